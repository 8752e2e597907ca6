"""Print an ncu --csv launch list (per launch: duration, DRAM bytes)."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]
ki, mi, vi, idi = h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value'), h.index('ID')
d = {}
order = []
for r in rows[hi + 1:]:
    key = (int(r[idi]), r[ki])
    if key not in d: order.append(key)
    d.setdefault(key, {})[r[mi]] = float(r[vi].replace(',', ''))
tot = sum(d[k].get('gpu__time_duration.sum', 0) for k in order)
for k in order:
    m = d[k]; t = m.get('gpu__time_duration.sum', 0)
    rd, wr = m.get('dram__bytes_read.sum', 0), m.get('dram__bytes_write.sum', 0)
    name = k[1].split('(')[0].replace('void ', '')[:48]
    print(f"{k[0]:3d} {name:48s} {t/1e3:9.1f} us {100*t/tot:5.1f}%  rd {rd/1e9:7.3f} GB wr {wr/1e9:7.3f} GB  {(rd+wr)/max(t,1):7.1f} GB/s")
