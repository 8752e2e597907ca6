"""Attribute an ncu SASS-level profile (per-address instruction counts and
stall samples) to kernel-body source lines through nvdisasm's inline chains.
usage: ncu_attr.py <ncu sass csv> <nvdisasm -g -gi listing of the same kernel> [ranges a-b:name ...]"""
import csv, re, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
hdr = rows[hi]
ia, ie, iss = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
prof = []
for r in rows[hi + 1:]:
    if not r or not r[0].startswith("0x"): continue
    prof.append((int(r[ia], 16), int(r[ie] or 0), int(r[iss] or 0)))
base = prof[0][0]
chain, outer = [], {}
for l in open(sys.argv[2]):
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        chain.append((m.group(1).split("/")[-1], int(m.group(2))))
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/\s+\S", l)
    if m and chain:
        outer[int(m.group(1), 16)] = chain[-1][1] if chain[-1][0] == "build.cu" else -1
        chain = []
ranges = [(int(x.split(":")[0].split("-")[0]), int(x.split(":")[0].split("-")[1]), x.split(":")[1]) for x in sys.argv[3:]]
agg, last = {}, -1
T = [0, 0]
for a, n, smp in prof:
    ln = outer.get(a - base, last)
    last = ln
    nm = next((r[2] for r in ranges if r[0] <= ln < r[1]), f"line{ln}")
    x = agg.setdefault(nm, [0, 0]); x[0] += n; x[1] += smp; T[0] += n; T[1] += smp
for k, v in sorted(agg.items(), key=lambda x: -x[1][0])[:40]:
    print(f"{k:20s} inst {v[0]/1e6:8.1f}M ({100*v[0]/T[0]:5.1f}%)  samples {100*v[1]/max(T[1],1):5.1f}%")
print("total", T[0] / 1e6)
