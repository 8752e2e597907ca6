import csv, re, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
hdr = rows[hi]
ia, ie, iss = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
isrc = hdr.index("Source")
prof = []
for r in rows[hi + 1:]:
    if not r or not r[0].startswith("0x"): continue
    prof.append((int(r[ia], 16), int(r[ie] or 0), int(r[iss] or 0), r[isrc]))
base = prof[0][0]
chain, info = [], {}
for l in open(sys.argv[2]):
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        chain.append((m.group(1).split("/")[-1], int(m.group(2))))
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/\s+\S", l)
    if m and chain:
        outer = [c for c in chain if c[0]=="build.cu"]
        info[int(m.group(1), 16)] = (chain[0], outer[-1] if outer else None, chain[-1])
        chain = []
lo, hi_ = int(sys.argv[3]), int(sys.argv[4])
agg = {}
T = 0
last=None
for a, n, smp, src in prof:
    x = info.get(a - base, last); last = x
    T += n
    if x is None or x[1] is None or not (lo <= x[1][1] < hi_): continue
    key = "%s:%d" % x[0]
    v = agg.setdefault(key, [0, 0]); v[0] += n; v[1] += smp
for k, v in sorted(agg.items(), key=lambda x: -x[1][0])[:45]:
    print(f"{k:24s} inst {v[0]/1e6:8.1f}M  {v[0]/2**26:6.2f}/key samples {v[1]}")
