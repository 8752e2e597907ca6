"""Aggregate ncu source-view samples / instructions over line ranges of build.cu."""
import csv, subprocess, sys
rep = sys.argv[1]; fsuffix = sys.argv[2]; ranges = sys.argv[3:]  # "a-b:name"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"] + (["-k", "regex:" + __import__("os").environ["KN"]] if __import__("os").environ.get("KN") else []), capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out)); hdr = None; fname = None; agg = {}; tot = [0, 0]
def num(x):
    try: return int(x)
    except: return 0
for r in rows:
    if r and r[0] == "File Path": fname = r[1]
    if r and r[0] == "Line No": hdr = r; continue
    if hdr and r and r[0] and r[0].isdigit():
        d = dict(zip(hdr[2:], r[2:])); ln = int(r[0])
        smp = num(d.get("Warp Stall Sampling (All Samples)", 0)); ins = num(d.get("Instructions Executed", 0))
        tot[0] += smp; tot[1] += ins
        name = "other:" + fname.split('/')[-1]
        if fname.endswith(fsuffix):
            for rg in ranges:
                ab, nm = rg.split(':'); a, b = map(int, ab.split('-'))
                if a <= ln < b: name = nm
        x = agg.setdefault(name, [0, 0]); x[0] += smp; x[1] += ins
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:24s} samples {100*v[0]/max(tot[0],1):5.1f}%  inst {100*v[1]/max(tot[1],1):5.1f}%  ({v[1]/1e6:.0f}M warp-inst)")
