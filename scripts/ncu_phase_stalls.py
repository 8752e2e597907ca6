"""Per-phase stall-reason breakdown: SASS rows attributed to the source line printed before them."""
import csv, subprocess, sys
rep, fsuffix = sys.argv[1], sys.argv[2]
ranges = [(int(r.split(':')[0].split('-')[0]), int(r.split(':')[0].split('-')[1]), r.split(':')[1]) for r in sys.argv[3:]]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"] + (["-k", "regex:" + __import__("os").environ["KN"]] if __import__("os").environ.get("KN") else []), capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out)); hdr = None; fname = ""; cur = "other"; agg = {}
def num(x):
    try: return int(x)
    except: return 0
for r in rows:
    if r and r[0] == "File Path": fname = r[1]; continue
    if r and r[0] == "Line No": hdr = r; continue
    if not hdr or not r: continue
    if r[0]:  # source row
        cur = "other"
        if fname.endswith(fsuffix) and r[0].isdigit():
            ln = int(r[0])
            for a, b, nm in ranges:
                if a <= ln < b: cur = nm
        continue
    d = dict(zip(hdr, r))
    a = agg.setdefault(cur, {})
    for k, v in d.items():
        if k.startswith("stall_") and "Not Issued" not in k:
            a[k[6:]] = a.get(k[6:], 0) + num(v)
    a["_inst"] = a.get("_inst", 0) + num(d.get("Instructions Executed", 0))
T = sum(sum(v for k, v in a.items() if k != "_inst") for a in agg.values()) or 1
for nm, a in sorted(agg.items(), key=lambda x: -sum(v for k, v in x[1].items() if k != "_inst")):
    tot = sum(v for k, v in a.items() if k != "_inst")
    top = sorted(((k, v) for k, v in a.items() if k != "_inst"), key=lambda x: -x[1])[:5]
    print(f"{nm:16s} {100*tot/T:5.1f}% of samples, {a['_inst']/1e6:7.1f}M inst | " + ", ".join(f"{k} {100*v/max(tot,1):.0f}%" for k, v in top))
