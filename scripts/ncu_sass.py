"""Top SASS instructions of an ncu report by stall samples, with the dominant stall reasons."""
import csv, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out)); h = rows[1]
reasons = [x for x in h if x.startswith('stall_') and 'Not Issued' not in x]
tot = {}
recs = []
for r in rows[2:]:
    d = dict(zip(h, r))
    try: smp = int(d['Warp Stall Sampling (All Samples)'] or 0)
    except: continue
    rs = {k: int(d[k] or 0) for k in reasons}
    for k, v in rs.items(): tot[k] = tot.get(k, 0) + v
    recs.append((smp, d['Address'][-5:], d['Source'][:60], sorted(rs.items(), key=lambda x: -x[1])[:3]))
T = sum(x[0] for x in recs) or 1
print("overall:", ", ".join(f"{k[6:]} {100*v/T:.1f}%" for k, v in sorted(tot.items(), key=lambda x: -x[1])[:8]))
for smp, a, s, rs in sorted(recs, reverse=True)[:top]:
    print(f"{100*smp/T:5.1f}% {a} {s:60s} " + " ".join(f"{k[6:]}={v}" for k, v in rs if v))
