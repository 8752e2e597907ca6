"""Per-source-line executed warp instructions and stall samples of one kernel in an ncu report.
usage: ncu_line_inst.py <report> <kernel regex> [top] [units]"""
import csv, subprocess, sys
rep, kn = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 50
units = float(sys.argv[4]) if len(sys.argv) > 4 else 1.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", "regex:" + kn,
                      "--launch-count", "1"], capture_output=True, text=True).stdout.splitlines()
hdr = None; fname = None; L = {}
for r in csv.reader(out):
    if r and r[0] == "File Path": fname = r[1].split('/')[-1]
    if r and r[0] == "Line No": hdr = r; continue
    if hdr and r and r[0].isdigit():
        d = dict(zip(hdr[2:], r[2:]))
        try: v = (int(d.get("Instructions Executed") or 0), int(d.get("Warp Stall Sampling (All Samples)") or 0))
        except ValueError: continue
        k = (fname, int(r[0])); o = L.get(k, (0, 0, r[1][:90])); L[k] = (o[0] + v[0], o[1] + v[1], o[2])
T = sum(x[0] for x in L.values()) or 1; S = sum(x[1] for x in L.values()) or 1
print(f"{T/1e6:.1f} M warp instructions ({T/units:.2f} per unit)")
for k, x in sorted(L.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100*x[0]/T:5.2f}% inst {x[0]/units:6.3f}/unit {100*x[1]/S:5.1f}% smp {k[0]}:{k[1]} {x[2]}")
