"""Summarise an ncu --set full report per CUDA source line (samples, instructions)."""
import csv, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"] + (["-k", "regex:" + __import__("os").environ["KN"]] if __import__("os").environ.get("KN") else []),
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
hdr = None; lines = []; fname = None
for r in rows:
    if r and r[0] == "File Path": fname = r[1]
    if r and r[0] == "Line No": hdr = r; continue
    if hdr and r and r[0]:
        d = dict(zip(hdr[2:], r[2:]))
        try:
            lines.append((int(d.get("Warp Stall Sampling (All Samples)", 0) or 0), int(d.get("Instructions Executed", 0) or 0),
                          d.get("Avg. Threads Executed", ""), fname.split('/')[-1] if fname else "", r[0], r[1][:90]))
        except ValueError:
            pass
tot = sum(l[0] for l in lines) or 1
totI = sum(l[1] for l in lines) or 1
print(f"total samples {tot}, warp instructions {totI}")
for l in sorted(lines, reverse=True)[:top]:
    print(f"{100*l[0]/tot:5.1f}% smp {100*l[1]/totI:5.1f}% inst thr={l[2]:>4} {l[3]}:{l[4]:>4} {l[5]}")
