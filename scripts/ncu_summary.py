"""Summarise the round's ncu evidence into profiles/.

  ncu_summary.py <launches.csv> <full.ncu-rep> <out.md> [--json profiles/ncu_summary.json]

launches.csv: `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
--clock-control none --csv` of a bench run (cold-cache, serialised launches: only the
kernels' shares of a step are comparable with bench.py, not the absolute times).
full.ncu-rep: `ncu --set full` of one launch of each hot kernel: DRAM traffic per
launch (the `traffic` field of bench.py's roofline), throughput, issue and stall data.
"""
import csv
import json
import re
import subprocess
import sys


def short(name):
    n = name.replace("void ", "").split("(")[0]
    base = n.split("<")[0].split("::")[-1]
    if base == "k_split":
        m = re.search(r"k_split<[^,]+,\s*[^,]+,\s*(\d)", n)
        return f"k_split{m.group(1)}" if m else base
    return base


def launch_list(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, mi, vi, idi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    d, order = {}, []
    for r in rows[hi + 1:]:
        key = (int(r[idi]), r[ki])
        if key not in d:
            order.append(key)
        d.setdefault(key, {})[r[mi]] = float(r[vi].replace(",", ""))
    agg = {}
    for k in order:
        m = d[k]
        a = agg.setdefault(short(k[1]), [0, 0.0, 0.0])
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0) / 1e3
        a[2] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
    return agg


FULL = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "lts__t_sector_hit_rate.pct", "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio"]


def full_capture(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    res = {}
    for r in rows[2:]:
        nm = short(r[h.index("Kernel Name")])
        if nm in res:
            continue
        m = {w: (r[h.index(w)] + (" " + units[h.index(w)] if units[h.index(w)] else "")) for w in FULL if w in h}
        b = 0.0
        for w in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = h.index(w)
            b += float(r[i].replace(",", "")) * scale.get(units[i], 1)
        m["dram_bytes"] = b
        res[nm] = m
    return res


def main():
    lst, rep, md = sys.argv[1], sys.argv[2], sys.argv[3]
    js = sys.argv[sys.argv.index("--json") + 1] if "--json" in sys.argv else None
    agg = launch_list(lst)
    full = full_capture(rep)
    tot = sum(a[1] for a in agg.values())
    lines = ["| kernel | launches | mean us/launch (ncu, cold) | share of the listed time | DRAM GB/launch |", "|---|---|---|---|---|"]
    for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| {k} | {a[0]} | {a[1]/a[0]:.1f} | {100*a[1]/tot:.1f}% | {a[2]/a[0]/1e9:.3f} |")
    lines += ["", "`ncu --set full`, one launch each:", ""]
    for k, m in full.items():
        lines.append(f"**{k}**")
        lines.append("")
        for w, v in m.items():
            lines.append(f"- `{w}` = {v}")
        lines.append("")
    open(md, "w").write("\n".join(lines) + "\n")
    if js:
        summ = {"source": {"launch_list": lst, "full": rep}, "kernels": {}}
        for k, a in agg.items():
            summ["kernels"].setdefault(k, {})["launch_list_dram_bytes_per_launch"] = a[2] / a[0]
            summ["kernels"][k]["ncu_us_per_launch"] = a[1] / a[0]
        for k, m in full.items():  # the `traffic` of bench.py: one --set full capture
            summ["kernels"].setdefault(k, {})["dram_bytes_per_launch"] = m["dram_bytes"]
            summ["kernels"][k]["full_metrics"] = m
        json.dump(summ, open(js, "w"), indent=1)
    print("\n".join(lines[:12]))


if __name__ == "__main__":
    main()
