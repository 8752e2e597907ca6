"""CUPTI trace (torch.profiler) of one warm build + lookup: every kernel,
memcpy, memset and sync on the device timeline with host-side gaps.

usage: python scripts/trace_build.py LOG2N {u64|str} [out.json]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2508_11443_b200 import hm  # noqa: E402
from workloads import gen_cuda  # noqa: E402

log2n = int(sys.argv[1]) if len(sys.argv) > 1 else 24
kind = sys.argv[2] if len(sys.argv) > 2 else "str"
n = 1 << log2n
if kind == "u64":
    k, v = gen_cuda.u64_keys(n)
    q, _, _ = gen_cuda.u64_queries(n, n)

    def build():
        return hm.HashMap.build_u64(k, v)

    def look(m):
        m.lookup(q)
else:
    c, o = gen_cuda.string_keys(n)
    v = torch.arange(n, dtype=torch.int64, device="cuda")
    qc, qo, _ = gen_cuda.string_queries(n, n)

    def build():
        return hm.HashMap.build_bytes(c, o, v)

    def look(m):
        m.lookup_bytes(qc, qo)

m = build()
look(m)
m2 = build()
m.free()
m = m2
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    m2 = build()
    m.free()
    b.record()
    torch.cuda.synchronize()
    look(m2)
    torch.cuda.synchronize()
print("build event ms", a.elapsed_time(b))
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start if ev else 0
prev_end = t0
for e in ev:
    s, d = e.time_range.start, e.time_range.end - e.time_range.start
    print(f"{(s - t0) / 1e3:9.3f} ms  gap {(s - prev_end) / 1e3:7.3f}  dur {d / 1e3:7.3f}  {e.name[:70]}")
    prev_end = e.time_range.end
cpu = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CPU]
tot = {}
for e in cpu:
    tot[e.name] = tot.get(e.name, 0) + (e.time_range.end - e.time_range.start)
for k_, v_ in sorted(tot.items(), key=lambda x: -x[1])[:15]:
    print(f"cpu {v_ / 1e3:8.3f} ms {k_[:80]}")
if len(sys.argv) > 3:
    prof.export_chrome_trace(sys.argv[3])
