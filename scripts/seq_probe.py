"""Build times of a sequence of (log2 n : flags) builds in one process, with the
per-kernel device times: shows host-side costs (pool mapping) that the kernel
times do not.  Usage: seq_probe.py 24:0,26:0,26:16"""
import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
from paper_2508_11443_b200 import hm
from workloads import gen_cuda
def run(lg, flags, reps=3, prof=False):
    n = 1 << lg
    k, v = gen_cuda.u64_keys(n)
    for r in range(reps):
        if prof: hm.profile_read(); hm.profile_enable(True)
        torch.cuda.synchronize(); t = time.perf_counter(); sys.stderr.write('[py] start %.3f\n' % (time.monotonic()*1e3)); sys.stderr.flush()
        m = hm.HashMap.build_u64(k, v, flags=flags)
        torch.cuda.synchronize(); dt = (time.perf_counter() - t) * 1e3
        st = hm.profile_read() if prof else {}
        hm.profile_enable(False)
        m.free()
        print(lg, flags, r, round(dt, 2), {a: round(b[1], 2) for a, b in st.items()}, flush=True)
seq = sys.argv[1].split(",")
for s in seq:
    lg, fl = s.split(":")
    run(int(lg), int(fl), prof=True)
