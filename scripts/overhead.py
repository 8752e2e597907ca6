"""Fixed per-call cost of a build/lookup: wall clock vs CUDA events vs the kernels' own time (hm_profile)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2508_11443_b200 import hm
from workloads import gen_cuda
for lg in (10, 16, 20, 26):
    n = 1 << lg
    k, v = gen_cuda.u64_keys(n)
    q, _, _ = gen_cuda.u64_queries(n, n)
    for _ in range(5):
        hm.HashMap.build_u64(k, v).free()
    reps = 200 if lg < 24 else 20
    torch.cuda.synchronize()
    hm.profile_read(); hm.profile_enable(True)
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    t0 = time.perf_counter(); e0.record()
    for _ in range(reps):
        hm.HashMap.build_u64(k, v).free()
    e1.record(); torch.cuda.synchronize(); t1 = time.perf_counter()
    st = hm.profile_read(); hm.profile_enable(False)
    kern = sum(b[1] for b in st.values()) / reps
    m = hm.HashMap.build_u64(k, v)
    ov = torch.empty(n, dtype=torch.int64, device='cuda'); of = torch.empty(n, dtype=torch.uint8, device='cuda')
    for _ in range(5):
        m.lookup(q, ov, of)
    torch.cuda.synchronize()
    hm.profile_read(); hm.profile_enable(True)
    t2 = time.perf_counter(); e0.record()
    for _ in range(reps):
        m.lookup(q, ov, of)
    e1.record(); torch.cuda.synchronize(); t3 = time.perf_counter()
    stl = hm.profile_read(); hm.profile_enable(False)
    print(f"2^{lg}: build wall {1e3*(t1-t0)/reps:.4f} ms, kernels {kern:.4f} ms {dict((a, round(b[1]/reps, 4)) for a, b in st.items())}; "
          f"lookup wall {1e3*(t3-t2)/reps:.4f} ms, events {e0.elapsed_time(e1)/reps:.4f}, kernels {sum(b[1] for b in stl.values())/reps:.4f}", flush=True)
    m.free()
