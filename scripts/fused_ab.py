"""A/B of the u64 build routes at 2^26 (default two kernels vs FLAG_FUSED_PASS2):
whole-build CUDA-event time and per-kernel times (hm_profile)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2508_11443_b200 import hm
from workloads import gen_cuda
n = 1 << int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 26
k, v = gen_cuda.u64_keys(n)
for rep in range(2):
    for flags in (0, hm.FLAG_FUSED_PASS2):
        for _ in range(3):
            hm.HashMap.build_u64(k, v, flags=flags).free()
        hm.profile_read(); hm.profile_enable(True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ms = []
        for _ in range(10):
            e0.record(); m = hm.HashMap.build_u64(k, v, flags=flags); e1.record(); torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1)); m.free()
        st = hm.profile_read(); hm.profile_enable(False)
        ms.sort()
        print(f"n=2^{n.bit_length()-1} flags={flags} build median {ms[5]:.4f} ms min {ms[0]:.4f}",
              {a: round(b[1] / b[0], 4) for a, b in st.items()}, flush=True)
