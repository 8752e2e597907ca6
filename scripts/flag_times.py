"""k_bucket time at 2^26 with build flags (testing knobs) vs none."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2508_11443_b200 import hm
from workloads import gen_cuda
n = 1 << 26
k, v = gen_cuda.u64_keys(n)
for flags in [0] + [int(x) for x in sys.argv[1:]]:
    for _ in range(2):
        hm.HashMap.build_u64(k, v, flags=flags).free()
    hm.profile_read(); hm.profile_enable(True)
    for _ in range(5):
        hm.HashMap.build_u64(k, v, flags=flags).free()
    st = hm.profile_read(); hm.profile_enable(False)
    print("flags", flags, {a: round(b[1] / b[0], 4) for a, b in st.items()})
