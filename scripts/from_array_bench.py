"""from_array (HM_FLAG_FROM_ARRAY) at 2^26 inputs: all distinct, and 2x duplicated (2^25 distinct)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2508_11443_b200 import hm
from workloads import gen_cuda
n = 1 << 26
k, v = gen_cuda.u64_keys(n)
k2 = torch.cat([k[: n // 2], k[: n // 2]])
for name, keys in (("distinct", k), ("2x duplicated", k2)):
    for _ in range(2):
        hm.HashMap.build_u64(keys, v, flags=hm.FLAG_FROM_ARRAY).free()
    torch.cuda.synchronize()
    hm.profile_read(); hm.profile_enable(True)
    ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(); m = hm.HashMap.build_u64(keys, v, flags=hm.FLAG_FROM_ARRAY); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b)); nn = m.info().n; m.free()
    st = hm.profile_read(); hm.profile_enable(False)
    print(name, "n_distinct", nn, "ms", round(min(ts), 3), {a: round(b[1] / b[0], 3) for a, b in st.items()})
