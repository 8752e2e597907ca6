"""Time the routing kernels (k_route_count/k_route_scatter) at 2^26 keys for world = 2, 8."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2508_11443_b200 import hm, dist
from workloads import gen_cuda
n = 1 << 26
k, v = gen_cuda.u64_keys(n)
ops = dist.GpuOps()
for world in (2, 8):
    for _ in range(2):
        ops.route(k, v, n * world, 0, 0, world)
    torch.cuda.synchronize()
    hm.profile_read(); hm.profile_enable(True)
    for _ in range(5):
        ops.route(k, v, n * world, 0, 0, world)
    torch.cuda.synchronize()
    st = hm.profile_read(); hm.profile_enable(False)
    print(world, {a: round(b[1] / b[0], 4) for a, b in st.items()})
