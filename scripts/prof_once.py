"""One warm build + one lookup at 2^N, for ncu launch lists / captures."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2508_11443_b200 import hm
from workloads import gen_cuda
log2n = int(sys.argv[1]) if len(sys.argv) > 1 else 26
kind = sys.argv[2] if len(sys.argv) > 2 else "u64"
n = 1 << log2n
if kind == "u64":
    k, v = gen_cuda.u64_keys(n)
    q, _, _ = gen_cuda.u64_queries(n, n)
    m = hm.HashMap.build_u64(k, v); m.free()
    m = hm.HashMap.build_u64(k, v)
    ov = torch.empty(n, dtype=torch.int64, device='cuda'); of = torch.empty(n, dtype=torch.uint8, device='cuda')
    m.lookup(q, ov, of); m.lookup(q, ov, of)
else:
    c, o = gen_cuda.string_keys(n)
    v = torch.arange(n, dtype=torch.int64, device='cuda')
    qc, qo, _ = gen_cuda.string_queries(n, n)
    m = hm.HashMap.build_bytes(c, o, v); m.free()
    m = hm.HashMap.build_bytes(c, o, v)
    m.lookup_bytes(qc, qo); m.lookup_bytes(qc, qo)
torch.cuda.synchronize()
print("done")
