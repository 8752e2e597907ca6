"""One 2^24 byte-key build and two lookups (for an ncu capture of k_lookup_bytes)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2508_11443_b200 import hm
from workloads import gen_cuda
n = 1 << 24
ctx, offs = gen_cuda.string_keys(n)
vals = torch.arange(n, dtype=torch.int64, device="cuda")
m = hm.HashMap.build_bytes(ctx, offs, vals)
qc, qo, ids = gen_cuda.string_queries(n, n)
for _ in range(2):
    m.lookup_bytes(qc, qo)
torch.cuda.synchronize()
print("done")
