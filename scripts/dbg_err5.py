import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2508_11443_b200 import hm
def dev(a): return torch.from_numpy(a.view(np.int64)).cuda()
for it in range(20):
    try:
        hm.HashMap.build_u64(dev(np.full(5, 9, np.uint64)), dev(np.arange(5, dtype=np.uint64)))
    except hm.HMError as e:
        if e.name != "SEED_EXHAUSTED": print("iter", it, e.name, e); break
    try:
        hm.HashMap.build_u64(dev(np.array([7, 7], np.uint64)), dev(np.array([1, 2], np.uint64)))
    except hm.HMError as e:
        if e.name != "DUPLICATE_KEY": print("iter", it, e.name, e); break
print("done")
