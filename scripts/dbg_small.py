import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2508_11443_b200 import hm
from workloads import gen
n = int(sys.argv[1]); seed = int(sys.argv[2]) if len(sys.argv) > 2 else 0
k = torch.from_numpy(gen.u64_keys(n).view(np.int64)).cuda(); v = torch.from_numpy(gen.u64_values(n).view(np.int64)).cuda()
t0 = time.time(); m = hm.HashMap.build_u64(k, v, seed=seed); print("built", n, seed, m.info(), time.time() - t0, flush=True)
q = torch.from_numpy(gen.u64_queries(n, 1000)[0].view(np.int64)).cuda()
m.lookup(q); torch.cuda.synchronize(); print("lookup ok", flush=True)
