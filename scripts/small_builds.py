"""Build time (CUDA events, median of 20) of u64 tables of 2^10 .. 2^24 keys, per library (HM_LIB_PATH)."""
import os, sys, subprocess
code = r'''
import os, sys, torch
sys.path.insert(0, os.environ["R"])
from paper_2508_11443_b200 import hm
from workloads import gen_cuda
out = []
for lg in (12, 14, 16, 18, 20, 22, 24):
    k, v = gen_cuda.u64_keys(1 << lg)
    for _ in range(3): hm.HashMap.build_u64(k, v).free()
    ts = []
    for _ in range(20):
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(); m = hm.HashMap.build_u64(k, v); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b)); m.free()
    ts.sort(); out.append(f"2^{lg} {ts[10]:.4f}")
print(" | ".join(out))
'''
for lib in [None] + sys.argv[1:]:
    env = dict(os.environ, R=os.getcwd())
    if lib: env["HM_LIB_PATH"] = os.path.abspath(lib)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    print(os.path.basename(lib) if lib else "default", (r.stdout.strip().splitlines() or [r.stderr[-300:]])[-1], flush=True)
