"""Time k_lookup_u64 at 2^26 with alternative library builds (HM_LIB_PATH)."""
import os, sys, subprocess
code = r'''
import os, sys, torch
sys.path.insert(0, os.environ["R"])
from paper_2508_11443_b200 import hm
from workloads import gen_cuda
n = 1 << 26
k, v = gen_cuda.u64_keys(n)
q, ev, ef = gen_cuda.u64_queries(n, n, with_expect=True)
m = hm.HashMap.build_u64(k, v)
ov = torch.empty(n, dtype=torch.int64, device="cuda"); of = torch.empty(n, dtype=torch.uint8, device="cuda")
for _ in range(3): m.lookup(q, ov, of)
hm.profile_read(); hm.profile_enable(True)
for _ in range(10): m.lookup(q, ov, of)
st = hm.profile_read()
print({a: round(b[1] / b[0], 4) for a, b in st.items()}, bool(torch.equal(of, ef)) and bool(torch.equal(ov, ev)))
'''
for lib in [None] + sys.argv[1:]:
    env = dict(os.environ, R=os.getcwd())
    if lib: env["HM_LIB_PATH"] = os.path.abspath(lib)
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    lines = out.stdout.strip().splitlines()
    print(os.path.basename(lib) if lib else "default", lines[-1] if lines else out.stderr[-300:])
