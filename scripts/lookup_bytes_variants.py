"""Time k_lookup_bytes (C3: 2^24 strings, 2^24 lookups at 50 % hit) with
alternative library builds (HM_LIB_PATH); outputs checked against the
queries' ids (hit iff id < n, value = id)."""
import os, sys, subprocess
code = r'''
import os, sys, torch
sys.path.insert(0, os.environ["R"])
from paper_2508_11443_b200 import hm
from workloads import gen_cuda
n = 1 << 24
ctx, offs = gen_cuda.string_keys(n)
vals = torch.arange(n, dtype=torch.int64, device="cuda")
m = hm.HashMap.build_bytes(ctx, offs, vals)
qc, qo, ids = gen_cuda.string_queries(n, n)
ov = torch.empty(n, dtype=torch.int64, device="cuda"); of = torch.empty(n, dtype=torch.uint8, device="cuda")
for _ in range(3): m.lookup_bytes(qc, qo, ov, of)
hm.profile_read(); hm.profile_enable(True)
for _ in range(10): m.lookup_bytes(qc, qo, ov, of)
st = hm.profile_read()
hit = ids < n
ok = bool(torch.equal(of.bool(), hit)) and bool(torch.equal(ov[hit], ids[hit])) and bool((ov[~hit] == 0).all())
print({a: round(b[1] / b[0], 4) for a, b in st.items()}, ok)
'''
for lib in [None] + sys.argv[1:]:
    env = dict(os.environ, R=os.getcwd())
    if lib: env["HM_LIB_PATH"] = os.path.abspath(lib)
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    lines = out.stdout.strip().splitlines()
    print(os.path.basename(lib) if lib else "default", lines[-1] if lines else out.stderr[-300:])
