"""C5 lookups (2^30 queries on a 2^27-key table) and C2 lookups with alternative library builds (HM_LIB_PATH)."""
import os, sys, subprocess
code = r'''
import os, sys, torch
sys.path.insert(0, os.environ["R"])
from paper_2508_11443_b200 import hm
from workloads import gen_cuda
out = {}
for lg, lq in ((26, 26), (27, 28)):
    n = 1 << lg
    k, v = gen_cuda.u64_keys(n)
    m = hm.HashMap.build_u64(k, v)
    q, ev, ef = gen_cuda.u64_queries(n, 1 << lq, with_expect=True)
    ov = torch.empty_like(q); of = torch.empty(q.numel(), dtype=torch.uint8, device="cuda")
    for _ in range(2): m.lookup(q, ov, of)
    hm.profile_read(); hm.profile_enable(True)
    for _ in range(5): m.lookup(q, ov, of)
    st = hm.profile_read(); hm.profile_enable(False)
    ok = bool(torch.equal(ov, ev)) and bool(torch.equal(of, ef))
    out[f"2^{lq} on 2^{lg}"] = (round(st["k_lookup_u64"][1] / st["k_lookup_u64"][0], 4), ok)
    m.free(); del k, v, q, ev, ef, ov, of; torch.cuda.empty_cache()
print(out)
'''
for lib in [None] + sys.argv[1:]:
    env = dict(os.environ, R=os.getcwd())
    if lib: env["HM_LIB_PATH"] = os.path.abspath(lib)
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    lines = out.stdout.strip().splitlines()
    print(os.path.basename(lib) if lib else "default", lines[-1] if lines else out.stderr[-300:])
