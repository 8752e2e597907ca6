"""u64 lookup kernel time at 2^26 queries on a 2^26 table and 2^28 on 2^27 (per library build, HM_LIB_PATH)."""
import os, sys, subprocess
code = r'''
import os, sys, torch
sys.path.insert(0, os.environ["R"])
from paper_2508_11443_b200 import hm
from workloads import gen_cuda
out = []
for lt, lq in ((26, 26), (27, 28)):
    k, v = gen_cuda.u64_keys(1 << lt)
    q, _, _ = gen_cuda.u64_queries(1 << lt, 1 << lq)
    m = hm.HashMap.build_u64(k, v)
    ov = torch.empty(1 << lq, dtype=torch.int64, device="cuda"); of = torch.empty(1 << lq, dtype=torch.uint8, device="cuda")
    for _ in range(3): m.lookup(q, ov, of)
    torch.cuda.synchronize(); hm.profile_read(); hm.profile_enable(True)
    for _ in range(5): m.lookup(q, ov, of)
    torch.cuda.synchronize(); st = hm.profile_read(); hm.profile_enable(False)
    m.free()
    # as in the bench step: each lookup right after a build (the compact directory fresh in L2)
    for _ in range(2):
        m = hm.HashMap.build_u64(k, v); m.lookup(q, ov, of); m.free()
    torch.cuda.synchronize(); hm.profile_read(); hm.profile_enable(True)
    for _ in range(5):
        m = hm.HashMap.build_u64(k, v); m.lookup(q, ov, of); m.free()
    torch.cuda.synchronize(); st2 = hm.profile_read(); hm.profile_enable(False)
    out.append(f"2^{lq} on 2^{lt}: repeated {st['k_lookup_u64'][1] / st['k_lookup_u64'][0]:.4f} ms, after build "
               f"{st2['k_lookup_u64'][1] / st2['k_lookup_u64'][0]:.4f} ms")
    del k, v, q, ov, of; torch.cuda.empty_cache()
print(" | ".join(out))
'''
libs = sys.argv[1:]
for lib in [None] + libs:
    env = dict(os.environ, R=os.getcwd())
    if lib: env["HM_LIB_PATH"] = os.path.abspath(lib)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    lines = r.stdout.strip().splitlines()
    print(os.path.basename(lib) if lib else "default", lines[-1] if lines else r.stderr[-300:], flush=True)
