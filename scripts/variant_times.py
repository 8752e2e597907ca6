"""Time builds/lookups with alternative library builds (HM_LIB_PATH) at 2^26."""
import os, sys, subprocess, glob
code = r'''
import os, sys, torch
sys.path.insert(0, os.environ["R"])
from paper_2508_11443_b200 import hm
from workloads import gen_cuda
n = 1 << 26
k, v = gen_cuda.u64_keys(n)
for _ in range(2):
    hm.HashMap.build_u64(k, v).free()
hm.profile_read(); hm.profile_enable(True)
for _ in range(3):
    hm.HashMap.build_u64(k, v).free()
st = hm.profile_read()
print({a: round(b[1] / b[0], 3) for a, b in st.items()})
'''
libs = sys.argv[1:] or sorted(glob.glob("paper_2508_11443_b200/libhm_*.so"))
for lib in [None] + libs:
    env = dict(os.environ, R=os.getcwd())
    if lib: env["HM_LIB_PATH"] = os.path.abspath(lib)
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    lines = out.stdout.strip().splitlines()
    print(os.path.basename(lib) if lib else "default", lines[-1] if lines else out.stderr[-300:])
