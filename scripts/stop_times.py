"""Marginal phase costs of k_bucket: whole-kernel time of builds cut after phase k."""
import os, sys, subprocess
code = r'''
import os, sys, torch
sys.path.insert(0, os.environ["R"])
from paper_2508_11443_b200 import hm
from workloads import gen_cuda
n = 1 << 26
k, v = gen_cuda.u64_keys(n)
for _ in range(2):
    try: hm.HashMap.build_u64(k, v).free()
    except Exception as e: pass
hm.profile_read(); hm.profile_enable(True)
for _ in range(3):
    try: hm.HashMap.build_u64(k, v).free()
    except Exception as e: pass
st = hm.profile_read()
print({a: round(b[1] / b[0], 3) for a, b in st.items()})
'''
for k in [int(x) for x in os.environ.get("MARKS", "1,2,3,4,5,6,7").split(",")] + [None]:
    env = dict(os.environ, R=os.getcwd())
    if k: env["HM_LIB_PATH"] = os.path.join(os.getcwd(), "paper_2508_11443_b200", f"libhm_stop{k}.so")
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    lines = out.stdout.strip().splitlines()
    print("stop after mark", k, lines[-1] if lines else out.stderr[-300:])
