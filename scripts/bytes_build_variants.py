"""Time the byte-key build (C3: 2^24 strings) with alternative library builds (HM_LIB_PATH)."""
import os, sys, subprocess
code = r'''
import os, sys, torch
sys.path.insert(0, os.environ["R"])
from paper_2508_11443_b200 import hm
from workloads import gen_cuda
n = 1 << 24
ctx, offs = gen_cuda.string_keys(n)
vals = torch.arange(n, dtype=torch.int64, device="cuda")
for _ in range(2): hm.HashMap.build_bytes(ctx, offs, vals).free()
hm.profile_read(); hm.profile_enable(True)
for _ in range(5): hm.HashMap.build_bytes(ctx, offs, vals).free()
st = hm.profile_read()
hm.profile_enable(False)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ms = []
for _ in range(5):
    torch.cuda.synchronize(); e0.record()
    m = hm.HashMap.build_bytes(ctx, offs, vals)
    e1.record(); torch.cuda.synchronize(); ms.append(e0.elapsed_time(e1)); m.free()
r = {a: round(b[1] / b[0], 4) for a, b in st.items()}
r["build_ms_min"] = round(min(ms), 4)
print(r)
'''
for lib in [None] + sys.argv[1:]:
    env = dict(os.environ, R=os.getcwd())
    if lib: env["HM_LIB_PATH"] = os.path.abspath(lib)
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    lines = out.stdout.strip().splitlines()
    print(os.path.basename(lib) if lib else "default", lines[-1] if lines else out.stderr[-300:])
