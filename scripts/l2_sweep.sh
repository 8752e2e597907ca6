for v in 32 48 64 72 80 96; do
  echo "== $v"; HM_L2_PERSIST=$v python - <<'PY' 2>&1 | grep -v Warning
import os, sys, torch
sys.path.insert(0, os.getcwd())
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
# the bench pattern: build then lookups
ts = []
for _ in range(3):
    m2 = hm.HashMap.build_u64(k, v); hm.profile_read()
    m2.lookup(q, ov, of); ts.append(hm.profile_read()["k_lookup_u64"][1]); m2.free()
print({a: round(b[1] / b[0], 4) for a, b in st.items()}, "after build:", [round(x, 3) for x in ts], bool(torch.equal(of, ef)))
PY
done
