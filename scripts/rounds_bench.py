"""NEXT-4 ablation: build time of the default construction (partition +
warp-per-bucket search in shared memory) vs the paper's sortless round-based
construction (HM_FLAG_ROUNDS), u64 keys, inputs resident in HBM.
Prints one JSON line per size with both times, the per-kernel breakdown of the
rounds build and its round count."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2508_11443_b200 import hm
from workloads import gen_cuda


def timed(k, v, flags, reps):
    for _ in range(2):
        hm.HashMap.build_u64(k, v, flags=flags).free()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        m = hm.HashMap.build_u64(k, v, flags=flags)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
        m.free()
    ts.sort()
    return ts[len(ts) // 2]


for lg in [int(x) for x in (sys.argv[1:] or ["20", "24", "26"])]:
    n = 1 << lg
    k, v = gen_cuda.u64_keys(n)
    t_def = timed(k, v, 0, 5)
    t_rnd = timed(k, v, hm.FLAG_ROUNDS, 5)
    hm.profile_read(); hm.profile_enable(True)
    hm.HashMap.build_u64(k, v, flags=hm.FLAG_ROUNDS).free()
    st = hm.profile_read(); hm.profile_enable(False)
    rounds = st.get("k_r_seg_hash", (0, 0))[0]
    br = {a: round(b[1], 3) for a, b in sorted(st.items(), key=lambda x: -x[1][1])}
    print(json.dumps({"n": n, "default_ms": round(t_def, 3), "rounds_ms": round(t_rnd, 3),
                      "ratio": round(t_rnd / t_def, 2), "rounds": rounds,
                      "default_Gkeys_s": round(n / t_def / 1e6, 3), "rounds_Gkeys_s": round(n / t_rnd / 1e6, 3),
                      "rounds_kernel_ms": br}), flush=True)
    del k, v
