"""Per-phase durations of k_bucket from the debug build (HM_LIB_PATH=.../libhm_timing.so):
globaltimer stamps at the HM_TMARK points of every CTA."""
import os, sys, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("HM_LIB_PATH", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2508_11443_b200", "libhm_timing.so"))
import numpy as np, torch
from paper_2508_11443_b200 import hm
from workloads import gen_cuda
lg = int(sys.argv[1]) if len(sys.argv) > 1 else 26
n = 1 << lg
k, v = gen_cuda.u64_keys(n)
for _ in range(2):
    m = hm.HashMap.build_u64(k, v); m.free()
hm.profile_read(); hm.profile_enable(True)
m = hm.HashMap.build_u64(k, v); torch.cuda.synchronize()
print('event ms per kernel', hm.profile_read()); hm.profile_enable(False)
L = hm.lib(); L.hm_debug_phase_times.argtypes = [C.c_void_p, C.c_uint64]
buf = np.zeros(65536 * 16 + 8192, np.uint64)
L.hm_debug_phase_times(buf.ctypes.data_as(C.c_void_p), 65536 * 16)
names = ["start", "load", "hist", "scan+group", "search", "lookback", "out", "dir"]
t = buf[: 65536 * 16].reshape(65536, 16).astype(np.int64)
t = t[t[:, 0] > 0][:, :len(names)]
d = np.diff(t, axis=1)
life = t[:, -1] - t[:, 0]
print("partitions", len(t), "kernel span us %.1f" % ((t[:, -1].max() - t[:, 0].min()) / 1e3))
print("CTA lifetime us: mean %.2f median %.2f max %.2f" % (life.mean() / 1e3, np.median(life) / 1e3, life.max() / 1e3))
for i in range(len(names) - 1):
    print(f"{names[i]:>12s} -> {names[i+1]:<12s} mean {d[:, i].mean()/1e3:7.2f} us  p50 {np.median(d[:, i])/1e3:7.2f}  p99 {np.percentile(d[:, i], 99)/1e3:7.2f}  share {100*d[:, i].mean()/life.mean():5.1f}%")
t2 = buf[: 65536 * 16].reshape(65536, 16).astype(np.int64)
t2 = t2[t2[:, 0] > 0]
if (t2[:, 8] > 0).all():
    for a, b, nm in [(2, 10, "scan"), (10, 3, "groupby"), (3, 9, "lookback (w0)"), (3, 8, "swarp+round0"), (8, 11, "retry round 1"), (8, 4, "retry rounds")]:
        ok = (t2[:, b] > 0) & (t2[:, a] > 0)
        x = (t2[:, b] - t2[:, a])[ok]
        print(f"  search part {nm:18s} mean {x.mean()/1e3:7.2f} us  p50 {np.median(x)/1e3:7.2f}")
    nr = t2[:, 12]
    print("  retry rounds per CTA: mean %.2f, dist %s" % (nr.mean(), np.bincount(nr.astype(int))[:8]))
