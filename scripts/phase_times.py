"""Per-phase durations of k_bucket from the debug build (HM_LIB_PATH=.../libhm_timing.so)."""
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
buf = np.zeros(65536 * 12 + 8192, np.uint64)
L.hm_debug_phase_times(buf.ctypes.data_as(C.c_void_p), 65536 * 12)
ka = buf[65536*12:].reshape(4096, 2).astype(np.int64); ka = ka[ka[:,0] > 0]
print('k_partition CTA span us', (ka[:,1].max()-ka[:,0].min())/1e3, 'ctas', len(ka))
KA_END = ka[:,1].max(); KA_START = ka[:,0].min()
np_ = n >> (int(sys.argv[2]) if len(sys.argv) > 2 else 12)
t = buf[: np_ * 12].reshape(np_, 12).astype(np.int64)
names = ["start", "P1", "P2", "P3", "P4ab", "P4c", "search", "lookback", "dir/cdir/single", "multiwrite", "end"]
d = np.diff(t[:, :11], axis=1)
print("partitions", np_, "kernel span us", (t[:, 10].max() - t[:, 0].min()) / 1e3, "gap K_A end -> first K_B CTA us", (t[:, 0].min() - KA_END) / 1e3, "K_A start -> K_B end us", (t[:,10].max()-KA_START)/1e3)
print("CTA lifetime us: mean %.1f median %.1f max %.1f" % (np.mean(t[:, 10] - t[:, 0]) / 1e3, np.median(t[:, 10] - t[:, 0]) / 1e3, np.max(t[:, 10] - t[:, 0]) / 1e3))
for i in range(10):
    print(f"{names[i]:>16s} -> {names[i+1]:<16s} mean {d[:, i].mean()/1e3:8.2f} us  p50 {np.median(d[:, i])/1e3:8.2f}  max {d[:, i].max()/1e3:8.2f}")
