"""Quick device timing of build and lookup (development aid, not the bench contract)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2508_11443_b200 import hm
from workloads import gen_cuda

def main(log2n=26, reps=5):
    if os.environ.get("L2FG"):
        from cuda.bindings import runtime as cudart
        torch.cuda.init(); torch.zeros(1, device='cuda')
        print("set L2 fetch granularity", os.environ["L2FG"], cudart.cudaDeviceSetLimit(cudart.cudaLimit.cudaLimitMaxL2FetchGranularity, int(os.environ["L2FG"])),
              cudart.cudaDeviceGetLimit(cudart.cudaLimit.cudaLimitMaxL2FetchGranularity))
    n = 1 << log2n
    k, v = gen_cuda.u64_keys(n)
    q, ev, ef = gen_cuda.u64_queries(n, n, with_expect=True)
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    for i in range(2):
        m = hm.HashMap.build_u64(k, v); m.free()
    ts = []
    for i in range(reps):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); m = hm.HashMap.build_u64(k, v); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
        if i < reps - 1: m.free()
    inf = m.info()
    print(f"build n=2^{log2n}: ms min {min(ts):.3f} med {sorted(ts)[len(ts)//2]:.3f} -> {n/min(ts)/1e6:.1f} Gkeys/s  S/n={inf.S/n:.4f}")
    ov = torch.empty(n, dtype=torch.int64, device='cuda'); of = torch.empty(n, dtype=torch.uint8, device='cuda')
    for i in range(3): m.lookup(q, ov, of)
    ts = []
    for i in range(10):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); m.lookup(q, ov, of); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    ok = bool(torch.equal(of, ef)) and bool(torch.equal(ov, ev))
    print(f"lookup nq=2^{log2n}: ms min {min(ts):.3f} -> {n/min(ts)/1e6:.1f} Gq/s correct={ok}")

if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 26)
