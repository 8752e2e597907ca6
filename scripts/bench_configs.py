"""Measure every BASELINE.json config on one GPU (build and lookup separately).

Not the driver's bench contract (bench.py is); this records the per-config
numbers and roofline fractions under profiles/.  Byte models per unit are
SURVEY.md §8(d): u64 build 56 B/key, u64 lookup 75.1 B/query, strings build
~156 B/key, strings lookup ~142 B/query.  Inputs are device-resident.
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2508_11443_b200 import hm  # noqa: E402
from workloads import gen_cuda  # noqa: E402

PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
B_BUILD_U64, B_LOOK_U64, B_BUILD_STR, B_LOOK_STR = 56.0, 75.11, 156.0, 142.0


def timed(fn, reps, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    hm.profile_read()
    hm.profile_enable(True)
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    hm.profile_enable(False)
    ks = {k: round(v[1] / v[0], 4) for k, v in hm.profile_read().items()}
    ts.sort()
    return ts[len(ts) // 2], ts[0], ks


def rate(units, ms):
    return units / (ms / 1e3) / 1e6


def u64_config(name, log2n, log2q, reps=5):
    n, nq = 1 << log2n, 1 << log2q
    k, v = gen_cuda.u64_keys(n)
    maps = []

    def build():
        m = hm.HashMap.build_u64(k, v)
        if maps:
            maps.pop().free()
        maps.append(m)

    bmed, bmin, bk = timed(build, reps)
    m = maps[0]
    chunk = min(nq, 1 << 28)
    q, _, _ = gen_cuda.u64_queries(n, chunk)
    ov = torch.empty(chunk, dtype=torch.int64, device="cuda")
    of = torch.empty(chunk, dtype=torch.uint8, device="cuda")
    reps_q = max(1, nq // chunk)

    def look():
        for _ in range(reps_q):
            m.lookup(q, ov, of)

    lmed, lmin, lk = timed(look, 5)
    m.free()
    out = {"config": name, "n": n, "nq": nq,
           "build_ms": round(bmed, 4), "build_mkeys_s": round(rate(n, bmed), 1),
           "build_roofline_frac": round(rate(n, bmed) * 1e6 * B_BUILD_U64 / 1e9 / PEAK, 4),
           "lookup_ms": round(lmed, 4), "lookup_mq_s": round(rate(nq, lmed), 1),
           "lookup_roofline_frac": round(rate(nq, lmed) * 1e6 * B_LOOK_U64 / 1e9 / PEAK, 4),
           "build_kernels_ms": bk, "lookup_kernels_ms": lk}
    del k, v, q, ov, of
    torch.cuda.empty_cache()
    return out


def str_config(name, log2n, reps=5):
    n = 1 << log2n
    ctx, offs = gen_cuda.string_keys(n)
    vals = torch.arange(n, dtype=torch.int64, device="cuda")
    maps = []

    def build():
        m = hm.HashMap.build_bytes(ctx, offs, vals)
        if maps:
            maps.pop().free()
        maps.append(m)

    bmed, bmin, bk = timed(build, reps)
    m = maps[0]
    qc, qo, _ = gen_cuda.string_queries(n, n)

    def look():
        m.lookup_bytes(qc, qo)

    lmed, lmin, lk = timed(look, 5)
    m.free()
    return {"config": name, "n": n, "nq": n, "ctx_bytes": int(ctx.numel()),
            "build_ms": round(bmed, 4), "build_mkeys_s": round(rate(n, bmed), 1),
            "build_roofline_frac": round(rate(n, bmed) * 1e6 * B_BUILD_STR / 1e9 / PEAK, 4),
            "lookup_ms": round(lmed, 4), "lookup_mq_s": round(rate(n, lmed), 1),
            "lookup_roofline_frac": round(rate(n, lmed) * 1e6 * B_LOOK_STR / 1e9 / PEAK, 4),
            "build_kernels_ms": bk, "lookup_kernels_ms": lk}


def paper_shape(reps=5):
    """NEXT-3: the paper's Table 1 shape: n = 10^7 keys, u64 keys and 5..25-byte
    strings, construction, lookup of every key (100 % hit) and membership of every key.  Values
    are u64 here (the paper's are i32).  Context only: the paper's numbers are A100."""
    n = 10_000_000
    out = []
    k, v = gen_cuda.u64_keys(n)
    maps = []

    def build():
        m = hm.HashMap.build_u64(k, v)
        if maps:
            maps.pop().free()
        maps.append(m)

    bmed, _, bk = timed(build, reps)
    m = maps[0]
    ov = torch.empty(n, dtype=torch.int64, device="cuda")
    of = torch.empty(n, dtype=torch.uint8, device="cuda")
    lmed, _, lk = timed(lambda: m.lookup(k, ov, of), reps)
    assert bool(torch.equal(ov, v)) and bool(of.all())
    mmed, _, mk = timed(lambda: m.contains(k), reps)
    m.free()
    out.append({"config": "P1 paper Table 1 shape, u64 keys, n = 10^7", "n": n,
                "construction_ms": round(bmed, 4), "lookup_all_ms": round(lmed, 4), "membership_all_ms": round(mmed, 4),
                "paper_a100_ms": {"construction": 18.3, "lookup": 3.3, "membership": 1.6},
                "build_kernels_ms": bk, "lookup_kernels_ms": lk, "membership_kernels_ms": mk})
    del k, v, ov, of
    ctx, offs = gen_cuda.string_keys(n, lens_range=(5, 25))
    vals = torch.arange(n, dtype=torch.int64, device="cuda")
    maps = []

    def build_s():
        m = hm.HashMap.build_bytes(ctx, offs, vals)
        if maps:
            maps.pop().free()
        maps.append(m)

    bmed, _, bk = timed(build_s, reps)
    m = maps[0]
    lmed, _, lk = timed(lambda: m.lookup_bytes(ctx, offs), reps)
    gv, gf = m.lookup_bytes(ctx, offs)
    assert bool(torch.equal(gv, vals)) and bool(gf.all())
    mmed, _, mk = timed(lambda: m.contains_bytes(ctx, offs), reps)
    m.free()
    out.append({"config": "P1 paper Table 1 shape, 5..25-byte strings, n = 10^7", "n": n, "ctx_bytes": int(ctx.numel()),
                "construction_ms": round(bmed, 4), "lookup_all_ms": round(lmed, 4), "membership_all_ms": round(mmed, 4),
                "paper_a100_ms": {"construction": 33.2, "lookup": 4.3, "membership": 2.8},
                "build_kernels_ms": bk, "lookup_kernels_ms": lk, "membership_kernels_ms": mk})
    torch.cuda.empty_cache()
    return out


def main():
    only = os.environ.get("ONLY", "C1,C2,C3,C4,C5,P1").split(",")
    todo = [
        ("C1", lambda: u64_config("C1 2^16 u64 + 2^16 lookups", 16, 16, reps=20)),
        ("C2", lambda: u64_config("C2 2^26 u64 + 2^26 lookups", 26, 26)),
        ("C3", lambda: str_config("C3 2^24 strings + 2^24 lookups", 24)),
        ("C4", lambda: u64_config("C4 2^29 u64 build (1 GPU)", 29, 26, reps=3)),
        ("C5", lambda: u64_config("C5 2^30 lookups on a 2^27 table (1 GPU)", 27, 30, reps=3)),
    ]
    res = [fn() for tag, fn in todo if tag in only]
    if "P1" in only:
        res += paper_shape()
    meta = {"gpu": torch.cuda.get_device_name(0), "peak_gbs": PEAK, "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())}
    for r in res:
        print(json.dumps(r))
    out = sys.argv[1] if len(sys.argv) > 1 else None
    if out:
        with open(out, "w") as f:
            json.dump({"meta": meta, "configs": res}, f, indent=1)


if __name__ == "__main__":
    main()
