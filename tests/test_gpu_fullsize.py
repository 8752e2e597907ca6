"""GPU parity at BASELINE.json's full sizes, in the launch configuration
bench.py times (default build options, device-resident inputs).

configs[1] (2^26 u64) and configs[2] (2^24 strings): every byte of the exported
table against the oracle, every lookup against the generator's ground truth.
configs[3]/[4] sizes (2^29 keys; 2^27-key table with 2^30 queries) on one GPU:
properties that hold at any size (S <= 4n, the directory is the exclusive scan
of s^2 and sums to n, every member found with its value, every absent key
misses, every query against the generator's ground truth) and every byte of
the table against the oracle, range by range through the oracle's shard
definition (bounded host memory).
"""
import numpy as np
import pytest

from oracle import oracle as O
from workloads import gen

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.slow]

MASK40 = np.uint64((1 << 40) - 1)


def _hm():
    from paper_2508_11443_b200 import hm
    return hm


def _dev_gen():
    from workloads import gen_cuda
    return gen_cuda


def _u(t):
    return t.cpu().numpy().view(np.uint64)


def _check_dir_properties(d, n, S):
    soff = d & MASK40
    s = (d >> np.uint64(40)) & np.uint64(0xFFFF)
    sq = s * s
    assert S <= 4 * n
    assert int(s.sum(dtype=np.uint64)) == n
    assert soff[0] == 0 and np.array_equal(soff[1:], soff[:-1] + sq[:-1])
    assert int(soff[-1] + sq[-1]) == S


def _check_full_by_shards(d, slots, keys, vals, n, seed, t1, S, nshards=64):
    """Every byte of the table against the oracle with bounded host memory:
    the single table is the concatenation, in bucket order, of the oracle's
    bucket-range shards (or_build_u64_shard — that identity is pinned on CPU
    by tests/test_dist_gloo.py and tests/test_oracle_fks.py), so range r of
    the exported directory (soff rebased to the range) and of the slots must
    equal the oracle's shard of the keys whose level-1 bucket falls in it.
    The shards are built in parallel host threads (ctypes releases the GIL)."""
    import os
    from concurrent.futures import ThreadPoolExecutor
    g = O.level1_buckets(keys, n, seed, t1)
    rid = (g * np.uint64(nshards) // np.uint64(n)).astype(np.uint8)  # floor(b K / n): range of bucket b
    del g
    order = np.argsort(rid, kind="stable")
    starts = np.concatenate([[0], np.cumsum(np.bincount(rid, minlength=nshards))])
    del rid
    soff = d & MASK40

    def one(r):
        lo, hi = -(-r * n // nshards), -(-(r + 1) * n // nshards)
        idx = order[starts[r]:starts[r + 1]]
        st, sh = O.build_u64_shard(keys[idx], vals[idx], n, lo, hi, t1, seed)
        assert st == "OK", st
        gd = d[lo:hi]
        base = int(soff[lo])
        rel = (gd & ~MASK40) | ((gd & MASK40) - np.uint64(base))
        ok_dir = np.array_equal(rel, sh.dir)
        ok_slots = slots[base:base + sh.S].tobytes() == sh.slots.tobytes()
        return r, ok_dir, ok_slots, sh.S

    with ThreadPoolExecutor(min(16, os.cpu_count() or 1)) as ex:
        res = list(ex.map(one, range(nshards)))
    bad = [(r, od, os_) for r, od, os_, _ in res if not (od and os_)]
    assert not bad, f"bucket ranges differing from the oracle (range, dir ok, slots ok): {bad[:5]}"
    assert sum(x[3] for x in res) == S


def test_config2_u64_2e26_full_table():
    hm, gc = _hm(), _dev_gen()
    n = 1 << 26
    k, v = gc.u64_keys(n)
    m = hm.HashMap.build_u64(k, v)
    d, slots, _ = m.export()
    inf = m.info()
    q, ev, ef = gc.u64_queries(n, n, with_expect=True)
    gv, gf = m.lookup(q)
    torch.cuda.synchronize()
    assert torch.equal(gf, ef) and torch.equal(gv, ev)
    keys, vals = _u(k), _u(v)
    del k, v
    m.free()
    _check_dir_properties(d, n, inf.S)
    ot = O.build_u64(keys, vals, 0)
    assert inf.S == ot.S and inf.t1 == int(ot.header["t1"])
    assert d.tobytes() == ot.dir.tobytes()
    assert slots.tobytes() == ot.slots.tobytes()
    # oracle lookups on a sample of the same queries
    qs = _u(q)[:: 64]
    ov, of = O.lookup_u64(ot, qs)
    assert np.array_equal(_u(gv)[::64], ov) and np.array_equal(gf.cpu().numpy()[::64], of)


def test_config3_strings_2e24_full_table():
    hm, gc = _hm(), _dev_gen()
    n = 1 << 24
    ctx, offs = gc.string_keys(n)
    vals = torch.arange(n, dtype=torch.int64, device="cuda")
    m = hm.HashMap.build_bytes(ctx, offs, vals)
    d, slots, mctx = m.export()
    inf = m.info()
    qc, qo, ids = gc.string_queries(n, n)
    gv, gf = m.lookup_bytes(qc, qo)
    member = ids < n
    assert torch.equal(gf.bool(), member)
    assert torch.equal(gv, torch.where(member, ids, torch.zeros_like(ids)))
    m.free()
    hctx, hoffs, hvals = ctx.cpu().numpy(), _u(offs), _u(vals)
    ot = O.build_bytes(hctx, hoffs, hvals, 0)
    assert inf.S == ot.S and inf.t1 == int(ot.header["t1"]) and inf.t0 == int(ot.header["t0"])
    assert d.tobytes() == ot.dir.tobytes()
    assert slots.tobytes() == ot.slots.tobytes()
    assert mctx.tobytes() == ot.ctx.tobytes()


def test_config4_u64_2e29_sampled():
    hm, gc = _hm(), _dev_gen()
    n = 1 << 29
    k, v = gc.u64_keys(n)
    m = hm.HashMap.build_u64(k, v)
    inf = m.info()
    # every member found with its value, every absent key misses (on device, in chunks)
    chunk = 1 << 27
    for lo in range(0, n, chunk):
        gv, gf = m.lookup(k[lo:lo + chunk])
        assert bool(gf.all()) and torch.equal(gv, v[lo:lo + chunk])
    absent, _ = gc.u64_keys(1 << 24, lo=n, with_values=False)
    gv, gf = m.lookup(absent)
    assert not bool(gf.any()) and not bool(gv.any())
    d, slots, _ = m.export()
    m.free()
    _check_dir_properties(d, n, inf.S)
    keys, vals = _u(k), _u(v)
    del k, v, absent
    torch.cuda.empty_cache()
    _check_full_by_shards(d, slots, keys, vals, n, 0, inf.t1, inf.S, nshards=64)


def test_config5_2e30_queries_on_2e27_table():
    hm, gc = _hm(), _dev_gen()
    n, nq = 1 << 27, 1 << 30
    k, v = gc.u64_keys(n)
    m = hm.HashMap.build_u64(k, v)
    inf = m.info()
    chunk = 1 << 28
    hits = 0
    for lo in range(0, nq, chunk):
        q, ev, ef = gc.u64_queries(n, chunk, lo=lo, with_expect=True)
        gv, gf = m.lookup(q)
        assert torch.equal(gf, ef) and torch.equal(gv, ev)
        hits += int(gf.sum())
        del q, ev, ef, gv, gf
    assert abs(hits / nq - 0.5) < 0.01
    d, slots, _ = m.export()
    m.free()
    _check_dir_properties(d, n, inf.S)
    keys, vals = _u(k), _u(v)
    del k, v
    _check_full_by_shards(d, slots, keys, vals, n, 0, inf.t1, inf.S, nshards=16)
