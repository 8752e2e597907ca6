"""GPU parity at BASELINE.json's full sizes, in the launch configuration
bench.py times (default build options, device-resident inputs).

configs[1] (2^26 u64) and configs[2] (2^24 strings): every byte of the exported
table against the oracle, every lookup against the generator's ground truth.
configs[3]/[4] sizes (2^29 keys; 2^27-key table with 2^30 queries) on one GPU:
properties that hold at any size (S <= 4n, the directory is the exclusive scan
of s^2 and sums to n, every member found with its value, every absent key
misses) plus sampled bucket ranges rebuilt by the oracle's shard definition.
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


def _check_sampled_ranges(m_dir, m_slots, keys, vals, n, seed, t1, rng, nranges=48, width=64):
    """Rebuild random bucket ranges with the oracle's shard definition and
    compare directory entries (relative soff, s, t) and slot bytes."""
    g = O.level1_buckets(keys, n, seed, t1)
    soff = m_dir & MASK40
    for lo in rng.integers(0, n - width, nranges):
        lo = int(lo)
        hi = lo + width
        sel = (g >= lo) & (g < hi)
        st, sh = O.build_u64_shard(keys[sel], vals[sel], n, lo, hi, t1, seed)
        assert st == "OK"
        gd = m_dir[lo:hi]
        base = int(soff[lo])
        rel = (gd & ~MASK40) | ((gd & MASK40) - np.uint64(base))
        assert np.array_equal(rel, sh.dir), f"directory differs in buckets [{lo},{hi})"
        assert m_slots[base:base + sh.S].tobytes() == sh.slots.tobytes(), f"slots differ in [{lo},{hi})"


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
    _check_sampled_ranges(d, slots, keys, vals, n, 0, inf.t1, np.random.default_rng(4))


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
    _check_sampled_ranges(d, slots, keys, vals, n, 0, inf.t1, np.random.default_rng(5))
