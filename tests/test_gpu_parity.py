"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle.

Bit-exact on every byte of the exported table (header fields, directory,
slots, context copy) and on every lookup output — all integer work
(DESIGN.md §5).  Sizes span many build partitions plus ragged tails; the
edge cases are the method's degenerate ones (n=1, tiny n with level-1
redraws, duplicates, empty strings).
"""
import numpy as np
import pytest

from oracle import oracle as O
from workloads import gen

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _hm():
    from paper_2508_11443_b200 import hm
    return hm


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).cuda()


def host(t):
    return t.cpu().numpy().view(np.uint64) if t.dtype == torch.int64 else t.cpu().numpy()


def assert_table_equal(m, ot):
    d, slots, ctx = m.export()
    inf = m.info()
    assert inf.n == ot.n and inf.S == ot.S
    assert inf.t1 == int(ot.header["t1"]) and inf.t0 == int(ot.header["t0"])
    assert inf.seed == int(ot.header["seed"])
    assert m.header_bytes() == ot.header_bytes()
    bad = np.nonzero(d != ot.dir)[0]
    assert len(bad) == 0, f"dir differs at {bad[:10]} gpu={d[bad[:3]]} oracle={ot.dir[bad[:3]]}"
    assert slots.tobytes() == ot.slots.tobytes(), "slots differ"
    if ctx is not None:
        assert ctx.tobytes() == ot.ctx.tobytes()


U64_CASES = [
    (1, 0, 0), (2, 0, 0), (5, 0, 0), (7, 3, 0), (100, 1, 0), (1000, 2, 0), (4133, 5, 0),
    (1 << 14, 0, 0), (50_000, 7, 0), (1 << 16, 0, 0), (1 << 16, 11, 0),
    # forced small partitions: many CTAs, long look-back chains, ragged last partition
    (70_001, 3, 6), (1 << 17, 4, 9), (300_007, 0, 12),
    # requests below 2^5 buckets per partition act as 2^5 (a compact-directory
    # record is one partition's): a two-pass build at this size
    (100_003, 2, 2),
]


@pytest.mark.parametrize("n,seed,log2_bp", U64_CASES)
def test_u64_build_and_lookup_parity(n, seed, log2_bp):
    hm = _hm()
    keys, vals = gen.u64_keys(n), gen.u64_values(n)
    ot = O.build_u64(keys, vals, seed)
    m = hm.HashMap.build_u64(dev(keys), dev(vals), seed=seed, log2_bp=log2_bp)
    assert_table_equal(m, ot)
    nq = max(2 * n, 1000)
    q, exp_found, exp_vals = gen.u64_queries(n, nq)
    ov, of = O.lookup_u64(ot, q)
    assert np.array_equal(of.astype(bool), exp_found) and np.array_equal(ov, exp_vals)
    gv, gf = m.lookup(dev(q))
    torch.cuda.synchronize()
    assert np.array_equal(host(gv), ov) and np.array_equal(host(gf), of)
    # membership only (no values)
    gf2 = m.contains(dev(q))
    assert np.array_equal(host(gf2), of)
    m.free()


def test_u64_many_seeds_small():
    hm = _hm()
    for n in (3, 6, 8, 13, 31):
        keys, vals = gen.u64_keys(n, lo=n * 1000), gen.u64_values(n)
        for seed in range(0, 60):
            ot = O.build_u64(keys, vals, seed)
            m = hm.HashMap.build_u64(dev(keys), dev(vals), seed=seed)
            assert_table_equal(m, ot)
            m.free()


def test_u64_compact_directory_escapes():
    """Lookups read a compact directory whose records escape to
    the full directory when a bucket has s >= 7 or t >= 15: exercise both."""
    hm = _hm()
    escapes = 0
    for n in (20, 24):
        keys, vals = gen.u64_keys(n, lo=7 * n), gen.u64_values(n)
        q = np.concatenate([keys, gen.u64_keys(3 * n, lo=100 * n)])
        for seed in range(300):
            ot = O.build_u64(keys, vals, seed)
            _, s, t = O.decode_dir(ot.dir)
            esc = bool(((s >= 7) | (t >= 15)).any())
            if not esc and seed % 10:
                continue
            escapes += esc
            m = hm.HashMap.build_u64(dev(keys), dev(vals), seed=seed)
            assert_table_equal(m, ot)
            ov, of = O.lookup_u64(ot, q)
            gv, gf = m.lookup(dev(q))
            assert np.array_equal(host(gv), ov) and np.array_equal(host(gf), of)
            m.free()
    assert escapes > 0
    # every record escaping (HM_FLAG_FULL_DIRECTORY) must give the same answers
    n = 70_001
    keys, vals = gen.u64_keys(n), gen.u64_values(n)
    q, _, _ = gen.u64_queries(n, 3 * n)
    ot = O.build_u64(keys, vals, 4)
    m = hm.HashMap.build_u64(dev(keys), dev(vals), seed=4, flags=hm.FLAG_FULL_DIRECTORY)
    assert_table_equal(m, ot)
    ov, of = O.lookup_u64(ot, q)
    gv, gf = m.lookup(dev(q))
    assert np.array_equal(host(gv), ov) and np.array_equal(host(gf), of)


def test_u64_order_invariance_and_host_path():
    hm = _hm()
    n = 123_457
    keys, vals = gen.u64_keys(n), gen.u64_values(n)
    perm = np.random.default_rng(0).permutation(n)
    m1 = hm.HashMap.build_u64(dev(keys), dev(vals), seed=9)
    m2 = hm.HashMap.build_u64(dev(keys[perm]), dev(vals[perm]), seed=9)
    m3 = hm.HashMap.build_u64(keys[perm], vals[perm], seed=9)  # host (numpy) buffers
    d1, s1, _ = m1.export()
    for m in (m2, m3):
        d, s, _ = m.export()
        assert d.tobytes() == d1.tobytes() and s.tobytes() == s1.tobytes()
    q, f, v = gen.u64_queries(n, 10_000)
    hv, hf = m3.lookup(q)  # host in, host out
    assert np.array_equal(hv, v) and np.array_equal(hf.astype(bool), f)


def test_u64_error_cases():
    hm = _hm()
    with pytest.raises(hm.HMError) as e:
        hm.HashMap.build_u64(dev(np.array([7, 7], np.uint64)), dev(np.array([1, 2], np.uint64)))
    assert e.value.name == "DUPLICATE_KEY"
    with pytest.raises(hm.HMError) as e:
        hm.HashMap.build_u64(dev(np.full(5, 9, np.uint64)), dev(np.arange(5, dtype=np.uint64)))
    assert e.value.name == "SEED_EXHAUSTED"
    keys = gen.u64_keys(100_000)
    keys[77_777] = keys[12]
    with pytest.raises(hm.HMError) as e:
        hm.HashMap.build_u64(dev(keys), dev(gen.u64_values(100_000)))
    assert e.value.name == "DUPLICATE_KEY"
    with pytest.raises(O.OracleError) as eo:
        O.build_u64(keys, gen.u64_values(100_000), 0)
    assert eo.value.name == "DUPLICATE_KEY"
    with pytest.raises(hm.HMError) as e:
        hm.HashMap.build_u64(dev(np.zeros(0, np.uint64)), dev(np.zeros(0, np.uint64)))
    assert e.value.name == "EMPTY"


def test_build_workspace_reuse_release_and_streams():
    """The cached build scratch (hm_release_workspace): shrinking and growing
    sizes, a second stream, and a release between builds all give the
    oracle's table."""
    hm = _hm()
    side = torch.cuda.Stream()
    for i, n in enumerate([300_000, 1000, 70_001, 300_000, 5]):
        keys, vals = gen.u64_keys(n), gen.u64_values(n)
        ot = O.build_u64(keys, vals, i)
        if i == 3:
            hm.release_workspace()
        k, v = dev(keys), dev(vals)
        if i % 2:
            torch.cuda.synchronize()
            with torch.cuda.stream(side):
                m = hm.HashMap.build_u64(k, v, seed=i)
            side.synchronize()
        else:
            m = hm.HashMap.build_u64(k, v, seed=i)
        assert_table_equal(m, ot)
        m.free()
    hm.release_workspace()


def test_u64_adversarial_values_and_keys():
    """Keys at the edges of u64 (0, 2^64-1, P, P+5, 2^32 boundaries)."""
    hm = _hm()
    P = (1 << 61) - 1
    special = [0, 1, (1 << 64) - 1, P, P + 5, 1 << 32, (1 << 32) - 1, (1 << 63), 5]
    keys = np.array(special + list(gen.u64_keys(991)), np.uint64)
    vals = np.array([(1 << 64) - 1 - i for i in range(len(keys))], np.uint64)
    for seed in range(5):
        ot = O.build_u64(keys, vals, seed)
        m = hm.HashMap.build_u64(dev(keys), dev(vals), seed=seed)
        assert_table_equal(m, ot)
        gv, gf = m.lookup(dev(keys))
        assert host(gf).all() and np.array_equal(host(gv), vals)


# ------------------------------------------------------------------ strings

STR_CASES = [(1, 0), (2, 1), (50, 0), (1000, 3), (20_000, 0), (70_000, 5)]


@pytest.mark.parametrize("n,seed", STR_CASES)
def test_bytes_build_and_lookup_parity(n, seed):
    hm = _hm()
    ctx, offs = gen.string_keys(n)
    vals = gen.u64_values(n) + np.uint64(1)
    ot = O.build_bytes(ctx, offs, vals, seed)
    m = hm.HashMap.build_bytes(torch.from_numpy(ctx).cuda(), dev(offs), dev(vals), seed=seed)
    assert_table_equal(m, ot)
    qctx, qoffs, f, v = gen.string_queries(n, max(2 * n, 500))
    ov, of = O.lookup_bytes(ot, qctx, qoffs)
    gv, gf = m.lookup_bytes(torch.from_numpy(qctx).cuda(), dev(qoffs))
    assert np.array_equal(host(gv), ov) and np.array_equal(host(gf), of)
    m.free()


def test_bytes_edge_strings_and_offsets():
    hm = _hm()
    strs = [b"", b"ab", b"ab\0", b"\0", b"\0\0\0\0", b"\0\0\0\0\0", b"x" * 64, b"y" * 1000, b"abc", b"abcd"]
    ctx, offs = gen.pack_bytes_list(strs)
    # non-zero first offset: the map copies bytes[offsets[0]..offsets[n])
    pre = np.frombuffer(b"PREFIX!", np.uint8)
    ctx2 = np.concatenate([pre, ctx])
    offs2 = offs + np.uint64(len(pre))
    vals = np.arange(10, 10 + len(strs), dtype=np.uint64)
    for seed in range(6):
        ot = O.build_bytes(ctx2, offs2, vals, seed)
        m = hm.HashMap.build_bytes(torch.from_numpy(ctx2).cuda(), dev(offs2), dev(vals), seed=seed)
        assert_table_equal(m, ot)
        needles = strs + [b"a", b"ab\0\0", b"x" * 63, b"y" * 999 + b"z", b"PREFIX!"]
        qc, qo = gen.pack_bytes_list(needles)
        ov, of = O.lookup_bytes(ot, qc, qo)
        gv, gf = m.lookup_bytes(qc, qo)  # host needles
        assert np.array_equal(gv, ov) and np.array_equal(gf, of)
    with pytest.raises(hm.HMError) as e:
        c, o = gen.pack_bytes_list([b"hello", b"world", b"hello"])
        hm.HashMap.build_bytes(torch.from_numpy(c).cuda(), dev(o), dev(np.arange(3, dtype=np.uint64)))
    assert e.value.name == "DUPLICATE_KEY"


def test_bytes_every_length_and_alignment():
    """Keys of every length 0..300 at every start alignment (the expanded
    fingerprint's chunk tails, its 128-byte table limit and the Horner path
    beyond it; warps whose byte range overflows the shared-memory stage)."""
    hm = _hm()
    rng = np.random.default_rng(11)
    strs = []
    for L in range(0, 301):
        for _ in range(3):
            strs.append(rng.integers(0, 256, size=L, dtype=np.uint8).tobytes() if L else b"")
    strs = list(dict.fromkeys(strs))  # (distinct; b"" once)
    strs += [b"\xff" * L for L in (1, 7, 8, 9, 63, 64, 65, 127, 128, 129)]
    order = rng.permutation(len(strs))
    strs = [strs[i] for i in order]
    ctx, offs = gen.pack_bytes_list(strs)
    vals = np.arange(1, len(strs) + 1, dtype=np.uint64)
    ot = O.build_bytes(ctx, offs, vals, 4)
    m = hm.HashMap.build_bytes(torch.from_numpy(ctx).cuda(), dev(offs), dev(vals), seed=4)
    assert_table_equal(m, ot)
    needles = strs + [s[:-1] + b"\x01" for s in strs if s] + [b"\xff" * 66]
    qc, qo = gen.pack_bytes_list(needles)
    ov, of = O.lookup_bytes(ot, qc, qo)
    gv, gf = m.lookup_bytes(torch.from_numpy(qc).cuda(), dev(qo))
    assert np.array_equal(host(gv), ov) and np.array_equal(host(gf), of)
    m.free()


@pytest.mark.parametrize("shift,prefix", [(3, 0), (3, 13), (8, 5), (0, 16), (0, 1)])
def test_bytes_unaligned_context_pointer(shift, prefix):
    """A key context that starts at any byte address (a tensor slice) with any
    first offset: the fingerprint stage aligns by address, and the map's copy
    of the context is written by the fingerprint kernel exactly when
    bytes + offsets[0] is 16-aligned, else by a copy."""
    hm = _hm()
    ctx, offs = gen.string_keys(5000)
    ctx2 = np.concatenate([np.full(prefix, 0x5A, np.uint8), ctx])
    offs2 = offs + np.uint64(prefix)
    vals = gen.u64_values(5000) + np.uint64(1)
    base = torch.zeros(shift + len(ctx2) + 32, dtype=torch.uint8, device="cuda")
    base[shift:shift + len(ctx2)] = torch.from_numpy(ctx2).cuda()
    t = base[shift:shift + len(ctx2)]
    ot = O.build_bytes(ctx2, offs2, vals, 2)
    m = hm.HashMap.build_bytes(t, dev(offs2), dev(vals), seed=2)
    assert_table_equal(m, ot)
    base.fill_(0)  # the map holds its own copy
    qc, qo, f, v = gen.string_queries(5000, 20_000)
    qbase = torch.zeros(len(qc) + 40, dtype=torch.uint8, device="cuda")
    qbase[shift + 5:shift + 5 + len(qc)] = torch.from_numpy(qc).cuda()
    ov, of = O.lookup_bytes(ot, qc, qo)
    gv, gf = m.lookup_bytes(qbase[shift + 5:shift + 5 + len(qc)], dev(qo))
    assert np.array_equal(host(gv), ov) and np.array_equal(host(gf), of)
    assert np.array_equal(host(gf).astype(bool), f)
    m.free()


@pytest.mark.parametrize("flags_name", ["FLAG_DIRECT_SLOTS", "FLAG_NO_ROUND0_ILP", "FLAG_ROUNDS", "FLAG_FUSED_PASS2"])
@pytest.mark.parametrize("n,seed,log2_bp", [(5, 0, 0), (4133, 5, 0), (70_001, 3, 6), (300_007, 1, 0)])
def test_u64_construction_routes_same_table(flags_name, n, seed, log2_bp):
    """The testing knobs change how k_bucket gets there (direct slot writes
    instead of the shared-memory source map; one round-0 attempt instead of
    two), and FLAG_ROUNDS replaces it with the paper's sortless rounds
     — never the table: all must equal the oracle byte for byte."""
    hm = _hm()
    keys, vals = gen.u64_keys(n, lo=3 * n), gen.u64_values(n)
    ot = O.build_u64(keys, vals, seed)
    m = hm.HashMap.build_u64(dev(keys), dev(vals), seed=seed, log2_bp=log2_bp, flags=getattr(hm, flags_name))
    assert_table_equal(m, ot)
    q, _, _ = gen.u64_queries(n, 2 * n + 100)
    ov, of = O.lookup_u64(ot, q)
    gv, gf = m.lookup(dev(q))
    assert np.array_equal(host(gv), ov) and np.array_equal(host(gf), of)
    m.free()


@pytest.mark.parametrize("n,seed,log2_bp", [(70_001, 2, 5), (300_007, 4, 6), (2_200_003, 6, 5), (1 << 20, 8, 5)])
def test_u64_fused_pipeline_same_table(n, seed, log2_bp):
    """HM_FLAG_FUSED_PASS2: two-pass builds (more than 1024 partitions) run
    radix pass 2 and the per-partition construction as one pipelined kernel
    (k_split2_bucket): a partition job waits for its coarse region's pass-2
    tiles and drops its L2 lines after loading them.  Ragged last regions (np
    not a multiple of the 256/512 partitions per region), 8- and 9-bit digits
    (np > 65536 at 2.2M keys and log2_bp = 5): the oracle's table and lookups,
    and the same bytes as the default two-kernel route."""
    hm = _hm()
    keys, vals = gen.u64_keys(n, lo=n), gen.u64_values(n)
    ot = O.build_u64(keys, vals, seed)
    m = hm.HashMap.build_u64(dev(keys), dev(vals), seed=seed, log2_bp=log2_bp, flags=hm.FLAG_FUSED_PASS2)
    assert_table_equal(m, ot)
    u = hm.HashMap.build_u64(dev(keys), dev(vals), seed=seed, log2_bp=log2_bp)
    assert_table_equal(u, ot)
    q, _, _ = gen.u64_queries(n, n + 1000)
    ov, of = O.lookup_u64(ot, q)
    gv, gf = m.lookup(dev(q))
    assert np.array_equal(host(gv), ov) and np.array_equal(host(gf), of)
    # back to back on the same stream: the scratch (sdone, pcount) is reset per build
    for _ in range(3):
        m2 = hm.HashMap.build_u64(dev(keys), dev(vals), seed=seed, log2_bp=log2_bp, flags=hm.FLAG_FUSED_PASS2)
        assert_table_equal(m2, ot)
        m2.free()
    m.free()
    u.free()


@pytest.mark.parametrize("flags_name", ["FLAG_DIRECT_SLOTS", "FLAG_NO_ROUND0_ILP", "FLAG_ROUNDS", "FLAG_FUSED_PASS2"])
def test_u64_construction_routes_duplicates(flags_name):
    hm = _hm()
    keys = gen.u64_keys(100_000)
    keys[91_234] = keys[5]
    with pytest.raises(hm.HMError) as e:
        hm.HashMap.build_u64(dev(keys), dev(gen.u64_values(100_000)), flags=getattr(hm, flags_name))
    assert e.value.name == "DUPLICATE_KEY"


def test_u64_duplicate_heavy_overflow_matches_oracle():
    """Thousands of copies of one key overflow a build partition; the GPU
    recounts the suspect partitions for the space bound (R7) and, like the
    oracle, exhausts level one (SEED_EXHAUSTED, R26).  With the bound holding
    (a huge n) the build falls back to the flat rounds (any bucket size), which
    report the equal keys as the oracle does (DUPLICATE_KEY)."""
    hm = _hm()
    n = 200_000
    keys = gen.u64_keys(n)
    keys[:2000] = keys[7]
    vals = gen.u64_values(n)
    with pytest.raises(O.OracleError) as eo:
        O.build_u64(keys, vals, 0)
    with pytest.raises(hm.HMError) as e:
        hm.HashMap.build_u64(dev(keys), dev(vals))
    assert e.value.name == eo.value.name == "SEED_EXHAUSTED"
    n = 2_000_000
    keys = gen.u64_keys(n)
    keys[:1500] = keys[11]
    vals = gen.u64_values(n)
    with pytest.raises(O.OracleError) as eo:
        O.build_u64(keys, vals, 0)
    with pytest.raises(hm.HMError) as e:
        hm.HashMap.build_u64(dev(keys), dev(vals))
    # (the bound holds: the flat rounds take over and find them, as the oracle's make2 does)
    assert e.value.name == eo.value.name == "DUPLICATE_KEY"
    # the map and the workspace stay usable after the degenerate builds
    keys, vals = gen.u64_keys(5000), gen.u64_values(5000)
    m = hm.HashMap.build_u64(dev(keys), dev(vals))
    assert_table_equal(m, O.build_u64(keys, vals, 0))
    m.free()


@pytest.mark.parametrize("n,ndistinct,seed", [(1, 1, 0), (10, 3, 1), (5000, 5000, 2), (300_000, 70_000, 3),
                                              (1 << 20, 1 << 18, 0)])
def test_u64_from_array_parity(n, ndistinct, seed):
    """from_array (HM_FLAG_FROM_ARRAY): duplicates allowed, the first occurrence
    keeps its value; the table equals the oracle's from_array byte for byte."""
    hm = _hm()
    rng = np.random.default_rng(n + seed)
    base = gen.u64_keys(ndistinct, lo=11)
    keys = base[rng.integers(0, ndistinct, size=n)] if n > ndistinct else base[rng.permutation(ndistinct)]
    vals = gen.u64_values(n, lo=100)
    ot = O.from_array_u64(keys, vals, seed)
    m = hm.HashMap.build_u64(dev(keys), dev(vals), seed=seed, flags=hm.FLAG_FROM_ARRAY)
    assert_table_equal(m, ot)
    q = np.concatenate([base, gen.u64_keys(1000, lo=10 * n + 7)])
    ov, of = O.lookup_u64(ot, q)
    gv, gf = m.lookup(dev(q))
    assert np.array_equal(host(gv), ov) and np.array_equal(host(gf), of)
    m.free()


def test_u64_from_array_heavy_duplication():
    """A million copies of one key among a few distinct ones: the dedup set
    meets them in one slot; the map holds 4 keys."""
    hm = _hm()
    n = 1_000_000
    keys = np.full(n, np.uint64(0xDEADBEEF12345678))
    keys[[10, 500_000, 999_999]] = gen.u64_keys(3, lo=5)
    vals = gen.u64_values(n, lo=0)
    ot = O.from_array_u64(keys, vals, 0)
    m = hm.HashMap.build_u64(dev(keys), dev(vals), flags=hm.FLAG_FROM_ARRAY)
    assert m.info().n == 4
    assert_table_equal(m, ot)
    gv, gf = m.lookup(dev(np.array([0xDEADBEEF12345678], np.uint64)))
    assert host(gv)[0] == 0 and host(gf)[0] == 1  # the first copy is input 0 with value 0
    m.free()


@pytest.mark.parametrize("n,ndistinct,seed", [(1, 1, 0), (40, 7, 1), (3000, 3000, 2), (200_000, 50_000, 3)])
def test_bytes_from_array_parity(n, ndistinct, seed):
    """from_array for byte keys (HM_FLAG_FROM_ARRAY): content duplicates, the
    first occurrence keeps its value, the distinct keys are packed in input
    order; table and context equal the oracle's byte for byte."""
    hm = _hm()
    rng = np.random.default_rng(n * 7 + seed)
    ids = rng.integers(0, ndistinct, size=n).astype(np.uint64) if n > ndistinct else \
        rng.permutation(ndistinct).astype(np.uint64)
    ctx, offs = gen.pack_strings(ids + np.uint64(5))
    vals = gen.u64_values(n, lo=1000)
    ot = O.from_array_bytes(ctx, offs, vals, seed)
    m = hm.HashMap.build_bytes(torch.from_numpy(ctx).cuda(), dev(offs), dev(vals), seed=seed,
                               flags=hm.FLAG_FROM_ARRAY)
    assert_table_equal(m, ot)
    qc, qo = gen.pack_strings(np.arange(0, ndistinct + 50, dtype=np.uint64) + np.uint64(5))
    ov, of = O.lookup_bytes(ot, qc, qo)
    gv, gf = m.lookup_bytes(torch.from_numpy(qc).cuda(), dev(qo))
    assert np.array_equal(host(gv), ov) and np.array_equal(host(gf), of)
    m.free()


def test_u64_rounds_ablation_large_and_from_array():
    """The sortless round-based construction (HM_FLAG_ROUNDS) at a
    size with tens of rounds: the same table as the default build (whose
    parity with the oracle is tested above) and, for from_array input, as the
    oracle's; byte keys are outside the ablation."""
    hm = _hm()
    n = 1 << 21
    keys, vals = gen.u64_keys(n), gen.u64_values(n)
    a = hm.HashMap.build_u64(dev(keys), dev(vals), seed=9)
    b = hm.HashMap.build_u64(dev(keys), dev(vals), seed=9, flags=hm.FLAG_ROUNDS)
    da, sa, _ = a.export()
    db, sb, _ = b.export()
    assert a.header_bytes() == b.header_bytes()
    assert np.array_equal(da, db) and sa.tobytes() == sb.tobytes()
    q, _, _ = gen.u64_queries(n, 1 << 20)
    va, fa = a.lookup(dev(q))
    vb, fb = b.lookup(dev(q))
    assert torch.equal(va, vb) and torch.equal(fa, fb)
    a.free()
    b.free()
    rng = np.random.default_rng(4)
    base = gen.u64_keys(50_000, lo=11)
    keys = base[rng.integers(0, 50_000, size=200_000)]
    vals = gen.u64_values(200_000, lo=3)
    m = hm.HashMap.build_u64(dev(keys), dev(vals), seed=2, flags=hm.FLAG_ROUNDS | hm.FLAG_FROM_ARRAY)
    assert_table_equal(m, O.from_array_u64(keys, vals, 2))
    m.free()
    c, o = gen.string_keys(100)
    with pytest.raises(hm.HMError) as e:
        hm.HashMap.build_bytes(torch.from_numpy(c).cuda(), dev(o), dev(gen.u64_values(100)), flags=hm.FLAG_ROUNDS)
    assert e.value.name == "INVALID_ARG"


@pytest.mark.parametrize("pinned", [True, False])
def test_u64_lookup_host_buffers_pipelined(pinned):
    """Host queries with host outputs above two chunks (2^23) take the chunked
    upload/lookup/download pipeline of hm_lookup_u64; answers equal the device
    path's (whose parity with the oracle is tested above), with and without
    a value output, from pinned and from pageable memory."""
    hm = _hm()
    n = 1 << 20
    keys, vals = gen.u64_keys(n), gen.u64_values(n)
    m = hm.HashMap.build_u64(dev(keys), dev(vals), seed=1)
    nq = (1 << 24) + (1 << 22) + 12345  # 2.5 chunks and a ragged tail
    q, _, _ = gen.u64_queries(n, nq)
    dv, df = m.lookup(dev(q))
    hq = torch.from_numpy(q.view(np.int64))
    hv = torch.empty(nq, dtype=torch.int64)
    hf = torch.empty(nq, dtype=torch.uint8)
    if pinned:
        hq, hv, hf = hq.pin_memory(), hv.pin_memory(), hf.pin_memory()
    m.lookup(hq, hv, hf)
    assert torch.equal(hv, dv.cpu()) and torch.equal(hf, df.cpu())
    hf2 = torch.zeros(nq, dtype=torch.uint8)
    m.contains(hq, hf2)
    assert torch.equal(hf2, df.cpu())
    m.free()


def test_user_allocator_hooks():
    """hm_opts.alloc / .free: every array a map owns comes from
    the hook (here torch's caching allocator) and goes back through it in
    hm_free, also on a failed build; the maps are the oracle's."""
    hm = _hm()
    live, calls = {}, {"alloc": 0, "free": 0}

    def alloc(n, st):
        p = torch.cuda.caching_allocator_alloc(n, device=0, stream=st or 0)
        live[p] = n
        calls["alloc"] += 1
        return p

    def free(p, n, st):
        assert live.pop(p) == n
        calls["free"] += 1
        torch.cuda.caching_allocator_delete(p)

    hm.set_allocator(alloc, free)
    try:
        n = 100_003
        keys, vals = gen.u64_keys(n), gen.u64_values(n)
        m = hm.HashMap.build_u64(dev(keys), dev(vals), seed=2)
        assert calls["alloc"] == 3 and len(live) == 3
        assert_table_equal(m, O.build_u64(keys, vals, 2))
        m.free()
        assert not live and calls["free"] == 3
        ctx, offs = gen.string_keys(5000)
        bv = gen.u64_values(5000)
        mb = hm.HashMap.build_bytes(torch.from_numpy(ctx).cuda(), dev(offs), dev(bv), seed=1)
        assert len(live) == 4  # dir, compact dir, slots, context copy
        assert_table_equal(mb, O.build_bytes(ctx, offs, bv, 1))
        mb.free()
        assert not live
        keys[777] = keys[3]
        with pytest.raises(hm.HMError) as e:
            hm.HashMap.build_u64(dev(keys), dev(vals))
        assert e.value.name == "DUPLICATE_KEY" and not live
    finally:
        hm.set_allocator(None, None)
    m = hm.HashMap.build_u64(dev(keys[:10]), dev(vals[:10]))  # the library's pool again
    assert not live
    m.free()


def test_bytes_from_array_heavy_duplication():
    """Byte keys repeated so often that a dedup partition overflows take the
    global fingerprint set (content-confirmed); the map equals the oracle's
    from_array: 300 000 copies of one string among 2 000 distinct ones."""
    hm = _hm()
    strs = [bytes(x) for x in gen.string_list(*gen.string_keys(2000))]
    idx = np.random.default_rng(5).integers(0, 2000, size=20_000)
    keys = [strs[i] for i in idx] + [strs[7]] * 300_000 + [b""] * 1000
    ctx, offs = gen.pack_bytes_list(keys)
    vals = gen.u64_values(len(keys), lo=9)
    ot = O.from_array_bytes(ctx, offs, vals, 4)
    hm.profile_read()
    hm.profile_enable(True)
    m = hm.HashMap.build_bytes(torch.from_numpy(ctx).cuda(), dev(offs), dev(vals), seed=4, flags=hm.FLAG_FROM_ARRAY)
    st = hm.profile_read()
    hm.profile_enable(False)
    assert "k_dedup_insert_bytes" in st  # (the global set decided)
    assert m.info().n == ot.n
    assert_table_equal(m, ot)
    m.free()


def test_u64_bucket_over_32_keys_takes_the_flat_rounds():
    """33 distinct keys in one level-1 bucket within the space bound: outside
    the partitioned search (s <= 32), so the build falls back to the flat
    rounds (HM_FLAG_ROUNDS' kernels, any s) — the table is still the oracle's."""
    hm = _hm()
    n, seed = 1024, 0
    c1 = O.derive(seed, 1, 0, 0)
    cand = gen.u64_keys(120_000, lo=77)
    b0 = O.hash_(c1, int(cand[0])) % n
    same, other = [], []
    for k in cand:
        b = O.hash_(c1, int(k)) % n
        if b == b0 and len(same) < 33:
            same.append(k)
        elif b != b0 and len(other) < n - 33:
            other.append(k)
        if len(same) == 33 and len(other) == n - 33:
            break
    keys = np.array(same + other, dtype=np.uint64)
    vals = gen.u64_values(n, lo=1)
    ot = O.build_u64(keys, vals, seed)
    assert int(ot.header["t1"]) == 0 and (ot.dir >> np.uint64(40) & np.uint64(0xFFFF)).max() == 33
    m = hm.HashMap.build_u64(dev(keys), dev(vals), seed=seed)
    assert_table_equal(m, ot)
    gv, gf = m.lookup(dev(keys))
    assert bool(gf.all()) and np.array_equal(host(gv), vals)
    m.free()


def test_bytes_duplicate_heavy_reports_duplicate_key():
    """Byte keys from_array_nodup with 1 500 copies of one string among 2*10^6
    (the space bound holds): equal keys are reported as DUPLICATE_KEY, as the
    oracle does, not TOO_LARGE."""
    hm = _hm()
    strs = gen.string_list(*gen.string_keys(2_000_000))
    keys = strs[:1_998_500] + [strs[3]] * 1500
    ctx, offs = gen.pack_bytes_list(keys)
    vals = gen.u64_values(len(keys))
    with pytest.raises(O.OracleError) as eo:
        O.build_bytes(ctx, offs, vals, 0)
    with pytest.raises(hm.HMError) as e:
        hm.HashMap.build_bytes(torch.from_numpy(ctx).cuda(), dev(offs), dev(vals))
    assert e.value.name == eo.value.name == "DUPLICATE_KEY"


def _fp_fixture():
    import os
    import sys
    sys.path.insert(0, os.path.dirname(__file__))
    from test_oracle_fpcoll import load_fixture
    return load_fixture()


@pytest.mark.parametrize("name", ["s2", "s3", "s5", "s9"])
def test_bytes_fingerprint_collision_redraws_t0(name):
    """Two different keys with equal fingerprints at (seed 0, t0 0) (the
    lattice-built fixture, tests/golden/fp_collision_seed0.txt; DESIGN R5,
    SURVEY 8(c) step 5): the GPU detects them in their level-1 bucket — a
    2-key bucket in round 0 (s2), 3- and 5-key buckets (s3, s5), a 9-key
    bucket in the warp-per-bucket search (s9) — redraws t0, and its table is
    the oracle's (t0 = 1) byte for byte."""
    hm = _hm()
    fx = _fp_fixture()
    strs = fx["sets"][name]
    ctx, offs = gen.pack_bytes_list(strs)
    vals = np.arange(100, 100 + len(strs), dtype=np.uint64)
    ot = O.build_bytes(ctx, offs, vals, 0)
    assert int(ot.header["t0"]) == 1
    m = hm.HashMap.build_bytes(torch.from_numpy(ctx).cuda(), dev(offs), dev(vals))
    assert m.info().t0 == 1
    assert_table_equal(m, ot)
    gv, gf = m.lookup_bytes(torch.from_numpy(ctx).cuda(), dev(offs))
    assert bool(gf.all()) and np.array_equal(host(gv), vals)
    m.free()


def test_bytes_fingerprint_collision_among_many_keys():
    """The colliding pair among 200 000 generated strings (equal fingerprints
    share a level-1 bucket at any n): redraw t0, the oracle's table."""
    hm = _hm()
    fx = _fp_fixture()
    a, b = fx["pair"]
    strs = gen.string_list(*gen.string_keys(200_000))
    strs[1234] = a
    strs[150_001] = b
    assert len(set(strs)) == len(strs)
    ctx, offs = gen.pack_bytes_list(strs)
    vals = gen.u64_values(len(strs), lo=9)
    ot = O.build_bytes(ctx, offs, vals, 0)
    assert int(ot.header["t0"]) == 1
    m = hm.HashMap.build_bytes(torch.from_numpy(ctx).cuda(), dev(offs), dev(vals))
    assert_table_equal(m, ot)
    m.free()


def test_bytes_bucket_over_32_keys_takes_the_flat_rounds():
    """33 distinct byte keys whose fingerprints share one level-1 bucket, within
    the space bound: outside the partitioned search (s <= 32), so the byte
    build falls back to the flat rounds (any s) — the oracle's table, not
    TOO_LARGE (make2 has no size cap)."""
    hm = _hm()
    n, seed = 1024, 0
    r0 = O.derive(seed, 0, 0, 0)[0]
    c1 = O.derive(seed, 1, 0, 0)
    cand = gen.string_list(*gen.string_keys(60_000, lo=5))
    bucket = [O.hash_(c1, O.fingerprint(x, r0)) % n for x in cand]
    b0 = bucket[0]
    same = [x for x, b in zip(cand, bucket) if b == b0][:33]
    other = [x for x, b in zip(cand, bucket) if b != b0][: n - 33]
    assert len(same) == 33 and len(other) == n - 33
    strs = same + other
    ctx, offs = gen.pack_bytes_list(strs)
    vals = gen.u64_values(n, lo=1)
    ot = O.build_bytes(ctx, offs, vals, seed)
    assert int(ot.header["t0"]) == 0 and int(ot.header["t1"]) == 0
    assert (ot.dir >> np.uint64(40) & np.uint64(0xFFFF)).max() == 33
    m = hm.HashMap.build_bytes(torch.from_numpy(ctx).cuda(), dev(offs), dev(vals), seed=seed)
    assert_table_equal(m, ot)
    gv, gf = m.lookup_bytes(torch.from_numpy(ctx).cuda(), dev(offs))
    assert bool(gf.all()) and np.array_equal(host(gv), vals)
    m.free()
