"""The seeded generators (workloads/gen.py) produce the paper-shaped inputs
(uniform, no duplicates) with the recipe of DESIGN.md §3."""
import numpy as np

from workloads import gen


def test_stream_matches_scalar_and_is_distinct():
    k = gen.u64_keys(1 << 16)
    assert len(np.unique(k)) == len(k)
    for i in (0, 1, 2, 12345, (1 << 16) - 1):
        assert int(k[i]) == gen.stream_py(gen.SEED_K, i)
    # members and absent keys are disjoint
    a = gen.u64_keys(1 << 16, lo=1 << 16)
    assert len(np.intersect1d(k, a)) == 0


def test_queries_half_hits():
    n, nq = 1 << 14, 1 << 16
    q, member, vals = gen.u64_queries(n, nq)
    keys = gen.u64_keys(n)
    pos = {int(x): i for i, x in enumerate(keys)}
    assert abs(member.mean() - 0.5) < 0.02
    for j in range(0, nq, 97):
        if member[j]:
            assert pos[int(q[j])] == int(vals[j])
        else:
            assert int(q[j]) not in pos and vals[j] == 0


def test_strings_shape():
    ctx, offs = gen.string_keys(5000)
    lens = np.diff(offs.astype(np.int64))
    assert lens.min() >= 4 and lens.max() <= 64 and abs(lens.mean() - 34) < 1.0
    s = gen.string_list(ctx, offs)
    assert len(set(s)) == len(s)
    assert s[7][:4] == int(gen.fmix32(np.array([7]))[0]).to_bytes(4, "little")
    qctx, qoffs, member, vals = gen.string_queries(5000, 4000)
    qs = gen.string_list(qctx, qoffs)
    pos = {x: i for i, x in enumerate(s)}
    for j in range(4000):
        assert (qs[j] in pos) == bool(member[j])
        if member[j]:
            assert pos[qs[j]] == int(vals[j])
