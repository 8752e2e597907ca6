"""Pins for the oracle's byte-string path (not gpu): keys are slices of a flat
context, the map keeps its own copy, and
needles come with their own context."""
import numpy as np
import pytest

from oracle import oracle as O
from workloads import gen

P = (1 << 61) - 1


def _assoc_check(t, strs, vals, needles):
    assoc = {s: int(v) for s, v in zip(strs, vals)}
    qctx, qoff = gen.pack_bytes_list(needles)
    v, f = O.lookup_bytes(t, qctx, qoff)
    for s, vv, ff in zip(needles, v, f):
        assert bool(ff) == (s in assoc), s
        assert int(vv) == assoc.get(s, 0)


def test_string_roundtrip_and_near_misses():
    n = 3000
    ctx, offs = gen.string_keys(n)
    strs = gen.string_list(ctx, offs)
    assert len(set(strs)) == n and all(4 <= len(s) <= 64 for s in strs)
    vals = gen.u64_values(n)
    t = O.build_bytes(ctx, offs, vals, 0)
    assert int(t.header["key_kind"]) == 1 and int(t.header["ctx_bytes"]) == len(ctx)
    assert t.ctx.tobytes() == ctx.tobytes()
    near = []
    for s in strs[:300]:
        near += [s[:-1], s + b"\0", bytes([s[0] ^ 1]) + s[1:], s[:-1] + bytes([s[-1] ^ 0x80])]
    _assoc_check(t, strs, vals, strs + near + [b"", b"a"])


def test_needles_from_foreign_context_with_offset():
    n = 500
    ctx, offs = gen.string_keys(n)
    strs = gen.string_list(ctx, offs)
    t = O.build_bytes(ctx, offs, gen.u64_values(n), 9)
    # same contents at different offsets of a different buffer
    pad = [b"zz" * (i % 5) for i in range(n)]
    qctx, qoff = gen.pack_bytes_list([p + s for p, s in zip(pad, strs)])
    qoff2 = qoff.copy()
    for i in range(n):
        qoff2[i] = qoff[i] + len(pad[i])
    # CSR needs q[i] = ctx[off[i]:off[i+1]] so build explicit slices via a lookup loop
    for i in range(0, n, 37):
        one_ctx = qctx[int(qoff2[i]):int(qoff[i + 1])]
        v, f = O.lookup_bytes(t, one_ctx, np.array([0, len(one_ctx)], np.uint64))
        assert f[0] == 1 and int(v[0]) == i


def test_slot_fields_follow_layout():
    n = 800
    ctx, offs = gen.string_keys(n, lo=1000)
    # the map copies bytes[offsets[0]..offsets[n]): shift offsets by a prefix
    pre = np.full(13, 7, np.uint8)
    ctx2 = np.concatenate([pre, ctx])
    offs2 = offs + np.uint64(13)
    vals = np.arange(5, 5 + n, dtype=np.uint64)
    t = O.build_bytes(ctx2, offs2, vals, 4)
    assert t.ctx.tobytes() == ctx.tobytes()
    r = O.derive(4, 0, 0, int(t.header["t0"]))[0]
    strs = gen.string_list(ctx, offs)
    pos = {s: i for i, s in enumerate(strs)}
    members = 0
    for sl in t.slots:
        s = t.ctx[int(sl["ctx_off"]):int(sl["ctx_off"]) + int(sl["len"])].tobytes()
        assert s in pos and int(sl["reserved"]) == 0
        assert int(sl["fp"]) == O.fingerprint(s, r)
        if int(sl["value"]) != 0:
            members += 1
            assert int(sl["value"]) == 5 + pos[s]
    assert members == n  # values are all non-zero here, fillers carry 0


def test_string_special_cases():
    # prefix pairs separate through the length term (R5)
    strs = [b"ab", b"ab\0", b"", b"\0", b"\0\0\0\0", b"\0\0\0\0\0"]
    ctx, offs = gen.pack_bytes_list(strs)
    t = O.build_bytes(ctx, offs, np.arange(1, 7, dtype=np.uint64), 0)
    _assoc_check(t, strs, np.arange(1, 7), strs + [b"a", b"\0\0", b"ab\0\0"])
    with pytest.raises(O.OracleError) as e:
        c, o = gen.pack_bytes_list([b"hello", b"world", b"hello"])
        O.build_bytes(c, o, np.arange(3, dtype=np.uint64), 0)
    assert e.value.name == "DUPLICATE_KEY"
    with pytest.raises(O.OracleError) as e:
        c, o = gen.pack_bytes_list([b"x" * 70000])
        O.build_bytes(c, o, np.arange(1, dtype=np.uint64), 0)
    assert e.value.name == "TOO_LARGE"


def test_string_fingerprints_distinct_and_deterministic():
    n = 20000
    ctx, offs = gen.string_keys(n)
    strs = gen.string_list(ctx, offs)
    r = O.derive(0, 0, 0, 0)[0]
    fps = [O.fingerprint(s, r) for s in strs[:5000]]
    assert len(set(fps)) == len(fps)
    t1 = O.build_bytes(ctx, offs, gen.u64_values(n), 0)
    # permuting the keys permutes ctx_off but not fp/value/len at each slot
    perm = np.random.default_rng(1).permutation(n)
    p_strs = [strs[i] for i in perm]
    c2, o2 = gen.pack_bytes_list(p_strs)
    t2 = O.build_bytes(c2, o2, gen.u64_values(n)[perm], 0)
    assert t1.dir.tobytes() == t2.dir.tobytes()
    for f in ("fp", "value", "len"):
        assert np.array_equal(t1.slots[f], t2.slots[f])


def test_oracle_from_array_bytes_first_occurrence_wins():
    """from_array for byte keys: each lookup returns the value of the key's
    first occurrence (brute-force scan); distinct inputs give from_array_nodup's
    table; the packed context holds the distinct keys in input order."""
    rng = np.random.default_rng(11)
    words = [b"", b"a", b"ab", b"ab\\0", b"abc", b"hello world", b"x" * 70, b"\\x00\\x01", b"zz"]
    idx = rng.integers(0, len(words), size=60)
    keys = [words[i] for i in idx]
    ctx = np.frombuffer(b"".join(keys), np.uint8)
    offs = np.zeros(len(keys) + 1, np.uint64)
    np.cumsum([len(k) for k in keys], out=offs[1:])
    vals = np.arange(500, 560, dtype=np.uint64)
    t = O.from_array_bytes(ctx, offs, vals, 2)
    distinct = list(dict.fromkeys(keys))
    assert int(t.header["n"]) == len(distinct)
    assert t.ctx.tobytes() == b"".join(distinct)
    qk = words + [b"abcd", b"hello worle"]
    qctx = np.frombuffer(b"".join(qk), np.uint8)
    qoffs = np.zeros(len(qk) + 1, np.uint64)
    np.cumsum([len(k) for k in qk], out=qoffs[1:])
    ov, of = O.lookup_bytes(t, qctx, qoffs)
    for k, v, f in zip(qk, ov.tolist(), of.tolist()):
        first = next((i for i, x in enumerate(keys) if x == k), None)
        assert (f, v) == ((0, 0) if first is None else (1, 500 + first))
    c2, o2 = gen.string_keys(300)
    v2 = gen.u64_values(300)
    a, b = O.from_array_bytes(c2, o2, v2, 1), O.build_bytes(c2, o2, v2, 1)
    assert a.dir.tobytes() == b.dir.tobytes() and a.slots.tobytes() == b.slots.tobytes()
