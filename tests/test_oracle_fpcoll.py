"""Pin of the fingerprint-collision redraw (not gpu): SURVEY §8(c) step 5 /
DESIGN.md R5 — the paper elides the sequence hash (§3.3), so
byte keys are hashed through a 61-bit fingerprint, and two different keys with
equal fingerprints make the build redraw the fingerprint point (t0 + 1).

The fixture (tests/golden/fp_collision_seed0.txt, scripts/make_fp_collision.py)
holds a pair of 32-byte keys whose fingerprints collide at (seed 0, t0 = 0),
found by lattice reduction.  Pinned here without the oracle's own fingerprint:
  * the collision by the closed form fp = sum_i w_i r^(m-i) + len (mod P) in
    Python integers, and its absence at t0 = 1;
  * the oracle's table for every fixture set equals a brute-force
    reconstruction at t0 = 1 straight from PAPER.md §2.2-§2.3 (first t1 with
    S <= 4n, first injective t per bucket, fillers = the lowest-slot member),
    built on those closed-form fingerprints and the pinned derive/hash.
"""
import os

import numpy as np
import pytest

from oracle import oracle as O
from workloads import gen

P = (1 << 61) - 1
GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "fp_collision_seed0.txt")


def load_fixture():
    d = {"sets": {}}
    with open(GOLDEN) as f:
        for line in f:
            if not line.strip() or line.startswith("#"):
                continue
            parts = line.split()
            if parts[0] == "r0":
                d["r0"] = int(parts[1], 16)
            elif parts[0] == "pair":
                d["pair"] = (bytes.fromhex(parts[1]), bytes.fromhex(parts[2]))
            elif parts[0] == "set":
                d["sets"][parts[1]] = [bytes.fromhex(x) for x in parts[2].split(",")]
    return d


def fp_closed_form(s: bytes, r: int) -> int:
    """R5 unrolled: acc = sum_{i<m} w_i r^(m-i) over zero-padded LE u32 words."""
    m = (len(s) + 3) // 4
    pad = s + b"\0" * (4 * m - len(s))
    acc = sum(int.from_bytes(pad[4 * i:4 * i + 4], "little") * pow(r, m - i, P) for i in range(m))
    return (acc + len(s)) % P


def reference_bytes_table(strs, vals, seed, r):
    """Brute-force byte-key table for fingerprint point r (closed-form fps)."""
    n = len(strs)
    fps = [fp_closed_form(s, r) for s in strs]
    offs_ctx = np.concatenate([[0], np.cumsum([len(s) for s in strs])]).astype(np.int64)
    for t1 in range(16):
        c1 = O.derive(seed, 1, 0, t1)
        g = [O.hash_(c1, f) % n for f in fps]
        shape = [g.count(b) for b in range(n)]
        if sum(s * s for s in shape) <= 4 * n:
            break
    else:
        return None
    offs, acc = [], 0
    for s in shape:
        offs.append(acc)
        acc += s * s
    S = acc
    dir_, slots = [], [None] * S
    for b in range(n):
        members = [i for i in range(n) if g[i] == b]
        s = len(members)
        if s == 0:
            dir_.append(offs[b])
            continue
        if s == 1:
            t, pos = 0, [0]
        else:
            assert len({fps[i] for i in members}) == s  # (no collision left at this r)
            for t in range(256):
                cs = O.derive(seed, 2, b, t)
                pos = [O.hash_(cs, fps[i]) % (s * s) for i in members]
                if len(set(pos)) == s:
                    break
        for i, p in zip(members, pos):
            slots[offs[b] + p] = (fps[i], int(vals[i]), int(offs_ctx[i]), len(strs[i]))
        low = members[pos.index(min(pos))]
        for j in range(s * s):
            if slots[offs[b] + j] is None:
                slots[offs[b] + j] = (fps[low], 0, int(offs_ctx[low]), len(strs[low]))
        dir_.append(offs[b] | (s << 40) | (t << 56))
    return t1, S, dir_, slots


def test_fixture_pair_collides_in_closed_form():
    fx = load_fixture()
    a, b = fx["pair"]
    r0 = O.derive(0, 0, 0, 0)[0]
    assert r0 == fx["r0"] == 0x1D2912234C98DAE3  # SURVEY §8(c) cross-check value
    assert a != b and len(a) == len(b) == 32
    assert fp_closed_form(a, r0) == fp_closed_form(b, r0)
    r1 = O.derive(0, 0, 0, 1)[0]
    assert fp_closed_form(a, r1) != fp_closed_form(b, r1)
    # the oracle's fingerprint agrees with the closed form on both points
    for r in (r0, r1):
        assert O.fingerprint(a, r) == fp_closed_form(a, r) and O.fingerprint(b, r) == fp_closed_form(b, r)


@pytest.mark.parametrize("name", ["s2", "s3", "s5", "s9"])
def test_oracle_redraws_t0_on_fingerprint_collision(name):
    fx = load_fixture()
    strs = fx["sets"][name]
    n = len(strs)
    a, b = fx["pair"]
    assert a in strs and b in strs and len(set(strs)) == n
    r0 = O.derive(0, 0, 0, 0)[0]
    # the fixture's intent: at t0 = 0 (t1 = 0 accepted) the pair's bucket has K keys
    fps0 = [fp_closed_form(s, r0) for s in strs]
    c1 = O.derive(0, 1, 0, 0)
    g = [O.hash_(c1, f) % n for f in fps0]
    assert sum(g.count(x) ** 2 for x in range(n)) <= 4 * n
    assert g.count(g[strs.index(a)]) == int(name[1:])
    ctx, offs = gen.pack_bytes_list(strs)
    vals = np.arange(100, 100 + n, dtype=np.uint64)
    t = O.build_bytes(ctx, offs, vals, 0)
    assert int(t.header["t0"]) == 1  # one redraw: r1 separates the pair
    r1 = O.derive(0, 0, 0, 1)[0]
    ref = reference_bytes_table(strs, vals, 0, r1)
    t1, S, d, sl = ref
    assert int(t.header["t1"]) == t1 and t.S == S
    assert [int(x) for x in t.dir] == d
    got = [(int(x["fp"]), int(x["value"]), int(x["ctx_off"]), int(x["len"])) for x in t.slots]
    assert got == sl
    assert all(int(x["reserved"]) == 0 for x in t.slots)
    v, f = O.lookup_bytes(t, ctx, offs)
    assert list(f) == [1] * n and [int(x) for x in v] == list(range(100, 100 + n))
