"""Pins for the oracle's primitives (not gpu).

Each test checks the oracle against something other than the oracle's own
formula: published generator outputs, worked examples printed in the paper,
closed forms and algebraic invariants that a dropped term / wrong shift /
transposed operand would break.  See DESIGN.md §5 for the pin table.
"""
import os
import random

import numpy as np
import pytest

from oracle import oracle as O

P = (1 << 61) - 1
M64 = (1 << 64) - 1
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
GAMMA = 0x9E3779B97F4A7C15
SALT = 0xD6E8FEB86659FD93


def _golden_hex(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return [int(l.strip(), 16) for l in f if l.strip() and not l.startswith("#")]


# ------------------------------------------------------------ mix64 / derive

def test_mix64_matches_published_splitmix64_seed0():
    # splitmix64 with state 0: k-th output = mix64(GAMMA*k)
    pub = _golden_hex("splitmix64_seed0.txt")
    for k, v in enumerate(pub, start=1):
        assert O.mix64((GAMMA * k) & M64) == v
    assert O.mix64(0) == 0


def _unxorshift(z, s):
    x = z
    for _ in range(64 // s + 1):
        x = z ^ (x >> s)
    return x


def _unmix64(z):
    """Textbook inverse of the splitmix64 output function (bijection on u64)."""
    z = _unxorshift(z, 31)
    z = (z * pow(0x94D049BB133111EB, -1, 1 << 64)) & M64
    z = _unxorshift(z, 27)
    z = (z * pow(0xBF58476D1CE4E5B9, -1, 1 << 64)) & M64
    z = _unxorshift(z, 30)
    return z


@pytest.mark.parametrize("level,bucket,attempt", [(0, 0, 0), (1, 0, 3), (2, 7, 3), (2, (1 << 40) + 5, 255)])
def test_derive_reduces_to_published_splitmix_stream(level, bucket, attempt):
    """R6: with the seed chosen so that u = 0, the three constants are the
    seed-0 splitmix64 outputs >> 3.  Pins the salt, the counter layout
    level<<60 | bucket<<8 | attempt, the output indices j+1 and the >>3."""
    ctr = (level << 60) | (bucket << 8) | attempt
    assert O.mix64(_unmix64(ctr)) == ctr
    seed = _unmix64(ctr) ^ SALT
    pub = _golden_hex("splitmix64_seed0.txt")
    a1, a2, b = O.derive(seed, level, bucket, attempt)
    assert (a1, a2, b) == (pub[0] >> 3, pub[1] >> 3, pub[2] >> 3)


def test_derive_ranges_and_distinctness():
    seen = set()
    for seed in range(3):
        for level in (0, 1, 2):
            for bucket in range(20):
                for t in range(4):
                    a1, a2, b = O.derive(seed, level, bucket, t)
                    assert 1 <= a1 < P and 1 <= a2 < P and 0 <= b < P
                    seen.add((a1, a2, b))
                    assert O.derive(seed, level, bucket, t) == (a1, a2, b)
    assert len(seen) == 3 * 3 * 20 * 4


# ------------------------------------------------------------------- hash (R4)

def test_hash_special_cases():
    x = 0x0123456789ABCDEF
    lo, hi = x & 0xFFFFFFFF, x >> 32
    assert O.hash_((1, 0, 0), x) == lo
    assert O.hash_((0, 1, 0), x) == hi
    assert O.hash_((1, 1, 0), x) == lo + hi
    assert O.hash_((5, 7, 11), 0) == 11
    # (-1)(2^32-1) + (-1)(2^32-1) + (-1)  mod P  = P - 2^33 + 1
    assert O.hash_((P - 1, P - 1, P - 1), M64) == P - (1 << 33) + 1
    # b is reduced too
    assert O.hash_((1, 1, P), 0) == 0


def test_hash_limb_linearity():
    rnd = random.Random(7)
    for _ in range(200):
        c = (rnd.randrange(1, P), rnd.randrange(1, P), rnd.randrange(P))
        x = rnd.getrandbits(64)
        if (x & 0xFFFFFFFF) != 0xFFFFFFFF:
            assert (O.hash_(c, x + 1) - O.hash_(c, x)) % P == c[0]
        if (x >> 32) != 0xFFFFFFFF:
            assert (O.hash_(c, x + (1 << 32)) - O.hash_(c, x)) % P == c[1]
        assert 0 <= O.hash_(c, x) < P


def test_hash_separates_x_and_x_plus_P():
    """R4 rejects (a*(x mod P)+b) because x, x+P always collide."""
    rnd = random.Random(3)
    for _ in range(50):
        c = (rnd.randrange(1, P), rnd.randrange(1, P), rnd.randrange(P))
        x = rnd.randrange(1 << 32)
        assert O.hash_(c, x) != O.hash_(c, x + P)


def test_hash_universality_statistics():
    """Pr[h(x)=h(y) mod 2^10] over random constants ~ 2^-10 (universal family)."""
    rnd = random.Random(11)
    trials, coll = 20000, 0
    x, y = rnd.getrandbits(64), rnd.getrandbits(64)
    for i in range(trials):
        c = O.derive(99, 2, i, 0)
        coll += (O.hash_(c, x) % 1024) == (O.hash_(c, y) % 1024)
    mu = trials / 1024
    assert abs(coll - mu) < 6 * mu ** 0.5


# ------------------------------------------------------------ fingerprint (R5)

def _words(s: bytes):
    m = (len(s) + 3) // 4
    padded = s + b"\0" * (4 * m - len(s))
    return [int.from_bytes(padded[4 * i:4 * i + 4], "little") for i in range(m)]


def test_fingerprint_closed_forms():
    rnd = random.Random(5)
    r = O.derive(0, 0, 0, 0)[0]
    assert O.fingerprint(b"", r) == 0
    assert O.fingerprint(b"a", r) == (0x61 * r + 1) % P
    assert O.fingerprint(b"abcd", 1) == (int.from_bytes(b"abcd", "little") + 4) % P
    for _ in range(100):
        s = bytes(rnd.getrandbits(8) for _ in range(rnd.randrange(0, 70)))
        # r = 0: every word is multiplied away, only the length survives
        assert O.fingerprint(s, 0) == len(s)
        # r = 1: sum of little-endian words plus length
        assert O.fingerprint(s, 1) == (sum(_words(s)) + len(s)) % P
        # polynomial form sum_i w_i r^(m-i) + len, evaluated without Horner
        w = _words(s)
        m = len(w)
        poly = sum(wi * pow(r, m - i, P) for i, wi in enumerate(w))
        assert O.fingerprint(s, r) == (poly + len(s)) % P


def test_fingerprint_prefix_pairs_differ_by_len_term():
    r = O.derive(0, 0, 0, 0)[0]
    for s in [b"ab", b"abcde", b"x" * 62]:
        if len(s) % 4:
            assert (O.fingerprint(s + b"\0", r) - O.fingerprint(s, r)) % P == 1


# ---------------------------------------------------------- Fig. 1 vocabulary

def test_groupby_paper_example():
    # groupby 4 [2,0,2] [x,y,z] = [[y],[],[x,z],[]]
    assert O.groupby(4, [2, 0, 2], ["x", "y", "z"]) == [["y"], [], ["x", "z"], []]


def test_hist_definition():
    # like scatter but duplicate indices are summed
    assert list(O.hist(3, [0, 2, 0], [5, 6, 7])) == [12, 0, 6]
    assert list(O.hist(4, [1, 1, 1], [1, 1, 1])) == [0, 3, 0, 0]


def test_presum_exclusive():
    # R2: exclusive; offset of bucket 0 is 0 (otherwise property 1, fails)
    assert list(O.presum([3, 1, 2])) == [0, 3, 4, 6]
    x = np.random.default_rng(0).integers(0, 9, 1000)
    p = O.presum(x)
    assert np.all(p[:-1] + x.astype(np.uint64) == p[1:])
