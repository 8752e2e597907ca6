"""Write tests/golden/fp_collision_seed0.txt: byte keys whose R5 fingerprints
collide at (table seed 0, t0 = 0), so that both the oracle and the CUDA path
must take the fingerprint redraw of SURVEY §8(c) step 5 (R5; the
sequence hash itself is elided by PAPER.md:719-722, §3.3).

Construction.  For two keys of the same length L = 4m, the R5 fingerprint is
fp = sum_{i<m} w_i r^(m-i) + L (mod P), w_i the little-endian u32 words, so two
keys collide iff the word difference d = w - w' satisfies
sum_i d_i r^(m-i) == 0 (mod P).  Those d form a lattice of determinant P in
Z^m; LLL (exact rational arithmetic, below) finds a vector with entries of
about P^(1/m), which is added to random base words kept inside [0, 2^32).

Only oracle/ is called (for r = a1 of derive(0,0,0,0), the level-1 constants
and the space bound); nothing here comes from the CUDA path.

Sets written (values are the key's index; keys in the listed order):
  s2   the pair alone (n = 2): one level-1 bucket of 2 keys at t0 = 0
  sK   the pair plus K-2 keys of the same level-1 bucket at (t0 = 0, t1 = 0)
       among n - K keys in other buckets, for K = 3, 5, 9 (the GPU's
       thread-per-bucket round 0, queued rounds and warp-per-bucket search)
"""
from __future__ import annotations

import os
import sys
from fractions import Fraction

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

P = (1 << 61) - 1
OUT = os.path.join(ROOT, "tests", "golden", "fp_collision_seed0.txt")


def lll(B, delta=Fraction(3, 4)):
    """Textbook LLL (Lenstra-Lenstra-Lovasz) on integer row vectors."""
    B = [list(map(int, b)) for b in B]
    n = len(B)

    def dot(u, v):
        return sum(a * b for a, b in zip(u, v))

    def gso():
        Bs, mu = [], [[Fraction(0)] * n for _ in range(n)]
        for i in range(n):
            v = [Fraction(x) for x in B[i]]
            for j in range(i):
                mu[i][j] = Fraction(dot(B[i], Bs[j])) / dot(Bs[j], Bs[j]) if dot(Bs[j], Bs[j]) else Fraction(0)
                v = [a - mu[i][j] * b for a, b in zip(v, Bs[j])]
            Bs.append(v)
        return Bs, mu

    Bs, mu = gso()
    k = 1
    while k < n:
        for j in range(k - 1, -1, -1):
            q = round(mu[k][j])
            if q:
                B[k] = [a - q * b for a, b in zip(B[k], B[j])]
                Bs, mu = gso()
        if dot(Bs[k], Bs[k]) >= (delta - mu[k][k - 1] ** 2) * dot(Bs[k - 1], Bs[k - 1]):
            k += 1
        else:
            B[k], B[k - 1] = B[k - 1], B[k]
            Bs, mu = gso()
            k = max(k - 1, 1)
    return B


def words_to_bytes(w):
    return b"".join(int(x).to_bytes(4, "little") for x in w)


def collision_pair(r: int, m: int, rng) -> tuple[bytes, bytes]:
    c = [pow(r, m - i, P) for i in range(m)]  # coefficient of word i
    inv = pow(c[m - 1], P - 2, P)
    basis = []
    for i in range(m - 1):
        v = [0] * m
        v[i] = 1
        v[m - 1] = (-c[i] * inv) % P
        basis.append(v)
    basis.append([0] * (m - 1) + [P])
    red = lll(basis)
    d = min((v for v in red if any(v)), key=lambda v: max(abs(x) for x in v))
    assert sum(di * ci for di, ci in zip(d, c)) % P == 0
    lim = max(abs(x) for x in d)
    assert lim < 1 << 20
    w = [int(x) for x in rng.integers(lim, (1 << 32) - lim, size=m)]
    w2 = [a + b for a, b in zip(w, d)]
    return words_to_bytes(w), words_to_bytes(w2)


def main():
    rng = np.random.default_rng(20250815)
    r0 = O.derive(0, 0, 0, 0)[0]
    a, b = collision_pair(r0, 8, rng)  # 32-byte keys
    assert a != b and O.fingerprint(a, r0) == O.fingerprint(b, r0)
    lines = [
        "# Byte keys with equal R5 fingerprints at table seed 0, t0 = 0 (written by",
        "# scripts/make_fp_collision.py from oracle/ only; see its docstring).",
        "# PAPER.md:719-722 (sequence hash elided) -> DESIGN.md R5; SURVEY §8(c) step 5.",
        f"r0 {r0:016x}",
        f"pair {a.hex()} {b.hex()}",
        f"set s2 {a.hex()},{b.hex()}",
    ]
    c1 = O.derive(0, 1, 0, 0)
    for K, n in ((3, 40), (5, 64), (9, 96)):
        fpa = O.fingerprint(a, r0)
        tgt = O.hash_(c1, fpa) % n
        same, other = [], []
        while len(same) < K - 2 or len(other) < n - K:
            L = int(rng.integers(4, 65))
            s = rng.integers(0, 256, size=L, dtype=np.uint8).tobytes()
            bk = O.hash_(c1, O.fingerprint(s, r0)) % n
            if bk == tgt and len(same) < K - 2:
                same.append(s)
            elif bk != tgt and len(other) < n - K:
                other.append(s)
        keys = [a, b] + same + other
        order = rng.permutation(len(keys))
        keys = [keys[i] for i in order]
        fps = np.array([O.fingerprint(s, r0) for s in keys], np.uint64)
        S = O.level1_S(fps, 0, 0)[0]
        assert S <= 4 * n, (K, S)  # t1 = 0 holds at t0 = 0: the pair's bucket has K keys
        lines.append(f"set s{K} " + ",".join(s.hex() for s in keys))
    with open(OUT, "w") as f:
        f.write("\n".join(lines) + "\n")
    print("wrote", OUT)


if __name__ == "__main__":
    main()
