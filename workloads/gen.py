"""Seeded synthetic workloads shaped like the paper's benchmark inputs.

PAPER.md:903-906 (§4 Benchmarks): "inserting n keys of two types (64-bit
integers and strings of 5--25 characters) ... The keys are uniformly
distributed and generated such that there are no duplicates."  The shapes used
here are the ones BASELINE.json names (u64 keys, 4-64 byte strings, 50% hit
lookups); the recipe is SURVEY.md §8(d) and is restated in DESIGN.md §3.

This module is shared by the tests, the oracle harness and bench.py. It holds
NONE of the method's arithmetic (no hash family, no seed schedule, no range
reduction): only a counter-based key stream.  The stream uses its own copy of
the splitmix64 output function; the method's constant schedule (R6)
is implemented separately by the oracle and by the CUDA library.

    stream(s, i) = splitmix_out(splitmix_out(s ^ 0xA0761D6478BD642F) + GAMMA*(i+1))

is a bijection in i (splitmix_out is a bijection on u64 and i -> GAMMA*(i+1) is
one too), so keys stream(SEED_K, i) are pairwise distinct by construction.

Workloads:
  u64 members    key_i = stream(SEED_K, i), i in [0, n);  value_i = i
  u64 absent     key_i for i in [n, 2n)   (disjoint from the members)
  queries (50%)  r = stream(SEED_Q, j); idx = (r mod 2^63) mod n;
                 r>>63 == 0 -> member key_idx, else absent key_{n+idx}
  strings        len_i = 4 + stream(SEED_L, i) mod 61        (uniform 4..64)
                 bytes[0:4]  = little-endian u32 fmix32(i)   (distinct for i < 2^32)
                 bytes[4:len] = little-endian bytes of stream(SEED_B, 8i+w), w=0..7
"""
from __future__ import annotations

import numpy as np

SEED_K, SEED_Q, SEED_L, SEED_B = 1, 2, 3, 4
GAMMA = 0x9E3779B97F4A7C15
STREAM_SALT = 0xA0761D6478BD642F
_M64 = (1 << 64) - 1


def _out_py(z: int) -> int:
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def _out_np(z: np.ndarray) -> np.ndarray:
    z = z.astype(np.uint64, copy=True)
    with np.errstate(over="ignore"):
        z ^= z >> np.uint64(30)
        z *= np.uint64(0xBF58476D1CE4E5B9)
        z ^= z >> np.uint64(27)
        z *= np.uint64(0x94D049BB133111EB)
        z ^= z >> np.uint64(31)
    return z


def stream_start(s: int) -> int:
    return _out_py((s ^ STREAM_SALT) & _M64)


def stream(s: int, idx) -> np.ndarray:
    """stream(s, i) for an array (or range) of indices i; returns uint64."""
    idx = np.asarray(idx, dtype=np.uint64)
    base = np.uint64(stream_start(s))
    with np.errstate(over="ignore"):
        x = base + np.uint64(GAMMA) * (idx + np.uint64(1))
    return _out_np(x)


def stream_py(s: int, i: int) -> int:
    return _out_py((stream_start(s) + GAMMA * (i + 1)) & _M64)


def u64_keys(n: int, lo: int = 0, seed_k: int = SEED_K) -> np.ndarray:
    """Member keys key_i, i in [lo, lo+n)."""
    return stream(seed_k, np.arange(lo, lo + n, dtype=np.uint64))


def u64_values(n: int, lo: int = 0) -> np.ndarray:
    return np.arange(lo, lo + n, dtype=np.uint64)


def query_plan(n: int, nq: int, lo: int = 0, seed_q: int = SEED_Q):
    """For queries j in [lo, lo+nq): (is_member bool[nq], idx uint64[nq]).

    The query is key_idx when is_member, else the absent key key_{n+idx}."""
    r = stream(seed_q, np.arange(lo, lo + nq, dtype=np.uint64))
    member = (r >> np.uint64(63)) == 0
    idx = (r & np.uint64((1 << 63) - 1)) % np.uint64(n)
    return member, idx


def u64_queries(n: int, nq: int, lo: int = 0, seed_k: int = SEED_K, seed_q: int = SEED_Q):
    """Returns (queries uint64[nq], expected_found bool[nq], expected_value uint64[nq])."""
    member, idx = query_plan(n, nq, lo, seed_q)
    kidx = np.where(member, idx, idx + np.uint64(n))
    q = stream(seed_k, kidx)
    vals = np.where(member, idx, np.uint64(0)).astype(np.uint64)
    return q, member, vals


# ---------------------------------------------------------------- strings

def fmix32(h: np.ndarray) -> np.ndarray:
    h = np.asarray(h, dtype=np.uint64) & np.uint64(0xFFFFFFFF)
    with np.errstate(over="ignore"):
        h ^= h >> np.uint64(16)
        h = (h * np.uint64(0x85EBCA6B)) & np.uint64(0xFFFFFFFF)
        h ^= h >> np.uint64(13)
        h = (h * np.uint64(0xC2B2AE35)) & np.uint64(0xFFFFFFFF)
        h ^= h >> np.uint64(16)
    return h


def string_lengths(idx: np.ndarray, seed_l: int = SEED_L, lens_range=(4, 64)) -> np.ndarray:
    """len = lmin + stream(SEED_L, id) mod (lmax - lmin + 1): 4..64 by default, 5..25 for the
    paper's Table 1 shape."""
    lmin, lmax = lens_range
    return (np.uint64(lmin) + stream(seed_l, idx) % np.uint64(lmax - lmin + 1)).astype(np.int64)


def string_rows(idx: np.ndarray, seed_b: int = SEED_B) -> np.ndarray:
    """Full 68-byte rows (4 prefix bytes + 64 stream bytes) for string ids idx."""
    idx = np.asarray(idx, dtype=np.uint64)
    m = idx.shape[0]
    rows = np.empty((m, 68), dtype=np.uint8)
    rows[:, 0:4] = fmix32(idx).astype("<u4").view(np.uint8).reshape(m, 4)
    w = stream(seed_b, (idx[:, None] * np.uint64(8) + np.arange(8, dtype=np.uint64)[None, :]).reshape(-1))
    rows[:, 4:68] = w.astype("<u8").view(np.uint8).reshape(m, 64)
    return rows


def pack_strings(idx: np.ndarray, seed_l: int = SEED_L, seed_b: int = SEED_B, lens_range=(4, 64)):
    """Flat context + CSR offsets (n+1, uint64) for the strings with ids idx."""
    idx = np.asarray(idx, dtype=np.uint64)
    lens = string_lengths(idx, seed_l, lens_range)
    offs = np.zeros(idx.shape[0] + 1, dtype=np.uint64)
    np.cumsum(lens, out=offs[1:])
    total = int(offs[-1])
    ctx = np.empty(total, dtype=np.uint8)
    chunk = 1 << 20
    for c0 in range(0, idx.shape[0], chunk):
        c1 = min(idx.shape[0], c0 + chunk)
        rows = string_rows(idx[c0:c1], seed_b)
        l = lens[c0:c1]
        mask = np.arange(68)[None, :] < l[:, None]
        ctx[int(offs[c0]):int(offs[c1])] = rows[mask]
    return ctx, offs


def string_keys(n: int, lo: int = 0):
    """Member strings i in [lo, lo+n): (ctx uint8[], offsets uint64[n+1])."""
    return pack_strings(np.arange(lo, lo + n, dtype=np.uint64))


def string_queries(n: int, nq: int, lo: int = 0):
    """Needles in their own context: (ctx, offsets, found, value)."""
    member, idx = query_plan(n, nq, lo)
    sid = np.where(member, idx, idx + np.uint64(n))
    ctx, offs = pack_strings(sid)
    vals = np.where(member, idx, np.uint64(0)).astype(np.uint64)
    return ctx, offs, member, vals


def string_list(ctx: np.ndarray, offs: np.ndarray):
    return [bytes(ctx[int(offs[i]):int(offs[i + 1])]) for i in range(len(offs) - 1)]


def pack_bytes_list(strs):
    """Pack a python list of bytes objects into (ctx, offsets)."""
    offs = np.zeros(len(strs) + 1, dtype=np.uint64)
    np.cumsum([len(s) for s in strs], out=offs[1:])
    ctx = np.frombuffer(b"".join(strs), dtype=np.uint8).copy() if strs else np.zeros(0, np.uint8)
    return ctx, offs
