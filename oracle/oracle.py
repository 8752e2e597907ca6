"""ctypes front-end of the CPU oracle (oracle/fks_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, by __graft_entry__.smoke() and by
bench.py's cpu_baseline / --impl reference legs.  Never imported by the product
package (paper_2508_11443_b200), and it imports nothing from it.

Every function here is argument marshalling around the C oracle; the
arithmetic lives in fks_oracle.c, which cites the paper passage per function.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "fks_oracle.c")
LIB = os.path.join(HERE, "liboracle.so")

STATUS = {
    0: "OK",
    1: "INVALID_ARG",
    2: "EMPTY",
    3: "DUPLICATE_KEY",
    4: "SEED_EXHAUSTED",
    5: "FP_EXHAUSTED",
    6: "TOO_LARGE",
    7: "OOM",
}

HEADER_DTYPE = np.dtype(
    [
        ("magic", "<u4"), ("spec_version", "<u4"), ("key_kind", "<u4"), ("reserved", "<u4"),
        ("n", "<u8"), ("S", "<u8"), ("seed", "<u8"), ("t1", "<u4"), ("t0", "<u4"),
        ("ctx_bytes", "<u8"),
    ]
)
SLOT_U64_DTYPE = np.dtype([("key", "<u8"), ("value", "<u8")])
SLOT_BYTES_DTYPE = np.dtype(
    [("fp", "<u8"), ("value", "<u8"), ("ctx_off", "<u8"), ("len", "<u4"), ("reserved", "<u4")]
)


class OracleError(RuntimeError):
    def __init__(self, code: int):
        super().__init__(f"oracle status {code} ({STATUS.get(code, '?')})")
        self.code = code
        self.name = STATUS.get(code, "?")


def build_lib(force: bool = False) -> str:
    """Compile the oracle with gcc (plain C, -O2)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        tmp = LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=gnu11", "-shared", "-fPIC", "-pthread", "-o", tmp, SRC])
        os.replace(tmp, LIB)
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build_lib()
        L = C.CDLL(LIB)
        u64, u32, p = C.c_uint64, C.c_uint32, C.c_void_p
        L.or_mix64.restype = u64
        L.or_mix64.argtypes = [u64]
        L.or_derive.argtypes = [u64, u32, u64, u32, p]
        L.or_hash.restype = u64
        L.or_hash.argtypes = [p, u64]
        L.or_fingerprint.restype = u64
        L.or_fingerprint.argtypes = [p, u64, u64]
        L.or_hist.argtypes = [u64, p, p, u64, p]
        L.or_presum.argtypes = [p, u64, p]
        L.or_groupby.argtypes = [u64, p, u64, p, p]
        L.or_build_u64.restype = C.c_int
        L.or_build_u64.argtypes = [p, p, u64, u64, C.POINTER(p)]
        L.or_build_bytes.restype = C.c_int
        L.or_build_bytes.argtypes = [p, p, p, u64, u64, C.POINTER(p)]
        L.or_lookup_u64.argtypes = [p, p, u64, p, p]
        L.or_lookup_bytes.argtypes = [p, p, p, u64, p, p]
        L.or_build_u64_shard.restype = C.c_int
        L.or_build_u64_shard.argtypes = [p, p, u64, u64, u64, u64, u32, u64, C.POINTER(p)]
        L.or_table_free.argtypes = [p]
        L.or_table_header.argtypes = [p, p]
        L.or_table_dir.restype = p
        L.or_table_dir.argtypes = [p]
        L.or_table_slots.restype = p
        L.or_table_slots.argtypes = [p]
        L.or_table_ctx.restype = p
        L.or_table_ctx.argtypes = [p]
        L.or_sizeof_header.restype = u64
        L.or_level1_buckets.argtypes = [p, u64, u64, u64, u32, p]
        L.or_build_u64_mt.argtypes = [p, p, u64, u64, C.c_int, C.POINTER(C.c_void_p)]
        L.or_level1_S.restype = u64
        L.or_level1_S.argtypes = [p, u64, u64, u32, p]
        assert L.or_sizeof_header() == HEADER_DTYPE.itemsize
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _u64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint64))


# ------------------------------------------------------------------ scalars

def mix64(x: int) -> int:
    return lib().or_mix64(x)


def derive(seed: int, level: int, bucket: int, attempt: int):
    out = np.zeros(3, np.uint64)
    lib().or_derive(seed, level, bucket, attempt, _ptr(out))
    return tuple(int(v) for v in out)


def hash_(c, x: int) -> int:
    ca = _u64(c)
    return lib().or_hash(_ptr(ca), x)


def fingerprint(s: bytes, r: int) -> int:
    buf = np.frombuffer(s, dtype=np.uint8).copy() if s else np.zeros(1, np.uint8)
    return lib().or_fingerprint(_ptr(buf), len(s), r)


# --------------------------------------------------------------- vocabulary

def hist(nbins: int, is_, vs) -> np.ndarray:
    is_, vs = _u64(is_), _u64(vs)
    out = np.zeros(nbins, np.uint64)
    lib().or_hist(nbins, _ptr(is_), _ptr(vs), len(is_), _ptr(out))
    return out


def presum(x) -> np.ndarray:
    """Exclusive prefix sum; returns n+1 entries (last = total)."""
    x = _u64(x)
    out = np.zeros(len(x) + 1, np.uint64)
    lib().or_presum(_ptr(x), len(x), _ptr(out))
    return out


def groupby(m: int, is_, vs):
    """groupby m is vs -> list of m lists."""
    is_ = _u64(is_)
    start = np.zeros(m + 1, np.uint64)
    items = np.zeros(max(1, len(is_)), np.uint64)
    lib().or_groupby(m, _ptr(is_), len(is_), _ptr(start), _ptr(items))
    return [[vs[int(i)] for i in items[int(start[g]):int(start[g + 1])]] for g in range(m)]


def level1_buckets(keys, n: int, seed: int, t1: int) -> np.ndarray:
    """g k for every key (mod n, the global key count)."""
    keys = _u64(keys)
    out = np.empty(len(keys), np.uint64)
    if len(keys):
        lib().or_level1_buckets(_ptr(keys), len(keys), n, seed, t1, _ptr(out))
    return out


def level1_S(keys, seed: int, t1: int):
    keys = _u64(keys)
    shape = np.zeros(len(keys), np.uint64)
    S = lib().or_level1_S(_ptr(keys), len(keys), seed, t1, _ptr(shape))
    return int(S), shape


# ------------------------------------------------------------------- tables

@dataclass
class Table:
    handle: int
    header: np.ndarray  # structured scalar (HEADER_DTYPE)
    dir: np.ndarray  # uint64[n]
    slots: np.ndarray  # structured [S]
    ctx: np.ndarray | None

    @property
    def n(self):
        return int(self.header["n"])

    @property
    def S(self):
        return int(self.header["S"])

    def header_bytes(self) -> bytes:
        return self.header.tobytes()

    def __del__(self):
        try:
            if self.handle:
                lib().or_table_free(self.handle)
                self.handle = 0
        except Exception:
            pass


def _wrap(h, kind: int) -> Table:
    L = lib()
    hdr = np.zeros(1, HEADER_DTYPE)
    L.or_table_header(h, _ptr(hdr))
    n, S = int(hdr["n"][0]), int(hdr["S"][0])
    d = np.ctypeslib.as_array(C.cast(L.or_table_dir(h), C.POINTER(C.c_uint64)), shape=(n,)).copy()
    sd = SLOT_U64_DTYPE if kind == 0 else SLOT_BYTES_DTYPE
    raw = C.cast(L.or_table_slots(h), C.POINTER(C.c_uint8))
    sl = np.ctypeslib.as_array(raw, shape=(S * sd.itemsize,)).copy().view(sd)
    ctx = None
    if kind == 1:
        cb = int(hdr["ctx_bytes"][0])
        if cb:
            ctx = np.ctypeslib.as_array(C.cast(L.or_table_ctx(h), C.POINTER(C.c_uint8)), shape=(cb,)).copy()
        else:
            ctx = np.zeros(0, np.uint8)
    return Table(h, hdr[0], d, sl, ctx)


def build_u64(keys, vals, seed: int = 0) -> Table:
    keys, vals = _u64(keys), _u64(vals)
    assert len(keys) == len(vals)
    h = C.c_void_p()
    st = lib().or_build_u64(_ptr(keys) if len(keys) else None, _ptr(vals) if len(vals) else None,
                            len(keys), seed, C.byref(h))
    if st != 0:
        raise OracleError(st)
    return _wrap(h.value, 0)


def build_u64_mt(keys, vals, seed: int = 0, threads: int = 0) -> Table:
    """The T-thread oracle (bucket ranges per thread): the same
    table as build_u64; CPU-baseline timing only."""
    keys, vals = _u64(keys), _u64(vals)
    T = threads or os.cpu_count() or 1
    h = C.c_void_p()
    st = lib().or_build_u64_mt(_ptr(keys), _ptr(vals), len(keys), seed, T, C.byref(h))
    if st != 0:
        raise OracleError(st)
    return _wrap(h.value, 0)


def from_array_u64(keys, vals, seed: int = 0) -> Table:
    """from_array: duplicates are
    allowed, the first occurrence (lowest input index) of every key keeps its
    value, and the map is the one from_array_nodup builds from those distinct
    keys (the table is a function of the key set, R13, so their order does not
    matter).  Plain definition: numpy's unique with return_index gives the
    first occurrence of each key."""
    keys, vals = _u64(keys), _u64(vals)
    assert len(keys) == len(vals)
    if len(keys) == 0:
        raise OracleError(2)
    _, first = np.unique(keys, return_index=True)
    first = np.sort(first)
    return build_u64(keys[first], vals[first], seed)


def build_u64_shard(keys, vals, n_global: int, b_lo: int, b_hi: int, t1: int, seed: int = 0):
    """(status_name, Table) of one bucket-range shard (fks_oracle.c or_build_u64_shard)."""
    keys, vals = _u64(keys), _u64(vals)
    h = C.c_void_p()
    kb = keys if len(keys) else np.zeros(1, np.uint64)
    vb = vals if len(vals) else np.zeros(1, np.uint64)
    st = lib().or_build_u64_shard(_ptr(kb), _ptr(vb), len(keys), n_global, b_lo, b_hi, t1, seed, C.byref(h))
    if not h.value:
        raise OracleError(st)
    t = _wrap(h.value, 0)
    if st != 0:
        t.slots = t.slots[:0]
    return STATUS[st], t


def lookup_u64(t: Table, q):
    q = _u64(q)
    vals = np.zeros(len(q), np.uint64)
    found = np.zeros(len(q), np.uint8)
    if len(q):
        lib().or_lookup_u64(t.handle, _ptr(q), len(q), _ptr(vals), _ptr(found))
    return vals, found


def build_bytes(ctx, offsets, vals, seed: int = 0) -> Table:
    ctx = np.ascontiguousarray(np.asarray(ctx, dtype=np.uint8))
    offsets, vals = _u64(offsets), _u64(vals)
    n = len(offsets) - 1
    assert len(vals) == n
    cbuf = ctx if len(ctx) else np.zeros(1, np.uint8)
    h = C.c_void_p()
    st = lib().or_build_bytes(_ptr(cbuf), _ptr(offsets), _ptr(vals) if n else None, n, seed, C.byref(h))
    if st != 0:
        raise OracleError(st)
    return _wrap(h.value, 1)


def from_array_bytes(ctx, offsets, vals, seed: int = 0) -> Table:
    """from_array for byte-string keys: the first
    occurrence of every key (by content) keeps its value; the distinct keys,
    packed in input order into a new context, go to from_array_nodup.  Plain
    definition: a Python dict over the key bytes."""
    ctx = np.ascontiguousarray(np.asarray(ctx, dtype=np.uint8))
    offsets, vals = _u64(offsets), _u64(vals)
    n = len(offsets) - 1
    if n <= 0:
        raise OracleError(2)
    seen, keep = set(), []
    for i in range(n):
        k = ctx[int(offsets[i]):int(offsets[i + 1])].tobytes()
        if k not in seen:
            seen.add(k)
            keep.append(i)
    parts = [ctx[int(offsets[i]):int(offsets[i + 1])] for i in keep]
    lens = np.array([len(x) for x in parts], dtype=np.uint64)
    noffs = np.zeros(len(keep) + 1, np.uint64)
    np.cumsum(lens, out=noffs[1:])
    nctx = np.concatenate(parts) if int(noffs[-1]) else np.zeros(0, np.uint8)
    return build_bytes(nctx, noffs, vals[np.array(keep, dtype=np.int64)], seed)


def lookup_bytes(t: Table, qctx, qoffsets):
    qctx = np.ascontiguousarray(np.asarray(qctx, dtype=np.uint8))
    qoffsets = _u64(qoffsets)
    nq = len(qoffsets) - 1
    vals = np.zeros(nq, np.uint64)
    found = np.zeros(nq, np.uint8)
    cbuf = qctx if len(qctx) else np.zeros(1, np.uint8)
    if nq:
        lib().or_lookup_bytes(t.handle, _ptr(cbuf), _ptr(qoffsets), nq, _ptr(vals), _ptr(found))
    return vals, found


def decode_dir(d: np.ndarray):
    d = _u64(d)
    soff = d & np.uint64((1 << 40) - 1)
    s = (d >> np.uint64(40)) & np.uint64(0xFFFF)
    t = d >> np.uint64(56)
    return soff, s, t
