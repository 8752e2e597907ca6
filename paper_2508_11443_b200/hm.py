"""Thin ctypes binding of libhm.so (include/hm.h) — argument marshalling only.

Every step of the hot path runs in the CUDA kernels behind the C-ABI; this
module converts torch tensors / numpy arrays into pointers and sizes, passes
the current CUDA stream, and turns statuses into exceptions.  There is no CPU
fallback: if libhm.so is missing or the device is not a B200 the calls raise.

Names follow include/hm.h: build_u64 / build_bytes (from_array_nodup,
PAPER.md:608-609), lookup / lookup_bytes, free.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HM_LIB_PATH") or os.path.join(PKG, "libhm.so")  # override: debug builds only

STATUS = {
    0: "OK", 1: "INVALID_ARG", 2: "EMPTY", 3: "DUPLICATE_KEY", 4: "SEED_EXHAUSTED",
    5: "FP_EXHAUSTED", 6: "TOO_LARGE", 7: "OOM", 8: "CUDA", 9: "NCCL", 10: "NO_DEVICE",
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


class HMError(RuntimeError):
    def __init__(self, code: int, detail: str = ""):
        self.code = code
        self.name = STATUS.get(code, "?")
        super().__init__(f"hm status {code} ({self.name}){': ' + detail if detail else ''}")


ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)
FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)


class _Opts(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("log2_bp", C.c_uint32), ("flags", C.c_uint32),
                ("alloc", ALLOC_FN), ("free", FREE_FN), ("alloc_ctx", C.c_void_p)]


class _Header(C.Structure):
    _fields_ = [(n, C.c_uint32 if d.kind == "u" and d.itemsize == 4 else C.c_uint64)
                for n, (d, _) in HEADER_DTYPE.fields.items()]


_lib = None


def lib():
    """Load libhm.so; raises if it has not been built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        p, u64, u32, i32 = C.c_void_p, C.c_uint64, C.c_uint32, C.c_int
        L.hm_build_u64.argtypes = [p, p, u64, C.POINTER(_Opts), p, C.POINTER(p)]
        L.hm_build_bytes.argtypes = [p, p, p, u64, C.POINTER(_Opts), p, C.POINTER(p)]
        L.hm_lookup_u64.argtypes = [p, p, u64, p, p, p]
        L.hm_lookup_bytes.argtypes = [p, p, p, u64, p, p, p]
        L.hm_free.argtypes = [p]
        L.hm_free.restype = None
        L.hm_info.argtypes = [p, C.POINTER(_Header)]
        L.hm_export.argtypes = [p, p, p, p]
        L.hm_status_str.restype = C.c_char_p
        L.hm_status_str.argtypes = [i32]
        L.hm_last_error.restype = C.c_char_p
        L.hm_version.restype = C.c_char_p
        L.hm_kernel_launches.restype = C.c_uint64
        L.hm_release_workspace.restype = C.c_int
        L.hm_profile_enable.argtypes = [C.c_int]
        L.hm_profile_enable.restype = None
        L.hm_profile_read.argtypes = [C.c_void_p, C.c_int]
        L.hm_profile_read.restype = C.c_int
        L.hm_route_u64.argtypes = [p, p, u64, u64, u64, u32, i32, p, p, p, p]
        L.hm_build_u64_shard.argtypes = [p, p, u64, u64, u64, u64, u32, C.POINTER(_Opts), p, C.POINTER(p),
                                         C.POINTER(u64)]
        L.hm_shard_set_base.argtypes = [p, u64]
        L.hm_route_queries_u64.argtypes = [p, p, u64, i32, p, p, p, p]
        L.hm_unroute_u64.argtypes = [p, p, p, u64, p, p, p]
        L.hm_assemble_u64.argtypes = [p, p, u64, u64, u64, u32, C.POINTER(_Opts), p, C.POINTER(p)]
        L.hm_build_u64_dist.argtypes = [p, p, u64, C.POINTER(_Opts), p, p, C.POINTER(p)]
        L.hm_lookup_u64_dist.argtypes = [p, p, u64, p, p, p, p]
        if hasattr(L, "hm_dist_decide"):  # (absent only from older debug builds, HM_LIB_PATH)
            L.hm_dist_bucket_range.argtypes = [u64, i32, i32, C.POINTER(u64), C.POINTER(u64)]
            L.hm_dist_bucket_range.restype = C.c_int
            L.hm_dist_decide.argtypes = [u64, u32, u64, i32, C.POINTER(u32)]
            L.hm_dist_decide.restype = C.c_int
            L.hm_dist_slot_base.argtypes = [p, i32, i32]
            L.hm_dist_slot_base.restype = u64
            L.hm_dist_exchange_plan.argtypes = [p, i32, i32, p, C.POINTER(u64), C.POINTER(u64)]
            L.hm_dist_exchange_plan.restype = C.c_int
        for f in ("hm_assemble_u64", "hm_build_u64_dist", "hm_lookup_u64_dist", "hm_build_u64", "hm_build_bytes", "hm_lookup_u64", "hm_lookup_bytes", "hm_info", "hm_export",
                  "hm_route_u64", "hm_build_u64_shard", "hm_shard_set_base", "hm_route_queries_u64",
                  "hm_unroute_u64"):
            getattr(L, f).restype = C.c_int
        _lib = L
    return _lib


def _check(code: int):
    if code != 0:
        raise HMError(code, lib().hm_last_error().decode(errors="replace"))


# ------------------------------------------------------------- marshalling

def _ptr(x, itemsize: int = 0, out: bool = False):
    """Pointer + keep-alive for a torch tensor (any device) or numpy array.

    itemsize: the element width the C call reads or writes (8 for keys, values,
    offsets and value outputs, 1 for byte contexts and found flags); a tensor of
    another width is refused instead of being read as the wrong type.  out: an
    output the library writes, which must be contiguous (a copy would lose the
    results)."""
    if x is None:
        return None, None
    try:
        import torch
        if isinstance(x, torch.Tensor):
            if itemsize and x.element_size() != itemsize:
                raise TypeError("expected a %d-byte element type, got %s" % (itemsize, x.dtype))
            if not x.is_contiguous():
                if out:
                    raise ValueError("output tensors must be contiguous")
                x = x.contiguous()
            return C.c_void_p(x.data_ptr()), x
    except ImportError:  # pragma: no cover
        pass
    if out:
        if not isinstance(x, np.ndarray) or not x.flags.c_contiguous:
            raise ValueError("output arrays must be contiguous numpy arrays or tensors")
        a = x
    else:
        a = np.ascontiguousarray(x)
    if itemsize and a.itemsize != itemsize:
        raise TypeError("expected a %d-byte element type, got %s" % (itemsize, a.dtype))
    return a.ctypes.data_as(C.c_void_p), a


def _numel(x) -> int:
    return int(x.numel()) if hasattr(x, "numel") else int(np.asarray(x).size)


def _stream(stream=None):
    if stream is not None:
        return C.c_void_p(int(stream))
    try:
        import torch
        if torch.cuda.is_available():
            return C.c_void_p(torch.cuda.current_stream().cuda_stream)
    except ImportError:  # pragma: no cover
        pass
    return C.c_void_p(0)


FLAG_FULL_DIRECTORY = 1  # HM_FLAG_FULL_DIRECTORY
FLAG_DIRECT_SLOTS = 2  # HM_FLAG_DIRECT_SLOTS (testing knob)
FLAG_NO_ROUND0_ILP = 4  # HM_FLAG_NO_ROUND0_ILP (testing knob)
FLAG_FROM_ARRAY = 8  # HM_FLAG_FROM_ARRAY: from_array (duplicates allowed, first occurrence kept)
FLAG_ROUNDS = 16  # HM_FLAG_ROUNDS: the paper's sortless round-based construction (ablation, u64 keys)
FLAG_FUSED_EXCHANGE = 32  # HM_FLAG_FUSED_EXCHANGE: build_u64_dist routes straight into the owners' NCCL windows
FLAG_FUSED_PASS2 = 64  # HM_FLAG_FUSED_PASS2: pass 2 + k_bucket as one pipelined kernel (alternative route, same table)


_allocator = None  # (alloc, free) ctypes callbacks of set_allocator
_allocators_alive = []  # every pair ever set: maps built with one call its free hook until hm_free


def set_allocator(alloc=None, free=None):
    """Allocator hooks (hm_opts.alloc / .free) for the arrays of the maps built
    from now on in this process: alloc(bytes, stream) -> device pointer (int),
    free(ptr, bytes, stream).  None, None: the library's own pool.  Maps keep
    the hooks they were built with until hm_free."""
    global _allocator
    if (alloc is None) != (free is None):
        raise ValueError("set both hooks or neither")
    if alloc is None:
        _allocator = None
        return
    a = ALLOC_FN(lambda n, st, ctx: alloc(int(n), st) or None)
    f = FREE_FN(lambda p, n, st, ctx: free(int(p), int(n), st))
    _allocator = (a, f)
    _allocators_alive.append(_allocator)


def _opts(seed: int, log2_bp: int = 0, flags: int = 0):
    o = _Opts(seed & ((1 << 64) - 1), log2_bp, flags)
    if _allocator is not None:
        o.alloc, o.free = _allocator
    return o


@dataclass
class Info:
    key_kind: int
    n: int
    S: int
    seed: int
    t1: int
    t0: int
    ctx_bytes: int


class HashMap:
    """An immutable FKS hash map living on one GPU (owned by libhm)."""

    def __init__(self, handle: int, key_kind: int):
        self._h = C.c_void_p(handle)
        self.key_kind = key_kind

    # -- build
    @classmethod
    def build_u64(cls, keys, vals, seed: int = 0, stream=None, log2_bp: int = 0, flags: int = 0) -> "HashMap":
        kp, kk = _ptr(keys, 8)
        vp, vk = _ptr(vals, 8)
        n = _numel(keys)
        if _numel(vals) != n:
            raise ValueError("keys and vals differ in length")
        h = C.c_void_p()
        o = _opts(seed, log2_bp, flags)
        _check(lib().hm_build_u64(kp, vp, n, C.byref(o), _stream(stream), C.byref(h)))
        return cls(h.value, 0)

    @classmethod
    def assemble_u64(cls, dir_, slots, n: int, S: int, seed: int, t1: int, flags: int = 0,
                     stream=None) -> "HashMap":
        """A map from a complete table (dir uint64[n], slots {key, value}[S] as
        2*S int64/uint64 words or the structured export), host or device."""
        dp, dk = _ptr(dir_)
        sp, sk = _ptr(slots)
        h = C.c_void_p()
        o = _opts(seed, 0, flags)
        _check(lib().hm_assemble_u64(dp, sp, n, S, seed & ((1 << 64) - 1), t1, C.byref(o), _stream(stream),
                                     C.byref(h)))
        return cls(h.value, 0)

    @classmethod
    def build_bytes(cls, ctx, offsets, vals, seed: int = 0, stream=None, log2_bp: int = 0, flags: int = 0) -> "HashMap":
        cp, ck = _ptr(ctx, 1)
        op, ok = _ptr(offsets, 8)
        vp, vk = _ptr(vals, 8)
        n = _numel(offsets) - 1
        if _numel(vals) != n:
            raise ValueError("offsets and vals disagree on n")
        h = C.c_void_p()
        o = _opts(seed, log2_bp, flags)
        _check(lib().hm_build_bytes(cp, op, vp, n, C.byref(o), _stream(stream), C.byref(h)))
        return cls(h.value, 1)

    # -- lookup
    def lookup(self, q, out_vals=None, out_found=None, stream=None):
        """Batched lookup of u64 queries; fills/returns (vals, found).

        With torch CUDA inputs and no outputs given, allocates device outputs."""
        nq = _numel(q)
        out_vals, out_found = self._outputs(q, nq, out_vals, out_found)
        qp, qk = _ptr(q, 8)
        vp, vk = _ptr(out_vals, 8, out=True)
        fp, fk = _ptr(out_found, 1, out=True)
        _check(lib().hm_lookup_u64(self._h, qp, nq, vp, fp, _stream(stream)))
        return out_vals, out_found

    def contains(self, q, out_found=None, stream=None):
        """Membership only: no value is read or written."""
        nq = _numel(q)
        _, out_found = self._outputs(q, nq, False, out_found)
        qp, qk = _ptr(q, 8)
        fp, fk = _ptr(out_found, 1, out=True)
        _check(lib().hm_lookup_u64(self._h, qp, nq, None, fp, _stream(stream)))
        return out_found

    def lookup_bytes(self, qctx, qoffsets, out_vals=None, out_found=None, stream=None):
        nq = _numel(qoffsets) - 1
        out_vals, out_found = self._outputs(qoffsets, nq, out_vals, out_found)
        cp, ck = _ptr(qctx, 1)
        op, ok = _ptr(qoffsets, 8)
        vp, vk = _ptr(out_vals, 8, out=True)
        fp, fk = _ptr(out_found, 1, out=True)
        _check(lib().hm_lookup_bytes(self._h, cp, op, nq, vp, fp, _stream(stream)))
        return out_vals, out_found

    def contains_bytes(self, qctx, qoffsets, out_found=None, stream=None):
        """Membership of byte-string needles: no value is written."""
        nq = _numel(qoffsets) - 1
        _, out_found = self._outputs(qoffsets, nq, False, out_found)
        cp, ck = _ptr(qctx, 1)
        op, ok = _ptr(qoffsets, 8)
        fp, fk = _ptr(out_found, 1, out=True)
        _check(lib().hm_lookup_bytes(self._h, cp, op, nq, None, fp, _stream(stream)))
        return out_found

    @staticmethod
    def _outputs(like, nq, out_vals, out_found):
        try:
            import torch
            is_t = isinstance(like, torch.Tensor)
        except ImportError:  # pragma: no cover
            is_t = False
        if is_t:
            import torch
            dev = like.device
            if out_vals is None:
                out_vals = torch.empty(nq, dtype=torch.int64, device=dev)
            if out_found is None:
                out_found = torch.empty(nq, dtype=torch.uint8, device=dev)
        else:
            if out_vals is None:
                out_vals = np.empty(nq, np.uint64)
            if out_found is None:
                out_found = np.empty(nq, np.uint8)
        if out_vals is False:
            out_vals = None
        return out_vals, out_found

    # -- introspection
    def info(self) -> Info:
        h = _Header()
        _check(lib().hm_info(self._h, C.byref(h)))
        return Info(h.key_kind, h.n, h.S, h.seed, h.t1, h.t0, h.ctx_bytes)

    def header_bytes(self) -> bytes:
        h = _Header()
        _check(lib().hm_info(self._h, C.byref(h)))
        return bytes(h)

    def export(self):
        """Host copies (dir uint64[n], slots structured[S], ctx uint8[] | None)."""
        inf = self.info()
        d = np.empty(inf.n, np.uint64)
        sd = SLOT_U64_DTYPE if self.key_kind == 0 else SLOT_BYTES_DTYPE
        raw = np.empty(max(1, inf.S) * sd.itemsize, np.uint8)
        ctx = np.empty(max(1, inf.ctx_bytes), np.uint8) if self.key_kind == 1 else None
        _check(lib().hm_export(self._h, d.ctypes.data_as(C.c_void_p), raw.ctypes.data_as(C.c_void_p),
                               ctx.ctypes.data_as(C.c_void_p) if ctx is not None else None))
        slots = raw[: inf.S * sd.itemsize].view(sd)
        if ctx is not None:
            ctx = ctx[: inf.ctx_bytes]
        return d, slots, ctx

    def free(self):
        if self._h and self._h.value:
            lib().hm_free(self._h)
            self._h = C.c_void_p(0)

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    def export_to(self, dir_out, slots_out):
        """Copy the directory (global soff for a shard) and the slots into
        caller tensors (device or host): dir_out int64[nb], slots_out int64[2*S]
        (u64 keys)."""
        dp, dk = _ptr(dir_out, 8, out=True)
        sp, sk = _ptr(slots_out, out=True)
        _check(lib().hm_export(self._h, dp, sp, None))

    # -- shards (multi-GPU)
    def set_base(self, slot_base: int):
        _check(lib().hm_shard_set_base(self._h, slot_base))

    def route_queries(self, q, world: int, send_q, perm, counts, stream=None):
        qp, qk = _ptr(q, 8)
        sp, sk = _ptr(send_q, 8, out=True)
        pp, pk = _ptr(perm, 8, out=True)
        cp, ck = _ptr(counts, 8, out=True)
        _check(lib().hm_route_queries_u64(self._h, qp, _numel(q), world, sp, pp, cp, _stream(stream)))


def route_u64(keys, vals, n_global: int, seed: int, t1: int, world: int, send_keys, send_vals, counts, stream=None):
    kp, kk = _ptr(keys, 8)
    vp, vk = _ptr(vals, 8)
    sk, skk = _ptr(send_keys, 8, out=True)
    sv, svk = _ptr(send_vals, 8, out=True)
    cp, ck = _ptr(counts, 8, out=True)
    _check(lib().hm_route_u64(kp, vp, _numel(keys), n_global, seed, t1, world, sk, sv, cp, _stream(stream)))


def build_u64_shard(keys, vals, n_global: int, b_lo: int, b_hi: int, t1: int, seed: int = 0, stream=None,
                    log2_bp: int = 0):
    kp, kk = _ptr(keys, 8)
    vp, vk = _ptr(vals, 8)
    h = C.c_void_p()
    S = C.c_uint64()
    o = _opts(seed, log2_bp)
    _check(lib().hm_build_u64_shard(kp, vp, _numel(keys), n_global, b_lo, b_hi, t1, C.byref(o), _stream(stream),
                                    C.byref(h), C.byref(S)))
    return HashMap(h.value, 0), int(S.value)


def build_u64_dist(keys, vals, nccl_comm: int, seed: int = 0, stream=None, log2_bp: int = 0,
                   flags: int = 0) -> "HashMap":
    """Collective sharded build over an NCCL communicator (hm_build_u64_dist;
    e.g. nccl_comm = the process group's backend ._comm_ptr()).  flags:
    FLAG_FUSED_EXCHANGE routes straight into the owners' windows."""
    kp, kk = _ptr(keys, 8)
    vp, vk = _ptr(vals, 8)
    h = C.c_void_p()
    o = _opts(seed, log2_bp, flags)
    _check(lib().hm_build_u64_dist(kp, vp, _numel(keys), C.byref(o), _stream(stream), C.c_void_p(int(nccl_comm)),
                                   C.byref(h)))
    return HashMap(h.value, 0)


def dist_release_windows(nccl_comm: int) -> None:
    """Free the receive windows FLAG_FUSED_EXCHANGE builds keep registered on
    this communicator (hm_dist_release_windows; collective: every rank)."""
    lib().hm_dist_release_windows.argtypes = [C.c_void_p]
    lib().hm_dist_release_windows.restype = C.c_int
    _check(lib().hm_dist_release_windows(C.c_void_p(int(nccl_comm))))


def lookup_u64_dist(shard: "HashMap", q, nccl_comm: int, out_vals=None, out_found=None, stream=None):
    """Collective routed lookup on the shards of build_u64_dist (hm_lookup_u64_dist)."""
    nq = _numel(q)
    out_vals, out_found = shard._outputs(q, nq, out_vals, out_found)
    qp, qk = _ptr(q, 8)
    vp, vk = _ptr(out_vals, 8, out=True)
    fp, fk = _ptr(out_found, 1, out=True)
    _check(lib().hm_lookup_u64_dist(shard._h, qp, nq, vp, fp, _stream(stream), C.c_void_p(int(nccl_comm))))
    return out_vals, out_found


def unroute_u64(vals_routed, found_routed, perm, out_vals, out_found, stream=None):
    a, ak = _ptr(vals_routed, 8)
    b, bk = _ptr(found_routed, 1)
    p, pk = _ptr(perm, 8)
    v, vk = _ptr(out_vals, 8, out=True)
    f, fk = _ptr(out_found, 1, out=True)
    _check(lib().hm_unroute_u64(a, b, p, _numel(perm), v, f, _stream(stream)))


DIST_REDRAW = 100  # HM_DIST_REDRAW


def dist_bucket_range(n_global: int, world: int, rank: int):
    """[lo, hi) of the level-1 buckets `rank` owns (hm_dist_bucket_range)."""
    lo, hi = C.c_uint64(), C.c_uint64()
    _check(lib().hm_dist_bucket_range(n_global, world, rank, C.byref(lo), C.byref(hi)))
    return int(lo.value), int(hi.value)


def dist_decide(n_global: int, t1: int, S_total: int, max_status: int):
    """(code, next_t1) of hm_dist_decide: 0 done, DIST_REDRAW route again with
    next_t1, else the status every rank reports."""
    nt = C.c_uint32(0)
    code = int(lib().hm_dist_decide(n_global, t1, S_total, max_status, C.byref(nt)))
    return code, int(nt.value)


def dist_slot_base(S_all, rank: int) -> int:
    a = np.ascontiguousarray(np.asarray(S_all, dtype=np.uint64))
    return int(lib().hm_dist_slot_base(a.ctypes.data_as(C.c_void_p), len(a), rank))


def dist_exchange_plan(C_matrix, world: int, rank: int):
    """(off[world], cap, recv) of hm_dist_exchange_plan for the count matrix
    C_matrix[q][r] (pairs rank q routes to owner r)."""
    cm = np.ascontiguousarray(np.asarray(C_matrix, dtype=np.uint64).reshape(world, world))
    off = np.zeros(world, np.uint64)
    cap, recv = C.c_uint64(), C.c_uint64()
    _check(lib().hm_dist_exchange_plan(cm.ctypes.data_as(C.c_void_p), world, rank, off.ctypes.data_as(C.c_void_p),
                                       C.byref(cap), C.byref(recv)))
    return [int(x) for x in off], int(cap.value), int(recv.value)


class _KStat(C.Structure):
    _fields_ = [("name", C.c_char * 32), ("launches", C.c_uint64), ("ms", C.c_double)]


def profile_enable(on: bool = True):
    """Bracket every libhm kernel launch with CUDA events on its stream."""
    lib().hm_profile_enable(1 if on else 0)


def profile_read() -> dict:
    """{kernel name: (launches, device ms)} since the last read (synchronises the events)."""
    buf = (_KStat * 64)()
    n = lib().hm_profile_read(buf, 64)
    return {buf[i].name.decode(): (int(buf[i].launches), float(buf[i].ms)) for i in range(min(n, 64))}


def kernel_launches() -> int:
    """Kernels launched by libhm so far in this process."""
    return int(lib().hm_kernel_launches())


def release_workspace() -> None:
    """Free the build scratch cached between builds on the current device."""
    _check(lib().hm_release_workspace())


def version() -> str:
    return lib().hm_version().decode()
