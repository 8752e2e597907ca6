"""Device-side generation of the workloads of workloads/gen.py (same recipe,
bit-identical; checked by tests/test_workloads_gpu.py).  Used by bench.py for
the multi-GiB inputs.  Not part of the product path."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from . import gen

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "gen_cuda.cu")
LIB = os.path.join(HERE, "libhmgen.so")
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        tmp = LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                               "-lineinfo", "-Xcompiler", "-fPIC", "-shared", "-o", tmp, SRC])
        os.replace(tmp, LIB)
    return LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB)
        p, u64 = C.c_void_p, C.c_uint64
        L.hg_u64_keys.argtypes = [u64, u64, u64, p, p, p]
        L.hg_queries.argtypes = [u64, u64, u64, u64, u64, p, p, p, p]
        L.hg_query_ids.argtypes = [u64, u64, u64, u64, p, p]
        L.hg_str_lens.argtypes = [u64, p, u64, u64, p, p, u64, u64]
        L.hg_str_bytes.argtypes = [u64, p, u64, u64, p, p, p]
        _lib = L
    return _lib


def _p(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def _s():
    import torch
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def u64_keys(n, lo=0, with_values=True, device="cuda"):
    import torch
    k = torch.empty(n, dtype=torch.int64, device=device)
    v = torch.empty(n, dtype=torch.int64, device=device) if with_values else None
    assert lib().hg_u64_keys(gen.SEED_K, lo, n, _p(k), _p(v), _s()) == 0
    return k, v


def u64_queries(n, nq, lo=0, with_expect=False, device="cuda"):
    import torch
    q = torch.empty(nq, dtype=torch.int64, device=device)
    ev = torch.empty(nq, dtype=torch.int64, device=device) if with_expect else None
    ef = torch.empty(nq, dtype=torch.uint8, device=device) if with_expect else None
    assert lib().hg_queries(gen.SEED_K, gen.SEED_Q, n, lo, nq, _p(q), _p(ev), _p(ef), _s()) == 0
    return q, ev, ef


def _strings(ids, lo, n, device, lens_range=(4, 64)):
    import torch
    lens = torch.empty(n, dtype=torch.int64, device=device)
    lmin, lmax = lens_range
    assert lib().hg_str_lens(gen.SEED_L, _p(ids), lo, n, _p(lens), _s(), lmin, lmax - lmin + 1) == 0
    offs = torch.zeros(n + 1, dtype=torch.int64, device=device)
    torch.cumsum(lens, 0, out=offs[1:])
    total = int(offs[-1].item())
    ctx = torch.empty(total + 8, dtype=torch.uint8, device=device)
    assert lib().hg_str_bytes(gen.SEED_B, _p(ids), lo, n, _p(offs), _p(ctx), _s()) == 0
    return ctx[:total], offs


def string_keys(n, lo=0, device="cuda", lens_range=(4, 64)):
    return _strings(None, lo, n, device, lens_range)


def string_queries(n, nq, lo=0, device="cuda", lens_range=(4, 64)):
    import torch
    ids = torch.empty(nq, dtype=torch.int64, device=device)
    assert lib().hg_query_ids(gen.SEED_Q, n, lo, nq, _p(ids), _s()) == 0
    ctx, offs = _strings(ids, 0, nq, device, lens_range)
    return ctx, offs, ids
