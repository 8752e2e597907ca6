"""The C-ABI library loads and exports every entry point include/hm.h declares
(no compute calls: this runs without a GPU)."""
import ctypes as C
import os
import re

import numpy as np

from paper_2508_11443_b200 import hm

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "hm.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hm_[a-z0-9_]+)\s*\(", src)))


def test_every_declared_symbol_is_exported():
    L = hm.lib()
    names = _declared()
    assert len(names) >= 14
    for n in names:
        assert hasattr(L, n), n


def test_status_strings_and_version():
    L = hm.lib()
    for code, name in hm.STATUS.items():
        assert L.hm_status_str(code).decode() == name
    assert "sm_100a" in hm.version()


def test_argument_errors_need_no_device():
    L = hm.lib()
    out = C.c_void_p()
    # n == 0 -> EMPTY (K is non-empty)
    assert L.hm_build_u64(None, None, 0, None, None, C.byref(out)) == 2
    assert out.value is None
    assert L.hm_build_bytes(None, None, None, 0, None, None, C.byref(out)) == 2
    # n > 2^30 -> TOO_LARGE
    k = np.zeros(1, np.uint64)
    assert L.hm_build_u64(k.ctypes.data_as(C.c_void_p), k.ctypes.data_as(C.c_void_p), (1 << 30) + 1, None, None,
                          C.byref(out)) == 6
    # NULL map / both outputs NULL -> INVALID_ARG
    assert L.hm_lookup_u64(None, None, 0, None, None, None) == 1
    assert L.hm_info(None, None) == 1
    L.hm_free(None)  # NULL-safe


def test_header_layout_matches_oracle():
    from oracle import oracle as O
    assert hm.HEADER_DTYPE == O.HEADER_DTYPE and hm.HEADER_DTYPE.itemsize == 56
    assert C.sizeof(hm._Header) == 56
    assert hm.SLOT_U64_DTYPE.itemsize == 16 and hm.SLOT_BYTES_DTYPE.itemsize == 32
