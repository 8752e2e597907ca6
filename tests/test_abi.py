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


def test_opts_layout_hooks_and_dist_argument_errors():
    L = hm.lib()
    assert C.sizeof(hm._Opts) == 40  # seed, log2_bp, flags, alloc, free, alloc_ctx
    out = C.c_void_p()
    k = np.zeros(4, np.uint64)
    kp = k.ctypes.data_as(C.c_void_p)
    o = hm._opts(0)
    o.alloc = hm.ALLOC_FN(lambda n, st, ctx: None)  # one hook without the other
    assert L.hm_build_u64(kp, kp, 4, C.byref(o), None, C.byref(out)) == 1
    assert L.hm_build_u64_dist(kp, kp, 4, None, None, None, C.byref(out)) == 1  # no communicator
    assert L.hm_lookup_u64_dist(None, kp, 4, kp, None, None, None) == 1
    assert L.hm_assemble_u64(kp, kp, 0, 1, 0, 0, None, None, C.byref(out)) == 2  # n == 0
    assert L.hm_assemble_u64(kp, kp, 4, 17, 0, 0, None, None, C.byref(out)) == 6  # S > 4n
    assert L.hm_assemble_u64(kp, kp, 4, 16, 0, 16, None, None, C.byref(out)) == 1  # t1 >= 16


def test_missing_library_fails_loudly(tmp_path):
    import subprocess
    import sys
    code = "from paper_2508_11443_b200 import hm\ntry:\n    hm.lib()\nexcept RuntimeError as e:\n    print('raised', e)\n"
    env = dict(os.environ, HM_LIB_PATH=str(tmp_path / "nope.so"), PYTHONPATH=ROOT)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=120)
    assert "raised" in r.stdout, r.stdout + r.stderr


def test_shard_build_rejects_single_table_flags():
    L = hm.lib()
    out, S = C.c_void_p(), C.c_uint64()
    k = np.zeros(4, np.uint64)
    kp = k.ctypes.data_as(C.c_void_p)
    for f in (hm.FLAG_FROM_ARRAY, hm.FLAG_ROUNDS):
        o = hm._opts(0, 0, f)
        assert L.hm_build_u64_shard(kp, kp, 4, 8, 0, 4, 0, C.byref(o), None, C.byref(out), C.byref(S)) == 1


def test_dist_decisions_need_no_device():
    """The sharded build's control decisions (hm_dist_*), shared by
    hm_build_u64_dist and dist.py: the space bound R7 with its 16 level-1
    draws, the max-status agreement, the bucket ranges owner(b) = floor(bG/n)
    and the slot bases."""
    REDRAW = hm.DIST_REDRAW
    assert hm.dist_decide(100, 0, 400, 0) == (0, 0)          # S = 4n: done
    assert hm.dist_decide(100, 0, 401, 0) == (REDRAW, 1)     # S > 4n: redraw t1 + 1
    assert hm.dist_decide(100, 14, 401, 0) == (REDRAW, 15)
    assert hm.dist_decide(100, 15, 401, 0)[0] == 4           # t1 = 15: SEED_EXHAUSTED (R7 cap)
    assert hm.dist_decide(100, 3, 10, 3)[0] == 3             # a shard failed: its status everywhere
    assert hm.dist_decide(100, 3, 10**9, 3)[0] == 3          # (a failure before the bound)
    for n in (1, 7, 100, 1 << 20, (1 << 30) + 0):
        for world in (1, 2, 3, 8, 64):
            prev = 0
            for r in range(world):
                lo, hi = hm.dist_bucket_range(n, world, r)
                assert lo == prev and lo == -(-r * n // world) and hi == -(-(r + 1) * n // world)
                # every bucket b of the range has owner floor(b*G/n) = r
                for b in {lo, hi - 1} if hi > lo else ():
                    assert b * world // n == r
                prev = hi
            assert prev == n
    with __import__("pytest").raises(hm.HMError):
        hm.dist_bucket_range(10, 2, 2)
    assert [hm.dist_slot_base([5, 7, 11], r) for r in range(3)] == [0, 5, 12]
