"""Compile libhm.so (the CUDA path + C-ABI) in-tree for sm_100a with nvcc."""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libhm.so")
SOURCES = ["capi.cu", "build.cu", "lookup.cu", "dedup.cu", "rounds.cu", "assemble.cu", "dist.cu"]
HEADERS = ["hm_internal.cuh", "hm_math.cuh", "route.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
def _nccl_dir() -> str:
    """The pip NCCL torch loads (same libnccl.so.2 in the process), else the system one."""
    import sysconfig
    d = os.path.join(sysconfig.get_paths()["purelib"], "nvidia", "nccl")
    return d if os.path.exists(os.path.join(d, "include", "nccl.h")) else ""


_NCCL = _nccl_dir()
NCCL_FLAGS = ([f"-I{_NCCL}/include", f"-L{_NCCL}/lib", f"-Xlinker=-rpath={_NCCL}/lib"] if _NCCL else []) + \
    ["-l:libnccl.so.2"]
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo", "-O3", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "-Xptxas", "-v",
]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(os.path.dirname(PKG), "include", "hm.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [NVCC, *FLAGS, "-o", tmp] + [os.path.join(CSRC, f) for f in SOURCES] + NCCL_FLAGS
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libhm.so")
    if verbose:
        sys.stderr.write(r.stderr)
    with open(os.path.join(PKG, "ptxas_info.txt"), "w") as f:
        f.write(r.stderr)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)


def build_variant(tag: str, defines: list[str]) -> str:
    """Debug/experiment builds (libhm_<tag>.so with extra -D flags); never loaded
    by the product path unless HM_LIB_PATH points at one."""
    out = os.path.join(PKG, f"libhm_{tag}.so")
    cmd = [NVCC, *[f for f in FLAGS if f != "-v" and f != "-Xptxas"], *[f"-D{d}" for d in defines], "-o", out] + \
        [os.path.join(CSRC, f) for f in SOURCES] + NCCL_FLAGS
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"nvcc failed building {out}")
    return out
