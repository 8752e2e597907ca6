"""B200-native static FKS hash maps (arXiv 2508.11443 hot path).

The product is libhm.so (CUDA kernels for sm_100a behind the C-ABI of
include/hm.h); `hm` is its thin ctypes binding and `dist` the multi-GPU
orchestration over torch.distributed.
"""
from .hm import HashMap, HMError, build_u64_shard, route_u64, unroute_u64, version  # noqa: F401
