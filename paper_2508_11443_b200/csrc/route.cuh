// route.cuh — the owner-rank scatter of the multi-GPU path,
// shared by the local-buffer kernel (lookup.cu) and the fused route +
// exchange kernel that stores straight into the owners' NCCL windows
// (dist.cu).  Included after hm_internal.cuh.
#pragma once

namespace hm {

// owner(b) = floor(b * G / n): contiguous bucket ranges.
__device__ __forceinline__ uint32_t owner_of(uint64_t b, uint64_t n, int world) {
  return uint32_t((b * uint64_t(world)) / n);
}

// Scatter by owner rank, a tile of kRTile keys per CTA: the rank of every key
// among the tile's keys with the same destination comes from a shared-memory
// atomicAdd, one global atomicAdd per (tile, destination) reserves its run
// (cursors[d]: the next free position in destination d's buffer; counts are
// exact, k_route_count ran first), and the tile is staged in shared memory in
// destination order so that the runs are written with consecutive lanes.
// perm[i] (queries) = the routed position of input i.  Out gives the base of
// destination d's key and value buffers: this rank's send buffers, or the
// owner's receive window mapped over NVLink.
constexpr int kRThreads = 512, kRPT = 8, kRTile = kRThreads * kRPT;
template <class Out>
__device__ __forceinline__ void route_scatter(const uint64_t* __restrict__ keys, const uint64_t* __restrict__ vals,
                                              uint64_t n, const L1Params& l1, int world,
                                              unsigned long long* __restrict__ cursors, const Out& out,
                                              uint64_t* __restrict__ perm) {
  __shared__ uint64_t s_k[kRTile];
  __shared__ uint8_t s_d[kRTile];
  __shared__ uint32_t s_cnt[64], s_pre[64];
  __shared__ unsigned long long s_base[64];
  const uint32_t tid = threadIdx.x;
  for (uint64_t t0 = uint64_t(blockIdx.x) * kRTile; t0 < n; t0 += uint64_t(gridDim.x) * kRTile) {
    const uint32_t nv = n - t0 < uint64_t(kRTile) ? uint32_t(n - t0) : uint32_t(kRTile);
    if (tid < 64) s_cnt[tid] = 0;
    __syncthreads();
    uint64_t k[kRPT];
    uint32_t d[kRPT], rk[kRPT];
#pragma unroll
    for (int j = 0; j < kRPT; j++) {
      const uint32_t i = j * kRThreads + tid;
      k[j] = i < nv ? __ldg(keys + t0 + i) : 0ull;
    }
#pragma unroll
    for (int j = 0; j < kRPT; j++) {
      const uint32_t i = j * kRThreads + tid;
      d[j] = 0;
      if (i < nv) {
        d[j] = owner_of(level1_bucket(l1, k[j]), l1.n, world);
        rk[j] = atomicAdd(&s_cnt[d[j]], 1u);
      }
    }
    __syncthreads();
    if (tid < 32) {  // tile prefix over the destinations (world <= 64: two per lane)
      const uint32_t a = s_cnt[2 * tid], b = s_cnt[2 * tid + 1];
      uint32_t x = a + b;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (tid >= uint32_t(o)) x += y;
      }
      x -= a + b;
      s_pre[2 * tid] = x;
      s_pre[2 * tid + 1] = x + a;
    }
    if (tid < uint32_t(world) && s_cnt[tid]) s_base[tid] = atomicAdd(&cursors[tid], (unsigned long long)s_cnt[tid]);
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kRPT; j++) {
      const uint32_t i = j * kRThreads + tid;
      if (i < nv) {
        const uint32_t pos = s_pre[d[j]] + rk[j];
        s_k[pos] = k[j];
        s_d[pos] = uint8_t(d[j]);
        if (perm) perm[t0 + i] = s_base[d[j]] + rk[j];
      }
    }
    __syncthreads();
    for (uint32_t i = tid; i < nv; i += kRThreads) {
      const uint32_t dd = s_d[i];
      out.keys(dd)[s_base[dd] + (i - s_pre[dd])] = s_k[i];
    }
    if (vals) {  // values follow the same permutation (staged through the same buffer)
      __syncthreads();
#pragma unroll
      for (int j = 0; j < kRPT; j++) {
        const uint32_t i = j * kRThreads + tid;
        if (i < nv) s_k[s_pre[d[j]] + rk[j]] = __ldg(vals + t0 + i);
      }
      __syncthreads();
      for (uint32_t i = tid; i < nv; i += kRThreads) {
        const uint32_t dd = s_d[i];
        out.vals(dd)[s_base[dd] + (i - s_pre[dd])] = s_k[i];
      }
    }
    __syncthreads();
  }
}

}  // namespace hm
