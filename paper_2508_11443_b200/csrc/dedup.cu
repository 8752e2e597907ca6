// dedup.cu — from_array: duplicates allowed, the
// first occurrence (lowest input index) of every key keeps its value, and the
// map is the one from_array_nodup builds from the distinct keys.
//
// A GPU hash set over the input keys (open addressing, linear probing, load
// factor <= 1/2, a 16-byte slot per distinct key holding the key and the lowest
// input index seen) followed by a compaction of the keys whose index is that lowest
// one.  Equal keys meet in one slot whatever their number, so any duplication
// pattern is handled (a million copies of one key are a million atomicMin on
// one address).  The compacted (key, value) arrays then go through the normal
// build with n = the number of distinct keys (R3).
#include <algorithm>

#include "hm_internal.cuh"

namespace hm {

// A slot is 16 bytes {key, meta}: meta = (lowest input index << 32) | state,
// so a probe touches one 32-byte sector.  A slot is claimed (EMPTY -> BUSY) by
// one thread's CAS on meta, which then writes the key and publishes READY
// (release); the others wait for READY before comparing keys, and an equal key
// lowers the index with a 64-bit atomicMin on meta (same state bits).
struct __align__(16) DedupSlot {
  uint64_t key, meta;
};
constexpr uint64_t kSlotEmpty = 0, kSlotBusy = 1, kSlotReady = 2;

__device__ __forceinline__ uint64_t ld_acquire_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t dedup_slot(uint64_t k, uint64_t mask) {
  return mix64(k ^ 0x3C6EF372FE94F82Bull) & mask;
}

__global__ void k_dedup_insert(const uint64_t* __restrict__ keys, uint64_t n, uint64_t mask, DedupSlot* set) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t k = __ldg(keys + i);
    uint64_t h = dedup_slot(k, mask);
    const uint64_t mine = (i << 32) | kSlotReady;
    while (true) {
      uint64_t* meta = &set[h].meta;
      uint64_t m = ld_acquire_u64(meta);
      if ((m & 3) == kSlotEmpty) {
        if (atomicCAS(reinterpret_cast<unsigned long long*>(meta), m, (i << 32) | kSlotBusy) == m) {
          set[h].key = k;
          st_release_u64(meta, mine);
          break;
        }
        continue;
      }
      while ((m & 3) == kSlotBusy) m = ld_acquire_u64(meta);
      if (set[h].key == k) {
        if (mine < m) atomicMin(reinterpret_cast<unsigned long long*>(meta), mine);
        break;
      }
      h = (h + 1) & mask;
    }
  }
}

// Keep input i iff it is the lowest index of its key: (key, value) go to the
// output at a warp-aggregated cursor position (order irrelevant: R13).
__global__ void k_dedup_compact(const uint64_t* __restrict__ keys, const uint64_t* __restrict__ vals, uint64_t n,
                                uint64_t mask, const DedupSlot* __restrict__ set, uint64_t* __restrict__ okeys,
                                uint64_t* __restrict__ ovals, unsigned long long* __restrict__ cursor) {
  const uint32_t lane = threadIdx.x & 31;
  for (uint64_t b = (blockIdx.x * uint64_t(blockDim.x)) & ~uint64_t(31); b < n; b += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t i = b + (threadIdx.x & ~31u) + lane;
    bool keep = false;
    uint64_t k = 0;
    if (i < n) {
      k = __ldg(keys + i);
      uint64_t h = dedup_slot(k, mask);
      DedupSlot sl = set[h];
      while (sl.key != k) {
        h = (h + 1) & mask;
        sl = set[h];
      }
      keep = (sl.meta >> 32) == i;
    }
    const uint32_t m = __ballot_sync(0xffffffffu, keep);
    if (!m) continue;
    const uint32_t leader = __ffs(m) - 1;
    unsigned long long p0 = 0;
    if (lane == leader) p0 = atomicAdd(cursor, (unsigned long long)__popc(m));
    p0 = __shfl_sync(0xffffffffu, p0, leader);
    if (keep) {
      const uint64_t p = p0 + __popc(m & ((1u << lane) - 1u));
      okeys[p] = k;
      ovals[p] = vals[i];
    }
  }
}

hm_status dedup_u64(const uint64_t* keys, const uint64_t* vals, uint64_t n, cudaStream_t st, uint64_t** out_keys,
                    uint64_t** out_vals, uint64_t* n_out) {
  *out_keys = *out_vals = nullptr;
  *n_out = 0;
  uint64_t cap = 1;
  while (cap < 2 * n) cap <<= 1;
  DedupSlot* set = nullptr;
  uint64_t *ok = nullptr, *ov = nullptr;
  unsigned long long* cur = nullptr;
  auto release = [&]() {
    if (cur) cudaFreeAsync(cur, st);
  };
  cudaError_t e;
  if ((e = cudaMallocAsync(reinterpret_cast<void**>(&cur), 8, st)) != cudaSuccess ||
      (e = cudaMallocAsync(reinterpret_cast<void**>(&ok), n * 8, st)) != cudaSuccess ||
      (e = cudaMallocAsync(reinterpret_cast<void**>(&ov), n * 8, st)) != cudaSuccess) {
    cudaGetLastError();
    release();
    if (ok) cudaFreeAsync(ok, st);
    set_error("from_array: out of device memory for the dedup set");
    return HM_ERR_OOM;
  }
  {  // the fast path: the build's radix passes and a shared-memory set per partition
    uint64_t m = 0;
    const hm_status ps = dedup_partitioned(keys, vals, n, st, ok, ov, &m);
    if (ps == HM_OK) {
      release();
      *out_keys = ok;
      *out_vals = ov;
      *n_out = m;
      return HM_OK;
    }
    if (ps != HM_ERR_TOO_LARGE) {
      release();
      cudaFreeAsync(ok, st);
      cudaFreeAsync(ov, st);
      return ps;
    }
  }
  // heavy duplication (a partition overflowed): the global set, cached build
  // scratch (hm_release_workspace frees it)
  {
    void* v = nullptr;
    const hm_status s = dedup_workspace(&v, cap * sizeof(DedupSlot), st);
    if (s != HM_OK) {
      release();
      cudaFreeAsync(ok, st);
      cudaFreeAsync(ov, st);
      return s;
    }
    set = reinterpret_cast<DedupSlot*>(v);
  }
  HM_CUDA_TRY(cudaMemsetAsync(set, 0, cap * sizeof(DedupSlot), st));
  HM_CUDA_TRY(cudaMemsetAsync(cur, 0, 8, st));
  const unsigned grid = unsigned(std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, uint64_t(num_sms()) * 8)));
  {
    LaunchScope ls_("k_dedup_insert", st);
    k_dedup_insert<<<grid, 256, 0, st>>>(keys, n, cap - 1, set);
  }
  {
    LaunchScope ls_("k_dedup_compact", st);
    k_dedup_compact<<<grid, 256, 0, st>>>(keys, vals, n, cap - 1, set, ok, ov, cur);
  }
  unsigned long long m = 0;
  HM_CUDA_TRY(cudaMemcpyAsync(&m, cur, 8, cudaMemcpyDeviceToHost, st));
  HM_CUDA_TRY(cudaStreamSynchronize(st));
  release();
  *out_keys = ok;
  *out_vals = ov;
  *n_out = m;
  return HM_OK;
}

}  // namespace hm
