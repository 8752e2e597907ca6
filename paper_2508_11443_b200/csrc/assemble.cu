// assemble.cu — a map from a complete table: the directory and the slots of
// the canonical layout, e.g. the concatenation of the exported
// shards of a distributed build (the replicated-lookup mode of SURVEY.md §8(f)
// NEXT-2) or an hm_export of a single table.
//
// The arrays are copied; the compact lookup directory is
// derived from them, a warp per 32 buckets, and the directory is checked on
// the way: soff_0 = 0, soff_{b+1} = soff_b + s_b^2, soff_{n-1} + s_{n-1}^2 = S
// and t = 0 for singletons and empty buckets (R12), so that every probe a
// lookup can make stays inside the slots.
#include <algorithm>

#include "hm_internal.cuh"

namespace hm {

__global__ void k_assemble_cdir(const uint64_t* __restrict__ dir, const KV16* __restrict__ slots, uint64_t n,
                                uint64_t S, L1Params l1, uint32_t full_dir, CDir* __restrict__ cdir,
                                unsigned int* __restrict__ bad) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t b0 = blockIdx.x * uint64_t(blockDim.x) + (threadIdx.x & ~31u); b0 < n; b0 += stride) {
    const uint64_t b = b0 + lane;
    uint32_t s = 0, t = 0;
    uint64_t so = 0;
    if (b < n) {
      const uint64_t d = dir[b];
      so = d & kMask40;
      s = uint32_t(d >> 40) & 0xFFFFu;
      t = uint32_t(d >> 56);
      const uint64_t next = b + 1 < n ? (dir[b + 1] & kMask40) : S;
      bool ok = so + uint64_t(s) * s == next && (b != 0 || so == 0) && (s >= 2 || t == 0);
      if (ok && s == 1 && so < S) t = tag4_of_hash(hash64(l1.c1, slots[so].key));  // the singleton tag (§6.2)
      if (!ok) atomicOr(bad, 1u);
    }
    uint32_t pa = __ballot_sync(0xffffffffu, s & 4), pb = __ballot_sync(0xffffffffu, s & 2),
             pc = __ballot_sync(0xffffffffu, s & 1);
    const uint32_t t0 = __ballot_sync(0xffffffffu, t & 1), t1 = __ballot_sync(0xffffffffu, t & 2),
                   t2 = __ballot_sync(0xffffffffu, t & 4), t3 = __ballot_sync(0xffffffffu, t & 8);
    if (__any_sync(0xffffffffu, s >= kCdirEscS || (s >= 2 && t >= kCdirEscT)) || full_dir) pa = pb = pc = 0xffffffffu;
    if (lane == 0) {
      CDir r;
      r.w[0] = uint32_t(so);
      r.w[1] = pa;
      r.w[2] = pb;
      r.w[3] = pc;
      r.w[4] = t0;
      r.w[5] = t1;
      r.w[6] = t2;
      r.w[7] = t3;
      cdir[b0 >> 5] = r;
    }
  }
}

// soff += base over a directory (hm_export of a shard into device memory)
__global__ void k_dir_rebase(uint64_t* __restrict__ d, uint64_t n, uint64_t base) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t x = d[i];
    d[i] = (x & ~kMask40) | ((x & kMask40) + base);
  }
}

hm_status assemble_cdir_launch(const uint64_t* dir, const void* slots, uint64_t n, uint64_t S, const L1Params& l1,
                               uint32_t full_dir, CDir* cdir, unsigned int* bad, cudaStream_t st) {
  const unsigned g = unsigned(std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, uint64_t(num_sms()) * 8)));
  {
    LaunchScope ls_("k_assemble_cdir", st);
    k_assemble_cdir<<<g, 256, 0, st>>>(dir, reinterpret_cast<const KV16*>(slots), n, S, l1, full_dir, cdir, bad);
  }
  HM_CUDA_TRY(cudaGetLastError());
  return HM_OK;
}

hm_status dir_rebase_launch(uint64_t* d, uint64_t n, uint64_t base, cudaStream_t st) {
  const unsigned g = unsigned(std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, uint64_t(num_sms()) * 8)));
  {
    LaunchScope ls_("k_dir_rebase", st);
    k_dir_rebase<<<g, 256, 0, st>>>(d, n, base);
  }
  HM_CUDA_TRY(cudaGetLastError());
  return HM_OK;
}

}  // namespace hm
