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
    set_error(std::string("from_array: out of device memory for the dedup set: ") + cudaGetErrorString(e));
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

// ------------------------------------------------------------ byte keys
// from_array for byte keys: fingerprints (any fixed point: they only group),
// the partitioned first-occurrence pass (keep[i] = 1 for the first occurrence
// of every distinct content, build.cu), then a stable compaction in input
// order — exclusive scans of keep and of the kept lengths give each survivor
// its index and its offset in a new packed context, exactly the context the
// oracle packs.
constexpr int kScanT = 1024, kScanPT = 4, kScanTile = kScanT * kScanPT;

// v[i] = keep[i] (mode 0) or keep[i] ? len_i : 0 (mode 1)
__global__ void k_keep_vals(const uint8_t* __restrict__ keep, const uint64_t* __restrict__ offs, uint64_t n, int mode,
                            uint64_t* __restrict__ v) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
    v[i] = keep[i] ? (mode ? offs[i + 1] - offs[i] : 1ull) : 0ull;
}

__device__ __forceinline__ uint64_t block_scan_excl_1024(uint64_t x, uint64_t* s_w, uint64_t* total) {
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t incl = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= uint32_t(o)) incl += y;
  }
  if (lane == 31) s_w[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    uint64_t w = s_w[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= uint32_t(o)) w += y;
    }
    s_w[lane] = w;
  }
  __syncthreads();
  *total = s_w[31];
  const uint64_t r = (warp ? s_w[warp - 1] : 0ull) + incl - x;
  __syncthreads();
  return r;
}

// in-place exclusive scan of a tile per block; the tile sums go to sums[]
__global__ void __launch_bounds__(kScanT) k_scan_tiles(uint64_t* __restrict__ v, uint64_t n,
                                                       uint64_t* __restrict__ sums) {
  __shared__ uint64_t s_w[32];
  const uint64_t t0 = uint64_t(blockIdx.x) * kScanTile + uint64_t(threadIdx.x) * kScanPT;
  uint64_t x[kScanPT], acc = 0;
#pragma unroll
  for (int j = 0; j < kScanPT; j++) {
    x[j] = t0 + j < n ? v[t0 + j] : 0ull;
    acc += x[j];
  }
  uint64_t tot;
  uint64_t run = block_scan_excl_1024(acc, s_w, &tot);
#pragma unroll
  for (int j = 0; j < kScanPT; j++) {
    if (t0 + j < n) v[t0 + j] = run;
    run += x[j];
  }
  if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

// exclusive scan of the tile sums in one block (sequential chunks per thread)
__global__ void __launch_bounds__(kScanT) k_scan_sums(uint64_t* __restrict__ sums, uint64_t m) {
  __shared__ uint64_t s_w[32];
  const uint64_t per = (m + kScanT - 1) / kScanT, a = threadIdx.x * per, b = min(a + per, m);
  uint64_t acc = 0;
  for (uint64_t i = a; i < b; i++) acc += sums[i];
  uint64_t tot;
  uint64_t run = block_scan_excl_1024(acc, s_w, &tot);
  for (uint64_t i = a; i < b; i++) {
    const uint64_t x = sums[i];
    sums[i] = run;
    run += x;
  }
}

__global__ void k_scan_add(uint64_t* __restrict__ v, uint64_t n, const uint64_t* __restrict__ sums) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
    v[i] += sums[i / kScanTile];
}

uint64_t scan_sums_len(uint64_t n) { return (n + kScanTile - 1) / kScanTile; }

// in-place exclusive scan of v[0, n); sums holds scan_sums_len(n) entries
hm_status scan_excl(uint64_t* v, uint64_t n, uint64_t* sums, cudaStream_t st) {
  const uint64_t tiles = (n + kScanTile - 1) / kScanTile;
  {
    LaunchScope ls_("k_scan_tiles", st);
    k_scan_tiles<<<unsigned(tiles), kScanT, 0, st>>>(v, n, sums);
  }
  {
    LaunchScope ls_("k_scan_sums", st);
    k_scan_sums<<<1, kScanT, 0, st>>>(sums, tiles);
  }
  {
    LaunchScope ls_("k_scan_add", st);
    const unsigned g = unsigned(std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, uint64_t(num_sms()) * 8)));
    k_scan_add<<<g, 256, 0, st>>>(v, n, sums);
  }
  HM_CUDA_TRY(cudaGetLastError());
  return HM_OK;
}

// survivors -> packed context, offsets and values (thread per input key)
__global__ void k_pack_kept(const uint8_t* __restrict__ bytes, const uint64_t* __restrict__ offs,
                            const uint64_t* __restrict__ vals, const uint8_t* __restrict__ keep, uint64_t n,
                            const uint64_t* __restrict__ pos, const uint64_t* __restrict__ bpos,
                            uint8_t* __restrict__ nctx, uint64_t* __restrict__ noffs, uint64_t* __restrict__ nvals) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
    if (!keep[i]) continue;
    const uint64_t p = pos[i], o = offs[i], len = offs[i + 1] - o, b = bpos[i];
    noffs[p] = b;
    nvals[p] = vals[i];
    for (uint64_t k = 0; k < len; k++) nctx[b + k] = bytes[o + k];
  }
}

// Byte keys, the fallback of heavy duplication (a dedup partition overflowed):
// the global set keyed by fingerprint, every hit confirmed by content against
// the slot's current lowest index (all indices in a slot hold equal bytes),
// so equal fingerprints of different keys take different slots.
__global__ void k_dedup_insert_bytes(const uint8_t* __restrict__ bytes, const uint64_t* __restrict__ offs,
                                     const uint64_t* __restrict__ fp, uint64_t n, uint64_t mask, DedupSlot* set) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t f = fp[i], o = offs[i];
    const uint32_t len = uint32_t(offs[i + 1] - o);
    uint64_t h = dedup_slot(f, mask);
    const uint64_t mine = (i << 32) | kSlotReady;
    while (true) {
      uint64_t* meta = &set[h].meta;
      uint64_t m = ld_acquire_u64(meta);
      if ((m & 3) == kSlotEmpty) {
        if (atomicCAS(reinterpret_cast<unsigned long long*>(meta), m, (i << 32) | kSlotBusy) == m) {
          set[h].key = f;
          st_release_u64(meta, mine);
          break;
        }
        continue;
      }
      while ((m & 3) == kSlotBusy) m = ld_acquire_u64(meta);
      if (set[h].key == f) {
        const uint64_t r = m >> 32, ro = offs[r];
        if (offs[r + 1] - ro == len && bytes_equal(bytes + ro, bytes + o, len)) {
          if (mine < m) atomicMin(reinterpret_cast<unsigned long long*>(meta), mine);
          break;
        }
      }
      h = (h + 1) & mask;
    }
  }
}

__global__ void k_dedup_keep_bytes(const uint8_t* __restrict__ bytes, const uint64_t* __restrict__ offs,
                                   const uint64_t* __restrict__ fp, uint64_t n, uint64_t mask,
                                   const DedupSlot* __restrict__ set, uint8_t* __restrict__ keep) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t f = fp[i], o = offs[i];
    const uint32_t len = uint32_t(offs[i + 1] - o);
    uint64_t h = dedup_slot(f, mask);
    while (true) {
      const DedupSlot sl = set[h];
      if (sl.key == f) {
        const uint64_t r = sl.meta >> 32, ro = offs[r];
        if (offs[r + 1] - ro == len && bytes_equal(bytes + ro, bytes + o, len)) {
          keep[i] = r == i ? 1 : 0;
          break;
        }
      }
      h = (h + 1) & mask;
    }
  }
}

static hm_status dedup_global_bytes(const uint8_t* bytes, const uint64_t* offs, const uint64_t* fp, uint64_t n,
                                    cudaStream_t st, uint8_t* keep) {
  uint64_t cap = 1024;
  while (cap < 2 * n) cap <<= 1;
  DedupSlot* set = nullptr;
  if (cudaMallocAsync(reinterpret_cast<void**>(&set), cap * sizeof(DedupSlot), st) != cudaSuccess) {
    cudaGetLastError();
    set_error("from_array: out of device memory for the dedup set");
    return HM_ERR_OOM;
  }
  HM_CUDA_TRY(cudaMemsetAsync(set, 0, cap * sizeof(DedupSlot), st));
  const unsigned g = unsigned(std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, uint64_t(num_sms()) * 8)));
  {
    LaunchScope ls_("k_dedup_insert_bytes", st);
    k_dedup_insert_bytes<<<g, 256, 0, st>>>(bytes, offs, fp, n, cap - 1, set);
  }
  {
    LaunchScope ls_("k_dedup_keep_bytes", st);
    k_dedup_keep_bytes<<<g, 256, 0, st>>>(bytes, offs, fp, n, cap - 1, set, keep);
  }
  const cudaError_t e = cudaGetLastError();
  cudaFreeAsync(set, st);
  if (e != cudaSuccess) return cuda_fail(e, "dedup_global_bytes");
  return HM_OK;
}

hm_status dedup_bytes(const uint8_t* bytes, const uint64_t* offs, const uint64_t* vals, uint64_t n, cudaStream_t st,
                      uint8_t** out_ctx, uint64_t** out_offs, uint64_t** out_vals, uint64_t* n_out) {
  *out_ctx = nullptr;
  *out_offs = *out_vals = nullptr;
  *n_out = 0;
  uint64_t *fp = nullptr, *pos = nullptr, *bpos = nullptr, *sums = nullptr;
  uint8_t* keep = nullptr;
  auto release = [&]() {
    for (void* q : {static_cast<void*>(fp), static_cast<void*>(pos), static_cast<void*>(bpos),
                    static_cast<void*>(sums), static_cast<void*>(keep)})
      if (q) cudaFreeAsync(q, st);
  };
  const uint64_t tiles = (n + kScanTile - 1) / kScanTile;
  if (cudaMallocAsync(reinterpret_cast<void**>(&fp), n * 8, st) != cudaSuccess ||
      cudaMallocAsync(reinterpret_cast<void**>(&pos), n * 8, st) != cudaSuccess ||
      cudaMallocAsync(reinterpret_cast<void**>(&bpos), n * 8, st) != cudaSuccess ||
      cudaMallocAsync(reinterpret_cast<void**>(&sums), tiles * 8 + 8, st) != cudaSuccess ||
      cudaMallocAsync(reinterpret_cast<void**>(&keep), n + 16, st) != cudaSuccess) {
    cudaGetLastError();
    release();
    set_error("from_array: out of device memory");
    return HM_ERR_OOM;
  }
  uint64_t o0 = 0, on = 0;
  HM_CUDA_TRY(cudaMemcpyAsync(&o0, offs, 8, cudaMemcpyDeviceToHost, st));
  HM_CUDA_TRY(cudaMemcpyAsync(&on, offs + n, 8, cudaMemcpyDeviceToHost, st));
  launch_fingerprint(bytes, offs, n, derive(seed_mix(0x46524F4D41525241ull), 0, 0, 0).a1, fp, st);
  HM_CUDA_TRY(cudaMemsetAsync(keep, 0, n, st));
  HM_CUDA_TRY(cudaStreamSynchronize(st));
  hm_status s = dedup_partitioned_bytes(bytes, offs, fp, vals, n, o0, st, keep);
  if (s == HM_ERR_TOO_LARGE) {  // heavy duplication: the global set decides every key
    set_error("");
    s = dedup_global_bytes(bytes, offs, fp, n, st, keep);
  }
  if (s != HM_OK) {
    release();
    return s;
  }
  const unsigned g = unsigned(std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, uint64_t(num_sms()) * 8)));
  k_keep_vals<<<g, 256, 0, st>>>(keep, offs, n, 0, pos);
  k_keep_vals<<<g, 256, 0, st>>>(keep, offs, n, 1, bpos);
  if ((s = scan_excl(pos, n, sums, st)) != HM_OK || (s = scan_excl(bpos, n, sums, st)) != HM_OK) {
    release();
    return s;
  }
  uint64_t lastp = 0, lastb = 0;
  uint8_t lastk = 0;
  HM_CUDA_TRY(cudaMemcpyAsync(&lastp, pos + n - 1, 8, cudaMemcpyDeviceToHost, st));
  HM_CUDA_TRY(cudaMemcpyAsync(&lastb, bpos + n - 1, 8, cudaMemcpyDeviceToHost, st));
  HM_CUDA_TRY(cudaMemcpyAsync(&lastk, keep + n - 1, 1, cudaMemcpyDeviceToHost, st));
  uint64_t lastlen = 0, ol = 0;
  HM_CUDA_TRY(cudaMemcpyAsync(&ol, offs + n - 1, 8, cudaMemcpyDeviceToHost, st));
  HM_CUDA_TRY(cudaStreamSynchronize(st));
  lastlen = on - ol;
  const uint64_t m = lastp + (lastk ? 1 : 0), tb = lastb + (lastk ? lastlen : 0);
  uint8_t* nctx = nullptr;
  uint64_t *noffs = nullptr, *nvals = nullptr;
  if (cudaMallocAsync(reinterpret_cast<void**>(&nctx), tb + 16, st) != cudaSuccess ||
      cudaMallocAsync(reinterpret_cast<void**>(&noffs), (m + 1) * 8, st) != cudaSuccess ||
      cudaMallocAsync(reinterpret_cast<void**>(&nvals), m * 8 + 8, st) != cudaSuccess) {
    cudaGetLastError();
    release();
    for (void* q : {static_cast<void*>(nctx), static_cast<void*>(noffs), static_cast<void*>(nvals)})
      if (q) cudaFreeAsync(q, st);
    set_error("from_array: out of device memory");
    return HM_ERR_OOM;
  }
  {
    LaunchScope ls_("k_pack_kept", st);
    k_pack_kept<<<g, 256, 0, st>>>(bytes, offs, vals, keep, n, pos, bpos, nctx, noffs, nvals);
  }
  HM_CUDA_TRY(cudaMemcpyAsync(noffs + m, &tb, 8, cudaMemcpyHostToDevice, st));
  HM_CUDA_TRY(cudaStreamSynchronize(st));  // (tb is a host variable)
  release();
  *out_ctx = nctx;
  *out_offs = noffs;
  *out_vals = nvals;
  *n_out = m;
  return HM_OK;
}

}  // namespace hm
