// build.cu — FKS construction on sm_100a (§2.2-§2.5, 220-499).
//
// The paper's flattened construction runs make2 for all buckets in bulk rounds
// (segrandom / seghashes / segcollisions / segresult).  This
// is the B200 design of DESIGN.md §6 instead — two kernels per level-1 attempt:
//
//   K_A  k_partition : stream (key, value), hash every key to its level-1
//        bucket g k = hash(c1, k) mod n and append it to the
//        build partition that owns a contiguous range of 2^log2_bp buckets.
//        A per-CTA shared-memory histogram ranks the tile's keys per partition
//        so that only one global atomic per (tile, partition) reserves space.
//   K_B  k_bucket    : one CTA per partition, everything else in shared memory:
//        hist of the partition's buckets, exclusive scans of s
//        and s^2 (presum, PAPER.md:229-230 with R1/R2), groupby
//        as a counting scatter of (key, index) into bucket order, the level-2
//        seed search make2 per bucket — a group of G lanes
//        per bucket (G = 2/4/8/32 by size class), one attempt per loop
//        iteration, __match_any_sync as the injectivity test — then a
//        decoupled look-back across partitions for the global slot base, and
//        the write of the directory and of the s^2 slots of every bucket
//        (members + filler, R10).
//
// One host synchronisation per attempt reads the device status (total S for
// the space bound R7, duplicate / exhaustion flags).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <map>
#include <mutex>
#include <type_traits>
#include <vector>

#include "hm_internal.cuh"

namespace hm {

constexpr int kAThreads = 512;
#ifndef HM_KB_THREADS
#define HM_KB_THREADS 512
#endif
#ifndef HM_KB_LOG2BP
#define HM_KB_LOG2BP 12
#endif
constexpr int kBThreads = HM_KB_THREADS;
constexpr int kBWarps = kBThreads / 32;
constexpr unsigned long long kFlagAgg = 1ull << 62, kFlagInc = 2ull << 62, kValMask = (1ull << 62) - 1;

// ----------------------------------------------------------------- sources
struct SrcU64 {
  const uint64_t* keys;
  const uint64_t* vals;
  __device__ __forceinline__ KV16 load(uint64_t i) const {
    KV16 e;
    e.key = __ldg(keys + i);
    e.value = __ldg(vals + i);
    return e;
  }
};
struct SrcBytes {
  const uint64_t* fp;
  const uint64_t* vals;
  const uint64_t* offs;
  uint64_t off0;
  __device__ __forceinline__ KV32 load(uint64_t i) const {
    KV32 e;
    const uint64_t o = __ldg(offs + i), o1 = __ldg(offs + i + 1);
    e.key = __ldg(fp + i);
    e.value = __ldg(vals + i);
    e.ctx_off = o - off0;
    e.len = uint32_t(o1 - o);
    e.reserved = 0;
    return e;
  }
};
// Equal hashed keys: the same key (duplicate) or a fingerprint collision?
struct SameU64 {
  __device__ __forceinline__ bool same(const KV16&, const KV16&) const { return true; }
};
struct SameBytes {
  const uint8_t* bytes;  // original context, element ctx_off is relative to off0
  uint64_t off0;
  __device__ bool same(const KV32& a, const KV32& b) const {
    if (a.len != b.len) return false;
    const uint8_t* pa = bytes + off0 + a.ctx_off;
    const uint8_t* pb = bytes + off0 + b.ctx_off;
    for (uint32_t i = 0; i < a.len; i++)
      if (pa[i] != pb[i]) return false;
    return true;
  }
};

// ------------------------------------------------------------- primitives
__device__ __forceinline__ void st_release(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Block-wide exclusive scan of u64 (kBThreads threads); also returns the total.
__device__ __forceinline__ unsigned long long block_excl_scan(unsigned long long v, unsigned long long* total,
                                                              unsigned long long* s_red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned long long x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_red[warp] = x;
  __syncthreads();
  if (warp == 0) {
    unsigned long long w = lane < kBWarps ? s_red[lane] : 0ull;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      unsigned long long y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < kBWarps) s_red[lane] = w;
  }
  __syncthreads();
  const unsigned long long before = warp ? s_red[warp - 1] : 0ull;
  *total = s_red[kBWarps - 1];
  __syncthreads();
  return before + x - v;
}

// Debug-only phase timestamps (compile with -DHM_PHASE_TIMING).
#ifdef HM_PHASE_TIMING
__device__ unsigned long long g_hm_phase[65536 * 12];
__device__ unsigned long long g_hm_ka[4096 * 2];
#define HM_TMARK(k)                                                     \
  do {                                                                  \
    if (threadIdx.x == 0) {                                             \
      unsigned long long t_;                                            \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));            \
      g_hm_phase[(s_p & 65535u) * 12 + (k)] = t_;                       \
    }                                                                   \
  } while (0)
extern "C" int hm_debug_phase_times(unsigned long long* host, unsigned long long n) {
  int e = int(cudaMemcpyFromSymbol(host, g_hm_phase, n * 8));
  if (!e) e = int(cudaMemcpyFromSymbol(host + n, g_hm_ka, 4096 * 2 * 8));
  return e;
}
#define HM_TKA(k)                                                       \
  do {                                                                  \
    if (threadIdx.x == 0 && blockIdx.x < 4096) {                        \
      unsigned long long t_;                                            \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));            \
      g_hm_ka[blockIdx.x * 2 + (k)] = t_;                               \
    }                                                                   \
  } while (0)
#elif defined(HM_STOP_AFTER)
// debug: cut the kernel after phase mark HM_STOP_AFTER (marginal phase costs)
#define HM_TMARK(k)                   \
  do {                                \
    if ((k) == HM_STOP_AFTER) return; \
  } while (0)
#define HM_TKA(k) \
  do {            \
  } while (0)
#else
#define HM_TKA(k) \
  do {            \
  } while (0)
#define HM_TMARK(k) \
  do {              \
  } while (0)
#endif

// ------------------------------------------------------------------ K_A
template <class Src, class E, int KPT, bool kSmemHist>
__global__ void __launch_bounds__(kAThreads) k_partition(Src src, BuildParams bp, E* __restrict__ pbuf,
                                                         unsigned int* __restrict__ pcount,
                                                         DevStatus* __restrict__ stt) {
  constexpr uint32_t kNone = 0x7FFFFFFFu, kLead = 0x80000000u;
  extern __shared__ unsigned int s_hist[];
  const uint32_t tid = threadIdx.x;
  if (kSmemHist) {
    for (uint32_t i = tid; i < bp.np; i += kAThreads) s_hist[i] = 0;
    __syncthreads();
  }
  HM_TKA(0);
  const uint64_t T = uint64_t(kAThreads) * KPT;
  const uint64_t ntiles = (bp.n_in + T - 1) / T;
  bool ovf = false, bad = false;
  for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    E e[KPT];
    uint32_t pp[KPT], rk[KPT];
    const uint64_t base = tile * T;
#pragma unroll
    for (int j = 0; j < KPT; j++) {
      const uint64_t idx = base + uint64_t(j) * kAThreads + tid;
      pp[j] = kNone;
      rk[j] = 0;
      if (idx < bp.n_in) e[j] = src.load(idx);
    }
    // g k = hash(c1, k) mod n -> owning partition; rank within the tile
#pragma unroll
    for (int j = 0; j < KPT; j++) {
      const uint64_t idx = base + uint64_t(j) * kAThreads + tid;
      if (idx < bp.n_in) {
        const uint64_t lb = level1_bucket(bp.l1, e[j].key) - bp.b_lo;
        if (lb >= bp.nb) {
          bad = true;
          continue;
        }
        pp[j] = uint32_t(lb >> bp.log2_bp);
        rk[j] = kSmemHist ? atomicAdd(&s_hist[pp[j]], 1u) : atomicAdd(&pcount[pp[j]], 1u);
      }
    }
    if (kSmemHist) {
      // one global reservation per (tile, partition), issued back to back by
      // the rank-0 element of each partition: counts first, then independent
      // atomics, then the bases
      __syncthreads();
#pragma unroll
      for (int j = 0; j < KPT; j++)
        if (pp[j] != kNone && rk[j] == 0) {
          rk[j] = s_hist[pp[j]];
          pp[j] |= kLead;
        }
#pragma unroll
      for (int j = 0; j < KPT; j++)
        if (pp[j] & kLead) rk[j] = atomicAdd(&pcount[pp[j] & ~kLead], rk[j]);
#pragma unroll
      for (int j = 0; j < KPT; j++)
        if (pp[j] & kLead) {
          pp[j] &= ~kLead;
          s_hist[pp[j]] = rk[j];
          rk[j] = 0;
        }
      __syncthreads();
    }
#pragma unroll
    for (int j = 0; j < KPT; j++) {
      if (pp[j] == kNone) continue;
      const uint32_t pos = (kSmemHist ? s_hist[pp[j]] : 0u) + rk[j];
      if (pos < bp.cap) pbuf[size_t(pp[j]) * bp.cap + pos] = e[j];
      else ovf = true;
    }
    if (kSmemHist) {
      __syncthreads();
#pragma unroll
      for (int j = 0; j < KPT; j++)
        if (pp[j] != kNone && rk[j] == 0) s_hist[pp[j]] = 0;
      __syncthreads();
    }
  }
  if (ovf) atomicOr(&stt->part_overflow, 1u);
  if (bad) atomicOr(&stt->pad, 1u);
  HM_TKA(1);
}

// ------------------------------------------------------------ K_A, two passes
// For large tables the partition step runs as two 128-way radix-partition
// passes over the partition id (high 7 bits, then low 7 bits): a 16K-way
// single pass writes ~one 16-byte element per partition per tile (scattered
// partial-sector stores), a 128-way pass writes runs of ~32 elements from a
// shared-memory staging tile, fully coalesced.  Ranking inside the tile uses
// warp ballots over the 7 digit bits and per-warp counters (no atomics).
constexpr int kSThreads = 512, kSPT = 4, kSTile = kSThreads * kSPT;
constexpr int kSWarps = kSThreads / 32, kSDigits = 256, kSBits = 8;  // 8-bit digits: up to 64K partitions in two passes

struct SplitArgs {
  // pass 2 source: the coarse buffer
  const void* cbuf;
  const unsigned int* ccount;
  uint32_t ccap;
  uint32_t tpc;  // tiles per coarse partition
  // destination
  void* dst;
  unsigned int* dcount;
  uint32_t dcap;
  uint32_t nreg;      // destination regions
  uint32_t nreg_src;  // pass 2: source (coarse) regions
};

template <class Src, class E, int PASS>
__global__ void __launch_bounds__(kSThreads, 2) k_split(Src src, BuildParams bp, SplitArgs a,
                                                        DevStatus* __restrict__ stt) {
  extern __shared__ __align__(16) uint8_t smem[];
  E* stage = reinterpret_cast<E*>(smem);
  uint8_t* sdig = smem + size_t(kSTile) * sizeof(E);
  __shared__ uint16_t s_wh[kSWarps][kSDigits];
  __shared__ uint32_t s_dstart[kSDigits], s_gbase[kSDigits];
  __shared__ unsigned long long s_red[kSWarps];

  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, lt = (1u << lane) - 1u;
  for (uint32_t i = tid; i < kSWarps * kSDigits / 2; i += kSThreads) reinterpret_cast<uint32_t*>(&s_wh[0][0])[i] = 0;
  // this CTA's elements
  uint64_t base;
  uint32_t nvalid, coarse = 0;
  const E* cb = reinterpret_cast<const E*>(a.cbuf);
  if (PASS == 1) {
    base = uint64_t(blockIdx.x) * kSTile;
    nvalid = bp.n_in - base < uint64_t(kSTile) ? uint32_t(bp.n_in - base) : uint32_t(kSTile);
  } else {
    coarse = blockIdx.x / a.tpc;
    const uint32_t k = blockIdx.x % a.tpc;
    const uint32_t cc = min(a.ccount[coarse], a.ccap);
    base = uint64_t(k) * kSTile;
    nvalid = cc > base ? (cc - base < uint64_t(kSTile) ? uint32_t(cc - base) : uint32_t(kSTile)) : 0u;
  }
  __syncthreads();
  if (nvalid == 0) return;
  E e[kSPT];
  uint32_t dg[kSPT], rk[kSPT];
  bool bad = false;
#pragma unroll
  for (int j = 0; j < kSPT; j++) {
    const uint32_t i = j * kSThreads + tid;
    if (i < nvalid) e[j] = PASS == 1 ? src.load(base + i) : cb[size_t(coarse) * a.ccap + base + i];
  }
#pragma unroll
  for (int j = 0; j < kSPT; j++) {
    const uint32_t i = j * kSThreads + tid;
    dg[j] = 0;
    if (i < nvalid) {
      const uint64_t lb = level1_bucket(bp.l1, e[j].key) - bp.b_lo;
      if (lb >= bp.nb) bad = true;
      const uint32_t p = uint32_t(lb >> bp.log2_bp);
      dg[j] = PASS == 1 ? ((p >> kSBits) & (kSDigits - 1)) : (p & (kSDigits - 1));
    }
  }
  // warp-ballot rank of every element among the warp's elements with its digit
#pragma unroll
  for (int j = 0; j < kSPT; j++) {
    const bool valid = j * kSThreads + tid < nvalid;
    uint32_t m = __ballot_sync(0xffffffffu, valid);
#pragma unroll
    for (int bit = 0; bit < kSBits; bit++) {
      const uint32_t bl = __ballot_sync(0xffffffffu, (dg[j] >> bit) & 1u);
      m &= ((dg[j] >> bit) & 1u) ? bl : ~bl;
    }
    const uint32_t below = m & lt;
    const uint32_t c = valid ? s_wh[warp][dg[j]] : 0u;
    __syncwarp();
    if (valid && below == 0) s_wh[warp][dg[j]] = uint16_t(c + __popc(m));
    __syncwarp();
    rk[j] = c + __popc(below);
  }
  __syncthreads();
  // digit-major offsets inside the tile; one global reservation per digit
  {
    uint32_t pre[kSWarps], tot = 0;
    if (tid < kSDigits) {
#pragma unroll
      for (int w = 0; w < kSWarps; w++) {
        pre[w] = tot;
        tot += s_wh[w][tid];
      }
    }
    unsigned long long t_all;
    const uint32_t ds = uint32_t(block_excl_scan(tot, &t_all, s_red));
    if (tid < kSDigits) {
#pragma unroll
      for (int w = 0; w < kSWarps; w++) s_wh[w][tid] = uint16_t(ds + pre[w]);
      s_dstart[tid] = ds;
      if (tot) {
        const uint32_t reg = PASS == 1 ? tid : coarse * kSDigits + tid;
        s_gbase[tid] = reg < a.nreg ? atomicAdd(&a.dcount[reg], tot) : 0xFFFFFFFFu;
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kSPT; j++) {
    if (j * kSThreads + tid < nvalid) {
      const uint32_t pos = s_wh[warp][dg[j]] + rk[j];
      stage[pos] = e[j];
      sdig[pos] = uint8_t(dg[j]);
    }
  }
  __syncthreads();
  // runs of equal digit are contiguous: consecutive threads write consecutive addresses
  E* dst = reinterpret_cast<E*>(a.dst);
  bool ovf = false;
  for (uint32_t i = tid; i < nvalid; i += kSThreads) {
    const uint32_t d = sdig[i];
    const uint32_t reg = PASS == 1 ? d : coarse * kSDigits + d;
    const uint32_t pos = s_gbase[d] + (i - s_dstart[d]);
    if (reg < a.nreg && pos < a.dcap) dst[size_t(reg) * a.dcap + pos] = stage[i];
    else ovf = true;
  }
  if (ovf) atomicOr(&stt->part_overflow, 1u);
  if (bad) atomicOr(&stt->pad, 1u);
}

// ------------------------------------------------------------------ K_B
// Size classes of multi-key buckets and the lane-group width G that searches
// one bucket: s=2 -> 2 lanes, s=3..4 -> 4, s=5..8 -> 8, s=9..32 -> 32.
constexpr int kNCls = 4;
__device__ __forceinline__ int size_class(uint32_t s) { return s == 2 ? 0 : s <= 4 ? 1 : s <= 8 ? 2 : s <= 32 ? 3 : 4; }
__device__ __forceinline__ int class_log2g(int c) { return c == 0 ? 1 : c == 1 ? 2 : c == 2 ? 3 : 5; }

template <class E>
__device__ __forceinline__ E shfl_elem(const E& e, int src) {
  constexpr int W = sizeof(E) / 8;
  const uint64_t* p = reinterpret_cast<const uint64_t*>(&e);
  E out;
  uint64_t* q = reinterpret_cast<uint64_t*>(&out);
#pragma unroll
  for (int w = 0; w < W; w++) q[w] = __shfl_sync(0xffffffffu, p[w], src);
  return out;
}

// make2 for one size class, K key registers per thread.
// Every thread owns one bucket at a time and makes one attempt per loop
// iteration: derive(seed,2,b,t), the s level-2 slots hash mod s^2, and an
// occupancy bitmap as `collision`.  Threads that finish take
// the next bucket of the class from a shared counter (one warp-aggregated
// atomic per refill), so the spread of attempt counts does not idle the warp.
template <int K, class E, class Same>
__device__ __forceinline__ void search_threads(const BuildParams& bp, const E* part, const uint64_t* skey,
                                               const uint16_t* list, uint32_t L,
                                               uint32_t* next, const uint16_t* sstart, const uint16_t* sidx,
                                               uint16_t* sA, uint8_t* s_t, const uint64_t* s_m2, uint64_t bbase,
                                               DevStatus* stt, const Same& same) {
  const uint32_t lane = threadIdx.x & 31, lt = (1u << lane) - 1u;
  bool have = false, drained = false;
  uint32_t lb = 0, st0 = 0, s = 2, t = 0;
  uint64_t k[K];
  FastMod fm{4, s_m2[2]};
#pragma unroll
  for (int j = 0; j < K; j++) k[j] = 0;
  while (true) {
    const bool need = !have && !drained;
    const uint32_t nm = __ballot_sync(0xffffffffu, need);
    if (nm) {
      const uint32_t leader = __ffs(nm) - 1;
      uint32_t b0 = 0;
      if (lane == leader) b0 = atomicAdd(next, uint32_t(__popc(nm)));
      b0 = __shfl_sync(0xffffffffu, b0, leader);
      if (need) {
        const uint32_t idx = b0 + __popc(nm & lt);
        if (idx < L) {
          lb = list[idx];
          st0 = sstart[lb];
          s = uint32_t(sstart[lb + 1]) - st0;
          t = 0;
          have = true;
          fm = FastMod{uint64_t(s) * s, s_m2[s]};
#pragma unroll
          for (int j = 0; j < K; j++) k[j] = uint32_t(j) < s ? skey[sidx[st0 + j]] : 0ull;
        } else {
          drained = true;
        }
      }
    }
    if (!__any_sync(0xffffffffu, have)) break;
    if (have) {
      const Consts c = derive(bp.smix, 2, bbase + lb, t);
      uint64_t bits = 0;
      bool coll = false;
      uint32_t h[K];
#pragma unroll
      for (int j = 0; j < K; j++) {
        h[j] = 0;
        if (uint32_t(j) < s) {
          const uint64_t hv = hash64(c, k[j]);
          // mod s^2: a mask when s is a power of two (always for the s = 2 class)
          h[j] = (K == 2 || (s & (s - 1)) == 0) ? uint32_t(hv) & (s * s - 1) : uint32_t(fastmod(hv, fm));
          const uint64_t bit = 1ull << h[j];
          coll |= (bits & bit) != 0;
          bits |= bit;
        }
      }
      bool done = false;
      if (!coll) {
#pragma unroll
        for (int j = 0; j < K; j++)
          if (uint32_t(j) < s) sA[st0 + j] = uint16_t(h[j]);
        done = true;
      } else {
        if (t == 0) {  // equal keys collide under every t: check the bucket once
          int di = -1, dj = -1;
#pragma unroll
          for (int i = 0; i < K; i++)
#pragma unroll
            for (int j = i + 1; j < K; j++)
              if (uint32_t(j) < s && k[i] == k[j] && di < 0) {
                di = i;
                dj = j;
              }
          if (di >= 0) {
            const bool d = same.same(part[sidx[st0 + di]], part[sidx[st0 + dj]]);
            atomicOr(d ? &stt->dup : &stt->fpcoll, 1u);
            done = true;
          }
        }
        if (!done) {
          if (t + 1 >= kT2Cap) {
            atomicOr(&stt->exhausted, 1u);
            t = 0;
            done = true;
          } else {
            t++;
          }
        }
      }
      if (done) {
        s_t[lb] = uint8_t(t);
        have = false;
      }
    }
  }
}

// make2 for the rare 9 <= s <= 32 buckets: a warp per bucket, a lane per key,
// __match_any_sync on the level-2 slots as the injectivity test.
template <class E, class Same>
__device__ __forceinline__ void search_warp(const BuildParams& bp, const E* part, const uint64_t* skey,
                                            const uint16_t* list, uint32_t L,
                                            const uint16_t* sstart, const uint16_t* sidx, uint16_t* sA, uint8_t* s_t,
                                            const uint64_t* s_m2, uint64_t bbase, DevStatus* stt, const Same& same) {
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (uint32_t idx = warp; idx < L; idx += kBWarps) {
    const uint32_t lb = list[idx], st0 = sstart[lb], s = uint32_t(sstart[lb + 1]) - st0;
    const bool mine = lane < s;
    const uint64_t key = mine ? skey[sidx[st0 + lane]] : 0ull;
    const uint32_t valid = __ballot_sync(0xffffffffu, mine);
    const uint32_t dm = __match_any_sync(0xffffffffu, key) & valid & ~(1u << lane);
    uint32_t t = 0;
    if (__any_sync(0xffffffffu, mine && dm != 0)) {
      if (mine && dm != 0) {
        const bool d = same.same(part[sidx[st0 + lane]], part[sidx[st0 + __ffs(dm) - 1]]);
        atomicOr(d ? &stt->dup : &stt->fpcoll, 1u);
      }
    } else {
      const FastMod fm{uint64_t(s) * s, s_m2[s]};
      uint32_t h = 0;
      for (t = 0; t < kT2Cap; t++) {
        const Consts c = derive(bp.smix, 2, bbase + lb, t);
        h = uint32_t(fastmod(hash64(c, key), fm));
        const uint32_t mh = __match_any_sync(0xffffffffu, mine ? h : (0x80000000u | lane));
        if (!__any_sync(0xffffffffu, mine && __popc(mh) > 1)) break;
      }
      if (t >= kT2Cap) {
        if (lane == 0) atomicOr(&stt->exhausted, 1u);
        t = 0;
      } else if (mine) {
        sA[st0 + lane] = uint16_t(h);
      }
    }
    if (lane == 0) s_t[lb] = uint8_t(t);
  }
}

// Table write of one class, thread per bucket: members at soff + h, unused
// slots get the lowest-slot member with value 0 (R10).
template <int K, class E>
__device__ __forceinline__ void write_threads(const uint16_t* list, uint32_t L, const uint16_t* sstart,
                                              const uint16_t* sidx, const uint16_t* sA, const E* part, E* slots,
                                              unsigned long long base, const uint32_t* s_cbase, const uint16_t* srel,
                                              uint32_t lgch) {
  for (uint32_t idx = threadIdx.x; idx < L; idx += kBThreads) {
    const uint32_t lb = list[idx], st0 = sstart[lb], s = uint32_t(sstart[lb + 1]) - st0;
    const uint64_t soff = base + s_cbase[lb >> lgch] + srel[lb];
    E e[K];
    uint32_t h[K];
#pragma unroll
    for (int j = 0; j < K; j++)  // all member loads in flight before any store
      if (uint32_t(j) < s) {
        h[j] = sA[st0 + j];
        e[j] = part[sidx[st0 + j]];
      }
    uint64_t bits = 0;
    uint32_t hmin = 0xFFFFu;
    int jmin = 0;
#pragma unroll
    for (int j = 0; j < K; j++) {
      if (uint32_t(j) < s) {
        slots[soff + h[j]] = e[j];
        bits |= 1ull << h[j];
        if (h[j] < hmin) {
          hmin = h[j];
          jmin = j;
        }
      }
    }
    E f = e[0];
#pragma unroll
    for (int j = 1; j < K; j++)
      if (j == jmin) f = e[j];
    f.value = 0;
    const uint32_t s2 = s * s;
    for (uint32_t x = 0; x < s2; x++)
      if (!((bits >> x) & 1)) slots[soff + x] = f;
  }
}

template <class E>
__device__ __forceinline__ void write_warp(const uint16_t* list, uint32_t L, const uint16_t* sstart,
                                           const uint16_t* sidx, const uint16_t* sA, const E* part, E* slots,
                                           unsigned long long base, const uint32_t* s_cbase, const uint16_t* srel,
                                           uint32_t lgch, uint32_t* bitsw) {
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (uint32_t idx = warp; idx < L; idx += kBWarps) {
    const uint32_t lb = list[idx], st0 = sstart[lb], s = uint32_t(sstart[lb + 1]) - st0;
    const uint64_t soff = base + s_cbase[lb >> lgch] + srel[lb];
    const bool mine = lane < s;
    uint32_t h = 0xFFFFu;
    E e;
    bitsw[lane] = 0;
    __syncwarp();
    if (mine) {
      h = sA[st0 + lane];
      e = part[sidx[st0 + lane]];
      slots[soff + h] = e;
      atomicOr(&bitsw[h >> 5], 1u << (h & 31));
    }
    const uint32_t hmin = __reduce_min_sync(0xffffffffu, h);
    const uint32_t who = __ffs(__ballot_sync(0xffffffffu, mine && h == hmin)) - 1;
    E f = shfl_elem(e, who);
    f.value = 0;
    __syncwarp();
    for (uint32_t x = lane; x < s * s; x += 32)
      if (!((bitsw[x >> 5] >> (x & 31)) & 1)) slots[soff + x] = f;
    __syncwarp();
  }
}

// Dynamic shared memory of k_bucket (all offsets 16-byte aligned).  Regions
// are reused once their first use is over (see the phase comments).
struct BucketSmem {
  size_t skey, sA, sidx, tmp, whist, sstart, st, total;
};
__host__ __device__ __forceinline__ size_t al16(size_t x) { return (x + 15) & ~size_t(15); }
__host__ __device__ __forceinline__ uint32_t bucket_chunk(uint32_t BP) {  // buckets per owner thread
  return BP / kBThreads > 2 ? BP / kBThreads : 2;
}
__host__ __device__ __forceinline__ BucketSmem bucket_smem_layout(uint32_t cap, uint32_t BP) {
  const uint32_t CH = bucket_chunk(BP), nown = BP / CH;
  size_t wh = size_t(kBWarps) * nown * 2;                      // P1-P3: per-warp owner counters
  wh = wh > size_t(CH) * kBThreads * 2 ? wh : size_t(CH) * kBThreads * 2;  // P4: per-thread bucket counters
  wh = wh > (size_t(cap) / 2 + 8) * 2 ? wh : (size_t(cap) / 2 + 8) * 2;   // then: class lists
  BucketSmem L;
  L.skey = 0;                                           // u64[cap]: the partition's keys (item order)
  L.sA = L.skey + al16(size_t(cap) * 8);                // u16[cap]: bucket of item i; later level-2 slot of position
  L.sidx = L.sA + al16(size_t(cap) * 2);                // u16[cap]: P1-P3 warp rank of item; P4+ position -> item
  L.tmp = L.sidx + al16(size_t(cap) * 2);               // u16[max(cap,BP)]: owner-grouped items; P4c+ slot offset in chunk
  L.whist = L.tmp + al16(size_t(cap > BP ? cap : BP) * 2);
  L.sstart = L.whist + al16(wh);                        // u16[BP+1]: first position of each bucket
  L.st = L.sstart + al16((size_t(BP) + 1) * 2);         // u8[BP]: attempt t of each bucket
  L.total = L.st + al16(BP);
  return L;
}

template <class E, class Same>
__global__ void __launch_bounds__(kBThreads, 1024 / kBThreads)
    k_bucket(BuildParams bp, const E* __restrict__ pbuf, const unsigned int* __restrict__ pcount,
             unsigned long long* __restrict__ lbstate, uint64_t* __restrict__ dir, CDir* __restrict__ cdir,
             E* __restrict__ slots, DevStatus* __restrict__ stt, Same same) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ uint64_t s_m2[33];
  __shared__ uint32_t s_p;
  __shared__ unsigned long long s_red[kBWarps];
  __shared__ unsigned long long s_base;
  __shared__ uint32_t s_cls_off[kNCls + 1];
  __shared__ uint32_t s_bits[kBWarps][32];
  __shared__ uint32_t s_cbase[kBThreads];  // slot offset of each thread's bucket chunk in the partition
  __shared__ uint32_t s_next[kNCls];        // work counters of the search classes

  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_p = atomicAdd(&stt->ticket, 1u);
  if (tid < 33) s_m2[tid] = tid ? ~0ull / (uint64_t(tid) * tid) : 0ull;
  __syncthreads();
  const uint32_t p = s_p;
  HM_TMARK(0);
  const uint32_t cap = bp.cap;
  const uint32_t BP = 1u << bp.log2_bp;
  const uint32_t CH = bucket_chunk(BP), lgch = 31 - __clz(CH), nown = BP / CH, obits = 31 - __clz(nown);
  const uint64_t lb0 = uint64_t(p) << bp.log2_bp;
  const uint32_t nbp = uint32_t(bp.nb - lb0 < uint64_t(BP) ? bp.nb - lb0 : uint64_t(BP));
  const uint32_t cnt_raw = pcount[p];
  const bool ovf = cnt_raw > cap;
  const uint32_t cnt = ovf ? 0u : cnt_raw;
  const BucketSmem SL = bucket_smem_layout(cap, BP);
  uint64_t* skey = reinterpret_cast<uint64_t*>(smem + SL.skey);
  uint16_t* sA = reinterpret_cast<uint16_t*>(smem + SL.sA);
  uint16_t* srk = reinterpret_cast<uint16_t*>(smem + SL.sidx);   // P1-P3
  uint16_t* sidx = srk;                                           // P4+
  uint16_t* tmp = reinterpret_cast<uint16_t*>(smem + SL.tmp);    // P3-P4b
  uint16_t* srel = tmp;                                           // P4c+
  uint16_t* whist = reinterpret_cast<uint16_t*>(smem + SL.whist); // P1-P3
  uint16_t* scnt = whist;                                         // P4a-P4b
  uint16_t* slist = whist;                                        // P4c+
  uint16_t* sstart = reinterpret_cast<uint16_t*>(smem + SL.sstart);
  uint8_t* s_t = smem + SL.st;
  for (uint32_t w = tid; w < kBWarps * nown / 2; w += kBThreads) reinterpret_cast<uint32_t*>(whist)[w] = 0;
  __syncthreads();
  const E* part = pbuf + size_t(p) * cap;
  const uint64_t bbase = bp.b_lo + lb0;  // global id of the partition's first bucket

  // groupby of the partition's items by bucket without shared
  // atomics: P1 ranks every item among the items of its owner thread (the
  // thread owning CH consecutive buckets) with `obits` warp ballots and
  // per-warp counters; P2 scans the counters; P3 scatters into owner order;
  // P4 groups each owner's ~CH items by bucket with thread-private counters.
  HM_TMARK(1);
  // ---- P1: level-1 bucket g k, warp-level owner rank
  const uint32_t lt = (1u << lane) - 1u;
  uint16_t* wh = whist + warp * nown;
  for (uint32_t i0 = warp * 32; i0 < cnt; i0 += 8 * kBThreads) {
    uint64_t ks[8];
    uint32_t lbs[8];
#pragma unroll
    for (int j = 0; j < 8; j++) {  // the partition's keys are read from HBM once, 8 loads in flight
      const uint32_t i = i0 + j * kBThreads + lane;
      ks[j] = i < cnt ? part[i].key : 0ull;
    }
#pragma unroll
    for (int j = 0; j < 8; j++) {
      const uint32_t i = i0 + j * kBThreads + lane;
      lbs[j] = 0;
      if (i < cnt) {
        skey[i] = ks[j];
        lbs[j] = uint32_t(level1_bucket(bp.l1, ks[j]) - bbase);
        if (lbs[j] >= nbp) {  // cannot happen for a well-routed partition; never index out of range
          atomicOr(&stt->pad, 1u);
          lbs[j] = 0;
        }
      }
    }
#pragma unroll
    for (int j = 0; j < 8; j++) {
      const uint32_t i = i0 + j * kBThreads + lane;
      const bool valid = i < cnt;
      const uint32_t o = lbs[j] >> lgch;
      uint32_t m = __ballot_sync(0xffffffffu, valid);
      for (uint32_t bit = 0; bit < obits; bit++) {
        const uint32_t bl = __ballot_sync(0xffffffffu, (o >> bit) & 1u);
        m &= ((o >> bit) & 1u) ? bl : ~bl;
      }
      const uint32_t below = m & lt;
      const uint32_t wc = valid ? wh[o] : 0u;
      __syncwarp();
      if (valid && below == 0) wh[o] = uint16_t(wc + __popc(m));
      __syncwarp();
      if (valid) {
        sA[i] = uint16_t(lbs[j]);
        srk[i] = uint16_t(wc + __popc(below));
      }
    }
  }
  __syncthreads();
  HM_TMARK(2);
  // ---- P2: owner totals and offsets (owner-major, warp-minor)
  uint32_t ostart = 0, otot = 0;
  {
    uint32_t pre[kBWarps];
    if (tid < nown) {
#pragma unroll
      for (int w = 0; w < kBWarps; w++) {
        pre[w] = otot;
        otot += whist[w * nown + tid];
      }
    }
    unsigned long long tot;
    ostart = uint32_t(block_excl_scan(otot, &tot, s_red));
    if (tid < nown) {
#pragma unroll
      for (int w = 0; w < kBWarps; w++) whist[w * nown + tid] = uint16_t(ostart + pre[w]);
    }
  }
  __syncthreads();
  HM_TMARK(3);
  // ---- P3: scatter items into owner order
  for (uint32_t i0 = warp * 32; i0 < cnt; i0 += kBThreads) {
    const uint32_t i = i0 + lane;
    if (i < cnt) tmp[wh[sA[i] >> lgch] + srk[i]] = uint16_t(i);
  }
  __syncthreads();
  HM_TMARK(4);
  // ---- P4a/b: each owner groups its items by bucket (thread-private counters)
  if (tid < nown) {
    for (uint32_t k = 0; k < CH; k++) scnt[k * kBThreads + tid] = 0;
    for (uint32_t q = ostart; q < ostart + otot; q++) scnt[(sA[tmp[q]] & (CH - 1)) * kBThreads + tid]++;
    uint32_t run = ostart;
    for (uint32_t k = 0; k < CH; k++) {
      const uint32_t c = scnt[k * kBThreads + tid];
      scnt[k * kBThreads + tid] = uint16_t(run);
      sstart[tid * CH + k] = uint16_t(run);
      run += c;
    }
    for (uint32_t q = ostart; q < ostart + otot; q++) {
      const uint32_t i = tmp[q];
      uint16_t* c = &scnt[(sA[i] & (CH - 1)) * kBThreads + tid];
      sidx[*c] = uint16_t(i);
      *c = uint16_t(*c + 1);
    }
  }
  if (tid == 0) sstart[BP] = uint16_t(cnt);
  __syncthreads();
  HM_TMARK(5);
  // ---- P4c: sizes, s^2 offsets (presum, R1/R2), class lists
  const uint32_t c0 = tid * CH, c1 = min(c0 + CH, nbp);
  uint32_t lsq = 0, maxs = 0;
  unsigned long long lcls = 0;
  for (uint32_t j = c0; j < c1; j++) {
    const uint32_t v = uint32_t(sstart[j + 1]) - sstart[j];
    lsq += v * v;
    maxs = max(maxs, v);
    if (v >= 2) {
      const int c = size_class(v);
      if (c < kNCls && uint64_t(v) * v <= bp.bound4n) lcls += 1ull << (16 * c);
    }
  }
  unsigned long long S_p, totB;
  const uint32_t exsq = uint32_t(block_excl_scan(lsq, &S_p, s_red));
  const unsigned long long exB = block_excl_scan(lcls, &totB, s_red);
  if (tid == 0) {
    s_cls_off[0] = 0;
    for (int c = 0; c < kNCls; c++) s_cls_off[c + 1] = s_cls_off[c] + uint32_t((totB >> (16 * c)) & 0xFFFF);
  }
  s_cbase[tid] = exsq;
  __syncthreads();
  {
    uint32_t ccur[kNCls];
#pragma unroll
    for (int c = 0; c < kNCls; c++) ccur[c] = s_cls_off[c] + uint32_t((exB >> (16 * c)) & 0xFFFF);
    bool huge = false, bfail = false;
    uint32_t fsq = 0;
    for (uint32_t j = c0; j < c1; j++) {
      const uint32_t v = uint32_t(sstart[j + 1]) - sstart[j];
      srel[j] = uint16_t(fsq);
      fsq += v * v;
      s_t[j] = 0;
      if (v >= 2) {
        const int c = size_class(v);
        if (uint64_t(v) * v > bp.bound4n) bfail = true;  // S > 4n: level one redraws
        else if (c >= kNCls) huge = true;
        else slist[ccur[c]++] = uint16_t(j);
      }
    }
    if (fsq > 0xFFFFu) huge = true;
    if (huge) atomicOr(&stt->huge, 1u);
    if (bfail || uint64_t(maxs) * maxs > bp.bound4n) atomicOr(&stt->bound_fail, 1u);
  }
  // publish the partition's aggregate S_p now (decoupled look-back); the
  // exclusive prefix is looked up after the search, when the predecessors
  // have long published theirs
  if (tid == 0) st_release(&lbstate[p], (p == 0 ? kFlagInc : kFlagAgg) | (S_p & kValMask));
  if (tid < kNCls) s_next[tid] = 0;
  __syncthreads();

  // from here: bucket lb holds positions [sstart[lb], sstart[lb+1]); sidx[pos] = item;
  // slot offset within the partition = s_cbase[lb / CH] + srel[lb]

  HM_TMARK(6);
  // level-2 seed search, map make2 over the multi-key buckets:
  // warp-per-bucket for 9 <= s <= 32, then thread-per-bucket classes from the
  // rarest (longest chains) to the most common, so the tail of the last class
  // is short and early warps go on to the singleton slots
  search_warp(bp, part, skey, slist + s_cls_off[3], s_cls_off[4] - s_cls_off[3], sstart, sidx, sA, s_t, s_m2, bbase, stt,
              same);
  search_threads<8>(bp, part, skey, slist + s_cls_off[2], s_cls_off[3] - s_cls_off[2], &s_next[2], sstart, sidx, sA, s_t,
                    s_m2, bbase, stt, same);
  search_threads<4>(bp, part, skey, slist + s_cls_off[1], s_cls_off[2] - s_cls_off[1], &s_next[1], sstart, sidx, sA, s_t,
                    s_m2, bbase, stt, same);
  search_threads<2>(bp, part, skey, slist + s_cls_off[0], s_cls_off[1] - s_cls_off[0], &s_next[0], sstart, sidx, sA, s_t,
                    s_m2, bbase, stt, same);
  HM_TMARK(7);
  // look-back: exclusive prefix of S over the partitions before p (warp 0,
  // lane i inspects partition q0 - i: the closest inclusive prefix plus the
  // aggregates in front of it give the base)
  if (warp == 0) {
    unsigned long long base = 0;
    if (p > 0) {
      int64_t q0 = int64_t(p) - 1;
      while (true) {
        const int64_t q = q0 - int64_t(lane);
        const unsigned long long v = q >= 0 ? ld_acquire(&lbstate[q]) : kFlagInc;
        const unsigned long long f = v & ~kValMask;
        const uint32_t notready = __ballot_sync(0xffffffffu, f == 0);
        const uint32_t incs = __ballot_sync(0xffffffffu, f == kFlagInc);
        const uint32_t upto = incs ? (__ffs(incs) - 1) : 31u;  // lanes 0..upto are needed
        const uint32_t need = upto == 31u ? 0xffffffffu : ((2u << upto) - 1u);
        if (notready & need) continue;  // a closer partition has not published yet
        unsigned long long x = lane <= upto ? (v & kValMask) : 0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        base += x;
        if (incs) break;
        q0 -= 32;
      }
      if (lane == 0) st_release(&lbstate[p], kFlagInc | ((base + S_p) & kValMask));
    }
    if (lane == 0) {
      if (p == bp.np - 1) stt->S = base + S_p;
      s_base = base;
    }
  }
  __syncthreads();
  const unsigned long long base = s_base;
  if (ovf) {
    if (tid == 0) atomicOr(&stt->part_overflow, 1u);
    return;
  }
  if (base + S_p > bp.slot_cap) {
    if (tid == 0) atomicOr(&stt->slot_overflow, 1u);
    return;
  }


  // singleton slots (R12: a singleton sits at soff) need no search result;
  // 8 element loads in flight per thread, then the stores
  for (uint32_t lb0s = 0; lb0s < nbp; lb0s += 8 * kBThreads) {
    E ev[8];
    uint64_t so[8];
#pragma unroll
    for (int j = 0; j < 8; j++) {
      const uint32_t lb = lb0s + j * kBThreads + tid;
      so[j] = ~0ull;
      if (lb < nbp) {
        const uint32_t st0 = sstart[lb];
        if (uint32_t(sstart[lb + 1]) - st0 == 1) {
          so[j] = base + s_cbase[lb >> lgch] + srel[lb];
          ev[j] = part[sidx[st0]];
        }
      }
    }
#pragma unroll
    for (int j = 0; j < 8; j++)
      if (so[j] != ~0ull) slots[so[j]] = ev[j];
  }

  HM_TMARK(8);
  // directory (coalesced) and compact directory record per 32 buckets (one per
  // warp iteration)
  for (uint32_t cb = 0; cb < nbp; cb += kBThreads) {
    const uint32_t lb = cb + tid;
    uint32_t s = 0, t = 0, st0 = 0;
    uint64_t soff = 0;
    if (lb < nbp) {
      st0 = sstart[lb];
      s = uint32_t(sstart[lb + 1]) - st0;
      t = s_t[lb];
      soff = base + s_cbase[lb >> lgch] + srel[lb];
      dir[lb0 + lb] = dir_entry(soff, s, t);
    }
    uint32_t pa = __ballot_sync(0xffffffffu, s & 4), pb = __ballot_sync(0xffffffffu, s & 2),
             pc = __ballot_sync(0xffffffffu, s & 1);
    const uint32_t t0 = __ballot_sync(0xffffffffu, t & 1), t1 = __ballot_sync(0xffffffffu, t & 2),
                   t2 = __ballot_sync(0xffffffffu, t & 4), t3 = __ballot_sync(0xffffffffu, t & 8);
    if (__any_sync(0xffffffffu, s >= kCdirEscS || t >= kCdirEscT) || (bp.flags & HM_FLAG_FULL_DIRECTORY))
      pa = pb = pc = 0xffffffffu;
    if (lane == 0 && lb < nbp) {
      CDir r;
      r.w[0] = uint32_t(soff);
      r.w[1] = pa;
      r.w[2] = pb;
      r.w[3] = pc;
      r.w[4] = t0;
      r.w[5] = t1;
      r.w[6] = t2;
      r.w[7] = t3;
      cdir[(lb0 + lb) >> 5] = r;
    }
  }
  HM_TMARK(9);
  // multi-key buckets: members at soff + h, every unused slot gets the
  // lowest-slot member with value 0 (R10)
  write_threads<2>(slist + s_cls_off[0], s_cls_off[1] - s_cls_off[0], sstart, sidx, sA, part, slots, base, s_cbase,
                   srel, lgch);
  write_threads<4>(slist + s_cls_off[1], s_cls_off[2] - s_cls_off[1], sstart, sidx, sA, part, slots, base, s_cbase,
                   srel, lgch);
  write_threads<8>(slist + s_cls_off[2], s_cls_off[3] - s_cls_off[2], sstart, sidx, sA, part, slots, base, s_cbase,
                   srel, lgch);
  write_warp(slist + s_cls_off[3], s_cls_off[4] - s_cls_off[3], sstart, sidx, sA, part, slots, base, s_cbase, srel,
             lgch, s_bits[warp]);
  HM_TMARK(10);
}

// ------------------------------------------------------------- host side
static size_t bucket_smem_bytes(uint32_t cap, uint32_t log2_bp) {
  return bucket_smem_layout(cap, 1u << log2_bp).total;
}

struct Plan {
  uint32_t log2_bp, np, cap;
  size_t smemB;
};

static Plan make_plan(uint64_t n_in, uint64_t nb, uint32_t log2_req, size_t smem_limit) {
  Plan pl{};
  const int sms = num_sms();
  // 8K buckets per partition (two CTAs of k_bucket per SM); 16K when that
  // would make more than 32K partitions (k_partition's shared histogram)
  uint32_t lg = log2_req ? log2_req : ((nb >> HM_KB_LOG2BP) > 32768 ? 14 : HM_KB_LOG2BP);
  if (!log2_req) {
    while (lg > 6 && (nb >> lg) < uint64_t(4 * sms)) lg--;
  }
  for (;; lg--) {
    const double BP = double(uint64_t(1) << lg);
    const double m = double(n_in) * BP / double(std::max<uint64_t>(nb, 1));
    double c = m + 8.0 * std::sqrt(std::max(m, 1.0)) + 64.0;
    uint32_t cap = uint32_t(std::min(65535.0, std::ceil(c / 32.0) * 32.0));
    if (cap > 65535u) cap = 65535u;
    const size_t sm = bucket_smem_bytes(cap, lg);
    if ((sm <= smem_limit && c <= 65535.0) || lg <= 1) {
      pl.log2_bp = lg;
      pl.cap = cap;
      pl.smemB = sm;
      break;
    }
  }
  pl.np = uint32_t((nb + (uint64_t(1) << pl.log2_bp) - 1) >> pl.log2_bp);
  return pl;
}

template <class T>
static hm_status dmalloc(T** p, size_t bytes, cudaStream_t st) {
  void* v = nullptr;
  cudaError_t e = cudaMallocAsync(&v, std::max<size_t>(bytes, 16), st);
  if (e != cudaSuccess) {
    cudaGetLastError();
    set_error(std::string("cudaMallocAsync(") + std::to_string(bytes) + ") failed: " + cudaGetErrorString(e));
    return HM_ERR_OOM;
  }
  *p = reinterpret_cast<T*>(v);
  return HM_OK;
}

// Build scratch, cached per (device, stream) between builds.  The partition
// buffers have the same sizes build after build; taking them from the
// stream-ordered pool each time cost up to 5.4 ms of page mapping per build
// (measured on the 2^24-string config, when the pool was fragmented by the
// maps' own arrays), so they stay allocated until hm_release_workspace().
// Reuse is safe because everything that touches a stream's workspace is
// ordered on that stream.
enum WsRole { WS_FP, WS_BAD, WS_PBUF, WS_PCOUNT, WS_LBSTATE, WS_DSTAT, WS_CBUF, WS_CCOUNT, WS_NROLES };
struct Workspace {
  void* p[WS_NROLES] = {};
  size_t bytes[WS_NROLES] = {};
};
static std::mutex g_ws_mu;
static std::map<std::pair<int, cudaStream_t>, Workspace> g_ws;

struct Scratch {
  cudaStream_t st;
  template <class T>
  hm_status alloc(WsRole role, T** out, size_t bytes) {
    int dev = 0;
    HM_CUDA_TRY(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(g_ws_mu);
    Workspace& w = g_ws[{dev, st}];
    bytes = std::max<size_t>(bytes, 16);
    if (w.bytes[role] < bytes) {
      if (w.p[role]) cudaFreeAsync(w.p[role], st);
      w.p[role] = nullptr;
      w.bytes[role] = 0;
      void* v = nullptr;
      hm_status s = dmalloc(&v, bytes, st);
      if (s != HM_OK) return s;
      w.p[role] = v;
      w.bytes[role] = bytes;
    }
    *out = reinterpret_cast<T*>(w.p[role]);
    return HM_OK;
  }
};

// Frees every cached workspace of the current device (stream-ordered on the
// stream that owns it).
hm_status release_workspace() {
  int dev = 0;
  HM_CUDA_TRY(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_ws_mu);
  for (auto it = g_ws.begin(); it != g_ws.end();) {
    if (it->first.first == dev) {
      for (int r = 0; r < WS_NROLES; r++)
        if (it->second.p[r]) cudaFreeAsync(it->second.p[r], it->first.second);
      it = g_ws.erase(it);
    } else {
      ++it;
    }
  }
  HM_CUDA_TRY(cudaDeviceSynchronize());
  return HM_OK;
}

// Builds one table for buckets [b_lo, b_lo+nb) of a level-1 function mod
// n_global from the n_in elements produced by `src`.
template <class Src, class E, class Same>
static hm_status build_core(Src src, Same same, uint64_t n_in, uint64_t n_global, uint64_t b_lo, uint64_t nb,
                            int t1_fixed, uint64_t seed, uint32_t log2_req, cudaStream_t st, BuildOut* out,
                            bool* fpcoll) {
  *fpcoll = false;
  int dev = 0;
  HM_CUDA_TRY(cudaGetDevice(&dev));
  int smem_optin = 0;
  HM_CUDA_TRY(cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  const size_t static_smem_B = 6144;  // upper bound for k_bucket static shared memory (4.5 KB)
  const uint32_t knob_flags = log2_req >> 16;
  log2_req &= 0xFFFFu;
  const Plan pl = make_plan(n_in, nb, log2_req, size_t(smem_optin) - static_smem_B);
  if (pl.smemB + static_smem_B > size_t(smem_optin)) {
    set_error("build plan does not fit in shared memory");
    return HM_ERR_TOO_LARGE;
  }
  const int sms = num_sms();
  const uint64_t smix = seed_mix(seed);

  Scratch sc{st};
  E* pbuf = nullptr;
  unsigned int* pcount = nullptr;
  unsigned long long* lbstate = nullptr;
  DevStatus* dstat = nullptr;
  hm_status s;
  if ((s = sc.alloc(WS_PBUF, &pbuf, size_t(pl.np) * pl.cap * sizeof(E))) != HM_OK) return s;
  if ((s = sc.alloc(WS_PCOUNT, &pcount, size_t(pl.np) * 4)) != HM_OK) return s;
  if ((s = sc.alloc(WS_LBSTATE, &lbstate, size_t(pl.np) * 8)) != HM_OK) return s;
  if ((s = sc.alloc(WS_DSTAT, &dstat, sizeof(DevStatus))) != HM_OK) return s;

  uint64_t* dir = nullptr;
  E* slots = nullptr;
  CDir* cdir = nullptr;
  if ((s = dmalloc(&dir, nb * 8, st)) != HM_OK) return s;
  if ((s = dmalloc(&cdir, ((nb + 31) / 32) * sizeof(CDir), st)) != HM_OK) {
    cudaFreeAsync(dir, st);
    return s;
  }
  const double sn = double(n_in);
  uint64_t slot_cap = uint64_t(2.0 * sn + 8.0 * std::sqrt(2.0 * sn + 1.0) + 1024.0);
  if (n_in <= 4096) slot_cap = std::max<uint64_t>(slot_cap, 4 * std::max<uint64_t>(n_in, 1));
  if ((s = dmalloc(&slots, slot_cap * sizeof(E), st)) != HM_OK) {
    cudaFreeAsync(dir, st);
    cudaFreeAsync(cdir, st);
    return s;
  }
  auto fail = [&](hm_status code) {
    cudaFreeAsync(dir, st);
    cudaFreeAsync(cdir, st);
    cudaFreeAsync(slots, st);
    return code;
  };

  // kernel configuration
  constexpr int KPT = sizeof(E) == 16 ? 16 : 8;
  const size_t smemA = size_t(pl.np) * 4;
  const bool smemHist = smemA <= size_t(smem_optin) - 1024 && !getenv("HM_KA_GLOBAL");
  auto kA_s = k_partition<Src, E, KPT, true>;
  auto kA_g = k_partition<Src, E, KPT, false>;
  auto kB = k_bucket<E, Same>;
  if (smemHist) HM_CUDA_TRY(cudaFuncSetAttribute(kA_s, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smemA)));
  HM_CUDA_TRY(cudaFuncSetAttribute(kB, cudaFuncAttributeMaxDynamicSharedMemorySize, int(pl.smemB)));
  int occA = 1;
  if (smemHist) HM_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occA, kA_s, kAThreads, smemA));
  else HM_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occA, kA_g, kAThreads, 0));
  occA = std::max(occA, 1);
  const uint64_t T = uint64_t(kAThreads) * KPT;
  const uint64_t ntiles = (n_in + T - 1) / T;
  const unsigned gridA = unsigned(std::max<uint64_t>(1, std::min<uint64_t>(ntiles, uint64_t(sms) * occA)));
  // large tables: two coalesced 128-way passes instead of one 16K-way scatter
  const bool two_pass = sizeof(E) == 16 && pl.np > 1024 && pl.np <= 65536 && !getenv("HM_ONE_PASS");
  uint32_t ncoarse = 0, ccap = 0, tpc = 0;
  E* cbuf = nullptr;
  unsigned int* ccount = nullptr;
  const size_t smemS = size_t(kSTile) * (sizeof(E) + 1);
  auto kS1 = k_split<Src, E, 1>;
  auto kS2 = k_split<Src, E, 2>;
  if (two_pass) {
    ncoarse = (pl.np + kSDigits - 1) / kSDigits;
    const double mc = double(n_in) * double(kSDigits) * double(uint64_t(1) << pl.log2_bp) / double(nb);
    ccap = uint32_t(mc + 8.0 * std::sqrt(mc + 1.0) + 1024.0);
    tpc = (ccap + kSTile - 1) / kSTile;
    if ((s = sc.alloc(WS_CBUF, &cbuf, size_t(ncoarse) * ccap * sizeof(E))) != HM_OK) return fail(s);
    if ((s = sc.alloc(WS_CCOUNT, &ccount, size_t(ncoarse) * 4)) != HM_OK) return fail(s);
    HM_CUDA_TRY(cudaFuncSetAttribute(kS1, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smemS)));
    HM_CUDA_TRY(cudaFuncSetAttribute(kS2, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smemS)));
  }

  BuildParams bp{};
  bp.smix = smix;
  bp.b_lo = b_lo;
  bp.nb = nb;
  bp.n_in = n_in;
  bp.bound4n = 4 * n_global;
  bp.log2_bp = pl.log2_bp;
  bp.np = pl.np;
  bp.cap = pl.cap;
  bp.flags = knob_flags;

  DevStatus hs{};
  const uint32_t t1_lo = t1_fixed >= 0 ? uint32_t(t1_fixed) : 0u;
  const uint32_t t1_hi = t1_fixed >= 0 ? uint32_t(t1_fixed) + 1 : kT1Cap;
  for (uint32_t t1 = t1_lo; t1 < t1_hi; t1++) {
    bp.l1 = make_l1(smix, t1, n_global);
    bp.slot_cap = slot_cap;
    HM_CUDA_TRY(cudaMemsetAsync(pcount, 0, size_t(pl.np) * 4, st));
    bool run_a = true;
    for (int pass = 0; pass < 3; pass++) {
      HM_CUDA_TRY(cudaMemsetAsync(lbstate, 0, size_t(pl.np) * 8, st));
      HM_CUDA_TRY(cudaMemsetAsync(dstat, 0, sizeof(DevStatus), st));
      if (run_a && ntiles > 0 && two_pass) {
        HM_CUDA_TRY(cudaMemsetAsync(ccount, 0, size_t(ncoarse) * 4, st));
        const SplitArgs a1{nullptr, nullptr, 0, 0, cbuf, ccount, ccap, ncoarse, 0};
        {
          LaunchScope ls_("k_split1", st);
          kS1<<<unsigned((n_in + kSTile - 1) / kSTile), kSThreads, smemS, st>>>(src, bp, a1, dstat);
        }
        HM_CUDA_TRY(cudaGetLastError());
        const SplitArgs a2{cbuf, ccount, ccap, tpc, pbuf, pcount, pl.cap, pl.np, ncoarse};
        {
          LaunchScope ls_("k_split2", st);
          kS2<<<ncoarse * tpc, kSThreads, smemS, st>>>(src, bp, a2, dstat);
        }
        HM_CUDA_TRY(cudaGetLastError());
      } else if (run_a && ntiles > 0) {
        {
          LaunchScope ls_("k_partition", st);
          if (smemHist) kA_s<<<gridA, kAThreads, smemA, st>>>(src, bp, pbuf, pcount, dstat);
          else kA_g<<<gridA, kAThreads, 0, st>>>(src, bp, pbuf, pcount, dstat);
        }
        HM_CUDA_TRY(cudaGetLastError());
      }
      run_a = false;
      {
        LaunchScope ls_("k_bucket", st);
        kB<<<pl.np, kBThreads, pl.smemB, st>>>(bp, pbuf, pcount, lbstate, dir, cdir, slots, dstat, same);
      }
      HM_CUDA_TRY(cudaGetLastError());
      HM_CUDA_TRY(cudaMemcpyAsync(&hs, dstat, sizeof(hs), cudaMemcpyDeviceToHost, st));
      HM_CUDA_TRY(cudaStreamSynchronize(st));
      if (hs.pad) {
        set_error("a routed key does not belong to this shard's bucket range");
        return fail(HM_ERR_INVALID_ARG);
      }
      if (hs.part_overflow) {
        set_error("build partition overflow (degenerate key distribution); not supported in this version");
        return fail(HM_ERR_TOO_LARGE);
      }
      if (hs.S > 4 * n_global || hs.bound_fail) break;  // R7: redraw level one
      if (hs.slot_overflow && !(hs.bound_fail)) {
        // more slots than the allocation: grow to exactly S and rerun K_B
        cudaFreeAsync(slots, st);
        slots = nullptr;
        slot_cap = hs.S;
        bp.slot_cap = slot_cap;
        if ((s = dmalloc(&slots, slot_cap * sizeof(E), st)) != HM_OK) {
          cudaFreeAsync(dir, st);
          cudaFreeAsync(cdir, st);
          return s;
        }
        continue;
      }
      break;
    }
    if (hs.S > 4 * n_global || hs.bound_fail) {
      if (t1_fixed < 0) continue;
      // a shard with a fixed t1: report the failed bound, the caller redraws
      out->dir = dir;
    out->cdir = cdir;
      out->slots = slots;
      out->S = std::max<uint64_t>(hs.S, 4 * n_global + 1);
      out->t1 = t1;
      return HM_OK;
    }
    if (hs.huge) {
      set_error("a level-1 bucket with more than 32 keys (degenerate input); not supported in this version");
      if (hs.dup) return fail(HM_ERR_DUPLICATE_KEY);
      return fail(HM_ERR_TOO_LARGE);
    }
    if (hs.dup) {
      set_error("duplicate keys in from_array_nodup input");
      return fail(HM_ERR_DUPLICATE_KEY);
    }
    if (hs.fpcoll) {
      *fpcoll = true;
      return fail(HM_OK);
    }
    if (hs.exhausted) {
      set_error("a level-2 bucket exhausted 256 attempts");
      return fail(HM_ERR_SEED_EXHAUSTED);
    }
    if (hs.slot_overflow) {
      set_error("slot allocation overflow");
      return fail(HM_ERR_CUDA);
    }
    out->dir = dir;
    out->cdir = cdir;
    out->slots = slots;
    out->S = hs.S;
    out->t1 = t1;
    return HM_OK;
  }
  set_error("level one exhausted 16 attempts without meeting the space bound S <= 4n");
  return fail(HM_ERR_SEED_EXHAUSTED);
}

hm_status build_u64_core(const uint64_t* keys, const uint64_t* vals, uint64_t n_in, uint64_t n_global,
                         uint64_t b_lo, uint64_t nb, int t1_fixed, uint64_t seed, uint32_t log2_bp,
                         cudaStream_t st, BuildOut* out) {
  bool fpc = false;
  return build_core<SrcU64, KV16, SameU64>(SrcU64{keys, vals}, SameU64{}, n_in, n_global, b_lo, nb, t1_fixed, seed,
                                           log2_bp, st, out, &fpc);
}

// ------------------------------------------------------------ byte keys
// Fingerprints (R5) of all keys, thread per key, expanded form (fingerprint_pw).
__global__ void __launch_bounds__(256) k_fingerprint(const uint8_t* __restrict__ bytes,
                                                     const uint64_t* __restrict__ offs, uint64_t n, uint64_t r,
                                                     uint64_t* __restrict__ fp) {
  __shared__ FpPow s_pw;
  if (threadIdx.x == 0) fp_pow_fill(&s_pw, r);
  __syncthreads();
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t o = offs[i], o1 = offs[i + 1];
    fp[i] = fingerprint_pw(bytes, o, o1 - o, r, &s_pw);
  }
}

__global__ void k_check_offsets(const uint64_t* __restrict__ offs, uint64_t n, unsigned int* bad) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t o = offs[i], o1 = offs[i + 1];
    if (o1 < o) atomicOr(bad, 1u);
    else if (o1 - o > 65535) atomicOr(bad, 2u);
  }
}

void launch_fingerprint(const uint8_t* bytes, const uint64_t* offs, uint64_t n, uint64_t r, uint64_t* fp,
                        cudaStream_t st) {
  const unsigned grid = unsigned(std::min<uint64_t>((n + 255) / 256, uint64_t(num_sms()) * 8));
  {
    LaunchScope ls_("k_fingerprint", st);
    k_fingerprint<<<std::max(grid, 1u), 256, 0, st>>>(bytes, offs, n, r, fp);
  }
}

hm_status build_bytes_core(const uint8_t* bytes, const uint64_t* offsets, const uint64_t* vals, uint64_t n,
                           uint64_t seed, uint32_t log2_bp, cudaStream_t st, BuildOut* out, uint32_t* t0_out,
                           uint64_t* r_out) {
  Scratch sc{st};
  uint64_t* fp = nullptr;
  unsigned int* bad = nullptr;
  hm_status s;
  if ((s = sc.alloc(WS_FP, &fp, n * 8)) != HM_OK) return s;
  if ((s = sc.alloc(WS_BAD, &bad, 4)) != HM_OK) return s;
  HM_CUDA_TRY(cudaMemsetAsync(bad, 0, 4, st));
  {
    const unsigned grid = unsigned(std::min<uint64_t>((n + 255) / 256, uint64_t(num_sms()) * 16));
    {
      LaunchScope ls_("k_check_offsets", st);
      k_check_offsets<<<std::max(grid, 1u), 256, 0, st>>>(offsets, n, bad);
    }
    HM_CUDA_TRY(cudaGetLastError());
  }
  unsigned int hbad = 0;
  uint64_t off0 = 0;
  HM_CUDA_TRY(cudaMemcpyAsync(&hbad, bad, 4, cudaMemcpyDeviceToHost, st));
  HM_CUDA_TRY(cudaMemcpyAsync(&off0, offsets, 8, cudaMemcpyDeviceToHost, st));
  HM_CUDA_TRY(cudaStreamSynchronize(st));
  if (hbad & 1u) {
    set_error("offsets are not non-decreasing");
    return HM_ERR_INVALID_ARG;
  }
  if (hbad & 2u) {
    set_error("a byte key is longer than 65535 bytes");
    return HM_ERR_TOO_LARGE;
  }
  const uint64_t smix = seed_mix(seed);
  for (uint32_t t0 = 0; t0 < kT0Cap; t0++) {
    const uint64_t r = derive(smix, 0, 0, t0).a1;
    launch_fingerprint(bytes, offsets, n, r, fp, st);
    HM_CUDA_TRY(cudaGetLastError());
    bool fpc = false;
    s = build_core<SrcBytes, KV32, SameBytes>(SrcBytes{fp, vals, offsets, off0}, SameBytes{bytes, off0}, n, n, 0, n,
                                               -1, seed, log2_bp, st, out, &fpc);
    if (s != HM_OK) return s;
    if (!fpc) {
      *t0_out = t0;
      *r_out = r;
      return HM_OK;
    }
  }
  set_error("fingerprint redraws exhausted (16)");
  return HM_ERR_FP_EXHAUSTED;
}

}  // namespace hm
