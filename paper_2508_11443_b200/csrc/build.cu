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
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <map>
#include <tuple>
#include <mutex>
#include <type_traits>
#include <vector>

#include "hm_internal.cuh"

namespace hm {

constexpr int kAThreads = 512;
#ifndef HM_KB_THREADS
#define HM_KB_THREADS 512
#endif
#ifndef HM_KB_MINB
#define HM_KB_MINB (1024 / HM_KB_THREADS)  // CTAs per SM the registers must allow
#endif
#ifndef HM_KB_THREADS_BYTES
#define HM_KB_THREADS_BYTES 512  // byte keys: only the fingerprints in shared memory, BP = 2^11, 2 CTAs per SM
#endif
#ifndef HM_KB_MINB_BYTES
#define HM_KB_MINB_BYTES 2
#endif
// k_bucket geometry per record type: threads per CTA, warps, CTAs per SM
template <class E>
struct KBCfg {
  static constexpr int T = sizeof(E) == 16 ? HM_KB_THREADS : HM_KB_THREADS_BYTES;
  // the single-table geometry k_bucket<E, Same, FIX_CAP> has built in: 4 buckets
  // per thread, cap = ceil((m + 8 sqrt(m) + 64) / 32) * 32 for m = 2^FIX_LOG2 (make_plan)
  static constexpr uint32_t FIX_LOG2 = T == 512 ? 11u : 10u;
  static constexpr uint32_t FIX_CAP = FIX_LOG2 == 11 ? 2496u : 1344u;
  static constexpr int W = T / 32;
  static constexpr int MINB = sizeof(E) == 16 ? HM_KB_MINB : HM_KB_MINB_BYTES;
  // bytes per item k_bucket keeps in shared memory: the whole 16-byte record
  // (key, value); for 32-byte byte-key records only the fingerprint (the out
  // phase gathers the records from the partition buffer, L2-resident by then)
#ifdef HM_KB_KEYS_ONLY
  static constexpr int SMEM_ITEM = 8;
#else
  static constexpr int SMEM_ITEM = sizeof(E) == 16 ? 16 : 8;
#endif
};

// The partition's items as k_bucket sees them: keys in shared memory (inside
// the 16-byte records, or a plain fingerprint array), records from shared
// memory (16-byte) or from the partition buffer in global memory (32-byte).
template <class E>
struct Items {
  const uint64_t* keys;
  const E* recs;
  static constexpr int kStride = KBCfg<E>::SMEM_ITEM / 8;
  __device__ __forceinline__ uint64_t key(uint32_t i) const { return keys[size_t(i) * kStride]; }
  __device__ __forceinline__ E rec(uint32_t i) const {
    if (KBCfg<E>::SMEM_ITEM == int(sizeof(E))) return recs[i];
    static_assert(sizeof(E) == 16 || sizeof(E) == 32, "record size");
    E e;
    const uint4* p = reinterpret_cast<const uint4*>(recs + i);
    const uint4 a = __ldg(p);
    memcpy(&e, &a, 16);
    if (sizeof(E) == 32) {
      const uint4 b = __ldg(p + 1);
      memcpy(reinterpret_cast<char*>(&e) + 16, &b, 16);
    }
    return e;
  }
};
#ifndef HM_SMEM_ALIAS
#define HM_SMEM_ALIAS 0  // k_bucket: alias rk with the rounds' lists and sA with the slot source map
#endif
#ifndef HM_FP_BATCH
#define HM_FP_BATCH 1  // k_bucket (byte keys): the fingerprints loaded five per thread at a time
#endif
#ifndef HM_OUT_FULL
#define HM_OUT_FULL 1  // k_bucket out phase: whole groups of slots without per-slot bounds checks
#endif
#ifndef HM_DIR_V4
#define HM_DIR_V4 1  // k_bucket: a whole partition's directory as one 32-byte store per thread
#endif
#ifndef HM_MOD_ALWAYS
#define HM_MOD_ALWAYS 1  // k_bucket search: mod s^2 by the reciprocal for every s in K > 2 chunks
#endif
#ifndef HM_PLACE_FLAT
#define HM_PLACE_FLAT 1  // k_bucket scan: class-list placement without a branch per bucket
#endif
#ifndef HM_EQ_INLINE2
#define HM_EQ_INLINE2 1  // k_bucket: the duplicate check of an s = 2 bucket inline (no call)
#endif
#ifndef HM_PRED_ATOM
#define HM_PRED_ATOM 1  // k_bucket: the search's chunk and list counters bumped by predicated atomics
#endif
#ifndef HM_LATE_RECORDS
#define HM_LATE_RECORDS 1  // k_bucket: the record copy completes its own barrier, waited for only before the search
#endif
#ifndef HM_FUSED_DISCARD
#define HM_FUSED_DISCARD 1  // k_split2_bucket: drop a consumed partition's L2 lines without write-back
#endif
#ifndef HM_FUSED_D
#define HM_FUSED_D 1  // k_split2_bucket: pass-2 tiles run D coarse regions ahead of the partitions
#endif
#ifndef HM_PF_DIST
#define HM_PF_DIST 148  // k_bucket: L2 prefetch of partition p + HM_PF_DIST (0: off; 148 measured best)
#endif
#ifndef HM_R0_LOGA2
#define HM_R0_LOGA2 0  // round 0: 2^0 lanes per s = 2 bucket
#endif
#ifndef HM_R0_LOGA
#define HM_R0_LOGA 2  // round 0: 2^2 adjacent lanes (attempts 0..3) per s >= 3 bucket
#endif
#ifndef HM_RETRY_LOGA
#define HM_RETRY_LOGA 3  // at most 2^3 lanes (attempts) per queued bucket and round
#endif
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
// from_array's dedup: {key, value, input index} records (KV32 with ctx_off = i).
struct SrcU64Idx {
  const uint64_t* keys;
  const uint64_t* vals;
  __device__ __forceinline__ KV32 load(uint64_t i) const {
    KV32 e;
    e.key = __ldg(keys + i);
    e.value = __ldg(vals + i);
    e.ctx_off = i;
    e.len = 0;
    e.reserved = 0;
    return e;
  }
};
// from_array of byte keys: {fingerprint, value, ctx_off, len, input index}.
struct SrcBytesIdx {
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
    e.reserved = uint32_t(i);
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
__device__ __forceinline__ uint32_t ld_acquire_u32(const unsigned int* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_relaxed_u32(const unsigned int* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Block-wide exclusive scan of u64 (NT threads); also returns the total.
template <int NT>
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
    unsigned long long w = lane < (NT / 32) ? s_red[lane] : 0ull;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      unsigned long long y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < (NT / 32)) s_red[lane] = w;
  }
  __syncthreads();
  const unsigned long long before = warp ? s_red[warp - 1] : 0ull;
  *total = s_red[(NT / 32) - 1];
  __syncthreads();
  return before + x - v;
}

// Debug-only phase timestamps (compile with -DHM_PHASE_TIMING).
#ifdef HM_PHASE_TIMING
__device__ unsigned long long g_hm_phase[65536 * 16];
__device__ unsigned long long g_hm_ka[4096 * 2];
#define HM_TMARK(k)                                                     \
  do {                                                                  \
    if (threadIdx.x == 0) {                                             \
      unsigned long long t_;                                            \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));            \
      g_hm_phase[(s_p & 65535u) * 16 + (k)] = t_;                       \
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
                                                         uint16_t* __restrict__ plb, unsigned int* __restrict__ pcount,
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
    uint32_t pp[KPT], rk[KPT], lc[KPT];
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
        const uint64_t h1 = hash64(bp.l1.c1, e[j].key);
        const uint64_t lb = level1_of_hash(bp.l1, h1) - bp.b_lo;
        if (lb >= bp.nb) {
          bad = true;
          continue;
        }
        pp[j] = uint32_t(lb >> bp.log2_bp);
        lc[j] = uint32_t(lb & ((1u << bp.log2_bp) - 1)) | (tag4_of_hash(h1) << 12);
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
      if (pos < bp.cap) {
        pbuf[size_t(pp[j]) * bp.cap + pos] = e[j];
        plb[size_t(pp[j]) * bp.cap + pos] = uint16_t(lc[j]);
      } else {
        ovf = true;
      }
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
// passes over the partition id (high bits, then low bits; 8- or 9-bit digits):
// an np-way single pass writes ~one 16-byte element per partition per tile
// (scattered partial-sector stores), a 256-way pass writes runs of ~16
// elements from a shared-memory staging tile.  Ranking inside the tile uses
// one shared-memory atomicAdd per element.
#ifndef HM_SPLIT_T
#define HM_SPLIT_T 512  // (>= the digit count 2^BITS: one digit per thread in the scan)
#endif
constexpr int kSThreads = HM_SPLIT_T;
// elements per thread: 8 x 16-byte or 4 x 32-byte records in registers
#ifndef HM_SPLIT_PT
#define HM_SPLIT_PT 6
#endif
#ifndef HM_SPLIT_PT_BYTES
#define HM_SPLIT_PT_BYTES 4
#endif
#ifndef HM_SPLIT_MINB
#define HM_SPLIT_MINB 2
#endif
template <class E>
__host__ __device__ constexpr int split_pt() {
  return sizeof(E) == 16 ? HM_SPLIT_PT : HM_SPLIT_PT_BYTES;
}
template <class E>
__host__ __device__ constexpr int split_tile() {
  return kSThreads * split_pt<E>();
}

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
  uint16_t* dst_lb;   // pass 2: the record's local bucket | tag4 << 12 for k_bucket (nullptr: none)
};

// One tile of a radix pass (bid: the tile; pass 2: coarse region bid / tpc,
// tile bid % tpc of it).  Also a job of the fused pass-2 + k_bucket kernel.
// The tile's work after its extent is known.  FULL: a whole tile (no
// per-record bounds checks); POW2: n is a power of two (level-one reduction
// by a mask) — both compile-time, so that the per-record loops carry no
// branches.
template <class Src, class E, int PASS, int BITS, int NT, bool FULL, bool POW2>
__device__ __forceinline__ void split_tile_rest(const Src& src, const BuildParams& bp, const SplitArgs& a,
                                                DevStatus* __restrict__ stt, uint8_t* smem, uint64_t base,
                                                uint32_t nvalid, uint32_t coarse, uint32_t* s_cnt,
                                                uint32_t* s_dstart, uint32_t* s_gbase, unsigned long long* s_red) {
  const uint32_t log2bp = bp.log2_bp, ccap = a.ccap, dcap = a.dcap;
  constexpr int kSDigits = 1 << BITS, kSBits = BITS, kSPT = split_pt<E>(), kSTile = NT * split_pt<E>();
  E* stage = reinterpret_cast<E*>(smem);
  uint16_t* sdig = reinterpret_cast<uint16_t*>(smem + size_t(kSTile) * sizeof(E));
  uint16_t* slbc = sdig + kSTile;  // pass 2: local bucket | tag4 << 12 of the staged record
  const uint32_t tid = threadIdx.x;
  const E* cb = reinterpret_cast<const E*>(a.cbuf);
  if (FULL) nvalid = kSTile;
  E e[kSPT];
  uint32_t dg[kSPT], rk[kSPT], lc[kSPT];
  bool bad = false;
#pragma unroll
  for (int j = 0; j < kSPT; j++) {
    const uint32_t i = j * NT + tid;
    if (FULL || i < nvalid) e[j] = PASS == 1 ? src.load(base + i) : cb[size_t(coarse) * ccap + base + i];
  }
#pragma unroll
  for (int j = 0; j < kSPT; j++) {
    const uint32_t i = j * NT + tid;
    dg[j] = 0;
    if (FULL || i < nvalid) {
      const uint64_t h1 = hash64(bp.l1.c1, e[j].key);
      const uint64_t lb = (POW2 ? (h1 & bp.l1.mask) : level1_of_hash(bp.l1, h1)) - bp.b_lo;
      if (lb >= bp.nb) bad = true;
      const uint32_t p = uint32_t(lb >> log2bp);
      dg[j] = PASS == 1 ? ((p >> kSBits) & (kSDigits - 1)) : (p & (kSDigits - 1));
      lc[j] = uint32_t(lb & ((1u << log2bp) - 1)) | (tag4_of_hash(h1) << 12);
    }
  }
  // rank of every element among the tile's elements with its digit: one
  // shared-memory atomicAdd (cheap on sm_100 for spread addresses,
  // scripts/micro/smem_atomics.cu); the order inside a digit is irrelevant
  // (the table is a function of the key set, R13)
#pragma unroll
  for (int j = 0; j < kSPT; j++)
    if (FULL || j * NT + tid < nvalid) rk[j] = atomicAdd(&s_cnt[dg[j]], 1u);
  __syncthreads();
  // digit-major offsets inside the tile; one global reservation per digit
  {
    const uint32_t tot = tid < kSDigits ? s_cnt[tid] : 0u;
    unsigned long long t_all;
    const uint32_t ds = uint32_t(block_excl_scan<NT>(tot, &t_all, s_red));
    if (tid < kSDigits) {
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
    if (FULL || j * NT + tid < nvalid) {
      const uint32_t pos = s_dstart[dg[j]] + rk[j];
      stage[pos] = e[j];
      sdig[pos] = uint16_t(dg[j]);
      if (PASS == 2) slbc[pos] = uint16_t(lc[j]);
    }
  }
  __syncthreads();
  // runs of equal digit are contiguous: consecutive threads write consecutive addresses
  E* dst = reinterpret_cast<E*>(a.dst);
  bool ovf = false;
  for (uint32_t i = tid; i < nvalid; i += NT) {
    const uint32_t d = sdig[i];
    const uint32_t reg = PASS == 1 ? d : coarse * kSDigits + d;
    const uint32_t pos = s_gbase[d] + (i - s_dstart[d]);
    if (reg < a.nreg && pos < dcap) {
      dst[size_t(reg) * dcap + pos] = stage[i];
      if (PASS == 2 && a.dst_lb) a.dst_lb[size_t(reg) * dcap + pos] = slbc[i];
    } else {
      ovf = true;
    }
  }
  if (ovf) atomicOr(&stt->part_overflow, 1u);
  if (bad) atomicOr(&stt->pad, 1u);
}

template <class Src, class E, int PASS, int BITS, int NT = kSThreads>
__device__ __forceinline__ void split_tile_body(const Src& src, const BuildParams& bp, const SplitArgs& a,
                                                DevStatus* __restrict__ stt, uint32_t bid, uint8_t* smem) {
  const uint32_t tpc = a.tpc, ccap = a.ccap;
  constexpr int kSDigits = 1 << BITS, kSTile = NT * split_pt<E>();
  __shared__ uint32_t s_cnt[kSDigits], s_dstart[kSDigits], s_gbase[kSDigits];
  __shared__ unsigned long long s_red[NT / 32];

  const uint32_t tid = threadIdx.x;
  for (uint32_t i = tid; i < kSDigits; i += NT) s_cnt[i] = 0;
  // this CTA's elements
  uint64_t base;
  uint32_t nvalid, coarse = 0;
  if (PASS == 1) {
    base = uint64_t(bid) * kSTile;
    nvalid = bp.n_in - base < uint64_t(kSTile) ? uint32_t(bp.n_in - base) : uint32_t(kSTile);
  } else {
    coarse = bid / tpc;
    const uint32_t k = bid % tpc;
    const uint32_t cc = min(a.ccount[coarse], ccap);
    base = uint64_t(k) * kSTile;
    nvalid = cc > base ? (cc - base < uint64_t(kSTile) ? uint32_t(cc - base) : uint32_t(kSTile)) : 0u;
  }
  __syncthreads();
  if (nvalid == 0) return;
  // (the tile's remaining work with its bounds and level-one reduction fixed at compile time)
  if (nvalid == uint32_t(kSTile)) {
    if (bp.l1.pow2)
      split_tile_rest<Src, E, PASS, BITS, NT, true, true>(src, bp, a, stt, smem, base, nvalid, coarse, s_cnt,
                                                          s_dstart, s_gbase, s_red);
    else
      split_tile_rest<Src, E, PASS, BITS, NT, true, false>(src, bp, a, stt, smem, base, nvalid, coarse, s_cnt,
                                                           s_dstart, s_gbase, s_red);
  } else {
    split_tile_rest<Src, E, PASS, BITS, NT, false, false>(src, bp, a, stt, smem, base, nvalid, coarse, s_cnt,
                                                          s_dstart, s_gbase, s_red);
  }
}

template <class Src, class E, int PASS, int BITS, int NT = kSThreads>
__global__ void __launch_bounds__(NT, NT == kSThreads ? HM_SPLIT_MINB : 2 * HM_SPLIT_MINB)
    k_split(Src src, BuildParams bp, SplitArgs a, DevStatus* __restrict__ stt) {
  extern __shared__ __align__(16) uint8_t smem[];
  split_tile_body<Src, E, PASS, BITS, NT>(src, bp, a, stt, blockIdx.x, smem);
}
#ifndef HM_SPLIT1_T
#define HM_SPLIT1_T 256  // pass 1 of 8-bit digits: 256-thread tiles, twice the CTAs per SM
#endif

// ------------------------------------------------------------------ K_B
// One CTA per build partition of BP = 2^log2_bp level-1 buckets; everything
// between reading the partition and writing its table slice happens in shared
// memory, so that global memory sees one bulk read of the partition and fully
// coalesced writes of the directory and the slots:
//   load   the partition's elements, one cp.async.bulk (TMA) into shared memory
//   hist   g k of every item and its rank in its bucket from a
//          shared-memory atomicAdd (hist) — measured on B200 at
//          ~4.6 SM-cycles per warp-wide spread-address atomic, 9x cheaper than
//          a warp-ballot rank over 11 bucket bits (scripts/micro/smem_atomics.cu)
//   scan   exclusive scans of s and s^2 (presum, R1/R2) and of
//          the size-class counts; groupby as a counting scatter
//   search make2 per multi-key bucket in CTA-wide rounds
//          (below); a finished bucket maps its s^2 slots to their source items:
//          members, and the lowest-slot member as value-0 filler elsewhere (R10)
//   out    decoupled look-back for the global slot base, then the slots
//          (consecutive lanes -> consecutive 16/32-byte records), the directory
//          and the compact directory.
constexpr int kNCls = 3;

__device__ __forceinline__ uint4 ld_stream_u4(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// atomicAdd on a shared counter by the lanes with `pred` only, as one
// predicated instruction (no divergent branch around it); other lanes get 0
__device__ __forceinline__ uint32_t atom_add_if(bool pred, uint32_t saddr, uint32_t v) {
  uint32_t r = 0;
  asm volatile("{ .reg .pred p; setp.ne.u32 p, %1, 0; @p atom.shared::cta.add.u32 %0, [%2], %3; }"
               : "+r"(r)
               : "r"(uint32_t(pred)), "r"(saddr), "r"(v)
               : "memory");
  return r;
}

// make2 for buckets with 2 <= s <= 8, in CTA-wide rounds.
// One attempt = derive(seed,2,b,t), the s level-2 slots hash mod s^2 and the
// occupancy bitmap as `collision`.  Every round is a list
// of buckets with A adjacent lanes per bucket, lane j trying attempt tb + j
// (tb: the bucket's next attempt, 0 in round 0); the lowest successful lane
// wins — the same t as trying them one by one (R13).  Round 0 is the class-
// ordered list (s = 5..8 | 3..4 | 2: the lanes of a warp share one
// key-register width K) with A = 4 for s >= 3 and A = 1 for s = 2 (success
// 3/4); the buckets that collide go to the next round's list (s >= 3 from the
// front, s = 2 from the back: ordered by width again) with A = lanes / list
// length (at most 2^HM_RETRY_LOGA).  Warps take 32-lane chunks from a shared
// counter (dynamic balance); one CTA barrier per round.  Every attempt is one
// lane's work from start to end, so the instruction count follows the attempts
// made (SASS attribution in profiles/r02/).

// Search state (shared memory).
struct SearchCtx {
  const uint16_t* sstart;
  const uint8_t* ss;
  const uint16_t* sidx;
  const uint32_t* soff;  // slot offset of each bucket inside the partition
  uint16_t* sA;          // level-2 slot of each grouped position (direct-slot partitions only)
  uint8_t* s_t;          // attempt t of each bucket (the next attempt to try while searching)
  uint16_t* src;         // slot -> item map (nullptr: not staged)
};

// Slots h[] of a bucket under constants c (K keys in registers); returns the
// occupancy bitmap, or 0 on a collision (s >= 2, so a valid map is never 0).
// For K <= 4 (s^2 <= 16) the bitmap is 32-bit.
template <int K>
__device__ __forceinline__ uint64_t slots_of(const Consts& c, const uint64_t* k, uint32_t s, const FastMod& fm,
                                             uint32_t* h) {
  using B = typename std::conditional<(K <= 4), uint32_t, uint64_t>::type;
  B bits = 0;
  bool coll = false;
#pragma unroll
  for (int j = 0; j < K; j++) {
    h[j] = 0;
    if (uint32_t(j) < s) {
      const uint64_t hv = hash64(c, k[j]);
#if HM_MOD_ALWAYS
      // (K > 2: the reciprocal for every s, exact for s = 4 and 8 too — no per-lane select)
      h[j] = K == 2 ? uint32_t(hv) & (s * s - 1) : uint32_t(fastmod(hv, fm));
#else
      h[j] = (K == 2 || (s & (s - 1)) == 0) ? uint32_t(hv) & (s * s - 1) : uint32_t(fastmod(hv, fm));
#endif
      const B bit = B(1) << h[j];
      coll |= (bits & bit) != 0;
      bits |= bit;
    }
  }
  return coll ? 0ull : uint64_t(bits);
}

// A finished bucket: its t, and its s^2 slots in the slot source map — member
// j at h[j], every other slot the member at the lowest occupied slot with
// value 0 (R10, bit 15): every slot is first written as filler (unrolled
// predicated stores) and the members over them.
template <int K>
__device__ __forceinline__ void bucket_done(const SearchCtx& X, uint32_t lb, uint32_t st0, uint32_t s, uint32_t t,
                                            const uint32_t* h, uint64_t bits) {
  X.s_t[lb] = uint8_t(t);
  uint32_t it[K], hmin = 0xFFFFu, fill = 0;
#pragma unroll
  for (int j = 0; j < K; j++)
    if (uint32_t(j) < s) {
      it[j] = X.sidx[st0 + j];
      if (h[j] < hmin) {
        hmin = h[j];
        fill = it[j];
      }
    }
  if (!X.src) {
#pragma unroll
    for (int j = 0; j < K; j++)
      if (uint32_t(j) < s) X.sA[st0 + j] = uint16_t(h[j]);
    return;
  }
  uint16_t* o = X.src + X.soff[lb];
  const uint16_t fv = uint16_t(fill | 0x8000u);
  const uint32_t s2 = s * s;
#pragma unroll
  for (int x = 0; x < K * K; x++)
    if (uint32_t(x) < s2) o[x] = fv;
#pragma unroll
  for (int j = 0; j < K; j++)
    if (uint32_t(j) < s) o[h[j]] = uint16_t(it[j]);
}

// Equal keys in a bucket (a duplicate, or equal fingerprints with different
// bytes) never separate: record which, once, and retire the bucket.
template <class E, class Same>
__device__ __noinline__ bool bucket_equal_keys_(Items<E> skv, const uint16_t* sstart, const uint8_t* ss,
                                                const uint16_t* sidx, uint8_t* s_t, uint32_t lb, DevStatus* stt,
                                                Same same) {
  const uint32_t st0 = sstart[lb], s = ss[lb];
  for (uint32_t i = 0; i < s; i++) {
    const uint32_t ii = sidx[st0 + i];
    for (uint32_t j = i + 1; j < s; j++) {
      const uint32_t jj = sidx[st0 + j];
      if (skv.key(jj) == skv.key(ii)) {
        atomicOr(same.same(skv.rec(ii), skv.rec(jj)) ? &stt->dup : &stt->fpcoll, 1u);
        s_t[lb] = 0;
        return true;
      }
    }
  }
  return false;
}
template <class E, class Same>
__device__ __forceinline__ bool bucket_equal_keys(const Items<E>& skv, const SearchCtx& X, uint32_t lb, DevStatus* stt,
                                                  const Same& same) {
#if HM_EQ_INLINE2
  // (the common case inline: a pair of distinct keys; the call only for s > 2
  // or an equal pair)
  if (X.ss[lb] == 2) {
    const uint32_t st0 = X.sstart[lb];
    if (skv.key(X.sidx[st0]) != skv.key(X.sidx[st0 + 1])) return false;
  }
#endif
  return bucket_equal_keys_(skv, X.sstart, X.ss, X.sidx, X.s_t, lb, stt, same);
}

// Attempt t of bucket lb (s keys, K-wide registers) on this lane.  Returns
// the occupancy bitmap (0: collision, or no bucket on this lane).
template <int K, class E>
__device__ __forceinline__ uint64_t lane_attempt(const BuildParams& bp, const Items<E>& skv, const SearchCtx& X, bool act,
                                                 uint32_t lb, uint32_t s, uint32_t t, const uint64_t* s_m2,
                                                 uint64_t bbase, uint32_t* h) {
  if (!act || t >= kT2Cap) return 0;
  const uint32_t st0 = X.sstart[lb];
  uint64_t k[K];
#pragma unroll
  for (int j = 0; j < K; j++) k[j] = uint32_t(j) < s ? skv.key(X.sidx[st0 + j]) : 0ull;
  FastMod fm{uint64_t(s) * s, 0};
  if (K > 2) fm.m = s_m2[s];
  return slots_of<K>(derive(bp.smix, 2, bbase + lb, t), k, s, fm, h);
}

// The key-register width follows the largest bucket among the warp's lanes.
template <class E>
__device__ __forceinline__ uint64_t lane_attempt_k(const BuildParams& bp, const Items<E>& skv, const SearchCtx& X, bool act,
                                                   uint32_t lb, uint32_t s, uint32_t t, const uint64_t* s_m2,
                                                   uint64_t bbase, uint32_t* h) {
  const uint32_t smax = __reduce_max_sync(0xffffffffu, act ? s : 0u);
  if (smax <= 2) return lane_attempt<2>(bp, skv, X, act, lb, s, t, s_m2, bbase, h);
  if (smax <= 4) return lane_attempt<4>(bp, skv, X, act, lb, s, t, s_m2, bbase, h);
  return lane_attempt<8>(bp, skv, X, act, lb, s, t, s_m2, bbase, h);
}

__device__ __forceinline__ void bucket_done_any(const SearchCtx& X, uint32_t lb, uint32_t s, uint32_t t,
                                                const uint32_t* h, uint64_t bits) {
  const uint32_t st0 = X.sstart[lb];
  if (s <= 2) bucket_done<2>(X, lb, st0, s, t, h, bits);
  else if (s <= 4) bucket_done<4>(X, lb, st0, s, t, h, bits);
  else bucket_done<8>(X, lb, st0, s, t, h, bits);
}

// Append lb to the next round's list (s >= 3 at the front, s = 2 at the back),
// warp-aggregated: one shared atomic per warp and side.
__device__ __forceinline__ void list_append(bool want, uint32_t lb, uint32_t s, uint16_t* nl, uint32_t lcap,
                                            uint32_t* ncnt, uint32_t ncnt_sa) {
  const uint32_t lane = threadIdx.x & 31, lt = (1u << lane) - 1u;
#pragma unroll
  for (int side = 0; side < 2; side++) {
    const bool mine = want && ((s >= 3) == (side == 0));
    const uint32_t m = __ballot_sync(0xffffffffu, mine);
    if (m) {
      const uint32_t leader = __ffs(m) - 1;
#if HM_PRED_ATOM
      uint32_t b = atom_add_if(lane == leader, ncnt_sa + 4u * side, uint32_t(__popc(m)));  // (ncnt_sa: &ncnt[0])
#else
      uint32_t b = 0;
      if (lane == leader) b = atomicAdd(&ncnt[side], uint32_t(__popc(m)));
#endif
      b = __shfl_sync(0xffffffffu, b, leader) + __popc(m & lt);
      if (mine) nl[side == 0 ? b : lcap - 1 - b] = uint16_t(lb);
    }
  }
}

// make2 for the rare 9 <= s <= 32 buckets: a warp per bucket, a lane per key,
// __match_any_sync on the level-2 slots as the injectivity test; then the
// bucket's s^2 slots are mapped as in bucket_done (bitsw: a per-warp bitmap).
template <class E, class Same>
__device__ __forceinline__ void search_warp(const BuildParams& bp, const Items<E>& skv, const SearchCtx& X,
                                            const uint16_t* list, uint32_t L, const uint64_t* s_m2, uint64_t bbase,
                                            DevStatus* stt, const Same& same, uint32_t* bitsw) {
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (uint32_t idx = warp; idx < L; idx += KBCfg<E>::W) {
    const uint32_t lb = list[idx], st0 = X.sstart[lb], s = X.ss[lb];
    const bool mine = lane < s;
    const uint32_t item = mine ? X.sidx[st0 + lane] : 0u;
    const uint64_t key = mine ? skv.key(item) : 0ull;
    const uint32_t valid = __ballot_sync(0xffffffffu, mine);
    const uint32_t dm = __match_any_sync(0xffffffffu, key) & valid & ~(1u << lane);
    uint32_t t = 0;
    if (__any_sync(0xffffffffu, mine && dm != 0)) {
      if (mine && dm != 0) {
        const bool d = same.same(skv.rec(item), skv.rec(X.sidx[st0 + __ffs(dm) - 1]));
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
      } else {
        if (mine && !X.src) X.sA[st0 + lane] = uint16_t(h);
        if (X.src) {
          uint16_t* o = X.src + X.soff[lb];
          bitsw[lane] = 0;
          __syncwarp();
          if (mine) atomicOr(&bitsw[h >> 5], 1u << (h & 31));
          const uint32_t hmin = __reduce_min_sync(0xffffffffu, mine ? h : 0xFFFFu);
          const uint32_t who = __ffs(__ballot_sync(0xffffffffu, mine && h == hmin)) - 1;
          const uint32_t fill = __shfl_sync(0xffffffffu, item, who);
          __syncwarp();
          for (uint32_t x = lane; x < s * s; x += 32)
            if (!((bitsw[x >> 5] >> (x & 31)) & 1)) o[x] = uint16_t(fill | 0x8000u);
          __syncwarp();
          if (mine) o[h] = uint16_t(item);
        }
      }
    }
    if (lane == 0) X.s_t[lb] = uint8_t(t);
  }
}

__host__ __device__ constexpr size_t al16(size_t x) { return (x + 15) & ~size_t(15); }
// Dynamic shared memory of k_bucket (all offsets 16-byte aligned), computed on
// the host and passed in BuildParams (kernel parameters live in the constant
// bank: no registers, no recomputation inside the kernel's loops).
__host__ __device__ constexpr BucketSmem bucket_smem_layout(uint32_t cap, uint32_t BP, uint32_t esz) {
  BucketSmem L{};
  L.smax = 2 * cap + 256;  // slots of the partition staged in shared memory (S_p is ~2 cnt)
  if (L.smax > 32768u) L.smax = 32768u;
  L.cls_off[0] = 0;                           // s = 2..8 (regions s = 5..8 | 3..4 | 2): at most cap/2 buckets
  L.cls_off[1] = L.cls_off[0];
  L.cls_off[2] = L.cls_off[1] + cap / 2 + 1;  // s = 9..32: cap/9
  L.cls_off[3] = L.cls_off[2] + cap / 9 + 1;
  L.skv = 0;                                               // [cap] items: 16-B records or 8-B fingerprints
  L.lbk = L.skv + al16(size_t(cap) * esz);                 // u16[cap]: local bucket of item i
#if HM_SMEM_ALIAS
  // (rk lives from hist to groupby, the rounds' lists from the search on: one
  // region; sA serves only direct-slot partitions, src only staged ones)
  L.sidx = L.lbk + al16(size_t(cap) * 2);                  // u16[cap]: grouped position -> item
  L.src = L.sidx + al16(size_t(cap) * 2);                  // u16[smax]: slot -> item / u16[cap]: sA
  L.sA = L.src;
  L.slist = L.src + al16(size_t(L.smax) * 2);              // u16[]: class lists
  L.queue = L.slist + al16(size_t(L.cls_off[kNCls]) * 2);  // u16[3][cap/2+1]: the rounds' lists / u16[cap]: rk
  L.rk = L.queue;
  L.ss = L.queue + al16(size_t(cap / 2 + 1) * 6 > size_t(cap) * 2 ? size_t(cap / 2 + 1) * 6 : size_t(cap) * 2);
#else
  L.rk = L.lbk + al16(size_t(cap) * 2);                    // u16[cap]: rank of item i in its bucket
  L.sidx = L.rk + al16(size_t(cap) * 2);                   // u16[cap]: grouped position -> item
  L.sA = L.sidx + al16(size_t(cap) * 2);                   // u16[cap]: level-2 slot of a grouped position
  L.src = L.sA + al16(size_t(cap) * 2);                    // u16[smax]: slot -> item (bit 15: filler, value 0)
  L.slist = L.src + al16(size_t(L.smax) * 2);              // u16[]: class lists
  L.queue = L.slist + al16(size_t(L.cls_off[kNCls]) * 2);  // u16[3][cap/2+1]: the rounds' lists
  L.ss = L.queue + al16(size_t(cap / 2 + 1) * 6);          // u8[BP]: bucket size s
#endif
  L.sstart = L.ss + al16(BP);                              // u16[BP]: first grouped position of each bucket
  L.soff = L.sstart + al16(size_t(BP) * 2);                // u32[BP]: histogram, then slot offset in the partition
  L.st = L.soff + al16(size_t(BP) * 4);                    // u8[BP]: attempt t of each bucket
  L.total = uint32_t(L.st + al16(BP));
  return L;
}

// Block-wide exclusive scan of two u64 values at once (NW warps).
template <int NW>
__device__ __forceinline__ void block_excl_scan2(unsigned long long& a, unsigned long long& b,
                                                 unsigned long long* ta, unsigned long long* tb,
                                                 unsigned long long (*s_red)[NW]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned long long x = a, y = b;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long u = __shfl_up_sync(0xffffffffu, x, o), v = __shfl_up_sync(0xffffffffu, y, o);
    if (lane >= o) {
      x += u;
      y += v;
    }
  }
  if (lane == 31) {
    s_red[0][warp] = x;
    s_red[1][warp] = y;
  }
  __syncthreads();
  if (warp == 0) {
    unsigned long long u = lane < NW ? s_red[0][lane] : 0ull, v = lane < NW ? s_red[1][lane] : 0ull;
#pragma unroll
    for (int o = 1; o < NW; o <<= 1) {
      const unsigned long long p = __shfl_up_sync(0xffffffffu, u, o), q = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) {
        u += p;
        v += q;
      }
    }
    if (lane < NW) {
      s_red[0][lane] = u;
      s_red[1][lane] = v;
    }
  }
  __syncthreads();
  const unsigned long long ba = warp ? s_red[0][warp - 1] : 0ull, bb = warp ? s_red[1][warp - 1] : 0ull;
  *ta = s_red[0][NW - 1];
  *tb = s_red[1][NW - 1];
  a = ba + x - a;
  b = bb + y - b;
}

// kFused: a job of k_split2_bucket — partition p_given, whose records pass 2
// is writing in the same kernel: wait until the tiles of its coarse region
// are all done (*sdone_c == tpc), and drop the partition's L2 lines without
// write-back once they are in shared memory (discard.global.L2: nothing reads
// them again).  Otherwise the partition is the next ticket.
// kCap != 0: the geometry of every single-table build of 2^16+ keys (2^11
// buckets per partition, capacity kCap) as compile-time constants, so that
// shared-memory addresses fold into the instructions' immediate offsets.
template <class E, class Same, bool kFused, uint32_t kCap>
__device__ __forceinline__ void bucket_body(const BuildParams& bp, const E* __restrict__ pbuf,
                                            const uint16_t* __restrict__ plb, const unsigned int* pcount,
                                            unsigned long long* __restrict__ lbstate, uint64_t* __restrict__ dir,
                                            CDir* __restrict__ cdir, E* __restrict__ slots,
                                            DevStatus* __restrict__ stt, const Same& same, uint8_t* smem,
                                            uint32_t p_given, const unsigned int* sdone_c, uint32_t tpc) {
  __shared__ uint64_t s_m2[33];
  __shared__ __align__(8) unsigned long long s_bar[2];  // bulk loads: [0] the codes, [1] the records
  __shared__ uint32_t s_p;
  __shared__ unsigned long long s_red2[2][KBCfg<E>::W];
  __shared__ unsigned long long s_base;
  __shared__ uint32_t s_c9, s_chunk[3], s_qn[3][2];
  __shared__ uint32_t s_bitsw[KBCfg<E>::W][32];

  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr bool kFix = kCap != 0;
  constexpr uint32_t kFixLog2 = KBCfg<E>::FIX_LOG2;
  constexpr BucketSmem kSL = bucket_smem_layout(kFix ? kCap : 32u, 1u << kFixLog2, KBCfg<E>::SMEM_ITEM);
#define HM_SL(f) (kFix ? kSL.f : bp.sl.f)
  const uint32_t cap = kFix ? kCap : bp.cap;
  const uint32_t log2bp = kFix ? kFixLog2 : bp.log2_bp;
  const uint32_t BP = 1u << log2bp;
  const uint32_t CH = (BP + KBCfg<E>::T - 1) / KBCfg<E>::T;  // buckets per thread in the scans
  uint64_t* skey = reinterpret_cast<uint64_t*>(smem + HM_SL(skv));  // (16-byte records, or fingerprints)
  uint16_t* lbk = reinterpret_cast<uint16_t*>(smem + HM_SL(lbk));
  uint16_t* rk = reinterpret_cast<uint16_t*>(smem + HM_SL(rk));
  uint16_t* sidx = reinterpret_cast<uint16_t*>(smem + HM_SL(sidx));
  uint16_t* sA = reinterpret_cast<uint16_t*>(smem + HM_SL(sA));
  uint16_t* src = reinterpret_cast<uint16_t*>(smem + HM_SL(src));
  uint16_t* slist = reinterpret_cast<uint16_t*>(smem + HM_SL(slist));
  uint16_t* rlist = reinterpret_cast<uint16_t*>(smem + HM_SL(queue));  // [3][lcap]
  uint8_t* ss = smem + HM_SL(ss);
  uint16_t* sstart = reinterpret_cast<uint16_t*>(smem + HM_SL(sstart));
  uint32_t* soff = reinterpret_cast<uint32_t*>(smem + HM_SL(soff));
  uint8_t* s_t = smem + HM_SL(st);
  const uint32_t lcap = cap / 2 + 1;

  if (tid == 0) {
    if (kFused) {
      s_p = p_given;
      // the coarse region's pass-2 tiles (release: __threadfence + atomicAdd
      // after their stores); then the bulk copy (async proxy) may read them
      uint32_t d;
      while ((d = ld_acquire_u32(sdone_c)) < tpc) __nanosleep(128);
      asm volatile("fence.proxy.async.global;" ::: "memory");
    } else {
      s_p = atomicAdd(&stt->ticket, 1u);
    }
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&s_bar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&s_bar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    s_c9 = 0;
#pragma unroll
    for (int i = 0; i < 3; i++) {
      s_chunk[i] = 0;
      s_qn[i][0] = s_qn[i][1] = 0;
    }
  }
  if (tid < 33) s_m2[tid] = g_m2.v[tid];  // (a compile-time table: no 64-bit division per CTA)
  if (BP == 4u * KBCfg<E>::T) reinterpret_cast<uint4*>(soff)[tid] = make_uint4(0u, 0u, 0u, 0u);  // the histogram
  else
    for (uint32_t j = tid; j < BP; j += KBCfg<E>::T) soff[j] = 0;
  __syncthreads();
  const uint32_t p = s_p;
  HM_TMARK(0);
  const uint64_t lb0 = uint64_t(p) << log2bp;
  const uint32_t nbp = uint32_t(bp.nb - lb0 < uint64_t(BP) ? bp.nb - lb0 : uint64_t(BP));
  const uint32_t cnt_raw = kFused ? ld_relaxed_u32(pcount + p) : pcount[p];
  const bool ovf = cnt_raw > cap;
  const uint32_t cnt = ovf ? 0u : cnt_raw;
  const uint64_t bbase = bp.b_lo + lb0;  // global id of the partition's first bucket

  // ---- load: one bulk copy (TMA) of the partition's elements into shared memory
#if HM_PF_DIST
  // (and an L2 prefetch of the partition a CTA takes about a wave later, so
  // that its load finds the lines in L2)
  if (!kFused && tid == 32 && p + HM_PF_DIST < bp.np) {
    const uint32_t q = p + HM_PF_DIST, cq = min(pcount[q], cap);
    const uint32_t qb = (cq * uint32_t(sizeof(E)) + 15u) & ~15u, ql = ((cq + 7) & ~7u) * 2;
    if (qb)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(pbuf + size_t(q) * cap), "r"(qb) : "memory");
    if (ql) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(plb + size_t(q) * cap), "r"(ql) : "memory");
  }
#endif
  const E* prec = pbuf + size_t(p) * cap;  // (the partition's records in global memory)
  if (tid == 0) {
    const uint32_t bytes = KBCfg<E>::SMEM_ITEM == int(sizeof(E)) ? cnt * uint32_t(sizeof(E)) : 0u;
    const uint32_t lbytes = ((cnt + 7) & ~7u) * 2;  // (16-byte multiple; cap is a multiple of 32)
    // the codes (all that hist, scan and groupby read) complete barrier 0, the
    // records (first read by the search) barrier 1: the record copy overlaps
    // hist, scan and groupby
    const uint32_t b0 = smem_u32(&s_bar[0]), b1 = smem_u32(&s_bar[HM_LATE_RECORDS ? 1 : 0]);
    if (cnt) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b0),
                   "r"(lbytes + (HM_LATE_RECORDS ? 0u : bytes))
                   : "memory");
      if (HM_LATE_RECORDS) {
        if (bytes)
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b1), "r"(bytes) : "memory");
        else
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(b1) : "memory");
      }
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_u32(lbk)),
          "l"(plb + size_t(p) * cap), "r"(lbytes), "r"(b0)
          : "memory");
      if (bytes)
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_u32(skey)),
            "l"(prec), "r"(bytes), "r"(b1)
            : "memory");
    } else {
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(b0) : "memory");
      if (HM_LATE_RECORDS) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(b1) : "memory");
    }
  }
  if constexpr (sizeof(E) == sizeof(KV32)) {  // (byte-key builds only)
    if (bp.cp_bytes && warp != 0) {
      // the side copy (BuildParams::cp_*): this partition's slice, 16-byte
      // units, HM_CP_UNROLL loads in flight per thread, streaming stores
#ifndef HM_CP_UNROLL
#define HM_CP_UNROLL 8
#endif
      constexpr int U = HM_CP_UNROLL;
      const uint64_t a = uint64_t(p) * bp.cp_slice, b = min(a + bp.cp_slice, bp.cp_bytes);
      const uint32_t nt = KBCfg<E>::T - 32;
      const uint4* src4 = reinterpret_cast<const uint4*>(bp.cp_src);
      uint4* dst4 = reinterpret_cast<uint4*>(bp.cp_dst);
      const uint64_t u0 = a >> 4, u1 = b >> 4;  // (full units; a is 16-aligned)
      for (uint64_t u = u0 + (tid - 32); u < u1; u += uint64_t(U) * nt) {
        uint4 v[U];
#pragma unroll
        for (int k = 0; k < U; k++)
          if (u + uint64_t(k) * nt < u1) v[k] = ld_stream_u4(src4 + u + uint64_t(k) * nt);
#pragma unroll
        for (int k = 0; k < U; k++)
          if (u + uint64_t(k) * nt < u1) __stcs(dst4 + u + uint64_t(k) * nt, v[k]);
      }
      if (b == bp.cp_bytes && (b & 15) && tid >= 32 && tid < 32 + (b & 15))  // (the last partial unit)
        bp.cp_dst[(b & ~uint64_t(15)) + (tid - 32)] = bp.cp_src[(b & ~uint64_t(15)) + (tid - 32)];
    }
  }
  // (warp 0 waits; the other warps wait at the CTA barrier that follows, with no issue slots)
  auto bulk_wait = [&](const unsigned long long* bar) {
    uint32_t done = 0;
    do {
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
          : "=r"(done)
          : "r"(smem_u32(bar))
          : "memory");
      if (!done) __nanosleep(64);
    } while (!done);
  };
  if (warp == 0) bulk_wait(&s_bar[0]);
  __syncthreads();
  HM_TMARK(1);

  // ---- hist: the local bucket of g k and the
  // key's tag came with the record from the partition pass (k_split pass 2 /
  // k_partition hashed it already); the rank among the items of its bucket
  // comes from the shared-memory counter
#if HM_FP_BATCH
  if constexpr (KBCfg<E>::SMEM_ITEM != int(sizeof(E))) {
    // byte keys: the fingerprints from the partition buffer, five loads in
    // flight per thread (the search reads them from shared memory)
    constexpr int U = 5;
    for (uint32_t i0 = tid; i0 < cnt; i0 += U * KBCfg<E>::T) {
      uint64_t f[U];
#pragma unroll
      for (int u = 0; u < U; u++) {
        const uint32_t i = i0 + u * KBCfg<E>::T;
        f[u] = i < cnt ? __ldg(reinterpret_cast<const unsigned long long*>(prec + i)) : 0ull;
      }
#pragma unroll
      for (int u = 0; u < U; u++) {
        const uint32_t i = i0 + u * KBCfg<E>::T;
        if (i < cnt) skey[i] = f[u];
      }
    }
  }
#endif
  for (uint32_t i = tid; i < cnt; i += KBCfg<E>::T) {
    if (!HM_FP_BATCH && KBCfg<E>::SMEM_ITEM != int(sizeof(E)))
      skey[i] = __ldg(reinterpret_cast<const unsigned long long*>(prec + i));
    const uint32_t code = lbk[i];
    uint32_t lb = code & 0xFFFu;
    if (lb >= nbp) {  // cannot happen for a well-routed partition; never index out of range
      atomicOr(&stt->pad, 1u);
      lb = 0;
    }
    lbk[i] = uint16_t(lb);
    rk[i] = uint16_t(atomicAdd(&soff[lb], 1u));
    s_t[lb] = uint8_t(code >> 12);  // kept for singletons only (the scan resets the rest)
  }
  __syncthreads();
  HM_TMARK(2);

  // ---- exclusive scans of s and s^2 (presum, R1/R2) and of
  // the class counts; thread t owns buckets [4t, 4t + 4) (BP = 4T: one 16-byte
  // load of the four counts) or [t*CH, t*CH + CH) otherwise
  bool huge = false, bfail = false;
  unsigned long long S_p;
  uint32_t Lall, L3;  // listed buckets, of them with s >= 3 (at the front)
  {
    const uint32_t c0 = tid * CH, c1 = min(c0 + CH, nbp);
    const bool vec = CH == 4;  // (CTA-uniform; entries past nbp are 0)
    uint32_t v4[4] = {0, 0, 0, 0};
    if (vec) {
      const uint4 q = *reinterpret_cast<const uint4*>(soff + c0);
      v4[0] = q.x;
      v4[1] = q.y;
      v4[2] = q.z;
      v4[3] = q.w;
    }
    // a = s | s^2 << 32; b = #(s=2) | #(s=3..4) << 21 | #(s=5..8) << 42
    unsigned long long a = 0, b = 0;
    if (vec) {
      uint32_t sum = 0, sq = 0, cls = 0;  // cls: the three counts in bytes 0..2
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const uint32_t v = v4[u];
        sum += v;
        sq += v * v;
        cls += (v == 2 ? 1u : 0u) + (v - 3u <= 1u ? 0x100u : 0u) + (v - 5u <= 3u ? 0x10000u : 0u);
      }
      a = uint64_t(sum) | (uint64_t(sq) << 32);
      b = uint64_t(cls & 0xFF) | (uint64_t((cls >> 8) & 0xFF) << 21) | (uint64_t(cls >> 16) << 42);
    } else {
      for (uint32_t j = c0; j < c1; j++) {
        const uint32_t v = soff[j];
        a += uint64_t(v) | (uint64_t(v * v) << 32);
        b += v == 2 ? 1ull : (v - 3u <= 1u ? (1ull << 21) : (v - 5u <= 3u ? (1ull << 42) : 0ull));
      }
    }
    unsigned long long ta, tb;
    block_excl_scan2<KBCfg<E>::W>(a, b, &ta, &tb, s_red2);
    S_p = ta >> 32;
    const uint32_t T2 = uint32_t(tb & 0x1FFFFF), T4 = uint32_t((tb >> 21) & 0x1FFFFF), T8 = uint32_t(tb >> 42);
    Lall = T2 + T4 + T8;
    L3 = T4 + T8;
    // list regions: [s = 5..8 | s = 3..4 | s = 2]
    uint32_t n8 = uint32_t(b >> 42), n4 = T8 + uint32_t((b >> 21) & 0x1FFFFF), n2 = T8 + T4 + uint32_t(b & 0x1FFFFF);
    uint32_t pos = uint32_t(a), sq = uint32_t(a >> 32);
    // (a bucket with s^2 > 4n means S > 4n: level one redraws, R7, and this
    // pass is discarded; s <= 8 buckets are listed all the same — only
    // reachable with n < 16)
    auto place = [&](uint32_t j, uint32_t v) {
#if HM_PLACE_FLAT
      // s = 2..8 branch-free (a predicated store); s >= 5 — the only sizes the
      // space bound can reject (s <= n) and the warp-per-bucket list — apart
      const uint32_t pos = v == 2 ? n2 : (v <= 4 ? n4 : n8);
      if (v - 2u <= 6u) slist[pos] = uint16_t(j);
      n2 += v == 2;
      n4 += v - 3u <= 1u;
      n8 += v - 5u <= 3u;
      if (v >= 5) {
        const bool over = uint64_t(v) * v > bp.bound4n;
        bfail |= over;
        if (v >= 9 && !over) {
          if (v <= 32) slist[HM_SL(cls_off[2]) + atomicAdd(&s_c9, 1u)] = uint16_t(j);
          else huge = true;
        }
      }
#else
      if (v < 2) return;
      const bool over = uint64_t(v) * v > bp.bound4n;
      bfail |= over;
      if (v <= 8) {
        slist[v == 2 ? n2 : (v <= 4 ? n4 : n8)] = uint16_t(j);
        n2 += v == 2;
        n4 += v - 3u <= 1u;
        n8 += v >= 5;
      } else if (!over) {
        if (v <= 32) slist[HM_SL(cls_off[2]) + atomicAdd(&s_c9, 1u)] = uint16_t(j);
        else huge = true;
      }
#endif
    };
    if (vec) {
      uint32_t st4 = *reinterpret_cast<const uint32_t*>(s_t + c0), ss4 = 0, ssk = 0;
      uint32_t so[4], sp[4];
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const uint32_t v = v4[u];
        sp[u] = pos;
        so[u] = sq;
        ss4 |= (v > 255 ? 255u : v) << (8 * u);
        if (v == 1) ssk |= 0xFFu << (8 * u);  // (a singleton keeps its key's tag for the compact directory)
        pos += v;
        sq += v * v;
      }
      *reinterpret_cast<uint4*>(soff + c0) = make_uint4(so[0], so[1], so[2], so[3]);
      *reinterpret_cast<uint2*>(sstart + c0) = make_uint2(sp[0] | (sp[1] << 16), sp[2] | (sp[3] << 16));
      *reinterpret_cast<uint32_t*>(ss + c0) = ss4;
      *reinterpret_cast<uint32_t*>(s_t + c0) = st4 & ssk;
#pragma unroll
      for (int u = 0; u < 4; u++) place(c0 + u, v4[u]);
    } else {
      for (uint32_t j = c0; j < c1; j++) {
        const uint32_t v = soff[j];
        ss[j] = uint8_t(v > 255 ? 255 : v);
        sstart[j] = uint16_t(pos);
        soff[j] = sq;
        if (v != 1) s_t[j] = 0;
        pos += v;
        sq += v * v;
        place(j, v);
      }
    }
    if (huge) atomicOr(&stt->huge, 1u);
    if (bfail) atomicOr(&stt->bound_fail, 1u);
  }
  // publish the partition's aggregate S_p now (decoupled look-back)
  if (tid == 0) st_release(&lbstate[p], (p == 0 ? kFlagInc : kFlagAgg) | (S_p & kValMask));
  __syncthreads();
  HM_TMARK(10);
  // ---- groupby: grouped position of every item; a singleton
  // (R12: its slot is soff) is mapped right here
  const bool staged = S_p <= HM_SL(smax) && !(bp.flags & HM_FLAG_DIRECT_SLOTS);
  for (uint32_t i = tid; i < cnt; i += KBCfg<E>::T) {
    const uint32_t lb = lbk[i];
    sidx[sstart[lb] + rk[i]] = uint16_t(i);
    if (staged && ss[lb] == 1) src[soff[lb]] = uint16_t(i);
  }
  if (HM_LATE_RECORDS && warp == 0) bulk_wait(&s_bar[1]);  // (the records, for the search)
  __syncthreads();
  HM_TMARK(3);
  if (kFused && HM_FUSED_DISCARD) {
    // the partition's records and codes are in shared memory: drop their L2
    // lines (only lines wholly inside this partition's buffer regions)
    auto drop = [&](const void* b0, size_t region, size_t used) {
      const uintptr_t a = reinterpret_cast<uintptr_t>(b0);
      const uintptr_t lo = (a + 127) & ~uintptr_t(127), hi = (a + region) & ~uintptr_t(127);
      const uintptr_t end = min(hi, (a + used + 127) & ~uintptr_t(127));
      for (uintptr_t x = lo + uintptr_t(tid) * 128; x < end; x += uintptr_t(KBCfg<E>::T) * 128)
        asm volatile("discard.global.L2 [%0], 128;" ::"l"(x) : "memory");
    };
    drop(prec, size_t(cap) * sizeof(E), size_t(cnt) * sizeof(E));
    drop(plb + size_t(p) * cap, size_t(cap) * 2, size_t(cnt) * 2);
  }

  // ---- level-2 seed search, map make2 over the multi-key buckets
  // (PAPER.md:286-292); every finished bucket maps its slots to their source
  // items (bucket_done)
  SearchCtx X{sstart, ss, sidx, soff, sA, s_t, staged ? src : nullptr};
  const Items<E> skv{skey, KBCfg<E>::SMEM_ITEM == int(sizeof(E)) ? reinterpret_cast<const E*>(skey) : prec};
  // look-back: exclusive prefix of S over the partitions before p (warp 0,
  // lane i inspects partition qb - i: the closest inclusive prefix plus the
  // aggregates in front of it give the base)
  auto look_back = [&]() {
    unsigned long long base = 0;
    if (p > 0) {
      int64_t qb = int64_t(p) - 1;
      while (true) {
        const int64_t qq = qb - int64_t(lane);
        const unsigned long long v = qq >= 0 ? ld_acquire(&lbstate[qq]) : kFlagInc;
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
        qb -= 32;
      }
      if (lane == 0) st_release(&lbstate[p], kFlagInc | ((base + S_p) & kValMask));
    }
    if (lane == 0) {
      if (p == bp.np - 1) stt->S = base + S_p;
      s_base = base;
    }
  };
  // warp 0 takes the look-back first (the partitions before p published their
  // aggregates right after their scans), then joins the search
  if (warp == 0) look_back();
  HM_TMARK(9);
  search_warp(bp, skv, X, slist + HM_SL(cls_off[2]), s_c9, s_m2, bbase, stt, same, s_bitsw[warp]);
  {
    uint32_t h[8];
    // round r: the list of round r-1's collisions (round 0: every listed
    // bucket, the class-ordered slist), A adjacent lanes per bucket trying
    // attempts tb .. tb + A - 1 (tb = s_t[lb]: 0 in round 0), 32-lane chunks
    // from a shared counter
    uint32_t cur = 0, nxt = 1, prv = 2;  // (the three lists rotate: r % 3, (r + 1) % 3, (r + 2) % 3)
    for (uint32_t r = 0;; r++) {
      const uint16_t* cl = r == 0 ? slist : rlist + cur * lcap;
      const uint32_t n3 = r == 0 ? Lall : s_qn[cur][0], L = r == 0 ? Lall : n3 + s_qn[cur][1];
#ifdef HM_PHASE_TIMING
      if (tid == 0) g_hm_phase[(s_p & 65535u) * 16 + 12] = r;  // (the round count)
      if (r == 1) HM_TMARK(8);
      if (r == 2) HM_TMARK(11);
#endif
      if (L == 0) break;
      if (tid == 0) {  // (the list two rounds back is not read any more)
        s_qn[prv][0] = s_qn[prv][1] = 0;
        s_chunk[prv] = 0;
      }
      // lanes per bucket: round 0 gives the s >= 3 buckets (the front of the
      // list) 2^HM_R0_LOGA lanes and the s = 2 ones 2^HM_R0_LOGA2; later rounds
      // A = lanes / list length (at most 2^HM_RETRY_LOGA)
      uint32_t logA = 0, logA2 = 0, L1 = L;
      if (r == 0) {
        const bool one = bp.flags & HM_FLAG_NO_ROUND0_ILP;
        logA = one ? 0u : uint32_t(HM_R0_LOGA);
        logA2 = one ? 0u : uint32_t(HM_R0_LOGA2);
        L1 = L3;
      } else {
        // the largest logA <= HM_RETRY_LOGA with L << logA <= T (T a power of two:
        // logA = log2 T - ceil(log2 L))
        static_assert((KBCfg<E>::T & (KBCfg<E>::T - 1)) == 0, "T is a power of two");
        const int lg = int(__ffs(KBCfg<E>::T) - 1) - (32 - __clz(L - 1));
        logA = uint32_t(min(max(lg, 0), HM_RETRY_LOGA));
      }
      const uint32_t W1 = L1 << logA, W = W1 + ((L - L1) << logA2);
#if HM_PRED_ATOM
      const uint32_t chunk_sa = smem_u32(&s_chunk[cur]), qn_sa = smem_u32(&s_qn[nxt][0]);
#else
      const uint32_t qn_sa = 0;
#endif
      for (;;) {
#if HM_PRED_ATOM
        uint32_t c = atom_add_if(lane == 0, chunk_sa, 32u);
#else
        uint32_t c = 0;
        if (lane == 0) c = atomicAdd(&s_chunk[cur], 32u);
#endif
        c = __shfl_sync(0xffffffffu, c, 0);
        if (c >= W) break;
        const uint32_t w = c + lane;
        const uint32_t lA = w < W1 ? logA : logA2, A = 1u << lA;
        const uint32_t g = w < W1 ? (w >> logA) : L1 + ((w - W1) >> logA2), j = w & (A - 1u);
        const uint32_t gmask = A == 32 ? 0xffffffffu : (((1u << A) - 1u) << (lane & ~(A - 1u)));
        const bool act = w < W;
        const uint32_t lb = act ? (g < n3 ? cl[g] : cl[lcap - 1 - (g - n3)]) : 0u;
        const uint32_t s = act ? ss[lb] : 0u, tb = act ? s_t[lb] : 0u;
        const uint64_t bits = lane_attempt_k(bp, skv, X, act, lb, s, tb + j, s_m2, bbase, h);
        const uint32_t om = __ballot_sync(0xffffffffu, bits != 0) & gmask;
        if (bits && lane == uint32_t(__ffs(om) - 1)) bucket_done_any(X, lb, s, tb + j, h, bits);
        bool again = false;
        if (act && j == 0 && om == 0) {
          if (tb == 0 && bucket_equal_keys(skv, X, lb, stt, same)) {
            // (equal keys collide under every t: retired, checked once)
          } else if (tb + A >= kT2Cap) {
            atomicOr(&stt->exhausted, 1u);
            s_t[lb] = 0;
          } else {
            s_t[lb] = uint8_t(tb + A);
            again = true;
          }
        }
        list_append(again, lb, s, rlist + nxt * lcap, lcap, s_qn[nxt], qn_sa);
      }
      __syncthreads();
      const uint32_t t3 = prv;
      prv = cur;
      cur = nxt;
      nxt = t3;
    }
  }
  HM_TMARK(4);
  const unsigned long long base = s_base;
  HM_TMARK(5);
  if (ovf) {
    if (tid == 0) atomicOr(&stt->part_overflow, 1u);
    return;
  }
  if (base + S_p > bp.slot_cap) {
    if (tid == 0) atomicOr(&stt->slot_overflow, 1u);
    return;
  }

  // ---- out: the partition's slots [base, base + S_p), consecutive lanes write
  // consecutive records
  if (staged) {
    E* out = slots + base;
    const uint32_t Sp = uint32_t(S_p);
    // (whole groups of 4T slots without per-slot bounds checks, then the rest)
    auto out_group = [&](uint32_t x0, auto full) {
      constexpr bool kFull = decltype(full)::value;
      E e[4];
#pragma unroll
      for (int j = 0; j < 4; j++) {
        const uint32_t x = x0 + j * KBCfg<E>::T + tid;
        if (kFull || x < Sp) {
          const uint32_t v = src[x], it = v & 0x7FFFu;
          e[j] = skv.rec(min(it, cnt - 1u));  // (an unmapped slot only in a pass that is redone; Sp > 0: cnt > 0)
          if (v & 0x8000u) e[j].value = 0;
        }
      }
#pragma unroll
      for (int j = 0; j < 4; j++) {
        const uint32_t x = x0 + j * KBCfg<E>::T + tid;
        if (kFull || x < Sp) out[x] = e[j];
      }
    };
    uint32_t x0 = 0;
#if HM_OUT_FULL
    // (byte keys only: their records come from the partition buffer in global
    // memory, and unchecked groups keep four gathers in flight — 0.924 ->
    // 0.847 ms at C3; the u64 records are in shared memory, 1.911 -> 1.938 ms)
    if constexpr (KBCfg<E>::SMEM_ITEM != int(sizeof(E)))
      for (; x0 + 4 * KBCfg<E>::T <= Sp; x0 += 4 * KBCfg<E>::T) out_group(x0, std::true_type{});
#endif
    for (; x0 < Sp; x0 += 4 * KBCfg<E>::T) out_group(x0, std::false_type{});
  } else {
    // a partition with more slots than the staging map (adversarial level-1
    // distribution within the global bound): direct writes, thread per bucket
    for (uint32_t lb = tid; lb < nbp; lb += KBCfg<E>::T) {
      const uint32_t s = ss[lb];
      if (s == 0 || s > 32) continue;
      E* out = slots + base + soff[lb];
      const uint32_t st0 = sstart[lb];
      if (s == 1) {
        out[0] = skv.rec(sidx[st0]);
        continue;
      }
      const uint32_t s2 = s * s;
      uint32_t hmin = 0xFFFFu, fill = 0;
      for (uint32_t j = 0; j < s; j++) {
        const uint32_t h = sA[st0 + j];
        if (h < hmin) {
          hmin = h;
          fill = sidx[st0 + j];
        }
      }
      E f = skv.rec(fill);
      f.value = 0;
      for (uint32_t x = 0; x < s2; x++) out[x] = f;
      for (uint32_t j = 0; j < s; j++) {
        const uint32_t h = sA[st0 + j];
        if (h < s2) out[h] = skv.rec(sidx[st0 + j]);
      }
    }
  }
  HM_TMARK(6);
  // directory: two buckets per lane, one 16-byte store (lb0 and the pair are
  // even, so the store is aligned)
#if HM_DIR_V4
  if (BP == 4u * KBCfg<E>::T && nbp == BP) {
    // a whole partition: four buckets per thread, one 32-byte store
    const uint32_t lb = 4 * tid;
    const uint4 so4 = *reinterpret_cast<const uint4*>(soff + lb);
    const uint32_t s4 = *reinterpret_cast<const uint32_t*>(ss + lb), t4 = *reinterpret_cast<const uint32_t*>(s_t + lb);
    uint64_t e[4];
    const uint32_t sov[4] = {so4.x, so4.y, so4.z, so4.w};
#pragma unroll
    for (int u = 0; u < 4; u++) {
      const uint32_t su = (s4 >> (8 * u)) & 0xFF, tu = su == 1 ? 0u : (t4 >> (8 * u)) & 0xFF;
      e[u] = dir_entry(base + sov[u], su, tu);
    }
    asm volatile("st.global.v4.u64 [%0], {%1, %2, %3, %4};" ::"l"(dir + lb0 + lb), "l"(e[0]), "l"(e[1]), "l"(e[2]),
                 "l"(e[3])
                 : "memory");
  } else
#endif
  for (uint32_t q = tid; 2 * q < nbp; q += KBCfg<E>::T) {
    const uint32_t lb = 2 * q;
    const uint2 so2 = *reinterpret_cast<const uint2*>(soff + lb);
    const uint32_t s2 = *reinterpret_cast<const uint16_t*>(ss + lb), t2 = *reinterpret_cast<const uint16_t*>(s_t + lb);
    const uint32_t sa = s2 & 0xFF, sb = s2 >> 8, ta = sa == 1 ? 0u : (t2 & 0xFF), tb = sb == 1 ? 0u : (t2 >> 8);
    const uint64_t ea = dir_entry(base + so2.x, sa, ta), eb = dir_entry(base + so2.y, sb, tb);
    if (lb + 1 < nbp) {
      *reinterpret_cast<ulonglong2*>(dir + lb0 + lb) = make_ulonglong2(ea, eb);
    } else {
      dir[lb0 + lb] = ea;
    }
  }
  // compact directory: a lane per 32-bucket record.  Bit i of the four sizes
  // (or attempts) packed in a word x is gathered with one multiply:
  // ((x >> i) & 0x01010101) * 0x01020408 puts the four bits at 24..27.
  for (uint32_t r = tid; 32 * r < nbp; r += KBCfg<E>::T) {
    const uint32_t* s32 = reinterpret_cast<const uint32_t*>(ss + 32 * r);
    const uint32_t* t32 = reinterpret_cast<const uint32_t*>(s_t + 32 * r);
    uint32_t w[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    uint32_t esc = 0;
    const uint32_t nr = nbp - 32 * r;  // (buckets past nbp count as s = 0, t = 0)
#pragma unroll
    for (int k = 0; k < 8; k++) {
      const uint32_t vb = nr >= uint32_t(4 * k + 4) ? 4u : (nr > uint32_t(4 * k) ? nr - 4 * k : 0u);
      const uint32_t bm = vb == 4 ? 0xFFFFFFFFu : ((1u << (8 * vb)) - 1u);
      const uint32_t x = s32[k] & bm, y = t32[k] & bm;
      // escapes: any s >= 7, or s >= 2 with t >= 15 (bytes < 128 after the mask: no carries)
      const uint32_t ge7 = (((x & 0x7F7F7F7Fu) + 0x79797979u) | x) & 0x80808080u;
      const uint32_t ge2 = (((x & 0x7F7F7F7Fu) + 0x7E7E7E7Eu) | x) & 0x80808080u;
      const uint32_t t15 = (((y & 0x7F7F7F7Fu) + 0x71717171u) | y) & 0x80808080u;
      esc |= ge7 | (ge2 & t15);
#pragma unroll
      for (int i = 0; i < 3; i++)
        w[1 + i] |= ((((x >> (2 - i)) & 0x01010101u) * 0x01020408u) >> 24) << (4 * k);
#pragma unroll
      for (int i = 0; i < 4; i++) w[4 + i] |= ((((y >> i) & 0x01010101u) * 0x01020408u) >> 24) << (4 * k);
    }
    if (esc || (bp.flags & HM_FLAG_FULL_DIRECTORY)) w[1] = w[2] = w[3] = 0xffffffffu;
    w[0] = uint32_t(base + soff[32 * r]);
    uint4* o = reinterpret_cast<uint4*>(cdir + ((lb0 >> 5) + r));
    o[0] = make_uint4(w[0], w[1], w[2], w[3]);
    o[1] = make_uint4(w[4], w[5], w[6], w[7]);
  }
  HM_TMARK(7);
#undef HM_SL
}

template <class E, class Same, uint32_t kCap>
__global__ void __launch_bounds__(KBCfg<E>::T, KBCfg<E>::MINB)
    k_bucket(BuildParams bp, const E* __restrict__ pbuf, const uint16_t* __restrict__ plb,
             const unsigned int* __restrict__ pcount,
             unsigned long long* __restrict__ lbstate, uint64_t* __restrict__ dir, CDir* __restrict__ cdir,
             E* __restrict__ slots, DevStatus* __restrict__ stt, Same same) {
  extern __shared__ __align__(16) uint8_t smem[];
  bucket_body<E, Same, false, kCap>(bp, pbuf, plb, pcount, lbstate, dir, cdir, slots, stt, same, smem, 0, nullptr,
                                    0);
}


// The fused pass 2 + k_bucket pipeline (u64 keys, HM_FLAG_FUSED_PASS2): one kernel whose CTAs take
// jobs in ticket order — the pass-2 tiles of coarse region c + D come before the
// k_bucket partitions of region c — so that a region's partitions are consumed
// from L2 shortly after pass 2 wrote them (and discarded there), and the
// bandwidth-bound tiles run beside the issue-bound partitions on the same SMs.
// A partition job waits for its region's tiles (per-region done counters);
// every job it can wait for holds an earlier ticket, so the wait always ends.
struct FuseArgs {
  unsigned int* sdone;  // per coarse region: pass-2 tiles finished
  uint32_t R, tpc, sdig, D;
};
__device__ __forceinline__ void fused_job(const FuseArgs& f, uint32_t j, bool* split, uint32_t* x) {
  const uint32_t D = min(f.D, f.R), pre = D * f.tpc;
  if (j < pre) {
    *split = true;
    *x = j;  // region j / tpc, tile j % tpc
    return;
  }
  j -= pre;
  const uint32_t full = f.R - D, seg = f.tpc + f.sdig;
  if (j < full * seg) {
    const uint32_t k = j / seg, r = j % seg;
    *split = r < f.tpc;
    *x = *split ? (k + D) * f.tpc + r : k * f.sdig + (r - f.tpc);
    return;
  }
  j -= full * seg;
  *split = false;
  *x = (full + j / f.sdig) * f.sdig + j % f.sdig;
}

template <class Src, class E, class Same, int BITS>
__global__ void __launch_bounds__(KBCfg<E>::T, KBCfg<E>::MINB)
    k_split2_bucket(Src src, BuildParams bp, SplitArgs a, FuseArgs f, const E* __restrict__ pbuf,
                    const uint16_t* __restrict__ plb, const unsigned int* pcount,
                    unsigned long long* __restrict__ lbstate, uint64_t* __restrict__ dir, CDir* __restrict__ cdir,
                    E* __restrict__ slots, DevStatus* __restrict__ stt, Same same) {
  extern __shared__ __align__(16) uint8_t smem[];
  if constexpr (KBCfg<E>::T != kSThreads) {  // (one block size for both job kinds; the host checks)
    return;
  } else {
    __shared__ uint32_t s_job;
    if (threadIdx.x == 0) s_job = atomicAdd(&stt->ticket, 1u);
    __syncthreads();
    bool split;
    uint32_t x;
    fused_job(f, s_job, &split, &x);
    if (split) {
      split_tile_body<Src, E, 2, BITS>(src, bp, a, stt, x, smem);
      __syncthreads();
      if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(&f.sdone[x / f.tpc], 1u);
      }
      return;
    }
    if (x >= bp.np) return;
    bucket_body<E, Same, true, 0>(bp, pbuf, plb, pcount, lbstate, dir, cdir, slots, stt, same, smem, x,
                               f.sdone + x / f.sdig, f.tpc);
  }
}

// ------------------------------------------------------- overflow check
// A build partition that overflowed its buffer (a degenerate level-1
// distribution: many equal keys, or an adversarial key set) lost records, so
// its S_p is unknown.  These two kernels recount the level-1 histogram of the
// suspect partitions straight from the input and sum their s^2, so that the
// space bound R7 decides as the oracle does (redraw level one, and after 16
// draws SEED_EXHAUSTED); if the bound holds the build reports TOO_LARGE (a
// bucket this version cannot hold).
template <class Src>
__global__ void k_heavy_hist(Src src, BuildParams bp, const uint32_t* __restrict__ hidx, uint32_t* __restrict__ hcnt) {
  const uint32_t BP = 1u << bp.log2_bp;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < bp.n_in; i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t lb = level1_bucket(bp.l1, src.load(i).key) - bp.b_lo;
    if (lb >= bp.nb) continue;
    const uint32_t h = hidx[lb >> bp.log2_bp];
    if (h != ~0u) atomicAdd(&hcnt[size_t(h) * BP + (lb & (BP - 1))], 1u);
  }
}
__global__ void k_heavy_sq(const uint32_t* __restrict__ hcnt, uint64_t total, unsigned long long* out) {
  unsigned long long acc = 0;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < total; i += uint64_t(gridDim.x) * blockDim.x)
    acc += uint64_t(hcnt[i]) * hcnt[i];
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0 && acc) atomicAdd(out, acc);
}

// ------------------------------------------------------------- host side
static size_t bucket_smem_bytes(uint32_t cap, uint32_t log2_bp, uint32_t esz) {
  return bucket_smem_layout(cap, 1u << log2_bp, esz).total;
}

// Per-device caches of the host-side launch configuration.
static std::mutex g_attr_mu;
static std::map<std::pair<int, const void*>, int> g_smem_set;                    // dynamic smem limit set
static std::map<std::tuple<int, const void*, int, size_t>, int> g_occ;           // blocks per SM
static cudaError_t device_smem(int* optin, int* per_sm) {
  static std::map<int, std::pair<int, int>> cache;  // device -> (opt-in per block, per SM)
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  {
    std::lock_guard<std::mutex> g(g_attr_mu);
    auto it = cache.find(dev);
    if (it != cache.end()) {
      *optin = it->second.first;
      *per_sm = it->second.second;
      return cudaSuccess;
    }
  }
  if ((e = cudaDeviceGetAttribute(optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev)) != cudaSuccess) return e;
  if ((e = cudaDeviceGetAttribute(per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev)) != cudaSuccess) return e;
  std::lock_guard<std::mutex> g(g_attr_mu);
  cache[dev] = {*optin, *per_sm};
  return cudaSuccess;
}
static cudaError_t ensure_smem(const void* fn, int bytes) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  {
    std::lock_guard<std::mutex> g(g_attr_mu);
    auto it = g_smem_set.find({dev, fn});
    if (it != g_smem_set.end() && it->second >= bytes) return cudaSuccess;
  }
  if ((e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes)) != cudaSuccess) return e;
  std::lock_guard<std::mutex> g(g_attr_mu);
  int& v = g_smem_set[{dev, fn}];
  v = std::max(v, bytes);
  return cudaSuccess;
}
static cudaError_t occupancy(int* blocks, const void* fn, int threads, size_t smem) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const auto key = std::make_tuple(dev, fn, threads, smem);
  {
    std::lock_guard<std::mutex> g(g_attr_mu);
    auto it = g_occ.find(key);
    if (it != g_occ.end()) {
      *blocks = it->second;
      return cudaSuccess;
    }
  }
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks, fn, threads, smem)) != cudaSuccess) return e;
  std::lock_guard<std::mutex> g(g_attr_mu);
  g_occ[key] = *blocks;
  return cudaSuccess;
}

struct Plan {
  uint32_t log2_bp, np, cap;
  size_t smemB;
};

// Partition geometry: the largest BP = 2^lg (at most 2^12: 64 groups of 64
// buckets) whose k_bucket shared memory lets KBCfg<E>::MINB CTAs share an SM
// (smem_two: the register-limited occupancy at 64 registers per thread); with
// at least 4 partitions per SM for small tables.  An
// explicit log2_req only has to fit one CTA per SM (smem_one).
static Plan make_plan(uint64_t n_in, uint64_t nb, uint32_t log2_req, uint32_t esz, size_t smem_two,
                      size_t smem_one) {
  Plan pl{};
  const int sms = num_sms();
  // (at least 2^5 buckets: a compact-directory record covers 32 buckets and
  // is written by the one partition that holds them)
  uint32_t lg = log2_req ? std::min<uint32_t>(std::max<uint32_t>(log2_req, 5u), 12u) : 12u;
  const size_t limit = log2_req ? smem_one : smem_two;
  if (!log2_req) {
#ifndef HM_PLAN_PPS
#define HM_PLAN_PPS 2  // small tables: at least this many build partitions per SM (4: 2^16 builds 0.100 -> 0.085 ms with 2)
#endif
    while (lg > 6 && (nb >> lg) < uint64_t(HM_PLAN_PPS * sms)) lg--;
  }
  for (;; lg--) {
    const double BP = double(uint64_t(1) << lg);
    const double m = double(n_in) * BP / double(std::max<uint64_t>(nb, 1));
    double c = m + 8.0 * std::sqrt(std::max(m, 1.0)) + 64.0;
    uint32_t cap = uint32_t(std::min(16383.0, std::ceil(c / 32.0) * 32.0));
    const size_t sm = bucket_smem_bytes(cap, lg, esz);
    if ((sm <= limit && c <= 16383.0) || lg <= 5) {
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
enum WsRole { WS_FP, WS_BAD, WS_PBUF, WS_PLB, WS_PCOUNT, WS_LBSTATE, WS_DSTAT, WS_CBUF, WS_CCOUNT, WS_DEDUP, WS_SDONE, WS_ZERO, WS_NROLES };
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

// Map arrays freed by hm_free, kept per (device, size) for the next build.
// Builds of a size take their dir/cdir/slots from here; without it the
// stream-ordered pool, fragmented by the other sizes, mapped fresh memory for
// a 2 GB slot array on build after build (50-100 ms each at 2^26, measured).
// Capped at kMapCacheCap bytes; hm_release_workspace() empties it.
static std::multimap<std::pair<int, size_t>, void*> g_mapcache;
static size_t g_mapcache_bytes = 0;
constexpr size_t kMapCacheCap = size_t(32) << 30;

thread_local UserAlloc tl_user_alloc;

hm_status map_alloc(void** p, size_t bytes, cudaStream_t st) {
  bytes = std::max<size_t>(bytes, 16);
  if (tl_user_alloc.alloc) {
    *p = tl_user_alloc.alloc(bytes, reinterpret_cast<void*>(st), tl_user_alloc.ctx);
    if (!*p) {
      set_error("the user allocator (hm_opts.alloc) returned NULL for " + std::to_string(bytes) + " bytes");
      return HM_ERR_OOM;
    }
    if (reinterpret_cast<uintptr_t>(*p) & 31u) {  // (32-byte slot and compact-directory records, 32-B vector loads)
      tl_user_alloc.free(*p, bytes, reinterpret_cast<void*>(st), tl_user_alloc.ctx);
      *p = nullptr;
      set_error("the user allocator (hm_opts.alloc) returned a pointer that is not 32-byte aligned");
      return HM_ERR_INVALID_ARG;
    }
    return HM_OK;
  }
  int dev = 0;
  HM_CUDA_TRY(cudaGetDevice(&dev));
  {
    std::lock_guard<std::mutex> lk(g_ws_mu);
    auto it = g_mapcache.find({dev, bytes});
    if (it != g_mapcache.end()) {
      *p = it->second;
      g_mapcache.erase(it);
      g_mapcache_bytes -= bytes;
      return HM_OK;
    }
  }
  return dmalloc(p, bytes, st);
}

void map_discard(void* p, size_t bytes, cudaStream_t st) {
  if (!p) return;
  if (tl_user_alloc.free) tl_user_alloc.free(p, std::max<size_t>(bytes, 16), reinterpret_cast<void*>(st), tl_user_alloc.ctx);
  else cudaFreeAsync(p, st);
}

void map_release(void* p, size_t bytes) {
  if (!p) return;
  bytes = std::max<size_t>(bytes, 16);
  int dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) {
    std::lock_guard<std::mutex> lk(g_ws_mu);
    if (g_mapcache_bytes + bytes <= kMapCacheCap) {
      g_mapcache.insert({{dev, bytes}, p});
      g_mapcache_bytes += bytes;
      return;
    }
  }
  cudaFree(p);
}

// The from_array dedup set (dedup.cu) lives in the same cache.
hm_status dedup_workspace(void** p, size_t bytes, cudaStream_t st) {
  Scratch sc{st};
  uint8_t* q = nullptr;
  hm_status s = sc.alloc(WS_DEDUP, &q, bytes);
  *p = q;
  return s;
}

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
  for (auto it = g_mapcache.begin(); it != g_mapcache.end();) {
    if (it->first.first == dev) {
      cudaFree(it->second);
      g_mapcache_bytes -= it->first.second;
      it = g_mapcache.erase(it);
    } else {
      ++it;
    }
  }
  HM_CUDA_TRY(cudaDeviceSynchronize());
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
  cudaGetLastError();
  return HM_OK;
}

// Builds one table for buckets [b_lo, b_lo+nb) of a level-1 function mod
// n_global from the n_in elements produced by `src`.
template <class Src, class E, class Same>
static hm_status build_core(Src src, Same same, uint64_t n_in, uint64_t n_global, uint64_t b_lo, uint64_t nb,
                            int t1_fixed, uint64_t seed, uint32_t log2_req, cudaStream_t st, BuildOut* out,
                            bool* fpcoll, SideJob* job = nullptr) {
  *fpcoll = false;
  // (device attributes, the kernels' static shared memory, their dynamic
  // shared-memory limits and occupancies are queried once per device: a
  // build's fixed cost is its launches, not these host calls)
  int smem_optin = 0, smem_sm = 0;
  HM_CUDA_TRY(device_smem(&smem_optin, &smem_sm));
  static std::atomic<size_t> static_smem_cache{0};  // k_bucket's static shared memory (~2.6 KB; one binary)
  size_t static_smem_B = static_smem_cache.load();
  if (!static_smem_B) {
    size_t v = 4096;
    cudaFuncAttributes fa{};
    if (cudaFuncGetAttributes(&fa, k_bucket<E, Same, 0>) == cudaSuccess) v = fa.sharedSizeBytes;
    else cudaGetLastError();
    if constexpr (sizeof(E) == sizeof(KV16)) {  // (the fused kernel holds pass 2's static arrays too)
      if (cudaFuncGetAttributes(&fa, k_split2_bucket<Src, E, Same, 9>) == cudaSuccess)
        v = std::max<size_t>(v, fa.sharedSizeBytes);
      else cudaGetLastError();
    }
    static_smem_B = v;
    static_smem_cache.store(v);
  }
  const uint32_t knob_flags = log2_req >> 16;
  log2_req &= 0xFFFFu;
  const Plan pl = make_plan(n_in, nb, log2_req, uint32_t(KBCfg<E>::SMEM_ITEM), size_t(smem_sm) / KBCfg<E>::MINB - 1024 - static_smem_B,
                            size_t(smem_optin) - static_smem_B);
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
  uint16_t* plb = nullptr;
  if ((s = sc.alloc(WS_PLB, &plb, size_t(pl.np) * pl.cap * 2)) != HM_OK) return s;
  // the counters a pass starts from zero, one block (one memset per level-1
  // draw): status | look-back words | partition counts | coarse counts
  const size_t z_lb = 256, z_pc = z_lb + size_t(pl.np) * 8, z_cc = z_pc + al16(size_t(pl.np) * 4),
               z_end = z_cc + al16(size_t(pl.np / 256 + 2) * 4);
  static_assert(sizeof(DevStatus) <= 256, "status block");
  uint8_t* zblk = nullptr;
  if ((s = sc.alloc(WS_ZERO, &zblk, z_end)) != HM_OK) return s;
  dstat = reinterpret_cast<DevStatus*>(zblk);
  lbstate = reinterpret_cast<unsigned long long*>(zblk + z_lb);
  pcount = reinterpret_cast<unsigned int*>(zblk + z_pc);

  uint64_t* dir = nullptr;
  E* slots = nullptr;
  CDir* cdir = nullptr;
  const size_t dir_bytes = nb * 8, cdir_bytes = ((nb + 31) / 32) * sizeof(CDir);
  if ((s = map_alloc(reinterpret_cast<void**>(&dir), dir_bytes, st)) != HM_OK) return s;
  if ((s = map_alloc(reinterpret_cast<void**>(&cdir), cdir_bytes, st)) != HM_OK) {
    map_discard(dir, dir_bytes, st);
    return s;
  }
  const double sn = double(n_in);
  uint64_t slot_cap = uint64_t(2.0 * sn + 8.0 * std::sqrt(2.0 * sn + 1.0) + 1024.0);
  if (n_in <= 4096) slot_cap = std::max<uint64_t>(slot_cap, 4 * std::max<uint64_t>(n_in, 1));
  if ((s = map_alloc(reinterpret_cast<void**>(&slots), slot_cap * sizeof(E), st)) != HM_OK) {
    map_discard(dir, dir_bytes, st);
    map_discard(cdir, cdir_bytes, st);
    return s;
  }
  auto fail = [&](hm_status code) {
    map_discard(dir, dir_bytes, st);
    map_discard(cdir, cdir_bytes, st);
    map_discard(slots, slot_cap * sizeof(E), st);
    return code;
  };

  // kernel configuration
  constexpr int KPT = sizeof(E) == 16 ? 16 : 8;
  const size_t smemA = size_t(pl.np) * 4;
  const bool smemHist = smemA <= size_t(smem_optin) - 1024;
  auto kA_s = k_partition<Src, E, KPT, true>;
  auto kA_g = k_partition<Src, E, KPT, false>;
  auto kB = pl.log2_bp == KBCfg<E>::FIX_LOG2 && pl.cap == KBCfg<E>::FIX_CAP ? k_bucket<E, Same, KBCfg<E>::FIX_CAP>
                                                                              : k_bucket<E, Same, 0>;
  if (smemHist) HM_CUDA_TRY(ensure_smem(reinterpret_cast<const void*>(kA_s), int(smemA)));
  HM_CUDA_TRY(ensure_smem(reinterpret_cast<const void*>(kB), int(pl.smemB)));
  int occA = 1;
  if (smemHist) HM_CUDA_TRY(occupancy(&occA, reinterpret_cast<const void*>(kA_s), kAThreads, smemA));
  else HM_CUDA_TRY(occupancy(&occA, reinterpret_cast<const void*>(kA_g), kAThreads, 0));
  occA = std::max(occA, 1);
  const uint64_t T = uint64_t(kAThreads) * KPT;
  const uint64_t ntiles = (n_in + T - 1) / T;
  const unsigned gridA = unsigned(std::max<uint64_t>(1, std::min<uint64_t>(ntiles, uint64_t(sms) * occA)));
  // large tables: two coalesced radix passes (256- or 512-way) over the
  // partition id instead of one np-way scatter
  const bool two_pass = pl.np > 1024 && pl.np <= (1u << 18);
  const int sbits = pl.np <= 65536 ? 8 : 9;
  const uint32_t sdig = 1u << sbits;
  uint32_t ncoarse = 0, ccap = 0, tpc = 0;
  E* cbuf = nullptr;
  unsigned int* ccount = nullptr;
  constexpr int kSTile = split_tile<E>();
  const size_t smemS = size_t(kSTile) * (sizeof(E) + 4);
  // pass 1: HM_SPLIT1_T-thread tiles for 8-bit digits (one digit per thread in the scan)
  auto kS1 = sbits == 8 ? k_split<Src, E, 1, 8, HM_SPLIT1_T> : k_split<Src, E, 1, 9>;
  const int s1T = sbits == 8 ? HM_SPLIT1_T : kSThreads;
  const int s1Tile = s1T * split_pt<E>();
  const size_t smemS1 = size_t(s1Tile) * (sizeof(E) + 4);
  auto kS2 = sbits == 8 ? k_split<Src, E, 2, 8> : k_split<Src, E, 2, 9>;
  if (two_pass) {
    ncoarse = (pl.np + sdig - 1) / sdig;
    const double mc = double(n_in) * double(sdig) * double(uint64_t(1) << pl.log2_bp) / double(nb);
    ccap = uint32_t(mc + 8.0 * std::sqrt(mc + 1.0) + 1024.0);
    tpc = (ccap + kSTile - 1) / kSTile;

    if ((s = sc.alloc(WS_CBUF, &cbuf, size_t(ncoarse) * ccap * sizeof(E))) != HM_OK) return fail(s);
    ccount = reinterpret_cast<unsigned int*>(zblk + z_cc);  // (ncoarse <= np / 256 + 1)
    HM_CUDA_TRY(ensure_smem(reinterpret_cast<const void*>(kS1), int(smemS1)));
    HM_CUDA_TRY(ensure_smem(reinterpret_cast<const void*>(kS2), int(smemS)));
  }
  // HM_FLAG_FUSED_PASS2 (u64 keys, opt-in): pass 2 and k_bucket as one pipelined kernel (k_split2_bucket)
  const bool fused = two_pass && sizeof(E) == sizeof(KV16) && !job && (knob_flags & HM_FLAG_FUSED_PASS2) &&
                     KBCfg<E>::T == kSThreads;
  const size_t smemF = std::max(smemS, pl.smemB);
  unsigned int* sdone = nullptr;
  if constexpr (sizeof(E) == sizeof(KV16)) {
    if (fused) {
      auto kF = sbits == 8 ? k_split2_bucket<Src, E, Same, 8> : k_split2_bucket<Src, E, Same, 9>;
      if ((s = sc.alloc(WS_SDONE, &sdone, size_t(ncoarse) * 4)) != HM_OK) return fail(s);
      HM_CUDA_TRY(ensure_smem(reinterpret_cast<const void*>(kF), int(smemF)));
    }
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
  bp.sl = bucket_smem_layout(pl.cap, 1u << pl.log2_bp, uint32_t(KBCfg<E>::SMEM_ITEM));
  for (int i = 0; i < 33; i++) bp.m2[i] = i ? ~0ull / (uint64_t(i) * i) : 0ull;

  DevStatus hs{};
  const uint32_t t1_lo = t1_fixed >= 0 ? uint32_t(t1_fixed) : 0u;
  const uint32_t t1_hi = t1_fixed >= 0 ? uint32_t(t1_fixed) + 1 : kT1Cap;
  for (uint32_t t1 = t1_lo; t1 < t1_hi; t1++) {
    bp.l1 = make_l1(smix, t1, n_global);
    bp.slot_cap = slot_cap;
    HM_CUDA_TRY(cudaMemsetAsync(zblk, 0, z_end, st));
    bool run_a = true;
    for (int pass = 0; pass < 3; pass++) {
      if (pass > 0) HM_CUDA_TRY(cudaMemsetAsync(zblk, 0, z_pc, st));  // (a rerun: status and look-back words)
      if (run_a && ntiles > 0 && two_pass) {
        const SplitArgs a1{nullptr, nullptr, 0, 0, cbuf, ccount, ccap, ncoarse, 0};
        {
          LaunchScope ls_("k_split1", st);
          kS1<<<unsigned((n_in + s1Tile - 1) / s1Tile), s1T, smemS1, st>>>(src, bp, a1, dstat);
        }
        HM_CUDA_TRY(cudaGetLastError());
        if (!fused) {
          const SplitArgs a2{cbuf, ccount, ccap, tpc, pbuf, pcount, pl.cap, pl.np, ncoarse, plb};
          LaunchScope ls_("k_split2", st);
          kS2<<<ncoarse * tpc, kSThreads, smemS, st>>>(src, bp, a2, dstat);
        }
        HM_CUDA_TRY(cudaGetLastError());
      } else if (run_a && ntiles > 0) {
        {
          LaunchScope ls_("k_partition", st);
          if (smemHist) kA_s<<<gridA, kAThreads, smemA, st>>>(src, bp, pbuf, plb, pcount, dstat);
          else kA_g<<<gridA, kAThreads, 0, st>>>(src, bp, pbuf, plb, pcount, dstat);
        }
        HM_CUDA_TRY(cudaGetLastError());
      }
      run_a = false;
      bp.cp_bytes = 0;
      if (job && !job->done && job->kbytes) {
        bp.cp_src = job->ksrc;
        bp.cp_dst = job->kdst;
        bp.cp_bytes = job->kbytes;
        bp.cp_slice = ((job->kbytes + pl.np - 1) / pl.np + 15) & ~uint64_t(15);
        job->done = true;
      } else if (job) {
        job->run(st);
      }
      if (fused) {
        // (a rerun after a slot overflow repeats pass 2 too: the partitions were
        // dropped from L2 as they were consumed; the coarse buffer is intact)
        if (pass > 0) HM_CUDA_TRY(cudaMemsetAsync(pcount, 0, size_t(pl.np) * 4, st));
        HM_CUDA_TRY(cudaMemsetAsync(sdone, 0, size_t(ncoarse) * 4, st));
        const SplitArgs a2{cbuf, ccount, ccap, tpc, pbuf, pcount, pl.cap, pl.np, ncoarse, plb};
        const FuseArgs fa{sdone, ncoarse, tpc, sdig, uint32_t(HM_FUSED_D)};
        if constexpr (sizeof(E) == sizeof(KV16)) {
          auto kF = sbits == 8 ? k_split2_bucket<Src, E, Same, 8> : k_split2_bucket<Src, E, Same, 9>;
          LaunchScope ls_("k_split2_bucket", st);
          kF<<<ncoarse * (tpc + sdig), KBCfg<E>::T, smemF, st>>>(src, bp, a2, fa, pbuf, plb, pcount, lbstate, dir,
                                                                  cdir, slots, dstat, same);
        }
      } else {
        LaunchScope ls_("k_bucket", st);
        kB<<<pl.np, KBCfg<E>::T, pl.smemB, st>>>(bp, pbuf, plb, pcount, lbstate, dir, cdir, slots, dstat, same);
      }
      HM_CUDA_TRY(cudaGetLastError());
      HM_CUDA_TRY(cudaMemcpyAsync(&hs, dstat, sizeof(hs), cudaMemcpyDeviceToHost, st));
      HM_CUDA_TRY(cudaStreamSynchronize(st));
      if (hs.pad) {
        set_error("a routed key does not belong to this shard's bucket range");
        return fail(HM_ERR_INVALID_ARG);
      }
      if (hs.part_overflow) {
        // recount the suspect partitions (k_heavy_*) for the space bound R7
        std::vector<unsigned int> hp(pl.np), hc(two_pass ? ncoarse : 0);
        HM_CUDA_TRY(cudaMemcpyAsync(hp.data(), pcount, size_t(pl.np) * 4, cudaMemcpyDeviceToHost, st));
        if (two_pass) HM_CUDA_TRY(cudaMemcpyAsync(hc.data(), ccount, size_t(ncoarse) * 4, cudaMemcpyDeviceToHost, st));
        HM_CUDA_TRY(cudaStreamSynchronize(st));
        std::vector<uint32_t> hidx(pl.np, ~0u);
        uint32_t nh = 0;
        for (uint32_t q = 0; q < pl.np; q++)
          if (hp[q] > pl.cap) hidx[q] = nh++;
        for (uint32_t c = 0; c < hc.size(); c++)
          if (hc[c] > ccap)
            for (uint32_t d = 0; d < sdig && c * sdig + d < pl.np; d++)
              if (hidx[c * sdig + d] == ~0u) hidx[c * sdig + d] = nh++;
        if (nh == 0 || nh > 1024) {
          set_error("build partition overflow (degenerate key distribution); not supported in this version");
          return fail(HM_ERR_TOO_LARGE);
        }
        const size_t BPz = size_t(1) << pl.log2_bp;
        uint32_t *d_hidx = nullptr, *d_hcnt = nullptr;
        unsigned long long* d_sq = nullptr;
        if ((s = dmalloc(&d_hidx, size_t(pl.np) * 4, st)) != HM_OK) return fail(s);
        if ((s = dmalloc(&d_hcnt, size_t(nh) * BPz * 4, st)) != HM_OK) return fail(s);
        if ((s = dmalloc(&d_sq, 8, st)) != HM_OK) return fail(s);
        HM_CUDA_TRY(cudaMemcpyAsync(d_hidx, hidx.data(), size_t(pl.np) * 4, cudaMemcpyHostToDevice, st));
        HM_CUDA_TRY(cudaMemsetAsync(d_hcnt, 0, size_t(nh) * BPz * 4, st));
        HM_CUDA_TRY(cudaMemsetAsync(d_sq, 0, 8, st));
        {
          LaunchScope ls_("k_heavy_hist", st);
          k_heavy_hist<Src><<<unsigned(sms) * 8, 256, 0, st>>>(src, bp, d_hidx, d_hcnt);
        }
        {
          LaunchScope ls_("k_heavy_sq", st);
          k_heavy_sq<<<unsigned(sms) * 4, 256, 0, st>>>(d_hcnt, uint64_t(nh) * BPz, d_sq);
        }
        unsigned long long heavy = 0;
        HM_CUDA_TRY(cudaMemcpyAsync(&heavy, d_sq, 8, cudaMemcpyDeviceToHost, st));
        HM_CUDA_TRY(cudaStreamSynchronize(st));
        cudaFreeAsync(d_hidx, st);
        cudaFreeAsync(d_hcnt, st);
        cudaFreeAsync(d_sq, st);
        if (hs.S + heavy > 4 * n_global) {  // R7: level one redraws, as the oracle does
          hs.S += heavy;
          hs.bound_fail = 1;
          hs.part_overflow = 0;
          break;
        }
        set_error("build partition overflow (degenerate key distribution) within the space bound; "
                  "not supported in this version");
        return fail(HM_ERR_TOO_LARGE);
      }
      if (hs.S > 4 * n_global || hs.bound_fail) break;  // R7: redraw level one
      if (hs.slot_overflow && !(hs.bound_fail)) {
        // more slots than the allocation: grow to exactly S and rerun K_B
        map_discard(slots, slot_cap * sizeof(E), st);
        slots = nullptr;
        slot_cap = hs.S;
        bp.slot_cap = slot_cap;
        if ((s = map_alloc(reinterpret_cast<void**>(&slots), slot_cap * sizeof(E), st)) != HM_OK) {
          map_discard(dir, dir_bytes, st);
          map_discard(cdir, cdir_bytes, st);
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
      out->bytes[0] = dir_bytes;
      out->bytes[1] = cdir_bytes;
      out->bytes[2] = slot_cap * sizeof(E);
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
    out->bytes[0] = dir_bytes;
    out->bytes[1] = cdir_bytes;
    out->bytes[2] = slot_cap * sizeof(E);
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
// Fingerprints (R5) of all keys, expanded form.  A warp takes 32 consecutive
// keys (a tile), stages their contiguous byte range in shared memory, and
// every lane fingerprints its key from there (fingerprint_sm32).  The staging
// is double-buffered with cp.async: while a warp fingerprints tile t, the
// bytes of its next tile are in flight and the offsets of the one after are
// being loaded, so each warp keeps two tiles of DRAM reads outstanding.  A
// range longer than the stage (keys of hundreds of bytes) is read directly.
// (Writing the map's context copy from the stage as well measured slower than
// the separate copy running beside the build: 2.25 vs 2.21 ms at C3.)
constexpr int kFpThreads = 256, kFpWarps = kFpThreads / 32, kFpStage16 = 96;  // (16-byte units per buffer)
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}
struct FpTile {
  uint64_t g0;  // 16-aligned address of the staged range
  bool staged;
};
#ifndef HM_FP_MINB
#define HM_FP_MINB 4
#endif
__global__ void __launch_bounds__(kFpThreads, HM_FP_MINB) k_fingerprint(const uint8_t* __restrict__ bytes,
                                                            const uint64_t* __restrict__ offs, uint64_t n, uint64_t r,
                                                            uint64_t* __restrict__ fp) {
  __shared__ FpPow s_pw;
  // (+1 unit: fingerprint_sm32 reads up to two words past a key)
  __shared__ __align__(16) uint4 s_stage[kFpWarps][2][kFpStage16 + 1];
  if (threadIdx.x == 0) fp_pow_fill(&s_pw, r);
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint64_t stride = uint64_t(gridDim.x) * kFpWarps * 32;
  const uint64_t B = reinterpret_cast<uintptr_t>(bytes);
  auto load_offs = [&](uint64_t t0, uint64_t& o, uint64_t& o1) {
    const uint64_t i = t0 + lane;
    o = i < n ? __ldg(offs + i) : 0;
    o1 = i < n ? __ldg(offs + i + 1) : 0;
  };
  // stage tile t0's bytes into buffer bf (one cp.async group, possibly empty)
  auto issue = [&](uint64_t t0, uint64_t o, uint64_t o1, int bf) {
    FpTile T{0, false};
    if (t0 < n) {  // (warp-uniform)
      const uint32_t lastl = n - 1 - t0 < 31 ? uint32_t(n - 1 - t0) : 31u;
      const uint64_t start = __shfl_sync(0xffffffffu, o, 0), end = __shfl_sync(0xffffffffu, o1, lastl);
      T.g0 = (B + start) & ~uint64_t(15);  // (an address: 16-aligned units of any byte pointer)
      const uint32_t units = end > start ? uint32_t((B + end - T.g0 + 15) >> 4) : 0u;  // (keys <= 65535 bytes)
      T.staged = units <= uint32_t(kFpStage16);
      if (T.staged)
        for (uint32_t k = lane; k < units; k += 32)
          cp_async16(&s_stage[w][bf][k], reinterpret_cast<const void*>(T.g0 + 16ull * k));
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    return T;
  };
  uint64_t t = (uint64_t(blockIdx.x) * kFpWarps + w) * 32;
  uint64_t o, o1, on, o1n;
  load_offs(t, o, o1);
  FpTile cur = issue(t, o, o1, 0);
  load_offs(t + stride, on, o1n);
  int bf = 0;
  for (; t < n; t += stride) {
    const FpTile nxt = issue(t + stride, on, o1n, bf ^ 1);
    uint64_t onn, o1nn;
    load_offs(t + 2 * stride, onn, o1nn);
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    __syncwarp();
    if (t + lane < n) {
      const uint64_t len = o1 - o;
      fp[t + lane] = cur.staged && len <= 4ull * kFpPowMax
                         ? fingerprint_sm32(reinterpret_cast<const uint32_t*>(s_stage[w][bf]), uint32_t(B + o - cur.g0),
                                            uint32_t(len), &s_pw)
                         : fingerprint_pw64(bytes, o, len, r, &s_pw);
    }
    __syncwarp();
    o = on;
    o1 = o1n;
    on = onn;
    o1n = o1nn;
    cur = nxt;
    bf ^= 1;
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
}

// (four keys per thread and iteration: eight loads in flight)
__global__ void k_check_offsets(const uint64_t* __restrict__ offs, uint64_t n, unsigned int* bad) {
  const uint64_t T = uint64_t(gridDim.x) * blockDim.x;
  uint32_t f = 0;
  for (uint64_t i0 = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i0 < n; i0 += 4 * T) {
    uint64_t o[4], o1[4];
#pragma unroll
    for (int u = 0; u < 4; u++) {
      const uint64_t i = i0 + u * T;
      o[u] = i < n ? __ldg(offs + i) : 0;
      o1[u] = i < n ? __ldg(offs + i + 1) : 0;
    }
#pragma unroll
    for (int u = 0; u < 4; u++) f |= o1[u] < o[u] ? 1u : (o1[u] - o[u] > 65535 ? 2u : 0u);
  }
  if (f) atomicOr(bad, f);
}

void launch_fingerprint(const uint8_t* bytes, const uint64_t* offs, uint64_t n, uint64_t r, uint64_t* fp,
                        cudaStream_t st) {
  // one wave of resident blocks (the grid-stride loop pipelines per warp)
  static int per_sm = 0;
  if (!per_sm && cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_fingerprint, kFpThreads, 0) != cudaSuccess)
    per_sm = 4;
  per_sm = std::max(per_sm, 1);
#ifndef HM_FP_WAVES
#define HM_FP_WAVES 4  // grid: 4 waves of resident blocks (0.319 -> 0.310 ms at C3; 16: 0.333)
#endif
  const unsigned grid =
      unsigned(std::min<uint64_t>((n + kFpThreads - 1) / kFpThreads, uint64_t(num_sms()) * per_sm * HM_FP_WAVES));
  {
    LaunchScope ls_("k_fingerprint", st);
    k_fingerprint<<<std::max(grid, 1u), kFpThreads, 0, st>>>(bytes, offs, n, r, fp);
  }
}

// The key context's validity (hm.h): offsets non-decreasing (INVALID_ARG) and
// every key at most 65535 bytes (TOO_LARGE, R23).  Runs before anything reads
// the bytes (the from_array dedup, the fingerprints).
hm_status check_offsets(const uint64_t* offsets, uint64_t n, cudaStream_t st) {
  Scratch sc{st};
  unsigned int* bad = nullptr;
  hm_status s;
  if ((s = sc.alloc(WS_BAD, &bad, 4)) != HM_OK) return s;
  HM_CUDA_TRY(cudaMemsetAsync(bad, 0, 4, st));
  const unsigned grid = unsigned(std::min<uint64_t>((n + 255) / 256, uint64_t(num_sms()) * 16));
  {
    LaunchScope ls_("k_check_offsets", st);
    k_check_offsets<<<std::max(grid, 1u), 256, 0, st>>>(offsets, n, bad);
  }
  HM_CUDA_TRY(cudaGetLastError());
  unsigned int hbad = 0;
  HM_CUDA_TRY(cudaMemcpyAsync(&hbad, bad, 4, cudaMemcpyDeviceToHost, st));
  HM_CUDA_TRY(cudaStreamSynchronize(st));
  if (hbad & 1u) {
    set_error("offsets are not non-decreasing");
    return HM_ERR_INVALID_ARG;
  }
  if (hbad & 2u) {
    set_error("a byte key is longer than 65535 bytes");
    return HM_ERR_TOO_LARGE;
  }
  return HM_OK;
}

// (the caller has validated the offsets with check_offsets)
hm_status build_bytes_core(const uint8_t* bytes, const uint64_t* offsets, const uint64_t* vals, uint64_t n,
                           uint64_t seed, uint32_t log2_bp, cudaStream_t st, BuildOut* out, uint32_t* t0_out,
                           uint64_t* r_out, SideJob* job, const uint64_t* off0_host) {
  Scratch sc{st};
  uint64_t* fp = nullptr;
  hm_status s;
  if ((s = sc.alloc(WS_FP, &fp, n * 8)) != HM_OK) return s;
  uint64_t off0 = off0_host ? *off0_host : 0;
  if (!off0_host) {
    HM_CUDA_TRY(cudaMemcpyAsync(&off0, offsets, 8, cudaMemcpyDeviceToHost, st));
    HM_CUDA_TRY(cudaStreamSynchronize(st));
  }
  const uint64_t smix = seed_mix(seed);
  for (uint32_t t0 = 0; t0 < kT0Cap; t0++) {
    const uint64_t r = derive(smix, 0, 0, t0).a1;
    launch_fingerprint(bytes, offsets, n, r, fp, st);
    HM_CUDA_TRY(cudaGetLastError());
    bool fpc = false;
    s = build_core<SrcBytes, KV32, SameBytes>(SrcBytes{fp, vals, offsets, off0}, SameBytes{bytes, off0}, n, n, 0, n,
                                               -1, seed, log2_bp, st, out, &fpc, job);
    if (s == HM_ERR_TOO_LARGE) {
      // a degenerate level-1 distribution within the space bound (a bucket of
      // more than 32 keys, an overflowing build partition): the flat rounds
      // take any bucket size and tell duplicates from fingerprint collisions
      set_error("");
      s = build_bytes_rounds(fp, vals, offsets, off0, bytes, n, seed, log2_bp >> 16, st, out, &fpc);
    }
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

// --------------------------------------------------- from_array, dedup
// The first occurrence of every key, through the build's own radix passes:
// {key, value, input index} records are partitioned by a level-1 hash (equal
// keys share a partition), and one CTA per partition keeps, in a shared-memory
// set keyed by the key, the lowest input index of every key; the records
// holding it go to the output.  A partition that overflows its buffer (heavy
// duplication) makes the caller fall back to the global set (dedup.cu).
constexpr int kDThreads = 512, kDTab = 4096;
__global__ void __launch_bounds__(kDThreads, 2) k_dedup_part(const KV32* __restrict__ pbuf,
                                                             const unsigned int* __restrict__ pcount, uint32_t cap,
                                                             uint64_t* __restrict__ okeys, uint64_t* __restrict__ ovals,
                                                             unsigned long long* __restrict__ cursor,
                                                             DevStatus* __restrict__ stt) {
  extern __shared__ __align__(16) uint8_t smem[];
  KV32* skv = reinterpret_cast<KV32*>(smem);
  uint32_t* tab = reinterpret_cast<uint32_t*>(smem + size_t(cap) * sizeof(KV32));  // local item index
  uint32_t* tmin = tab + kDTab;                                                    // lowest input index
  __shared__ uint32_t s_n;
  __shared__ unsigned long long s_base;
  const uint32_t p = blockIdx.x, tid = threadIdx.x;
  const uint32_t cnt_raw = pcount[p];
  if (cnt_raw > cap) {  // (records were lost: the global set decides)
    if (tid == 0) atomicOr(&stt->part_overflow, 1u);
    return;
  }
  const uint32_t cnt = cnt_raw;
  for (uint32_t i = tid; i < kDTab; i += kDThreads) {
    tab[i] = ~0u;
    tmin[i] = ~0u;
  }
  if (tid == 0) s_n = 0;
  for (uint32_t i = tid; i < cnt; i += kDThreads) skv[i] = pbuf[size_t(p) * cap + i];
  __syncthreads();
  for (uint32_t i = tid; i < cnt; i += kDThreads) {
    const uint64_t k = skv[i].key;
    uint32_t h = uint32_t(mix64(k ^ 0x5851F42D4C957F2Dull)) & (kDTab - 1);
    while (true) {
      const uint32_t cur = atomicCAS(&tab[h], ~0u, i);
      if (cur == ~0u || skv[cur].key == k) break;
      h = (h + 1) & (kDTab - 1);
    }
    atomicMin(&tmin[h], uint32_t(skv[i].ctx_off));
    skv[i].len = h;  // (the item's slot, for the survivor test)
  }
  __syncthreads();
  uint32_t rk[(8192 + kDThreads - 1) / kDThreads];
  uint32_t nloc = 0;
  for (uint32_t i = tid, j = 0; i < cnt; i += kDThreads, j++) {
    rk[j] = ~0u;
    if (tmin[skv[i].len] == uint32_t(skv[i].ctx_off)) {
      rk[j] = atomicAdd(&s_n, 1u);
      nloc++;
    }
  }
  __syncthreads();
  if (tid == 0) s_base = atomicAdd(cursor, (unsigned long long)s_n);
  __syncthreads();
  for (uint32_t i = tid, j = 0; i < cnt; i += kDThreads, j++)
    if (rk[j] != ~0u) {
      okeys[s_base + rk[j]] = skv[i].key;
      ovals[s_base + rk[j]] = skv[i].value;
    }
}

// The same for byte keys: the set is keyed by the fingerprint and confirmed
// by content (equal fingerprints with different bytes are different keys and
// take different slots); a first occurrence sets keep[input index] = 1.
__global__ void __launch_bounds__(kDThreads, 2) k_dedup_part_bytes(const KV32* __restrict__ pbuf,
                                                                   const unsigned int* __restrict__ pcount, uint32_t cap,
                                                                   const uint8_t* __restrict__ bytes, uint64_t off0,
                                                                   uint8_t* __restrict__ keep,
                                                                   DevStatus* __restrict__ stt) {
  extern __shared__ __align__(16) uint8_t smem[];
  KV32* skv = reinterpret_cast<KV32*>(smem);
  uint32_t* tab = reinterpret_cast<uint32_t*>(smem + size_t(cap) * sizeof(KV32));
  uint32_t* tmin = tab + kDTab;
  uint16_t* slotof = reinterpret_cast<uint16_t*>(tmin + kDTab);
  const uint32_t p = blockIdx.x, tid = threadIdx.x;
  const uint32_t cnt_raw = pcount[p];
  if (cnt_raw > cap) {
    if (tid == 0) atomicOr(&stt->part_overflow, 1u);
    return;
  }
  const uint32_t cnt = cnt_raw;
  for (uint32_t i = tid; i < kDTab; i += kDThreads) {
    tab[i] = ~0u;
    tmin[i] = ~0u;
  }
  for (uint32_t i = tid; i < cnt; i += kDThreads) skv[i] = pbuf[size_t(p) * cap + i];
  __syncthreads();
  for (uint32_t i = tid; i < cnt; i += kDThreads) {
    const KV32 e = skv[i];
    uint32_t h = uint32_t(mix64(e.key ^ 0x5851F42D4C957F2Dull)) & (kDTab - 1);
    while (true) {
      const uint32_t cur = atomicCAS(&tab[h], ~0u, i);
      if (cur == ~0u) break;
      const KV32 c = skv[cur];
      if (c.key == e.key && c.len == e.len &&
          bytes_equal(bytes + off0 + c.ctx_off, bytes + off0 + e.ctx_off, e.len))
        break;
      h = (h + 1) & (kDTab - 1);
    }
    atomicMin(&tmin[h], e.reserved);
    slotof[i] = uint16_t(h);
  }
  __syncthreads();
  for (uint32_t i = tid; i < cnt; i += kDThreads)
    if (tmin[slotof[i]] == skv[i].reserved) keep[skv[i].reserved] = 1;
}

hm_status dedup_partitioned_bytes(const uint8_t* bytes, const uint64_t* offs, const uint64_t* fp,
                                  const uint64_t* vals, uint64_t n, uint64_t off0, cudaStream_t st, uint8_t* keep) {
  const int sms = num_sms();
  uint32_t lg = 10;  // (32-byte records: partitions of ~1024 records, 2 CTAs per SM)
  while (lg > 6 && (n >> lg) < uint64_t(4 * sms)) lg--;
  const double m = double(uint64_t(1) << lg);
  const uint32_t cap = uint32_t(std::ceil((m + 8.0 * std::sqrt(m) + 64.0) / 32.0) * 32.0);
  const uint32_t np = uint32_t((n + (uint64_t(1) << lg) - 1) >> lg);
  if (np > (1u << 18) || cap * 4 > kDTab * 3) return HM_ERR_TOO_LARGE;
  BuildParams bp{};
  bp.smix = seed_mix(0x46524F4D41525241ull);
  bp.l1 = make_l1(bp.smix, 0, n);
  bp.nb = n;
  bp.n_in = n;
  bp.log2_bp = lg;
  bp.np = np;
  bp.cap = cap;
  Scratch sc{st};
  KV32 *pbuf = nullptr, *cbuf = nullptr;
  unsigned int *pcount = nullptr, *ccount = nullptr;
  DevStatus* dstat = nullptr;
  hm_status s;
  const int sbits = np <= 65536 ? 8 : 9;
  const uint32_t sdig = 1u << sbits, ncoarse = (np + sdig - 1) / sdig;
  const double mc = double(sdig) * m;
  const uint32_t ccap = uint32_t(mc + 8.0 * std::sqrt(mc + 1.0) + 1024.0);
  constexpr int kSTile = split_tile<KV32>();
  const uint32_t tpc = (ccap + kSTile - 1) / kSTile;
  if ((s = sc.alloc(WS_PBUF, &pbuf, size_t(np) * cap * sizeof(KV32))) != HM_OK) return s;
  if ((s = sc.alloc(WS_PCOUNT, &pcount, size_t(np) * 4)) != HM_OK) return s;
  if ((s = sc.alloc(WS_CBUF, &cbuf, size_t(ncoarse) * ccap * sizeof(KV32))) != HM_OK) return s;
  if ((s = sc.alloc(WS_CCOUNT, &ccount, size_t(ncoarse) * 4)) != HM_OK) return s;
  if ((s = sc.alloc(WS_DSTAT, &dstat, sizeof(DevStatus))) != HM_OK) return s;
  HM_CUDA_TRY(cudaMemsetAsync(pcount, 0, size_t(np) * 4, st));
  HM_CUDA_TRY(cudaMemsetAsync(ccount, 0, size_t(ncoarse) * 4, st));
  HM_CUDA_TRY(cudaMemsetAsync(dstat, 0, sizeof(DevStatus), st));
  uint64_t o0 = off0;
  const size_t smemS = size_t(kSTile) * (sizeof(KV32) + 4);
  auto kS1 = sbits == 8 ? k_split<SrcBytesIdx, KV32, 1, 8> : k_split<SrcBytesIdx, KV32, 1, 9>;
  auto kS2 = sbits == 8 ? k_split<SrcBytesIdx, KV32, 2, 8> : k_split<SrcBytesIdx, KV32, 2, 9>;
  HM_CUDA_TRY(cudaFuncSetAttribute(kS1, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smemS)));
  HM_CUDA_TRY(cudaFuncSetAttribute(kS2, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smemS)));
  const SrcBytesIdx src{fp, vals, offs, o0};
  const SplitArgs a1{nullptr, nullptr, 0, 0, cbuf, ccount, ccap, ncoarse, 0};
  {
    LaunchScope ls_("k_split1", st);
    kS1<<<unsigned((n + kSTile - 1) / kSTile), kSThreads, smemS, st>>>(src, bp, a1, dstat);
  }
  const SplitArgs a2{cbuf, ccount, ccap, tpc, pbuf, pcount, cap, np, ncoarse};
  {
    LaunchScope ls_("k_split2", st);
    kS2<<<ncoarse * tpc, kSThreads, smemS, st>>>(src, bp, a2, dstat);
  }
  const size_t smemD = size_t(cap) * sizeof(KV32) + size_t(kDTab) * 8 + size_t(cap) * 2;
  HM_CUDA_TRY(cudaFuncSetAttribute(k_dedup_part_bytes, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smemD)));
  {
    LaunchScope ls_("k_dedup_part", st);
    k_dedup_part_bytes<<<np, kDThreads, smemD, st>>>(pbuf, pcount, cap, bytes, o0, keep, dstat);
  }
  HM_CUDA_TRY(cudaGetLastError());
  DevStatus hs{};
  HM_CUDA_TRY(cudaMemcpyAsync(&hs, dstat, sizeof(hs), cudaMemcpyDeviceToHost, st));
  HM_CUDA_TRY(cudaStreamSynchronize(st));
  if (hs.part_overflow || hs.pad) return HM_ERR_TOO_LARGE;
  return HM_OK;
}

// Returns HM_OK with *n_out distinct keys in (okeys, ovals) (device arrays of n
// entries the caller owns), or HM_ERR_TOO_LARGE when a partition overflowed.
hm_status dedup_partitioned(const uint64_t* keys, const uint64_t* vals, uint64_t n, cudaStream_t st,
                            uint64_t* okeys, uint64_t* ovals, uint64_t* n_out) {
  const int sms = num_sms();
  // partitions of ~2048 records (cap 2496): 2 CTAs per SM for k_dedup_part
  uint32_t lg = 11;
  while (lg > 6 && (n >> lg) < uint64_t(4 * sms)) lg--;
  const double m = double(uint64_t(1) << lg);
  const uint32_t cap = uint32_t(std::ceil((m + 8.0 * std::sqrt(m) + 64.0) / 32.0) * 32.0);
  const uint32_t np = uint32_t((n + (uint64_t(1) << lg) - 1) >> lg);
  if (np > (1u << 18) || cap * 4 > kDTab * 3) return HM_ERR_TOO_LARGE;
  BuildParams bp{};
  bp.smix = seed_mix(0x46524F4D41525241ull);  // (any level-1 function groups equal keys)
  bp.l1 = make_l1(bp.smix, 0, n);
  bp.b_lo = 0;
  bp.nb = n;
  bp.n_in = n;
  bp.log2_bp = lg;
  bp.np = np;
  bp.cap = cap;
  Scratch sc{st};
  KV32 *pbuf = nullptr, *cbuf = nullptr;
  unsigned int *pcount = nullptr, *ccount = nullptr;
  DevStatus* dstat = nullptr;
  hm_status s;
  const int sbits = np <= 65536 ? 8 : 9;
  const uint32_t sdig = 1u << sbits, ncoarse = (np + sdig - 1) / sdig;
  const double mc = double(n) * double(sdig) * m / double(n);
  const uint32_t ccap = uint32_t(mc + 8.0 * std::sqrt(mc + 1.0) + 1024.0);
  constexpr int kSTile = split_tile<KV32>();
  const uint32_t tpc = (ccap + kSTile - 1) / kSTile;
  if ((s = sc.alloc(WS_PBUF, &pbuf, size_t(np) * cap * sizeof(KV32))) != HM_OK) return s;
  if ((s = sc.alloc(WS_PCOUNT, &pcount, size_t(np) * 4)) != HM_OK) return s;
  if ((s = sc.alloc(WS_CBUF, &cbuf, size_t(ncoarse) * ccap * sizeof(KV32))) != HM_OK) return s;
  if ((s = sc.alloc(WS_CCOUNT, &ccount, size_t(ncoarse) * 4)) != HM_OK) return s;
  if ((s = sc.alloc(WS_DSTAT, &dstat, sizeof(DevStatus))) != HM_OK) return s;
  unsigned long long* cur = reinterpret_cast<unsigned long long*>(&dstat->S);  // (S is unused here)
  HM_CUDA_TRY(cudaMemsetAsync(pcount, 0, size_t(np) * 4, st));
  HM_CUDA_TRY(cudaMemsetAsync(ccount, 0, size_t(ncoarse) * 4, st));
  HM_CUDA_TRY(cudaMemsetAsync(dstat, 0, sizeof(DevStatus), st));
  const size_t smemS = size_t(kSTile) * (sizeof(KV32) + 4);
  auto kS1 = sbits == 8 ? k_split<SrcU64Idx, KV32, 1, 8> : k_split<SrcU64Idx, KV32, 1, 9>;
  auto kS2 = sbits == 8 ? k_split<SrcU64Idx, KV32, 2, 8> : k_split<SrcU64Idx, KV32, 2, 9>;
  HM_CUDA_TRY(cudaFuncSetAttribute(kS1, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smemS)));
  HM_CUDA_TRY(cudaFuncSetAttribute(kS2, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smemS)));
  const SrcU64Idx src{keys, vals};
  const SplitArgs a1{nullptr, nullptr, 0, 0, cbuf, ccount, ccap, ncoarse, 0};
  {
    LaunchScope ls_("k_split1", st);
    kS1<<<unsigned((n + kSTile - 1) / kSTile), kSThreads, smemS, st>>>(src, bp, a1, dstat);
  }
  const SplitArgs a2{cbuf, ccount, ccap, tpc, pbuf, pcount, cap, np, ncoarse};
  {
    LaunchScope ls_("k_split2", st);
    kS2<<<ncoarse * tpc, kSThreads, smemS, st>>>(src, bp, a2, dstat);
  }
  const size_t smemD = size_t(cap) * sizeof(KV32) + size_t(kDTab) * 8;
  HM_CUDA_TRY(cudaFuncSetAttribute(k_dedup_part, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smemD)));
  {
    LaunchScope ls_("k_dedup_part", st);
    k_dedup_part<<<np, kDThreads, smemD, st>>>(pbuf, pcount, cap, okeys, ovals, cur, dstat);
  }
  HM_CUDA_TRY(cudaGetLastError());
  DevStatus hs{};
  HM_CUDA_TRY(cudaMemcpyAsync(&hs, dstat, sizeof(hs), cudaMemcpyDeviceToHost, st));
  HM_CUDA_TRY(cudaStreamSynchronize(st));
  if (hs.part_overflow || hs.pad) return HM_ERR_TOO_LARGE;
  *n_out = hs.S;
  return HM_OK;
}

}  // namespace hm
