// lookup.cu — batched lookups and multi-GPU routing kernels (sm_100a).
//
// lookup is the membership test of PAPER.md:244-245
// extended to a map: two dependent random probes (directory entry, slot) and a
// key compare.  Each thread keeps QPT independent queries in flight so that the
// chip has enough outstanding 32-byte sectors to cover DRAM latency (Little's
// law).
#include <algorithm>

#include "hm_internal.cuh"
#include "route.cuh"

namespace hm {

constexpr int kLThreads = 256;

__device__ __forceinline__ uint64_t ld_stream_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.global.nc.L1::no_allocate.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}
// Random probes bypass L1 (.cg): an L1 miss would be promoted to a full
// 128-byte line request, four times the one 32-byte sector a probe needs.
__device__ __forceinline__ uint64_t ld_dir(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ KV16 ld_slot16(const KV16* p) {
  KV16 e;
  asm volatile("ld.global.cg.v2.u64 {%0, %1}, [%2];" : "=l"(e.key), "=l"(e.value) : "l"(p));
  return e;
}
__device__ __forceinline__ KV32 ld_slot32(const KV32* p) {
  KV32 e;
  uint64_t w3;
  asm volatile("ld.global.cg.L2::64B.v4.u64 {%0, %1, %2, %3}, [%4];"
               : "=l"(e.key), "=l"(e.value), "=l"(e.ctx_off), "=l"(w3)
               : "l"(p));
  e.len = uint32_t(w3);
  e.reserved = uint32_t(w3 >> 32);
  return e;
}
__device__ __forceinline__ void st_stream_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.global.L1::no_allocate.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// level-2 range reduction mod s^2 (R22): reciprocal table for s <= 32
__device__ __forceinline__ uint64_t mod_s2(uint64_t h, uint32_t s, const uint64_t* s_m2) {
  const uint64_t d = uint64_t(s) * s;
  if (s <= 32) {
    const FastMod fm{d, s_m2[s]};
    return fastmod(h, fm);
  }
  return h % d;
}

// probe-2 slot index of key k in bucket b (global id) with directory entry d
#ifndef HM_SLOT_FLAT
#define HM_SLOT_FLAT 1  // lookups: the level-2 hash computed for every lane, the singleton case selected (no branch)
#endif
__device__ __forceinline__ uint64_t slot_index(uint64_t smix, uint64_t b, uint64_t d, uint64_t k,
                                               const uint64_t* s_m2) {
  const uint32_t s = uint32_t((d >> 40) & 0xFFFF);
  const uint64_t soff = d & kMask40;
#if HM_SLOT_FLAT
  // (a warp's queries mix singletons and multi-key buckets, so the level-2
  // hash costs the warp the same either way; without the branch the four
  // queries of a thread interleave)
  const Consts c = derive(smix, 2, b, uint32_t(d >> 56));
  const uint64_t hv = hash64(c, k);
  if (s > 32) return s <= 1 ? soff : soff + hv % (uint64_t(s) * s);  // (never for distinct keys; R22)
  const FastMod fm{uint64_t(s) * s, s_m2[s]};
  return s <= 1 ? soff : soff + fastmod(hv, fm);  // R12: a singleton's slot is soff
#else
  if (s <= 1) return soff;  // R12
  const Consts c = derive(smix, 2, b, uint32_t(d >> 56));
  return soff + mod_s2(hash64(c, k), s, s_m2);
#endif
}

// L2 cache policies: the compact directory should stay resident (evict_last);
// query streams, slot probes and outputs pass through (evict_first).
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t ld_q(const uint64_t* p, uint64_t pol) {
  uint64_t v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ CDir ld_cdir(const CDir* p, uint64_t pol) {
  CDir r;
  uint64_t a, b, c, d;
#ifndef HM_CDIR_PF
#define HM_CDIR_PF "128B"  // (neighbouring records are reused: 2^26 lookups 1.46 -> 1.41 ms vs 64B)
#endif
  asm volatile("ld.global.cg.L2::cache_hint.L2::" HM_CDIR_PF ".v4.u64 {%0, %1, %2, %3}, [%4], %5;"
               : "=l"(a), "=l"(b), "=l"(c), "=l"(d)
               : "l"(p), "l"(pol));
  r.w[0] = uint32_t(a);
  r.w[1] = uint32_t(a >> 32);
  r.w[2] = uint32_t(b);
  r.w[3] = uint32_t(b >> 32);
  r.w[4] = uint32_t(c);
  r.w[5] = uint32_t(c >> 32);
  r.w[6] = uint32_t(d);
  r.w[7] = uint32_t(d >> 32);
  return r;
}
__device__ __forceinline__ KV16 ld_slot16_ef(const KV16* p, uint64_t pol) {
  KV16 e;
  asm volatile("ld.global.cg.L2::cache_hint.L2::64B.v2.u64 {%0, %1}, [%2], %3;"
               : "=l"(e.key), "=l"(e.value)
               : "l"(p), "l"(pol));
  return e;
}
__device__ __forceinline__ void st_ef_u64(uint64_t* p, uint64_t v, uint64_t pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.u64 [%0], %1, %2;" ::"l"(p), "l"(v), "l"(pol) : "memory");
}

// Decode bucket lb from its compact-directory record into a full directory
// entry (soff | s<<40 | t<<56); escapes read the full directory (DRAM).
__device__ __forceinline__ uint64_t cdir_entry(const CDir& r, uint64_t lb, const uint64_t* dir, bool* escaped) {
  const uint32_t j = uint32_t(lb & 31), bit = 1u << j, below = bit - 1u;
  const uint32_t s = ((r.w[1] & bit) ? 4u : 0u) | ((r.w[2] & bit) ? 2u : 0u) | ((r.w[3] & bit) ? 1u : 0u);
  const uint32_t t = ((r.w[4] & bit) ? 1u : 0u) | ((r.w[5] & bit) ? 2u : 0u) | ((r.w[6] & bit) ? 4u : 0u) |
                     ((r.w[7] & bit) ? 8u : 0u);
  *escaped = s == kCdirEscS || (s >= 2 && t == kCdirEscT);  // (a singleton's t planes hold its tag)
  const uint64_t soff = uint64_t(r.w[0]) + cdir_prefix_sq(r.w[1] & below, r.w[2] & below, r.w[3] & below);
  return dir_entry(soff, s, t);
}

// u64 lookup: probe 1 reads the L2-resident compact directory, probe 2 the
// slot (the one DRAM line a query needs); 4 queries in flight per thread.
// POW2: the table's n is a power of two (level-one reduction by a mask, no
// per-query branch; every benchmark configuration)
template <int QPT, bool POW2>
__global__ void __launch_bounds__(kLThreads) k_lookup_u64(LookupParams lp, const uint64_t* __restrict__ q,
                                                          uint64_t nq, uint64_t* __restrict__ ov,
                                                          uint8_t* __restrict__ of) {
  __shared__ uint64_t s_m2[33];
  // (computed here: a global-memory table costs a dependent load at every CTA start, 1.32 -> 1.39 ms)
  if (threadIdx.x < 33) s_m2[threadIdx.x] = threadIdx.x ? ~0ull / (uint64_t(threadIdx.x) * threadIdx.x) : 0ull;
  __syncthreads();
  const uint64_t pol_keep = policy_evict_last(), pol_stream = policy_evict_first();
  const KV16* __restrict__ slots = reinterpret_cast<const KV16*>(lp.slots);
  const uint64_t per = uint64_t(kLThreads) * QPT;
  for (uint64_t base = blockIdx.x * per; base < nq; base += uint64_t(gridDim.x) * per) {
    uint64_t key[QPT], b[QPT], d[QPT];
    uint32_t tag[QPT];
    CDir rec[QPT];
#pragma unroll
    for (int j = 0; j < QPT; j++) {
      const uint64_t idx = base + uint64_t(j) * kLThreads + threadIdx.x;
      key[j] = idx < nq ? ld_q(q + idx, pol_stream) : 0ull;
    }
    // L1 + L2: g q and the (compact) directory probe
#pragma unroll
    for (int j = 0; j < QPT; j++) {
      const uint64_t idx = base + uint64_t(j) * kLThreads + threadIdx.x;
      const uint64_t h1 = hash64(lp.l1.c1, key[j]);
      b[j] = (POW2 ? (h1 & lp.l1.mask) : level1_of_hash(lp.l1, h1)) - lp.b_lo;
      tag[j] = tag4_of_hash(h1);
      const bool ok = idx < nq && b[j] < lp.nb;
      if (!ok) b[j] = 0;
      rec[j] = ld_cdir(lp.cdir + (b[j] >> 5), pol_keep);
      if (!ok) rec[j].w[1] = rec[j].w[2] = rec[j].w[3] = 0;  // s = 0: no probe
    }
#pragma unroll
    for (int j = 0; j < QPT; j++) {
      bool esc;
      d[j] = cdir_entry(rec[j], b[j], lp.dir, &esc);
      if (esc) d[j] = ld_dir(lp.dir + b[j]);
      // a singleton whose key tag differs: a miss without the slot probe
      else if (((d[j] >> 40) & 0xFFFF) == 1 && uint32_t(d[j] >> 56) != tag[j]) d[j] = 0;
    }
    // L3 + L4: slot index and the slot probe
    KV16 e[QPT];
#pragma unroll
    for (int j = 0; j < QPT; j++) {
      const bool live = ((d[j] >> 40) & 0xFFFF) != 0;
      e[j].key = ~key[j];
      e[j].value = 0;
      if (live) e[j] = ld_slot16_ef(slots + slot_index(lp.smix, b[j] + lp.b_lo, d[j], key[j], s_m2), pol_stream);
    }
#pragma unroll
    for (int j = 0; j < QPT; j++) {
      const uint64_t idx = base + uint64_t(j) * kLThreads + threadIdx.x;
      if (idx < nq) {
        const bool hit = e[j].key == key[j];
        if (ov) st_ef_u64(ov + idx, hit ? e[j].value : 0ull, pol_stream);
        if (of) of[idx] = hit ? 1 : 0;
      }
    }
  }
}

hm_status lookup_u64_launch(const hm_map* m, const uint64_t* q, uint64_t nq, uint64_t* out_vals,
                            uint8_t* out_found, cudaStream_t st) {
  if (nq == 0) return HM_OK;
  LookupParams lp{};
  lp.l1 = m->l1;
  lp.smix = m->smix;
  lp.b_lo = m->b_lo;
  lp.nb = m->nb;
  lp.dir = m->dir;
  lp.cdir = m->cdir;
  lp.slots = m->slots;
#ifndef HM_LOOKUP_QPT
#define HM_LOOKUP_QPT 4
#endif
  constexpr int QPT = HM_LOOKUP_QPT;
  const uint64_t per = uint64_t(kLThreads) * QPT;
  const uint64_t blocks = (nq + per - 1) / per;
#ifndef HM_LOOKUP_CPS
#define HM_LOOKUP_CPS 96  // grid: CTAs per SM, 3-4 resident at a time (the block scheduler balances the SMs: 8 -> 64 cut 2^26 lookups 1.42 -> 1.33 ms; 96: 2^28 on 2^27 -1 %)
#endif
  const unsigned grid = unsigned(std::min<uint64_t>(blocks, uint64_t(num_sms()) * HM_LOOKUP_CPS));
  {
    LaunchScope ls_("k_lookup_u64", st);
#ifndef HM_LOOKUP_POW2
#define HM_LOOKUP_POW2 1
#endif
    if (HM_LOOKUP_POW2 && lp.l1.pow2) k_lookup_u64<QPT, true><<<grid, kLThreads, 0, st>>>(lp, q, nq, out_vals, out_found);
    else k_lookup_u64<QPT, false><<<grid, kLThreads, 0, st>>>(lp, q, nq, out_vals, out_found);
  }
  HM_CUDA_TRY(cudaGetLastError());
  return HM_OK;
}

// ------------------------------------------------------------ byte keys

// Byte-key lookup: fingerprint the needle (R5,
// expanded form), probe the compact directory and the 32-byte slot, and on a
// fingerprint + length match compare the bytes with the map's context copy.
#ifndef HM_LOOKUP_BYTES_QPT
#define HM_LOOKUP_BYTES_QPT 1
#endif

// A key of at most 64 bytes as eight little-endian 8-byte chunks (zero past
// the key), from the at most nine aligned words it touches: every load is
// issued before the first is used (one memory round trip per key, where a
// chunk-at-a-time loop pays one per chunk).
constexpr uint32_t kRegKey = 64;
__device__ __forceinline__ void key_chunks(const uint8_t* p, uint32_t len, uint64_t (&c)[8]) {
  const uintptr_t A = reinterpret_cast<uintptr_t>(p);
  const unsigned long long* w = reinterpret_cast<const unsigned long long*>(A & ~uintptr_t(7));
  const uint32_t sh = uint32_t(A & 7) * 8, nw = len ? (uint32_t(A & 7) + len + 7) >> 3 : 0u;
  uint64_t u[9];
#pragma unroll
  for (int i = 0; i < 9; i++) u[i] = uint32_t(i) < nw ? __ldg(w + i) : 0ull;
#pragma unroll
  for (int i = 0; i < 8; i++) {
    uint64_t x = sh ? (u[i] >> sh) | (u[i + 1] << (64 - sh)) : u[i];
    const int rem = int(len) - 8 * i;
    if (rem < 8) x = rem <= 0 ? 0ull : x & ((1ull << (8 * rem)) - 1ull);
    c[i] = x;
  }
}
// fingerprint_pw64 of a key held as chunks (len <= 64): chunk i carries words
// 2i and 2i+1, weighted r^(nw-2i) and r^(nw-2i-1).  Branch-free: chunks past
// the key are 0 and their exponents (down to -15) read the table's zero pad;
// len = 0 gives 0 as fingerprint_pw64 does.
__device__ __forceinline__ uint64_t fingerprint_chunks(const uint64_t (&c)[8], uint32_t len, const FpPow* pw) {
  // P[-k] = r^(nw-k), 0 below r^0 (the pad: FpPow is one array of uint4)
  const uint4* P = reinterpret_cast<const uint4*>(pw) + kFpPowPad + ((len + 3) >> 2);
  uint64_t a0 = 0, a1 = 0, a2 = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) {
    fp3_acc(a0, a1, a2, uint32_t(c[i]), P[-2 * i]);
    fp3_acc(a0, a1, a2, uint32_t(c[i] >> 32), P[-2 * i - 1]);
  }
  return fp3_finish(a0, a1, a2, len);
}
#ifndef HM_LB_MINB
#define HM_LB_MINB 4  // (64 registers; 1 / 3: 1.01 / 1.00 ms vs 0.87 at C3, 5: spills)
#endif
template <int QPT, bool POW2>
__global__ void __launch_bounds__(kLThreads, HM_LB_MINB) k_lookup_bytes(LookupParams lp, const uint8_t* __restrict__ qb,
                                                            const uint64_t* __restrict__ qo, uint64_t nq,
                                                            uint64_t* __restrict__ ov, uint8_t* __restrict__ of) {
  __shared__ uint64_t s_m2[33];
  __shared__ FpPow s_pw;
  // (computed here: a global-memory table costs a dependent load at every CTA start, 1.32 -> 1.39 ms)
  if (threadIdx.x < 33) s_m2[threadIdx.x] = threadIdx.x ? ~0ull / (uint64_t(threadIdx.x) * threadIdx.x) : 0ull;
  if (threadIdx.x == 64) fp_pow_fill(&s_pw, lp.r_fp);
  __syncthreads();
  const uint64_t pol_keep = policy_evict_last();
  const KV32* __restrict__ slots = reinterpret_cast<const KV32*>(lp.slots);
  const uint64_t per = uint64_t(kLThreads) * QPT;
  for (uint64_t base = blockIdx.x * per; base < nq; base += uint64_t(gridDim.x) * per) {
    uint64_t fp[QPT], b[QPT], d[QPT], off[QPT], len[QPT];
    uint64_t kc[QPT][8];  // (keys <= kRegKey bytes: the needle's chunks, kept for the comparison)
    CDir rec[QPT];
#pragma unroll
    for (int j = 0; j < QPT; j++) {
      const uint64_t idx = base + uint64_t(j) * kLThreads + threadIdx.x;
      off[j] = 0;
      len[j] = 0;
      fp[j] = 0;
      if (idx < nq) {
        off[j] = qo[idx];
        len[j] = qo[idx + 1] - off[j];
      }
      key_chunks(qb + off[j], len[j] <= kRegKey ? uint32_t(len[j]) : 0u, kc[j]);
      if (idx < nq)
        fp[j] = len[j] <= kRegKey ? fingerprint_chunks(kc[j], uint32_t(len[j]), &s_pw)
                                  : fingerprint_pw64(qb, off[j], len[j], lp.r_fp, &s_pw);
    }
    uint32_t tag[QPT];
#pragma unroll
    for (int j = 0; j < QPT; j++) {
      const uint64_t idx = base + uint64_t(j) * kLThreads + threadIdx.x;
      const uint64_t h1 = hash64(lp.l1.c1, fp[j]);
      b[j] = (POW2 ? (h1 & lp.l1.mask) : level1_of_hash(lp.l1, h1)) - lp.b_lo;
      tag[j] = tag4_of_hash(h1);
      const bool ok = idx < nq && b[j] < lp.nb;
      if (!ok) b[j] = 0;
      rec[j] = ld_cdir(lp.cdir + (b[j] >> 5), pol_keep);
      if (!ok) rec[j].w[1] = rec[j].w[2] = rec[j].w[3] = 0;
    }
#pragma unroll
    for (int j = 0; j < QPT; j++) {
      bool esc;
      d[j] = cdir_entry(rec[j], b[j], lp.dir, &esc);
      if (esc) d[j] = ld_dir(lp.dir + b[j]);
      // a singleton whose key tag differs: a miss without the slot probe
      else if (((d[j] >> 40) & 0xFFFF) == 1 && uint32_t(d[j] >> 56) != tag[j]) d[j] = 0;
    }
    // all slot probes in flight before the first comparison
    KV32 e[QPT];
#pragma unroll
    for (int j = 0; j < QPT; j++) {
      e[j].key = ~fp[j];  // (no probe: never equal)
      e[j].len = 0;
      if (((d[j] >> 40) & 0xFFFF) != 0) e[j] = ld_slot32(slots + slot_index(lp.smix, b[j] + lp.b_lo, d[j], fp[j], s_m2));
    }
#pragma unroll
    for (int j = 0; j < QPT; j++) {
      const uint64_t idx = base + uint64_t(j) * kLThreads + threadIdx.x;
      if (idx >= nq) continue;
      bool hit = false;
      uint64_t v = 0;
      if (e[j].key == fp[j] && e[j].len == len[j]) {
        if (len[j] <= kRegKey) {
          uint64_t mc[8];
          key_chunks(lp.ctx + e[j].ctx_off, e[j].len, mc);
          uint64_t diff = 0;
#pragma unroll
          for (int i = 0; i < 8; i++) diff |= mc[i] ^ kc[j][i];
          hit = diff == 0;
        } else {
          hit = bytes_equal64(lp.ctx + e[j].ctx_off, qb + off[j], e[j].len);
        }
        if (hit) v = e[j].value;
      }
      if (ov) ov[idx] = v;
      if (of) of[idx] = hit ? 1 : 0;
    }
  }
}

hm_status lookup_bytes_launch(const hm_map* m, const uint8_t* qb, const uint64_t* qo, uint64_t nq,
                              uint64_t* out_vals, uint8_t* out_found, cudaStream_t st) {
  if (nq == 0) return HM_OK;
  LookupParams lp{};
  lp.l1 = m->l1;
  lp.smix = m->smix;
  lp.b_lo = m->b_lo;
  lp.nb = m->nb;
  lp.dir = m->dir;
  lp.cdir = m->cdir;
  lp.slots = m->slots;
  lp.ctx = m->ctx;
  lp.r_fp = m->r_fp;
  const uint64_t blocks = (nq + kLThreads * HM_LOOKUP_BYTES_QPT - 1) / (kLThreads * HM_LOOKUP_BYTES_QPT);
#ifndef HM_LOOKUP_BYTES_CPS
#define HM_LOOKUP_BYTES_CPS 8  // grid: CTAs per SM (grid-stride)
#endif
  const unsigned grid = unsigned(std::min<uint64_t>(blocks, uint64_t(num_sms()) * HM_LOOKUP_BYTES_CPS));
  {
    LaunchScope ls_("k_lookup_bytes", st);
    if (HM_LOOKUP_POW2 && lp.l1.pow2)
      k_lookup_bytes<HM_LOOKUP_BYTES_QPT, true><<<grid, kLThreads, 0, st>>>(lp, qb, qo, nq, out_vals, out_found);
    else
      k_lookup_bytes<HM_LOOKUP_BYTES_QPT, false><<<grid, kLThreads, 0, st>>>(lp, qb, qo, nq, out_vals, out_found);
  }
  HM_CUDA_TRY(cudaGetLastError());
  return HM_OK;
}

// ------------------------------------------------------- multi-GPU routing

__global__ void __launch_bounds__(512) k_route_count(const uint64_t* __restrict__ keys, uint64_t n, L1Params l1,
                                                     int world, unsigned long long* __restrict__ counts) {
  __shared__ unsigned int s_c[64];
  if (threadIdx.x < 64) s_c[threadIdx.x] = 0;
  __syncthreads();
  constexpr int U = 8;  // keys in flight per thread
  for (uint64_t b0 = uint64_t(blockIdx.x) * blockDim.x * U; b0 < n; b0 += uint64_t(gridDim.x) * blockDim.x * U) {
    uint64_t k[U];
#pragma unroll
    for (int j = 0; j < U; j++) {
      const uint64_t i = b0 + uint64_t(j) * blockDim.x + threadIdx.x;
      k[j] = i < n ? __ldg(keys + i) : 0ull;
    }
#pragma unroll
    for (int j = 0; j < U; j++) {
      const uint64_t i = b0 + uint64_t(j) * blockDim.x + threadIdx.x;
      if (i < n) atomicAdd(&s_c[owner_of(level1_bucket(l1, k[j]), l1.n, world)], 1u);
    }
  }
  __syncthreads();
  if (threadIdx.x < world && s_c[threadIdx.x]) atomicAdd(&counts[threadIdx.x], (unsigned long long)s_c[threadIdx.x]);
}

__global__ void k_route_prefix(const unsigned long long* counts, int world, unsigned long long* cursors) {
  if (threadIdx.x == 0) {
    unsigned long long acc = 0;
    for (int r = 0; r < world; r++) {
      cursors[r] = acc;
      acc += counts[r];
    }
  }
}

struct OutLocal {  // this rank's send buffers, grouped by destination
  uint64_t* sk;
  uint64_t* sv;
  __device__ __forceinline__ uint64_t* keys(uint32_t) const { return sk; }
  __device__ __forceinline__ uint64_t* vals(uint32_t) const { return sv; }
};
__global__ void __launch_bounds__(kRThreads) k_route_scatter(const uint64_t* __restrict__ keys,
                                                             const uint64_t* __restrict__ vals, uint64_t n, L1Params l1,
                                                             int world, unsigned long long* __restrict__ cursors,
                                                             uint64_t* __restrict__ sk, uint64_t* __restrict__ sv,
                                                             uint64_t* __restrict__ perm) {
  route_scatter(keys, sv ? vals : nullptr, n, l1, world, cursors, OutLocal{sk, sv}, perm);
}

static hm_status route_common(const uint64_t* keys, const uint64_t* vals, uint64_t n, const L1Params& l1, int world,
                              uint64_t* sk, uint64_t* sv, uint64_t* perm, uint64_t* counts, cudaStream_t st) {
  if (world < 1 || world > 64) return HM_ERR_INVALID_ARG;
  unsigned long long* cur = nullptr;
  HM_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&cur), 64 * 8, st));
  cudaError_t e = cudaMemsetAsync(counts, 0, size_t(world) * 8, st);
  const unsigned grid = unsigned(std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, uint64_t(num_sms()) * 8)));
  if (e == cudaSuccess && n) {
    {
      LaunchScope ls_("k_route_count", st);
      const unsigned gc = unsigned(std::max<uint64_t>(1, std::min<uint64_t>((n + 4095) / 4096, uint64_t(num_sms()) * 4)));
      k_route_count<<<gc, 512, 0, st>>>(keys, n, l1, world, reinterpret_cast<unsigned long long*>(counts));
    }
    {
      LaunchScope ls_("k_route_prefix", st);
      k_route_prefix<<<1, 32, 0, st>>>(reinterpret_cast<unsigned long long*>(counts), world, cur);
    }
    {
      LaunchScope ls_("k_route_scatter", st);
      const unsigned gs = unsigned(std::max<uint64_t>(1, std::min<uint64_t>((n + kRTile - 1) / kRTile, uint64_t(num_sms()) * 2)));
      k_route_scatter<<<gs, kRThreads, 0, st>>>(keys, vals, n, l1, world, cur, sk, sv, perm);
    }
    e = cudaGetLastError();
  }
  cudaFreeAsync(cur, st);
  if (e != cudaSuccess) return cuda_fail(e, "route");
  return HM_OK;
}

// counts[d] = keys of this rank owned by rank d (device u64[world], zeroed here)
hm_status route_count_launch(const uint64_t* keys, uint64_t n, const L1Params& l1, int world, uint64_t* counts,
                             cudaStream_t st) {
  if (world < 1 || world > 64) return HM_ERR_INVALID_ARG;
  HM_CUDA_TRY(cudaMemsetAsync(counts, 0, size_t(world) * 8, st));
  if (n) {
    LaunchScope ls_("k_route_count", st);
    const unsigned gc = unsigned(std::max<uint64_t>(1, std::min<uint64_t>((n + 4095) / 4096, uint64_t(num_sms()) * 4)));
    k_route_count<<<gc, 512, 0, st>>>(keys, n, l1, world, reinterpret_cast<unsigned long long*>(counts));
  }
  HM_CUDA_TRY(cudaGetLastError());
  return HM_OK;
}

hm_status route_u64_launch(const uint64_t* keys, const uint64_t* vals, uint64_t n, const L1Params& l1, int world,
                           uint64_t* sk, uint64_t* sv, uint64_t* counts, cudaStream_t st) {
  return route_common(keys, vals, n, l1, world, sk, sv, nullptr, counts, st);
}

hm_status route_queries_launch(const L1Params& l1, const uint64_t* q, uint64_t nq, int world, uint64_t* sq,
                               uint64_t* perm, uint64_t* counts, cudaStream_t st) {
  return route_common(q, nullptr, nq, l1, world, sq, nullptr, perm, counts, st);
}

__global__ void k_unroute(const uint64_t* __restrict__ vr, const uint8_t* __restrict__ fr,
                          const uint64_t* __restrict__ perm, uint64_t nq, uint64_t* __restrict__ ov,
                          uint8_t* __restrict__ of) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < nq; i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t p = perm[i];
    if (ov) ov[i] = vr[p];
    if (of) of[i] = fr[p];
  }
}

hm_status unroute_launch(const uint64_t* vr, const uint8_t* fr, const uint64_t* perm, uint64_t nq, uint64_t* ov,
                         uint8_t* of, cudaStream_t st) {
  if (!nq) return HM_OK;
  const unsigned grid = unsigned(std::min<uint64_t>((nq + 255) / 256, uint64_t(num_sms()) * 8));
  {
    LaunchScope ls_("k_unroute", st);
    k_unroute<<<grid, 256, 0, st>>>(vr, fr, perm, nq, ov, of);
  }
  HM_CUDA_TRY(cudaGetLastError());
  return HM_OK;
}

}  // namespace hm
