// hm_math.cuh — device arithmetic of the FKS hot path (sm_100a).
//
//  * constant schedule  `random` made deterministic as
//    the counter schedule of DESIGN.md R6;
//  * the universal family `hash` of DESIGN.md R4:
//    hash((a1,a2,b), x) = (a1*(x mod 2^32) + a2*(x >> 32) + b) mod (2^61-1);
//  * exact range reduction `mod n` / `mod s^2` (R22) with a
//    precomputed reciprocal instead of the 64-bit division subroutine;
//  * the 61-bit polynomial fingerprint of byte keys (R5).
//
// Everything is integer arithmetic; 64x64->128 products use __umul64hi, and
// the Mersenne modulus is reduced with shifts and masks (no division).
#pragma once
#include <cstdint>

namespace hm {

constexpr uint64_t kP = (1ull << 61) - 1;          // Mersenne prime (R4)
constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ull;  // splitmix64 increment (R6)
constexpr uint64_t kSeedSalt = 0xD6E8FEB86659FD93ull;
constexpr uint32_t kT1Cap = 16, kT2Cap = 256, kT0Cap = 16;
constexpr uint64_t kMask40 = (1ull << 40) - 1;

struct Consts {  // (a1, a2, b)
  uint64_t a1, a2, b;
};

// z * c mod 2^64.  On the device as three 32-bit multiply-adds (the low
// product widened, both cross terms added into its high word) where nvcc emits
// four; on the host the plain product.
__host__ __device__ __forceinline__ uint64_t mul64_lo(uint64_t z, uint64_t c) {
#if defined(__CUDA_ARCH__) && !defined(HM_PLAIN_MUL)
  uint64_t r;
  asm("{ .reg .u32 wl, wh; .reg .u64 w;\n\t"
      "mul.wide.u32 w, %1, %3;\n\t"
      "mov.b64 {wl, wh}, w;\n\t"
      "mad.lo.u32 wh, %2, %3, wh;\n\t"
      "mad.lo.u32 wh, %1, %4, wh;\n\t"
      "mov.b64 %0, {wl, wh}; }"
      : "=l"(r)
      : "r"(uint32_t(z)), "r"(uint32_t(z >> 32)), "r"(uint32_t(c)), "r"(uint32_t(c >> 32)));
  return r;
#else
  return z * c;
#endif
}

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = mul64_lo(z ^ (z >> 30), 0xBF58476D1CE4E5B9ull);
  z = mul64_lo(z ^ (z >> 27), 0x94D049BB133111EBull);
  return z ^ (z >> 31);
}

__host__ __device__ __forceinline__ uint64_t field_of(uint64_t z) {
  uint64_t v = z >> 3;
  return v == kP ? 0 : v;
}

// seed_mix = mix64(seed ^ kSeedSalt) is hoisted per table (one per build).
__host__ __device__ __forceinline__ uint64_t seed_mix(uint64_t seed) { return mix64(seed ^ kSeedSalt); }

// derive(seed, level, bucket, attempt) -> (a1, a2, b)   (R6)
__host__ __device__ __forceinline__ Consts derive(uint64_t smix, uint32_t level, uint64_t bucket,
                                                  uint32_t attempt) {
  const uint64_t ctr = (uint64_t(level) << 60) | (bucket << 8) | uint64_t(attempt);
  const uint64_t u = mix64(smix ^ ctr);
  Consts c;
  c.a1 = field_of(mix64(u + kGamma));
  c.a2 = field_of(mix64(u + 2 * kGamma));
  c.b = field_of(mix64(u + 3 * kGamma));
  if (c.a1 == 0) c.a1 = 1;
  if (c.a2 == 0) c.a2 = 1;
  return c;
}

__host__ __device__ __forceinline__ uint64_t umulhi(uint64_t a, uint64_t b) {
#if defined(__CUDA_ARCH__)
  return __umul64hi(a, b);
#else
  return (uint64_t)(((unsigned __int128)a * b) >> 64);
#endif
}

// Reduce the 128-bit value hi*2^64 + lo (hi < 2^40) modulo P = 2^61-1,
// using 2^61 == 1 (mod P), hence 2^64 == 8.
__host__ __device__ __forceinline__ uint64_t mod_p128(uint64_t hi, uint64_t lo) {
  uint64_t x = (lo & kP) + (lo >> 61) + (hi << 3);
  x = (x & kP) + (x >> 61);
  return x >= kP ? x - kP : x;
}

// The universal family (R4):  (a1*xl + a2*xh + b) mod P with xl, xh the 32-bit
// limbs of x and a1, a2, b < P.  Computed on 32-bit pieces of the constants:
//   a*x = al*x + (ah*x)*2^32  (al < 2^32, ah < 2^29),
// with (ah1*xl + ah2*xh) = R < 2^62 folded as R*2^32 = (R >> 29) + (R mod 2^29)*2^32
// (mod P, since 2^61 = 1), and the two 64-bit products al*x folded to < 2^61+8
// before the sum, so every intermediate fits in 64 bits.
__host__ __device__ __forceinline__ uint64_t hash64(const Consts& c, uint64_t x) {
  const uint32_t xl = uint32_t(x), xh = uint32_t(x >> 32);
  const uint64_t p = uint64_t(uint32_t(c.a1)) * xl;          // < 2^64
  const uint64_t q = uint64_t(uint32_t(c.a2)) * xh;          // < 2^64
  const uint64_t r = uint64_t(uint32_t(c.a1 >> 32)) * xl + uint64_t(uint32_t(c.a2 >> 32)) * xh;  // < 2^62
  const uint64_t fp_ = (p & kP) + (p >> 61);
  const uint64_t fq = (q & kP) + (q >> 61);
  const uint64_t fr = (r >> 29) + ((r & ((1ull << 29) - 1)) << 32);
  uint64_t s = fp_ + fq + fr + c.b;                          // < 4*2^61 + 16
  s = (s & kP) + (s >> 61);
  return s >= kP ? s - kP : s;
}

// (a*b) mod P for a, b < 2^62.
__host__ __device__ __forceinline__ uint64_t mulmod_p(uint64_t a, uint64_t b) {
  const uint64_t lo = a * b, hi = umulhi(a, b);
  // value = hi*2^64 + lo < 2^124: fold the top: hi*2^64 = hi*8 (mod P), hi < 2^60
  uint64_t x = (lo & kP) + (lo >> 61);
  // hi*8 may be up to 2^63: fold it separately
  uint64_t h8 = hi << 3;                 // < 2^63
  uint64_t y = (h8 & kP) + (h8 >> 61);   // < 2^61 + 4
  x += y;                                // < 2^62 + small
  x = (x & kP) + (x >> 61);
  return x >= kP ? x - kP : x;
}

// Exact x mod d for x < 2^62 and 1 <= d < 2^32, with m = floor((2^64-1)/d):
// q = umulhi(x, m) underestimates floor(x/d) by at most 1 (x/2^64 < 1/4), so
// one correction gives the exact remainder (R22).
struct FastMod {
  uint64_t d, m;
};
__host__ __device__ __forceinline__ FastMod make_fastmod(uint64_t d) {
  FastMod f;
  f.d = d;
  f.m = ~0ull / d;
  return f;
}
__host__ __device__ __forceinline__ uint64_t fastmod(uint64_t x, const FastMod& f) {
  // x < 2^62: x*m/2^64 >= x/d - 2x/2^64 > x/d - 1/2, so q >= floor(x/d) - 1
  // and a single correction suffices
  const uint64_t q = umulhi(x, f.m);
  const uint64_t r = x - q * f.d;
  return r >= f.d ? r - f.d : r;
}

// floor((2^64 - 1) / s^2) for s = 1..32 (index 0 unused): the reciprocals of
// the level-2 moduli (R22), a compile-time table in global memory, so that a
// kernel copies it into shared memory with one coalesced load instead of 33
// 64-bit divisions (or constant-bank loads at 33 distinct addresses).
struct M2Table {
  uint64_t v[33];
};
__host__ __device__ constexpr M2Table make_m2_table() {
  M2Table t{};
  for (int i = 1; i <= 32; i++) t.v[i] = ~0ull / (uint64_t(i) * uint64_t(i));
  return t;
}
#if defined(__CUDACC__)
static __device__ const M2Table g_m2 = make_m2_table();
#endif

// Level-one range reduction `mod n`: mask when n is a power of
// two (all benchmark configs), reciprocal otherwise.
struct L1Params {
  Consts c1;
  uint64_t n;       // level-1 modulus (global key count)
  uint64_t mmagic;  // ~0 / n
  uint64_t mask;    // n-1 when n is a power of two, else 0
  int pow2;
};
__host__ __device__ __forceinline__ uint64_t level1_of_hash(const L1Params& p, uint64_t h) {
  if (p.pow2) return h & p.mask;
  FastMod f{p.n, p.mmagic};
  return fastmod(h, f);
}
__host__ __device__ __forceinline__ uint64_t level1_bucket(const L1Params& p, uint64_t key) {
  return level1_of_hash(p, hash64(p.c1, key));
}
// A 4-bit filter tag of a key from the top bits of its level-1 hash value
// (bits 57..60; the bucket uses the low bits, n <= 2^30).  Not part of the
// table contract: only the compact lookup directory stores it (§6.2).
__host__ __device__ __forceinline__ uint32_t tag4_of_hash(uint64_t h) { return uint32_t(h >> 57) & 15u; }

// Directory entry: soff | s<<40 | t<<56.
__host__ __device__ __forceinline__ uint64_t dir_entry(uint64_t soff, uint64_t s, uint64_t t) {
  return soff | (s << 40) | (t << 56);
}

// Compact lookup directory: one 32-byte record per 32
// consecutive buckets, small enough (1 B/bucket) to stay resident in L2 so
// that probe 1 of a lookup does not touch DRAM:
//   w[0] = soff of the record's first bucket (u32)
//   w[1..3] = bit-planes of s (bit 2, bit 1, bit 0): bit j = that bit of s_j
//   w[4..7] = bit-planes of t (bit 0..3)
// s_j = 7 or t_j = 15 means "read the full directory entry"; a record with any
// s >= 7 or t >= 15 (s >= 2) stores all-ones s planes (every bucket escapes).
// A singleton bucket has t = 0 (R12), so its t planes hold instead the 4-bit
// tag of its key (tag4_of_hash): a lookup whose tag differs is a miss without
// the slot probe (no false negatives; cuts ~15/16 of the DRAM probes of absent
// keys that land on singletons).
// soff_j = w[0] + sum_{i<j} s_i^2, where with s = 4a+2b+c (bits):
//   s^2 = 16a + 4b + c + 16ab + 8ac + 4bc  -> six popcounts over masked planes.
struct CDir {
  uint32_t w[8];
};
constexpr uint32_t kCdirEscS = 7, kCdirEscT = 15;

__host__ __device__ __forceinline__ uint32_t cdir_prefix_sq(uint32_t a, uint32_t b, uint32_t c) {
#if defined(__CUDA_ARCH__)
  return 16u * __popc(a) + 4u * __popc(b) + __popc(c) + 16u * __popc(a & b) + 8u * __popc(a & c) +
         4u * __popc(b & c);
#else
  return 16u * __builtin_popcount(a) + 4u * __builtin_popcount(b) + __builtin_popcount(c) +
         16u * __builtin_popcount(a & b) + 8u * __builtin_popcount(a & c) + 4u * __builtin_popcount(b & c);
#endif
}

#if defined(__CUDACC__)
// Fingerprint (R5): acc = (acc + w_i) * r mod P over little-endian u32 words
// (zero padded), fp = acc + len mod P.  Thread per key; the words are
// assembled from 4-byte aligned loads with a funnel shift.
__device__ __forceinline__ uint32_t ld_u32(const uint8_t* p) { return __ldg(reinterpret_cast<const uint32_t*>(p)); }

__device__ __forceinline__ uint64_t fingerprint_dev(const uint8_t* bytes, uint64_t off, uint64_t len, uint64_t r) {
  uint64_t acc = 0;
  if (len == 0) return 0;
  const uint64_t abase = off & ~uint64_t(3);
  const uint32_t sh = uint32_t(off & 3) * 8;
  const uint64_t last_aligned = (off + len - 1) & ~uint64_t(3);
  const uint64_t nw = (len + 3) >> 2;
  uint32_t cur = ld_u32(bytes + abase);
  for (uint64_t i = 0; i < nw; i++) {
    const uint64_t na = abase + 4 * (i + 1);
    const uint32_t nxt = na <= last_aligned ? ld_u32(bytes + na) : 0u;
    uint32_t w = sh ? __funnelshift_r(cur, nxt, sh) : cur;
    const uint64_t rem = len - 4 * i;
    if (rem < 4) w &= (1u << (8 * rem)) - 1u;
    acc = mulmod_p(acc + w, r);
    cur = nxt;
  }
  uint64_t f = acc + len;
  f = (f & kP) + (f >> 61);
  return f >= kP ? f - kP : f;
}

// The same fingerprint in expanded form.  Unrolling the Horner recurrence
// acc_{i+1} = (acc_i + w_i) * r gives, exactly (mod P),
//   acc_nw = sum_{i < nw} w_i * r^(nw - i),
// so with the powers r^1 .. r^kFpPowMax tabulated once per block the words are
// independent.  Each power is split into 21-bit limbs, r^e = l0 + l1*2^21 +
// l2*2^42 (l2 < 2^19), and each limb product w*l (< 2^53) is accumulated in
// its own 64-bit sum with no reduction: a word costs three multiply-adds, and
// 32 words keep every sum below 2^58.  fp3_finish folds the three sums once.
// Keys longer than 4*kFpPowMax bytes take the Horner loop above.
constexpr int kFpPowMax = 32, kFpPowPad = 16;
struct FpPow {
  uint4 z[kFpPowPad];      // zeros: exponents down to -16 read as 0 (chunks past a key, lookup.cu)
  uint4 p[kFpPowMax + 1];  // {l0, l1, l2, 0} of r^e
};
// One thread of the block fills the table; the caller synchronises.
__device__ inline void fp_pow_fill(FpPow* pw, uint64_t r) {
  for (int e = 0; e < kFpPowPad; e++) pw->z[e] = make_uint4(0u, 0u, 0u, 0u);
  uint64_t p = 1;
  for (int e = 0; e <= kFpPowMax; e++) {
    pw->p[e] = make_uint4(uint32_t(p & 0x1FFFFF), uint32_t((p >> 21) & 0x1FFFFF), uint32_t(p >> 42), 0u);
    p = mulmod_p(p, r);
  }
}

// (a0 + a1*2^21 + a2*2^42 + len) mod P for a0, a1 < 2^58, a2 < 2^56, using
// 2^61 == 1: a1*2^21 == (a1 >> 40) + (a1 mod 2^40)*2^21 and a2*2^42 ==
// (a2 >> 19) + (a2 mod 2^19)*2^42; the sum stays below 2^63.
__device__ __forceinline__ uint64_t fp3_finish(uint64_t a0, uint64_t a1, uint64_t a2, uint32_t len) {
  uint64_t f = a0 + (a1 >> 40) + ((a1 & 0xFFFFFFFFFFull) << 21) + (a2 >> 19) + ((a2 & 0x7FFFFull) << 42) + len;
  f = (f & kP) + (f >> 61);
  return f >= kP ? f - kP : f;
}

__device__ __forceinline__ void fp3_acc(uint64_t& a0, uint64_t& a1, uint64_t& a2, uint32_t w, const uint4& p) {
  a0 += uint64_t(w) * p.x;
  a1 += uint64_t(w) * p.y;
  a2 += uint64_t(w) * p.z;
}

// Byte equality of two keys of length len at arbitrary alignments: 4-byte
// aligned loads on both sides, realigned with a funnel shift (the word holding
// a key's last byte is the last one read, so nothing past the key is touched).
__device__ __forceinline__ bool bytes_equal(const uint8_t* a, const uint8_t* b, uint32_t len) {
  if (len == 0) return true;
  const uintptr_t A = reinterpret_cast<uintptr_t>(a), B = reinterpret_cast<uintptr_t>(b);
  const uint32_t* wa = reinterpret_cast<const uint32_t*>(A & ~uintptr_t(3));
  const uint32_t* wb = reinterpret_cast<const uint32_t*>(B & ~uintptr_t(3));
  const uint32_t sa = uint32_t(A & 3) * 8, sb = uint32_t(B & 3) * 8;
  const uint32_t* la = reinterpret_cast<const uint32_t*>((A + len - 1) & ~uintptr_t(3));
  const uint32_t* lb = reinterpret_cast<const uint32_t*>((B + len - 1) & ~uintptr_t(3));
  uint32_t ca = __ldg(wa), cb = __ldg(wb);
  for (uint32_t i = 0, k = 1; i < len; i += 4, k++) {
    const uint32_t na = wa + k <= la ? __ldg(wa + k) : 0u, nb = wb + k <= lb ? __ldg(wb + k) : 0u;
    uint32_t x = sa ? __funnelshift_r(ca, na, sa) : ca, y = sb ? __funnelshift_r(cb, nb, sb) : cb;
    const uint32_t rem = len - i;
    if (rem < 4) {
      const uint32_t m = (1u << (8 * rem)) - 1u;
      x &= m;
      y &= m;
    }
    if (x != y) return false;
    ca = na;
    cb = nb;
  }
  return true;
}

// The 8-byte chunks of [p, p + len), len >= 1, from 8-byte aligned loads
// realigned with shifts (the aligned word holding the last byte is the last
// one read, as in bytes_equal): half the load instructions of the 4-byte
// path, which matters where each lane reads its own key (the lookups).
struct ChunkStream {
  const uint64_t* w;
  const uint64_t* last;
  uint32_t sh;
  uint64_t cur;
  __device__ __forceinline__ ChunkStream(const uint8_t* p, uint32_t len) {
    const uintptr_t A = reinterpret_cast<uintptr_t>(p);
    w = reinterpret_cast<const uint64_t*>(A & ~uintptr_t(7));
    last = reinterpret_cast<const uint64_t*>((A + len - 1) & ~uintptr_t(7));
    sh = uint32_t(A & 7) * 8;
    cur = __ldg(reinterpret_cast<const unsigned long long*>(w));
  }
  __device__ __forceinline__ uint64_t next() {
    const uint64_t* nw = w + 1;
    const uint64_t nxt = nw <= last ? __ldg(reinterpret_cast<const unsigned long long*>(nw)) : 0ull;
    const uint64_t x = sh ? (cur >> sh) | (nxt << (64 - sh)) : cur;
    w = nw;
    cur = nxt;
    return x;
  }
};

__device__ __forceinline__ bool bytes_equal64(const uint8_t* a, const uint8_t* b, uint32_t len) {
  if (len == 0) return true;
  ChunkStream A(a, len), B(b, len);
  for (uint32_t i = 0; i < len; i += 8) {
    uint64_t x = A.next(), y = B.next();
    const uint32_t rem = len - i;
    if (rem < 8) {
      const uint64_t m = (1ull << (8 * rem)) - 1ull;
      x &= m;
      y &= m;
    }
    if (x != y) return false;
  }
  return true;
}

// The expanded fingerprint over ChunkStream (8-byte chunks = two words):
// chunk c holds words 2c and 2c+1, weighted r^(nw-2c) and r^(nw-2c-1); the
// last chunk is masked to the key's bytes (its second word is then zero when
// nw is odd, and takes r^0).
__device__ __forceinline__ uint64_t fingerprint_pw64(const uint8_t* bytes, uint64_t off, uint64_t len, uint64_t r,
                                                     const FpPow* pw) {
  if (len == 0) return 0;
  if (len > 4 * kFpPowMax) return fingerprint_dev(bytes, off, len, r);
  const uint32_t L = uint32_t(len);
  ChunkStream S(bytes + off, L);
  uint64_t a0 = 0, a1 = 0, a2 = 0;
  uint32_t e = (L + 3) >> 2;
  for (uint32_t c = 0; c < (L >> 3); c++, e -= 2) {
    const uint64_t x = S.next();
    fp3_acc(a0, a1, a2, uint32_t(x), pw->p[e]);
    fp3_acc(a0, a1, a2, uint32_t(x >> 32), pw->p[e - 1]);
  }
  if (L & 7) {
    const uint64_t x = S.next() & ((1ull << (8 * (L & 7))) - 1ull);
    fp3_acc(a0, a1, a2, uint32_t(x), pw->p[e]);
    fp3_acc(a0, a1, a2, uint32_t(x >> 32), pw->p[e - 1]);
  }
  return fp3_finish(a0, a1, a2, L);
}

// The same over a shared-memory copy: u holds the 4-byte words of the bytes
// from a 4-aligned position (one readable word past the last one), the key
// starts rel bytes in (1 <= len <= 4 * kFpPowMax); its words are realigned
// with 32-bit funnel shifts.
__device__ __forceinline__ uint64_t fingerprint_sm32(const uint32_t* u, uint32_t rel, uint32_t len, const FpPow* pw) {
  if (len == 0) return 0;
  const uint32_t sh = (rel & 3) * 8;
  const uint32_t* q = u + (rel >> 2);
  uint64_t a0 = 0, a1 = 0, a2 = 0;
  uint32_t e = (len + 3) >> 2, cur = q[0];
  for (uint32_t c = 0; c < (len >> 3); c++, e -= 2, q += 2) {
    const uint32_t m = q[1], n = q[2];
    fp3_acc(a0, a1, a2, __funnelshift_r(cur, m, sh), pw->p[e]);
    fp3_acc(a0, a1, a2, __funnelshift_r(m, n, sh), pw->p[e - 1]);
    cur = n;
  }
  if (len & 7) {
    const uint32_t m = q[1], n = q[2], t = len & 7;
    uint32_t w0 = __funnelshift_r(cur, m, sh), w1 = __funnelshift_r(m, n, sh);
    if (t < 4) w0 &= (1u << (8 * t)) - 1u;
    w1 = t > 4 ? w1 & ((1u << (8 * (t - 4))) - 1u) : 0u;
    fp3_acc(a0, a1, a2, w0, pw->p[e]);
    fp3_acc(a0, a1, a2, w1, pw->p[e - 1]);
  }
  return fp3_finish(a0, a1, a2, len);
}

#endif

}  // namespace hm
