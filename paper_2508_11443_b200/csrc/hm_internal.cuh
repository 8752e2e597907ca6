// hm_internal.cuh — shared host/device declarations of libhm (not part of the ABI).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "../../include/hm.h"
#include "hm_math.cuh"

namespace hm {

// Partition-buffer elements double as slot records: the first
// u64 is the hashed key (the key itself, or the fingerprint of a byte key).
struct __align__(16) KV16 {  // u64 keys: {key, value}
  uint64_t key, value;
};
struct __align__(32) KV32 {  // byte keys: {fp, value, ctx_off, len, 0}
  uint64_t key, value, ctx_off;
  uint32_t len, reserved;
};

// Device-detected conditions of one build pass (all zero-initialised).
struct DevStatus {
  unsigned int dup;            // two equal keys (DUPLICATE_KEY)
  unsigned int exhausted;      // some bucket needed 256 attempts
  unsigned int fpcoll;         // equal fingerprints, different bytes (redraw t0)
  unsigned int part_overflow;  // a build partition exceeded its capacity
  unsigned int slot_overflow;  // S exceeded the slot allocation
  unsigned int huge;           // a bucket with s > 32 and s^2 <= 4n (fallback path)
  unsigned int bound_fail;     // some bucket has s^2 > 4n (=> S > 4n)
  unsigned int ticket;         // partition ticket for the ordered look-back
  unsigned long long S;        // total slots of this pass
  unsigned long long max_count;// largest partition count
  unsigned int nhuge;          // entries in the huge-bucket list
  unsigned int pad;
};

constexpr int kMaxHuge = 1024;

// Shared-memory layout of k_bucket (byte offsets into the dynamic region).
constexpr int kNClsL = 3;
struct BucketSmem {
  uint32_t skv, lbk, rk, sidx, sA, src, slist, queue, ss, sstart, soff, st, total;
  uint32_t smax;                 // capacity of the slot source map
  uint32_t cls_off[kNClsL + 1];  // class-list regions in slist
};

struct BuildParams {
  L1Params l1;
  uint64_t smix;      // seed_mix(seed)
  uint64_t b_lo;      // first global bucket of this (shard) table
  uint64_t nb;        // local bucket count
  uint64_t n_in;      // number of input elements
  uint64_t slot_cap;  // allocated slots
  uint64_t bound4n;   // 4 * n_global (R7)
  uint32_t log2_bp;   // buckets per partition = 1 << log2_bp
  uint32_t np;        // partitions
  uint32_t cap;       // partition capacity (elements)
  uint32_t flags;     // HM_FLAG_* (hm.h)
  BucketSmem sl;      // k_bucket shared-memory layout
  uint64_t m2[33];    // floor((2^64 - 1) / s^2) for the exact mod s^2 (R22), s <= 32
  // a side copy k_bucket does while its first warp waits for the partition's
  // bulk load (the byte-key context, SideJob): partition p copies bytes
  // [p*cp_slice, (p+1)*cp_slice) of cp_src to cp_dst (both 16-aligned)
  const uint8_t* cp_src;
  uint8_t* cp_dst;
  uint64_t cp_bytes, cp_slice;
};

struct LookupParams {
  L1Params l1;
  uint64_t smix;
  uint64_t b_lo, nb;
  const uint64_t* dir;
  const CDir* cdir;
  const void* slots;
  // byte keys
  const uint8_t* ctx;
  uint64_t r_fp;
};

}  // namespace hm

struct hm_map {
  int device;
  uint32_t key_kind;     // 0 u64, 1 bytes
  uint64_t n_global;     // level-1 modulus
  uint64_t b_lo, nb;     // bucket range held
  uint64_t S;            // local slots
  uint64_t slot_base;    // global base of the local slots (shards)
  uint64_t seed;
  uint32_t t1, t0;
  bool is_shard;
  hm::L1Params l1;
  uint64_t smix;
  uint64_t r_fp;         // byte keys: fingerprint point (a1 of derive(seed,0,0,t0))
  size_t abytes[3];      // map_alloc sizes of dir, cdir, slots (0: plain cudaMalloc)
  hm_free_fn ufree;      // the user's free hook (hm_opts) when the arrays came from its alloc
  void* uctx;
  size_t ctx_alloc;      // allocation size of ctx (user hook)
  uint64_t* dir;         // nb entries, local soff
  hm::CDir* cdir;        // compact lookup directory, ceil(nb/32) records
  void* slots;           // S records
  uint8_t* ctx;          // byte keys: context copy
  uint64_t ctx_bytes;
};

namespace hm {
void set_error(const std::string& s);
hm_status cuda_fail(cudaError_t e, const char* where);
L1Params make_l1(uint64_t smix, uint32_t t1, uint64_t n_global);
int num_sms();
// Scope around every kernel launch of this library: counts it
// (hm_kernel_launches) and, when hm_profile_enable(1) is on, brackets it with
// CUDA events recorded on the launching stream (hm_profile_read).
struct LaunchScope {
  const char* name;
  cudaStream_t st;
  cudaEvent_t e0 = nullptr;
  LaunchScope(const char* n, cudaStream_t s);
  ~LaunchScope();
};

// build.cu
// Work a build enqueues once, on its stream, right before the first k_bucket
// launch (the radix passes are done): the byte-key build copies the key
// context then, so that the copy shares DRAM with the latency-bound k_bucket
// rather than with the bandwidth-bound fingerprint and radix passes.
struct SideJob {
  void (*fn)(void* ctx, cudaStream_t st) = nullptr;
  void* ctx = nullptr;
  // or, with kbytes set, a copy done inside the first k_bucket launch
  // (BuildParams::cp_*; 16-aligned pointers)
  const uint8_t* ksrc = nullptr;
  uint8_t* kdst = nullptr;
  uint64_t kbytes = 0;
  bool done = false;
  void run(cudaStream_t st) {
    if (fn && !done) fn(ctx, st);
    done = true;
  }
};
struct BuildOut {
  uint64_t* dir = nullptr;
  CDir* cdir = nullptr;
  void* slots = nullptr;
  uint64_t S = 0;
  uint32_t t1 = 0;
  size_t bytes[3] = {0, 0, 0};  // allocation sizes of dir, cdir, slots (map_alloc)
};
// Device arrays of a map (dir, cdir, slots) come from map_alloc and go back
// through map_release when the map is freed (after a device synchronisation):
// freed arrays are kept, up to a cap, for the next build of the same sizes.
hm_status map_alloc(void** p, size_t bytes, cudaStream_t st);
void map_release(void* p, size_t bytes);
// A map array that is not handed out (a failed build): back to the user's
// free hook when one is active on this thread, else to the pool.
void map_discard(void* p, size_t bytes, cudaStream_t st);
// The user's allocator hooks of the build running on this thread (hm_opts),
// set by the C-ABI entry points for the duration of a build.
struct UserAlloc {
  hm_alloc_fn alloc = nullptr;
  hm_free_fn free = nullptr;
  void* ctx = nullptr;
};
extern thread_local UserAlloc tl_user_alloc;
struct UserAllocScope {
  explicit UserAllocScope(const hm_opts* o) {
    tl_user_alloc = o && o->alloc && o->free ? UserAlloc{o->alloc, o->free, o->alloc_ctx} : UserAlloc{};
  }
  ~UserAllocScope() { tl_user_alloc = UserAlloc{}; }
};
// t1_fixed < 0: search t1 = 0..15 with the space bound of this table.
hm_status release_workspace();
hm_status build_u64_core(const uint64_t* keys, const uint64_t* vals, uint64_t n_in, uint64_t n_global,
                         uint64_t b_lo, uint64_t nb, int t1_fixed, uint64_t seed, uint32_t log2_bp,
                         cudaStream_t st, BuildOut* out);
hm_status check_offsets(const uint64_t* offsets, uint64_t n, cudaStream_t st);
hm_status build_bytes_core(const uint8_t* bytes, const uint64_t* offsets, const uint64_t* vals, uint64_t n,
                           uint64_t seed, uint32_t log2_bp, cudaStream_t st, BuildOut* out, uint32_t* t0_out,
                           uint64_t* r_out, SideJob* job = nullptr, const uint64_t* off0_host = nullptr);
hm_status dedup_workspace(void** p, size_t bytes, cudaStream_t st);  // build.cu's cached scratch
hm_status dedup_partitioned_bytes(const uint8_t* bytes, const uint64_t* offs, const uint64_t* fp,
                                  const uint64_t* vals, uint64_t n, uint64_t off0, cudaStream_t st, uint8_t* keep);
void launch_fingerprint(const uint8_t* bytes, const uint64_t* offs, uint64_t n, uint64_t r, uint64_t* fp,
                        cudaStream_t st);
hm_status dedup_bytes(const uint8_t* bytes, const uint64_t* offs, const uint64_t* vals, uint64_t n, cudaStream_t st,
                      uint8_t** out_ctx, uint64_t** out_offs, uint64_t** out_vals, uint64_t* n_out);
hm_status dedup_partitioned(const uint64_t* keys, const uint64_t* vals, uint64_t n, cudaStream_t st, uint64_t* okeys,
                            uint64_t* ovals, uint64_t* n_out);
// dedup.cu: from_array's distinct (first-occurrence) keys, device arrays owned by the caller
hm_status dedup_u64(const uint64_t* keys, const uint64_t* vals, uint64_t n, cudaStream_t st, uint64_t** out_keys,
                    uint64_t** out_vals, uint64_t* n_out);
// rounds.cu: the sortless round-based construction (HM_FLAG_ROUNDS ablation)
// (a shard: buckets [b_lo, b_lo + nb) of the level-1 function mod n_global with t1 = t1_fixed >= 0)
hm_status build_u64_rounds(const uint64_t* keys, const uint64_t* vals, uint64_t n_in, uint64_t n_global,
                           uint64_t b_lo, uint64_t nb, int t1_fixed, uint64_t seed, uint32_t flags, cudaStream_t st,
                           BuildOut* out);
hm_status build_bytes_rounds(const uint64_t* fp, const uint64_t* vals, const uint64_t* offs, uint64_t off0,
                             const uint8_t* bytes, uint64_t n, uint64_t seed, uint32_t flags, cudaStream_t st,
                             BuildOut* out, bool* fpcoll);
// assemble.cu
hm_status assemble_cdir_launch(const uint64_t* dir, const void* slots, uint64_t n, uint64_t S, const L1Params& l1,
                               uint32_t full_dir, CDir* cdir, unsigned int* bad, cudaStream_t st);
hm_status dir_rebase_launch(uint64_t* d, uint64_t n, uint64_t base, cudaStream_t st);
// lookup.cu
hm_status lookup_u64_launch(const hm_map* m, const uint64_t* q, uint64_t nq, uint64_t* out_vals,
                            uint8_t* out_found, cudaStream_t st);
hm_status lookup_bytes_launch(const hm_map* m, const uint8_t* qb, const uint64_t* qo, uint64_t nq,
                              uint64_t* out_vals, uint8_t* out_found, cudaStream_t st);
hm_status route_count_launch(const uint64_t* keys, uint64_t n, const L1Params& l1, int world, uint64_t* counts,
                             cudaStream_t st);
hm_status route_u64_launch(const uint64_t* keys, const uint64_t* vals, uint64_t n, const L1Params& l1,
                           int world, uint64_t* sk, uint64_t* sv, uint64_t* counts, cudaStream_t st);
hm_status route_queries_launch(const L1Params& l1, const uint64_t* q, uint64_t nq, int world, uint64_t* sq,
                               uint64_t* perm, uint64_t* counts, cudaStream_t st);
hm_status unroute_launch(const uint64_t* vr, const uint8_t* fr, const uint64_t* perm, uint64_t nq,
                         uint64_t* ov, uint8_t* of, cudaStream_t st);
}  // namespace hm

#define HM_CUDA_TRY(expr)                                              \
  do {                                                                 \
    cudaError_t e__ = (expr);                                          \
    if (e__ != cudaSuccess) return ::hm::cuda_fail(e__, #expr);        \
  } while (0)
