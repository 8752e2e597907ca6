/*
 * hm.h — C-ABI of the B200-native static FKS hash map (libhm.so).
 *
 * Method: "Towards Efficient Hash Maps in Functional Array Languages"
 * (arXiv 2508.11443).  Citations are PAPER.md line numbers (the LaTeX source)
 * with the section they fall in; R<k> are the readings of the paper listed in
 * DESIGN.md §2.
 *
 * The library builds the two-level FKS hash set of §2.2 —
 *   g k = (hash const k) mod n,  shape = hist of g (squared: s_b^2 slots),
 *   offsets = presum shape,      h k = offsets[g k] + (hash consts[g k] k mod s_b^2)
 * — extended to a hash map by an accompanying value per slot,
 * and answers batched lookups (PAPER.md:244-245 membership test, §3.2 lookup).
 *
 * Conventions for every entry point:
 *  - All pointers are DEVICE pointers of the map's device unless stated
 *    otherwise.  The build and lookup entry points also accept HOST pointers
 *    (pageable or pinned) for their array arguments; they are detected with
 *    cudaPointerGetAttributes and staged through device memory inside the call
 *    (this is the end-to-end path bench.py times).  Mixing host and device
 *    arrays in one call is allowed.
 *  - `stream` is a cudaStream_t passed as void* (NULL = the legacy default
 *    stream).  Kernels run on that stream only.
 *  - Sizes are element counts unless named *_bytes.
 *  - No entry point ever falls back to a CPU implementation.  Errors are
 *    returned as hm_status; a human-readable detail for the last failure on the
 *    calling thread is available from hm_last_error().
 *  - Every result is a deterministic function of (seed, key set[, context
 *    order for byte keys]); internal parallel order never changes it (R13).
 */
#ifndef HM_H_
#define HM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HM_SPEC_VERSION 1u
#define HM_MAGIC 0x31544D48u /* "HMT1" little-endian */

typedef enum {
  HM_OK = 0,
  HM_ERR_INVALID_ARG = 1,    /* NULL where required, bad offsets, both outputs NULL ... */
  HM_ERR_EMPTY = 2,          /* n == 0: K is a non-empty set (§2.2)        */
  HM_ERR_DUPLICATE_KEY = 3,  /* from_array_nodup precondition violated  */
  HM_ERR_SEED_EXHAUSTED = 4, /* level one: t1 reached 16 (R7); or a bucket reached t = 256 (R8) */
  HM_ERR_FP_EXHAUSTED = 5,   /* byte keys: fingerprint redraw t0 reached 16 (R5)          */
  HM_ERR_TOO_LARGE = 6,      /* n > 2^30, or a byte key longer than 65535 bytes (R23)     */
  HM_ERR_OOM = 7,            /* device allocation failed                                   */
  HM_ERR_CUDA = 8,           /* a CUDA runtime error (detail in hm_last_error)             */
  HM_ERR_NCCL = 9,           /* an NCCL call of hm_*_dist failed (detail in hm_last_error) */
  HM_ERR_NO_DEVICE = 10      /* no CUDA device / wrong architecture                       */
} hm_status;

typedef struct hm_map hm_map; /* opaque; immutable after build; bound to its device */

/* Build options.  NULL means all defaults. */
/* Allocator hooks for the arrays a map owns.  alloc returns
 * `bytes` of device memory of the current device, 32-B aligned (the slot and
 * compact-directory records are read with 32-byte vector loads; a pointer that
 * is not 32-B aligned is handed back to free and the build returns
 * HM_ERR_INVALID_ARG), usable in stream order on `stream` (NULL: failure ->
 * HM_ERR_OOM); free gets back the pointer and the size it was allocated with. */
typedef void* (*hm_alloc_fn)(size_t bytes, void* stream, void* ctx);
typedef void (*hm_free_fn)(void* ptr, size_t bytes, void* stream, void* ctx);

typedef struct {
  uint64_t seed;       /* table seed: selects the constant schedule (R6). default 0  */
  uint32_t log2_bp;    /* 0 = auto. log2 of the level-1 buckets per build partition (5..12; smaller values act as 5) */
  uint32_t flags;      /* 0, or HM_FLAG_* below; other bits -> HM_ERR_INVALID_ARG     */
  /* NULL, NULL: the library's stream-ordered pool (cudaMallocAsync, with freed
   * maps' arrays cached per size, see hm_release_workspace).  Both set: every
   * array the built map owns (directory, compact directory, slots, the byte
   * context copy) comes from alloc(bytes, build stream, alloc_ctx) and returns
   * through free(ptr, bytes, stream, alloc_ctx) — from hm_free (stream NULL,
   * after a device synchronisation) or, on a failed build, on the build
   * stream.  Build scratch stays library-managed.  One hook alone:
   * HM_ERR_INVALID_ARG. */
  hm_alloc_fn alloc;
  hm_free_fn free;
  void* alloc_ctx;
} hm_opts;

/* Lookups of this map bypass the L2-resident compact directory and read the
 * full directory entry for every query (a testing/diagnostic knob: the
 * results are identical, only slower).  The table itself is unchanged. */
#define HM_FLAG_FULL_DIRECTORY 1u
/* Testing knobs of the construction (the table is identical, only the route
 * differs): DIRECT_SLOTS makes every build partition write its slots straight
 * from the search (the path of a partition whose slots exceed the shared-memory
 * staging map); NO_ROUND0_ILP tries one attempt per bucket in round 0 and
 * leaves the rest to the lane-parallel rounds. */
#define HM_FLAG_DIRECT_SLOTS 2u
#define HM_FLAG_NO_ROUND0_ILP 4u
/* Alternative route of the u64 construction (same table): radix pass 2 and
 * the per-partition construction as one pipelined kernel (k_split2_bucket):
 * a partition job takes its records from L2 right after the pass-2 tiles of
 * its region wrote them and drops the lines there without write-back (the
 * build's DRAM traffic falls by ~2 GB per 2^26 keys), but the two job kinds
 * sharing the SMs issue more slowly than the two kernels (measured 3.05 vs
 * 2.70 ms at 2^26), so it is not the default.  Byte keys ignore
 * it. */
#define HM_FLAG_FUSED_PASS2 64u
/* from_array: the keys may repeat;
 * the first occurrence (lowest input index) of every key keeps its value, and
 * the map is the one the default build (from_array_nodup) makes from the
 * distinct keys — hm_info's n is their number; byte keys are compared by
 * content and the distinct ones are packed in input order into the map's
 * context (any duplication pattern; heavy duplication of byte keys takes a
 * global fingerprint set confirmed by content). */
#define HM_FLAG_FROM_ARRAY 8u
/* Ablation (u64 keys only; byte keys -> HM_ERR_INVALID_ARG): build level two
 * with the paper's sortless round-based construction (PAPER.md:443-499,
 * §2.5: flat arrays, hist for collisions, presum renumbering, one grid-wide
 * pass per round) instead of the partitioned warp-per-bucket search.  The
 * table is identical (R13); only the construction route and its speed
 * differ.  log2_bp is ignored. */
#define HM_FLAG_ROUNDS 16u
/* hm_build_u64_dist only: the route kernel stores
 * every (key, value) straight into its owner's receive window over NVLink (a
 * symmetric window: ncclMemAlloc + ncclCommWindowRegister, peer pointers from
 * NCCL 2.28's device API) instead of the grouped ncclSend/ncclRecv all-to-all
 * after it; the shards are the same.  Needs every rank in one NVLink domain
 * (a single node).  Other calls: HM_ERR_INVALID_ARG. */
#define HM_FLAG_FUSED_EXCHANGE 32u
/* (The receive windows of HM_FLAG_FUSED_EXCHANGE builds stay registered on
 * their communicator for the next builds; hm_dist_release_windows, called by
 * every rank of the communicator — it is collective — frees them.) */

/* Table header, 56 bytes, little-endian (DESIGN.md §4 "Table layout"). */
typedef struct {
  uint32_t magic;        /* HM_MAGIC                                   */
  uint32_t spec_version; /* HM_SPEC_VERSION                            */
  uint32_t key_kind;     /* 0 = u64 keys, 1 = byte-string keys         */
  uint32_t reserved;     /* 0                                          */
  uint64_t n;            /* number of keys = number of level-1 buckets (R3) */
  uint64_t S;            /* total slots = sum over buckets of s_b^2    */
  uint64_t seed;         /* table seed                                 */
  uint32_t t1;           /* level-1 attempt (first with S <= 4n, R7)   */
  uint32_t t0;           /* byte keys: fingerprint attempt (R5); 0 for u64 */
  uint64_t ctx_bytes;    /* byte keys: size of the map's context copy  */
} hm_header;

/* ------------------------------------------------------------------ build
 * hm_build_u64 — from_array_nodup for 64-bit integer keys (PAPER.md:608-609,
 * 623-624; construction §2.2-§2.5).
 *   keys[n], vals[n]: the key/value pairs (u64 each).  Keys must be pairwise
 *                     distinct; violations are detected and reported as
 *                     HM_ERR_DUPLICATE_KEY (never a hang, never a wrong table).
 *   opts:   NULL or build options.
 *   stream: the stream all work is ordered on.
 *   out:    receives the new map (NULL on failure).
 * Synchronous: the call waits on `stream` once at the end to learn the total
 * slot count and the device-detected error flags; inputs may be freed when it
 * returns.  The map owns its directory u64[n] and its slot array {key,value}[S]
 * (16 B per slot), allocated with cudaMallocAsync on `stream`.
 * Errors: HM_ERR_EMPTY (n==0), HM_ERR_TOO_LARGE (n>2^30), HM_ERR_INVALID_ARG
 * (NULL keys/vals/out), HM_ERR_DUPLICATE_KEY, HM_ERR_SEED_EXHAUSTED,
 * HM_ERR_OOM, HM_ERR_CUDA.  Precedence (R26): level-1 exhaustion,
 * then duplicates, then level-2 exhaustion. */
hm_status hm_build_u64(const uint64_t* keys, const uint64_t* vals, uint64_t n,
                       const hm_opts* opts, void* stream, hm_map** out);

/* hm_build_bytes — from_array_nodup for byte-string keys (slices of a flat
 * context, §3.1; slice keys PAPER.md:726-746).
 *   bytes:   the flat context; key i is bytes[offsets[i] .. offsets[i+1]).
 *   offsets: u64[n+1], CSR, non-decreasing; offsets[0] need not be 0.
 *   vals:    u64[n].
 * The map stores a COPY of bytes[offsets[0] .. offsets[n])
 * and 32-byte slots {u64 fp, u64 value, u64 ctx_off, u32 len, u32 0}[S], with
 * ctx_off relative to offsets[0].  Keys are hashed through a 61-bit polynomial
 * fingerprint (R5); two different keys with equal fingerprints trigger a
 * redraw of the fingerprint point (t0), equal keys are DUPLICATE_KEY.
 * Errors: as hm_build_u64, plus HM_ERR_TOO_LARGE for a key longer than 65535
 * bytes and HM_ERR_FP_EXHAUSTED.  Synchronous like hm_build_u64. */
hm_status hm_build_bytes(const uint8_t* bytes, const uint64_t* offsets, const uint64_t* vals,
                         uint64_t n, const hm_opts* opts, void* stream, hm_map** out);

/* ----------------------------------------------------------------- lookup
 * hm_lookup_u64 — batched lookup: for each query
 * q[i], b = g q; probe the directory dir[b]; an empty bucket misses (R9);
 * j = soff_b + (hash consts_b q mod s_b^2) (singletons: j = soff_b, R12);
 * hit iff slot[j].key == q.
 *   out_vals[nq]:  value on a hit, 0 on a miss (R24).  May be NULL
 *                  (membership only).
 *   out_found[nq]: 1 on a hit, 0 on a miss.  May be NULL.  Not both NULL.
 * Asynchronous and stream-ordered when all arrays are device memory; when any
 * array is host memory the call stages it and returns after the results are
 * on the host; with host queries and host (or NULL) outputs beyond 2^24
 * queries the batch moves in 2^23-query chunks whose upload, lookups and
 * download overlap (two library copy streams, ordered with `stream` by
 * events; pinned host memory is needed for the overlap).  A map may serve
 * concurrent lookups from several streams.
 * Errors: HM_ERR_INVALID_ARG (NULL map/q with nq>0, both outputs NULL, wrong
 * key kind), HM_ERR_CUDA. */
hm_status hm_lookup_u64(const hm_map* map, const uint64_t* q, uint64_t nq, uint64_t* out_vals,
                        uint8_t* out_found, void* stream);

/* hm_lookup_bytes — batched lookup of byte-string needles given in their OWN
 * context: needle i is
 * qbytes[qoffsets[i] .. qoffsets[i+1]).  A hit requires equal fingerprint,
 * equal length and equal bytes against the map's context copy.  Outputs and
 * errors as hm_lookup_u64. */
hm_status hm_lookup_bytes(const hm_map* map, const uint8_t* qbytes, const uint64_t* qoffsets,
                          uint64_t nq, uint64_t* out_vals, uint8_t* out_found, void* stream);

/* ---------------------------------------------------------------- lifetime */
/* NULL-safe; waits for the device's pending work.  The map's device arrays are
 * kept for reuse by the next build of the same size (see
 * hm_release_workspace) unless that cache is full. */
void hm_free(hm_map* map);

/* Header of the (logical) table.  host_out: host pointer. */
hm_status hm_info(const hm_map* map, hm_header* host_out);

/* hm_export — copy the table out for parity checks and for replication
 * (DESIGN.md §4).  Each destination may be host or device memory (of the
 * map's device); a device directory is rebased on the device:
 *   host_dir:   u64[n]  entry b = soff_b | s_b<<40 | t_b<<56 (may be NULL)
 *   host_slots: S slots of 16 B (u64 keys) or 32 B (byte keys) (may be NULL)
 *   host_ctx:   ctx_bytes bytes of the map's context copy (byte keys; may be NULL)
 * For a shard (hm_build_u64_shard) the directory covers the shard's bucket
 * range and soff is GLOBAL (the shard's slot base is added). Synchronous. */
hm_status hm_export(const hm_map* map, uint64_t* host_dir, void* host_slots, uint8_t* host_ctx);

/* hm_assemble_u64 — a map (u64 keys) from a complete table in the layout of
 * dir u64[n] (soff | s<<40 | t<<56, soff global), slots
 * {u64 key, u64 value}[S], as hm_export writes them — for a distributed build,
 * the shards' exports concatenated in rank order, which is the single table
 * (the replicated-lookup mode; dist.replicate_dist).
 * seed and t1 are the table's (hm_info).  dir/slots: host or device pointers,
 * copied (the caller keeps ownership).  The compact lookup directory is
 * derived on the device.  Checked: soff_0 = 0, soff_{b+1} = soff_b + s_b^2,
 * soff_{n-1} + s_{n-1}^2 = S and t = 0 where s < 2 (else HM_ERR_INVALID_ARG),
 * so that no lookup probe leaves the slots; the keys themselves are trusted
 * (a table whose keys do not hash to their slots gives misses, not faults).
 * n == 0: HM_ERR_EMPTY; S > 4n or n > 2^30: HM_ERR_TOO_LARGE; opts: seed and
 * log2_bp ignored, flags 0 or HM_FLAG_FULL_DIRECTORY. */
hm_status hm_assemble_u64(const uint64_t* dir, const void* slots, uint64_t n, uint64_t S, uint64_t seed, uint32_t t1,
                          const hm_opts* opts, void* stream, hm_map** out);

const char* hm_status_str(hm_status s);
const char* hm_last_error(void); /* thread-local; "" if none */
const char* hm_version(void);
/* Number of CUDA kernels this library has launched in this process (all
 * devices, all threads): the evidence bench.py reports as gpu_launches. */
uint64_t hm_kernel_launches(void);

/* hm_release_workspace — free the build scratch this library caches between
 * builds (per device and stream: partition buffers and their bucket codes,
 * fingerprints, the from_array dedup set; about 44 B per key for u64 builds,
 * 52 B per key for byte-key builds) on the current device, and trim the
 * device's default stream-ordered memory pool, whose release threshold the
 * library raises on first use (freed table memory otherwise goes back to the
 * driver at every synchronisation and is re-mapped by the next build), and
 * free the arrays of freed maps that the library keeps (per device and size,
 * at most 32 GB) for the next build of the same size.  Live maps are not
 * affected.  Synchronises the device. */
hm_status hm_release_workspace(void);

/* Per-kernel device timing (diagnostics, used by bench.py for the roofline).
 * While enabled, every kernel launch of this library is bracketed by two CUDA
 * events recorded on the stream it is launched on.  hm_profile_read
 * synchronises those events, aggregates them per kernel name since the last
 * read, writes up to `max` entries to host array `out`, clears the record and
 * returns the number of distinct kernels. */
typedef struct {
  char name[32];     /* kernel name, e.g. "k_bucket" */
  uint64_t launches; /* launches since the last read */
  double ms;         /* summed event-to-event device time */
} hm_kernel_stat;
void hm_profile_enable(int on);
int hm_profile_read(hm_kernel_stat* out, int max);

/* ------------------------------------------------- multi-GPU building blocks
 * Bucket-range sharding: with G ranks and the
 * global key count n (= number of level-1 buckets), rank r owns buckets
 * [lo_r, lo_{r+1}) with lo_r = ceil(r*n/G), i.e. owner(b) = floor(b*G/n).
 * The exchange between the two steps is done by the caller (NCCL all-to-all
 * through torch.distributed); these entry points are the kernels on each side. */

/* hm_route_u64 — level-1 hash each (key, value) with the level-1 constants of
 * attempt t1 and partition the pairs by owner rank (stable within a rank is
 * NOT guaranteed).
 *   keys/vals[n_local]: this rank's input pairs.
 *   n_global: the global n (the level-1 modulus).
 *   send_keys/send_vals[n_local]: output, grouped by destination rank.
 *   send_counts[world]: output (device, u64): pairs destined to each rank.
 * Asynchronous. */
hm_status hm_route_u64(const uint64_t* keys, const uint64_t* vals, uint64_t n_local,
                       uint64_t n_global, uint64_t seed, uint32_t t1, int world,
                       uint64_t* send_keys, uint64_t* send_vals, uint64_t* send_counts,
                       void* stream);

/* hm_build_u64_dist — collective build of the bucket-range-sharded table over
 * an NCCL communicator.  Every rank of
 * `nccl_comm` (an ncclComm_t, e.g. torch's ProcessGroupNCCL._comm_ptr(); the
 * library uses the libnccl.so.2 the process has loaded) calls it with its own
 * keys/vals[n_local] (device pointers): the global n is their sum; rank r
 * receives the shard of level-1 buckets [ceil(r n / G), ceil((r+1) n / G)).
 * The shards together are exactly the single table hm_build_u64 builds from
 * the union of the keys (hm_export of a shard writes global soff).  All ranks
 * return the same status (max over ranks); duplicates anywhere in the union:
 * HM_ERR_DUPLICATE_KEY.  Synchronous on `stream`.  Free with hm_free.
 * A rank that fails before the status agreement (a device allocation, an
 * NCCL error) returns alone and leaves the others inside NCCL: abort the
 * communicator (ncclCommAbort) as for any collective. */
hm_status hm_build_u64_dist(const uint64_t* keys, const uint64_t* vals, uint64_t n_local, const hm_opts* opts,
                            void* stream, void* nccl_comm, hm_map** out);

/* hm_lookup_u64_dist — collective lookup on the shards of hm_build_u64_dist:
 * each rank passes its own queries q[nq] (device) and receives its own
 * answers in out_vals / out_found (device, as hm_lookup_u64).  Queries are
 * routed to the owner of their level-1 bucket, answered there and routed
 * back.  Every rank must call it (nq may be 0).  Synchronous for the count
 * exchange; the results are complete in `stream` order. */
hm_status hm_dist_release_windows(void* nccl_comm);

hm_status hm_lookup_u64_dist(const hm_map* shard, const uint64_t* q, uint64_t nq, uint64_t* out_vals,
                             uint8_t* out_found, void* stream, void* nccl_comm);

/* The control decisions of the sharded build, shared by hm_build_u64_dist and
 * any other orchestration of the per-rank pieces (paper_2508_11443_b200/dist.py
 * over torch.distributed), so that both take them the same way.  Host-only:
 * no device is touched.
 *
 * hm_dist_bucket_range — [*lo, *hi) of the level-1 buckets rank `rank` of
 * `world` owns with n = n_global buckets: lo_r = ceil(r n / G).
 * Returns HM_ERR_INVALID_ARG for world < 1, rank outside [0, world). */
hm_status hm_dist_bucket_range(uint64_t n_global, int world, int rank, uint64_t* lo, uint64_t* hi);

/* hm_dist_decide — after every rank built its shard with level-1 attempt t1
 * and the ranks agreed on S_total = sum_r S_r (all-reduce sum) and
 * max_status = max_r status_r (all-reduce max):
 *   returns HM_OK when the build is done (max_status 0 and the global space
 *     bound S_total <= 4 n_global holds, R7);
 *   returns max_status (nonzero) when some shard failed: every rank reports it;
 *   otherwise the bound failed: with t1 + 1 < 16, *next_t1 = t1 + 1 and the
 *     return value is HM_DIST_REDRAW (route again with *next_t1); at t1 = 15,
 *     HM_ERR_SEED_EXHAUSTED (PAPER.md has no bound; R7, R26). */
#define HM_DIST_REDRAW 100
int hm_dist_decide(uint64_t n_global, uint32_t t1, uint64_t S_total, int max_status, uint32_t* next_t1);

/* hm_dist_slot_base — the global slot base of rank `rank`: sum of S_all[q]
 * for q < rank (the exclusive prefix of the shards' slot counts, from an
 * all-gather of S_r). */
uint64_t hm_dist_slot_base(const uint64_t* S_all, int world, int rank);

/* hm_dist_exchange_plan — the fused route + exchange's placement
 * (HM_FLAG_FUSED_EXCHANGE): from the all-gathered count matrix
 * C[q * world + r] (pairs rank q routes to owner r), off[r] = where this
 * rank's run starts in owner r's receive buffer (sum of C[q][r] for q < rank),
 * *recv = pairs this rank receives (sum of C[q][rank]), *cap = the largest
 * receive count over the ranks (the symmetric window's size).  Host-only. */
hm_status hm_dist_exchange_plan(const uint64_t* C, int world, int rank, uint64_t* off, uint64_t* cap,
                                uint64_t* recv);

/* hm_build_u64_shard — build the shard of the global table that holds level-1
 * buckets [b_lo, b_hi) of a table with n_global keys, from exactly the keys
 * routed to it, with level-1 attempt t1 fixed by the caller.  The caller
 * checks the global space bound sum_r S_r <= 4 n_global (R7) and redraws t1
 * if it fails.  On return *S_local holds the shard's slot count.  The shard's
 * global slot base (exclusive prefix of S_r over ranks) is set with
 * hm_shard_set_base.  Errors as hm_build_u64 (duplicates within the shard are
 * reported; SEED_EXHAUSTED only for level-2 exhaustion). Synchronous.
 * opts->flags: FULL_DIRECTORY and the construction testing knobs only
 * (FROM_ARRAY, ROUNDS: HM_ERR_INVALID_ARG — single-table paths). */
hm_status hm_build_u64_shard(const uint64_t* keys, const uint64_t* vals, uint64_t n_recv,
                             uint64_t n_global, uint64_t b_lo, uint64_t b_hi, uint32_t t1,
                             const hm_opts* opts, void* stream, hm_map** out, uint64_t* S_local);

hm_status hm_shard_set_base(hm_map* map, uint64_t slot_base);

/* hm_route_queries_u64 — partition queries by owner rank of their level-1
 * bucket. send_q[nq] grouped by rank, perm[nq] (u64): position in send_q of
 * query i, send_counts[world] (u64, device). Asynchronous. */
hm_status hm_route_queries_u64(const hm_map* map, const uint64_t* q, uint64_t nq, int world,
                               uint64_t* send_q, uint64_t* perm, uint64_t* send_counts,
                               void* stream);

/* hm_unroute_u64 — out_vals[i] = vals_routed[perm[i]], out_found likewise
 * (either output may be NULL). Asynchronous. */
hm_status hm_unroute_u64(const uint64_t* vals_routed, const uint8_t* found_routed,
                         const uint64_t* perm, uint64_t nq, uint64_t* out_vals,
                         uint8_t* out_found, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* HM_H_ */
