/*
 * fks_oracle.c — the CPU ORACLE for the FKS static hash map.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  The
 * product path (paper_2508_11443_b200/) never links, imports or calls it, and
 * shares no code with it: no headers, no helpers, no constant tables.
 *
 * It is a plain, slow, obviously-correct sequential implementation of what the
 * hot path computes, written from the paper:
 *   - §2.2 "The Construction"   PAPER.md:220-247  (h, g, shape, offsets; the
 *                                                  well-formed / collision-free
 *                                                  properties; the arr table)
 *   - §2.3 "Functional Construction" PAPER.md:249-308 (make1, hashes,
 *                                                  collision, make2)
 *   - Fig. 1 vocabulary         PAPER.md:145-218  (hist, presum, groupby, sum)
 *   - §3.1 contexts             PAPER.md:558-581  (string keys = slices of a
 *                                                  flat byte context)
 * with the readings listed in DESIGN.md §2 (R1..R26) for
 * everything the paper leaves open: the hash family (R4), the sequence
 * fingerprint (R5), the deterministic `random` schedule (R6), the level-1
 * space bound (R7), attempt caps (R8), empty buckets (R9), filler slots (R10),
 * singletons (R12) and the table layout.
 *
 * All arithmetic is exact integer arithmetic: 128-bit products and the C `%`
 * operator.  No blocking, fusion or reordering beyond the paper's functional
 * formulation.  Pins: tests/test_oracle_*.py.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

/* --------------------------------------------------------------- statuses
 * Numeric values are part of the C-ABI contract; the oracle
 * defines its own copy. */
enum {
  OR_OK = 0,
  OR_ERR_INVALID_ARG = 1,
  OR_ERR_EMPTY = 2,          /* n == 0: K must be non-empty     */
  OR_ERR_DUPLICATE_KEY = 3,  /* from_array_nodup precondition  */
  OR_ERR_SEED_EXHAUSTED = 4, /* t1 reached 16, or some bucket reached t=256  */
  OR_ERR_FP_EXHAUSTED = 5,   /* strings: t0 reached 16                       */
  OR_ERR_TOO_LARGE = 6,      /* n > 2^30 or a key longer than 65535 bytes    */
  OR_ERR_OOM = 7
};

#define OR_P ((1ULL << 61) - 1)          /* Mersenne prime 2^61-1 (R4)     */
#define OR_GAMMA 0x9E3779B97F4A7C15ULL  /* splitmix64 increment (R6)       */
#define OR_SEED_SALT 0xD6E8FEB86659FD93ULL
#define OR_T1_CAP 16u   /* R7 */
#define OR_T2_CAP 256u  /* R8 */
#define OR_T0_CAP 16u   /* R5 */
#define OR_MAX_N (1ULL << 30) /* R23 */
#define OR_MAGIC 0x31544D48u  /* "HMT1" little-endian */
#define OR_SPEC_VERSION 1u

/* ------------------------------------------------------- random (R6)
 * PAPER.md:164 "random : unit -> [c]int": the constants
 * must make `hash` a universal family.  Made deterministic as a counter
 * schedule:  ctr = level<<60 | bucket<<8 | attempt,
 *            u   = mix64(mix64(seed ^ SALT) ^ ctr),
 *            z_j = mix64(u + GAMMA*(j+1))   (the j-th splitmix64 output from u)
 * with mix64 the splitmix64 output function. */
uint64_t or_mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

static uint64_t or_field(uint64_t z) { /* a uniform-ish element of [0, P) */
  uint64_t v = z >> 3;
  return v == OR_P ? 0 : v;
}

/* out = (a1, a2, b): a1, a2 in [1, P), b in [0, P). */
void or_derive(uint64_t seed, uint32_t level, uint64_t bucket, uint32_t attempt,
               uint64_t out[3]) {
  uint64_t ctr = ((uint64_t)level << 60) | (bucket << 8) | (uint64_t)attempt;
  uint64_t u = or_mix64(or_mix64(seed ^ OR_SEED_SALT) ^ ctr);
  uint64_t z0 = or_mix64(u + OR_GAMMA * 1);
  uint64_t z1 = or_mix64(u + OR_GAMMA * 2);
  uint64_t z2 = or_mix64(u + OR_GAMMA * 3);
  out[0] = or_field(z0);
  if (out[0] == 0) out[0] = 1;
  out[1] = or_field(z1);
  if (out[1] == 0) out[1] = 1;
  out[2] = or_field(z2);
}

/* ------------------------------------------------------------ hash (R4)
 * PAPER.md:165 "hash : [c]int -> alpha -> int"; "based on a universal hash
 * function".  Carter-Wegman dot product over the two
 * 32-bit limbs of x, in the field Z_P:
 *   hash((a1,a2,b), x) = (a1*(x mod 2^32) + a2*(x >> 32) + b) mod P. */
uint64_t or_hash(const uint64_t c[3], uint64_t x) {
  u128 lo = (u128)(x & 0xFFFFFFFFULL);
  u128 hi = (u128)(x >> 32);
  u128 v = (u128)c[0] * lo + (u128)c[1] * hi + (u128)c[2];
  return (uint64_t)(v % (u128)OR_P);
}

/* ------------------------------------------------------ fingerprint (R5)
 * PAPER.md:719-722 leaves the sequence hash open ("somewhat complicated ...
 * outside the scope of this paper").  Reading R5: Horner evaluation over
 * little-endian u32 words (zero padded) in Z_P at point r, plus the length:
 *   acc = 0; for each word w: acc = (acc + w) * r mod P;  fp = (acc + len) mod P */
uint64_t or_fingerprint(const uint8_t* s, uint64_t len, uint64_t r) {
  uint64_t acc = 0;
  uint64_t nwords = (len + 3) / 4;
  for (uint64_t i = 0; i < nwords; i++) {
    uint64_t w = 0;
    for (uint64_t k = 0; k < 4; k++) {
      uint64_t p = 4 * i + k;
      if (p < len) w |= (uint64_t)s[p] << (8 * k);
    }
    acc = (uint64_t)((((u128)acc + (u128)w) * (u128)r) % (u128)OR_P);
  }
  return (uint64_t)(((u128)acc + (u128)len) % (u128)OR_P);
}

/* --------------------------------------------- Fig. 1 vocabulary
 * hist n is vs: n bins initialised to 0, vs[i] added into bin is[i]
 * (PAPER.md:211-214). */
void or_hist(uint64_t nbins, const uint64_t* is, const uint64_t* vs, uint64_t m,
             uint64_t* out) {
  for (uint64_t b = 0; b < nbins; b++) out[b] = 0;
  for (uint64_t i = 0; i < m; i++) out[is[i]] += vs[i];
}

/* presum: prefix sum.  Reading R2: EXCLUSIVE, with
 * out[n] = the total (so out has n+1 entries). */
void or_presum(const uint64_t* x, uint64_t n, uint64_t* out) {
  uint64_t acc = 0;
  for (uint64_t i = 0; i < n; i++) {
    out[i] = acc;
    acc += x[i];
  }
  out[n] = acc;
}

/* groupby m is vs: an irregular [m][]alpha, elements kept
 * in input order within each group.  Represented flat: group g is
 * out_items[out_start[g] .. out_start[g+1]). Items are indices into vs. */
void or_groupby(uint64_t m, const uint64_t* is, uint64_t n, uint64_t* out_start,
                uint64_t* out_items) {
  uint64_t* ones = (uint64_t*)malloc(sizeof(uint64_t) * (n ? n : 1));
  uint64_t* size = (uint64_t*)malloc(sizeof(uint64_t) * (m ? m : 1));
  uint64_t* fill = (uint64_t*)malloc(sizeof(uint64_t) * (m ? m : 1));
  for (uint64_t i = 0; i < n; i++) ones[i] = 1;
  or_hist(m, is, ones, n, size);
  or_presum(size, m, out_start);
  for (uint64_t g = 0; g < m; g++) fill[g] = out_start[g];
  for (uint64_t i = 0; i < n; i++) out_items[fill[is[i]]++] = i;
  free(ones);
  free(size);
  free(fill);
}

/* ------------------------------------------------- level two
 * hashes cs keys = map ((mod m^2) . hash cs) keys
 * collision hs   = (or . map (>1) . hist m^2 hs) (rep m 1)
 * make2 keys     = redraw cs until not (collision (hashes cs keys))
 *                  (PAPER.md:286-292); the k-th redraw uses derive(seed,2,b,k)
 *                  (R6) and the first success is kept (R13), capped at 256
 *                  attempts (R8).                                            */
static int or_collision(const uint64_t* hs, uint64_t m) {
  uint64_t m2 = m * m;
  uint64_t* bins = (uint64_t*)malloc(sizeof(uint64_t) * m2);
  uint64_t* ones = (uint64_t*)malloc(sizeof(uint64_t) * m);
  for (uint64_t i = 0; i < m; i++) ones[i] = 1;
  or_hist(m2, hs, ones, m, bins);
  int any = 0;
  for (uint64_t j = 0; j < m2; j++) any = any || (bins[j] > 1);
  free(bins);
  free(ones);
  return any;
}

/* Returns the attempt index t (< OR_T2_CAP) or -1 when exhausted; fills
 * hs_out with the level-two slot of every key under the returned t. */
static int or_make2(uint64_t seed, uint64_t bucket, const uint64_t* keys, uint64_t m,
                    uint64_t* hs_out) {
  uint64_t m2 = m * m;
  for (uint32_t t = 0; t < OR_T2_CAP; t++) {
    uint64_t cs[3];
    or_derive(seed, 2, bucket, t, cs);
    for (uint64_t i = 0; i < m; i++) hs_out[i] = or_hash(cs, keys[i]) % m2;
    if (!or_collision(hs_out, m)) return (int)t;
  }
  return -1;
}

/* ---------------------------------------------------------------- tables */
typedef struct {
  uint32_t magic, spec_version, key_kind, reserved;
  uint64_t n, S, seed;
  uint32_t t1, t0;
  uint64_t ctx_bytes;
} or_header; /* 56 bytes */

typedef struct { uint64_t key, value; } or_slot_u64;
typedef struct { uint64_t fp, value, ctx_off; uint32_t len, reserved; } or_slot_bytes;

#define OR_DIR(soff, s, t) ((uint64_t)(soff) | ((uint64_t)(s) << 40) | ((uint64_t)(t) << 56))

/* Level one for a fixed attempt t1 (§2.2 g/shape):
 *   const  = derive(seed,1,0,t1)
 *   hashes = map ((mod n) . hash const) keys
 *   shape  = hist n hashes (rep n 1)                  (unsquared sizes, R1)
 * Returns S = sum (map (^2) shape). */
static uint64_t or_level1(uint64_t seed, uint32_t t1, const uint64_t* keys, uint64_t n,
                          uint64_t* hashes, uint64_t* shape) {
  uint64_t c1[3];
  or_derive(seed, 1, 0, t1, c1);
  for (uint64_t i = 0; i < n; i++) hashes[i] = or_hash(c1, keys[i]) % n;
  uint64_t* ones = (uint64_t*)malloc(sizeof(uint64_t) * n);
  for (uint64_t i = 0; i < n; i++) ones[i] = 1;
  or_hist(n, hashes, ones, n, shape);
  free(ones);
  uint64_t S = 0;
  for (uint64_t b = 0; b < n; b++) S += shape[b] * shape[b];
  return S;
}

/*
 * The shared FKS core used by both key kinds.  `hkeys` are the integers that
 * are hashed (the u64 keys, or the fingerprints for strings).  `same_key(i,j)`
 * decides whether two items with equal hkeys are the same key (always true
 * for u64; byte comparison for strings).  Emits dir[n] and the member slot of
 * every item (member_slot[i] = global slot index).  Status per §8(c) step 3:
 * duplicate -> DUPLICATE_KEY, else equal-hkey-different-key -> *fp_collision,
 * else a bucket reaching 256 attempts -> SEED_EXHAUSTED.
 */
typedef int (*or_same_fn)(void* ctx, uint64_t i, uint64_t j);

static int or_fks(uint64_t seed, const uint64_t* hkeys, uint64_t n, or_same_fn same,
                  void* same_ctx, uint64_t* dir, uint64_t* member_slot, uint64_t* S_out,
                  uint32_t* t1_out, int* fp_collision) {
  uint64_t* hashes = (uint64_t*)malloc(sizeof(uint64_t) * n);
  uint64_t* shape = (uint64_t*)malloc(sizeof(uint64_t) * n);
  uint64_t* sq = (uint64_t*)malloc(sizeof(uint64_t) * n);
  uint64_t* offsets = (uint64_t*)malloc(sizeof(uint64_t) * (n + 1));
  uint64_t* gstart = (uint64_t*)malloc(sizeof(uint64_t) * (n + 1));
  uint64_t* gitems = (uint64_t*)malloc(sizeof(uint64_t) * n);
  if (!hashes || !shape || !sq || !offsets || !gstart || !gitems) return OR_ERR_OOM;

  /* Step 1 — level one with the space bound (R7): first t1 with S <= 4n. */
  uint32_t t1 = 0;
  uint64_t S = 0;
  for (;; t1++) {
    if (t1 >= OR_T1_CAP) {
      free(hashes); free(shape); free(sq); free(offsets); free(gstart); free(gitems);
      return OR_ERR_SEED_EXHAUSTED;
    }
    S = or_level1(seed, t1, hkeys, n, hashes, shape);
    if (S <= 4 * n) break;
  }

  /* Step 2 — offsets = presum (map (^2) shape)  (R1, R2);
   * groupby n hashes keys.          */
  for (uint64_t b = 0; b < n; b++) sq[b] = shape[b] * shape[b];
  or_presum(sq, n, offsets);
  or_groupby(n, hashes, n, gstart, gitems);

  /* Step 3 — map make2 over the groups. */
  int dup = 0, exhausted = 0, fpcoll = 0;
  uint64_t* bkeys = (uint64_t*)malloc(sizeof(uint64_t) * n);
  uint64_t* bhs = (uint64_t*)malloc(sizeof(uint64_t) * n);
  for (uint64_t b = 0; b < n; b++) {
    uint64_t s = shape[b];
    uint64_t soff = offsets[b];
    const uint64_t* items = gitems + gstart[b];
    if (s == 0) { /* R9: empty bucket stores just its offset */
      dir[b] = OR_DIR(soff, 0, 0);
      continue;
    }
    /* equal keys can never be separated: record and skip (§8(c) step 3) */
    int skip = 0;
    for (uint64_t i = 0; i < s; i++)
      for (uint64_t j = i + 1; j < s; j++)
        if (hkeys[items[i]] == hkeys[items[j]]) {
          if (same(same_ctx, items[i], items[j])) dup = 1; else fpcoll = 1;
          skip = 1;
        }
    if (skip) { dir[b] = OR_DIR(soff, s, 0); continue; }
    if (s == 1) { /* R12: singleton, t = 0, slot = soff, level two not hashed */
      member_slot[items[0]] = soff;
      dir[b] = OR_DIR(soff, 1, 0);
      continue;
    }
    for (uint64_t i = 0; i < s; i++) bkeys[i] = hkeys[items[i]];
    int t = or_make2(seed, b, bkeys, s, bhs);
    if (t < 0) { exhausted = 1; dir[b] = OR_DIR(soff, s, 0); continue; }
    for (uint64_t i = 0; i < s; i++) member_slot[items[i]] = soff + bhs[i];
    dir[b] = OR_DIR(soff, s, (uint64_t)t);
  }
  free(bkeys); free(bhs);
  free(hashes); free(shape); free(sq); free(offsets); free(gstart); free(gitems);
  *S_out = S;
  *t1_out = t1;
  *fp_collision = fpcoll;
  if (dup) return OR_ERR_DUPLICATE_KEY;
  if (fpcoll) return OR_OK; /* caller redraws t0 */
  if (exhausted) return OR_ERR_SEED_EXHAUSTED;
  return OR_OK;
}

static int or_same_u64(void* ctx, uint64_t i, uint64_t j) {
  (void)ctx; (void)i; (void)j;
  return 1; /* equal u64 keys are the same key */
}

/* Fill the table (R10): every key at h k, every unused slot
 * of a non-empty bucket gets the bucket member at its lowest occupied slot
 * (value 0).  `occupant[j]` = item index + 1 at slot j, 0 if unused. */
static void or_occupancy(const uint64_t* dir, uint64_t nb, const uint64_t* member_slot,
                         uint64_t nkeys, uint64_t S, uint64_t* occupant) {
  for (uint64_t j = 0; j < S; j++) occupant[j] = 0;
  for (uint64_t i = 0; i < nkeys; i++) occupant[member_slot[i]] = i + 1;
  for (uint64_t b = 0; b < nb; b++) {
    uint64_t s = (dir[b] >> 40) & 0xFFFF;
    if (s == 0) continue;
    uint64_t soff = dir[b] & ((1ULL << 40) - 1);
    uint64_t lowest = 0;
    for (uint64_t j = soff; j < soff + s * s; j++)
      if (occupant[j]) { lowest = occupant[j]; break; }
    for (uint64_t j = soff; j < soff + s * s; j++)
      if (!occupant[j]) occupant[j] = lowest | (1ULL << 63); /* filler mark */
  }
}

/* ------------------------------------------------------- u64 build / lookup */
typedef struct {
  or_header hdr;
  uint64_t* dir;   /* n        */
  void* slots;     /* S slots  */
  uint8_t* ctx;    /* strings: the map's copy of its key context          */
} or_table;

void or_table_free(or_table* t) {
  if (!t) return;
  free(t->dir);
  free(t->slots);
  free(t->ctx);
  free(t);
}

/* from_array_nodup for u64 keys. */
int or_build_u64(const uint64_t* keys, const uint64_t* vals, uint64_t n, uint64_t seed,
                 or_table** out) {
  *out = NULL;
  if (n == 0) return OR_ERR_EMPTY;
  if (!keys || !vals) return OR_ERR_INVALID_ARG;
  if (n > OR_MAX_N) return OR_ERR_TOO_LARGE;
  uint64_t* dir = (uint64_t*)malloc(sizeof(uint64_t) * n);
  uint64_t* mslot = (uint64_t*)malloc(sizeof(uint64_t) * n);
  if (!dir || !mslot) return OR_ERR_OOM;
  uint64_t S = 0;
  uint32_t t1 = 0;
  int fpc = 0;
  int st = or_fks(seed, keys, n, or_same_u64, NULL, dir, mslot, &S, &t1, &fpc);
  if (st != OR_OK) { free(dir); free(mslot); return st; }
  uint64_t* occ = (uint64_t*)malloc(sizeof(uint64_t) * S);
  or_slot_u64* slots = (or_slot_u64*)calloc(S ? S : 1, sizeof(or_slot_u64));
  or_occupancy(dir, n, mslot, n, S, occ);
  for (uint64_t j = 0; j < S; j++) {
    uint64_t o = occ[j];
    uint64_t i = (o & ~(1ULL << 63)) - 1;
    slots[j].key = keys[i];
    slots[j].value = (o >> 63) ? 0 : vals[i];
  }
  free(occ);
  free(mslot);
  or_table* t = (or_table*)calloc(1, sizeof(or_table));
  t->hdr.magic = OR_MAGIC;
  t->hdr.spec_version = OR_SPEC_VERSION;
  t->hdr.key_kind = 0;
  t->hdr.n = n;
  t->hdr.S = S;
  t->hdr.seed = seed;
  t->hdr.t1 = t1;
  t->hdr.t0 = 0;
  t->hdr.ctx_bytes = 0;
  t->dir = dir;
  t->slots = slots;
  *out = t;
  return OR_OK;
}

/* lookup (membership test PAPER.md:244-247):
 * b = g q; probe dir[b]; s = 0 -> none; j = offsets[b] + (hash consts[b] q
 * mod s^2) (s = 1: no level-two hash, R12); hit iff arr[j] = q. */
void or_lookup_u64(const or_table* t, const uint64_t* q, uint64_t nq, uint64_t* out_vals,
                   uint8_t* out_found) {
  uint64_t n = t->hdr.n;
  uint64_t c1[3];
  or_derive(t->hdr.seed, 1, 0, t->hdr.t1, c1);
  const or_slot_u64* slots = (const or_slot_u64*)t->slots;
  for (uint64_t i = 0; i < nq; i++) {
    uint64_t b = or_hash(c1, q[i]) % n;
    uint64_t d = t->dir[b];
    uint64_t s = (d >> 40) & 0xFFFF;
    uint64_t soff = d & ((1ULL << 40) - 1);
    uint64_t v = 0;
    uint8_t f = 0;
    if (s != 0) {
      uint64_t j = soff;
      if (s > 1) {
        uint64_t cs[3];
        or_derive(t->hdr.seed, 2, b, (uint32_t)(d >> 56), cs);
        j += or_hash(cs, q[i]) % (s * s);
      }
      if (slots[j].key == q[i]) { v = slots[j].value; f = 1; }
    }
    if (out_vals) out_vals[i] = v;
    if (out_found) out_found[i] = f;
  }
}

/* ------------------------------------------------------ byte-string keys
 * Keys are slices (offset, length) of one flat context,
 * given as CSR offsets[n+1]; the map stores a copy of its context
 * bytes[offsets[0]..offsets[n]).                        */
typedef struct {
  const uint8_t* bytes;
  const uint64_t* offsets;
} or_strctx;

static int or_same_bytes(void* vctx, uint64_t i, uint64_t j) {
  or_strctx* c = (or_strctx*)vctx;
  uint64_t li = c->offsets[i + 1] - c->offsets[i];
  uint64_t lj = c->offsets[j + 1] - c->offsets[j];
  if (li != lj) return 0;
  return memcmp(c->bytes + c->offsets[i], c->bytes + c->offsets[j], li) == 0;
}

int or_build_bytes(const uint8_t* bytes, const uint64_t* offsets, const uint64_t* vals,
                   uint64_t n, uint64_t seed, or_table** out) {
  *out = NULL;
  if (n == 0) return OR_ERR_EMPTY;
  if (!offsets || !vals) return OR_ERR_INVALID_ARG;
  if (n > OR_MAX_N) return OR_ERR_TOO_LARGE;
  for (uint64_t i = 0; i < n; i++) {
    if (offsets[i + 1] < offsets[i]) return OR_ERR_INVALID_ARG;
    if (offsets[i + 1] - offsets[i] > 65535) return OR_ERR_TOO_LARGE;
  }
  uint64_t* fp = (uint64_t*)malloc(sizeof(uint64_t) * n);
  uint64_t* dir = (uint64_t*)malloc(sizeof(uint64_t) * n);
  uint64_t* mslot = (uint64_t*)malloc(sizeof(uint64_t) * n);
  or_strctx sc = {bytes, offsets};
  uint64_t S = 0;
  uint32_t t1 = 0, t0 = 0;
  /* §8(c) step 5: wrap steps 1-3 in a loop over t0 (fingerprint redraws). */
  for (;; t0++) {
    if (t0 >= OR_T0_CAP) { free(fp); free(dir); free(mslot); return OR_ERR_FP_EXHAUSTED; }
    uint64_t c0[3];
    or_derive(seed, 0, 0, t0, c0);
    uint64_t r = c0[0];
    for (uint64_t i = 0; i < n; i++)
      fp[i] = or_fingerprint(bytes + offsets[i], offsets[i + 1] - offsets[i], r);
    int fpc = 0;
    int st = or_fks(seed, fp, n, or_same_bytes, &sc, dir, mslot, &S, &t1, &fpc);
    if (st != OR_OK) { free(fp); free(dir); free(mslot); return st; }
    if (!fpc) break;
  }
  uint64_t* occ = (uint64_t*)malloc(sizeof(uint64_t) * S);
  or_slot_bytes* slots = (or_slot_bytes*)calloc(S ? S : 1, sizeof(or_slot_bytes));
  or_occupancy(dir, n, mslot, n, S, occ);
  for (uint64_t j = 0; j < S; j++) {
    uint64_t o = occ[j];
    uint64_t i = (o & ~(1ULL << 63)) - 1;
    slots[j].fp = fp[i];
    slots[j].value = (o >> 63) ? 0 : vals[i];
    slots[j].ctx_off = offsets[i] - offsets[0];
    slots[j].len = (uint32_t)(offsets[i + 1] - offsets[i]);
    slots[j].reserved = 0;
  }
  free(occ);
  free(mslot);
  free(fp);
  uint64_t cb = offsets[n] - offsets[0];
  or_table* t = (or_table*)calloc(1, sizeof(or_table));
  t->ctx = (uint8_t*)malloc(cb ? cb : 1);
  if (cb) memcpy(t->ctx, bytes + offsets[0], cb);
  t->hdr.magic = OR_MAGIC;
  t->hdr.spec_version = OR_SPEC_VERSION;
  t->hdr.key_kind = 1;
  t->hdr.n = n;
  t->hdr.S = S;
  t->hdr.seed = seed;
  t->hdr.t1 = t1;
  t->hdr.t0 = t0;
  t->hdr.ctx_bytes = cb;
  t->dir = dir;
  t->slots = slots;
  *out = t;
  return OR_OK;
}

/* String lookup: the needle is hashed with the map's fingerprint point and
 * compared by content against the map's own context (PAPER.md:580-581,
 * 780-789: needle and haystack each come with their own context). */
void or_lookup_bytes(const or_table* t, const uint8_t* qbytes, const uint64_t* qoffsets,
                     uint64_t nq, uint64_t* out_vals, uint8_t* out_found) {
  uint64_t n = t->hdr.n;
  uint64_t c0[3], c1[3];
  or_derive(t->hdr.seed, 0, 0, t->hdr.t0, c0);
  or_derive(t->hdr.seed, 1, 0, t->hdr.t1, c1);
  const or_slot_bytes* slots = (const or_slot_bytes*)t->slots;
  for (uint64_t i = 0; i < nq; i++) {
    const uint8_t* q = qbytes + qoffsets[i];
    uint64_t len = qoffsets[i + 1] - qoffsets[i];
    uint64_t f = or_fingerprint(q, len, c0[0]);
    uint64_t b = or_hash(c1, f) % n;
    uint64_t d = t->dir[b];
    uint64_t s = (d >> 40) & 0xFFFF;
    uint64_t soff = d & ((1ULL << 40) - 1);
    uint64_t v = 0;
    uint8_t hit = 0;
    if (s != 0) {
      uint64_t j = soff;
      if (s > 1) {
        uint64_t cs[3];
        or_derive(t->hdr.seed, 2, b, (uint32_t)(d >> 56), cs);
        j += or_hash(cs, f) % (s * s);
      }
      const or_slot_bytes* sl = &slots[j];
      if (sl->fp == f && sl->len == len && memcmp(t->ctx + sl->ctx_off, q, len) == 0) {
        v = sl->value;
        hit = 1;
      }
    }
    if (out_vals) out_vals[i] = v;
    if (out_found) out_found[i] = hit;
  }
}

/* --------------------------------------------------------- accessors (ctypes) */
void or_table_header(const or_table* t, or_header* out) { *out = t->hdr; }
const uint64_t* or_table_dir(const or_table* t) { return t->dir; }
const void* or_table_slots(const or_table* t) { return t->slots; }
const uint8_t* or_table_ctx(const or_table* t) { return t->ctx; }
uint64_t or_sizeof_header(void) { return sizeof(or_header); }

/* Level-one statistics for a fixed t1 (used by the closed-form pins). */
uint64_t or_level1_S(const uint64_t* keys, uint64_t n, uint64_t seed, uint32_t t1,
                     uint64_t* shape_out) {
  uint64_t* hashes = (uint64_t*)malloc(sizeof(uint64_t) * n);
  uint64_t S = or_level1(seed, t1, keys, n, hashes, shape_out);
  free(hashes);
  return S;
}

/* ------------------------------------------------------------ shards
 * The bucket-range shard of the logical table:
 * buckets [b_lo, b_hi) of g k = hash(derive(seed,1,0,t1), k) mod n_global,
 * built from exactly the keys whose bucket falls in the range, with the same
 * steps 2-3 as or_fks (presum of s^2 over the range, make2 per bucket, R10
 * filler).  dir has b_hi-b_lo entries with soff relative to the shard;
 * concatenating the shards of all ranks, each soff shifted by the slot count of
 * the ranks before it, gives the single table.  No level-1 loop: the caller
 * checks the GLOBAL bound sum S_r <= 4 n_global (R7). */
int or_build_u64_shard(const uint64_t* keys, const uint64_t* vals, uint64_t n_recv, uint64_t n_global,
                       uint64_t b_lo, uint64_t b_hi, uint32_t t1, uint64_t seed, or_table** out) {
  *out = NULL;
  if (n_global == 0) return OR_ERR_EMPTY;
  if (b_hi < b_lo || b_hi > n_global) return OR_ERR_INVALID_ARG;
  uint64_t nb = b_hi - b_lo;
  uint64_t c1[3];
  or_derive(seed, 1, 0, t1, c1);
  uint64_t* lb = (uint64_t*)malloc(sizeof(uint64_t) * (n_recv ? n_recv : 1));
  for (uint64_t i = 0; i < n_recv; i++) {
    uint64_t g = or_hash(c1, keys[i]) % n_global;
    if (g < b_lo || g >= b_hi) { free(lb); return OR_ERR_INVALID_ARG; }
    lb[i] = g - b_lo;
  }
  uint64_t* shape = (uint64_t*)calloc(nb ? nb : 1, sizeof(uint64_t));
  uint64_t* ones = (uint64_t*)malloc(sizeof(uint64_t) * (n_recv ? n_recv : 1));
  for (uint64_t i = 0; i < n_recv; i++) ones[i] = 1;
  or_hist(nb, lb, ones, n_recv, shape);
  free(ones);
  uint64_t* sq = (uint64_t*)malloc(sizeof(uint64_t) * (nb ? nb : 1));
  uint64_t* offsets = (uint64_t*)malloc(sizeof(uint64_t) * (nb + 1));
  uint64_t* gstart = (uint64_t*)malloc(sizeof(uint64_t) * (nb + 1));
  uint64_t* gitems = (uint64_t*)malloc(sizeof(uint64_t) * (n_recv ? n_recv : 1));
  for (uint64_t b = 0; b < nb; b++) sq[b] = shape[b] * shape[b];
  or_presum(sq, nb, offsets);
  or_groupby(nb, lb, n_recv, gstart, gitems);
  uint64_t S = offsets[nb];
  uint64_t* dir = (uint64_t*)malloc(sizeof(uint64_t) * (nb ? nb : 1));
  uint64_t* mslot = (uint64_t*)malloc(sizeof(uint64_t) * (n_recv ? n_recv : 1));
  uint64_t* bkeys = (uint64_t*)malloc(sizeof(uint64_t) * (n_recv ? n_recv : 1));
  uint64_t* bhs = (uint64_t*)malloc(sizeof(uint64_t) * (n_recv ? n_recv : 1));
  int dup = 0, exhausted = 0, bound = 0;
  for (uint64_t b = 0; b < nb; b++) {
    uint64_t s = shape[b], soff = offsets[b];
    const uint64_t* items = gitems + gstart[b];
    dir[b] = OR_DIR(soff, s, 0);
    if (s == 0) continue;
    if (s * s > 4 * n_global) { bound = 1; continue; }
    int skip = 0;
    for (uint64_t i = 0; i < s; i++)
      for (uint64_t j = i + 1; j < s; j++)
        if (keys[items[i]] == keys[items[j]]) { dup = 1; skip = 1; }
    if (skip) continue;
    if (s == 1) { mslot[items[0]] = soff; continue; }
    for (uint64_t i = 0; i < s; i++) bkeys[i] = keys[items[i]];
    int t = or_make2(seed, b_lo + b, bkeys, s, bhs);
    if (t < 0) { exhausted = 1; continue; }
    for (uint64_t i = 0; i < s; i++) mslot[items[i]] = soff + bhs[i];
    dir[b] = OR_DIR(soff, s, (uint64_t)t);
  }
  free(bkeys); free(bhs); free(lb); free(shape); free(sq); free(offsets); free(gstart); free(gitems);
  or_table* tb = (or_table*)calloc(1, sizeof(or_table));
  tb->hdr.magic = OR_MAGIC;
  tb->hdr.spec_version = OR_SPEC_VERSION;
  tb->hdr.n = nb;
  tb->hdr.S = S;
  tb->hdr.seed = seed;
  tb->hdr.t1 = t1;
  tb->dir = dir;
  if (!dup && !exhausted && !bound && S <= 4 * n_global) {
    uint64_t* occ = (uint64_t*)malloc(sizeof(uint64_t) * (S ? S : 1));
    or_slot_u64* slots = (or_slot_u64*)calloc(S ? S : 1, sizeof(or_slot_u64));
    or_occupancy(dir, nb, mslot, n_recv, S, occ);
    for (uint64_t j = 0; j < S; j++) {
      uint64_t o = occ[j];
      uint64_t i = (o & ~(1ULL << 63)) - 1;
      slots[j].key = keys[i];
      slots[j].value = (o >> 63) ? 0 : vals[i];
    }
    free(occ);
    tb->slots = slots;
  } else {
    tb->slots = calloc(1, sizeof(or_slot_u64));
    tb->hdr.S = (bound && S <= 4 * n_global) ? 4 * n_global + 1 : S;
  }
  free(mslot);
  *out = tb;
  if (dup) return OR_ERR_DUPLICATE_KEY;
  if (exhausted) return OR_ERR_SEED_EXHAUSTED;
  return OR_OK;
}

/* g k = hash(derive(seed,1,0,t1), k) mod n for every key: used
 * by the full-size tests to select the keys of sampled bucket ranges. */
void or_level1_buckets(const uint64_t* keys, uint64_t m, uint64_t n, uint64_t seed, uint32_t t1, uint64_t* out) {
  uint64_t c1[3];
  or_derive(seed, 1, 0, t1, c1);
  for (uint64_t i = 0; i < m; i++) out[i] = or_hash(c1, keys[i]) % n;
}

/* ------------------------------------------- T-thread variant (CPU baseline)
 * SURVEY §8(d) "Oracle timing": the same construction with the level-1
 * buckets split into T contiguous ranges, one thread per range — the
 * multi-GPU partitioning (§8(e)) on host threads.  Steps, in the order of
 * or_fks: level one (hash every key, shape by atomic increments, S; redraw
 * t1 while S > 4n, R7); offsets = presum(shape^2) and the group starts; the
 * keys grouped by bucket (any order inside a bucket: make2's first successful
 * t, the member slots and the lowest-slot filler do not depend on it); then
 * each thread runs make2 (the same or_make2) over its bucket range and writes
 * that range's directory entries and slots.  Same table as or_build_u64 (a
 * test checks the bytes); timing only, never called by the product. */
#include <pthread.h>

typedef struct {
  const uint64_t* keys; const uint64_t* vals; uint64_t n, seed;
  uint32_t t1; int T, id;
  uint64_t* hashes; uint32_t* shape; uint64_t* offs; uint64_t* gstart; uint64_t* gcur; uint64_t* gitems;
  uint64_t* dir; or_slot_u64* slots;
  uint64_t partS; int dup, exhausted;
} or_mt_arg;

static void* or_mt_level1(void* p) {
  or_mt_arg* a = (or_mt_arg*)p;
  uint64_t c1[3];
  or_derive(a->seed, 1, 0, a->t1, c1);
  uint64_t lo = a->n * a->id / a->T, hi = a->n * (a->id + 1) / a->T;
  for (uint64_t i = lo; i < hi; i++) {
    a->hashes[i] = or_hash(c1, a->keys[i]) % a->n;
    __atomic_fetch_add(&a->shape[a->hashes[i]], 1u, __ATOMIC_RELAXED);
  }
  return NULL;
}

static void* or_mt_sq(void* p) {
  or_mt_arg* a = (or_mt_arg*)p;
  uint64_t lo = a->n * a->id / a->T, hi = a->n * (a->id + 1) / a->T, S = 0;
  for (uint64_t b = lo; b < hi; b++) S += (uint64_t)a->shape[b] * a->shape[b];
  a->partS = S;
  return NULL;
}

static void* or_mt_group(void* p) {
  or_mt_arg* a = (or_mt_arg*)p;
  uint64_t lo = a->n * a->id / a->T, hi = a->n * (a->id + 1) / a->T;
  for (uint64_t i = lo; i < hi; i++) {
    uint64_t pos = __atomic_fetch_add(&a->gcur[a->hashes[i]], 1ull, __ATOMIC_RELAXED);
    a->gitems[pos] = i;
  }
  return NULL;
}

static void* or_mt_level2(void* p) {
  or_mt_arg* a = (or_mt_arg*)p;
  uint64_t lo = a->n * a->id / a->T, hi = a->n * (a->id + 1) / a->T;
  uint64_t* bkeys = (uint64_t*)malloc(sizeof(uint64_t) * 64);
  uint64_t* bhs = (uint64_t*)malloc(sizeof(uint64_t) * 64);
  uint64_t cap = 64;
  for (uint64_t b = lo; b < hi; b++) {
    uint64_t s = a->shape[b], soff = a->offs[b];
    const uint64_t* items = a->gitems + a->gstart[b];
    if (s == 0) { a->dir[b] = OR_DIR(soff, 0, 0); continue; }
    int skip = 0;
    for (uint64_t i = 0; i < s && !skip; i++)
      for (uint64_t j = i + 1; j < s; j++)
        if (a->keys[items[i]] == a->keys[items[j]]) { a->dup = 1; skip = 1; break; }
    if (skip) { a->dir[b] = OR_DIR(soff, s, 0); continue; }
    if (s > cap) {
      cap = s;
      bkeys = (uint64_t*)realloc(bkeys, sizeof(uint64_t) * cap);
      bhs = (uint64_t*)realloc(bhs, sizeof(uint64_t) * cap);
    }
    int t = 0;
    if (s == 1) bhs[0] = 0; /* R12 */
    else {
      for (uint64_t i = 0; i < s; i++) bkeys[i] = a->keys[items[i]];
      t = or_make2(a->seed, b, bkeys, s, bhs);
      if (t < 0) { a->exhausted = 1; a->dir[b] = OR_DIR(soff, s, 0); continue; }
    }
    a->dir[b] = OR_DIR(soff, s, (uint64_t)t);
    /* the bucket's slots (R10): members at h, the rest
     * the member at the lowest occupied slot with value 0 */
    uint64_t low = 0;
    for (uint64_t i = 1; i < s; i++) if (bhs[i] < bhs[low]) low = i;
    for (uint64_t j = 0; j < s * s; j++) {
      a->slots[soff + j].key = a->keys[items[low]];
      a->slots[soff + j].value = 0;
    }
    for (uint64_t i = 0; i < s; i++) {
      a->slots[soff + bhs[i]].key = a->keys[items[i]];
      a->slots[soff + bhs[i]].value = a->vals[items[i]];
    }
  }
  free(bkeys);
  free(bhs);
  return NULL;
}

static void or_mt_run(or_mt_arg* args, int T, void* (*fn)(void*)) {
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * T);
  for (int i = 0; i < T; i++) pthread_create(&th[i], NULL, fn, &args[i]);
  for (int i = 0; i < T; i++) pthread_join(th[i], NULL);
  free(th);
}

int or_build_u64_mt(const uint64_t* keys, const uint64_t* vals, uint64_t n, uint64_t seed, int T,
                    or_table** out) {
  *out = NULL;
  if (n == 0) return OR_ERR_EMPTY;
  if (!keys || !vals || T < 1) return OR_ERR_INVALID_ARG;
  if (n > OR_MAX_N) return OR_ERR_TOO_LARGE;
  uint64_t* hashes = (uint64_t*)malloc(sizeof(uint64_t) * n);
  uint32_t* shape = (uint32_t*)malloc(sizeof(uint32_t) * n);
  uint64_t* offs = (uint64_t*)malloc(sizeof(uint64_t) * (n + 1));
  uint64_t* gstart = (uint64_t*)malloc(sizeof(uint64_t) * (n + 1));
  uint64_t* gcur = (uint64_t*)malloc(sizeof(uint64_t) * n);
  uint64_t* gitems = (uint64_t*)malloc(sizeof(uint64_t) * n);
  uint64_t* dir = (uint64_t*)malloc(sizeof(uint64_t) * n);
  or_mt_arg* args = (or_mt_arg*)calloc(T, sizeof(or_mt_arg));
  if (!hashes || !shape || !offs || !gstart || !gcur || !gitems || !dir || !args) return OR_ERR_OOM;
  for (int i = 0; i < T; i++) {
    args[i] = (or_mt_arg){keys, vals, n, seed, 0, T, i, hashes, shape, offs, gstart, gcur, gitems, dir, NULL, 0, 0, 0};
  }
  uint32_t t1 = 0;
  uint64_t S = 0;
  for (;; t1++) {
    if (t1 >= OR_T1_CAP) {
      free(hashes); free(shape); free(offs); free(gstart); free(gcur); free(gitems); free(dir); free(args);
      return OR_ERR_SEED_EXHAUSTED;
    }
    memset(shape, 0, sizeof(uint32_t) * n);
    for (int i = 0; i < T; i++) args[i].t1 = t1;
    or_mt_run(args, T, or_mt_level1);
    or_mt_run(args, T, or_mt_sq);
    S = 0;
    for (int i = 0; i < T; i++) S += args[i].partS;
    if (S <= 4 * n) break;
  }
  /* presums (sequential: one pass over n) */
  uint64_t acc = 0, accg = 0;
  for (uint64_t b = 0; b < n; b++) {
    offs[b] = acc;
    gstart[b] = accg;
    gcur[b] = accg;
    acc += (uint64_t)shape[b] * shape[b];
    accg += shape[b];
  }
  offs[n] = acc;
  gstart[n] = accg;
  or_mt_run(args, T, or_mt_group);
  or_slot_u64* slots = (or_slot_u64*)calloc(S ? S : 1, sizeof(or_slot_u64));
  for (int i = 0; i < T; i++) args[i].slots = slots;
  or_mt_run(args, T, or_mt_level2);
  int dup = 0, exhausted = 0;
  for (int i = 0; i < T; i++) { dup |= args[i].dup; exhausted |= args[i].exhausted; }
  free(hashes); free(shape); free(offs); free(gstart); free(gcur); free(gitems); free(args);
  if (dup || exhausted) { free(dir); free(slots); return dup ? OR_ERR_DUPLICATE_KEY : OR_ERR_SEED_EXHAUSTED; }
  or_table* t = (or_table*)calloc(1, sizeof(or_table));
  t->hdr.magic = OR_MAGIC;
  t->hdr.spec_version = OR_SPEC_VERSION;
  t->hdr.key_kind = 0;
  t->hdr.n = n;
  t->hdr.S = S;
  t->hdr.seed = seed;
  t->hdr.t1 = t1;
  t->dir = dir;
  t->slots = slots;
  *out = t;
  return OR_OK;
}
