// rounds.cu — the paper's sortless, round-based construction as a GPU
// ablation (HM_FLAG_ROUNDS, u64 keys).
//
// PAPER.md:443-499 (§2.5 "Sortless Construction") builds level two without a
// sort: every key carries the rank of its non-empty level-1 bucket
// (`koffsets`), and `segmake'_2` runs rounds over flat
// arrays:
//   segrandom     constants for every still-active bucket
//   seghashes     o' + hash(cs, key) mod s^2, o' = presum of s^2
//                 over the active buckets
//   segcollisions hist over the flat slot space, OR per bucket
//   segresult     finished buckets keep their constants
//   keys'         keys of colliding buckets, renumbered by the
//                 presum of the collision flags; recurse.
// Each step here is one grid-wide kernel over global memory (atomics for
// `hist`, device scans for `presum`, warp-aggregated appends for `filter`);
// the host reads two counters per round to size the next one (the recursion
// depth is data dependent).  Round r tries attempt t = r for every active
// bucket, so a bucket finishes at its first successful t: the table is the
// canonical one (R13), identical to the default build's — the same dir, cdir
// and slots, and the same lookup kernels read it.
//
// This is the design the default build (build.cu: partition, then one CTA per
// 2048 buckets searching in shared memory) replaces; it exists to measure the
// difference.  Not a product path: no shards, no byte keys.
#include <algorithm>
#include <cstdio>
#include <vector>

#include "hm_internal.cuh"

namespace hm {

hm_status scan_excl(uint64_t* v, uint64_t n, uint64_t* sums, cudaStream_t st);  // dedup.cu
uint64_t scan_sums_len(uint64_t n);

namespace {

constexpr int kRT = 256;

struct RoundsParams {
  uint64_t smix;
  uint64_t b_lo;  // global id of local bucket 0 (a shard's bucket range; 0 for one table)
  uint64_t m2[33];  // floor((2^64-1) / s^2), s <= 32 (R22)
};

struct __align__(16) ActKey {  // an active key: the key, its input index, its bucket's rank o
  uint64_t key;
  uint32_t idx, o;
};

__device__ __forceinline__ uint32_t level2_slot(const RoundsParams& P, uint64_t b, uint32_t t, uint32_t s,
                                                uint64_t key) {
  if (s == 1) return 0;  // R12
  const uint64_t hv = hash64(derive(P.smix, 2, P.b_lo + b, t), key);
  const uint64_t s2 = uint64_t(s) * s;
  if ((s2 & (s2 - 1)) == 0) return uint32_t(hv & (s2 - 1));
  if (s <= 32) {
    FastMod f{s2, P.m2[s]};
    return uint32_t(fastmod(hv, f));
  }
  return uint32_t(hv % s2);
}

// The keys the rounds hash and the slot records they write: u64 keys
// ({key, value}) or byte keys ({fingerprint, value, ctx_off, len}, the
// fingerprints of the current t0).
struct RSrcU64 {
  const uint64_t* keys;
  const uint64_t* vals;
  __device__ __forceinline__ uint64_t key(uint64_t i) const { return keys[i]; }
  __device__ __forceinline__ KV16 rec(uint64_t i) const {
    KV16 e;
    e.key = keys[i];
    e.value = vals[i];
    return e;
  }
};
struct RSrcBytes {
  const uint64_t* fp;
  const uint64_t* vals;
  const uint64_t* offs;
  uint64_t off0;
  __device__ __forceinline__ uint64_t key(uint64_t i) const { return fp[i]; }
  __device__ __forceinline__ KV32 rec(uint64_t i) const {
    KV32 e;
    e.key = fp[i];
    e.value = vals[i];
    e.ctx_off = offs[i] - off0;
    e.len = uint32_t(offs[i + 1] - offs[i]);
    e.reserved = 0;
    return e;
  }
};

#define HM_GRID_LOOP(i, n) \
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < (n); i += uint64_t(gridDim.x) * blockDim.x)

// make_1: the level-1 bucket of every key and `shape = hist n hashes`
// (local buckets b - b_lo of a shard's range [b_lo, b_lo + nb))
template <class Src>
__global__ void k_r_l1_hist(Src src, uint64_t n, L1Params l1, uint64_t b_lo, uint64_t nb,
                            uint32_t* __restrict__ kb, unsigned int* __restrict__ shape, unsigned int* __restrict__ bad) {
  HM_GRID_LOOP(i, n) {
    const uint64_t b = level1_bucket(l1, src.key(i)) - b_lo;
    if (b >= nb) {
      atomicOr(bad, 1u);
      kb[i] = 0;
      continue;
    }
    kb[i] = uint32_t(b);
    atomicAdd(shape + b, 1u);
  }
}

// per bucket: s^2 (for the slot offsets and R7) and (s != 0) (for `offsets`,
// P:458); entry n is 0 so that the exclusive scans end with the totals
__global__ void k_r_l1_prep(const unsigned int* __restrict__ shape, uint64_t n, uint64_t* __restrict__ sq,
                            uint64_t* __restrict__ nz) {
  HM_GRID_LOOP(b, n + 1) {
    const uint64_t s = b < n ? shape[b] : 0;
    sq[b] = s * s;
    nz[b] = s != 0;
  }
}

// ishape = filter (!= 0) (zip (iota n) shape)
__global__ void k_r_init_active(const unsigned int* __restrict__ shape, const uint64_t* __restrict__ rank, uint64_t n,
                                uint32_t* __restrict__ A) {
  HM_GRID_LOOP(b, n) {
    if (shape[b]) A[rank[b]] = uint32_t(b);
  }
}

// okeys = zip koffsets keys
template <class Src>
__global__ void k_r_init_keys(Src src, const uint32_t* __restrict__ kb,
                              const uint64_t* __restrict__ rank, uint64_t n, ActKey* __restrict__ ak) {
  HM_GRID_LOOP(i, n) {
    ActKey a;
    a.key = src.key(i);
    a.idx = uint32_t(i);
    a.o = uint32_t(rank[kb[i]]);
    ak[i] = a;
  }
}

// offsets = presum (map (\s -> s^2) shape) over the active buckets
__global__ void k_r_seg_sq(const uint32_t* __restrict__ A, const unsigned int* __restrict__ shape, uint64_t m,
                           uint64_t* __restrict__ foff) {
  HM_GRID_LOOP(o, m + 1) {
    const uint64_t s = o < m ? shape[A[o]] : 0;
    foff[o] = s * s;
  }
}

// seghashes + the `hist` of segcollisions
__global__ void k_r_seg_hash(const ActKey* __restrict__ ak, uint64_t nk, const uint32_t* __restrict__ A,
                             const unsigned int* __restrict__ shape, const uint64_t* __restrict__ foff, RoundsParams P,
                             uint32_t t, uint32_t* __restrict__ hk, unsigned int* __restrict__ flat) {
  HM_GRID_LOOP(j, nk) {
    const ActKey a = ak[j];
    const uint32_t b = A[a.o];
    const uint32_t h = level2_slot(P, b, t, shape[b], a.key);
    hk[j] = h;
    atomicAdd(flat + foff[a.o] + h, 1u);
  }
}

// segcollisions: a bucket collides when any of its flat slots counts > 1
__global__ void k_r_seg_coll(const ActKey* __restrict__ ak, uint64_t nk, const uint64_t* __restrict__ foff,
                             const uint32_t* __restrict__ hk, const unsigned int* __restrict__ flat,
                             uint64_t* __restrict__ coll) {
  HM_GRID_LOOP(j, nk) {
    const uint32_t o = ak[j].o;
    if (flat[foff[o] + hk[j]] > 1u) coll[o] = 1;
  }
}

// segresult: finished buckets record t; the colliding ones form
// ishape', renumbered by presum collisions
__global__ void k_r_seg_result(const uint32_t* __restrict__ A, uint64_t m, const uint64_t* __restrict__ noff,
                               uint32_t t, uint32_t* __restrict__ A2, uint8_t* __restrict__ tb) {
  HM_GRID_LOOP(o, m) {
    const uint32_t b = A[o];
    if (noff[o + 1] != noff[o]) A2[noff[o]] = b;
    else tb[b] = uint8_t(t);
  }
}

// keys' = filter (collisions[o]) keys, renumbered; the keys of
// finished buckets keep their slot.  Every key also clears its flat counter
// for the next round.
__global__ void k_r_seg_keys(const ActKey* __restrict__ ak, uint64_t nk, const uint64_t* __restrict__ foff,
                             const uint32_t* __restrict__ hk, const uint64_t* __restrict__ noff,
                             unsigned int* __restrict__ flat, ActKey* __restrict__ ak2,
                             unsigned long long* __restrict__ cursor, uint32_t* __restrict__ hkey) {
  const uint32_t lane = threadIdx.x & 31;
  // (warp-uniform trip count so that the append can use warp ballots)
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t j0 = blockIdx.x * uint64_t(blockDim.x) + (threadIdx.x & ~31u); j0 < nk; j0 += stride) {
    const uint64_t j = j0 + lane;
    bool keep = false;
    ActKey a{};
    uint32_t h = 0;
    if (j < nk) {
      a = ak[j];
      h = hk[j];
      flat[foff[a.o] + h] = 0u;
      keep = noff[a.o + 1] != noff[a.o];
      if (!keep) hkey[a.idx] = h;
    }
    const uint32_t bal = __ballot_sync(0xffffffffu, keep);
    if (bal) {
      unsigned long long base = 0;
      if (lane == 0) base = atomicAdd(cursor, (unsigned long long)__popc(bal));
      base = __shfl_sync(0xffffffffu, base, 0);
      if (keep) {
        a.o = uint32_t(noff[a.o]);
        ak2[base + __popc(bal & ((1u << lane) - 1u))] = a;
      }
    }
  }
}

// ---- the table (R10, R12): filler selection, fillers, members, directory
__global__ void k_r_fin_min(const uint32_t* __restrict__ kb, const unsigned int* __restrict__ shape,
                            const uint32_t* __restrict__ hkey, uint64_t n, unsigned long long* __restrict__ fsel) {
  HM_GRID_LOOP(i, n) {
    const uint32_t b = kb[i];
    if (shape[b] >= 2) atomicMin(fsel + b, (unsigned long long)((uint64_t(hkey[i]) << 32) | i));
  }
}

template <class Src, class E>
__global__ void k_r_fin_fill(const unsigned int* __restrict__ shape, const uint64_t* __restrict__ soff,
                             const unsigned long long* __restrict__ fsel, Src src,
                             uint64_t n, E* __restrict__ slots) {
  HM_GRID_LOOP(b, n) {
    const uint32_t s = shape[b];
    if (s < 2) continue;
    E f = src.rec(uint32_t(fsel[b]));
    f.value = 0;
    E* out = slots + soff[b];
    for (uint32_t x = 0; x < s * s; x++) out[x] = f;
  }
}

template <class Src, class E>
__global__ void k_r_fin_members(Src src, const uint32_t* __restrict__ kb, const unsigned int* __restrict__ shape,
                                const uint64_t* __restrict__ soff, const uint32_t* __restrict__ hkey, L1Params l1,
                                uint64_t n, E* __restrict__ slots, uint8_t* __restrict__ tb) {
  HM_GRID_LOOP(i, n) {
    const uint32_t b = kb[i];
    const E e = src.rec(i);
    const uint64_t k = e.key;
    slots[soff[b] + hkey[i]] = e;
    if (shape[b] == 1) tb[b] = uint8_t(tag4_of_hash(hash64(l1.c1, k)));  // the cdir tag of a singleton
  }
}

// dir entries and compact records, a warp per 32 buckets (the layout k_bucket writes)
__global__ void k_r_fin_dir(const unsigned int* __restrict__ shape, const uint64_t* __restrict__ soff,
                            const uint8_t* __restrict__ tb, uint64_t n, uint32_t full_dir, uint64_t* __restrict__ dir,
                            CDir* __restrict__ cdir) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t b0 = blockIdx.x * uint64_t(blockDim.x) + (threadIdx.x & ~31u); b0 < n; b0 += stride) {
    const uint64_t b = b0 + lane;
    uint32_t s = 0, t = 0;
    uint64_t so = 0;
    if (b < n) {
      s = shape[b];
      t = s ? tb[b] : 0u;
      so = soff[b];
      dir[b] = dir_entry(so, s, s == 1 ? 0u : t);
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

template <class T>
hm_status ralloc(std::vector<void*>& owned, T** p, size_t bytes, cudaStream_t st) {
  void* v = nullptr;
  const cudaError_t e = cudaMallocAsync(&v, std::max<size_t>(bytes, 16), st);
  if (e != cudaSuccess) {
    cudaGetLastError();
    set_error(std::string("cudaMallocAsync(") + std::to_string(bytes) + ") failed: " + cudaGetErrorString(e));
    return HM_ERR_OOM;
  }
  owned.push_back(v);
  *p = reinterpret_cast<T*>(v);
  return HM_OK;
}

struct Owned {
  cudaStream_t st;
  std::vector<void*> v;
  ~Owned() {
    for (void* p : v) cudaFreeAsync(p, st);
  }
};

}  // namespace

#define HM_RLAUNCH(name, grid, ...)                        \
  do {                                                     \
    LaunchScope ls_(#name, st);                            \
    name<<<(grid), kRT, 0, st>>>(__VA_ARGS__);             \
  } while (0)

// Equal keys left in a bucket that exhausted its attempts: u64 keys are
// duplicates; equal fingerprints of byte keys are duplicates when the bytes are
// equal too, else a fingerprint collision (the caller redraws t0).
struct SameHostU64 {
  hm_status operator()(uint32_t, uint32_t, cudaStream_t, bool* fpcoll) const {
    *fpcoll = false;
    return HM_OK;
  }
};
struct SameHostBytes {
  const uint8_t* bytes;
  const uint64_t* offs;
  hm_status operator()(uint32_t i, uint32_t j, cudaStream_t st, bool* fpcoll) const {
    uint64_t oi[2], oj[2];
    HM_CUDA_TRY(cudaMemcpyAsync(oi, offs + i, 16, cudaMemcpyDeviceToHost, st));
    HM_CUDA_TRY(cudaMemcpyAsync(oj, offs + j, 16, cudaMemcpyDeviceToHost, st));
    HM_CUDA_TRY(cudaStreamSynchronize(st));
    bool same = oi[1] - oi[0] == oj[1] - oj[0];
    if (same && oi[1] > oi[0]) {
      std::vector<uint8_t> a(oi[1] - oi[0]), b(oj[1] - oj[0]);
      HM_CUDA_TRY(cudaMemcpyAsync(a.data(), bytes + oi[0], a.size(), cudaMemcpyDeviceToHost, st));
      HM_CUDA_TRY(cudaMemcpyAsync(b.data(), bytes + oj[0], b.size(), cudaMemcpyDeviceToHost, st));
      HM_CUDA_TRY(cudaStreamSynchronize(st));
      same = a == b;
    }
    *fpcoll = !same;
    return HM_OK;
  }
};

template <class Src, class E, class SameHost>
static hm_status build_rounds_core(Src src, SameHost same, uint64_t n_in, uint64_t n_global, uint64_t b_lo,
                                   uint64_t nb, int t1_fixed, uint64_t seed, uint32_t flags, cudaStream_t st,
                                   BuildOut* out, bool* fpcoll) {
  *fpcoll = false;
  Owned ow{st, {}};
  const uint64_t smix = seed_mix(seed);
  const unsigned gmax = unsigned(num_sms()) * 8;
  auto grid = [&](uint64_t m) { return unsigned(std::max<uint64_t>(1, std::min<uint64_t>((m + kRT - 1) / kRT, gmax))); };
  RoundsParams P{};
  P.smix = smix;
  P.b_lo = b_lo;
  for (int i = 1; i <= 32; i++) P.m2[i] = ~0ull / (uint64_t(i) * i);
  const uint64_t n = nb;  // (the bucket count; the keys are n_in)

  uint32_t *kb, *A, *A2, *hk, *hkey;
  unsigned int *shape, *flat, *bad;
  uint64_t *soff, *rank, *foff, *coll, *sums;
  ActKey *ak, *ak2;
  unsigned long long *fsel, *cursor;
  uint8_t* tb;
  hm_status s;
  const size_t nsums = scan_sums_len(n + 1);
  if ((s = ralloc(ow.v, &kb, n_in * 4, st)) || (s = ralloc(ow.v, &shape, n * 4, st)) ||
      (s = ralloc(ow.v, &soff, (n + 1) * 8, st)) || (s = ralloc(ow.v, &rank, (n + 1) * 8, st)) ||
      (s = ralloc(ow.v, &sums, nsums * 8, st)) || (s = ralloc(ow.v, &bad, 4, st)))
    return s;

  // level one (make_1) with the space bound R7 (a shard: the
  // caller's t1, the caller checks the global bound)
  uint32_t t1 = t1_fixed >= 0 ? uint32_t(t1_fixed) : 0u;
  uint64_t S = 0, m = 0;
  for (;; t1++) {
    if (t1 == kT1Cap) {
      set_error("level one exhausted 16 attempts without meeting the space bound S <= 4n");
      return HM_ERR_SEED_EXHAUSTED;
    }
    const L1Params l1 = make_l1(smix, t1, n_global);
    HM_CUDA_TRY(cudaMemsetAsync(shape, 0, n * 4, st));
    HM_CUDA_TRY(cudaMemsetAsync(bad, 0, 4, st));
    HM_RLAUNCH(k_r_l1_hist, grid(n_in), src, n_in, l1, b_lo, nb, kb, shape, bad);
    HM_RLAUNCH(k_r_l1_prep, grid(n + 1), shape, n, soff, rank);
    if ((s = scan_excl(soff, n + 1, sums, st)) != HM_OK) return s;
    unsigned int hbad = 0;
    HM_CUDA_TRY(cudaMemcpyAsync(&S, soff + n, 8, cudaMemcpyDeviceToHost, st));
    HM_CUDA_TRY(cudaMemcpyAsync(&hbad, bad, 4, cudaMemcpyDeviceToHost, st));
    HM_CUDA_TRY(cudaStreamSynchronize(st));
    if (hbad) {
      set_error("a routed key does not belong to this shard's bucket range");
      return HM_ERR_INVALID_ARG;
    }
    if (S <= 4 * n_global) break;
    if (t1_fixed >= 0) {  // a shard over the global bound on its own: the caller redraws level one
      void* arr[3] = {nullptr, nullptr, nullptr};
      const size_t bytes[3] = {16, sizeof(CDir), 16};
      for (int a = 0; a < 3; a++)
        if ((s = map_alloc(&arr[a], bytes[a], st)) != HM_OK) {
          for (int b = 0; b < a; b++) map_discard(arr[b], bytes[b], st);
          return s;
        }
      out->dir = static_cast<uint64_t*>(arr[0]);
      out->cdir = static_cast<CDir*>(arr[1]);
      out->slots = arr[2];
      for (int a = 0; a < 3; a++) out->bytes[a] = bytes[a];
      out->S = S;
      out->t1 = t1;
      return HM_OK;
    }
  }
  if ((s = scan_excl(rank, n + 1, sums, st)) != HM_OK) return s;
  HM_CUDA_TRY(cudaMemcpyAsync(&m, rank + n, 8, cudaMemcpyDeviceToHost, st));
  HM_CUDA_TRY(cudaStreamSynchronize(st));

  if ((s = ralloc(ow.v, &A, m * 4, st)) || (s = ralloc(ow.v, &A2, m * 4, st)) ||
      (s = ralloc(ow.v, &hk, n_in * 4, st)) || (s = ralloc(ow.v, &hkey, n_in * 4, st)) ||
      (s = ralloc(ow.v, &flat, S * 4, st)) || (s = ralloc(ow.v, &foff, (m + 1) * 8, st)) ||
      (s = ralloc(ow.v, &coll, (m + 1) * 8, st)) || (s = ralloc(ow.v, &ak, n_in * sizeof(ActKey), st)) ||
      (s = ralloc(ow.v, &ak2, n_in * sizeof(ActKey), st)) || (s = ralloc(ow.v, &fsel, n * 8, st)) ||
      (s = ralloc(ow.v, &cursor, 8, st)) || (s = ralloc(ow.v, &tb, n, st)))
    return s;
  HM_CUDA_TRY(cudaMemsetAsync(flat, 0, S * 4, st));
  HM_CUDA_TRY(cudaMemsetAsync(tb, 0, n, st));
  HM_RLAUNCH(k_r_init_active, grid(n), shape, rank, n, A);
  HM_RLAUNCH(k_r_init_keys, grid(n_in), src, kb, rank, n_in, ak);

  // level two: segmake'_2 rounds, round r = attempt t = r
  uint64_t nk = n_in;
  uint32_t r = 0;
  for (; m > 0 && r < kT2Cap; r++) {
    HM_RLAUNCH(k_r_seg_sq, grid(m + 1), A, shape, m, foff);
    if ((s = scan_excl(foff, m + 1, sums, st)) != HM_OK) return s;
    HM_RLAUNCH(k_r_seg_hash, grid(nk), ak, nk, A, shape, foff, P, r, hk, flat);
    HM_CUDA_TRY(cudaMemsetAsync(coll, 0, (m + 1) * 8, st));
    HM_RLAUNCH(k_r_seg_coll, grid(nk), ak, nk, foff, hk, flat, coll);
    if ((s = scan_excl(coll, m + 1, sums, st)) != HM_OK) return s;
    HM_RLAUNCH(k_r_seg_result, grid(m), A, m, coll, r, A2, tb);
    HM_CUDA_TRY(cudaMemsetAsync(cursor, 0, 8, st));
    HM_RLAUNCH(k_r_seg_keys, grid(nk), ak, nk, foff, hk, coll, flat, ak2, cursor, hkey);
    uint64_t cnt[2] = {0, 0};
    HM_CUDA_TRY(cudaMemcpyAsync(&cnt[0], coll + m, 8, cudaMemcpyDeviceToHost, st));
    HM_CUDA_TRY(cudaMemcpyAsync(&cnt[1], cursor, 8, cudaMemcpyDeviceToHost, st));
    HM_CUDA_TRY(cudaStreamSynchronize(st));
    m = cnt[0];
    nk = cnt[1];
    std::swap(A, A2);
    std::swap(ak, ak2);
  }
  if (m > 0) {  // some bucket failed 256 attempts: equal keys among the remaining ones?
    std::vector<ActKey> h(nk);
    HM_CUDA_TRY(cudaMemcpyAsync(h.data(), ak, nk * sizeof(ActKey), cudaMemcpyDeviceToHost, st));
    HM_CUDA_TRY(cudaStreamSynchronize(st));
    std::sort(h.begin(), h.end(), [](const ActKey& a, const ActKey& b) { return a.key < b.key; });
    bool dup = false, coll = false;
    for (uint64_t j = 1; j < nk; j++)
      if (h[j].key == h[j - 1].key) {
        bool fc = false;
        hm_status s2 = same(h[j - 1].idx, h[j].idx, st, &fc);
        if (s2 != HM_OK) return s2;
        (fc ? coll : dup) = true;
      }
    if (dup) {  // (duplicates first, then fingerprint collisions: SURVEY 8(c) step 5)
      set_error("duplicate keys in from_array_nodup input");
      return HM_ERR_DUPLICATE_KEY;
    }
    if (coll) {
      *fpcoll = true;
      return HM_OK;
    }
    set_error("a level-2 bucket exhausted 256 attempts");
    return HM_ERR_SEED_EXHAUSTED;
  }

  // the table
  uint64_t* dir = nullptr;
  CDir* cdir = nullptr;
  E* slots = nullptr;
  std::vector<void*> res;
  const size_t bytes_[3] = {n * 8, ((n + 31) / 32) * sizeof(CDir), S * sizeof(E)};
  const size_t* bytes = bytes_;
  auto fail = [&](hm_status code) {
    for (size_t a = 0; a < res.size(); a++) map_discard(res[a], bytes_[a], st);
    return code;
  };
  void* arr[3] = {nullptr, nullptr, nullptr};
  for (int a = 0; a < 3; a++) {
    if ((s = map_alloc(&arr[a], bytes[a], st)) != HM_OK) return fail(s);
    res.push_back(arr[a]);
  }
  dir = static_cast<uint64_t*>(arr[0]);
  cdir = static_cast<CDir*>(arr[1]);
  slots = static_cast<E*>(arr[2]);
  const L1Params l1 = make_l1(smix, t1, n_global);
  HM_CUDA_TRY(cudaMemsetAsync(fsel, 0xFF, n * 8, st));
  HM_RLAUNCH(k_r_fin_min, grid(n_in), kb, shape, hkey, n_in, fsel);
  HM_RLAUNCH(k_r_fin_fill, grid(n), shape, soff, fsel, src, n, slots);
  HM_RLAUNCH(k_r_fin_members, grid(n_in), src, kb, shape, soff, hkey, l1, n_in, slots, tb);
  HM_RLAUNCH(k_r_fin_dir, grid(n), shape, soff, tb, n, flags & HM_FLAG_FULL_DIRECTORY, dir, cdir);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(cuda_fail(e, "rounds build"));
  out->dir = dir;
  out->cdir = cdir;
  out->slots = slots;
  for (int a = 0; a < 3; a++) out->bytes[a] = bytes[a];
  out->S = S;
  out->t1 = t1;
  return HM_OK;
}

hm_status build_u64_rounds(const uint64_t* keys, const uint64_t* vals, uint64_t n_in, uint64_t n_global,
                           uint64_t b_lo, uint64_t nb, int t1_fixed, uint64_t seed, uint32_t flags, cudaStream_t st,
                           BuildOut* out) {
  bool fc = false;
  return build_rounds_core<RSrcU64, KV16>(RSrcU64{keys, vals}, SameHostU64{}, n_in, n_global, b_lo, nb, t1_fixed,
                                          seed, flags, st, out, &fc);
}

// Byte keys (their fingerprints fp[n] under the current t0): any bucket size,
// the same table as the partitioned build (a fallback for degenerate level-1
// distributions); *fpcoll: equal fingerprints with different bytes.
hm_status build_bytes_rounds(const uint64_t* fp, const uint64_t* vals, const uint64_t* offs, uint64_t off0,
                             const uint8_t* bytes, uint64_t n, uint64_t seed, uint32_t flags, cudaStream_t st,
                             BuildOut* out, bool* fpcoll) {
  return build_rounds_core<RSrcBytes, KV32>(RSrcBytes{fp, vals, offs, off0}, SameHostBytes{bytes, offs}, n, n, 0, n,
                                            -1, seed, flags, st, out, fpcoll);
}

}  // namespace hm
