// capi.cu — the extern "C" boundary of libhm (include/hm.h).
//
// Argument validation, host-buffer staging for the end-to-end path, map
// lifetime, export for parity, and the multi-GPU building blocks.  Every
// compute step is one of the kernels in build.cu / lookup.cu; nothing here
// computes on the CPU.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "hm_internal.cuh"

namespace hm {

static thread_local std::string g_last_error;
static std::atomic<uint64_t> g_launches{0};
static std::atomic<int> g_profile{0};

struct ProfRec {
  const char* name;
  cudaEvent_t e0, e1;
};
static std::mutex g_prof_mu;
static std::vector<ProfRec> g_prof_pending;
static std::vector<cudaEvent_t> g_event_pool;

static cudaEvent_t get_event() {
  {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    if (!g_event_pool.empty()) {
      cudaEvent_t e = g_event_pool.back();
      g_event_pool.pop_back();
      return e;
    }
  }
  cudaEvent_t e = nullptr;
  if (cudaEventCreate(&e) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return e;
}

LaunchScope::LaunchScope(const char* n, cudaStream_t s) : name(n), st(s) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (g_profile.load(std::memory_order_relaxed)) {
    e0 = get_event();
    if (e0) cudaEventRecord(e0, st);
  }
}

LaunchScope::~LaunchScope() {
  if (!e0) return;
  cudaEvent_t e1 = get_event();
  if (!e1) return;
  cudaEventRecord(e1, st);
  std::lock_guard<std::mutex> lk(g_prof_mu);
  g_prof_pending.push_back({name, e0, e1});
}

void set_error(const std::string& s) { g_last_error = s; }

hm_status cuda_fail(cudaError_t e, const char* where) {
  cudaGetLastError();  // clear sticky-free errors
  set_error(std::string(where) + ": " + cudaGetErrorString(e));
  if (e == cudaErrorMemoryAllocation) return HM_ERR_OOM;
  if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver || e == cudaErrorNoKernelImageForDevice)
    return HM_ERR_NO_DEVICE;
  return HM_ERR_CUDA;
}

L1Params make_l1(uint64_t smix, uint32_t t1, uint64_t n_global) {
  L1Params p{};
  p.c1 = derive(smix, 1, 0, t1);
  p.n = n_global;
  p.mmagic = ~0ull / n_global;
  p.pow2 = (n_global & (n_global - 1)) == 0;
  p.mask = p.pow2 ? n_global - 1 : 0;
  return p;
}

int num_sms() {
  static int cache[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!cache[dev]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = v > 0 ? v : 148;
    // keep freed scratch in the stream-ordered pool between builds (warm pool)
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  }
  return cache[dev];
}

static hm_status check_device() {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    cudaGetLastError();
    set_error("no CUDA device visible");
    return HM_ERR_NO_DEVICE;
  }
  int dev = 0, major = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  if (major != 10) {
    set_error("libhm is built for sm_100a (B200) only");
    return HM_ERR_NO_DEVICE;
  }
  // Keep freed stream-ordered memory in the device's pool instead of handing it
  // back to the driver at every synchronisation (the default threshold, 0):
  // re-mapping a table's gigabytes costs ~10 ms per build otherwise.
  // hm_release_workspace() trims the pool.
  static bool configured[64] = {};
  if (dev >= 0 && dev < 64 && !configured[dev]) {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    cudaGetLastError();
    configured[dev] = true;
  }
  return HM_OK;
}

static bool is_device_ptr(const void* p) {
  if (!p) return true;
  cudaPointerAttributes a{};
  cudaError_t e = cudaPointerGetAttributes(&a, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// Device view of a caller array: the pointer itself, or a staged copy.
struct Staged {
  cudaStream_t st;
  std::vector<void*> tmp;
  ~Staged() {
    for (void* p : tmp) cudaFreeAsync(p, st);
  }
  template <class T>
  hm_status in(const T* host_or_dev, size_t count, const T** dev) {
    if (!host_or_dev || is_device_ptr(host_or_dev)) {
      *dev = host_or_dev;
      return HM_OK;
    }
    void* d = nullptr;
    HM_CUDA_TRY(cudaMallocAsync(&d, std::max<size_t>(count * sizeof(T), 16), st));
    tmp.push_back(d);
    HM_CUDA_TRY(cudaMemcpyAsync(d, host_or_dev, count * sizeof(T), cudaMemcpyHostToDevice, st));
    *dev = reinterpret_cast<const T*>(d);
    return HM_OK;
  }
  template <class T>
  hm_status out(T* host_or_dev, size_t count, T** dev, bool* staged) {
    *staged = false;
    if (!host_or_dev || is_device_ptr(host_or_dev)) {
      *dev = host_or_dev;
      return HM_OK;
    }
    void* d = nullptr;
    HM_CUDA_TRY(cudaMallocAsync(&d, std::max<size_t>(count * sizeof(T), 16), st));
    tmp.push_back(d);
    *dev = reinterpret_cast<T*>(d);
    *staged = true;
    return HM_OK;
  }
};

static bool hooks_ok(const hm_opts* o) { return !o || (!o->alloc) == (!o->free); }

// the map takes the user's free hook when its arrays came from the user's alloc
static void adopt_hooks(hm_map* m) {
  if (tl_user_alloc.alloc) {
    m->ufree = tl_user_alloc.free;
    m->uctx = tl_user_alloc.ctx;
  }
}

static hm_map* new_map() {
  hm_map* m = new hm_map;
  std::memset(m, 0, sizeof(*m));
  cudaGetDevice(&m->device);
  return m;
}

}  // namespace hm

using namespace hm;

extern "C" {

const char* hm_version(void) { return "hm 0.1 (sm_100a, spec v1)"; }

uint64_t hm_kernel_launches(void) { return g_launches.load(std::memory_order_relaxed); }

hm_status hm_release_workspace(void) {
  g_last_error.clear();
  hm_status s = check_device();
  if (s != HM_OK) return s;
  return release_workspace();
}

void hm_profile_enable(int on) { g_profile.store(on ? 1 : 0); }

int hm_profile_read(hm_kernel_stat* out, int max) {
  std::vector<ProfRec> recs;
  {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    recs.swap(g_prof_pending);
  }
  std::vector<hm_kernel_stat> agg;
  for (const ProfRec& r : recs) {
    float ms = 0.f;
    cudaEventSynchronize(r.e1);
    if (cudaEventElapsedTime(&ms, r.e0, r.e1) != cudaSuccess) {
      cudaGetLastError();
      ms = 0.f;
    }
    size_t k = 0;
    for (; k < agg.size(); k++)
      if (std::strncmp(agg[k].name, r.name, sizeof(agg[k].name)) == 0) break;
    if (k == agg.size()) {
      hm_kernel_stat z{};
      std::strncpy(z.name, r.name, sizeof(z.name) - 1);
      agg.push_back(z);
    }
    agg[k].launches += 1;
    agg[k].ms += ms;
  }
  {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    for (const ProfRec& r : recs) {
      g_event_pool.push_back(r.e0);
      g_event_pool.push_back(r.e1);
    }
  }
  const int n = int(std::min<size_t>(agg.size(), size_t(max > 0 ? max : 0)));
  for (int i = 0; i < n; i++) out[i] = agg[i];
  return int(agg.size());
}

const char* hm_last_error(void) { return g_last_error.c_str(); }

const char* hm_status_str(hm_status s) {
  switch (s) {
    case HM_OK: return "OK";
    case HM_ERR_INVALID_ARG: return "INVALID_ARG";
    case HM_ERR_EMPTY: return "EMPTY";
    case HM_ERR_DUPLICATE_KEY: return "DUPLICATE_KEY";
    case HM_ERR_SEED_EXHAUSTED: return "SEED_EXHAUSTED";
    case HM_ERR_FP_EXHAUSTED: return "FP_EXHAUSTED";
    case HM_ERR_TOO_LARGE: return "TOO_LARGE";
    case HM_ERR_OOM: return "OOM";
    case HM_ERR_CUDA: return "CUDA";
    case HM_ERR_NCCL: return "NCCL";
    case HM_ERR_NO_DEVICE: return "NO_DEVICE";
  }
  return "UNKNOWN";
}

hm_status hm_build_u64(const uint64_t* keys, const uint64_t* vals, uint64_t n, const hm_opts* opts, void* stream,
                       hm_map** out) {
  g_last_error.clear();
  if (!out) return HM_ERR_INVALID_ARG;
  *out = nullptr;
  if (n == 0) return HM_ERR_EMPTY;
  if (!keys || !vals) return HM_ERR_INVALID_ARG;
  if (n > (1ull << 30)) return HM_ERR_TOO_LARGE;
  if (opts && (opts->flags & ~uint32_t(HM_FLAG_FULL_DIRECTORY | HM_FLAG_DIRECT_SLOTS | HM_FLAG_NO_ROUND0_ILP |
                                         HM_FLAG_FROM_ARRAY | HM_FLAG_ROUNDS | HM_FLAG_FUSED_PASS2)))
    return HM_ERR_INVALID_ARG;
  if (!hooks_ok(opts)) return HM_ERR_INVALID_ARG;
  UserAllocScope ua_(opts);
  hm_status s = check_device();
  if (s != HM_OK) return s;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  Staged sg{st, {}};
  const uint64_t *dk, *dv;
  if ((s = sg.in(keys, n, &dk)) != HM_OK) return s;
  if ((s = sg.in(vals, n, &dv)) != HM_OK) return s;
  const uint64_t seed = opts ? opts->seed : 0;
  uint64_t *uk = nullptr, *uv = nullptr;
  if (opts && (opts->flags & HM_FLAG_FROM_ARRAY)) {  // from_array: the distinct keys first
    uint64_t nu = 0;
    if ((s = dedup_u64(dk, dv, n, st, &uk, &uv, &nu)) != HM_OK) return s;
    dk = uk;
    dv = uv;
    n = nu;
  }
  BuildOut bo;
  if (opts && (opts->flags & HM_FLAG_ROUNDS)) {
    s = build_u64_rounds(dk, dv, n, n, 0, n, -1, seed, opts->flags, st, &bo);
  } else {
    s = build_u64_core(dk, dv, n, n, 0, n, -1, seed, opts ? (opts->log2_bp | (opts->flags << 16)) : 0, st, &bo);
    // a degenerate level-1 distribution within the space bound (a bucket of more
    // than 32 keys, an overflowing build partition: many equal keys, or an
    // adversarial key set) is outside the partitioned search; the flat rounds
    // handle any bucket size and report equal keys as DUPLICATE_KEY
    if (s == HM_ERR_TOO_LARGE) {
      set_error("");
      s = build_u64_rounds(dk, dv, n, n, 0, n, -1, seed, opts ? opts->flags : 0u, st, &bo);
    }
  }
  if (uk) {
    cudaFreeAsync(uk, st);
    cudaFreeAsync(uv, st);
  }
  if (s != HM_OK) return s;
  hm_map* m = new_map();
  m->key_kind = 0;
  m->n_global = n;
  m->b_lo = 0;
  m->nb = n;
  m->S = bo.S;
  m->seed = seed;
  m->t1 = bo.t1;
  m->smix = seed_mix(seed);
  m->l1 = make_l1(m->smix, bo.t1, n);
  m->dir = bo.dir;
  m->cdir = bo.cdir;
  m->slots = bo.slots;
  for (int a = 0; a < 3; a++) m->abytes[a] = bo.bytes[a];
  adopt_hooks(m);
  *out = m;
  return HM_OK;
}

static hm_status copy_streams(cudaStream_t* up, cudaStream_t* down);

hm_status hm_build_bytes(const uint8_t* bytes, const uint64_t* offsets, const uint64_t* vals, uint64_t n,
                         const hm_opts* opts, void* stream, hm_map** out) {
  g_last_error.clear();
  if (!out) return HM_ERR_INVALID_ARG;
  *out = nullptr;
  if (n == 0) return HM_ERR_EMPTY;
  if (!offsets || !vals) return HM_ERR_INVALID_ARG;
  if (n > (1ull << 30)) return HM_ERR_TOO_LARGE;
  if (opts && (opts->flags & ~uint32_t(HM_FLAG_FULL_DIRECTORY | HM_FLAG_DIRECT_SLOTS | HM_FLAG_NO_ROUND0_ILP |
                                         HM_FLAG_FROM_ARRAY)))
    return HM_ERR_INVALID_ARG;
  if (!hooks_ok(opts)) return HM_ERR_INVALID_ARG;
  UserAllocScope ua_(opts);
  hm_status s = check_device();
  if (s != HM_OK) return s;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  Staged sg{st, {}};
  const uint64_t *doff, *dv;
  if ((s = sg.in(offsets, n + 1, &doff)) != HM_OK) return s;
  if ((s = sg.in(vals, n, &dv)) != HM_OK) return s;
  // context extent: offsets[0] .. offsets[n]
  uint64_t o0 = 0, on = 0;
  HM_CUDA_TRY(cudaMemcpyAsync(&o0, doff, 8, cudaMemcpyDeviceToHost, st));
  HM_CUDA_TRY(cudaMemcpyAsync(&on, doff + n, 8, cudaMemcpyDeviceToHost, st));
  HM_CUDA_TRY(cudaStreamSynchronize(st));
  if (on < o0) return HM_ERR_INVALID_ARG;
  if (on > o0 && !bytes) return HM_ERR_INVALID_ARG;
  const uint8_t* db = bytes;
  if (bytes && !is_device_ptr(bytes)) {
    // stage exactly the used extent, keeping absolute offsets valid
    void* d = nullptr;
    HM_CUDA_TRY(cudaMallocAsync(&d, std::max<uint64_t>(on + 16, 16), st));
    sg.tmp.push_back(d);
    if (on > o0)
      HM_CUDA_TRY(cudaMemcpyAsync(reinterpret_cast<uint8_t*>(d) + o0, bytes + o0, on - o0, cudaMemcpyHostToDevice, st));
    db = reinterpret_cast<const uint8_t*>(d);
  }
  // offsets non-decreasing, keys <= 65535 bytes: checked before anything reads the bytes
  if ((s = check_offsets(doff, n, st)) != HM_OK) return s;
  const uint64_t seed = opts ? opts->seed : 0;
  if (opts && (opts->flags & HM_FLAG_FROM_ARRAY)) {  // from_array: the distinct keys, packed in input order
    uint8_t* pc = nullptr;
    uint64_t *po = nullptr, *pv = nullptr, m = 0;
    if ((s = dedup_bytes(db, doff, dv, n, st, &pc, &po, &pv, &m)) != HM_OK) return s;
    sg.tmp.push_back(pc);
    sg.tmp.push_back(po);
    sg.tmp.push_back(pv);
    db = pc;
    doff = po;
    dv = pv;
    n = m;
    o0 = 0;
    HM_CUDA_TRY(cudaMemcpyAsync(&on, po + m, 8, cudaMemcpyDeviceToHost, st));
    HM_CUDA_TRY(cudaStreamSynchronize(st));
  }
  // The map's copy of the key context is allocated now and copied
  // on a library stream while the build kernels run (the copy engine is idle
  // during the build), joined before the map is returned.
  const uint64_t ctx_bytes = on - o0;
  const size_t ctx_alloc = std::max<uint64_t>(ctx_bytes + 16, 16);
  uint8_t* ctxc = nullptr;
  {
    void* c = nullptr;
    if (tl_user_alloc.alloc) {
      c = tl_user_alloc.alloc(ctx_alloc, stream, tl_user_alloc.ctx);
      if (!c) {
        set_error("the user allocator (hm_opts.alloc) returned NULL for the context copy");
        return HM_ERR_OOM;
      }
    } else {
      const cudaError_t e = cudaMallocAsync(&c, ctx_alloc, st);
      if (e != cudaSuccess) return cuda_fail(e, "context copy");
    }
    ctxc = reinterpret_cast<uint8_t*>(c);
  }
  auto free_ctx = [&]() {
    if (tl_user_alloc.free) tl_user_alloc.free(ctxc, ctx_alloc, stream, tl_user_alloc.ctx);
    else cudaFreeAsync(ctxc, st);
  };
  // The copy happens inside the first k_bucket launch (its warps copy a slice
  // each while the partition's bulk load is in flight), or, for a context not
  // 16-aligned, as a copy on a library stream enqueued right before k_bucket
  // (SideJob): either way it overlaps the latency-bound k_bucket instead of
  // competing with the bandwidth-bound fingerprint and radix passes
  // (DESIGN.md §6.4).
  struct CtxCopy {
    uint8_t* dst;
    const uint8_t* src;
    uint64_t bytes;
    cudaStream_t cs;
    cudaEvent_t ev_in, ev_copied;
    cudaError_t err;
  } cc{ctxc, db + o0, ctx_bytes, nullptr, nullptr, nullptr, cudaSuccess};
  {
    cudaStream_t unused;
    hm_status s2 = copy_streams(&cc.cs, &unused);
    cudaError_t e = s2 == HM_OK ? cudaEventCreateWithFlags(&cc.ev_in, cudaEventDisableTiming) : cudaErrorUnknown;
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&cc.ev_copied, cudaEventDisableTiming);
    if (e != cudaSuccess) {
      if (cc.ev_in) cudaEventDestroy(cc.ev_in);
      if (cc.ev_copied) cudaEventDestroy(cc.ev_copied);
      free_ctx();
      return cuda_fail(e, "context copy");
    }
  }
  SideJob job;
  if (ctx_bytes && (reinterpret_cast<uintptr_t>(db + o0) & 15) == 0) {  // (ctxc: 256-aligned)
    job.ksrc = db + o0;
    job.kdst = ctxc;
    job.kbytes = ctx_bytes;
  }
  job.ctx = &cc;
  job.fn = [](void* p, cudaStream_t s_) {
    CtxCopy* c = static_cast<CtxCopy*>(p);
    cudaError_t e = cudaEventRecord(c->ev_in, s_);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(c->cs, c->ev_in, 0);
#ifndef HM_DEBUG_NO_CTX_COPY  // (timing experiments only: the map's context stays unwritten)
    if (e == cudaSuccess && c->bytes) e = cudaMemcpyAsync(c->dst, c->src, c->bytes, cudaMemcpyDeviceToDevice, c->cs);
#endif
    if (e == cudaSuccess) e = cudaEventRecord(c->ev_copied, c->cs);
    c->err = e;
  };
  BuildOut bo;
  uint32_t t0 = 0;
  uint64_t r = 0;
  s = build_bytes_core(db, doff, dv, n, seed, opts ? (opts->log2_bp | (opts->flags << 16)) : 0, st, &bo, &t0, &r,
                       &job, &o0);
  const bool in_kernel = job.done && job.kbytes;  // (k_bucket copied the context)
  if (s == HM_OK && !job.done) {  // (a build that never reached k_bucket)
    job.kbytes = 0;
    job.run(st);
  }
  if (job.done && !in_kernel) cudaStreamWaitEvent(st, cc.ev_copied, 0);  // (the copy read db before its staging is freed)
  cudaEventDestroy(cc.ev_in);
  cudaEventDestroy(cc.ev_copied);
  if (s == HM_OK && cc.err != cudaSuccess) {
    map_discard(bo.dir, bo.bytes[0], st);
    map_discard(bo.cdir, bo.bytes[1], st);
    map_discard(bo.slots, bo.bytes[2], st);
    free_ctx();
    return cuda_fail(cc.err, "context copy");
  }
  if (s != HM_OK) {
    free_ctx();
    return s;
  }
  hm_map* m = new_map();
  m->key_kind = 1;
  m->n_global = n;
  m->nb = n;
  m->S = bo.S;
  m->seed = seed;
  m->t1 = bo.t1;
  m->t0 = t0;
  m->r_fp = r;
  m->smix = seed_mix(seed);
  m->l1 = make_l1(m->smix, bo.t1, n);
  m->dir = bo.dir;
  m->cdir = bo.cdir;
  m->slots = bo.slots;
  for (int a = 0; a < 3; a++) m->abytes[a] = bo.bytes[a];
  adopt_hooks(m);
  m->ctx_bytes = ctx_bytes;
  if (tl_user_alloc.alloc) m->ctx_alloc = ctx_alloc;
  m->ctx = ctxc;
  const cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) {
    hm_free(m);
    return cuda_fail(e, "build_bytes");
  }
  *out = m;
  return HM_OK;
}

static hm_status lookup_common(const hm_map* map, uint64_t nq, uint64_t* out_vals, uint8_t* out_found,
                               cudaStream_t st, Staged& sg, uint64_t** dvo, uint8_t** dfo, bool* sv, bool* sf) {
  hm_status s;
  if ((s = sg.out(out_vals, nq, dvo, sv)) != HM_OK) return s;
  if ((s = sg.out(out_found, nq, dfo, sf)) != HM_OK) return s;
  (void)map;
  (void)st;
  return HM_OK;
}

static hm_status finish_outputs(uint64_t nq, uint64_t* out_vals, uint8_t* out_found, uint64_t* dvo, uint8_t* dfo,
                                bool sv, bool sf, cudaStream_t st) {
  if (sv) HM_CUDA_TRY(cudaMemcpyAsync(out_vals, dvo, nq * 8, cudaMemcpyDeviceToHost, st));
  if (sf) HM_CUDA_TRY(cudaMemcpyAsync(out_found, dfo, nq, cudaMemcpyDeviceToHost, st));
  if (sv || sf) HM_CUDA_TRY(cudaStreamSynchronize(st));
  return HM_OK;
}

// Host queries and host outputs: the batch goes through in chunks so that the
// upload of chunk c+1, the lookups of chunk c and the download of chunk c-1
// overlap (copy engines in both directions, PCIe full duplex) instead of
// upload, lookups, download one after the other.  Two library streams per
// device carry the copies; events order them with the caller's stream.
constexpr uint64_t kPipeChunk = uint64_t(1) << 23;
static hm_status copy_streams(cudaStream_t* up, cudaStream_t* down) {
  static std::mutex mu;
  static cudaStream_t s_up[64] = {}, s_down[64] = {};
  int dev = 0;
  HM_CUDA_TRY(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) return HM_ERR_INVALID_ARG;
  std::lock_guard<std::mutex> lk(mu);
  if (!s_up[dev]) {
    HM_CUDA_TRY(cudaStreamCreateWithFlags(&s_up[dev], cudaStreamNonBlocking));
    HM_CUDA_TRY(cudaStreamCreateWithFlags(&s_down[dev], cudaStreamNonBlocking));
  }
  *up = s_up[dev];
  *down = s_down[dev];
  return HM_OK;
}

static hm_status lookup_u64_pipelined(const hm_map* map, const uint64_t* q, uint64_t nq, uint64_t* out_vals,
                                      uint8_t* out_found, cudaStream_t st) {
  cudaStream_t up, down;
  hm_status s;
  if ((s = copy_streams(&up, &down)) != HM_OK) return s;
  uint64_t* dq = nullptr;
  uint64_t* dv = nullptr;
  uint8_t* df = nullptr;
  std::vector<cudaEvent_t> ev;
  auto cleanup = [&]() {
    if (dq) cudaFreeAsync(dq, st);
    if (dv) cudaFreeAsync(dv, st);
    if (df) cudaFreeAsync(df, st);
    for (cudaEvent_t e : ev) cudaEventDestroy(e);
  };
  auto event = [&](cudaEvent_t* e) {
    cudaError_t r = cudaEventCreateWithFlags(e, cudaEventDisableTiming);
    if (r == cudaSuccess) ev.push_back(*e);
    return r;
  };
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&dq), nq * 8, st);
  if (e == cudaSuccess && out_vals) e = cudaMallocAsync(reinterpret_cast<void**>(&dv), nq * 8, st);
  if (e == cudaSuccess && out_found) e = cudaMallocAsync(reinterpret_cast<void**>(&df), nq, st);
  cudaEvent_t e0, e_end;
  if (e == cudaSuccess) e = event(&e0);
  if (e == cudaSuccess) e = cudaEventRecord(e0, st);  // (the buffers and the caller's prior work)
  if (e == cudaSuccess) e = cudaStreamWaitEvent(up, e0, 0);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(down, e0, 0);
  for (uint64_t c0 = 0; e == cudaSuccess && c0 < nq; c0 += kPipeChunk) {
    const uint64_t cn = std::min(kPipeChunk, nq - c0);
    cudaEvent_t e_in, e_k;
    if ((e = event(&e_in)) != cudaSuccess || (e = event(&e_k)) != cudaSuccess) break;
    if ((e = cudaMemcpyAsync(dq + c0, q + c0, cn * 8, cudaMemcpyHostToDevice, up)) != cudaSuccess) break;
    if ((e = cudaEventRecord(e_in, up)) != cudaSuccess || (e = cudaStreamWaitEvent(st, e_in, 0)) != cudaSuccess) break;
    if ((s = lookup_u64_launch(map, dq + c0, cn, dv ? dv + c0 : nullptr, df ? df + c0 : nullptr, st)) != HM_OK) {
      cleanup();
      return s;
    }
    if ((e = cudaEventRecord(e_k, st)) != cudaSuccess || (e = cudaStreamWaitEvent(down, e_k, 0)) != cudaSuccess) break;
    if (dv && (e = cudaMemcpyAsync(out_vals + c0, dv + c0, cn * 8, cudaMemcpyDeviceToHost, down)) != cudaSuccess) break;
    if (df && (e = cudaMemcpyAsync(out_found + c0, df + c0, cn, cudaMemcpyDeviceToHost, down)) != cudaSuccess) break;
  }
  if (e == cudaSuccess) e = event(&e_end);
  if (e == cudaSuccess) e = cudaEventRecord(e_end, down);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(st, e_end, 0);  // (frees after the last download)
  cleanup();
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "pipelined lookup");
  return HM_OK;
}

hm_status hm_lookup_u64(const hm_map* map, const uint64_t* q, uint64_t nq, uint64_t* out_vals, uint8_t* out_found,
                        void* stream) {
  if (!map || (!q && nq) || (!out_vals && !out_found) || map->key_kind != 0) return HM_ERR_INVALID_ARG;
  if (nq == 0) return HM_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (nq > 2 * kPipeChunk && !is_device_ptr(q) &&
      (!out_vals || !is_device_ptr(out_vals)) && (!out_found || !is_device_ptr(out_found)))
    return lookup_u64_pipelined(map, q, nq, out_vals, out_found, st);
  Staged sg{st, {}};
  const uint64_t* dq;
  uint64_t* dvo;
  uint8_t* dfo;
  bool sv, sf;
  hm_status s;
  if ((s = sg.in(q, nq, &dq)) != HM_OK) return s;
  if ((s = lookup_common(map, nq, out_vals, out_found, st, sg, &dvo, &dfo, &sv, &sf)) != HM_OK) return s;
  if ((s = lookup_u64_launch(map, dq, nq, dvo, dfo, st)) != HM_OK) return s;
  return finish_outputs(nq, out_vals, out_found, dvo, dfo, sv, sf, st);
}

hm_status hm_lookup_bytes(const hm_map* map, const uint8_t* qbytes, const uint64_t* qoffsets, uint64_t nq,
                          uint64_t* out_vals, uint8_t* out_found, void* stream) {
  if (!map || (!qoffsets && nq) || (!out_vals && !out_found) || map->key_kind != 1) return HM_ERR_INVALID_ARG;
  if (nq == 0) return HM_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  Staged sg{st, {}};
  const uint64_t* dqo;
  hm_status s;
  if ((s = sg.in(qoffsets, nq + 1, &dqo)) != HM_OK) return s;
  const uint8_t* dqb = qbytes;
  if (qbytes && !is_device_ptr(qbytes)) {
    uint64_t o0 = 0, on = 0;
    HM_CUDA_TRY(cudaMemcpyAsync(&o0, dqo, 8, cudaMemcpyDeviceToHost, st));
    HM_CUDA_TRY(cudaMemcpyAsync(&on, dqo + nq, 8, cudaMemcpyDeviceToHost, st));
    HM_CUDA_TRY(cudaStreamSynchronize(st));
    void* d = nullptr;
    HM_CUDA_TRY(cudaMallocAsync(&d, on + 16, st));
    sg.tmp.push_back(d);
    if (on > o0)
      HM_CUDA_TRY(cudaMemcpyAsync(reinterpret_cast<uint8_t*>(d) + o0, qbytes + o0, on - o0, cudaMemcpyHostToDevice, st));
    dqb = reinterpret_cast<const uint8_t*>(d);
  }
  uint64_t* dvo;
  uint8_t* dfo;
  bool sv, sf;
  if ((s = lookup_common(map, nq, out_vals, out_found, st, sg, &dvo, &dfo, &sv, &sf)) != HM_OK) return s;
  if ((s = lookup_bytes_launch(map, dqb, dqo, nq, dvo, dfo, st)) != HM_OK) return s;
  return finish_outputs(nq, out_vals, out_found, dvo, dfo, sv, sf, st);
}

void hm_free(hm_map* map) {
  if (!map) return;
  int cur = 0;
  cudaGetDevice(&cur);
  if (cur != map->device) cudaSetDevice(map->device);
  cudaDeviceSynchronize();
  void* arr[3] = {map->dir, map->cdir, map->slots};
  for (int a = 0; a < 3; a++) {
    if (!arr[a]) continue;
    if (map->ufree) map->ufree(arr[a], map->abytes[a], nullptr, map->uctx);
    else if (map->abytes[a]) map_release(arr[a], map->abytes[a]);
    else cudaFree(arr[a]);
  }
  if (map->ctx) {
    if (map->ufree) map->ufree(map->ctx, map->ctx_alloc, nullptr, map->uctx);
    else cudaFree(map->ctx);
  }
  if (cur != map->device) cudaSetDevice(cur);
  delete map;
}

hm_status hm_info(const hm_map* map, hm_header* h) {
  if (!map || !h) return HM_ERR_INVALID_ARG;
  std::memset(h, 0, sizeof(*h));
  h->magic = HM_MAGIC;
  h->spec_version = HM_SPEC_VERSION;
  h->key_kind = map->key_kind;
  h->n = map->is_shard ? map->nb : map->n_global;
  h->S = map->S;
  h->seed = map->seed;
  h->t1 = map->t1;
  h->t0 = map->t0;
  h->ctx_bytes = map->ctx_bytes;
  return HM_OK;
}

hm_status hm_export(const hm_map* map, uint64_t* host_dir, void* host_slots, uint8_t* host_ctx) {
  if (!map) return HM_ERR_INVALID_ARG;
  if (host_dir) {
    if (is_device_ptr(host_dir)) {  // device destination: copy and rebase on the device
      HM_CUDA_TRY(cudaMemcpy(host_dir, map->dir, map->nb * 8, cudaMemcpyDeviceToDevice));
      if (map->slot_base) {
        hm_status s = dir_rebase_launch(host_dir, map->nb, map->slot_base, 0);
        if (s != HM_OK) return s;
      }
    } else {
      HM_CUDA_TRY(cudaMemcpy(host_dir, map->dir, map->nb * 8, cudaMemcpyDeviceToHost));
      if (map->slot_base)
        for (uint64_t i = 0; i < map->nb; i++) {
          const uint64_t d = host_dir[i];
          host_dir[i] = (d & ~kMask40) | ((d & kMask40) + map->slot_base);
        }
    }
  }
  if (host_slots && map->S)
    HM_CUDA_TRY(cudaMemcpy(host_slots, map->slots, map->S * (map->key_kind ? 32 : 16), cudaMemcpyDefault));
  if (host_ctx && map->ctx_bytes) HM_CUDA_TRY(cudaMemcpy(host_ctx, map->ctx, map->ctx_bytes, cudaMemcpyDefault));
  HM_CUDA_TRY(cudaDeviceSynchronize());
  return HM_OK;
}

hm_status hm_assemble_u64(const uint64_t* dir, const void* slots, uint64_t n, uint64_t S, uint64_t seed, uint32_t t1,
                          const hm_opts* opts, void* stream, hm_map** out) {
  g_last_error.clear();
  if (!out) return HM_ERR_INVALID_ARG;
  *out = nullptr;
  if (n == 0) return HM_ERR_EMPTY;
  if (!dir || !slots || S == 0) return HM_ERR_INVALID_ARG;
  if (n > (1ull << 30) || S > 4 * n) return HM_ERR_TOO_LARGE;
  if (t1 >= kT1Cap || (opts && (opts->flags & ~uint32_t(HM_FLAG_FULL_DIRECTORY)))) return HM_ERR_INVALID_ARG;
  if (!hooks_ok(opts)) return HM_ERR_INVALID_ARG;
  UserAllocScope ua_(opts);
  hm_status s = check_device();
  if (s != HM_OK) return s;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const size_t bytes[3] = {n * 8, ((n + 31) / 32) * sizeof(CDir), S * 16};
  void* arr[3] = {nullptr, nullptr, nullptr};
  auto fail = [&](hm_status code) {
    for (int a = 0; a < 3; a++)
      if (arr[a]) map_discard(arr[a], bytes[a], st);
    return code;
  };
  for (int a = 0; a < 3; a++)
    if ((s = map_alloc(&arr[a], bytes[a], st)) != HM_OK) return fail(s);
  unsigned int* bad = nullptr;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&bad), 4, st);
  if (e != cudaSuccess) return fail(cuda_fail(e, "assemble"));
  auto fail2 = [&](hm_status code) {
    cudaFreeAsync(bad, st);
    return fail(code);
  };
  if ((e = cudaMemcpyAsync(arr[0], dir, bytes[0], cudaMemcpyDefault, st)) != cudaSuccess ||
      (e = cudaMemcpyAsync(arr[2], slots, bytes[2], cudaMemcpyDefault, st)) != cudaSuccess ||
      (e = cudaMemsetAsync(bad, 0, 4, st)) != cudaSuccess)
    return fail2(cuda_fail(e, "assemble copies"));
  const uint64_t smix = seed_mix(seed);
  const L1Params l1 = make_l1(smix, t1, n);
  if ((s = assemble_cdir_launch(static_cast<uint64_t*>(arr[0]), arr[2], n, S, l1,
                                opts ? (opts->flags & HM_FLAG_FULL_DIRECTORY) : 0u, static_cast<CDir*>(arr[1]), bad,
                                st)) != HM_OK)
    return fail2(s);
  unsigned int hbad = 0;
  if ((e = cudaMemcpyAsync(&hbad, bad, 4, cudaMemcpyDeviceToHost, st)) != cudaSuccess ||
      (e = cudaStreamSynchronize(st)) != cudaSuccess)
    return fail2(cuda_fail(e, "assemble"));
  cudaFreeAsync(bad, st);
  if (hbad) {
    set_error("not a table: directory offsets do not follow soff_{b+1} = soff_b + s_b^2 up to S, or a bucket "
              "with s < 2 has t != 0");
    return fail(HM_ERR_INVALID_ARG);
  }
  hm_map* m = new_map();
  m->key_kind = 0;
  m->n_global = n;
  m->b_lo = 0;
  m->nb = n;
  m->S = S;
  m->seed = seed;
  m->t1 = t1;
  m->smix = smix;
  m->l1 = l1;
  m->dir = static_cast<uint64_t*>(arr[0]);
  m->cdir = static_cast<CDir*>(arr[1]);
  m->slots = arr[2];
  for (int a = 0; a < 3; a++) m->abytes[a] = bytes[a];
  adopt_hooks(m);
  *out = m;
  return HM_OK;
}

// ------------------------------------------------------------- multi-GPU
hm_status hm_route_u64(const uint64_t* keys, const uint64_t* vals, uint64_t n_local, uint64_t n_global, uint64_t seed,
                       uint32_t t1, int world, uint64_t* send_keys, uint64_t* send_vals, uint64_t* send_counts,
                       void* stream) {
  if ((!keys || !vals || !send_keys || !send_vals) && n_local) return HM_ERR_INVALID_ARG;
  if (!send_counts || world < 1 || world > 64 || n_global == 0 || t1 >= kT1Cap) return HM_ERR_INVALID_ARG;
  hm_status s = check_device();
  if (s != HM_OK) return s;
  const L1Params l1 = make_l1(seed_mix(seed), t1, n_global);
  return route_u64_launch(keys, vals, n_local, l1, world, send_keys, send_vals, send_counts,
                          reinterpret_cast<cudaStream_t>(stream));
}

hm_status hm_build_u64_shard(const uint64_t* keys, const uint64_t* vals, uint64_t n_recv, uint64_t n_global,
                             uint64_t b_lo, uint64_t b_hi, uint32_t t1, const hm_opts* opts, void* stream,
                             hm_map** out, uint64_t* S_local) {
  g_last_error.clear();
  if (!out || !S_local) return HM_ERR_INVALID_ARG;
  *out = nullptr;
  if (n_global == 0) return HM_ERR_EMPTY;
  if (n_global > (1ull << 30)) return HM_ERR_TOO_LARGE;
  if (b_hi < b_lo || b_hi > n_global || t1 >= kT1Cap) return HM_ERR_INVALID_ARG;
  if (n_recv && (!keys || !vals)) return HM_ERR_INVALID_ARG;
  if (!hooks_ok(opts)) return HM_ERR_INVALID_ARG;
  // (from_array and the rounds ablation are single-table paths)
  if (opts && (opts->flags & ~uint32_t(HM_FLAG_FULL_DIRECTORY | HM_FLAG_DIRECT_SLOTS | HM_FLAG_NO_ROUND0_ILP |
                                         HM_FLAG_FUSED_PASS2)))
    return HM_ERR_INVALID_ARG;
  UserAllocScope ua_(opts);
  hm_status s = check_device();
  if (s != HM_OK) return s;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const uint64_t seed = opts ? opts->seed : 0;
  const uint64_t nb = b_hi - b_lo;
  BuildOut bo;
  if (nb == 0) {
    // an empty bucket range: nothing to build, an empty shard
    hm_map* m = new_map();
    m->is_shard = true;
    m->n_global = n_global;
    m->b_lo = b_lo;
    m->seed = seed;
    m->t1 = t1;
    m->smix = seed_mix(seed);
    m->l1 = make_l1(m->smix, t1, n_global);
    HM_CUDA_TRY(cudaMalloc(&m->dir, 16));
    HM_CUDA_TRY(cudaMalloc(&m->cdir, sizeof(CDir)));
    HM_CUDA_TRY(cudaMalloc(&m->slots, 16));
    *S_local = 0;
    *out = m;
    return HM_OK;
  }
  s = build_u64_core(keys, vals, n_recv, n_global, b_lo, nb, int(t1), seed, opts ? (opts->log2_bp | (opts->flags << 16)) : 0, st, &bo);
  // a degenerate level-1 distribution within the bound (as in hm_build_u64):
  // the flat rounds restricted to the shard's bucket range, any bucket size,
  // equal keys -> DUPLICATE_KEY
  if (s == HM_ERR_TOO_LARGE && n_recv) {
    set_error("");
    s = build_u64_rounds(keys, vals, n_recv, n_global, b_lo, nb, int(t1), seed, opts ? opts->flags : 0u, st, &bo);
  }
  if (s != HM_OK) return s;
  hm_map* m = new_map();
  m->is_shard = true;
  m->key_kind = 0;
  m->n_global = n_global;
  m->b_lo = b_lo;
  m->nb = nb;
  m->S = bo.S;
  m->seed = seed;
  m->t1 = t1;
  m->smix = seed_mix(seed);
  m->l1 = make_l1(m->smix, t1, n_global);
  m->dir = bo.dir;
  m->cdir = bo.cdir;
  m->slots = bo.slots;
  for (int a = 0; a < 3; a++) m->abytes[a] = bo.bytes[a];
  adopt_hooks(m);
  *S_local = bo.S;
  *out = m;
  return HM_OK;
}

hm_status hm_dist_bucket_range(uint64_t n_global, int world, int rank, uint64_t* lo, uint64_t* hi) {
  if (world < 1 || rank < 0 || rank >= world || !lo || !hi) return HM_ERR_INVALID_ARG;
  const unsigned __int128 n = n_global;
  *lo = uint64_t((n * uint64_t(rank) + uint64_t(world) - 1) / uint64_t(world));
  *hi = uint64_t((n * uint64_t(rank + 1) + uint64_t(world) - 1) / uint64_t(world));
  return HM_OK;
}

int hm_dist_decide(uint64_t n_global, uint32_t t1, uint64_t S_total, int max_status, uint32_t* next_t1) {
  if (max_status != 0) return max_status;
  if (S_total <= 4 * n_global) return HM_OK;  // R7
  if (t1 + 1 >= kT1Cap) {
    set_error("level one exhausted 16 attempts without meeting S <= 4n");
    return HM_ERR_SEED_EXHAUSTED;
  }
  if (next_t1) *next_t1 = t1 + 1;
  return HM_DIST_REDRAW;
}

hm_status hm_dist_exchange_plan(const uint64_t* C, int world, int rank, uint64_t* off, uint64_t* cap,
                                uint64_t* recv) {
  if (!C || !off || !cap || !recv || world < 1 || world > 64 || rank < 0 || rank >= world) return HM_ERR_INVALID_ARG;
  *cap = 0;
  *recv = 0;
  for (int r = 0; r < world; r++) {
    uint64_t tot = 0;
    for (int q = 0; q < world; q++) {
      if (q == rank) off[r] = tot;
      tot += C[size_t(q) * world + r];
    }
    *cap = std::max(*cap, tot);
    if (r == rank) *recv = tot;
  }
  return HM_OK;
}

uint64_t hm_dist_slot_base(const uint64_t* S_all, int world, int rank) {
  uint64_t b = 0;
  for (int q = 0; q < rank && q < world; q++) b += S_all[q];
  return b;
}

hm_status hm_shard_set_base(hm_map* map, uint64_t slot_base) {
  if (!map) return HM_ERR_INVALID_ARG;
  map->slot_base = slot_base;
  return HM_OK;
}

hm_status hm_route_queries_u64(const hm_map* map, const uint64_t* q, uint64_t nq, int world, uint64_t* send_q,
                               uint64_t* perm, uint64_t* send_counts, void* stream) {
  if (!map || (nq && (!q || !send_q || !perm)) || !send_counts || world < 1 || world > 64) return HM_ERR_INVALID_ARG;
  return route_queries_launch(map->l1, q, nq, world, send_q, perm, send_counts,
                              reinterpret_cast<cudaStream_t>(stream));
}

hm_status hm_unroute_u64(const uint64_t* vals_routed, const uint8_t* found_routed, const uint64_t* perm, uint64_t nq,
                         uint64_t* out_vals, uint8_t* out_found, void* stream) {
  if (nq && (!perm || (out_vals && !vals_routed) || (out_found && !found_routed))) return HM_ERR_INVALID_ARG;
  return unroute_launch(vals_routed, found_routed, perm, nq, out_vals, out_found,
                        reinterpret_cast<cudaStream_t>(stream));
}

}  // extern "C"
