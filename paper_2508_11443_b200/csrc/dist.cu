// dist.cu — the multi-GPU build and lookup as single C calls over an NCCL
// communicator (SURVEY.md §8(b) `hm_build_u64_dist` / `hm_lookup_u64_dist`,
// §8(e)): the steps of DESIGN.md §7 — allreduce(n), route, all-to-all of the
// counts and of the pairs, shard build with a fixed t1, allreduce of S (sum,
// the global bound R7) and of the status (max), allgather of S_r for the
// slot base; lookups route, exchange, probe the local shard, exchange back
// and unroute.  The kernels are the ones behind hm_route_u64 /
// hm_build_u64_shard / hm_route_queries_u64 / hm_lookup_u64 / hm_unroute_u64;
// the all-to-all-v is a group of ncclSend/ncclRecv.  The communicator may be
// torch's (ProcessGroupNCCL._comm_ptr()): the library links the same
// libnccl.so.2.
#include <nccl.h>
#include <nccl_device.h>  // (NCCL 2.28 device API: window peer pointers)

#include <algorithm>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "hm_internal.cuh"
#include "route.cuh"

namespace hm {
namespace {

#define HM_NCCL_TRY(expr)                                                                 \
  do {                                                                                    \
    ncclResult_t r__ = (expr);                                                            \
    if (r__ != ncclSuccess) {                                                             \
      set_error(std::string("NCCL: ") + ncclGetErrorString(r__) + " in " #expr);         \
      return HM_ERR_NCCL;                                                                 \
    }                                                                                     \
  } while (0)

struct DevBufs {  // stream-ordered temporaries, freed on the stream
  cudaStream_t st;
  std::vector<void*> v;
  ~DevBufs() {
    for (void* p : v) cudaFreeAsync(p, st);
  }
  template <class T>
  hm_status get(T** p, size_t count) {
    void* q = nullptr;
    const cudaError_t e = cudaMallocAsync(&q, std::max<size_t>(count * sizeof(T), 16), st);
    if (e != cudaSuccess) {
      cudaGetLastError();
      set_error("dist: out of device memory");
      return HM_ERR_OOM;
    }
    v.push_back(q);
    *p = static_cast<T*>(q);
    return HM_OK;
  }
};

// every rank sends sc[r] elements to rank r and learns rc[r] (device u64[world])
hm_status exchange_counts(const uint64_t* d_sc, uint64_t* d_rc, std::vector<uint64_t>& sc, std::vector<uint64_t>& rc,
                          int world, ncclComm_t c, cudaStream_t st) {
  HM_NCCL_TRY(ncclGroupStart());
  for (int r = 0; r < world; r++) {
    HM_NCCL_TRY(ncclSend(d_sc + r, 1, ncclUint64, r, c, st));
    HM_NCCL_TRY(ncclRecv(d_rc + r, 1, ncclUint64, r, c, st));
  }
  HM_NCCL_TRY(ncclGroupEnd());
  sc.assign(world, 0);
  rc.assign(world, 0);
  HM_CUDA_TRY(cudaMemcpyAsync(sc.data(), d_sc, world * 8, cudaMemcpyDeviceToHost, st));
  HM_CUDA_TRY(cudaMemcpyAsync(rc.data(), d_rc, world * 8, cudaMemcpyDeviceToHost, st));
  HM_CUDA_TRY(cudaStreamSynchronize(st));
  return HM_OK;
}

// all-to-all-v of elem-byte elements, grouped by destination in `send`
hm_status all_to_all_v(const void* send, const std::vector<uint64_t>& sc, void* recv, const std::vector<uint64_t>& rc,
                       size_t elem, int world, ncclComm_t c, cudaStream_t st) {
  uint64_t so = 0, ro = 0;
  HM_NCCL_TRY(ncclGroupStart());
  for (int r = 0; r < world; r++) {
    if (sc[r]) HM_NCCL_TRY(ncclSend(static_cast<const char*>(send) + so * elem, sc[r] * elem, ncclUint8, r, c, st));
    if (rc[r]) HM_NCCL_TRY(ncclRecv(static_cast<char*>(recv) + ro * elem, rc[r] * elem, ncclUint8, r, c, st));
    so += sc[r];
    ro += rc[r];
  }
  HM_NCCL_TRY(ncclGroupEnd());
  return HM_OK;
}

// ------------------------------------------- fused route + exchange (NEXT-2)
// With HM_FLAG_FUSED_EXCHANGE the route kernel stores every (key, value)
// straight into its owner's receive window (registered with
// ncclCommWindowRegister, NCCL_WIN_COLL_SYMMETRIC, and mapped over NVLink:
// ncclGetPeerPointer), at the position the count matrix gives this rank in
// the owner's buffer — the transfer overlaps the scatter tile by tile instead
// of following it as an all-to-all.
struct OutWindow {
  ncclWindow_t win;
  size_t vals_off;  // byte offset of the values in every rank's window
  __device__ __forceinline__ uint64_t* keys(uint32_t d) const {
    return static_cast<uint64_t*>(ncclGetPeerPointer(win, 0, int(d)));
  }
  __device__ __forceinline__ uint64_t* vals(uint32_t d) const {
    return static_cast<uint64_t*>(ncclGetPeerPointer(win, vals_off, int(d)));
  }
};
__global__ void __launch_bounds__(kRThreads) k_route_scatter_win(const uint64_t* __restrict__ keys,
                                                                 const uint64_t* __restrict__ vals, uint64_t n,
                                                                 L1Params l1, int world,
                                                                 unsigned long long* __restrict__ cursors,
                                                                 OutWindow out) {
  route_scatter(keys, vals, n, l1, world, cursors, out, nullptr);
  __threadfence_system();  // (the peer stores are visible once the exchange's barrier completes)
}

// The receive window of one build: keys [0, cap) then values [cap, 2 cap), cap
// the largest count any rank receives (the same size on every rank: a
// symmetric window).  Registration is collective; so is release().
struct RecvWindow {
  void* buf = nullptr;
  ncclWindow_t win = nullptr;
  ncclComm_t comm = nullptr;
  uint64_t cap = 0;
  hm_status open(ncclComm_t c, uint64_t cap_elems) {
    comm = c;
    cap = std::max<uint64_t>(cap_elems, 1);
    const size_t bytes = (2 * cap * 8 + 4095) & ~size_t(4095);
    HM_NCCL_TRY(ncclMemAlloc(&buf, bytes));
    HM_NCCL_TRY(ncclCommWindowRegister(comm, buf, bytes, &win, NCCL_WIN_COLL_SYMMETRIC));
    return HM_OK;
  }
  hm_status release() {
    if (win) HM_NCCL_TRY(ncclCommWindowDeregister(comm, win));
    if (buf) HM_NCCL_TRY(ncclMemFree(buf));
    win = nullptr;
    buf = nullptr;
    return HM_OK;
  }
};

// Registered windows are kept per communicator and reused while large enough
// (registration is collective and costs milliseconds); every rank takes the
// same decision (cap is the global maximum).  hm_dist_release_windows frees
// them (collective).
static std::mutex g_win_mu;
static std::map<ncclComm_t, RecvWindow> g_win;

static hm_status window_for(ncclComm_t comm, uint64_t cap, RecvWindow** out) {
  std::lock_guard<std::mutex> lk(g_win_mu);
  RecvWindow& w = g_win[comm];
  if (!w.win || w.cap < cap) {
    hm_status s;
    if ((s = w.release()) != HM_OK) return s;
    if ((s = w.open(comm, cap + cap / 4 + 1024)) != HM_OK) return s;  // (headroom for the next builds)
  }
  *out = &w;
  return HM_OK;
}

// Route this rank's pairs into the owners' windows: counts, their all-gather
// (the G x G matrix C[q][r]), the window, the fused scatter, one barrier.
// On return rk/rv point into this rank's window (nrecv pairs).
hm_status fused_exchange(const uint64_t* keys, const uint64_t* vals, uint64_t n_local, const L1Params& l1, int world,
                         int rank, ncclComm_t comm, cudaStream_t st, uint64_t* d_small, const uint64_t** rk,
                         const uint64_t** rv, uint64_t* nrecv) {
  uint64_t* d_c = nullptr;  // [world] own counts, then [world][world] all of them, then [world] cursors
  const cudaError_t ea = cudaMallocAsync(reinterpret_cast<void**>(&d_c), (size_t(world) * world + 2 * world) * 8, st);
  if (ea != cudaSuccess) return cuda_fail(ea, "fused exchange");
  uint64_t* d_all = d_c + world;
  unsigned long long* d_cur = reinterpret_cast<unsigned long long*>(d_all + size_t(world) * world);
  hm_status s = route_count_launch(keys, n_local, l1, world, d_c, st);
  if (s != HM_OK) return s;
  HM_NCCL_TRY(ncclAllGather(d_c, d_all, world, ncclUint64, comm, st));
  std::vector<uint64_t> C(size_t(world) * world);
  HM_CUDA_TRY(cudaMemcpyAsync(C.data(), d_all, C.size() * 8, cudaMemcpyDeviceToHost, st));
  HM_CUDA_TRY(cudaStreamSynchronize(st));
  uint64_t cap = 0, mine = 0;
  std::vector<uint64_t> off(world, 0);  // where this rank's run starts in every owner's buffer
  if ((s = hm_dist_exchange_plan(C.data(), world, rank, off.data(), &cap, &mine)) != HM_OK) return s;
  RecvWindow* w = nullptr;
  if ((s = window_for(comm, cap, &w)) != HM_OK) return s;
  HM_CUDA_TRY(cudaMemcpyAsync(d_cur, off.data(), size_t(world) * 8, cudaMemcpyHostToDevice, st));
  if (n_local) {
    LaunchScope ls_("k_route_scatter_win", st);
    const unsigned gs =
        unsigned(std::max<uint64_t>(1, std::min<uint64_t>((n_local + kRTile - 1) / kRTile, uint64_t(num_sms()) * 2)));
    k_route_scatter_win<<<gs, kRThreads, 0, st>>>(keys, vals, n_local, l1, world, d_cur, OutWindow{w->win, w->cap * 8});
  }
  HM_CUDA_TRY(cudaGetLastError());
  // every rank's stores have landed once every rank's scatter is done
  HM_NCCL_TRY(ncclAllReduce(d_small + 3, d_small + 3, 1, ncclUint64, ncclSum, comm, st));
  cudaFreeAsync(d_c, st);
  *rk = static_cast<const uint64_t*>(w->buf);
  *rv = static_cast<const uint64_t*>(w->buf) + w->cap;
  *nrecv = mine;
  return HM_OK;
}

}  // namespace
}  // namespace hm

using namespace hm;

extern "C" {

hm_status hm_build_u64_dist(const uint64_t* keys, const uint64_t* vals, uint64_t n_local, const hm_opts* opts,
                            void* stream, void* nccl_comm, hm_map** out) {
  if (!out || !nccl_comm || (n_local && (!keys || !vals))) return HM_ERR_INVALID_ARG;
  *out = nullptr;
  ncclComm_t comm = static_cast<ncclComm_t>(nccl_comm);
  int world = 0, rank = 0;
  HM_NCCL_TRY(ncclCommCount(comm, &world));
  HM_NCCL_TRY(ncclCommUserRank(comm, &rank));
  if (world < 1 || world > 64) return HM_ERR_INVALID_ARG;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  DevBufs db{st, {}};
  hm_status s;
  uint64_t *d_small, *sk = nullptr, *sv = nullptr;
  if ((s = db.get(&d_small, 4 + 2 * size_t(world) + size_t(world))) != HM_OK) return s;
  uint64_t* d_sc = d_small + 4;
  uint64_t* d_rc = d_sc + world;
  uint64_t* d_sall = d_rc + world;
  // (1) the global n
  HM_CUDA_TRY(cudaMemcpyAsync(d_small, &n_local, 8, cudaMemcpyHostToDevice, st));
  HM_NCCL_TRY(ncclAllReduce(d_small, d_small, 1, ncclUint64, ncclSum, comm, st));
  uint64_t n = 0;
  HM_CUDA_TRY(cudaMemcpyAsync(&n, d_small, 8, cudaMemcpyDeviceToHost, st));
  HM_CUDA_TRY(cudaStreamSynchronize(st));
  if (n == 0) return HM_ERR_EMPTY;
  if (n > (1ull << 30)) return HM_ERR_TOO_LARGE;
  uint64_t lo = 0, hi = 0;
  if ((s = hm_dist_bucket_range(n, world, rank, &lo, &hi)) != HM_OK) return s;
  const uint64_t seed = opts ? opts->seed : 0;
  const bool fused = opts && (opts->flags & HM_FLAG_FUSED_EXCHANGE);
  hm_opts shard_opts{};
  if (opts) {
    shard_opts = *opts;
    shard_opts.flags &= ~uint32_t(HM_FLAG_FUSED_EXCHANGE);
  }
  if (!fused && ((s = db.get(&sk, n_local)) != HM_OK || (s = db.get(&sv, n_local)) != HM_OK)) return s;
  hm_map* m = nullptr;
  uint64_t S_local = 0;
  HM_CUDA_TRY(cudaMemsetAsync(d_small + 3, 0, 8, st));
  for (uint32_t t1 = 0;;) {
    // (2) route, exchange counts and pairs (fused: straight into the owners' windows)
    DevBufs rb{st, {}};
    const uint64_t *rk = nullptr, *rv = nullptr;
    uint64_t nrecv = 0;
    if (fused) {
      const L1Params l1 = make_l1(seed_mix(seed), t1, n);
      if ((s = fused_exchange(keys, vals, n_local, l1, world, rank, comm, st, d_small, &rk, &rv, &nrecv)) != HM_OK)
        return s;
    } else {
      if ((s = hm_route_u64(keys, vals, n_local, n, seed, t1, world, sk, sv, d_sc, stream)) != HM_OK) return s;
      std::vector<uint64_t> sc, rc;
      if ((s = exchange_counts(d_sc, d_rc, sc, rc, world, comm, st)) != HM_OK) return s;
      for (uint64_t x : rc) nrecv += x;
      uint64_t *bk, *bv;
      if ((s = rb.get(&bk, nrecv)) != HM_OK || (s = rb.get(&bv, nrecv)) != HM_OK) return s;
      if ((s = all_to_all_v(sk, sc, bk, rc, 8, world, comm, st)) != HM_OK) return s;
      if ((s = all_to_all_v(sv, sc, bv, rc, 8, world, comm, st)) != HM_OK) return s;
      rk = bk;
      rv = bv;
    }
    // (3) the shard, then the global bound and the status, agreed by all ranks
    const hm_status bs = hm_build_u64_shard(rk, rv, nrecv, n, lo, hi, t1, opts ? &shard_opts : nullptr, stream, &m,
                                            &S_local);
    // (fused: the shard build has copied the window's pairs; the window stays
    // registered for the next build)
    const std::string local_err = bs != HM_OK ? hm_last_error() : std::string();
    uint64_t red[2] = {bs == HM_OK ? S_local : 0, uint64_t(bs)};
    HM_CUDA_TRY(cudaMemcpyAsync(d_small, red, 16, cudaMemcpyHostToDevice, st));
    HM_NCCL_TRY(ncclAllReduce(d_small, d_small, 1, ncclUint64, ncclSum, comm, st));
    HM_NCCL_TRY(ncclAllReduce(d_small + 1, d_small + 1, 1, ncclUint64, ncclMax, comm, st));
    HM_CUDA_TRY(cudaMemcpyAsync(red, d_small, 16, cudaMemcpyDeviceToHost, st));
    HM_CUDA_TRY(cudaStreamSynchronize(st));
    const int d = hm_dist_decide(n, t1, red[0], int(red[1]), &t1);
    if (d == HM_OK) break;
    hm_free(m);
    m = nullptr;
    if (d != HM_DIST_REDRAW) {
      if (red[1] != 0)
        set_error(local_err.empty() ? "a shard build failed on another rank (max status over ranks)" : local_err);
      return hm_status(d);
    }
  }
  // (4) the slot base: exclusive prefix of S_r
  HM_CUDA_TRY(cudaMemcpyAsync(d_small + 2, &S_local, 8, cudaMemcpyHostToDevice, st));
  HM_NCCL_TRY(ncclAllGather(d_small + 2, d_sall, 1, ncclUint64, comm, st));
  std::vector<uint64_t> sall(world);
  HM_CUDA_TRY(cudaMemcpyAsync(sall.data(), d_sall, world * 8, cudaMemcpyDeviceToHost, st));
  HM_CUDA_TRY(cudaStreamSynchronize(st));
  const uint64_t base = hm_dist_slot_base(sall.data(), world, rank);
  if ((s = hm_shard_set_base(m, base)) != HM_OK) {
    hm_free(m);
    return s;
  }
  *out = m;
  return HM_OK;
}

hm_status hm_dist_release_windows(void* nccl_comm) {
  if (!nccl_comm) return HM_ERR_INVALID_ARG;
  std::lock_guard<std::mutex> lk(g_win_mu);
  auto it = g_win.find(static_cast<ncclComm_t>(nccl_comm));
  if (it == g_win.end()) return HM_OK;
  const hm_status s = it->second.release();
  g_win.erase(it);
  return s;
}

hm_status hm_lookup_u64_dist(const hm_map* shard, const uint64_t* q, uint64_t nq, uint64_t* out_vals,
                             uint8_t* out_found, void* stream, void* nccl_comm) {
  if (!shard || !nccl_comm || (nq && !q) || (!out_vals && !out_found)) return HM_ERR_INVALID_ARG;
  ncclComm_t comm = static_cast<ncclComm_t>(nccl_comm);
  int world = 0;
  HM_NCCL_TRY(ncclCommCount(comm, &world));
  if (world < 1 || world > 64) return HM_ERR_INVALID_ARG;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  DevBufs db{st, {}};
  hm_status s;
  uint64_t *d_c, *sq, *perm;
  if ((s = db.get(&d_c, 2 * size_t(world))) != HM_OK || (s = db.get(&sq, nq)) != HM_OK ||
      (s = db.get(&perm, nq)) != HM_OK)
    return s;
  if ((s = hm_route_queries_u64(shard, q, nq, world, sq, perm, d_c, stream)) != HM_OK) return s;
  std::vector<uint64_t> sc, rc;
  if ((s = exchange_counts(d_c, d_c + world, sc, rc, world, comm, st)) != HM_OK) return s;
  uint64_t nrecv = 0;
  for (uint64_t x : rc) nrecv += x;
  uint64_t *rq, *rv, *bv;
  uint8_t *rf, *bf;
  if ((s = db.get(&rq, nrecv)) != HM_OK || (s = db.get(&rv, nrecv)) != HM_OK || (s = db.get(&rf, nrecv)) != HM_OK ||
      (s = db.get(&bv, nq)) != HM_OK || (s = db.get(&bf, nq)) != HM_OK)
    return s;
  if ((s = all_to_all_v(sq, sc, rq, rc, 8, world, comm, st)) != HM_OK) return s;
  if (nrecv && (s = hm_lookup_u64(shard, rq, nrecv, rv, rf, stream)) != HM_OK) return s;
  // the answers travel back along the reverse splits
  if ((s = all_to_all_v(rv, rc, bv, sc, 8, world, comm, st)) != HM_OK) return s;
  if ((s = all_to_all_v(rf, rc, bf, sc, 1, world, comm, st)) != HM_OK) return s;
  return hm_unroute_u64(bv, bf, perm, nq, out_vals, out_found, stream);
}

}  // extern "C"
