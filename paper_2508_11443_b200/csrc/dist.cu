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

#include <algorithm>
#include <string>
#include <vector>

#include "hm_internal.cuh"

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
  if ((s = db.get(&sk, n_local)) != HM_OK || (s = db.get(&sv, n_local)) != HM_OK) return s;
  hm_map* m = nullptr;
  uint64_t S_local = 0;
  for (uint32_t t1 = 0;;) {
    // (2) route, exchange counts and pairs
    if ((s = hm_route_u64(keys, vals, n_local, n, seed, t1, world, sk, sv, d_sc, stream)) != HM_OK) return s;
    std::vector<uint64_t> sc, rc;
    if ((s = exchange_counts(d_sc, d_rc, sc, rc, world, comm, st)) != HM_OK) return s;
    uint64_t nrecv = 0;
    for (uint64_t x : rc) nrecv += x;
    DevBufs rb{st, {}};
    uint64_t *rk, *rv;
    if ((s = rb.get(&rk, nrecv)) != HM_OK || (s = rb.get(&rv, nrecv)) != HM_OK) return s;
    if ((s = all_to_all_v(sk, sc, rk, rc, 8, world, comm, st)) != HM_OK) return s;
    if ((s = all_to_all_v(sv, sc, rv, rc, 8, world, comm, st)) != HM_OK) return s;
    // (3) the shard, then the global bound and the status, agreed by all ranks
    const hm_status bs = hm_build_u64_shard(rk, rv, nrecv, n, lo, hi, t1, opts, stream, &m, &S_local);
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
