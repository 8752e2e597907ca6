// gen_cuda.cu — device copy of the seeded workload recipe of workloads/gen.py
// (DESIGN.md §3), for the multi-GiB bench inputs.  Holds none of the method's
// arithmetic: only the splitmix64 key stream and the murmur3 fmix32 prefix.
#include <cstdint>

namespace {
constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ull;
constexpr uint64_t kSalt = 0xA0761D6478BD642Full;

__host__ __device__ __forceinline__ uint64_t out64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t stream_at(uint64_t start, uint64_t i) { return out64(start + kGamma * (i + 1)); }
__device__ __forceinline__ uint32_t fmix32(uint32_t h) {
  h ^= h >> 16; h *= 0x85EBCA6Bu; h ^= h >> 13; h *= 0xC2B2AE35u; h ^= h >> 16;
  return h;
}

__global__ void k_u64_keys(uint64_t start, uint64_t lo, uint64_t n, uint64_t* out, uint64_t* vals) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
    out[i] = stream_at(start, lo + i);
    if (vals) vals[i] = lo + i;
  }
}

// queries j in [lo, lo+nq): r = stream(SEED_Q, j); idx = (r mod 2^63) mod n;
// member key_idx if r>>63 == 0 else absent key_{n+idx}
__global__ void k_queries(uint64_t start_k, uint64_t start_q, uint64_t n, uint64_t lo, uint64_t nq, uint64_t* q,
                          uint64_t* expv, uint8_t* expf) {
  for (uint64_t j = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; j < nq; j += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t r = stream_at(start_q, lo + j);
    const uint64_t idx = (r & ((1ull << 63) - 1)) % n;
    const bool member = (r >> 63) == 0;
    q[j] = stream_at(start_k, member ? idx : idx + n);
    if (expv) expv[j] = member ? idx : 0;
    if (expf) expf[j] = member ? 1 : 0;
  }
}

// string ids (member i or absent n+idx) for queries; ids for members = lo + i
__global__ void k_query_ids(uint64_t start_q, uint64_t n, uint64_t lo, uint64_t nq, uint64_t* ids) {
  for (uint64_t j = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; j < nq; j += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t r = stream_at(start_q, lo + j);
    const uint64_t idx = (r & ((1ull << 63) - 1)) % n;
    ids[j] = (r >> 63) == 0 ? idx : idx + n;
  }
}

__global__ void k_str_lens(uint64_t start_l, const uint64_t* ids, uint64_t lo, uint64_t n, int64_t* lens,
                           uint64_t lmin, uint64_t lspan) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t id = ids ? ids[i] : lo + i;
    lens[i] = int64_t(lmin + stream_at(start_l, id) % lspan);
  }
}

// one thread per string: bytes[0:4] = LE fmix32(id), bytes[4:len] = LE bytes of stream(SEED_B, 8 id + w)
__global__ void k_str_bytes(uint64_t start_b, const uint64_t* ids, uint64_t lo, uint64_t n, const uint64_t* offs,
                            uint8_t* ctx) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t id = ids ? ids[i] : lo + i;
    const uint64_t o = offs[i], len = offs[i + 1] - o;
    uint8_t* p = ctx + o;
    const uint32_t h = fmix32(uint32_t(id));
    for (uint64_t b = 0; b < len; b++) {
      uint8_t v;
      if (b < 4) v = uint8_t(h >> (8 * b));
      else {
        const uint64_t w = stream_at(start_b, 8 * id + (b - 4) / 8);
        v = uint8_t(w >> (8 * ((b - 4) % 8)));
      }
      p[b] = v;
    }
  }
}
}  // namespace

extern "C" {
uint64_t hg_stream_start(uint64_t s) { return out64(s ^ kSalt); }
int hg_u64_keys(uint64_t seed_k, uint64_t lo, uint64_t n, uint64_t* out, uint64_t* vals, void* stream) {
  if (!n) return 0;
  k_u64_keys<<<1184, 256, 0, (cudaStream_t)stream>>>(hg_stream_start(seed_k), lo, n, out, vals);
  return (int)cudaGetLastError();
}
int hg_queries(uint64_t seed_k, uint64_t seed_q, uint64_t n, uint64_t lo, uint64_t nq, uint64_t* q, uint64_t* expv,
               uint8_t* expf, void* stream) {
  if (!nq) return 0;
  k_queries<<<1184, 256, 0, (cudaStream_t)stream>>>(hg_stream_start(seed_k), hg_stream_start(seed_q), n, lo, nq, q,
                                                     expv, expf);
  return (int)cudaGetLastError();
}
int hg_query_ids(uint64_t seed_q, uint64_t n, uint64_t lo, uint64_t nq, uint64_t* ids, void* stream) {
  if (!nq) return 0;
  k_query_ids<<<1184, 256, 0, (cudaStream_t)stream>>>(hg_stream_start(seed_q), n, lo, nq, ids);
  return (int)cudaGetLastError();
}
// lengths lmin + stream(SEED_L, id) mod lspan (the default recipe: 4 + mod 61, i.e. 4..64 bytes;
// the paper's Table 1 shape: 5 + mod 21, i.e. 5..25)
int hg_str_lens(uint64_t seed_l, const uint64_t* ids, uint64_t lo, uint64_t n, int64_t* lens, void* stream,
                uint64_t lmin, uint64_t lspan) {
  if (!n) return 0;
  k_str_lens<<<1184, 256, 0, (cudaStream_t)stream>>>(hg_stream_start(seed_l), ids, lo, n, lens, lmin, lspan);
  return (int)cudaGetLastError();
}
int hg_str_bytes(uint64_t seed_b, const uint64_t* ids, uint64_t lo, uint64_t n, const uint64_t* offs, uint8_t* ctx,
                 void* stream) {
  if (!n) return 0;
  k_str_bytes<<<1184, 256, 0, (cudaStream_t)stream>>>(hg_stream_start(seed_b), ids, lo, n, offs, ctx);
  return (int)cudaGetLastError();
}
}
