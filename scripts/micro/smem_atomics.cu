// Microbenchmark: shared-memory atomicAdd throughput (random spread addresses,
// 2048 u32 counters) vs. ballot-rank and match.any, per SM on this B200.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t rng(uint32_t x) { x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x; }
template <int MODE>
__global__ void k(int iters, uint32_t* out) {
  __shared__ uint32_t cnt[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) cnt[i] = 0;
  __syncthreads();
  uint32_t x = rng(threadIdx.x * 7919 + blockIdx.x * 104729), acc = 0;
  for (int it = 0; it < iters; it++) {
    x = rng(x + it);
    const uint32_t b = x & 2047;
    if (MODE == 0) acc += atomicAdd(&cnt[b], 1u);                 // ATOMS with return
    else if (MODE == 1) atomicAdd(&cnt[b], 1u);                   // RED-like (no use of return)
    else if (MODE == 2) acc += __match_any_sync(0xffffffffu, b);  // match.any
    else if (MODE == 3) {                                         // 11 ballots
      uint32_t m = 0xffffffffu;
#pragma unroll
      for (int bit = 0; bit < 11; bit++) { uint32_t bl = __ballot_sync(0xffffffffu, (b >> bit) & 1); m &= ((b >> bit) & 1) ? bl : ~bl; }
      acc += m;
    } else acc += cnt[b];                                         // plain LDS
  }
  __syncthreads();
  if (acc == 0x12345) out[0] = acc + cnt[threadIdx.x & 2047];
}
int main() {
  uint32_t* d; cudaMalloc(&d, 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const char* nm[] = {"ATOMS(ret)", "ATOMS(noret)", "MATCH.ANY", "11 ballots", "LDS"};
  for (int mode = 0; mode < 5; mode++) for (int th : {512, 1024}) {
    const int iters = 4096, blocks = sms * (2048 / th);
    for (int r = 0; r < 2; r++) {
      cudaEventRecord(a);
      switch (mode) { case 0: k<0><<<blocks, th>>>(iters, d); break; case 1: k<1><<<blocks, th>>>(iters, d); break;
        case 2: k<2><<<blocks, th>>>(iters, d); break; case 3: k<3><<<blocks, th>>>(iters, d); break; default: k<4><<<blocks, th>>>(iters, d); }
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      const double ops = double(blocks) * th * iters;
      if (r) printf("%-14s threads/CTA %4d: %.3f ms, %.2f Gops/s chip, %.2f SM-cycles per warp-op @1.965GHz\n", nm[mode], th, ms, ops / ms / 1e6,
                    (ms * 1e-3 * 1.965e9) / (ops / 32 / sms));
    }
  }
  return 0;
}
