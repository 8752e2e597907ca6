// Random 8-byte gathers over a 4 GiB array with different load flavours:
// how many DRAM bytes does each fetch?
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint64_t mixr(uint64_t z){z=(z^(z>>30))*0xBF58476D1CE4E5B9ull;z=(z^(z>>27))*0x94D049BB133111EBull;return z^(z>>31);}
template<int F> __device__ __forceinline__ uint64_t ld(const uint64_t* p){
  uint64_t v;
  if (F==0) asm volatile("ld.global.ca.u64 %0,[%1];":"=l"(v):"l"(p));
  if (F==1) asm volatile("ld.global.cg.u64 %0,[%1];":"=l"(v):"l"(p));
  if (F==2) asm volatile("ld.global.cs.u64 %0,[%1];":"=l"(v):"l"(p));
  if (F==3) asm volatile("ld.global.cv.u64 %0,[%1];":"=l"(v):"l"(p));
  if (F==4) asm volatile("ld.global.nc.u64 %0,[%1];":"=l"(v):"l"(p));
  if (F==5) asm volatile("ld.relaxed.gpu.global.u64 %0,[%1];":"=l"(v):"l"(p));
  if (F==6) asm volatile("ld.global.lu.u64 %0,[%1];":"=l"(v):"l"(p));
  if (F==8) asm volatile("ld.global.nc.L2::64B.u64 %0,[%1];":"=l"(v):"l"(p));
  if (F==9) asm volatile("ld.global.L2::64B.u64 %0,[%1];":"=l"(v):"l"(p));
  if (F==10) asm volatile("ld.global.nc.L1::no_allocate.L2::64B.u64 %0,[%1];":"=l"(v):"l"(p));
  if (F==11) asm volatile("ld.global.cg.L2::64B.u64 %0,[%1];":"=l"(v):"l"(p));
  if (F==12) asm volatile("ld.global.nc.L2::128B.u64 %0,[%1];":"=l"(v):"l"(p));
  if (F==7) { uint64_t pol; asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;":"=l"(pol)); asm volatile("ld.global.L2::cache_hint.u64 %0,[%1], %2;":"=l"(v):"l"(p),"l"(pol)); }
  return v;
}
template<int F> __global__ void k(const uint64_t* a, uint64_t n, uint64_t m, uint64_t* out){
  uint64_t acc=0;
  for (uint64_t i = blockIdx.x*(uint64_t)blockDim.x+threadIdx.x; i < m; i += (uint64_t)gridDim.x*blockDim.x){
    uint64_t j = mixr(i*0x9E3779B97F4A7C15ull+F) % n;
    acc += ld<F>(a + j);
  }
  if (acc == 42) out[0] = acc;
}
// cp.async 8-byte gather into smem
__global__ void kca(const uint64_t* a, uint64_t n, uint64_t m, uint64_t* out){
  __shared__ uint64_t buf[256];
  uint64_t acc=0;
  for (uint64_t i = blockIdx.x*(uint64_t)blockDim.x+threadIdx.x; i < m; i += (uint64_t)gridDim.x*blockDim.x){
    uint64_t j = mixr(i*0x9E3779B97F4A7C15ull+9) % n;
    unsigned sa = (unsigned)__cvta_generic_to_shared(&buf[threadIdx.x]);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;"::"r"(sa),"l"(a+j));
    asm volatile("cp.async.wait_all;");
    acc += buf[threadIdx.x];
  }
  if (acc == 42) out[0] = acc;
}
int main(){
  uint64_t n = (4ull<<30)/8, m = 1ull<<26;
  uint64_t *a, *o; cudaMalloc(&a, n*8); cudaMalloc(&o, 8); cudaMemset(a, 1, n*8);
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
#define RUN(K,name) K<<<148*8,256>>>(a,n,m,o); cudaEventRecord(e0); K<<<148*8,256>>>(a,n,m,o); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms,e0,e1); printf("%-12s %7.3f ms  %6.2f Gld/s\n", name, ms, m/ms/1e6);
  RUN(k<0>,"ca") RUN(k<1>,"cg") RUN(k<2>,"cs") RUN(k<3>,"cv") RUN(k<4>,"nc") RUN(k<5>,"relaxed") RUN(k<6>,"lu") RUN(k<7>,"evict_first") RUN(kca,"cp.async8")
  RUN(k<8>,"nc.L2::64B") RUN(k<9>,"L2::64B") RUN(k<10>,"nc.noal.L2::64B") RUN(k<11>,"cg.L2::64B") RUN(k<12>,"nc.L2::128B")
  return 0;
}
