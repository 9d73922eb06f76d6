// HBM ceilings for the access mixes of the hot kernels (diagnostic, not product code):
// read-only, write-only (16 B and 32 B stores, with/without evict_first), and
// "bf16 read -> fp32 write" (1:2 bytes, the segmented backward's V -> dV mix).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
__device__ __forceinline__ uint64_t pol_first() {
  uint64_t p; asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p)); return p;
}
__global__ void wr16(uint4* q, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, s = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += s) q[i] = make_uint4(i, 1, 2, 3);
}
__global__ void wr32(uint4* q, size_t n, int hint) {   // n in 32-byte units
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, s = (size_t)gridDim.x * blockDim.x;
  const uint64_t pol = pol_first();
  for (; i < n; i += s) {
    uint4* o = q + 2 * i;
    if (hint)
      asm volatile("st.global.L2::cache_hint.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8}, %9;" ::"l"(o),
                   "r"(unsigned(i)), "r"(1u), "r"(2u), "r"(3u), "r"(4u), "r"(5u), "r"(6u), "r"(7u), "l"(pol) : "memory");
    else
      asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(o),
                   "r"(unsigned(i)), "r"(1u), "r"(2u), "r"(3u), "r"(4u), "r"(5u), "r"(6u), "r"(7u) : "memory");
  }
}
// each thread: read 16 B of bf16 (8 values), write 32 B of fp32
__global__ void cvt(const uint4* __restrict__ p, uint4* q, size_t n, int hint) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, s = (size_t)gridDim.x * blockDim.x;
  const uint64_t pol = pol_first();
  for (; i < n; i += s) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p + i), "l"(pol));
    unsigned w[8] = {v.x << 16, v.x & 0xffff0000u, v.y << 16, v.y & 0xffff0000u,
                     v.z << 16, v.z & 0xffff0000u, v.w << 16, v.w & 0xffff0000u};
    uint4* o = q + 2 * i;
    if (hint)
      asm volatile("st.global.L2::cache_hint.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8}, %9;" ::"l"(o),
                   "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]), "l"(pol) : "memory");
    else
      asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(o),
                   "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]) : "memory");
  }
}
int main() {
  const size_t bytes = (size_t)8 << 30;
  uint4 *p, *q;
  cudaMalloc(&p, bytes); cudaMalloc(&q, bytes);
  cudaMemset(p, 1, bytes); cudaMemset(q, 1, bytes);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto timeit = [&](auto fn) {
    float best = 1e9;
    for (int r = 0; r < 6; ++r) {
      cudaEventRecord(a); fn(); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); if (r && ms < best) best = ms;
    }
    return best;
  };
  for (int bps : {4, 8}) {
    float ms = timeit([&] { wr16<<<sms * bps, 512>>>(q, bytes / 16); });
    printf("write-only 16B %d blk/SM: %.3f ms = %.0f GB/s\n", bps, ms, bytes / ms / 1e6);
    for (int h : {0, 1}) {
      ms = timeit([&] { wr32<<<sms * bps, 512>>>(q, bytes / 32, h); });
      printf("write-only 32B hint=%d %d blk/SM: %.3f ms = %.0f GB/s\n", h, bps, ms, bytes / ms / 1e6);
    }
    for (int h : {0, 1}) {
      // read bytes/2... write 'bytes': 16 B read + 32 B write per thread-iteration
      ms = timeit([&] { cvt<<<sms * bps, 512>>>(p, q, bytes / 32, h); });
      printf("bf16->fp32 (r:w 1:2) hint=%d %d blk/SM: %.3f ms = %.0f GB/s (r+w)\n", h, bps, ms,
             1.5 * bytes / ms / 1e6);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
