#include <cstdio>
#include <cuda_runtime.h>
__global__ void rd(const uint4* __restrict__ p, size_t n, unsigned* out) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  unsigned acc = 0;
  for (; i + 3 * stride < n; i += 4 * stride) {
    uint4 a, b, c, d;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w) : "l"(p + i));
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w) : "l"(p + i + stride));
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(c.x), "=r"(c.y), "=r"(c.z), "=r"(c.w) : "l"(p + i + 2 * stride));
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(d.x), "=r"(d.y), "=r"(d.z), "=r"(d.w) : "l"(p + i + 3 * stride));
    acc ^= a.x ^ b.y ^ c.z ^ d.w;
  }
  if (acc == 0x12345678) *out = acc;
}
__global__ void cp(const uint4* __restrict__ p, uint4* q, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) q[i] = p[i];
}
int main() {
  size_t bytes = (size_t)8 << 30; size_t n = bytes / 16;
  uint4 *p, *q; unsigned* o;
  cudaMalloc(&p, bytes); cudaMalloc(&q, bytes / 2); cudaMalloc(&o, 4);
  cudaMemset(p, 1, bytes);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int blocks_per_sm : {4, 8, 16}) {
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(a); rd<<<sms * blocks_per_sm, 512>>>(p, n, o); cudaEventRecord(b);
      cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
    }
    printf("read-only %d blk/SM: %.3f ms = %.0f GB/s\n", blocks_per_sm, best, bytes / best / 1e6);
  }
  float best = 1e9;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a); cp<<<sms * 8, 512>>>(p, q, n / 2); cudaEventRecord(b);
    cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
  }
  printf("copy 4 GiB: %.3f ms = %.0f GB/s (r+w)\n", best, bytes / best / 1e6);
  return 0;
}
