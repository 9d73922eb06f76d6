// Counter-based synthetic inputs; an independent CUDA
// implementation of the generator in synthetic/gen.py (checked bit for bit by
// tests/test_gpu_synth.py).  Not method arithmetic: it only produces inputs.
#include "internal.cuh"

namespace ml {
namespace {

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

template <typename T>
__global__ void synth_kernel(T* out, int64_t n_rows, int64_t n_cols, int64_t row0, uint64_t base,
                             float scale, int cls) {
  const int64_t n = n_rows * n_cols;
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
       e += int64_t(gridDim.x) * blockDim.x) {
    const uint64_t i = uint64_t(row0) * uint64_t(n_cols) + uint64_t(e);
    const uint64_t u = splitmix64(base + i);
    float f;
    if (cls == 0) f = float(int64_t(u >> 40) - (int64_t(1) << 23)) * (1.0f / 8388608.0f);
    else if (cls == 1) f = float(int64_t((u >> 60) & 15u) - 8) * 0.125f;
    else f = float(int64_t((u >> 58) & 63u)) * (1.0f / 64.0f);
    const float v = __fmul_rn(f, scale);
    if constexpr (sizeof(T) == 2) out[e] = __float2bfloat16_rn(v);
    else out[e] = v;
  }
}

__global__ void synth_index_kernel(int32_t* out, int64_t n_rows, int64_t n_cols, int64_t row0,
                                   uint64_t base, uint64_t modulus) {
  const int64_t n = n_rows * n_cols;
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
       e += int64_t(gridDim.x) * blockDim.x) {
    const uint64_t i = uint64_t(row0) * uint64_t(n_cols) + uint64_t(e);
    out[e] = int32_t(splitmix64(base + i) % modulus);
  }
}

}  // namespace

mlStatus launch_synth(void* out, int64_t n_rows, int64_t n_cols, int64_t row0, uint64_t seed,
                      uint32_t tag, float scale, int cls, mlDtype dt, int64_t modulus,
                      cudaStream_t s) {
  if (n_rows <= 0 || n_cols <= 0) return ML_OK;
  if (cls < 0 || cls > 3) return fail(ML_ERR_ARG, "synth: unknown class");
  const uint64_t base = seed * 0x9E3779B97F4A7C15ull + uint64_t(tag) * 0xD1B54A32D192ED03ull;
  const int64_t n = n_rows * n_cols;
  const unsigned grid = unsigned(std::min<int64_t>((n + 255) / 256, int64_t(num_sms()) * 32));
  if (cls == 3) {
    if (modulus <= 0) return fail(ML_ERR_ARG, "synth: index class needs a positive modulus");
    synth_index_kernel<<<grid, 256, 0, s>>>(static_cast<int32_t*>(out), n_rows, n_cols, row0, base,
                                            uint64_t(modulus));
  } else if (dt == ML_BF16) {
    synth_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>(static_cast<__nv_bfloat16*>(out), n_rows,
                                                     n_cols, row0, base, scale, cls);
  } else {
    synth_kernel<float><<<grid, 256, 0, s>>>(static_cast<float*>(out), n_rows, n_cols, row0, base,
                                             scale, cls);
  }
  ML_LAUNCH_CHECK("synth");
  return ML_OK;
}

}  // namespace ml
