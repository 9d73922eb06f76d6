// qk-normalisation ("We use qk-normalization when needed";
// reading Q12 in DESIGN.md: each query half and each half-key row is
// L2-normalised at score time, x / max(||x||, 1e-6), non-learned).
// The raw products stay on the tensor cores; the normalisation is applied as
// fp32 scale factors: s = (q.k) * inv_q * inv_k.  Backward: the selected
// score gradients are scaled by inv_q * inv_k (so the products give
// G = inv * d(x_hat)) and projected: dx = G - x_hat (x_hat . G) (or G when
// ||x|| <= eps).
#include "internal.cuh"

namespace ml {
namespace {

constexpr float kQkEps = 1e-6f;

// one warp per row of Dh elements: inv[r] = 1 / max(||x_r||, eps)
template <typename T>
__global__ void row_inv_norm_kernel(const T* x, int64_t rows, int Dh, float* inv) {
  const int64_t r = int64_t(blockIdx.x) * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const T* xr = x + r * Dh;
  float ss = 0.f;
  for (int c = lane; c < Dh; c += 32) {
    const float v = to_f(xr[c]);
    ss = fmaf(v, v, ss);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if (lane == 0) inv[r] = 1.f / fmaxf(sqrtf(ss), kQkEps);
}

// out[r] (=|+=) G[r] - x_hat (x_hat . G[r]),  x_hat = x[r] / max(||x[r]||, eps)
template <typename T>
__global__ void qk_proj_kernel(const T* x, int64_t rows, int Dh, const float* G, float* out,
                               int accumulate) {
  const int64_t r = int64_t(blockIdx.x) * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const T* xr = x + r * Dh;
  const float* gr = G + r * Dh;
  float ss = 0.f, dot = 0.f;
  for (int c = lane; c < Dh; c += 32) {
    const float v = to_f(xr[c]);
    ss = fmaf(v, v, ss);
    dot = fmaf(v, gr[c], dot);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ss += __shfl_xor_sync(0xffffffffu, ss, o);
    dot += __shfl_xor_sync(0xffffffffu, dot, o);
  }
  const float n = sqrtf(ss);
  const bool proj = n > kQkEps;
  const float inv = 1.f / fmaxf(n, kQkEps);
  const float c = dot * inv;                 // x_hat . G
  float* orow = out + r * Dh;
  for (int e = lane; e < Dh; e += 32) {
    const float res = proj ? gr[e] - to_f(xr[e]) * inv * c : gr[e];
    orow[e] = accumulate ? orow[e] + res : res;
  }
}

}  // namespace

mlStatus launch_row_inv_norm(const void* x, int64_t rows, int Dh, mlDtype dt, float* inv,
                             cudaStream_t s) {
  if (rows <= 0) return ML_OK;
  const unsigned grid = unsigned((rows + 7) / 8);
  if (dt == ML_BF16)
    row_inv_norm_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(x), rows, Dh, inv);
  else
    row_inv_norm_kernel<float><<<grid, 256, 0, s>>>(static_cast<const float*>(x), rows, Dh, inv);
  ML_LAUNCH_CHECK("qk_inv_norm");
  return ML_OK;
}

mlStatus launch_qk_proj(const void* x, int64_t rows, int Dh, mlDtype dt, const float* G, float* out,
                        bool accumulate, cudaStream_t s) {
  if (rows <= 0) return ML_OK;
  const unsigned grid = unsigned((rows + 7) / 8);
  if (dt == ML_BF16)
    qk_proj_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(x), rows, Dh, G, out,
                                                       accumulate ? 1 : 0);
  else
    qk_proj_kernel<float><<<grid, 256, 0, s>>>(static_cast<const float*>(x), rows, Dh, G, out,
                                               accumulate ? 1 : 0);
  ML_LAUNCH_CHECK("qk_proj");
  return ML_OK;
}

}  // namespace ml
