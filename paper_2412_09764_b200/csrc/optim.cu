// Sparse (lazy, row-wise) Adam(W) on the touched memory-value rows (SURVEY
// f1): consumes the compact value gradient of
// the "reverse_indices" backward directly -- no dense gradient, no memset.
//   c = ++steps[r]; m = b1 m + (1-b1) g; v = b2 v + (1-b2) g^2;
//   V[r] -= lr * ( m/(1-b1^c) / (sqrt(v/(1-b2^c)) + eps) + wd * V[r] )
// Rows are distinct, so every row is owned by one CTA (no atomics).
#include "internal.cuh"

namespace ml {
namespace {

__device__ __forceinline__ float4 grad4(const float* p, int64_t i) {
  return *reinterpret_cast<const float4*>(p + i);
}
__device__ __forceinline__ float4 grad4(const __nv_bfloat16* p, int64_t i) {
  const uint2 u = *reinterpret_cast<const uint2*>(p + i);
  const float2 a = bf2_to_f2(u.x), b = bf2_to_f2(u.y);
  return make_float4(a.x, a.y, b.x, b.y);
}

// 8 consecutive elements per thread and iteration (two float4 of m, v and the
// gradient, one 16-byte vector of a bf16 table row): every access is a full
// vector, and a 2048-wide row is one pass of 256 threads
template <typename T>
__device__ __forceinline__ void load8(const T* p, float* f);
template <>
__device__ __forceinline__ void load8<float>(const float* p, float* f) {
  const float4 a = reinterpret_cast<const float4*>(p)[0], b = reinterpret_cast<const float4*>(p)[1];
  f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w; f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
}
template <>
__device__ __forceinline__ void load8<__nv_bfloat16>(const __nv_bfloat16* p, float* f) {
  const uint4 u = *reinterpret_cast<const uint4*>(p);
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float2 t = bf2_to_f2(w[e]);
    f[2 * e] = t.x;
    f[2 * e + 1] = t.y;
  }
}
template <typename T>
__device__ __forceinline__ void store8(T* p, const float* f);
template <>
__device__ __forceinline__ void store8<float>(float* p, const float* f) {
  reinterpret_cast<float4*>(p)[0] = make_float4(f[0], f[1], f[2], f[3]);
  reinterpret_cast<float4*>(p)[1] = make_float4(f[4], f[5], f[6], f[7]);
}
template <>
__device__ __forceinline__ void store8<__nv_bfloat16>(__nv_bfloat16* p, const float* f) {
  *reinterpret_cast<uint4*>(p) = make_uint4(f2_to_bf2(f[0], f[1]), f2_to_bf2(f[2], f[3]),
                                            f2_to_bf2(f[4], f[5]), f2_to_bf2(f[6], f[7]));
}

template <typename T, typename G>
__global__ void __launch_bounds__(256, 4) sparse_adam_kernel(const int32_t* rows, const G* dV,
                                                          const int32_t* Uptr, int32_t dv, T* V,
                                                          float* Vm, float* m, float* v,
                                                          int32_t* steps, mlAdamParams hp) {
  __shared__ float s_bc1, s_bc2;
  const int32_t U = *Uptr;
  for (int32_t i = blockIdx.x; i < U; i += gridDim.x) {
    const int64_t r = rows[i];
    if (threadIdx.x == 0) {
      const int c = ++steps[r];
      s_bc1 = 1.f - powf(hp.beta1, float(c));
      s_bc2 = 1.f - powf(hp.beta2, float(c));
    }
    __syncthreads();
    const float bc1 = s_bc1, bc2 = s_bc2;
    for (int c0 = threadIdx.x * 8; c0 < dv; c0 += blockDim.x * 8) {
      float gs[8], ms[8], vs[8], w8[8];
      load8<G>(dV + int64_t(i) * dv + c0, gs);
      load8<float>(m + r * dv + c0, ms);
      load8<float>(v + r * dv + c0, vs);
      if (Vm) load8<float>(Vm + r * dv + c0, w8);
      else load8<T>(V + r * dv + c0, w8);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        ms[e] = hp.beta1 * ms[e] + (1.f - hp.beta1) * gs[e];
        vs[e] = hp.beta2 * vs[e] + (1.f - hp.beta2) * gs[e] * gs[e];
        const float upd = (ms[e] / bc1) / (sqrtf(vs[e] / bc2) + hp.eps) + hp.weight_decay * w8[e];
        w8[e] = w8[e] - hp.lr * upd;
      }
      store8<float>(m + r * dv + c0, ms);
      store8<float>(v + r * dv + c0, vs);
      if (Vm) store8<float>(Vm + r * dv + c0, w8);
      store8<T>(V + r * dv + c0, w8);
    }
    __syncthreads();
  }
}

// rows whose width is not a multiple of 8 (fp32 tables): 4 elements per access
template <typename T, typename G>
__global__ void __launch_bounds__(256) sparse_adam4_kernel(const int32_t* rows, const G* dV,
                                                          const int32_t* Uptr, int32_t dv, T* V,
                                                          float* Vm, float* m, float* v,
                                                          int32_t* steps, mlAdamParams hp) {
  __shared__ float s_bc1, s_bc2;
  const int32_t U = *Uptr;
  for (int32_t i = blockIdx.x; i < U; i += gridDim.x) {
    const int64_t r = rows[i];
    if (threadIdx.x == 0) {
      const int c = ++steps[r];
      s_bc1 = 1.f - powf(hp.beta1, float(c));
      s_bc2 = 1.f - powf(hp.beta2, float(c));
    }
    __syncthreads();
    const float bc1 = s_bc1, bc2 = s_bc2;
    for (int c0 = threadIdx.x * 4; c0 < dv; c0 += blockDim.x * 4) {
      const float4 g = grad4(dV, int64_t(i) * dv + c0);
      float4* mp = reinterpret_cast<float4*>(m + r * dv + c0);
      float4* vp = reinterpret_cast<float4*>(v + r * dv + c0);
      float4 mm = *mp, vv = *vp;
      float w4[4];
      if (Vm) {
        const float4 t = *reinterpret_cast<const float4*>(Vm + r * dv + c0);
        w4[0] = t.x; w4[1] = t.y; w4[2] = t.z; w4[3] = t.w;
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) w4[e] = to_f(V[r * dv + c0 + e]);
      }
      const float gs[4] = {g.x, g.y, g.z, g.w};
      float ms[4] = {mm.x, mm.y, mm.z, mm.w}, vs[4] = {vv.x, vv.y, vv.z, vv.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        ms[e] = hp.beta1 * ms[e] + (1.f - hp.beta1) * gs[e];
        vs[e] = hp.beta2 * vs[e] + (1.f - hp.beta2) * gs[e] * gs[e];
        const float upd = (ms[e] / bc1) / (sqrtf(vs[e] / bc2) + hp.eps) + hp.weight_decay * w4[e];
        w4[e] = w4[e] - hp.lr * upd;
      }
      *mp = make_float4(ms[0], ms[1], ms[2], ms[3]);
      *vp = make_float4(vs[0], vs[1], vs[2], vs[3]);
      if (Vm) *reinterpret_cast<float4*>(Vm + r * dv + c0) = make_float4(w4[0], w4[1], w4[2], w4[3]);
      if constexpr (sizeof(T) == 4) {
        *reinterpret_cast<float4*>(reinterpret_cast<float*>(V) + r * dv + c0) =
            make_float4(w4[0], w4[1], w4[2], w4[3]);
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) V[r * dv + c0 + e] = __float2bfloat16_rn(w4[e]);
      }
    }
    __syncthreads();
  }
}

}  // namespace

mlStatus launch_sparse_adam(const int32_t* rows, const void* dV, mlDtype gdt, const int32_t* U,
                            int64_t cap, int32_t dv, void* V, mlDtype dt, float* Vm, float* m,
                            float* v, int32_t* steps, const mlAdamParams& hp, cudaStream_t s) {
  if (cap <= 0) return ML_OK;
  if (dv % 4) return fail(ML_ERR_CONFIG, "sparse_adam: dv must be a multiple of 4");
  const unsigned grid = unsigned(std::min<int64_t>(cap, int64_t(num_sms()) * 8));
  const float* g32 = static_cast<const float*>(dV);
  const __nv_bfloat16* g16 = static_cast<const __nv_bfloat16*>(dV);
  if (dt == ML_BF16) {
    __nv_bfloat16* Vb = static_cast<__nv_bfloat16*>(V);
    if (gdt == ML_BF16)
      sparse_adam_kernel<__nv_bfloat16, __nv_bfloat16><<<grid, 256, 0, s>>>(rows, g16, U, dv, Vb, Vm, m, v, steps, hp);
    else
      sparse_adam_kernel<__nv_bfloat16, float><<<grid, 256, 0, s>>>(rows, g32, U, dv, Vb, Vm, m, v, steps, hp);
  } else if (dv % 8) {    // bf16 rows are 16-byte multiples, so only fp32 tables get here
    sparse_adam4_kernel<float, float><<<grid, 256, 0, s>>>(rows, g32, U, dv, static_cast<float*>(V),
                                                           Vm, m, v, steps, hp);
  } else {
    sparse_adam_kernel<float, float><<<grid, 256, 0, s>>>(rows, g32, U, dv, static_cast<float*>(V),
                                                          Vm, m, v, steps, hp);
  }
  ML_LAUNCH_CHECK("sparse_adam");
  return ML_OK;
}

}  // namespace ml
