// The two other EmbeddingBag backward strategies benchmarked in PAPER.md
// §3.1.4, kept as controls for the sorted "reverse_indices" kernel:
//   "atomics": accumulation via atomic additions -- every (token, position)
//              adds w * dy[t] into dV[idx] with vector float atomics;
//   "lock":    "row-level atomic lock where we amortize the cost of memory
//              lock over the embedding dimension" -- a team acquires a spin
//              lock on the destination row once, then adds the whole row.
// Both write a dense fp32 dV [N, dv] (accumulate; the caller zeroes it) and
// are not bitwise deterministic (arrival order of the adds).
#include "internal.cuh"

namespace ml {
namespace {

struct CtrlParams {
  const int32_t* idx; const float* w; int32_t B; int32_t T; int64_t N;
  const char* dy; int64_t ldy_bytes;
  float* dV; int64_t ldv;      // dense fp32 [N, dv]
  int* locks;                  // [N] (lock strategy)
  int* flag;
};

// one team of NT threads per token, VEC columns per thread (like the forward)
template <typename T, int NT>
__global__ void __launch_bounds__(256) bag_bwd_atomic_kernel(CtrlParams p) {
  constexpr int VEC = Vec<T>::N;
  constexpr int TPC = 256 / NT;
  extern __shared__ int2 s_iw[];
  const int team = threadIdx.x / NT, tl = threadIdx.x % NT;
  const int64_t t0 = int64_t(blockIdx.x) * TPC;
  const int B = p.B;
  for (int e = threadIdx.x; e < TPC * B; e += 256) {
    const int64_t t = t0 + e / B;
    int ix = 0;
    float wv = 0.f;
    if (t < p.T) {
      ix = p.idx[t * B + e % B];
      wv = p.w[t * B + e % B];
      if (uint64_t(uint32_t(ix)) >= uint64_t(p.N)) { atomicExch(p.flag, 1); ix = 0; wv = 0.f; }
    }
    s_iw[e] = make_int2(ix, __float_as_int(wv));
  }
  __syncthreads();
  const int64_t t = t0 + team;
  if (t >= p.T) return;
  const int64_t col = int64_t(blockIdx.y) * NT * VEC + int64_t(tl) * VEC;
  float f[VEC];
  Vec<T>::load(ldg_nc_v4(p.dy + t * p.ldy_bytes + col * int64_t(sizeof(T))), f);
  const int2* my = s_iw + team * B;
  for (int j = 0; j < B; ++j) {
    const float wv = __int_as_float(my[j].y);
    float* dst = p.dV + int64_t(my[j].x) * p.ldv + col;
#pragma unroll
    for (int v = 0; v < VEC; v += 4)
      atomicAdd(reinterpret_cast<float4*>(dst + v),
                make_float4(wv * f[v], wv * f[v + 1], wv * f[v + 2], wv * f[v + 3]));
  }
}

// one CTA (blockDim = row vectors of one column slice, >= 32) per token
template <typename T>
__global__ void __launch_bounds__(256) bag_bwd_lock_kernel(CtrlParams p) {
  constexpr int VEC = Vec<T>::N;
  const int64_t t = blockIdx.x;
  const int64_t col = (int64_t(blockIdx.y) * blockDim.x + threadIdx.x) * VEC;
  const bool act = col < p.ldv;
  __shared__ int s_ix;
  __shared__ float s_w;
  float f[VEC];
  if (act) Vec<T>::load(ldg_nc_v4(p.dy + t * p.ldy_bytes + col * int64_t(sizeof(T))), f);
  for (int j = 0; j < p.B; ++j) {
    if (threadIdx.x == 0) {
      int ix = p.idx[t * p.B + j];
      float wv = p.w[t * p.B + j];
      if (uint64_t(uint32_t(ix)) >= uint64_t(p.N)) { atomicExch(p.flag, 1); ix = 0; wv = 0.f; }
      // row lock (one per destination row, per column slice) -- spin with backoff
      int* lk = p.locks + int64_t(blockIdx.y) * p.N + ix;
      unsigned ns = 32;
      while (atomicCAS(lk, 0, 1) != 0) {
        __nanosleep(ns);
        if (ns < 1024) ns <<= 1;
      }
      __threadfence();
      s_ix = ix;
      s_w = wv;
    }
    __syncthreads();
    if (act) {
      float* dst = p.dV + int64_t(s_ix) * p.ldv + col;
#pragma unroll
      for (int v = 0; v < VEC; v += 4) {
        float4 a = __ldcg(reinterpret_cast<const float4*>(dst + v));
        a.x += s_w * f[v]; a.y += s_w * f[v + 1]; a.z += s_w * f[v + 2]; a.w += s_w * f[v + 3];
        __stcg(reinterpret_cast<float4*>(dst + v), a);
      }
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) atomicExch(p.locks + int64_t(blockIdx.y) * p.N + s_ix, 0);
  }
}

template <typename T>
mlStatus dispatch_atomic(int nt, dim3 grid, size_t smem, const CtrlParams& p, cudaStream_t s) {
#define ML_ATOM_CASE(NTV)                                                     \
  case NTV:                                                                   \
    bag_bwd_atomic_kernel<T, NTV><<<grid, 256, smem, s>>>(p);                 \
    break;
  switch (nt) {
    ML_ATOM_CASE(1) ML_ATOM_CASE(2) ML_ATOM_CASE(4) ML_ATOM_CASE(8) ML_ATOM_CASE(16)
    ML_ATOM_CASE(32) ML_ATOM_CASE(64) ML_ATOM_CASE(128) ML_ATOM_CASE(256)
    default: return fail(ML_ERR_CONFIG, "atomics: unsupported team size");
  }
#undef ML_ATOM_CASE
  ML_LAUNCH_CHECK("embbag_bwd_atomics");
  return ML_OK;
}

}  // namespace

mlStatus launch_bag_bwd_ctrl(int strategy, const mlBagShape& sh, const int32_t* idx, const float* w,
                             const void* dy, float* dV, int* locks, cudaStream_t s) {
  if (sh.T == 0) return ML_OK;
  const int64_t es = int64_t(dtype_size(sh.dtype));
  const int64_t vu = int64_t(sh.dv) * es / 16;
  CtrlParams p;
  p.idx = idx; p.w = w; p.B = sh.B; p.T = sh.T; p.N = sh.N;
  p.dy = static_cast<const char*>(dy); p.ldy_bytes = int64_t(sh.dv) * es;
  p.dV = dV; p.ldv = sh.dv; p.locks = locks; p.flag = index_flag_ptr();
  if (strategy == 0) {  // atomics
    const int nt = int(vu < 256 ? vu : 256);
    const int tpc = 256 / nt;
    const size_t smem = size_t(tpc) * sh.B * sizeof(int2);
    if (smem > 48 * 1024) return fail(ML_ERR_UNSUPPORTED, "atomics: bag too large");
    dim3 grid{unsigned((sh.T + tpc - 1) / tpc), unsigned(vu / nt), 1u};
    if (sh.dtype == ML_BF16) return dispatch_atomic<__nv_bfloat16>(nt, grid, smem, p, s);
    return dispatch_atomic<float>(nt, grid, smem, p, s);
  }
  // lock
  const int threads = vu <= 32 ? 32 : (vu >= 256 ? 256 : int(vu));
  dim3 grid{unsigned(sh.T), unsigned(vu > 256 ? vu / 256 : 1), 1u};
  if (sh.dtype == ML_BF16) bag_bwd_lock_kernel<__nv_bfloat16><<<grid, threads, 0, s>>>(p);
  else bag_bwd_lock_kernel<float><<<grid, threads, 0, s>>>(p);
  ML_LAUNCH_CHECK("embbag_bwd_lock");
  return ML_OK;
}

}  // namespace ml
