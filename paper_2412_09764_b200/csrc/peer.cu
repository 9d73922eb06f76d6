// PEER-style rank-1 experts over product keys (PAPER.md
// P:139; reading Q21 in DESIGN.md): key i owns (U[i], V[i]); for the
// selected keys of token t (idx, w from the product-key lookup)
//   h[t,j] = U[idx[t,j]] . x[t]          (peer_dot: a token-major gather-dot)
//   a[t,j] = w[t,j] * silu(h[t,j])       (peer_act)
//   y[t]   = sum_j a[t,j] V[idx[t,j]]    (the bag forward)
// and in the backward, from da[t,j] = <dy[t], V[idx[t,j]]> (the bag backward's
// score gradient):  dh = da * w * silu'(h),  dwr = da * silu(h)  (peer_dact).
#include "internal.cuh"

namespace ml {
namespace {

template <int N, int O>
struct WarpTR {   // butterfly transpose-reduce: lane l ends with the warp sum of value (l >> (5 - log2 N))
  __device__ __forceinline__ static void run(float* a, int lane) {
    const bool up = (lane & O) != 0;
#pragma unroll
    for (int i = 0; i < N / 2; ++i) {
      const float lo = a[i], hi = a[i + N / 2];
      a[i] = (up ? hi : lo) + __shfl_xor_sync(0xffffffffu, up ? lo : hi, O);
    }
    WarpTR<N / 2, O / 2>::run(a, lane);
  }
};
template <int O>
struct WarpTR<1, O> {
  __device__ __forceinline__ static void run(float* a, int) {
#pragma unroll
    for (int o = O; o > 0; o >>= 1) a[0] += __shfl_xor_sync(0xffffffffu, a[0], o);
  }
};

// One CTA per (token, column slice): the thread's 16 bytes of x[t] stay in
// registers, the selected table rows stream 16 at a time; the 16 partial dots
// of a batch are reduced by a warp butterfly and one shared exchange.
template <typename T>
__global__ void __launch_bounds__(256) peer_dot_kernel(const char* Ut, int64_t ld_bytes, int64_t N,
                                                       const int32_t* idx, int32_t B, const char* x,
                                                       int vec_units, float* h_part, int64_t P) {
  constexpr int VEC = Vec<T>::N;
  constexpr int R = 16;
  __shared__ int s_idx[1024];
  __shared__ float s_red[2][8][R];
  const int64_t t = blockIdx.x;
  const int slice = blockIdx.y;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  for (int j = tid; j < B; j += blockDim.x) {
    int ix = idx[t * B + j];
    if (uint64_t(uint32_t(ix)) >= uint64_t(N)) ix = 0;   // clamped (index flag set by the bag kernels)
    s_idx[j] = ix;
  }
  const int u = slice * blockDim.x + tid;
  const bool act = u < vec_units;
  const int64_t colb = int64_t(u) * 16;
  float2 f[VEC / 2];
  {
    uint4 d = make_uint4(0, 0, 0, 0);
    if (act) d = ldg_nc_v4(x + t * ld_bytes + colb);
    Vec<T>::load(d, reinterpret_cast<float*>(f));
  }
  __syncthreads();
  int buf = 0;
  for (int j0 = 0; j0 < B; j0 += R) {
    uint4 r[R];
#pragma unroll
    for (int q = 0; q < R; ++q) {
      r[q] = make_uint4(0, 0, 0, 0);
      if (act && j0 + q < B) r[q] = ldg_nc_v4(Ut + int64_t(s_idx[j0 + q]) * ld_bytes + colb);
    }
    float part[R];
#pragma unroll
    for (int q = 0; q < R; ++q) {
      float2 g[VEC / 2];
      Vec<T>::load(r[q], reinterpret_cast<float*>(g));
      float2 acc = make_float2(0.f, 0.f);
#pragma unroll
      for (int v = 0; v < VEC / 2; ++v) acc = ffma2(f[v], g[v], acc);
      part[q] = acc.x + acc.y;
    }
    WarpTR<R, 16>::run(part, lane);           // lane l: warp sum of slot (l >> 1) & 15
    if ((lane & 1) == 0) s_red[buf][warp][lane >> 1] = part[0];
    __syncthreads();
    if (tid < R && j0 + tid < B) {
      float tot = 0.f;
      for (int w2 = 0; w2 < nw; ++w2) tot += s_red[buf][w2][tid];
      h_part[int64_t(slice) * P + t * B + j0 + tid] = tot;
    }
    buf ^= 1;
  }
}

__global__ void peer_act_kernel(const float* h_part, int ns, int64_t P, const float* w, float* h,
                                float* a) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= P) return;
  float s = 0.f;
  for (int k = 0; k < ns; ++k) s += h_part[int64_t(k) * P + i];
  h[i] = s;
  a[i] = w[i] * silu_f(s);
}

__global__ void peer_dact_kernel(const float* da_part, int ns, int64_t P, const float* w,
                                 const float* h, float* dh, float* dwr) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= P) return;
  float da = 0.f;
  for (int k = 0; k < ns; ++k) da += da_part[int64_t(k) * P + i];
  const float x = h[i];
  const float sg = sigmoid_f(x);
  dh[i] = da * w[i] * (sg * (1.f + x * (1.f - sg)));
  dwr[i] = da * (x * sg);
}

}  // namespace

int peer_dot_slices(int32_t D, mlDtype dt) {
  const int64_t vu = int64_t(D) * int64_t(dtype_size(dt)) / 16;
  return int(vu <= 256 ? 1 : (vu + 255) / 256);
}

mlStatus launch_peer_dot(const void* Ut, int64_t N, int32_t D, const int32_t* idx, int32_t T,
                         int32_t B, const void* x, mlDtype dt, float* h_part, cudaStream_t s) {
  if (T <= 0) return ML_OK;
  if (B > 1024) return fail(ML_ERR_UNSUPPORTED, "peer: H*k > 1024");
  const int64_t es = int64_t(dtype_size(dt));
  const int64_t vu = int64_t(D) * es / 16;
  const int threads = vu <= 32 ? 32 : (vu >= 256 ? 256 : int(vu));
  const int ns = int((vu + threads - 1) / threads);
  dim3 grid{unsigned(T), unsigned(ns), 1u};
  const int64_t P = int64_t(T) * B;
  auto c = [](const void* p) { return static_cast<const char*>(p); };
  if (dt == ML_BF16)
    peer_dot_kernel<__nv_bfloat16><<<grid, threads, 0, s>>>(c(Ut), D * es, N, idx, B, c(x), int(vu),
                                                            h_part, P);
  else
    peer_dot_kernel<float><<<grid, threads, 0, s>>>(c(Ut), D * es, N, idx, B, c(x), int(vu), h_part,
                                                    P);
  ML_LAUNCH_CHECK("peer_dot");
  return ML_OK;
}

mlStatus launch_peer_act(const float* h_part, int ns, int64_t P, const float* w, float* h, float* a,
                         cudaStream_t s) {
  if (P <= 0) return ML_OK;
  peer_act_kernel<<<unsigned((P + 255) / 256), 256, 0, s>>>(h_part, ns, P, w, h, a);
  ML_LAUNCH_CHECK("peer_act");
  return ML_OK;
}

mlStatus launch_peer_dact(const float* da_part, int ns, int64_t P, const float* w, const float* h,
                          float* dh, float* dwr, cudaStream_t s) {
  if (P <= 0) return ML_OK;
  peer_dact_kernel<<<unsigned((P + 255) / 256), 256, 0, s>>>(da_part, ns, P, w, h, dh, dwr);
  ML_LAUNCH_CHECK("peer_dact");
  return ML_OK;
}

}  // namespace ml
