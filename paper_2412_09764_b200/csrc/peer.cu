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

// Warp-per-row variant for rows of 512-byte multiples: one CTA (8 warps) per
// (token, <= 4 KiB column slice); each warp keeps its lanes' 16-byte pieces of
// x[t] in registers and owns rows j = warp, warp + 8, ...; two rows per step
// (2 x NCH 16-byte loads per lane in flight), warp-shuffle reductions only.
template <typename T, int NCH>
__global__ void __launch_bounds__(256, 3) peer_dot_warp_kernel(const char* Ut, int64_t ld_bytes,
                                                            int64_t N, const int32_t* idx, int32_t B,
                                                            const char* x, float* h_part, int64_t P) {
  constexpr int VEC = Vec<T>::N;
  __shared__ int s_idx[1024];
  const int64_t t = blockIdx.x;
  const int slice = blockIdx.y;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t col0 = int64_t(slice) * 4096 + lane * 16;
  // the bag's indices are staged once (clamped): the row loads of every step
  // then depend on a shared-memory read, not a global one
  for (int j = threadIdx.x; j < B; j += blockDim.x) {
    int ix = idx[t * B + j];
    if (uint64_t(uint32_t(ix)) >= uint64_t(N)) ix = 0;
    s_idx[j] = ix;
  }
  // x[t]'s slice in shared memory (read at use): the registers go to the row
  // loads in flight, 3 CTAs/SM
  __shared__ uint4 s_x[NCH * 32];
  for (int e = threadIdx.x; e < NCH * 32; e += blockDim.x)
    s_x[e] = ldg_nc_v4(x + t * ld_bytes + int64_t(slice) * 4096 + int64_t(e) * 16);
  __syncthreads();
  for (int j0 = warp; j0 < B; j0 += 16) {
    const int j1 = j0 + 8;
    const int r0 = s_idx[j0];
    const int r1 = j1 < B ? s_idx[j1] : r0;
    uint4 a[NCH], b[NCH];
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      a[c] = ldg_nc_v4(Ut + int64_t(r0) * ld_bytes + col0 + c * 512);
      b[c] = ldg_nc_v4(Ut + int64_t(r1) * ld_bytes + col0 + c * 512);
    }
    float2 pa = make_float2(0.f, 0.f), pb = make_float2(0.f, 0.f);
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      float2 xf[VEC / 2], fa[VEC / 2], fb[VEC / 2];
      Vec<T>::load(s_x[c * 32 + lane], reinterpret_cast<float*>(xf));
      Vec<T>::load(a[c], reinterpret_cast<float*>(fa));
      Vec<T>::load(b[c], reinterpret_cast<float*>(fb));
#pragma unroll
      for (int v = 0; v < VEC / 2; ++v) {
        pa = ffma2(xf[v], fa[v], pa);
        pb = ffma2(xf[v], fb[v], pb);
      }
    }
    float sv[2] = {pa.x + pa.y, pb.x + pb.y};
    WarpTR<2, 16>::run(sv, lane);              // lane l: warp sum of row (l >> 4)
    if (lane == 0) h_part[int64_t(slice) * P + t * B + j0] = sv[0];
    if (lane == 16 && j1 < B) h_part[int64_t(slice) * P + t * B + j1] = sv[0];
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

// rows of 512, 1024, 2048 or k*4096 bytes take the warp-per-row kernel
static bool peer_warp_path(int64_t rowb) {
  return rowb == 512 || rowb == 1024 || rowb == 2048 || (rowb >= 4096 && rowb % 4096 == 0);
}

int peer_dot_slices(int32_t D, mlDtype dt) {
  const int64_t rowb = int64_t(D) * int64_t(dtype_size(dt));
  if (peer_warp_path(rowb)) return int(rowb >= 4096 ? rowb / 4096 : 1);
  const int64_t vu = rowb / 16;
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
  const int64_t P = int64_t(T) * B;
  auto c = [](const void* p) { return static_cast<const char*>(p); };
  const int64_t rowb = int64_t(D) * es;
  if (peer_warp_path(rowb)) {
    // warp-per-row path: slices of <= 4 KiB, NCH 512-byte chunks each
    const int nch = int(rowb >= 4096 ? 8 : rowb / 512);
    dim3 g2{unsigned(T), unsigned(rowb >= 4096 ? rowb / 4096 : 1), 1u};
#define ML_PEER_DOT(TT, NC)                                                                      \
  peer_dot_warp_kernel<TT, NC><<<g2, 256, 0, s>>>(c(Ut), rowb, N, idx, B, c(x), h_part, P)
#define ML_PEER_DOT_T(TT)                                                                        \
  switch (nch) {                                                                                 \
    case 1: ML_PEER_DOT(TT, 1); break;                                                           \
    case 2: ML_PEER_DOT(TT, 2); break;                                                           \
    case 4: ML_PEER_DOT(TT, 4); break;                                                           \
    case 8: ML_PEER_DOT(TT, 8); break;                                                           \
    default: return fail(ML_ERR_UNSUPPORTED, "peer: row width");                                 \
  }
    if (dt == ML_BF16) { ML_PEER_DOT_T(__nv_bfloat16) } else { ML_PEER_DOT_T(float) }
#undef ML_PEER_DOT_T
#undef ML_PEER_DOT
    ML_LAUNCH_CHECK("peer_dot");
    return ML_OK;
  }
  dim3 grid{unsigned(T), unsigned(ns), 1u};
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
