// Layout kernels of the dim-sharded memory group (§3.1.2, P:167:
// "each worker gathers the partial embeddings corresponding to its own
// portion of the indices"): after the all-to-all a rank holds, for its T_loc
// tokens, G column slices [G][T_loc][dv/G]; unpack interleaves them into
// [T_loc][dv] rows and (optionally) applies the Memory+ gate
// z = y * silu(g) (Eq. 2) in the same pass.  pack is the reverse
// (the dy slices of the backward exchange).
#include "internal.cuh"

namespace ml {
namespace {

template <typename T, bool GATE>
__global__ void unpack_kernel(const char* recv, int G, int64_t T_loc, int64_t vs, const char* gate,
                              char* y, char* z) {
  // one thread per 16-byte vector of the [T_loc, dv] output; vs = vectors per slice
  const int64_t nvec = int64_t(G) * T_loc * vs;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nvec;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t t = i / (G * vs);
    const int64_t r = i - t * (G * vs);
    const int64_t g = r / vs, c = r - g * vs;
    const uint4 v = ldg_nc_v4(recv + ((g * T_loc + t) * vs + c) * 16);
    if (y) stg_v4(y + i * 16, v);
    if constexpr (GATE) {
      float f[Vec<T>::N], gg[Vec<T>::N];
      Vec<T>::load(v, f);
      Vec<T>::load(ldg_nc_v4(gate + i * 16), gg);
#pragma unroll
      for (int e = 0; e < Vec<T>::N; ++e) f[e] = f[e] * silu_f(gg[e]);
      stg_v4(z + i * 16, Vec<T>::pack(f));
    }
  }
}

__global__ void pack_kernel(const char* src, int G, int64_t T_loc, int64_t vs, char* dst) {
  const int64_t nvec = int64_t(G) * T_loc * vs;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nvec;
       i += int64_t(gridDim.x) * blockDim.x) {
    // i indexes dst [G][T_loc][vs]
    const int64_t g = i / (T_loc * vs);
    const int64_t r = i - g * (T_loc * vs);
    const int64_t t = r / vs, c = r - t * vs;
    stg_v4(dst + i * 16, ldg_nc_v4(src + ((t * G + g) * vs + c) * 16));
  }
}

// pack straight into G destination buffers (block g -> dst.p[g]): the dy
// slices of the backward stored into their owners' exchange regions
struct DstBlocks { char* p[kMaxOutBlocks]; };
__global__ void pack_peers_kernel(const char* src, int G, int64_t T_loc, int64_t vs,
                                  const __grid_constant__ DstBlocks dst) {
  const int64_t nvec = int64_t(G) * T_loc * vs;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nvec;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t g = i / (T_loc * vs);
    const int64_t r = i - g * (T_loc * vs);
    const int64_t t = r / vs, c = r - t * vs;
    stg_v4(dst.p[g] + r * 16, ldg_nc_v4(src + ((t * G + g) * vs + c) * 16));
  }
}

// out[i] = sum over g = 0..G-1 (in rank order: deterministic) of slots[g][i]
__global__ void sum_ranks_kernel(const float* slots, int G, int64_t n, float* out) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    float t = 0.f;
    for (int g = 0; g < G; ++g) t += slots[int64_t(g) * n + i];
    out[i] = t;
  }
}

unsigned grid_for(int64_t n) {
  const int64_t b = (n + 255) / 256;
  return unsigned(std::min<int64_t>(b, int64_t(num_sms()) * 16));
}

}  // namespace

mlStatus launch_group_pack_peers(const void* src, int G, int64_t T_loc, int32_t dv_slice,
                                 void* const* dst, mlDtype dt, cudaStream_t s) {
  const int64_t vs = int64_t(dv_slice) * int64_t(dtype_size(dt)) / 16;
  const int64_t n = int64_t(G) * T_loc * vs;
  if (n <= 0) return ML_OK;
  if (G > kMaxOutBlocks) return fail(ML_ERR_CONFIG, "group pack: G <= 64");
  DstBlocks d{};
  for (int g = 0; g < G; ++g) d.p[g] = static_cast<char*>(dst[g]);
  pack_peers_kernel<<<grid_for(n), 256, 0, s>>>(static_cast<const char*>(src), G, T_loc, vs, d);
  ML_LAUNCH_CHECK("group_pack");
  return ML_OK;
}

mlStatus launch_sum_ranks(const float* slots, int G, int64_t n, float* out, cudaStream_t s) {
  if (n <= 0) return ML_OK;
  sum_ranks_kernel<<<grid_for(n), 256, 0, s>>>(slots, G, n, out);
  ML_LAUNCH_CHECK("group_sum_ranks");
  return ML_OK;
}

mlStatus launch_group_unpack(const void* recv, int G, int64_t T_loc, int32_t dv_slice,
                             const void* gate, void* y, void* z, mlDtype dt, cudaStream_t s) {
  const int64_t vs = int64_t(dv_slice) * int64_t(dtype_size(dt)) / 16;
  const int64_t n = int64_t(G) * T_loc * vs;
  if (n <= 0) return ML_OK;
  auto c = [](const void* p) { return static_cast<const char*>(p); };
  auto m = [](void* p) { return static_cast<char*>(p); };
  if (gate) {
    if (dt == ML_BF16)
      unpack_kernel<__nv_bfloat16, true><<<grid_for(n), 256, 0, s>>>(c(recv), G, T_loc, vs, c(gate), m(y), m(z));
    else
      unpack_kernel<float, true><<<grid_for(n), 256, 0, s>>>(c(recv), G, T_loc, vs, c(gate), m(y), m(z));
  } else {
    unpack_kernel<float, false><<<grid_for(n), 256, 0, s>>>(c(recv), G, T_loc, vs, nullptr, m(y), nullptr);
  }
  ML_LAUNCH_CHECK("group_unpack");
  return ML_OK;
}

mlStatus launch_group_pack(const void* src, int G, int64_t T_loc, int32_t dv_slice, void* dst,
                           mlDtype dt, cudaStream_t s) {
  const int64_t vs = int64_t(dv_slice) * int64_t(dtype_size(dt)) / 16;
  const int64_t n = int64_t(G) * T_loc * vs;
  if (n <= 0) return ML_OK;
  pack_kernel<<<grid_for(n), 256, 0, s>>>(static_cast<const char*>(src), G, T_loc, vs,
                                          static_cast<char*>(dst));
  ML_LAUNCH_CHECK("group_pack");
  return ML_OK;
}

}  // namespace ml
