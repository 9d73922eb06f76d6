// EmbeddingBag forward (Eq. 1 "y = s V_I"; §3.1.4 P:176:
// "we expect this operation to be solely limited by the GPU memory
// bandwidth").  Also used, with fp32 output, for the query gradient of the
// product-key lookup (dq = sum_j ds_j K[a_j], a bag over the half-key table).
//
// Design (sm_100a, HBM-bound): a "team" of NT threads owns one bag (token)
// and a slice of NT*16 bytes of the value row; each thread streams 16-byte
// vectors of UNROLL rows at once (ld.global.nc.L1::no_allocate.v4) into fp32
// accumulators, so a CTA keeps 256 * UNROLL * 16 B of loads in flight.  The
// bag's (idx, w) pairs are staged once in shared memory.  The Memory+ gate
// (Eq. 2) is applied in the epilogue: out = y * silu(g).
#include "internal.cuh"

#include <cstdlib>

namespace ml {

__device__ int g_index_error;

int* index_flag_ptr() {
  static int* p = nullptr;
  if (!p) cudaGetSymbolAddress(reinterpret_cast<void**>(&p), g_index_error);
  return p;
}

bool check_indices_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("ML_CHECK_INDICES");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

mlStatus check_index_flag(cudaStream_t s) {
  if (!check_indices_enabled()) return ML_OK;
  int h = 0;
  ML_CUDA_TRY(cudaMemcpyAsync(&h, index_flag_ptr(), sizeof(int), cudaMemcpyDeviceToHost, s));
  ML_CUDA_TRY(cudaStreamSynchronize(s));
  if (h) {
    int z = 0;
    ML_CUDA_TRY(cudaMemcpyAsync(index_flag_ptr(), &z, sizeof(int), cudaMemcpyHostToDevice, s));
    ML_CUDA_TRY(cudaStreamSynchronize(s));
    return fail(ML_ERR_INDEX, "index outside [0, N) in a bag (clamped to row 0, weight 0)");
  }
  return ML_OK;
}

namespace {

struct BagParams {
  const char* V; int64_t ldv_bytes; int64_t N;
  const int32_t* idx; const float* w; int32_t B; int32_t nbags;
  char* out; int64_t ldo; int32_t out_col0;
  const char* gate; char* y_ungated;
  int* flag;
  // blocked output (BLK): bag b's row goes to block b / block_rows, row
  // b % block_rows -- e.g. each token block straight into its owner rank's
  // exchange region over peer memory (memory group, fused exchange)
  char* blocks[kMaxOutBlocks]; int32_t block_rows;
};

// UNROLL = 8 rows per thread in flight at 4 CTAs/SM (<= 64 registers): 32
// resident warps per SM keep 128 KiB of row loads outstanding (measured
// 1.28 ms at C2 vs 1.33-1.34 for 16 rows at 1-2 CTAs/SM)
template <typename Tin, bool OUT_F32, int NT, int UNROLL, bool GATE, int MINB, bool BLK = false>
__global__ void __launch_bounds__(256, MINB) bag_fwd_kernel(const __grid_constant__ BagParams p) {
  constexpr int VEC = Vec<Tin>::N;
  constexpr int TPC = 256 / NT;
  extern __shared__ int2 s_iw[];  // [TPC][B] (row, weight bits)
  const int team = threadIdx.x / NT;
  const int tl = threadIdx.x % NT;
  const int64_t bag0 = int64_t(blockIdx.x) * TPC;
  const int B = p.B;

  for (int e = threadIdx.x; e < TPC * B; e += 256) {
    const int64_t b = bag0 + e / B;
    int ix = 0;
    float wv = 0.f;
    if (b < p.nbags) {
      const int64_t o = b * B + (e % B);
      ix = __ldg(p.idx + o);
      wv = __ldg(p.w + o);
      if (static_cast<uint64_t>(static_cast<int64_t>(ix)) >= static_cast<uint64_t>(p.N)) {
        atomicExch(p.flag, 1);
        ix = 0;
        wv = 0.f;
      }
    }
    s_iw[e] = make_int2(ix, __float_as_int(wv));
  }
  __syncthreads();

  const int64_t bag = bag0 + team;
  if (bag >= p.nbags) return;
  const int64_t col = int64_t(blockIdx.y) * NT * VEC + int64_t(tl) * VEC;
  const char* vbase = p.V + col * int64_t(sizeof(Tin));
  const int2* my = s_iw + team * B;

  float acc[VEC];
#pragma unroll
  for (int v = 0; v < VEC; ++v) acc[v] = 0.f;

  for (int j0 = 0; j0 < B; j0 += UNROLL) {
    uint4 r[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const int j = j0 + u;
      if (j < B) r[u] = ldg_nc_v4(vbase + int64_t(my[j].x) * p.ldv_bytes);
    }
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const int j = j0 + u;
      if (j < B) {
        float f[VEC];
        Vec<Tin>::load(r[u], f);
        const float wv = __int_as_float(my[j].y);
#pragma unroll
        for (int v = 0; v < VEC; ++v) acc[v] = fmaf(wv, f[v], acc[v]);
      }
    }
  }

  const int64_t oelem = bag * p.ldo + p.out_col0 + col;
  if constexpr (GATE) {
    const int64_t off = oelem * int64_t(sizeof(Tin));
    float g[VEC];
    Vec<Tin>::load(ldg_v4(p.gate + off), g);
    if (p.y_ungated) stg_v4(p.y_ungated + off, Vec<Tin>::pack(acc));
#pragma unroll
    for (int v = 0; v < VEC; ++v) acc[v] = acc[v] * silu_f(g[v]);
  }
  if constexpr (OUT_F32) {
    float* o = reinterpret_cast<float*>(p.out) + oelem;
#pragma unroll
    for (int v = 0; v < VEC; v += 4)
      stg_v4(o + v, make_uint4(__float_as_uint(acc[v]), __float_as_uint(acc[v + 1]),
                               __float_as_uint(acc[v + 2]), __float_as_uint(acc[v + 3])));
  } else if constexpr (BLK) {
    const int32_t blk = int32_t(bag / p.block_rows);
    const int64_t o = (bag - int64_t(blk) * p.block_rows) * p.ldo + p.out_col0 + col;
    stg_v4(p.blocks[blk] + o * int64_t(sizeof(Tin)), Vec<Tin>::pack(acc));
  } else {
    stg_v4(p.out + oelem * int64_t(sizeof(Tin)), Vec<Tin>::pack(acc));
  }
}

template <typename Tin, bool OUT_F32, bool GATE, bool BLK = false>
mlStatus dispatch_nt(int nt, dim3 grid, size_t smem, const BagParams& p, cudaStream_t s,
                     const char* name) {
#define ML_BAG_CASE(NTV)                                                              \
  case NTV: {                                                                         \
    auto k = bag_fwd_kernel<Tin, OUT_F32, NTV, 8, GATE, 4, BLK>;                      \
    if (smem > 48 * 1024)                                                             \
      ML_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                       int(smem)));                                   \
    k<<<grid, 256, smem, s>>>(p);                                                     \
    break;                                                                            \
  }
  switch (nt) {
    ML_BAG_CASE(1) ML_BAG_CASE(2) ML_BAG_CASE(4) ML_BAG_CASE(8) ML_BAG_CASE(16)
    ML_BAG_CASE(32) ML_BAG_CASE(64) ML_BAG_CASE(128) ML_BAG_CASE(256)
    default: return fail(ML_ERR_CONFIG, "bag: unsupported team size");
  }
#undef ML_BAG_CASE
  ML_LAUNCH_CHECK(name);
  return ML_OK;
}

}  // namespace

mlStatus check_cols(int32_t dv, mlDtype dt, const char* what) {
  const int64_t bytes = int64_t(dv) * int64_t(dtype_size(dt));
  if (dv <= 0 || bytes % 16)
    return fail(ML_ERR_CONFIG, std::string(what) + ": row bytes must be a positive multiple of 16");
  const int64_t vu = bytes / 16;
  if ((vu & (vu - 1)) != 0 && vu % 256 != 0)
    return fail(ML_ERR_CONFIG, std::string(what) +
                                   ": (row bytes / 16) must be a power of two or a multiple of 256");
  return ML_OK;
}

mlStatus launch_bag_fwd(const BagFwdArgs& a, cudaStream_t s) {
  ML_TRY(check_cols(a.dv, a.dtype, "bag"));
  if (a.B < 1 || a.B > 1024) return fail(ML_ERR_CONFIG, "bag size B must be in [1, 1024]");
  if (a.nbags <= 0) return ML_OK;
  const int64_t vu = int64_t(a.dv) * int64_t(dtype_size(a.dtype)) / 16;
  const int nt = int(vu < 256 ? vu : 256);
  const int slices = int(vu / nt);
  const int tpc = 256 / nt;
  const size_t smem = size_t(tpc) * size_t(a.B) * sizeof(int2);
  if (smem > 200 * 1024) return fail(ML_ERR_UNSUPPORTED, "bag: bag too large for the team layout");
  const int64_t nblk = (int64_t(a.nbags) + tpc - 1) / tpc;
  if (nblk > 0x7FFFFFFF || slices > 65535) return fail(ML_ERR_UNSUPPORTED, "bag: grid too large");
  BagParams p;
  const size_t es = dtype_size(a.dtype);
  p.V = static_cast<const char*>(a.V);
  p.ldv_bytes = a.ldv * int64_t(es);
  p.N = a.N;
  p.idx = a.idx;
  p.w = a.w;
  p.B = a.B;
  p.nbags = a.nbags;
  p.out = static_cast<char*>(a.out);
  p.ldo = a.ldo;
  p.out_col0 = a.out_col0;
  p.gate = static_cast<const char*>(a.gate);
  p.y_ungated = static_cast<char*>(a.y_ungated);
  p.flag = index_flag_ptr();
  p.block_rows = 0;
  dim3 grid{unsigned(nblk), unsigned(slices), 1u};
  const bool gate = a.gate != nullptr;
  if (gate && a.out_f32) return fail(ML_ERR_UNSUPPORTED, "bag: gated output must be of the value dtype");
  if (a.out_blocks) {
    if (gate || a.out_f32 || a.y_ungated || a.block_rows <= 0 ||
        (int64_t(a.nbags) + a.block_rows - 1) / a.block_rows > kMaxOutBlocks)
      return fail(ML_ERR_UNSUPPORTED, "bag: blocked output is ungated, of the value dtype, <= 64 blocks");
    const int nblocks = int((int64_t(a.nbags) + a.block_rows - 1) / a.block_rows);
    for (int b = 0; b < nblocks; ++b) p.blocks[b] = static_cast<char*>(a.out_blocks[b]);
    p.block_rows = a.block_rows;
    return a.dtype == ML_BF16 ? dispatch_nt<__nv_bfloat16, false, false, true>(nt, grid, smem, p, s, a.name)
                              : dispatch_nt<float, false, false, true>(nt, grid, smem, p, s, a.name);
  }
  if (a.dtype == ML_BF16) {
    if (a.out_f32) return dispatch_nt<__nv_bfloat16, true, false>(nt, grid, smem, p, s, a.name);
    return gate ? dispatch_nt<__nv_bfloat16, false, true>(nt, grid, smem, p, s, a.name)
                : dispatch_nt<__nv_bfloat16, false, false>(nt, grid, smem, p, s, a.name);
  }
  if (a.out_f32) return dispatch_nt<float, true, false>(nt, grid, smem, p, s, a.name);
  return gate ? dispatch_nt<float, false, true>(nt, grid, smem, p, s, a.name)
              : dispatch_nt<float, false, false>(nt, grid, smem, p, s, a.name);
}

}  // namespace ml
