// Memory+ gate pieces (Eq. 2; silu(x) = x sigmoid(x)):
// the elementwise backward and the dense W1/W2 products (library GEMMs on
// cuBLASLt with fp32 accumulation), plus the compact->dense dV scatter.
#include "internal.cuh"

#include <cstdio>

#include <algorithm>
#include <cstdlib>

#include <cublasLt.h>

#include <map>
#include <mutex>
#include <tuple>

namespace ml {
namespace {

// z = y*silu(g); dy = dz*silu(g); dg = dz*y*sigmoid(g)*(1 + g*(1 - sigmoid(g)))
template <typename T>
__global__ void gate_bwd_kernel(const char* dz, const char* g, const char* y, char* z, char* dy,
                                char* dg, int64_t nvec) {
  constexpr int VEC = Vec<T>::N;
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= nvec) return;
  const int64_t off = i * 16;
  float fdz[VEC], fg[VEC], fy[VEC], oz[VEC], ody[VEC], odg[VEC];
  Vec<T>::load(ldg_nc_v4(dz + off), fdz);
  Vec<T>::load(ldg_nc_v4(g + off), fg);
  Vec<T>::load(ldg_nc_v4(y + off), fy);
#pragma unroll
  for (int v = 0; v < VEC; ++v) {
    const float sg = sigmoid_f(fg[v]);
    const float si = fg[v] * sg;
    oz[v] = fy[v] * si;
    ody[v] = fdz[v] * si;
    odg[v] = fdz[v] * fy[v] * (sg * (1.0f + fg[v] * (1.0f - sg)));
  }
  stg_v4(z + off, Vec<T>::pack(oz));
  stg_v4(dy + off, Vec<T>::pack(ody));
  stg_v4(dg + off, Vec<T>::pack(odg));
}

__device__ __forceinline__ float4 load4(const float* p, int64_t i) {
  return reinterpret_cast<const float4*>(p)[i];
}
__device__ __forceinline__ float4 load4(const __nv_bfloat16* p, int64_t i) {
  const uint2 u = reinterpret_cast<const uint2*>(p)[i];
  const float2 a = bf2_to_f2(u.x), b = bf2_to_f2(u.y);
  return make_float4(a.x, a.y, b.x, b.y);
}

template <typename G>
__global__ void scatter_rows_kernel(const int32_t* rows, const G* dV, const int32_t* U,
                                    int32_t dv4, float* dense) {
  const int64_t r = blockIdx.x;
  if (r >= *U) return;
  const int64_t dst = rows[r];
  float4* d = reinterpret_cast<float4*>(dense + dst * int64_t(dv4) * 4);
  for (int c = threadIdx.x; c < dv4; c += blockDim.x) {
    float4 a = load4(dV, r * int64_t(dv4) + c), b = d[c];
    b.x += a.x; b.y += a.y; b.z += a.z; b.w += a.w;
    d[c] = b;
  }
}

// ------------------------------------------------------------ cuBLASLt
cublasLtHandle_t lt_handle() {
  static cublasLtHandle_t h = nullptr;
  static std::once_flag once;
  std::call_once(once, [] { cublasLtCreate(&h); });
  return h;
}

}  // namespace

mlStatus launch_gate_bwd(const void* dz, const void* g, const void* y, void* z, void* dy, void* dg,
                         int64_t n, mlDtype dt, cudaStream_t s) {
  if (n <= 0) return ML_OK;
  const int64_t nvec = n * int64_t(dtype_size(dt)) / 16;
  const unsigned grid = unsigned((nvec + 255) / 256);
  auto c = [](const void* p) { return static_cast<const char*>(p); };
  auto m = [](void* p) { return static_cast<char*>(p); };
  if (dt == ML_BF16)
    gate_bwd_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>(c(dz), c(g), c(y), m(z), m(dy), m(dg), nvec);
  else
    gate_bwd_kernel<float><<<grid, 256, 0, s>>>(c(dz), c(g), c(y), m(z), m(dy), m(dg), nvec);
  ML_LAUNCH_CHECK("gate_bwd");
  return ML_OK;
}

mlStatus launch_scatter_rows(const int32_t* rows, const void* dV, mlDtype gdt, const int32_t* U,
                             int64_t cap, int32_t dv, float* dense, cudaStream_t s) {
  if (cap <= 0) return ML_OK;
  if (dv % 4) return fail(ML_ERR_CONFIG, "grad_apply: dv must be a multiple of 4");
  if (gdt == ML_BF16)
    scatter_rows_kernel<__nv_bfloat16><<<unsigned(cap), 128, 0, s>>>(
        rows, static_cast<const __nv_bfloat16*>(dV), U, dv / 4, dense);
  else
    scatter_rows_kernel<float><<<unsigned(cap), 128, 0, s>>>(rows, static_cast<const float*>(dV),
                                                             U, dv / 4, dense);
  ML_LAUNCH_CHECK("scatter_rows");
  return ML_OK;
}

static bool tune_log() {
  static const bool v = [] { const char* e = std::getenv("ML_GEMM_TUNE_LOG"); return e && e[0] == '1'; }();
  return v;
}

mlStatus gemm_rm(bool transA, bool transB, int64_t M, int64_t N, int64_t K, const void* A,
                 int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc, mlDtype ab,
                 bool c_f32, void* ws, size_t ws_bytes, cudaStream_t s, float beta) {
  return gemm_rm_batched(transA, transB, M, N, K, A, lda, 0, B, ldb, 0, C, ldc, 0, 1, ab, c_f32, ws,
                         ws_bytes, s, beta);
}

mlStatus gemm_rm_batched(bool transA, bool transB, int64_t M, int64_t N, int64_t K, const void* A,
                         int64_t lda, int64_t strideA, const void* B, int64_t ldb, int64_t strideB,
                         void* C, int64_t ldc, int64_t strideC, int batch, mlDtype ab, bool c_f32,
                         void* ws, size_t ws_bytes, cudaStream_t s, float beta) {
  if (M <= 0 || N <= 0) return ML_OK;
  cublasLtHandle_t h = lt_handle();
  if (!h) return fail(ML_ERR_CUDA, "cublasLtCreate failed");
  // Row-major C[M,N] = op(A) op(B)  <=>  column-major C^T[N,M] = op(B)^T op(A)^T:
  // first operand = B buffer, second = A buffer.
  const cudaDataType_t tab = ab == ML_BF16 ? CUDA_R_16BF : CUDA_R_32F;
  const cudaDataType_t tc = c_f32 ? CUDA_R_32F : tab;
  cublasOperation_t op1 = transB ? CUBLAS_OP_T : CUBLAS_OP_N;
  cublasOperation_t op2 = transA ? CUBLAS_OP_T : CUBLAS_OP_N;
  cublasLtMatmulDesc_t desc = nullptr;
  cublasLtMatrixLayout_t l1 = nullptr, l2 = nullptr, lc = nullptr;
  mlStatus st = ML_OK;
  auto ck = [&](cublasStatus_t r, const char* what) {
    if (r != CUBLAS_STATUS_SUCCESS && st == ML_OK)
      st = fail(ML_ERR_CUDA, std::string("cublasLt ") + what + " status " + std::to_string(int(r)));
  };
  ck(cublasLtMatmulDescCreate(&desc, CUBLAS_COMPUTE_32F, CUDA_R_32F), "desc");
  if (st == ML_OK) {
    ck(cublasLtMatmulDescSetAttribute(desc, CUBLASLT_MATMUL_DESC_TRANSA, &op1, sizeof(op1)), "ta");
    ck(cublasLtMatmulDescSetAttribute(desc, CUBLASLT_MATMUL_DESC_TRANSB, &op2, sizeof(op2)), "tb");
    // stored (column-major) shapes of the two operands
    ck(cublasLtMatrixLayoutCreate(&l1, tab, transB ? K : N, transB ? N : K, ldb), "l1");
    ck(cublasLtMatrixLayoutCreate(&l2, tab, transA ? M : K, transA ? K : M, lda), "l2");
    ck(cublasLtMatrixLayoutCreate(&lc, tc, N, M, ldc), "lc");
    if (batch > 1 && st == ML_OK) {
      const int32_t bc = batch;
      ck(cublasLtMatrixLayoutSetAttribute(l1, CUBLASLT_MATRIX_LAYOUT_BATCH_COUNT, &bc, sizeof(bc)), "b1");
      ck(cublasLtMatrixLayoutSetAttribute(l2, CUBLASLT_MATRIX_LAYOUT_BATCH_COUNT, &bc, sizeof(bc)), "b2");
      ck(cublasLtMatrixLayoutSetAttribute(lc, CUBLASLT_MATRIX_LAYOUT_BATCH_COUNT, &bc, sizeof(bc)), "bc");
      ck(cublasLtMatrixLayoutSetAttribute(l1, CUBLASLT_MATRIX_LAYOUT_STRIDED_BATCH_OFFSET, &strideB,
                                          sizeof(strideB)), "s1");
      ck(cublasLtMatrixLayoutSetAttribute(l2, CUBLASLT_MATRIX_LAYOUT_STRIDED_BATCH_OFFSET, &strideA,
                                          sizeof(strideA)), "s2");
      ck(cublasLtMatrixLayoutSetAttribute(lc, CUBLASLT_MATRIX_LAYOUT_STRIDED_BATCH_OFFSET, &strideC,
                                          sizeof(strideC)), "sc");
    }
  }
  cublasLtMatmulPreference_t pref = nullptr;
  cublasLtMatmulHeuristicResult_t heur = {};
  int nres = 0;
  if (st == ML_OK) {
    ck(cublasLtMatmulPreferenceCreate(&pref), "pref");
    uint64_t wsb = ws_bytes;
    ck(cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &wsb,
                                            sizeof(wsb)), "pref ws");
    // heuristic results cached per problem signature (the query costs tens of us)
    static std::mutex mu;
    static std::map<std::tuple<int, int, int64_t, int64_t, int64_t, int64_t, int64_t, int64_t, int, int, size_t, int, int>,
                    cublasLtMatmulHeuristicResult_t> cache;
    const auto key = std::make_tuple(int(transA), int(transB), M, N, K, lda, ldb, ldc, int(ab),
                                     int(c_f32), ws_bytes, int(beta != 0.f), batch);
    {
      std::lock_guard<std::mutex> lk(mu);
      auto it = cache.find(key);
      if (it != cache.end()) {
        heur = it->second;
        nres = 1;
      }
    }
    if (!nres) {
      // the heuristic's first choice is not always the fastest on this part
      // (measured: the [T, S] x [S, Dh] query-gradient GEMM 68 vs 54 us): for
      // overwriting GEMMs (beta = 0) the top candidates are timed once, on the
      // first call of each problem signature, and the fastest is cached
      static const bool tune = [] { const char* e = std::getenv("ML_GEMM_TUNE"); return !(e && e[0] == '0'); }();
      constexpr int kCand = 8;
      cublasLtMatmulHeuristicResult_t all[kCand] = {};
      ck(cublasLtMatmulAlgoGetHeuristic(h, desc, l1, l2, lc, lc, pref, kCand, all, &nres), "heuristic");
      if (nres > 0) heur = all[0];
      cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
      ML_CUDA_TRY(cudaStreamIsCapturing(s, &cap));
      if (st == ML_OK && tune && nres > 1 && beta == 0.f && cap == cudaStreamCaptureStatusNone) {
        // per host thread: concurrent callers (one thread per rank of a hub
        // group) must not record into each other's timing events
        thread_local cudaEvent_t e0 = nullptr, e1 = nullptr;
        if (!e0) {
          ML_CUDA_TRY(cudaEventCreate(&e0));
          ML_CUDA_TRY(cudaEventCreate(&e1));
        }
        // 8 candidates, best of 5 runs each (with 4, C2's fastest kernel for
        // the 16384 x 2048 x 2048 GEMMs, the 6th candidate, was never timed).
        // No device-wide sync: a rank thread of a hub group would wait on
        // streams that wait on the other ranks' host threads
        const float alpha = 1.f;
        float best = 1e30f;
        for (int c = 0; c < nres && st == ML_OK; ++c) {
          float t = 1e30f;
          for (int rep = 0; rep < 5 && st == ML_OK; ++rep) {
            ML_CUDA_TRY(cudaEventRecord(e0, s));
            ck(cublasLtMatmul(h, desc, &alpha, B, l1, A, l2, &beta, C, lc, C, lc, &all[c].algo, ws,
                              ws_bytes, s), "matmul (tuning)");
            ML_CUDA_TRY(cudaEventRecord(e1, s));
            ML_CUDA_TRY(cudaEventSynchronize(e1));
            float ms = 0.f;
            ML_CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
            t = std::min(t, ms);
          }
          if (t < best) {
            best = t;
            heur = all[c];
          }
          if (tune_log())
            std::fprintf(stderr, "gemm tune M=%lld N=%lld K=%lld tA=%d tB=%d cand %d: %.1f us\n",
                         (long long)M, (long long)N, (long long)K, int(transA), int(transB), c, t * 1e3f);
        }
      }
      if (st == ML_OK && nres == 0) st = fail(ML_ERR_CUDA, "cublasLt: no algorithm");
      if (st == ML_OK) {
        std::lock_guard<std::mutex> lk(mu);
        cache[key] = heur;
      }
    }
  }
  if (st == ML_OK) {
    const float alpha = 1.f;
    timing_mark(nullptr, s);
    ck(cublasLtMatmul(h, desc, &alpha, B, l1, A, l2, &beta, C, lc, C, lc, &heur.algo, ws, ws_bytes,
                      s), "matmul");
    timing_mark("cublasLt_gemm", s);
  }
  if (pref) cublasLtMatmulPreferenceDestroy(pref);
  if (lc) cublasLtMatrixLayoutDestroy(lc);
  if (l2) cublasLtMatrixLayoutDestroy(l2);
  if (l1) cublasLtMatrixLayoutDestroy(l1);
  if (desc) cublasLtMatmulDescDestroy(desc);
  return st;
}

}  // namespace ml
