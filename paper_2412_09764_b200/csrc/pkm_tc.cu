// Half-key scoring on the 5th-generation tensor cores (§3.1.1,
// "we first split the query as q1, q2 ... the top-k indices and scores
// obtained from the respective key sets K1, K2"):
//
//   S_half[t, h, half, a] = sum_i q[t, h, half*Dh + i] * K_half[h, a, i]
//
// bf16 x bf16 -> fp32 on tcgen05 (kind::f16, M = 128 tokens, N = up to 256
// keys, K = 16 per instruction) with the accumulator in TMEM.  Warp roles in a
// persistent 256-thread CTA (one per SM):
//   warp 0   TMA producer: 128x64 query tile + BNx64 key tile per stage
//            (128-byte swizzle, mbarrier complete_tx), 3-stage ring
//   warp 1   MMA issuer (one elected thread), commits free smem stages and
//            signals a double-buffered TMEM accumulator
//   warp 2   TMEM allocator
//   warps 4-7 epilogue: tcgen05.ld 32x32b (thread = token row) -> a 32x32 fp32
//            tile in shared memory (128-byte swizzle, double-buffered per warp)
//            -> TMA tensor store to the [T, H*2, S] scores (bulk async groups)
// The selection (half top-k) consumes the scores in pkm.cu.
#include "internal.cuh"

#include <cuda.h>

#include <cstdlib>
#include <mutex>

namespace ml {
namespace {

constexpr int kBM = 128;     // tokens per tile (UMMA_M)
constexpr int kBK = 64;      // K elements per stage = one 128-byte swizzle atom of bf16
constexpr int kStages = 4;
constexpr int kStageFloats = 32 * 32;  // one epilogue staging tile: 32 token rows x 32 scores
constexpr int kStageBufs = kStages > 3 ? 1 : 2;   // staging tiles per epilogue warp
constexpr int kThreads = 256;
constexpr uint32_t kSpinLimit = 1u << 28;  // bounded waits: trap instead of hanging

struct TcParams {
  float* scores;
  int T, H, S, Dh, Dk;
  int BN, n_sub, k_chunks, m_tiles, tiles;
  uint32_t idesc;
  uint32_t tmem_cols;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t ok = 0, n = 0;
  while (true) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
    if (ok) return;
    if (++n > kSpinLimit) __trap();
  }
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                            int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
// TMA tensor store of one [32 tokens][1][32 scores] box (bulk async group)
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* src, int c0, int c1,
                                             int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// K-major operand, 128-byte swizzle: 8-row x 128-byte atoms, 1024 B apart (SBO)
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= uint64_t((saddr >> 4) & 0x3FFFu);   // start address (16-byte units)
  d |= uint64_t(1) << 16;                   // leading byte offset (unused for SW128 K-major)
  d |= uint64_t(1024 >> 4) << 32;           // stride byte offset: next 8-row group
  d |= uint64_t(1) << 46;                   // descriptor version (sm_100)
  d |= uint64_t(2) << 61;                   // layout: SWIZZLE_128B
  return d;
}
__device__ __forceinline__ void umma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__global__ void __launch_bounds__(kThreads, 1)
    pkm_scores_tc_kernel(const __grid_constant__ CUtensorMap tmQ,
                         const __grid_constant__ CUtensorMap tmK1,
                         const __grid_constant__ CUtensorMap tmK2,
                         const __grid_constant__ CUtensorMap tmS, TcParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte aligned carve-up (swizzle-128B atoms need it)
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t bytes_a = kBM * kBK * 2;
  const uint32_t bytes_b = uint32_t(p.BN) * kBK * 2;
  uint8_t* sA = base;
  uint8_t* sB = base + kStages * bytes_a;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + kStages * bytes_b);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  // epilogue staging: two [32 rows][32] fp32 tiles per epilogue warp (1024-byte aligned)
  float* stage_all = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(full) + 1024);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmQ)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmK1)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmK2)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmS)) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(p.tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < p.tiles; t += gridDim.x) {
        const int mt = t % p.m_tiles, hh = t / p.m_tiles;
        const int h = hh >> 1, half = hh & 1;
        const CUtensorMap* tmK = half ? &tmK2 : &tmK1;
        for (int n = 0; n < p.n_sub; ++n) {
          for (int kc = 0; kc < p.k_chunks; ++kc) {
            mbar_wait(&empty[stage], phase ^ 1);
            mbar_expect_tx(&full[stage], bytes_a + bytes_b);
            tma_load_2d(sA + stage * bytes_a, &tmQ, &full[stage], h * p.Dk + half * p.Dh + kc * kBK,
                        mt * kBM);
            tma_load_2d(sB + stage * bytes_b, tmK, &full[stage], kc * kBK, h * p.S + n * p.BN);
            if (++stage == kStages) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = blockIdx.x; t < p.tiles; t += gridDim.x) {
        for (int n = 0; n < p.n_sub; ++n) {
          mbar_wait(&tempty[acc], acc_phase ^ 1);
          tc_fence_after();
          const uint32_t dcol = tmem_base + uint32_t(acc * p.BN);
          for (int kc = 0; kc < p.k_chunks; ++kc) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            const uint64_t ad = sw128_desc(smem_u32(sA + stage * bytes_a));
            const uint64_t bd = sw128_desc(smem_u32(sB + stage * bytes_b));
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k)  // 16 bf16 = 32 bytes = 2 descriptor units
              umma_f16(dcol, ad + 2 * k, bd + 2 * k, p.idesc, (kc | k) != 0 ? 1u : 0u);
            umma_commit(&empty[stage]);
            if (++stage == kStages) {
              stage = 0;
              phase ^= 1;
            }
          }
          umma_commit(&tfull[acc]);
          if (++acc == 2) {
            acc = 0;
            acc_phase ^= 1;
          }
        }
      }
    }
  } else if (warp >= 4) {  // ---------------- epilogue: TMEM -> fp32 scores
    const int q4 = warp & 3;
    int acc = 0;
    uint32_t acc_phase = 0;
    int it = 0;
    float* stg0 = stage_all + (warp - 4) * kStageBufs * kStageFloats;
    for (int t = blockIdx.x; t < p.tiles; t += gridDim.x) {
      const int mt = t % p.m_tiles, hh = t / p.m_tiles;
      const int row0 = mt * kBM + q4 * 32;   // this warp's 32 token rows
      for (int n = 0; n < p.n_sub; ++n) {
        mbar_wait(&tfull[acc], acc_phase);
        tc_fence_after();
        for (int c0 = 0; c0 < p.BN; c0 += 32, ++it) {
          uint32_t r[32];
          tmem_ld32(tmem_base + (uint32_t(q4 * 32) << 16) + uint32_t(acc * p.BN + c0), r);
          float* stg = stg0 + (it % kStageBufs) * kStageFloats;
          // the store issued from this buffer kStageBufs chunks ago must have read it
          if (lane == 0) {
            if constexpr (kStageBufs == 2) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            else asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          }
          __syncwarp();
          // row `lane`, 16-byte chunk v at position v ^ (lane & 7): the 128-byte
          // swizzle of the tensor map (conflict-free, 8 lanes per 128-B phase)
#pragma unroll
          for (int v = 0; v < 8; ++v)
            *reinterpret_cast<uint4*>(stg + lane * 32 + ((v ^ (lane & 7)) << 2)) =
                make_uint4(r[4 * v], r[4 * v + 1], r[4 * v + 2], r[4 * v + 3]);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {   // rows past T are clipped by the tensor map
            tma_store_3d(&tmS, stg, n * p.BN + c0, hh, row0);
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
        }
        tc_fence_before();
        mbar_arrive(&tempty[acc]);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(p.tmem_cols));
  }
}

// ------------------------------------------------------------ host
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  return fn;
}

mlStatus make_map(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer,
                  uint64_t row_bytes, uint32_t box_inner, uint32_t box_outer) {
  EncodeFn f = encode_fn();
  if (!f) return fail(ML_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {row_bytes};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = f(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box,
                 estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(ML_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
  return ML_OK;
}

int tc_bn(int S) { return S >= 256 ? 256 : S; }

}  // namespace

bool pkm_scores_tc_eligible(const mlPkmShape& sh) {
  static int force_simt = -1;
  if (force_simt < 0) {
    const char* e = std::getenv("ML_PKM_SIMT");
    force_simt = (e && e[0] == '1') ? 1 : 0;
  }
  if (force_simt) return false;
  if (sh.dtype != ML_BF16) return false;    // fp32 inputs: exact fp32 FMA on the SIMT path
  const int Dh = sh.Dk / 2;
  if (Dh % kBK) return false;
  const int BN = tc_bn(sh.S);
  if (BN < 32 || (BN & (BN - 1)) || sh.S % BN) return false;
  return sh.T > 0;
}

mlStatus launch_pkm_scores_tc(const mlPkmShape& sh, const void* q, const void* K1, const void* K2,
                              float* scores, cudaStream_t s) {
  const int Dh = sh.Dk / 2;
  TcParams p;
  p.scores = scores;
  p.T = sh.T; p.H = sh.H; p.S = sh.S; p.Dh = Dh; p.Dk = sh.Dk;
  p.BN = tc_bn(sh.S);
  p.n_sub = sh.S / p.BN;
  p.k_chunks = Dh / kBK;
  p.m_tiles = (sh.T + kBM - 1) / kBM;
  p.tiles = p.m_tiles * sh.H * 2;
  // instruction descriptor: D fp32, A/B bf16, both K-major, N = BN, M = 128
  p.idesc = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(p.BN >> 3) << 17) | (uint32_t(kBM >> 4) << 24);
  uint32_t cols = 32;
  while (cols < uint32_t(2 * p.BN)) cols <<= 1;
  p.tmem_cols = cols;
  CUtensorMap mq, mk1, mk2;
  ML_TRY(make_map(&mq, q, uint64_t(sh.H) * sh.Dk, uint64_t(sh.T), uint64_t(sh.H) * sh.Dk * 2, kBK, kBM));
  ML_TRY(make_map(&mk1, K1, uint64_t(Dh), uint64_t(sh.H) * sh.S, uint64_t(Dh) * 2, kBK, p.BN));
  ML_TRY(make_map(&mk2, K2, uint64_t(Dh), uint64_t(sh.H) * sh.S, uint64_t(Dh) * 2, kBK, p.BN));
  CUtensorMap ms;
  {
    EncodeFn f = encode_fn();
    if (!f) return fail(ML_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    // scores [T][H*2][S] fp32; box = 32 scores x 1 (head, half) x 32 tokens
    cuuint64_t dims[3] = {uint64_t(sh.S), uint64_t(sh.H) * 2, uint64_t(sh.T)};
    cuuint64_t strides[2] = {uint64_t(sh.S) * 4, uint64_t(sh.H) * 2 * sh.S * 4};
    cuuint32_t box[3] = {32, 1, 32};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = f(&ms, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, scores, dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(ML_ERR_CUDA, "cuTensorMapEncodeTiled (scores) failed: " + std::to_string(int(r)));
  }
  const size_t smem = 1024 + size_t(kStages) * (kBM * kBK * 2 + size_t(p.BN) * kBK * 2) + 1024 +
                      size_t(4) * kStageBufs * kStageFloats * sizeof(float);
  static size_t configured = 0;
  if (smem > configured) {
    ML_CUDA_TRY(cudaFuncSetAttribute(pkm_scores_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(smem)));
    configured = smem;
  }
  const int grid = std::min(p.tiles, num_sms());
  pkm_scores_tc_kernel<<<grid, kThreads, smem, s>>>(mq, mk1, mk2, ms, p);
  ML_LAUNCH_CHECK("pkm_scores_tc");
  return ML_OK;
}

}  // namespace ml
