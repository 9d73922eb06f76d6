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
#include "tc_util.cuh"

#include <cuda.h>

#include <cmath>
#include <cstdlib>
#include <mutex>

namespace ml {
namespace {
using namespace tc;

constexpr int kBM = 128;     // tokens per tile (UMMA_M)
constexpr int kBK = 64;      // K elements per stage = one 128-byte swizzle atom of bf16
constexpr int kStages = 4;
constexpr int kStageFloats = 32 * 32;  // one epilogue staging tile: 32 token rows x 32 scores
#ifndef ML_SCORE_STAGE_BUFS
#define ML_SCORE_STAGE_BUFS 1
#endif
// staging tiles per epilogue warp (build switch; 2 tiles with the 4 stages
// fit in 226 KiB and measured equal at C2: 0.166-0.175 ms either way,
// scripts/gpu_ab_so_scores.sh)
constexpr int kStageBufs = ML_SCORE_STAGE_BUFS;
constexpr int kThreads = 256;
// epilogue warps of the single-CTA scoring kernel (build switch): 8 = two
// warps per TMEM lane quarter, each draining half of a subtile's columns
// (C2: 0.166-0.168 vs 0.170 ms with 4, scripts/gpu_ab_so_scores.sh)
#ifndef ML_SCORE_EPI_WARPS
#define ML_SCORE_EPI_WARPS 8
#endif
constexpr int kEpiWarps = ML_SCORE_EPI_WARPS;
constexpr int kThreadsS = 128 + 32 * kEpiWarps;

struct TcParams {
  float* scores;
  float* cmax;      // nullable: [T][H*2][S/32] chunk maxima
  int T, H, S, Dh, Dk;
  int BN, n_sub, k_chunks, m_tiles, tiles;
  uint32_t idesc;
  uint32_t tmem_cols;
};

// ---------------- TMA producer (one thread): the 128-token query tile and the
// BN-key half-key tile of every K-chunk of every subtile, STAGES-deep ring
template <int STAGES, bool SLEEP = false>
__device__ __forceinline__ void tc_producer(const CUtensorMap* tmQ, const CUtensorMap* tmK1,
                                            const CUtensorMap* tmK2, uint8_t* sA, uint8_t* sB,
                                            uint64_t* full, uint64_t* empty, uint32_t bytes_a,
                                            uint32_t bytes_b, const TcParams& p) {
  int stage = 0;
  uint32_t phase = 0;
  for (int t = blockIdx.x; t < p.tiles; t += gridDim.x) {
    const int mt = t % p.m_tiles, hh = t / p.m_tiles;
    const int h = hh >> 1, half = hh & 1;
    const CUtensorMap* tmK = half ? tmK2 : tmK1;
    for (int n = 0; n < p.n_sub; ++n) {
      for (int kc = 0; kc < p.k_chunks; ++kc) {
        mbar_wait_t<SLEEP>(&empty[stage], phase ^ 1);
        mbar_expect_tx(&full[stage], bytes_a + bytes_b);
        tma_load_2d(sA + stage * bytes_a, tmQ, &full[stage], h * p.Dk + half * p.Dh + kc * kBK,
                    mt * kBM);
        tma_load_2d(sB + stage * bytes_b, tmK, &full[stage], kc * kBK, h * p.S + n * p.BN);
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  }
}

// ---------------- MMA issuer (one thread): D[acc] = Q_tile x K_tile^T per
// subtile into a double-buffered TMEM accumulator; commits free smem stages
template <int STAGES, bool SLEEP = false>
__device__ __forceinline__ void tc_mma(uint8_t* sA, uint8_t* sB, uint64_t* full, uint64_t* empty,
                                       uint64_t* tfull, uint64_t* tempty, uint32_t bytes_a,
                                       uint32_t bytes_b, uint32_t tmem_base, const TcParams& p) {
  int stage = 0;
  uint32_t phase = 0;
  int acc = 0;
  uint32_t acc_phase = 0;
  for (int t = blockIdx.x; t < p.tiles; t += gridDim.x) {
    for (int n = 0; n < p.n_sub; ++n) {
      mbar_wait_t<SLEEP>(&tempty[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t dcol = tmem_base + uint32_t(acc * p.BN);
      for (int kc = 0; kc < p.k_chunks; ++kc) {
        mbar_wait_t<SLEEP>(&full[stage], phase);
        tc_fence_after();
        const uint64_t ad = sw128_desc(smem_u32(sA + stage * bytes_a));
        const uint64_t bd = sw128_desc(smem_u32(sB + stage * bytes_b));
#pragma unroll
        for (int k = 0; k < kBK / 16; ++k)  // 16 bf16 = 32 bytes = 2 descriptor units
          umma_f16(dcol, ad + 2 * k, bd + 2 * k, p.idesc, (kc | k) != 0 ? 1u : 0u);
        umma_commit(&empty[stage]);
        if (++stage == STAGES) {
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

__global__ void __launch_bounds__(kThreadsS, 1)
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
      mbar_init(&tempty[i], 32 * kEpiWarps);
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
    if (lane == 0) tc_producer<kStages>(&tmQ, &tmK1, &tmK2, sA, sB, full, empty, bytes_a, bytes_b, p);
  } else if (warp == 1) {
    if (lane == 0) tc_mma<kStages>(sA, sB, full, empty, tfull, tempty, bytes_a, bytes_b, tmem_base, p);
  } else if (warp >= 4) {  // ---------------- epilogue: TMEM -> fp32 scores
    const int q4 = warp & 3;
    // column part of each subtile this warp drains (kEpiWarps / 4 parts)
    const int nparts = min(kEpiWarps / 4, p.BN / 32), part = (warp - 4) >> 2;
    const int cw = part < nparts ? p.BN / nparts : 0, cbeg = part * (p.BN / nparts);
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
        float cm[8];          // this row's chunk maxima of the subtile (BN / 32 <= 8)
        for (int c0 = cbeg; c0 < cbeg + cw; c0 += 32, ++it) {
          uint32_t r[32];
          tmem_ld32(tmem_base + (uint32_t(q4 * 32) << 16) + uint32_t(acc * p.BN + c0), r);
          if (p.cmax) {
            float m = __uint_as_float(r[0]);
#pragma unroll
            for (int j = 1; j < 32; ++j) m = fmaxf(m, __uint_as_float(r[j]));
#pragma unroll
            for (int j = 0; j < 8; ++j)
              if (j == (c0 >> 5)) cm[j] = m;
          }
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
        if (p.cmax && row0 + lane < p.T && part < nparts) {
          float* dst = p.cmax + (int64_t(row0 + lane) * p.H * 2 + hh) * (p.S >> 5) + (n * p.BN >> 5);
          if (nparts > 1) {   // this warp's chunks only
#pragma unroll
            for (int j = 0; j < 8; ++j)
              if (j >= (cbeg >> 5) && j < ((cbeg + cw) >> 5)) dst[j] = cm[j];
          } else if (p.BN == 256) {   // 32 contiguous bytes per row
            reinterpret_cast<float4*>(dst)[0] = make_float4(cm[0], cm[1], cm[2], cm[3]);
            reinterpret_cast<float4*>(dst)[1] = make_float4(cm[4], cm[5], cm[6], cm[7]);
          } else {
#pragma unroll
            for (int j = 0; j < 8; ++j)
              if (j < (p.BN >> 5)) dst[j] = cm[j];
          }
        }
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


// ---- CTA-pair scoring (cta_group::2, M = 256 tokens): the two CTAs of a
// cluster take adjacent 128-token m-tiles of the same (h, half); each loads
// its own query rows and HALF of every 256-key subtile, the leader issues one
// M = 256 MMA per k-step, each CTA accumulates its rows in its own TMEM and
// runs the same epilogue (scores by TMA store, chunk maxima).  Per CTA the
// key bytes per stage halve.
constexpr int kStagesP = 6;

template <bool CHUNKS>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    pkm_scores_tc2_kernel(const __grid_constant__ CUtensorMap tmQ,
                          const __grid_constant__ CUtensorMap tmK1,
                          const __grid_constant__ CUtensorMap tmK2,
                          const __grid_constant__ CUtensorMap tmS, TcParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t bytes_a = kBM * kBK * 2;
  const uint32_t bytes_b = uint32_t(p.BN / 2) * kBK * 2;
  uint8_t* sA = base;
  uint8_t* sB = base + kStagesP * bytes_a;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + kStagesP * bytes_b);
  uint64_t* empty = full + kStagesP;
  uint64_t* tfull = empty + kStagesP;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  float* stage_all = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(full) + 1024);

  const uint32_t rank = cluster_ctarank();
  const int cl = int(blockIdx.x >> 1), ncl = int(gridDim.x >> 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kStagesP; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 256);
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
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(p.tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // unit -> (m-tile pair mp, hh = h*2 + half); p.m_tiles holds the pair count
  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer (both CTAs)
      int stage = 0;
      uint32_t phase = 0;
      for (int u = cl; u < p.tiles; u += ncl) {
        const int mp = u % p.m_tiles, hh = u / p.m_tiles;
        const int h = hh >> 1, half = hh & 1;
        const int mt = 2 * mp + int(rank);
        const CUtensorMap* tmK = half ? &tmK2 : &tmK1;
        for (int n = 0; n < p.n_sub; ++n) {
          for (int kc = 0; kc < p.k_chunks; ++kc) {
            mbar_wait_t<true>(&empty[stage], phase ^ 1);
            if (rank == 0) mbar_expect_tx(&full[stage], 2 * (bytes_a + bytes_b));
            const uint32_t lbar = mapa_shared(smem_u32(&full[stage]), 0);
            tma_load_2d_pair(sA + stage * bytes_a, &tmQ, lbar, h * p.Dk + half * p.Dh + kc * kBK,
                             mt * kBM);
            tma_load_2d_pair(sB + stage * bytes_b, tmK, lbar, kc * kBK,
                             h * p.S + n * p.BN + int(rank) * (p.BN / 2));
            if (++stage == kStagesP) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {  // ---------------- MMA issuer: the leader
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int u = cl; u < p.tiles; u += ncl) {
        for (int n = 0; n < p.n_sub; ++n) {
          mbar_wait_t<true>(&tempty[acc], acc_phase ^ 1);
          tc_fence_after();
          const uint32_t dcol = tmem_base + uint32_t(acc * p.BN);
          for (int kc = 0; kc < p.k_chunks; ++kc) {
            mbar_wait_t<true>(&full[stage], phase);
            tc_fence_after();
            const uint64_t ad = sw128_desc(smem_u32(sA + stage * bytes_a));
            const uint64_t bd = sw128_desc(smem_u32(sB + stage * bytes_b));
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k)
              umma_f16_pair(dcol, ad + 2 * k, bd + 2 * k, p.idesc, (kc | k) != 0 ? 1u : 0u);
            umma_commit_pair(&empty[stage]);
            if (++stage == kStagesP) {
              stage = 0;
              phase ^= 1;
            }
          }
          umma_commit_pair(&tfull[acc]);
          if (++acc == 2) {
            acc = 0;
            acc_phase ^= 1;
          }
        }
      }
    }
  } else if (warp >= 4) {  // ---------------- epilogue (both CTAs): own rows
    const int q4 = warp & 3;
    int acc = 0;
    uint32_t acc_phase = 0;
    int it = 0;
    float* stg0 = stage_all + (warp - 4) * 2 * kStageFloats;
    for (int u = cl; u < p.tiles; u += ncl) {
      const int mp = u % p.m_tiles, hh = u / p.m_tiles;
      const int mt = 2 * mp + int(rank);
      const int row0 = mt * kBM + q4 * 32;
      for (int n = 0; n < p.n_sub; ++n) {
        mbar_wait(&tfull[acc], acc_phase);
        tc_fence_after();
        float cm[8];
        for (int c0 = 0; c0 < p.BN; c0 += 32, ++it) {
          uint32_t r[32];
          tmem_ld32(tmem_base + (uint32_t(q4 * 32) << 16) + uint32_t(acc * p.BN + c0), r);
          if constexpr (CHUNKS) {
            float m = __uint_as_float(r[0]);
#pragma unroll
            for (int j = 1; j < 32; ++j) m = fmaxf(m, __uint_as_float(r[j]));
#pragma unroll
            for (int j = 0; j < 8; ++j)
              if (j == (c0 >> 5)) cm[j] = m;
          }
          float* stg = stg0 + (it & 1) * kStageFloats;
          if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          __syncwarp();
#pragma unroll
          for (int v = 0; v < 8; ++v)
            *reinterpret_cast<uint4*>(stg + lane * 32 + ((v ^ (lane & 7)) << 2)) =
                make_uint4(r[4 * v], r[4 * v + 1], r[4 * v + 2], r[4 * v + 3]);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            tma_store_3d(&tmS, stg, n * p.BN + c0, hh, row0);
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
        }
        tc_fence_before();
        if (rank == 0) mbar_arrive(&tempty[acc]);
        else mbar_arrive_remote(mapa_shared(smem_u32(&tempty[acc]), 0));
        if (CHUNKS && row0 + lane < p.T) {
          float* dst = p.cmax + (int64_t(row0 + lane) * p.H * 2 + hh) * (p.S >> 5) + (n * p.BN >> 5);
          reinterpret_cast<float4*>(dst)[0] = make_float4(cm[0], cm[1], cm[2], cm[3]);
          reinterpret_cast<float4*>(dst)[1] = make_float4(cm[4], cm[5], cm[6], cm[7]);
        }
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
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(p.tmem_cols));
  }
}

// ============================================================================
// Scoring fused with the half top-k filter (no score matrix in HBM; opt-in).
//
// The epilogue thread that owns token row r of a 128-token tile (tcgen05.ld
// 32x32b: thread = TMEM lane = row) sees every score of its (t, h, half) row,
// S / BN subtiles of BN = 256 keys, and keeps only a small candidate set that
// provably contains the row's k best ("the top-k indices ... obtained
// from the respective key sets"; ties resolved later by (score, lower index)):
//  * subtile 0's mean / standard deviation place a ladder of levels
//    L_j = L_0 + j*delta; theta_0 = the highest level with >= k of the
//    subtile's 256 scores at or above it (binary search, exact counts) -- a
//    valid lower bound of the row's k-th largest score whatever the
//    statistics were (they only place the levels);
//  * every subtile is filtered with v >= theta; survivors (score, key index)
//    go to a per-thread list in shared memory, which therefore holds every
//    score seen so far that is >= theta;
//  * when a list would overflow, theta is raised to the highest of the next
//    levels with >= k list entries at or above it (exact counts, by the
//    previous point) and the entries below it are dropped.
// All top-k scores of the row are >= the final theta >= the theta in force
// when they were seen, so all of them are candidates.  The row's candidates
// are written as 64-bit keys; rows whose list still overflowed are listed for
// an exact fallback.  The selection among the candidates happens in the
// combine kernel (pkm.cu).
constexpr int kSelStages = 3;     // ring depth (shared memory goes to the candidate lists)
constexpr int kCand = 96;         // candidate list capacity per row
constexpr int kLevels = 48;       // threshold ladder
constexpr int kEpi = 128;         // epilogue threads (one per tile row)

struct SelOut {
  uint64_t* cand;      // [rows][kCand] keys (ord(score) << 32 | ~a), first cnt valid
  int32_t* cnt;        // [rows]: candidates, or -1 (overflow: exact fallback)
  int32_t* fail_rows;  // list of rows needing the fallback
  int32_t* fail_n;     // its length (zeroed before the launch)
  float z0, dz;        // ladder: L_0 = mean + z0 sd, delta = dz sd
  int k;
  int probe;           // timing probes (ML_SEL_PROBE): 1 = TMEM loads only, 2 = + ladder and
                       // histogram, 3 = + survivor masks (no list writes), 0 = full
};

__device__ __forceinline__ uint64_t sel_key(float v, uint32_t a) {
  return (uint64_t(ord_f32(v)) << 32) | uint64_t(0xFFFFFFFFu - a);
}

__global__ void __launch_bounds__(kThreads, 1)
    pkm_scores_select_tc_kernel(const __grid_constant__ CUtensorMap tmQ,
                                const __grid_constant__ CUtensorMap tmK1,
                                const __grid_constant__ CUtensorMap tmK2, TcParams p, SelOut o) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte aligned, keeping the pointer's shared-space provenance (STS/LDS
  // for the candidate lists instead of generic stores)
  uint8_t* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t bytes_a = kBM * kBK * 2;
  const uint32_t bytes_b = uint32_t(p.BN) * kBK * 2;
  uint8_t* sA = base;
  uint8_t* sB = base + kSelStages * bytes_a;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + kSelStages * bytes_b);
  uint64_t* empty = full + kSelStages;
  uint64_t* tfull = empty + kSelStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  // per-row lists, [slot][row] so that every lane always hits its own bank
  float* c_val = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(full) + 256);
  uint16_t* c_key = reinterpret_cast<uint16_t*>(c_val + kCand * kEpi);
  uint32_t* stage = reinterpret_cast<uint32_t*>(c_key + kCand * kEpi);   // [row][8]: filter staging

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kSelStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], kEpi);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmQ)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmK1)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmK2)) : "memory");
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
    if (lane == 0) tc_producer<kSelStages, true>(&tmQ, &tmK1, &tmK2, sA, sB, full, empty, bytes_a, bytes_b, p);
  } else if (warp == 1) {
    if (lane == 0) tc_mma<kSelStages, true>(sA, sB, full, empty, tfull, tempty, bytes_a, bytes_b, tmem_base, p);
  } else if (warp >= 4) {
    const int q4 = warp & 3;
    const int er = q4 * 32 + lane;          // this thread's tile row (= TMEM lane)
    float* cv = c_val + er;                 // cv[e * kEpi]: e-th candidate score
    uint16_t* ck = c_key + er;
    const int H2 = 2 * p.H;
    int acc = 0;
    uint32_t acc_phase = 0;
    constexpr int NC = 256 / 32;            // 32-column chunks per subtile (BN = 256)
    // bit i of the result: score i of the 32-column chunk r is >= th (two
    // instructions per score: the sign of v - th funnel-shifted in; -0 as th
    // so that a -0 score counts as >= +0)
    auto ge_mask = [](const uint32_t* r, float th0) {
      const float th = th0 == 0.f ? -0.f : th0;
      uint32_t neg = 0;
#pragma unroll
      for (int i = 0; i < 32; ++i)
        neg = __funnelshift_l(__float_as_uint(__uint_as_float(r[i]) - th), neg, 1);
      return __brev(~neg);
    };
    for (int t = blockIdx.x; t < p.tiles; t += gridDim.x) {
      const int mt = t % p.m_tiles, hh = t / p.m_tiles;
      const int tok = mt * kBM + er;
      const bool valid = tok < p.T;
      int cnt = 0;
      bool ovf = false;
      float L0 = 0.f, delta = 1.f;
      // theta = L_lt: the list holds every score seen so far that is >= theta,
      // and at least k scores seen so far are >= theta (lt = -1: none yet)
      int lt = -1;
      float theta = -INFINITY;
      auto level = [&](int j) { return fmaf(float(j), delta, L0); };
      // raise theta to the highest of the next 8 levels with >= k list entries
      // at or above it (the list holds all scores >= theta, so these are the
      // exact counts), then drop the entries below it (order kept)
      auto compact = [&]() {
        int c8[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        float lv[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) lv[j] = level(lt + 1 + j);
#pragma unroll 1
        for (int e = 0; e < cnt; ++e) {
          const float v = cv[e * kEpi];
#pragma unroll
          for (int j = 0; j < 8; ++j) c8[j] += v >= lv[j] ? 1 : 0;
        }
        int up = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) up += (c8[j] >= o.k && lt + 1 + j < kLevels) ? 1 : 0;
        if (up > 0) {
          lt += up;
          theta = level(lt);
        }
        int w = 0;
#pragma unroll 1
        for (int e = 0; e < cnt; ++e) {
          const float v = cv[e * kEpi];
          const uint16_t kk = ck[e * kEpi];
          cv[w * kEpi] = v;                 // w <= e: harmless when not kept
          ck[w * kEpi] = kk;
          w += v >= theta ? 1 : 0;
        }
        cnt = w;
      };
      for (int n = 0; n < p.n_sub; ++n) {
        mbar_wait(&tfull[acc], acc_phase);
        tc_fence_after();
        const uint32_t ta = tmem_base + (uint32_t(q4 * 32) << 16) + uint32_t(acc * p.BN);
        uint32_t ra[32], rb[32];
        // walk the subtile's 8 chunks with the next TMEM load in flight
        auto walk = [&](auto&& fn) {
          tmem_ld32_nowait(ta, ra);
          tmem_wait_ld(ra);
#pragma unroll 1
          for (int c = 0; c < NC; c += 2) {
            tmem_ld32_nowait(ta + uint32_t(32 * (c + 1)), rb);
            fn(ra, c);
            tmem_wait_ld(rb);
            if (c + 2 < NC) tmem_ld32_nowait(ta + uint32_t(32 * (c + 2)), ra);
            fn(rb, c + 1);
            if (c + 2 < NC) tmem_wait_ld(ra);
          }
        };
        if (n == 0 && o.probe != 1) {
          // the ladder from the subtile's mean / sd, then theta_0 = the highest
          // level with >= k of the subtile's 256 scores at or above it (binary
          // search; every count is exact)
          float sum = 0.f, sq = 0.f;
          walk([&](const uint32_t* r, int) {
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              const float v = __uint_as_float(r[i]);
              sum += v;
              sq = fmaf(v, v, sq);
            }
          });
          const float mu = sum / float(p.BN);
          const float sd = sqrtf(fmaxf(sq / float(p.BN) - mu * mu, 0.f));
          delta = fmaxf(sd * o.dz, fmaxf(fabsf(mu), 1e-20f) * 1e-6f);
          L0 = fmaf(o.z0, sd, mu);
          int lo = -1, hi = kLevels;        // count(>= L_lo) >= k (lo = -1: -inf), count(>= L_hi) < k
#pragma unroll 1
          while (__any_sync(0xffffffffu, hi - lo > 1)) {
            const int mid = (lo + hi) >> 1;
            const float lm = level(mid);
            int c = 0;
            walk([&](const uint32_t* r, int) { c += __popc(ge_mask(r, lm)); });
            if (hi - lo > 1) {
              if (c >= o.k) lo = mid;
              else hi = mid;
            }
          }
          lt = lo;
          theta = lt >= 0 ? level(lt) : -INFINITY;
        }
        // filter: survivors (v >= theta) are staged in 8-score groups and
        // copied to the list; a list that would overflow is first compacted
        // (theta raised), and if it still does not fit the row falls back
        const int col_base = n * p.BN;
        walk([&](const uint32_t* r, int c) {
          if (o.probe == 1 || o.probe == 2) {
            uint32_t x = 0;
#pragma unroll
            for (int i = 0; i < 32; ++i) x ^= r[i];
            if (x == 0x12345678u) cnt += 1;
            return;
          }
          uint32_t m = ge_mask(r, (ovf || !valid) ? INFINITY : theta);
          if (o.probe == 3) {
            if (m == 0x12345678u) cnt += 1;
            return;
          }
          if (__any_sync(0xffffffffu, cnt + __popc(m) > kCand)) {
            if (cnt + __popc(m) > kCand) {
              compact();
              m = ge_mask(r, (ovf || !valid) ? INFINITY : theta);
              const int room = kCand - cnt;
              if (__popc(m) > room) {       // still no room: keep what fits, fall back
                ovf = true;
                while (__popc(m) > room) m &= ~(1u << (31 - __clz(m)));
              }
            }
          }
          const uint32_t col0 = uint32_t(col_base + 32 * c);
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            const uint32_t mg = (m >> (8 * g)) & 0xFFu;
            if (__any_sync(0xffffffffu, mg != 0u)) {
              uint4* st = reinterpret_cast<uint4*>(stage + er * 8);
              st[0] = make_uint4(r[8 * g + 0], r[8 * g + 1], r[8 * g + 2], r[8 * g + 3]);
              st[1] = make_uint4(r[8 * g + 4], r[8 * g + 5], r[8 * g + 6], r[8 * g + 7]);
#pragma unroll 1
              for (uint32_t b = mg; b; b &= b - 1u) {
                const int i = __ffs(b) - 1;
                cv[cnt * kEpi] = __uint_as_float(stage[er * 8 + i]);
                ck[cnt * kEpi] = uint16_t(col0 + uint32_t(8 * g + i));
                ++cnt;
              }
            }
          }
        });
        tc_fence_before();
        mbar_arrive(&tempty[acc]);          // the accumulator is free for the next subtile
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
      if (__any_sync(0xffffffffu, cnt > o.k)) compact();
      if (valid) {
        const int64_t row = int64_t(tok) * H2 + hh;
        if (ovf || cnt < o.k) {
          o.cnt[row] = -1;
          o.fail_rows[atomicAdd(o.fail_n, 1)] = int32_t(row);
        } else {
          uint64_t* dst = o.cand + row * kCand;
#pragma unroll 1
          for (int e = 0; e < cnt; ++e) dst[e] = sel_key(cv[e * kEpi], ck[e * kEpi]);
          o.cnt[row] = cnt;
        }
      }
    }
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
                              float* scores, cudaStream_t s, float* cmax) {
  const int Dh = sh.Dk / 2;
  TcParams p;
  p.scores = scores;
  p.cmax = cmax;
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
                      size_t(kEpiWarps) * kStageBufs * kStageFloats * sizeof(float);
  static size_t configured = 0;
  if (smem > configured) {
    ML_CUDA_TRY(cudaFuncSetAttribute(pkm_scores_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(smem)));
    configured = smem;
  }
  // opt-in (ML_PKM_PAIR=1): measured equal to the single-CTA kernel (C2 0.168
  // vs 0.163 ms, S = 4096 0.649 vs 0.644, S = 8192 0.714 vs 0.721) -- the
  // score stores, not the key-tile loads the pair halves, bound it
  static const bool pair_env = [] {
    const char* e = std::getenv("ML_PKM_PAIR");
    return e && e[0] == '1';
  }();
  if (pair_env && p.BN == 256) {
    // CTA pairs: 128-key boxes of the key tables, m-tile pairs
    CUtensorMap mh1, mh2;
    ML_TRY(make_map(&mh1, K1, uint64_t(Dh), uint64_t(sh.H) * sh.S, uint64_t(Dh) * 2, kBK, p.BN / 2));
    ML_TRY(make_map(&mh2, K2, uint64_t(Dh), uint64_t(sh.H) * sh.S, uint64_t(Dh) * 2, kBK, p.BN / 2));
    TcParams pp = p;
    pp.m_tiles = (p.m_tiles + 1) / 2;
    pp.tiles = pp.m_tiles * sh.H * 2;
    pp.idesc = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(p.BN >> 3) << 17) | (uint32_t(256 >> 4) << 24);
    const size_t smem2 = 1024 + size_t(kStagesP) * (kBM * kBK * 2 + size_t(p.BN / 2) * kBK * 2) + 1024 +
                         size_t(4) * 2 * kStageFloats * sizeof(float);
    static bool attr2 = false;
    if (!attr2) {
      ML_CUDA_TRY(cudaFuncSetAttribute(pkm_scores_tc2_kernel<false>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem2)));
      ML_CUDA_TRY(cudaFuncSetAttribute(pkm_scores_tc2_kernel<true>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem2)));
      attr2 = true;
    }
    const int ncl = std::min(pp.tiles, num_sms() / 2);
    if (cmax)
      pkm_scores_tc2_kernel<true><<<2 * ncl, kThreads, smem2, s>>>(mq, mh1, mh2, ms, pp);
    else
      pkm_scores_tc2_kernel<false><<<2 * ncl, kThreads, smem2, s>>>(mq, mh1, mh2, ms, pp);
    ML_LAUNCH_CHECK("pkm_scores_tc");
    return ML_OK;
  }
  const int grid = std::min(p.tiles, num_sms());
  pkm_scores_tc_kernel<<<grid, kThreadsS, smem, s>>>(mq, mk1, mk2, ms, p);
  ML_LAUNCH_CHECK("pkm_scores_tc");
  return ML_OK;
}


// ---- fused scoring + half top-k filter (pkm_scores_select_tc_kernel)
// Opt-in (ML_PKM_FUSED=1): measured slower than the score-matrix path at C2
// (DESIGN.md §6): the per-row list management of 4 epilogue warps is latency-
// and divergence-bound.
bool pkm_select_tc_eligible(const mlPkmShape& sh) {
  static int on = -1;
  if (on < 0) {
    const char* e = std::getenv("ML_PKM_FUSED");
    on = (e && e[0] == '1') ? 1 : 0;
  }
  if (!on || sh.qk_norm) return false;
  if (!pkm_scores_tc_eligible(sh)) return false;
  return sh.S >= 512 && sh.S % 256 == 0 && sh.S <= 65535 && sh.k <= 32;
}

int pkm_select_cap() { return kCand; }

// upper-tail standard normal quantile z with P(Z > z) = pr (Acklam's rational
// approximation, |rel err| < 1.2e-9; the ladder needs no more)
static double normal_isf(double pr) {
  const double a[] = {-3.969683028665376e+01, 2.209460984245205e+02, -2.759285104469687e+02,
                      1.383577518672690e+02, -3.066479806614716e+01, 2.506628277459239e+00};
  const double b[] = {-5.447609879822406e+01, 1.615858368580409e+02, -1.556989798598866e+02,
                      6.680131188771972e+01, -1.328068155288572e+01};
  const double c[] = {-7.784894002430293e-03, -3.223964580411365e-01, -2.400758277161838e+00,
                      -2.549732539343734e+00, 4.374664141464968e+00, 2.938163982698783e+00};
  const double d[] = {7.784695709041462e-03, 3.224671290700398e-01, 2.445134137142996e+00,
                      3.754408661907416e+00};
  const double q = 1.0 - pr;   // lower-tail probability
  double x;
  if (q < 0.02425) {
    const double u = std::sqrt(-2 * std::log(q));
    x = (((((c[0] * u + c[1]) * u + c[2]) * u + c[3]) * u + c[4]) * u + c[5]) /
        ((((d[0] * u + d[1]) * u + d[2]) * u + d[3]) * u + 1);
  } else if (q > 1 - 0.02425) {
    const double u = std::sqrt(-2 * std::log(1 - q));
    x = -(((((c[0] * u + c[1]) * u + c[2]) * u + c[3]) * u + c[4]) * u + c[5]) /
        ((((d[0] * u + d[1]) * u + d[2]) * u + d[3]) * u + 1);
  } else {
    const double u = q - 0.5, r = u * u;
    x = (((((a[0] * r + a[1]) * r + a[2]) * r + a[3]) * r + a[4]) * r + a[5]) * u /
        (((((b[0] * r + b[1]) * r + b[2]) * r + b[3]) * r + b[4]) * r + 1);
  }
  return x;
}

mlStatus launch_pkm_select_tc(const mlPkmShape& sh, const void* q, const void* K1, const void* K2,
                              uint64_t* cand, int32_t* cnt, int32_t* fail_rows, int32_t* fail_n,
                              cudaStream_t s) {
  const int Dh = sh.Dk / 2;
  TcParams p;
  p.scores = nullptr;
  p.cmax = nullptr;
  p.T = sh.T; p.H = sh.H; p.S = sh.S; p.Dh = Dh; p.Dk = sh.Dk;
  p.BN = 256;
  p.n_sub = sh.S / p.BN;
  p.k_chunks = Dh / kBK;
  p.m_tiles = (sh.T + kBM - 1) / kBM;
  p.tiles = p.m_tiles * sh.H * 2;
  p.idesc = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(p.BN >> 3) << 17) | (uint32_t(kBM >> 4) << 24);
  p.tmem_cols = 512;
  SelOut o;
  o.cand = cand; o.cnt = cnt; o.fail_rows = fail_rows; o.fail_n = fail_n; o.k = sh.k;
  static const int probe = [] { const char* e = std::getenv("ML_SEL_PROBE"); return e ? std::atoi(e) : 0; }();
  o.probe = probe;
  // ladder: from well below subtile 0's k-th largest (so that >= k of its 256
  // scores are counted at L_0) to above the row's expected k-th largest
  const double za = normal_isf(double(sh.k) / p.BN) - 1.0;
  const double zb = normal_isf(double(sh.k) / sh.S) + 0.3;
  o.z0 = float(za);
  o.dz = float((zb - za) / (kLevels - 1));
  CUtensorMap mq, mk1, mk2;
  ML_TRY(make_map(&mq, q, uint64_t(sh.H) * sh.Dk, uint64_t(sh.T), uint64_t(sh.H) * sh.Dk * 2, kBK, kBM));
  ML_TRY(make_map(&mk1, K1, uint64_t(Dh), uint64_t(sh.H) * sh.S, uint64_t(Dh) * 2, kBK, p.BN));
  ML_TRY(make_map(&mk2, K2, uint64_t(Dh), uint64_t(sh.H) * sh.S, uint64_t(Dh) * 2, kBK, p.BN));
  const size_t smem = 1024 + size_t(kSelStages) * (kBM * kBK * 2 + size_t(p.BN) * kBK * 2) + 256 +
                      size_t(kCand) * kEpi * (4 + 2) + size_t(kEpi) * 8 * 4;
  static size_t configured = 0;
  if (smem > configured) {
    ML_CUDA_TRY(cudaFuncSetAttribute(pkm_scores_select_tc_kernel,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    configured = smem;
  }
  ML_CUDA_TRY(cudaMemsetAsync(fail_n, 0, sizeof(int32_t), s));
  const int grid = std::min(p.tiles, num_sms());
  pkm_scores_select_tc_kernel<<<grid, kThreads, smem, s>>>(mq, mk1, mk2, p, o);
  ML_LAUNCH_CHECK("pkm_scores_topk_tc");
  return ML_OK;
}
}  // namespace ml
