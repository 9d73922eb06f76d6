// Key / query backward contractions on the 5th-generation tensor cores
// ("keys ... are trainable parameters").
// With ds the bf16 [T, H, 2, S] matrix of the selected half-key score
// gradients (softmax_bwd, sub-keys deduplicated per (t, h, half)):
//   dq[t, h, half, :]   = sum_a ds[t, h, half, a] * K_half[h, a, :]     (MODE_DQ)
//   dK_half[h, a, :]   += sum_t ds[t, h, half, a] * q[t, h, half, :]    (MODE_DK)
// one problem per (h, half).  tcgen05.mma kind::f16 (bf16 x bf16 -> fp32 in
// TMEM), M = 128, N = BN (<= 256), K = 16 per instruction; operands staged by
// TMA with the 128-byte swizzle.  dq reads ds K-major (keys contiguous) and
// the key table MN-major (the head dim contiguous); dK reads ds MN-major
// (keys contiguous along M) and q MN-major (the head dim contiguous along N):
// no operand is transposed in memory.  Warp roles as the scoring kernel
// (pkm_tc.cu): TMA producer, MMA issuer, TMEM allocator, 4 epilogue warps
// (thread = accumulator row) storing fp32 rows (dq) or adding into them (dK).
#include "internal.cuh"
#include "tc_util.cuh"

namespace ml {
namespace {
using namespace tc;

constexpr int kBM = 128;       // accumulator rows per tile
constexpr int kBK = 64;        // K per stage (one 128-byte atom of bf16)
constexpr int kStagesB = 4;
constexpr int kThreadsB = 256;

enum Mode { MODE_DQ = 0, MODE_DK = 1 };

// the exponent an fp16 operand copy was made with (to_f16_* kernels below):
// 0 while max|x| is in [2^-2, 2^14), else ds_f16_exp
__device__ __forceinline__ int op_f16_exp(const float* amax) {
  const float m = *amax;
  return (m >= 0.25f && m < 16384.f) ? 0 : ds_f16_exp(amax);
}

struct BwdParams {
  int T, H, S, Dh, Dk, k;
  int BN, n_tiles, m_tiles, k_chunks, tiles;
  int split, stages;         // split: A = hi + lo (two bf16 tiles per stage)
  uint32_t idesc, tmem_cols;
  float* dq;                 // MODE_DQ: [T, H*Dk]
  float* dK1; float* dK2;    // MODE_DK: [H*S, Dh] each, accumulate
  // fp16 operands (pkm_bwd_f16): ds scaled by 2^e_ds, the B operand by
  // 2^e_op (ds_f16_exp of the bounds); the epilogue multiplies by 2^-(e_ds + e_op)
  const float* ds_bound;
  const float* op_bound;
};

// Smem descriptor of a 128-byte-swizzled tile.  K-major (an 8-row x 128-byte
// atom per 8 rows of M/N, atoms 1024 B apart): LBO unused, SBO = 1024.
// MN-major (rows are K; 64 contiguous M/N elements per 128-byte row; 8-row
// atoms 1024 B apart along K = SBO; the next 64 M/N elements LBO bytes on).
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= uint64_t((saddr >> 4) & 0x3FFFu);
  d |= uint64_t((lbo_bytes >> 4) & 0x3FFFu) << 16;
  d |= uint64_t((sbo_bytes >> 4) & 0x3FFFu) << 32;
  d |= uint64_t(1) << 46;                   // descriptor version (sm_100)
  d |= uint64_t(2) << 61;                   // SWIZZLE_128B
  return d;
}

template <int MODE>
__global__ void __launch_bounds__(kThreadsB, 1)
    pkm_bwd_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB1,
                      const __grid_constant__ CUtensorMap tmB2, const __grid_constant__ CUtensorMap tmD,
                      const __grid_constant__ CUtensorMap tmAlo, BwdParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t bytes_a = kBM * kBK * 2;
  const uint32_t bytes_as = bytes_a << p.split;     // A bytes per stage (hi [+ lo])
  const uint32_t bytes_b = uint32_t(p.BN) * kBK * 2;
  const int stages = p.stages;
  uint8_t* sA = base;
  uint8_t* sB = base + stages * bytes_as;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + stages * bytes_b);
  uint64_t* empty = full + kStagesB;
  uint64_t* tfull = empty + kStagesB;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  // dq epilogue staging: two [32 rows][32] fp32 tiles per epilogue warp
  // (1024-byte aligned, 128-byte swizzle of the store's tensor map)
  float* stage_all = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(full) + 1024);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < stages; ++i) {
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
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB1)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB2)) : "memory");
    if (p.split) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmAlo)) : "memory");
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
  const int nb = p.BN / 64;       // 64-column boxes of B per stage

  // tile t -> (problem pr = h*2 + half, mt, nt)
  auto decode = [&](int t, int& pr, int& mt, int& nt) {
    nt = t % p.n_tiles;
    const int r = t / p.n_tiles;
    mt = r % p.m_tiles;
    pr = r / p.m_tiles;
  };

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < p.tiles; t += gridDim.x) {
        int pr, mt, nt;
        decode(t, pr, mt, nt);
        const int h = pr >> 1, half = pr & 1;
        const CUtensorMap* tmB = half ? &tmB2 : &tmB1;
        for (int kc = 0; kc < p.k_chunks; ++kc) {
          mbar_wait_t<true>(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], bytes_as + bytes_b);
          uint8_t* a = sA + stage * bytes_as;
          uint8_t* b = sB + stage * bytes_b;
          if constexpr (MODE == MODE_DQ) {
            // A = ds (K-major): keys [pr*S + kc*64, +64) x tokens [mt*128, +128)
            tma_load_2d(a, &tmA, &full[stage], pr * p.S + kc * kBK, mt * kBM);
            if (p.split) tma_load_2d(a + bytes_a, &tmAlo, &full[stage], pr * p.S + kc * kBK, mt * kBM);
            // B = K_half[h] (MN-major): head-dim boxes x keys [h*S + kc*64, +64)
            for (int j = 0; j < nb; ++j)
              tma_load_2d(b + j * 8192, tmB, &full[stage], nt * p.BN + j * 64, h * p.S + kc * kBK);
          } else {
            // A = ds (MN-major): keys [pr*S + mt*128 + j*64, +64) x tokens [kc*64, +64)
            for (int j = 0; j < 2; ++j)
              tma_load_2d(a + j * 8192, &tmA, &full[stage], pr * p.S + mt * kBM + j * 64, kc * kBK);
            if (p.split)
              for (int j = 0; j < 2; ++j)
                tma_load_2d(a + bytes_a + j * 8192, &tmAlo, &full[stage], pr * p.S + mt * kBM + j * 64,
                            kc * kBK);
            // B = q (MN-major): head-dim boxes of (h, half) x tokens [kc*64, +64)
            for (int j = 0; j < nb; ++j)
              tma_load_2d(b + j * 8192, &tmB1, &full[stage], h * p.Dk + half * p.Dh + nt * p.BN + j * 64,
                          kc * kBK);
          }
          if (++stage == stages) {
            stage = 0;
            phase ^= 1;
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
        mbar_wait_t<true>(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t dcol = tmem_base + uint32_t(acc * p.BN);
        for (int kc = 0; kc < p.k_chunks; ++kc) {
          mbar_wait_t<true>(&full[stage], phase);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + stage * bytes_as), b0 = smem_u32(sB + stage * bytes_b);
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k) {
            // K-major: the next 16 K = 32 bytes along the row; MN-major: the
            // next 16 K rows = two 8-row atoms = 2048 bytes
            const uint64_t ad = MODE == MODE_DQ ? desc_sw128(a0 + 32 * k, 16, 1024)
                                                : desc_sw128(a0 + 2048 * k, 8192, 1024);
            const uint64_t bd = desc_sw128(b0 + 2048 * k, 8192, 1024);
            umma_f16(dcol, ad, bd, p.idesc, (kc | k) != 0 ? 1u : 0u);
            if (p.split) umma_f16(dcol, ad + ((bytes_a >> 4) & 0x3FFFu), bd, p.idesc, 1u);  // + lo x B
          }
          umma_commit(&empty[stage]);
          if (++stage == stages) {
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
  } else if (warp >= 4) {  // ---------------- epilogue: TMEM -> fp32 rows
    const int q4 = warp & 3;
    const float ds_inv =
        p.ds_bound ? ldexpf(1.f, -(ds_f16_exp_ds(p.ds_bound, p.k) + op_f16_exp(p.op_bound))) : 1.f;
    int sbuf = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = blockIdx.x; t < p.tiles; t += gridDim.x) {
      int pr, mt, nt;
      decode(t, pr, mt, nt);
      const int h = pr >> 1, half = pr & 1;
      const int row = mt * kBM + q4 * 32 + lane;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      float* dst;
      bool valid;
      if constexpr (MODE == MODE_DQ) {
        valid = row < p.T;
        dst = p.dq + int64_t(row) * p.H * p.Dk + h * p.Dk + half * p.Dh + nt * p.BN;
      } else {
        valid = true;                        // S % 128 == 0
        dst = (half ? p.dK2 : p.dK1) + (int64_t(h) * p.S + row) * p.Dh + nt * p.BN;
      }
      for (int c0 = 0; c0 < p.BN; c0 += 32) {
        uint32_t r[32];
        tmem_ld32(tmem_base + (uint32_t(q4 * 32) << 16) + uint32_t(acc * p.BN + c0), r);
#pragma unroll
        for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * ds_inv);
        if constexpr (MODE == MODE_DQ) {
          // stage the 32x32 fp32 chunk (128-byte swizzle) and TMA-store it;
          // rows past T are clipped by the tensor map
          float* stg = stage_all + ((warp - 4) * 2 + (sbuf & 1)) * 1024;
          if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          __syncwarp();
#pragma unroll
          for (int v = 0; v < 8; ++v)
            *reinterpret_cast<uint4*>(stg + lane * 32 + ((v ^ (lane & 7)) << 2)) =
                make_uint4(r[4 * v], r[4 * v + 1], r[4 * v + 2], r[4 * v + 3]);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            asm volatile(
                "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                    reinterpret_cast<uint64_t>(&tmD)),
                "r"(smem_u32(stg)), "r"(h * p.Dk + half * p.Dh + nt * p.BN + c0),
                "r"(mt * kBM + q4 * 32)
                : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
          ++sbuf;
          continue;
        }
        if (valid) {
          float4* d4 = reinterpret_cast<float4*>(dst + c0);
#pragma unroll
          for (int v = 0; v < 8; ++v) {
            float4 x = make_float4(__uint_as_float(r[4 * v]), __uint_as_float(r[4 * v + 1]),
                                   __uint_as_float(r[4 * v + 2]), __uint_as_float(r[4 * v + 3]));
            if constexpr (MODE == MODE_DK) {
              const float4 o = d4[v];
              x.x += o.x; x.y += o.y; x.z += o.z; x.w += o.w;
            }
            d4[v] = x;
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
    if (MODE == MODE_DQ && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
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

// ---- CTA-pair form (cta_group::2, M = 256): the two CTAs of a cluster take
// two adjacent 128-row m-tiles of the same (h, half, n-tile); each loads its
// own A rows and HALF of the B columns, the leader issues one M = 256 MMA per
// k-step, each CTA accumulates its rows in its own TMEM.  Per CTA the B bytes
// per stage halve (the key / query tile is shared across the pair), so the
// TMA traffic that bounds the single-CTA kernel drops by a third.
constexpr int kStagesP = 6;

template <int MODE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreadsB, 1)
    pkm_bwd_tc2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB1,
                       const __grid_constant__ CUtensorMap tmB2, const __grid_constant__ CUtensorMap tmD,
                       BwdParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t bytes_a = kBM * kBK * 2;                      // this CTA's 128 rows x 64 K
  const uint32_t bytes_b = uint32_t(p.BN / 2) * kBK * 2;       // this CTA's half of the N columns
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
      mbar_init(&tempty[i], 256);     // both CTAs' epilogue threads (leader's copy is used)
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB1)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB2)) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(p.tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();                      // peer barriers initialised, TMEM allocated in both
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int nbh = p.BN / 128;          // 64-column B boxes per CTA per stage

  // unit -> (problem pr = h*2 + half, m-tile pair mp, n-tile nt)
  auto decode = [&](int u, int& pr, int& mp, int& nt) {
    nt = u % p.n_tiles;
    const int r = u / p.n_tiles;
    mp = r % p.m_tiles;               // m_tiles holds the PAIR count here
    pr = r / p.m_tiles;
  };

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer (both CTAs, each its own rows / columns)
      int stage = 0;
      uint32_t phase = 0;
      for (int u = cl; u < p.tiles; u += ncl) {
        int pr, mp, nt;
        decode(u, pr, mp, nt);
        const int h = pr >> 1, half = pr & 1;
        const int mt = 2 * mp + int(rank);
        const CUtensorMap* tmB = half ? &tmB2 : &tmB1;
        for (int kc = 0; kc < p.k_chunks; ++kc) {
          mbar_wait_t<true>(&empty[stage], phase ^ 1);
          if (rank == 0) mbar_expect_tx(&full[stage], 2 * (bytes_a + bytes_b));
          const uint32_t lbar = mapa_shared(smem_u32(&full[stage]), 0);
          uint8_t* a = sA + stage * bytes_a;
          uint8_t* b = sB + stage * bytes_b;
          if constexpr (MODE == MODE_DQ) {
            tma_load_2d_pair(a, &tmA, lbar, pr * p.S + kc * kBK, mt * kBM);
            for (int j = 0; j < nbh; ++j)
              tma_load_2d_pair(b + j * 8192, tmB, lbar, nt * p.BN + int(rank) * (p.BN / 2) + j * 64,
                               h * p.S + kc * kBK);
          } else {
            for (int j = 0; j < 2; ++j)
              tma_load_2d_pair(a + j * 8192, &tmA, lbar, pr * p.S + mt * kBM + j * 64, kc * kBK);
            for (int j = 0; j < nbh; ++j)
              tma_load_2d_pair(b + j * 8192, &tmB1, lbar,
                               h * p.Dk + half * p.Dh + nt * p.BN + int(rank) * (p.BN / 2) + j * 64,
                               kc * kBK);
          }
          if (++stage == kStagesP) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {  // ---------------- MMA issuer: the leader only
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int u = cl; u < p.tiles; u += ncl) {
        mbar_wait_t<true>(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t dcol = tmem_base + uint32_t(acc * p.BN);
        for (int kc = 0; kc < p.k_chunks; ++kc) {
          mbar_wait_t<true>(&full[stage], phase);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + stage * bytes_a), b0 = smem_u32(sB + stage * bytes_b);
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k) {
            const uint64_t ad = MODE == MODE_DQ ? desc_sw128(a0 + 32 * k, 16, 1024)
                                                : desc_sw128(a0 + 2048 * k, 8192, 1024);
            const uint64_t bd = desc_sw128(b0 + 2048 * k, 8192, 1024);
            umma_f16_pair(dcol, ad, bd, p.idesc, (kc | k) != 0 ? 1u : 0u);
          }
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
  } else if (warp >= 4) {  // ---------------- epilogue (both CTAs): own rows from own TMEM
    const int q4 = warp & 3;
    const float ds_inv =
        p.ds_bound ? ldexpf(1.f, -(ds_f16_exp_ds(p.ds_bound, p.k) + op_f16_exp(p.op_bound))) : 1.f;
    int sbuf = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = cl; u < p.tiles; u += ncl) {
      int pr, mp, nt;
      decode(u, pr, mp, nt);
      const int h = pr >> 1, half = pr & 1;
      const int mt = 2 * mp + int(rank);
      const int row = mt * kBM + q4 * 32 + lane;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      float* dst;
      bool valid;
      if constexpr (MODE == MODE_DQ) {
        valid = row < p.T;
        dst = p.dq + int64_t(row) * p.H * p.Dk + h * p.Dk + half * p.Dh + nt * p.BN;
      } else {
        valid = true;
        dst = (half ? p.dK2 : p.dK1) + (int64_t(h) * p.S + row) * p.Dh + nt * p.BN;
      }
      for (int c0 = 0; c0 < p.BN; c0 += 32) {
        uint32_t r[32];
        tmem_ld32(tmem_base + (uint32_t(q4 * 32) << 16) + uint32_t(acc * p.BN + c0), r);
#pragma unroll
        for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * ds_inv);
        if constexpr (MODE == MODE_DQ) {
          float* stg = stage_all + ((warp - 4) * 2 + (sbuf & 1)) * 1024;
          if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          __syncwarp();
#pragma unroll
          for (int v = 0; v < 8; ++v)
            *reinterpret_cast<uint4*>(stg + lane * 32 + ((v ^ (lane & 7)) << 2)) =
                make_uint4(r[4 * v], r[4 * v + 1], r[4 * v + 2], r[4 * v + 3]);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            asm volatile(
                "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                    reinterpret_cast<uint64_t>(&tmD)),
                "r"(smem_u32(stg)), "r"(h * p.Dk + half * p.Dh + nt * p.BN + c0),
                "r"(mt * kBM + q4 * 32)
                : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
          ++sbuf;
          continue;
        }
        if (valid) {
          float4* d4 = reinterpret_cast<float4*>(dst + c0);
#pragma unroll
          for (int v = 0; v < 8; ++v) {
            float4 x = make_float4(__uint_as_float(r[4 * v]), __uint_as_float(r[4 * v + 1]),
                                   __uint_as_float(r[4 * v + 2]), __uint_as_float(r[4 * v + 3]));
            const float4 o = d4[v];
            x.x += o.x; x.y += o.y; x.z += o.z; x.w += o.w;
            d4[v] = x;
          }
        }
      }
      tc_fence_before();
      if (rank == 0) mbar_arrive(&tempty[acc]);
      else mbar_arrive_remote(mapa_shared(smem_u32(&tempty[acc]), 0));
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
    if (MODE == MODE_DQ && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();                      // both CTAs done before the pair's TMEM is freed
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(p.tmem_cols));
  }
}

// fp16 copies of the bf16 q / key operands.  One pass converts at scale 1
// (exact for |x| in [2^-14, 65504]) and records max|x| (one atomic per
// block); a second launch redoes the conversion at 2^e (ds_f16_exp) only when
// that max leaves [2^-2, 2^14) (overflow risk, or a tensor so small that fp16
// subnormals would cost precision) and otherwise exits at once.  The epilogue
// reads the exponent the copy was made with from op_f16_exp.
__global__ void __launch_bounds__(256) to_f16_pass1_kernel(const __nv_bfloat16* __restrict__ x, int64_t n,
                                                           float* amax, __half* __restrict__ y) {
  float m = 0.f;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  const int64_t t0 = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  const bool vec = ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 15) == 0;
  const int64_t n8 = vec ? n / 8 : 0;
  for (int64_t i = t0; i < n8; i += stride) {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(x) + i);
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
    uint4 o;
    __half2* oh = reinterpret_cast<__half2*>(&o);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 f = __bfloat1622float2(h[j]);
      m = fmaxf(m, fmaxf(fabsf(f.x), fabsf(f.y)));
      oh[j] = __floats2half2_rn(f.x, f.y);
    }
    reinterpret_cast<uint4*>(y)[i] = o;
  }
  for (int64_t i = n8 * 8 + t0; i < n; i += stride) {
    const float f = __bfloat162float(x[i]);
    m = fmaxf(m, fabsf(f));
    y[i] = __float2half_rn(f);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
  __shared__ float s_m[8];
  if ((threadIdx.x & 31) == 0) s_m[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {      // one atomic per block (same-address atomics serialise)
    for (int i = 1; i < 8; ++i) m = fmaxf(m, s_m[i]);
    atomicMax(reinterpret_cast<int*>(amax), __float_as_int(m));   // values >= 0
  }
}

__global__ void __launch_bounds__(256) to_f16_redo_kernel(const __nv_bfloat16* __restrict__ x, int64_t n,
                                                          const float* amax, __half* __restrict__ y) {
  const int e = op_f16_exp(amax);
  if (e == 0) return;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    y[i] = __float2half_rn(ldexpf(__bfloat162float(x[i]), e));
}

int bn_for(int Dh) { return Dh % 256 == 0 ? 256 : (Dh % 128 == 0 ? 128 : 64); }

}  // namespace

bool pkm_bwd_tc_eligible(const mlPkmShape& sh) {
  static int off = -1;
  if (off < 0) {
    const char* e = std::getenv("ML_PKM_BWD_TC");
    off = (e && e[0] == '0') ? 1 : 0;
  }
  const int Dh = sh.Dk / 2;
  return !off && sh.dtype == ML_BF16 && sh.S % 128 == 0 && Dh % 64 == 0 && sh.T > 0;
}

bool pkm_bwd_split(const mlPkmShape& sh) {
  static int on = -1;
  if (on < 0) {
    const char* e = std::getenv("ML_PKM_BWD_SPLIT");
    on = (e && e[0] == '1') ? 1 : 0;
  }
  return on && pkm_bwd_tc_eligible(sh) && softmax_bwd_full_rows(sh);
}

bool pkm_bwd_f16(const mlPkmShape& sh) {
  static int on = -1;
  if (on < 0) {
    const char* e = std::getenv("ML_PKM_BWD_F16");
    on = (e && e[0] == '1') ? 1 : 0;
  }
  return on && !sh.qk_norm && pkm_bwd_tc_eligible(sh) && softmax_bwd_full_rows(sh) && !pkm_bwd_split(sh);
}

static unsigned f16_grid(int64_t n) {
  return unsigned(std::min<int64_t>((n / 8 + 255) / 256 + 1, int64_t(num_sms()) * 8));
}

mlStatus launch_pkm_bwd_f16_keys(const mlPkmShape& sh, const void* K1, const void* K2,
                                 const PkmBwdF16& f, cudaStream_t s) {
  const int64_t nk = int64_t(sh.H) * sh.S * (sh.Dk / 2);
  const auto* k1 = static_cast<const __nv_bfloat16*>(K1);
  const auto* k2 = static_cast<const __nv_bfloat16*>(K2);
  ML_CUDA_TRY(cudaMemsetAsync(f.bound + 2, 0, sizeof(float), s));
  to_f16_pass1_kernel<<<f16_grid(nk), 256, 0, s>>>(k1, nk, f.bound + 2, f.K16);
  ML_LAUNCH_CHECK("pkm_bwd_f16_convert");
  to_f16_pass1_kernel<<<f16_grid(nk), 256, 0, s>>>(k2, nk, f.bound + 2, f.K16 + nk);
  ML_LAUNCH_CHECK("pkm_bwd_f16_convert");
  to_f16_redo_kernel<<<unsigned(num_sms()), 256, 0, s>>>(k1, nk, f.bound + 2, f.K16);
  ML_LAUNCH_CHECK("pkm_bwd_f16_redo");
  to_f16_redo_kernel<<<unsigned(num_sms()), 256, 0, s>>>(k2, nk, f.bound + 2, f.K16 + nk);
  ML_LAUNCH_CHECK("pkm_bwd_f16_redo");
  return ML_OK;
}

mlStatus launch_pkm_bwd_f16_query(const mlPkmShape& sh, const void* q, const PkmBwdF16& f,
                                  cudaStream_t s) {
  const int64_t nq = int64_t(sh.T) * sh.H * sh.Dk;
  const auto* qb = static_cast<const __nv_bfloat16*>(q);
  ML_CUDA_TRY(cudaMemsetAsync(f.bound + 1, 0, sizeof(float), s));
  to_f16_pass1_kernel<<<f16_grid(nq), 256, 0, s>>>(qb, nq, f.bound + 1, f.q16);
  ML_LAUNCH_CHECK("pkm_bwd_f16_convert");
  to_f16_redo_kernel<<<unsigned(num_sms()), 256, 0, s>>>(qb, nq, f.bound + 1, f.q16);
  ML_LAUNCH_CHECK("pkm_bwd_f16_redo");
  return ML_OK;
}

// dq (overwrite) and dK1/dK2 (accumulate) from ds [T, H, 2, S] bf16
// (ds + ds_lo when ds_lo != NULL)
mlStatus launch_pkm_bwd_tc(const mlPkmShape& sh, const __nv_bfloat16* ds, const __nv_bfloat16* ds_lo,
                           const void* q,
                           const void* K1, const void* K2, float* dq, float* dK1, float* dK2,
                           cudaStream_t s, const PkmBwdF16* f16) {
  if (f16 && ds_lo) return fail(ML_ERR_UNSUPPORTED, "pkm_bwd_tc: fp16 operands and the split are exclusive");
  if (f16) {          // the fp16 copies replace the bf16 operands
    q = f16->q16;
    K1 = f16->K16;
    K2 = f16->K16 + int64_t(sh.H) * sh.S * (sh.Dk / 2);
  }
  const int Dh = sh.Dk / 2;
  const int64_t HS2 = int64_t(sh.H) * 2 * sh.S;
  BwdParams p;
  p.T = sh.T; p.H = sh.H; p.S = sh.S; p.Dh = Dh; p.Dk = sh.Dk; p.k = sh.k;
  p.BN = bn_for(Dh);
  p.n_tiles = Dh / p.BN;
  p.tmem_cols = 32;
  while (p.tmem_cols < uint32_t(2 * p.BN)) p.tmem_cols <<= 1;
  p.dq = dq; p.dK1 = dK1; p.dK2 = dK2;
  p.ds_bound = f16 ? f16->bound : nullptr;
  p.op_bound = nullptr;
  // A (atype, bits 7-9) and B (btype, bits 10-12): both bf16 (1) or both fp16 (0)
  const uint32_t atype = f16 ? 0u : ((1u << 7) | (1u << 10));
  p.split = ds_lo ? 1 : 0;
  p.stages = ds_lo ? 3 : kStagesB;
  const uint32_t base_idesc = (1u << 4) | atype | (uint32_t(p.BN >> 3) << 17) |
                              (uint32_t(kBM >> 4) << 24);
  const size_t smem = 1024 + size_t(p.stages) * ((kBM * kBK * 2 << p.split) + size_t(p.BN) * kBK * 2) + 1024 +
                      size_t(4) * 2 * 1024 * sizeof(float);
  static size_t configured[2] = {0, 0};
  const int grid_max = num_sms();
  // CTA pairs (cta_group::2): 256-column n-tiles, whole 256-row key pairs for dK
  static const bool pair_env = [] {
    const char* e = std::getenv("ML_PKM_BWD_PAIR");
    return !(e && e[0] == '0');
  }();
  if (pair_env && !ds_lo && p.BN == 256 && sh.S % 256 == 0) {
    const size_t smem2 = 1024 + size_t(kStagesP) * (kBM * kBK * 2 + size_t(p.BN / 2) * kBK * 2) + 1024 +
                         size_t(4) * 2 * 1024 * sizeof(float);
    static bool attr2 = false;
    if (!attr2) {
      ML_CUDA_TRY(cudaFuncSetAttribute(pkm_bwd_tc2_kernel<MODE_DQ>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem2)));
      ML_CUDA_TRY(cudaFuncSetAttribute(pkm_bwd_tc2_kernel<MODE_DK>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem2)));
      attr2 = true;
    }
    const uint32_t idesc2 = (1u << 4) | atype | (uint32_t(p.BN >> 3) << 17) |
                            (uint32_t(256 >> 4) << 24);
    const int ncl_max = grid_max / 2;
    {   // dq
      CUtensorMap ma, mb1, mb2, md;
      ML_TRY(make_map(&ma, ds, uint64_t(HS2), uint64_t(sh.T), uint64_t(HS2) * 2, kBK, kBM));
      ML_TRY(make_map(&mb1, K1, uint64_t(Dh), uint64_t(sh.H) * sh.S, uint64_t(Dh) * 2, 64, kBK));
      ML_TRY(make_map(&mb2, K2, uint64_t(Dh), uint64_t(sh.H) * sh.S, uint64_t(Dh) * 2, 64, kBK));
      EncodeFn f = encode_fn();
      if (!f) return fail(ML_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
      cuuint64_t dims[2] = {uint64_t(sh.H) * sh.Dk, uint64_t(sh.T)};
      cuuint64_t strides[1] = {uint64_t(sh.H) * sh.Dk * 4};
      cuuint32_t box[2] = {32, 32};
      cuuint32_t estr[2] = {1, 1};
      CUresult r = f(&md, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dq, dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) return fail(ML_ERR_CUDA, "cuTensorMapEncodeTiled (dq) failed: " + std::to_string(int(r)));
      BwdParams pq = p;
      pq.m_tiles = ((sh.T + kBM - 1) / kBM + 1) / 2;      // 128-row m-tile PAIRS
      pq.k_chunks = sh.S / kBK;
      pq.tiles = sh.H * 2 * pq.m_tiles * pq.n_tiles;
      pq.idesc = idesc2 | (1u << 16);
      if (f16) pq.op_bound = f16->bound + 2;
      const int ncl = std::min(pq.tiles, ncl_max);
      if (f16 && f16->keys_ready) ML_CUDA_TRY(cudaStreamWaitEvent(s, f16->keys_ready, 0));
      pkm_bwd_tc2_kernel<MODE_DQ><<<2 * ncl, kThreadsB, smem2, s>>>(ma, mb1, mb2, md, pq);
      ML_LAUNCH_CHECK("pkm_dq_tc");
    }
    {   // dK
      CUtensorMap ma, mb;
      ML_TRY(make_map(&ma, ds, uint64_t(HS2), uint64_t(sh.T), uint64_t(HS2) * 2, 64, kBK));
      ML_TRY(make_map(&mb, q, uint64_t(sh.H) * sh.Dk, uint64_t(sh.T), uint64_t(sh.H) * sh.Dk * 2, 64, kBK));
      BwdParams pk = p;
      pk.m_tiles = sh.S / 256;                             // 256-key pairs
      pk.k_chunks = (sh.T + kBK - 1) / kBK;
      pk.tiles = sh.H * 2 * pk.m_tiles * pk.n_tiles;
      pk.idesc = idesc2 | (1u << 15) | (1u << 16);
      if (f16) pk.op_bound = f16->bound + 1;
      const int ncl = std::min(pk.tiles, ncl_max);
      if (f16 && f16->q16_ready) ML_CUDA_TRY(cudaStreamWaitEvent(s, f16->q16_ready, 0));
      pkm_bwd_tc2_kernel<MODE_DK><<<2 * ncl, kThreadsB, smem2, s>>>(ma, mb, mb, mb, pk);
      ML_LAUNCH_CHECK("pkm_dK_tc");
    }
    return ML_OK;
  }
  // ---- dq = ds K: A K-major (ds rows), B MN-major (key table)
  {
    CUtensorMap ma, mb1, mb2, mlo;
    ML_TRY(make_map(&ma, ds, uint64_t(HS2), uint64_t(sh.T), uint64_t(HS2) * 2, kBK, kBM));
    mlo = ma;
    if (ds_lo) ML_TRY(make_map(&mlo, ds_lo, uint64_t(HS2), uint64_t(sh.T), uint64_t(HS2) * 2, kBK, kBM));
    ML_TRY(make_map(&mb1, K1, uint64_t(Dh), uint64_t(sh.H) * sh.S, uint64_t(Dh) * 2, 64, kBK));
    ML_TRY(make_map(&mb2, K2, uint64_t(Dh), uint64_t(sh.H) * sh.S, uint64_t(Dh) * 2, 64, kBK));
    BwdParams pq = p;
    pq.m_tiles = (sh.T + kBM - 1) / kBM;
    pq.k_chunks = sh.S / kBK;
    pq.tiles = sh.H * 2 * pq.m_tiles * pq.n_tiles;
    pq.idesc = base_idesc | (1u << 16);          // B MN-major
    if (f16) pq.op_bound = f16->bound + 2;
    if (smem > configured[0]) {
      ML_CUDA_TRY(cudaFuncSetAttribute(pkm_bwd_tc_kernel<MODE_DQ>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
      configured[0] = smem;
    }
    CUtensorMap md;   // dq [T][H*Dk] fp32, 32 x 32 boxes, 128-byte swizzle
    {
      EncodeFn f = encode_fn();
      if (!f) return fail(ML_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
      cuuint64_t dims[2] = {uint64_t(sh.H) * sh.Dk, uint64_t(sh.T)};
      cuuint64_t strides[1] = {uint64_t(sh.H) * sh.Dk * 4};
      cuuint32_t box[2] = {32, 32};
      cuuint32_t estr[2] = {1, 1};
      CUresult r = f(&md, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dq, dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) return fail(ML_ERR_CUDA, "cuTensorMapEncodeTiled (dq) failed: " + std::to_string(int(r)));
    }
    if (f16 && f16->keys_ready) ML_CUDA_TRY(cudaStreamWaitEvent(s, f16->keys_ready, 0));
    pkm_bwd_tc_kernel<MODE_DQ><<<std::min(pq.tiles, grid_max), kThreadsB, smem, s>>>(ma, mb1, mb2, md, mlo, pq);
    ML_LAUNCH_CHECK("pkm_dq_tc");
  }
  // ---- dK += ds^T q: A MN-major (ds, keys along M), B MN-major (q)
  {
    CUtensorMap ma, mb, mlo;
    ML_TRY(make_map(&ma, ds, uint64_t(HS2), uint64_t(sh.T), uint64_t(HS2) * 2, 64, kBK));
    mlo = ma;
    if (ds_lo) ML_TRY(make_map(&mlo, ds_lo, uint64_t(HS2), uint64_t(sh.T), uint64_t(HS2) * 2, 64, kBK));
    ML_TRY(make_map(&mb, q, uint64_t(sh.H) * sh.Dk, uint64_t(sh.T), uint64_t(sh.H) * sh.Dk * 2, 64, kBK));
    BwdParams pk = p;
    pk.m_tiles = sh.S / kBM;
    pk.k_chunks = (sh.T + kBK - 1) / kBK;
    pk.tiles = sh.H * 2 * pk.m_tiles * pk.n_tiles;
    pk.idesc = base_idesc | (1u << 15) | (1u << 16);   // A and B MN-major
    if (f16) pk.op_bound = f16->bound + 1;
    if (smem > configured[1]) {
      ML_CUDA_TRY(cudaFuncSetAttribute(pkm_bwd_tc_kernel<MODE_DK>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
      configured[1] = smem;
    }
    if (f16 && f16->q16_ready) ML_CUDA_TRY(cudaStreamWaitEvent(s, f16->q16_ready, 0));
    pkm_bwd_tc_kernel<MODE_DK><<<std::min(pk.tiles, grid_max), kThreadsB, smem, s>>>(ma, mb, mb, mb, mlo, pk);
    ML_LAUNCH_CHECK("pkm_dK_tc");
  }
  return ML_OK;
}

}  // namespace ml
