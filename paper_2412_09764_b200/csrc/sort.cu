// Device-wide scan, stable LSD radix sort of (key, position) pairs and run
// detection: the "preprocessing to inverse the token_id to embedding_id
// mapping, so that each row in the embedding gradient can know which token
// will contribute to it" of the "reverse_indices" backward (§3.1.4,
// P:176).  Stability keeps positions ascending inside each run, which fixes
// the summation order of every gradient row (determinism).
//
// Sort design: 4096 keys per CTA (8 warps x 16 rounds x 32); each warp ranks
// its 512 keys with __match_any_sync and warp-private digit counters, the
// CTA combines warps in order, a device-wide exclusive scan over the
// digit-major [digit][block] count matrix gives every (digit, block) its
// output offset; the scatter stages the block's pairs in digit order in
// shared memory and writes each digit run contiguously.  Digits are <= 11
// bits; passes = ceil(bits / 11) (2 for a 2^20-row table).
#include "internal.cuh"

#include <algorithm>
#include <cstdlib>

namespace ml {
namespace {

constexpr int kScanThreads = 512;
constexpr int kScanItems = 4;
constexpr int kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ int block_excl_scan(int v, int* s_warp, int* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[wid] = x;
  __syncthreads();
  if (wid == 0) {
    const int nw = blockDim.x >> 5;
    int t = lane < nw ? s_warp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    if (lane < nw) s_warp[lane] = t;
  }
  __syncthreads();
  const int warp_off = wid ? s_warp[wid - 1] : 0;
  *total = s_warp[(blockDim.x >> 5) - 1];
  __syncthreads();
  return warp_off + x - v;
}

__global__ void __launch_bounds__(kScanThreads) scan_reduce_kernel(const int32_t* in, int64_t n,
                                                                   int32_t* tmp) {
  __shared__ int s_warp[32];
  const int64_t base = int64_t(blockIdx.x) * kScanTile + threadIdx.x * kScanItems;
  int sum = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i)
    if (base + i < n) sum += in[base + i];
  int total;
  block_excl_scan(sum, s_warp, &total);
  if (threadIdx.x == 0) tmp[blockIdx.x] = total;
}

// Single CTA: exclusive scan of the nb block sums, in place; total -> *total.
__global__ void __launch_bounds__(1024) scan_blocks_kernel(int32_t* tmp, int64_t nb,
                                                           int32_t* total) {
  __shared__ int s_warp[32];
  int carry = 0;
  for (int64_t c0 = 0; c0 < nb; c0 += 1024 * 4) {
    const int64_t base = c0 + threadIdx.x * 4;
    int v[4], sum = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      v[i] = (base + i < nb) ? tmp[base + i] : 0;
      sum += v[i];
    }
    int tot;
    int ex = block_excl_scan(sum, s_warp, &tot) + carry;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (base + i < nb) tmp[base + i] = ex;
      ex += v[i];
    }
    carry += tot;
  }
  if (threadIdx.x == 0 && total) *total = carry;
}

__global__ void __launch_bounds__(kScanThreads) scan_down_kernel(const int32_t* in, int32_t* out,
                                                                 int64_t n, const int32_t* tmp) {
  __shared__ int s_warp[32];
  const int64_t base = int64_t(blockIdx.x) * kScanTile + threadIdx.x * kScanItems;
  int v[kScanItems], sum = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    v[i] = (base + i < n) ? in[base + i] : 0;
    sum += v[i];
  }
  int total;
  int ex = block_excl_scan(sum, s_warp, &total) + tmp[blockIdx.x];
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    if (base + i < n) out[base + i] = ex;
    ex += v[i];
  }
}

// ------------------------------------------------------------ radix sort
constexpr int kSortWarps = 8;
#ifndef ML_SORT_ROUNDS
#define ML_SORT_ROUNDS 16
#endif
constexpr int kSortRounds = ML_SORT_ROUNDS;   // keys per thread per tile (A/B: -DML_SORT_ROUNDS)
constexpr int kSortTile = kSortWarps * kSortRounds * 32;  // 4096
constexpr int kMaxDigitBits = 11;

struct SortPassParams {
  const int32_t* kin; const int32_t* vin;  // vin == nullptr -> value = position
  int32_t* kout; int32_t* vout;
  int64_t n; int nblocks; int shift; int dbits; uint32_t key_limit;
  int32_t* counts;  // [nbins][nblocks]; scanned in place between the kernels
  int* flag;
  // single-pass ("onesweep") mode: per-(tile, digit) status words published
  // and looked back over, global digit offsets of this pass, a tile ticket
  uint32_t* status; const int32_t* goff; int32_t* tile_ctr;
};

constexpr uint32_t kStAgg = 1u << 30;     // tile's own count available
constexpr uint32_t kStInc = 2u << 30;     // inclusive prefix available
constexpr uint32_t kStMask = (1u << 30) - 1;
constexpr uint32_t kSortSpin = 1u << 26;

// First pass: a key outside [0, key_limit) (an index outside [0, N)) is
// sorted as row 0 and its position value carries kClampedPos, so the
// segmented pass gives it weight 0 (memlayer.h: "clamped to row 0 with
// weight 0"); the index flag is raised for ML_CHECK_INDICES.
__device__ __forceinline__ int32_t load_key(const SortPassParams& p, int64_t i, bool first,
                                            bool* clamped = nullptr) {
  int32_t k = p.kin[i];
  if (first && static_cast<uint32_t>(k) >= p.key_limit) {
    atomicExch(p.flag, 1);
    k = 0;
    if (clamped) *clamped = true;
  }
  return k;
}

// dynamic smem: s_cnt[kSortWarps][nbins]
__global__ void __launch_bounds__(256) sort_hist_kernel(SortPassParams p, bool first) {
  extern __shared__ int s_dyn[];
  const int nbins = 1 << p.dbits;
  int* s_cnt = s_dyn;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int d = threadIdx.x; d < kSortWarps * nbins; d += 256) s_cnt[d] = 0;
  __syncthreads();
  const int64_t wbase = int64_t(blockIdx.x) * kSortTile + int64_t(wid) * kSortRounds * 32;
  const uint32_t mask = uint32_t(nbins - 1);
  int32_t key[kSortRounds];
#pragma unroll
  for (int r = 0; r < kSortRounds; ++r) {       // all loads first
    const int64_t i = wbase + r * 32 + lane;
    key[r] = i < p.n ? load_key(p, i, first) : 0;
  }
#pragma unroll
  for (int r = 0; r < kSortRounds; ++r) {
    const int64_t i = wbase + r * 32 + lane;
    const bool valid = i < p.n;
    const uint32_t dig = valid ? ((uint32_t(key[r]) >> p.shift) & mask) : 0x10000u;
    const unsigned peers = __match_any_sync(0xffffffffu, dig);
    if (valid && lane == __ffs(peers) - 1) s_cnt[wid * nbins + dig] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  for (int d = threadIdx.x; d < nbins; d += 256) {
    int t = 0;
#pragma unroll
    for (int w = 0; w < kSortWarps; ++w) t += s_cnt[w * nbins + d];
    p.counts[int64_t(d) * p.nblocks + blockIdx.x] = t;
  }
}

// Stable scatter of one pass.  Each warp ranks its 512 keys (match_any), the
// block places all 4096 (key, value) pairs in digit order in shared memory,
// then writes every digit's run contiguously (coalesced) at its global offset.
// dynamic smem: s_cnt[kSortWarps][nbins], s_dstart[nbins], s_goff[nbins],
//               s_key[kSortTile], s_val[kSortTile]
// ML_SORT_MINB (build switch): blocks per SM of the scatter kernel; 3 spills
// (80 registers) and measured 163 vs 143 us per 2-pass C2 sort
#ifndef ML_SORT_MINB
#define ML_SORT_MINB 2
#endif
// (A variant writing each key straight to its global slot, without the
// shared-memory staging, measured 155 vs 144 us per 2-pass sort of 2.1M keys.)
template <bool ONESWEEP, int ROUNDS = kSortRounds>
__global__ void __launch_bounds__(256, ML_SORT_MINB) sort_scatter_kernel(SortPassParams p, bool first) {
  constexpr int TILE = kSortWarps * ROUNDS * 32;
  extern __shared__ int s_dyn[];
  const int nbins = 1 << p.dbits;
  int* s_cnt = s_dyn;
  int* s_dstart = s_cnt + kSortWarps * nbins;
  int* s_goff = s_dstart + nbins;
  int32_t* s_key = s_goff + nbins;
  int32_t* s_val = s_key + TILE;
  __shared__ int s_warp[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t mask = uint32_t(nbins - 1);
  __shared__ int s_tile;
  for (int d = threadIdx.x; d < kSortWarps * nbins; d += 256) s_cnt[d] = 0;
  if constexpr (ONESWEEP) {   // tiles in ticket order: every predecessor is resident or done
    if (threadIdx.x == 0) s_tile = atomicAdd(p.tile_ctr, 1);
  }
  __syncthreads();
  const int tile = ONESWEEP ? s_tile : int(blockIdx.x);
  const int64_t bbase = int64_t(tile) * TILE;
  const int64_t wbase = bbase + int64_t(wid) * ROUNDS * 32;
  const int nvalid = int(p.n - bbase < TILE ? p.n - bbase : TILE);
  int32_t key[ROUNDS], val[ROUNDS];
  uint32_t dig[ROUNDS];
  unsigned peers[ROUNDS];
#pragma unroll
  for (int r = 0; r < ROUNDS; ++r) {
    const int64_t i = wbase + r * 32 + lane;
    const bool valid = i < p.n;
    bool clamped = false;
    key[r] = valid ? load_key(p, i, first, &clamped) : 0;
    val[r] = valid ? (p.vin ? p.vin[i] : (int32_t(i) | (clamped ? kClampedPos : 0))) : 0;
  }
#pragma unroll
  for (int r = 0; r < ROUNDS; ++r) {
    const int64_t i = wbase + r * 32 + lane;
    const bool valid = i < p.n;
    dig[r] = valid ? ((uint32_t(key[r]) >> p.shift) & mask) : 0x10000u;
    peers[r] = __match_any_sync(0xffffffffu, dig[r]);
    if (valid && lane == __ffs(peers[r]) - 1) s_cnt[wid * nbins + dig[r]] += __popc(peers[r]);
    __syncwarp();
  }
  __syncthreads();
  // block-local digit starts (exclusive scan of the block's digit totals),
  // per-(warp, digit) local offsets, global offsets of the block's digit runs
  const int per = nbins / 256 > 0 ? nbins / 256 : 1;   // digits per thread (nbins >= 256 or 1 each)
  int tot_local[8];
  int sum = 0;
  for (int j = 0; j < per; ++j) {
    const int d = threadIdx.x * per + j;
    int t = 0;
    if (d < nbins) {
      for (int w = 0; w < kSortWarps; ++w) t += s_cnt[w * nbins + d];
    }
    tot_local[j] = t;
    sum += t;
  }
  int total;
  int ex = block_excl_scan(sum, s_warp, &total);
  if constexpr (ONESWEEP) {
    // publish this tile's digit counts, then look back over the predecessors
    // (decoupled look-back) for the exclusive prefix of every digit
    for (int j = 0; j < per; ++j) {
      const int d = threadIdx.x * per + j;
      if (d < nbins) {
        volatile uint32_t* st = p.status + int64_t(tile) * nbins + d;
        *st = (tile == 0 ? kStInc : kStAgg) | uint32_t(tot_local[j]);
      }
    }
    __threadfence();
    // all of this thread's digits walk back together: one round of independent
    // status loads per predecessor tile, until every digit found an inclusive
    // prefix (tile 0 publishes inclusive values)
    // kLB predecessors per digit per round of loads (all independent), so a
    // walk over aggregate-only predecessors takes 1/kLB of the round trips
    constexpr int kLB = 4;
    uint32_t excl[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    int ptj[8];
    uint32_t open = 0;
    for (int j = 0; j < 8; ++j) {
      ptj[j] = tile - 1;
      if (j < per && threadIdx.x * per + j < nbins && tile > 0) open |= 1u << j;
    }
    uint32_t spins = 0;
    const volatile uint32_t* stp = p.status;
    while (open) {
      uint32_t v[8][kLB];
#pragma unroll
      for (int j = 0; j < 8; ++j)
#pragma unroll
        for (int q = 0; q < kLB; ++q) {
          v[j][q] = 2u << 30;    // before tile 0: an inclusive prefix of 0
          if ((open >> j & 1u) && ptj[j] - q >= 0)
            v[j][q] = stp[int64_t(ptj[j] - q) * nbins + threadIdx.x * per + j];
        }
      bool progress = false;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (!(open >> j & 1u)) continue;
#pragma unroll
        for (int q = 0; q < kLB; ++q) {
          const uint32_t f = v[j][q] >> 30;
          if (f == 0) break;                 // not published yet: retry from here
          excl[j] += v[j][q] & kStMask;
          --ptj[j];
          progress = true;
          if (f == 2) {
            open &= ~(1u << j);
            break;
          }
        }
      }
      if (!progress && ++spins > kSortSpin) __trap();
    }
    for (int j = 0; j < per; ++j) {
      const int d = threadIdx.x * per + j;
      if (d >= nbins) continue;
      if (tile > 0) {
        volatile uint32_t* st = p.status + int64_t(tile) * nbins + d;
        *st = kStInc | (excl[j] + uint32_t(tot_local[j]));
      }
      s_goff[d] = p.goff[d] + int(excl[j]);
    }
  }
  for (int j = 0; j < per; ++j) {
    const int d = threadIdx.x * per + j;
    if (d < nbins) {
      s_dstart[d] = ex;
      if constexpr (!ONESWEEP) s_goff[d] = p.counts[int64_t(d) * p.nblocks + blockIdx.x];
      int run = ex;
      for (int w = 0; w < kSortWarps; ++w) {
        const int c = s_cnt[w * nbins + d];
        s_cnt[w * nbins + d] = run;
        run += c;
      }
    }
    ex += tot_local[j];
  }
  __syncthreads();
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll
  for (int r = 0; r < ROUNDS; ++r) {
    const int64_t i = wbase + r * 32 + lane;
    const bool valid = i < p.n;
    int dst = 0;
    if (valid) dst = s_cnt[wid * nbins + dig[r]] + __popc(peers[r] & lt);
    __syncwarp();
    if (valid && lane == __ffs(peers[r]) - 1) s_cnt[wid * nbins + dig[r]] += __popc(peers[r]);
    __syncwarp();
    if (valid) {
      s_key[dst] = key[r];
      s_val[dst] = val[r];
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < nvalid; e += 256) {
    const int32_t k = s_key[e];
    const int d = int((uint32_t(k) >> p.shift) & mask);
    const int64_t g = int64_t(s_goff[d]) + (e - s_dstart[d]);
    p.kout[g] = k;
    p.vout[g] = s_val[e];
  }
}

// ---- single-pass sort support: one read of the keys builds the global digit
// histograms of every pass; one CTA turns them into per-pass digit offsets.
// ghist: [passes][nbins] counts -> exclusive offsets; ghist[passes*nbins + pass]
// are the tile tickets (zeroed here).
__global__ void __launch_bounds__(256) sort_ghist_kernel(const int32_t* keys, int64_t n,
                                                         uint32_t key_limit, int passes,
                                                         int dbits, int32_t* ghist, int* flag) {
  extern __shared__ int s_h[];   // [passes][nbins]
  const int nbins = 1 << dbits;
  for (int i = threadIdx.x; i < passes * nbins; i += blockDim.x) s_h[i] = 0;
  __syncthreads();
  const uint32_t mask = uint32_t(nbins - 1);
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    uint32_t k = uint32_t(keys[i]);
    if (k >= key_limit) {
      atomicExch(flag, 1);
      k = 0;
    }
    for (int ps = 0; ps < passes; ++ps) atomicAdd(&s_h[ps * nbins + ((k >> (ps * dbits)) & mask)], 1);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < passes * nbins; i += blockDim.x)
    if (s_h[i]) atomicAdd(&ghist[i], s_h[i]);
}

__global__ void __launch_bounds__(1024) sort_gscan_kernel(int32_t* ghist, int passes, int nbins) {
  __shared__ int s_warp[32];
  for (int ps = 0; ps < passes; ++ps) {
    int32_t* h = ghist + ps * nbins;
    const int per = (nbins + 1023) / 1024;
    int v[2] = {0, 0}, sum = 0;
    for (int j = 0; j < per; ++j) {
      const int d = threadIdx.x * per + j;
      v[j] = d < nbins ? h[d] : 0;
      sum += v[j];
    }
    int tot;
    int ex = block_excl_scan(sum, s_warp, &tot);
    for (int j = 0; j < per; ++j) {
      const int d = threadIdx.x * per + j;
      if (d < nbins) h[d] = ex;
      ex += v[j];
    }
    __syncthreads();
  }
  if (threadIdx.x < passes) ghist[passes * nbins + threadIdx.x] = 0;
}

// ------------------------------------------------------------ runs
// Two single-pass kernels (tiles of kScanTile, ticket order, decoupled
// look-back over one status word per tile); every array is read and written
// coalesced (tiles staged in shared memory, scanned blocked).
__device__ __forceinline__ uint32_t lookback_prefix(uint32_t* status, int tile, uint32_t total) {
  // thread 0 of the tile: publish, walk back, publish the inclusive prefix
  volatile uint32_t* st = status;
  st[tile] = (tile == 0 ? kStInc : kStAgg) | total;
  __threadfence();
  uint32_t excl = 0, spins = 0;
  for (int pt = tile - 1; pt >= 0;) {
    const uint32_t v = st[pt];
    if ((v >> 30) == 0) {
      if (++spins > kSortSpin) __trap();
      continue;
    }
    excl += v & kStMask;
    if ((v >> 30) == 2) break;
    --pt;
  }
  if (tile > 0) st[tile] = kStInc | (excl + total);
  return excl;
}

// Warp 0 of the tile: publish the tile's count, then walk back 32
// predecessors at a time (one status word per lane, the nearest one with an
// inclusive prefix ends the walk), publish the inclusive prefix.
constexpr int kRunItems = 4;
constexpr int kRunTile = kScanThreads * kRunItems;   // 2048 positions per tile
__device__ __forceinline__ uint32_t lookback_prefix_warp(uint64_t* status, int tile, uint32_t total,
                                                         int lane) {
  // 64-bit status words: flag in bits 62-63 (1 = aggregate, 2 = inclusive),
  // the count below (any n < 2^31)
  constexpr uint64_t kAgg = uint64_t(1) << 62, kInc = uint64_t(2) << 62;
  constexpr uint64_t kMask = kAgg - 1;
  volatile uint64_t* st = status;
  if (lane == 0) {
    st[tile] = (tile == 0 ? kInc : kAgg) | total;
    __threadfence();
  }
  __syncwarp();
  uint64_t excl = 0;
  for (int pt = tile - 1; pt >= 0; pt -= 32) {
    const int idx = pt - lane;
    uint64_t v = kInc;              // before tile 0: an inclusive prefix of 0
    if (idx >= 0) v = st[idx];
    uint32_t spins = 0;
    while ((v >> 62) == 0) {
      if (++spins > kSortSpin) __trap();
      v = st[idx];
    }
    const unsigned inc = __ballot_sync(0xffffffffu, (v >> 62) == 2);
    const int lim = inc ? __ffs(inc) - 1 : 31;     // lanes 0..lim contribute
    uint64_t c = lane <= lim ? (v & kMask) : 0u;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    excl += c;
    if (inc) break;
  }
  if (lane == 0 && tile > 0) st[tile] = kInc | (excl + total);
  return uint32_t(excl);
}

// run id of every position (rid), run_begin, rows (the distinct keys), *U
__global__ void __launch_bounds__(kScanThreads) run_scan1_kernel(const int32_t* skey, int64_t n,
                                                                 int32_t* rid, int32_t* run_begin,
                                                                 int32_t* rows_out, int32_t* U,
                                                                 uint64_t* status, int32_t* ticket) {
  __shared__ int s_warp[32];
  __shared__ int s_tile;
  __shared__ uint32_t s_prefix;
  __shared__ int32_t s_k[kRunTile + 1];   // s_k[0]: the key before the tile
  __shared__ int32_t s_r[kRunTile];
  __shared__ int32_t s_w[kRunTile];
  if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1);
  __syncthreads();
  const int tile = s_tile;
  const int64_t t0 = int64_t(tile) * kRunTile;
  for (int x = threadIdx.x; x < kRunTile; x += kScanThreads)
    s_k[1 + x] = t0 + x < n ? skey[t0 + x] : 0;
  if (threadIdx.x == 0) s_k[0] = tile > 0 ? skey[t0 - 1] : 0;
  __syncthreads();
  const int x0 = threadIdx.x * kRunItems;
  int f[kRunItems], sum = 0;
#pragma unroll
  for (int i = 0; i < kRunItems; ++i) {
    const int64_t ix = t0 + x0 + i;
    f[i] = (ix < n && (ix == 0 || s_k[1 + x0 + i] != s_k[x0 + i])) ? 1 : 0;
    sum += f[i];
  }
  int total;
  const int ex = block_excl_scan(sum, s_warp, &total);
  if (threadIdx.x < 32) {
    const uint32_t pre = lookback_prefix_warp(status, tile, uint32_t(total), threadIdx.x);
    if (threadIdx.x == 0) s_prefix = pre;
  }
  __syncthreads();
  const int pre = int(s_prefix);
  int e = pre + ex;
#pragma unroll
  for (int i = 0; i < kRunItems; ++i) {
    e += f[i];
    s_r[x0 + i] = e - 1;
  }
  __syncthreads();
  for (int x = threadIdx.x; x < kRunTile; x += kScanThreads)
    if (t0 + x < n) rid[t0 + x] = s_r[x];
  __syncthreads();
  // the tile's runs have the contiguous ids [pre, pre + total): stage their
  // first positions and keys, then store both coalesced
  e = ex;
#pragma unroll
  for (int i = 0; i < kRunItems; ++i) {
    if (f[i]) {
      s_r[e] = int32_t(t0 + x0 + i);
      s_w[e] = s_k[1 + x0 + i];
    }
    e += f[i];
  }
  __syncthreads();
  for (int x = threadIdx.x; x < total; x += kScanThreads) {
    run_begin[pre + x] = s_r[x];
    if (rows_out) rows_out[pre + x] = s_w[x];
  }
  if (t0 + kRunTile >= n && threadIdx.x == 0) {   // the last tile
    run_begin[pre + total] = int32_t(n);
    *U = pre + total;
  }
}

// pieces of the runs longer than kPieceLen: their exclusive scan over runs,
// written at each long run's first position (piece_base), and n_slots
__global__ void __launch_bounds__(kScanThreads) run_scan2_kernel(const int32_t* run_begin,
                                                                 const int32_t* U, int32_t* piece_base,
                                                                 int32_t* n_slots, int ntiles,
                                                                 uint64_t* status, int32_t* ticket) {
  __shared__ int s_warp[32];
  __shared__ int s_tile;
  __shared__ uint32_t s_prefix;
  __shared__ int32_t s_b[kRunTile + 1];
  if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1);
  __syncthreads();
  const int tile = s_tile;
  const int64_t r0 = int64_t(tile) * kRunTile;
  const int64_t u = *U;
  for (int x = threadIdx.x; x <= kRunTile; x += kScanThreads)
    s_b[x] = r0 + x <= u ? run_begin[r0 + x] : 0;
  __syncthreads();
  const int x0 = threadIdx.x * kRunItems;
  int np[kRunItems], sum = 0;
#pragma unroll
  for (int i = 0; i < kRunItems; ++i) {
    np[i] = 0;
    if (r0 + x0 + i < u) {
      const int32_t len = s_b[x0 + i + 1] - s_b[x0 + i];
      np[i] = len > kPieceLen ? (len + kPieceLen - 1) / kPieceLen : 0;
    }
    sum += np[i];
  }
  int total;
  const int ex = block_excl_scan(sum, s_warp, &total);
  if (threadIdx.x < 32) {
    const uint32_t pre = lookback_prefix_warp(status, tile, uint32_t(total), threadIdx.x);
    if (threadIdx.x == 0) s_prefix = pre;
  }
  __syncthreads();
  int e = int(s_prefix) + ex;
#pragma unroll
  for (int i = 0; i < kRunItems; ++i) {
    if (np[i]) piece_base[s_b[x0 + i]] = e;
    e += np[i];
  }
  if (tile == ntiles - 1 && threadIdx.x == kScanThreads - 1 && n_slots) *n_slots = e;
}

// ---------------------------------------------------------------- counting sort
// For a key range no larger than twice the key count (the value-row sort of a
// step with at least N/2 positions, e.g. C2: 2.1M positions over 2^20 rows):
// one histogram, one scan and one atomic-cursor scatter place every pair in
// its run; the scatter order inside a run is arbitrary, so each run's
// positions are then sorted ascending -- exactly the order the stable radix
// sort produces (the values of a run are distinct positions).  Clamped keys
// are handled as in load_key.  Run lengths: <= kFixShort by one thread,
// longer runs by one CTA (shared-memory bitonic chunks + merge passes).
constexpr int kFixShort = 32;
constexpr int kFixMed = 256;       // runs of 33..256 positions: one warp each
constexpr int kFixSmem = 8192;
constexpr uint32_t kPosMask = 0x7fffffffu;   // strips kClampedPos for ordering

__global__ void __launch_bounds__(256) csort_hist_kernel(const int32_t* __restrict__ keys, int64_t n,
                                                         uint32_t limit, int32_t* __restrict__ cnt,
                                                         int* flag) {
  // warp-aggregated: one atomic per distinct key of a warp's 32 keys (a
  // key shared by many positions -- the sparse key backward's sentinel --
  // would otherwise serialise on one counter)
  const int lane = threadIdx.x & 31;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t b0 = blockIdx.x * int64_t(blockDim.x) + (threadIdx.x & ~31); b0 < n; b0 += stride) {
    const int64_t i = b0 + lane;
    uint32_t k = 0xFFFFFFE0u | uint32_t(lane);    // distinct per lane when i >= n
    if (i < n) {
      k = uint32_t(keys[i]);
      if (k >= limit) {
        atomicExch(flag, 1);
        k = 0;
      }
    }
    const unsigned peers = __match_any_sync(0xffffffffu, k);
    if (i < n && lane == __ffs(peers) - 1) atomicAdd(cnt + k, __popc(peers));
  }
}

// cur: exclusive run offsets on entry, run ends on exit; uid (nullable):
// run id of every row, written to rid per position
__global__ void __launch_bounds__(256) csort_scatter_kernel(const int32_t* __restrict__ keys, int64_t n,
                                                            uint32_t limit, int32_t* __restrict__ cur,
                                                            int32_t* __restrict__ kout,
                                                            int32_t* __restrict__ vout,
                                                            const int32_t* __restrict__ uid,
                                                            int32_t* __restrict__ rid) {
  const int lane = threadIdx.x & 31;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t b0 = blockIdx.x * int64_t(blockDim.x) + (threadIdx.x & ~31); b0 < n; b0 += stride) {
    const int64_t i = b0 + lane;
    uint32_t k = 0xFFFFFFE0u | uint32_t(lane);    // distinct per lane when i >= n
    bool clamped = false;
    if (i < n) {
      k = uint32_t(keys[i]);
      clamped = k >= limit;
      if (clamped) k = 0;
    }
    // warp-aggregated cursor: the group's leader reserves popc slots, lanes
    // take them in lane (= position) order
    const unsigned peers = __match_any_sync(0xffffffffu, k);
    const int leader = __ffs(peers) - 1;
    int32_t o0 = 0;
    if (i < n && lane == leader) o0 = atomicAdd(cur + k, __popc(peers));
    o0 = __shfl_sync(0xffffffffu, o0, leader);
    if (i < n) {
      const int32_t o = o0 + __popc(peers & ((1u << lane) - 1u));
      kout[o] = int32_t(k);
      vout[o] = int32_t(i) | (clamped ? kClampedPos : 0);
      if (uid) rid[o] = uid[k];
    }
  }
}

// The runs of the counting sort straight from the per-row counts (replaces
// find_runs' two passes over the sorted positions): one scan over the N rows
// of (count, row touched, pieces of a run longer than kPieceLen) gives every
// touched row its first position, run id and piece base.  tmp: [3][nt + 1].
__device__ __forceinline__ void row_triple(const int32_t* cnt, int64_t N, int64_t r, int& c, int& u, int& pc) {
  c = r < N ? cnt[r] : 0;
  u = c > 0 ? 1 : 0;
  pc = c > kPieceLen ? (c + kPieceLen - 1) / kPieceLen : 0;
}

__global__ void __launch_bounds__(kScanThreads) rowscan_reduce_kernel(const int32_t* __restrict__ cnt,
                                                                      int64_t N, int32_t* tmp,
                                                                      int64_t tstride) {
  __shared__ int s_warp[32];
  const int64_t base = int64_t(blockIdx.x) * kScanTile + threadIdx.x * kScanItems;
  int sc = 0, su = 0, sp = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    int c, u, pc;
    row_triple(cnt, N, base + i, c, u, pc);
    sc += c; su += u; sp += pc;
  }
  int tc, tu, tp;
  block_excl_scan(sc, s_warp, &tc);
  block_excl_scan(su, s_warp, &tu);
  block_excl_scan(sp, s_warp, &tp);
  if (threadIdx.x == 0) {
    tmp[blockIdx.x] = tc;
    tmp[tstride + blockIdx.x] = tu;
    tmp[2 * tstride + blockIdx.x] = tp;
  }
}

// cnt: counts in, exclusive offsets out (the scatter's cursors); tot: the
// three totals (n, U, pieces) from the top-level scans
__global__ void __launch_bounds__(kScanThreads) rowscan_down_kernel(
    int32_t* __restrict__ cnt, int64_t N, int64_t n, const int32_t* __restrict__ tmp, int64_t tstride,
    const int32_t* __restrict__ tot, int32_t* __restrict__ uid, int32_t* __restrict__ run_begin,
    int32_t* __restrict__ rows_out, int32_t* __restrict__ piece_base, int32_t* U, int32_t* n_slots) {
  __shared__ int s_warp[32];
  const int64_t base = int64_t(blockIdx.x) * kScanTile + threadIdx.x * kScanItems;
  int c[kScanItems], u[kScanItems], pc[kScanItems], sc = 0, su = 0, sp = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    row_triple(cnt, N, base + i, c[i], u[i], pc[i]);
    sc += c[i]; su += u[i]; sp += pc[i];
  }
  int t;
  int ec = block_excl_scan(sc, s_warp, &t) + tmp[blockIdx.x];
  int eu = block_excl_scan(su, s_warp, &t) + tmp[tstride + blockIdx.x];
  int ep = block_excl_scan(sp, s_warp, &t) + tmp[2 * tstride + blockIdx.x];
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    const int64_t r = base + i;
    if (r < N) {
      cnt[r] = ec;
      uid[r] = eu;
      if (c[i] > 0) {
        run_begin[eu] = ec;
        if (rows_out) rows_out[eu] = int32_t(r);
        if (pc[i]) piece_base[ec] = ep;
      }
    }
    ec += c[i]; eu += u[i]; ep += pc[i];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *U = tot[1];
    *n_slots = tot[2];
    run_begin[tot[1]] = int32_t(n);
  }
}

// one thread per run head: short runs sorted in place, long ones listed
// (runs of keys >= order_limit keep the scatter's order: their positions'
// order is irrelevant to the caller)
__global__ void __launch_bounds__(256) csort_fix_kernel(const int32_t* __restrict__ kout,
                                                        int32_t* __restrict__ vout,
                                                        const int32_t* __restrict__ end, int64_t n,
                                                        int32_t* __restrict__ long_list,
                                                        int32_t* __restrict__ n_long,
                                                        uint32_t order_limit, int64_t med_off) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int32_t k = kout[i];
    if (i > 0 && kout[i - 1] == k) continue;
    if (uint32_t(k) >= order_limit) continue;
    const int len = int(int64_t(end[k]) - i);
    if (len <= 1) continue;
    if (len > kFixShort) {     // n_long[0]: CTA runs (list from the front), n_long[1]:
      if (len > kFixMed)       // warp runs (list from long_list + med_off)
        long_list[atomicAdd(n_long, 1)] = int32_t(i);
      else
        long_list[med_off + atomicAdd(n_long + 1, 1)] = int32_t(i);
      continue;
    }
    const uint32_t M = kPosMask;
    auto cs = [M](int32_t& p, int32_t& q) {
      if ((uint32_t(p) & M) > (uint32_t(q) & M)) { const int32_t t = p; p = q; q = t; }
    };
    if (len <= 4) {           // most runs (C2: mean 2.3): a sorting network in registers
      int32_t x0 = vout[i], x1 = vout[i + 1];
      int32_t x2 = len > 2 ? vout[i + 2] : int32_t(0x7fffffff);
      int32_t x3 = len > 3 ? vout[i + 3] : int32_t(0x7fffffff);
      cs(x0, x1); cs(x2, x3); cs(x0, x2); cs(x1, x3); cs(x1, x2);
      vout[i] = x0;
      vout[i + 1] = x1;
      if (len > 2) vout[i + 2] = x2;
      if (len > 3) vout[i + 3] = x3;
      continue;
    }
    if (len <= 8) {           // Batcher's odd-even merge network for 8 (19 exchanges)
      int32_t x[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) x[j] = j < len ? vout[i + j] : int32_t(0x7fffffff);
      cs(x[0], x[1]); cs(x[2], x[3]); cs(x[4], x[5]); cs(x[6], x[7]);
      cs(x[0], x[2]); cs(x[1], x[3]); cs(x[4], x[6]); cs(x[5], x[7]);
      cs(x[1], x[2]); cs(x[5], x[6]);
      cs(x[0], x[4]); cs(x[1], x[5]); cs(x[2], x[6]); cs(x[3], x[7]);
      cs(x[2], x[4]); cs(x[3], x[5]);
      cs(x[1], x[2]); cs(x[3], x[4]); cs(x[5], x[6]);
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (j < len) vout[i + j] = x[j];
      continue;
    }
    int32_t a[kFixShort];
    for (int j = 0; j < len; ++j) a[j] = vout[i + j];
    for (int j = 1; j < len; ++j) {      // insertion sort on the position
      const int32_t x = a[j];
      int t = j - 1;
      while (t >= 0 && (uint32_t(a[t]) & kPosMask) > (uint32_t(x) & kPosMask)) {
        a[t + 1] = a[t];
        --t;
      }
      a[t + 1] = x;
    }
    for (int j = 0; j < len; ++j) vout[i + j] = a[j];
  }
}

// one warp per medium run (33..kFixMed positions): a bitonic sort of the run
// (padded to a power of two) in the warp's shared-memory slice
__global__ void __launch_bounds__(256) csort_med_kernel(const int32_t* __restrict__ kout,
                                                       int32_t* __restrict__ vout,
                                                       const int32_t* __restrict__ end,
                                                       const int32_t* __restrict__ med_list,
                                                       const int32_t* __restrict__ n_med) {
  __shared__ uint32_t s_all[8][kFixMed];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t* sw = s_all[wid];
  const int nm = *n_med;
  for (int r = blockIdx.x * 8 + wid; r < nm; r += gridDim.x * 8) {
    const int64_t b = med_list[r];
    const int len = int(int64_t(end[kout[b]]) - b);
    int p2 = 64;
    while (p2 < len) p2 <<= 1;
    for (int j = lane; j < p2; j += 32) sw[j] = j < len ? uint32_t(vout[b + j]) : 0xffffffffu;
    __syncwarp();
    for (int k = 2; k <= p2; k <<= 1) {
      for (int j = k >> 1; j > 0; j >>= 1) {
        for (int t = lane; t < p2 / 2; t += 32) {
          const int i0 = (t / j) * 2 * j + (t & (j - 1)), i1 = i0 + j;
          const uint32_t x = sw[i0], y = sw[i1];
          if (((x & kPosMask) > (y & kPosMask)) == ((i0 & k) == 0)) {
            sw[i0] = y;
            sw[i1] = x;
          }
        }
        __syncwarp();
      }
    }
    for (int j = lane; j < len; j += 32) vout[b + j] = int32_t(sw[j]);
    __syncwarp();
  }
}

// one CTA per long run (grid-stride over the list); tmp: scratch of n values
__global__ void __launch_bounds__(256) csort_long_kernel(const int32_t* __restrict__ kout,
                                                         int32_t* __restrict__ vout,
                                                         int32_t* __restrict__ tmp,
                                                         const int32_t* __restrict__ end,
                                                         const int32_t* __restrict__ long_list,
                                                         const int32_t* __restrict__ n_long) {
  __shared__ uint32_t s[kFixSmem];
  const int nl = *n_long;
  const int tid = threadIdx.x;
  for (int r = blockIdx.x; r < nl; r += gridDim.x) {
    const int64_t b = long_list[r];
    const int64_t L = int64_t(end[kout[b]]) - b;
    int32_t* v = vout + b;
    for (int64_t c0 = 0; c0 < L; c0 += kFixSmem) {      // chunks sorted in shared memory
      const int m = int(L - c0 < kFixSmem ? L - c0 : kFixSmem);
      int p2 = 64;
      while (p2 < m) p2 <<= 1;
      for (int j = tid; j < p2; j += 256) s[j] = j < m ? uint32_t(v[c0 + j]) : 0xffffffffu;
      __syncthreads();
      for (int k = 2; k <= p2; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
          for (int t = tid; t < p2 / 2; t += 256) {
            const int i0 = (t / j) * 2 * j + (t & (j - 1)), i1 = i0 + j;
            const uint32_t x = s[i0], y = s[i1];
            if (((x & kPosMask) > (y & kPosMask)) == ((i0 & k) == 0)) {
              s[i0] = y;
              s[i1] = x;
            }
          }
          __syncthreads();
        }
      }
      for (int j = tid; j < m; j += 256) v[c0 + j] = int32_t(s[j]);
      __syncthreads();
    }
    int32_t* src = v;
    int32_t* dst = tmp + b;
    for (int64_t w = kFixSmem; w < L; w <<= 1) {         // merge passes (merge path per thread)
      for (int64_t s0 = 0; s0 < L; s0 += 2 * w) {
        const int32_t* A = src + s0;
        const int64_t na = L - s0 < w ? L - s0 : w;
        const int32_t* B = A + na;
        const int64_t nb = L - s0 - na < w ? L - s0 - na : w;
        const int64_t m = na + nb;
        const int64_t o0 = m * tid / 256, o1 = m * (tid + 1) / 256;
        int64_t lo = o0 - nb > 0 ? o0 - nb : 0, hi = o0 < na ? o0 : na;
        while (lo < hi) {
          const int64_t mid = (lo + hi) >> 1;
          if ((uint32_t(A[mid]) & kPosMask) <= (uint32_t(B[o0 - mid - 1]) & kPosMask)) lo = mid + 1;
          else hi = mid;
        }
        int64_t ia = lo, ib = o0 - lo;
        for (int64_t o = o0; o < o1; ++o) {
          const bool takeA = ib >= nb ||
              (ia < na && (uint32_t(A[ia]) & kPosMask) <= (uint32_t(B[ib]) & kPosMask));
          dst[s0 + o] = takeA ? A[ia++] : B[ib++];
        }
      }
      __syncthreads();
      int32_t* t = src;
      src = dst;
      dst = t;
    }
    if (src != v) {
      for (int64_t j = tid; j < L; j += 256) v[j] = src[j];
    }
    __syncthreads();
  }
}

}  // namespace

// ------------------------------------------------------------ host side
int64_t scan_tmp_elems(int64_t n) { return (n + kScanTile - 1) / kScanTile + 1; }

mlStatus scan_exclusive(const int32_t* in, int32_t* out, int64_t n, int32_t* tmp, int32_t* total,
                        cudaStream_t s) {
  if (n <= 0) {
    if (total) ML_CUDA_TRY(cudaMemsetAsync(total, 0, sizeof(int32_t), s));
    return ML_OK;
  }
  const int64_t nb = (n + kScanTile - 1) / kScanTile;
  scan_reduce_kernel<<<unsigned(nb), kScanThreads, 0, s>>>(in, n, tmp);
  ML_LAUNCH_CHECK("scan_reduce");
  scan_blocks_kernel<<<1, 1024, 0, s>>>(tmp, nb, total);
  ML_LAUNCH_CHECK("scan_blocks");
  scan_down_kernel<<<unsigned(nb), kScanThreads, 0, s>>>(in, out, n, tmp);
  ML_LAUNCH_CHECK("scan_down");
  return ML_OK;
}

static int sort_nblocks(int64_t n) { return int((n + kSortTile - 1) / kSortTile); }


// The counting sort (csort_*) needs one counter per key; it is used when the
// key range 2^bits is at most twice the key count, and only then are the
// counters sized for it.
static bool counting_sort_fits(int64_t n, int bits) {
  return bits >= 1 && bits <= 30 && (int64_t(1) << bits) <= 2 * n;
}

void sort_carve(Carver& c, int64_t n, int bits, SortBufs& b) {
  const int nb = sort_nblocks(n);
  b.k[0] = c.take<int32_t>(n);
  b.v[0] = c.take<int32_t>(n);
  b.k[1] = c.take<int32_t>(n);
  b.v[1] = c.take<int32_t>(n);
  // counting sort: [2^bits] counters + [2^bits] run ids of the rows; scan
  // scratch for three row scans
  const bool cf = counting_sort_fits(n, bits);
  const int64_t ncnt = std::max<int64_t>((int64_t(1) << kMaxDigitBits) * nb,
                                         cf ? int64_t(2) << bits : 0);
  b.counts = c.take<int32_t>(ncnt);
  b.scan_tmp = c.take<int32_t>(std::max<int64_t>(scan_tmp_elems(ncnt),
                                                 cf ? 3 * scan_tmp_elems(int64_t(1) << bits) : 0));
  b.ghist = c.take<int32_t>(3 * (int64_t(1) << kMaxDigitBits) + 8);
}

static int sort_passes(int bits) { return (bits + kMaxDigitBits - 1) / kMaxDigitBits; }

static bool counting_applies(int64_t n, int bits, int64_t key_limit) {
  static const bool on = [] {
    const char* e = std::getenv("ML_SORT_COUNTING");
    return !(e && e[0] == '0');
  }();
  if (bits < 1) bits = 1;
  // n <= 8 * key_limit (ML_SORT_COUNTING_MAX_PER_KEY): short runs on
  // average.  The fixup sorts runs of 33..256 positions with one warp, longer
  // ones with one CTA.  Measured: with every long run on a CTA, ~128
  // positions per key (C3's sparse key backward) cost 0.92 ms against the
  // radix sort's 0.43; at 32 per key (C5 per rank, 70 % of them one
  // sentinel key whose atomics serialise) the counting sort only broke even
  // (10.93-10.99 vs 10.87-10.91 ms); at 8 per key (C4 per rank) it wins
  // (1.66 vs 1.695 ms), at 2 (C2) too (5.05-5.10 vs 5.13)
  static const int64_t per_key = [] {
    const char* e = std::getenv("ML_SORT_COUNTING_MAX_PER_KEY");
    return e ? std::max<int64_t>(1, std::atoll(e)) : int64_t(8);
  }();
  return on && sort_passes(bits) >= 2 && key_limit > 0 && key_limit <= (int64_t(1) << bits) &&
         counting_sort_fits(n, bits) && n <= per_key * key_limit && n < (int64_t(1) << 31) - 1;
}

// The counting sort (csort_* kernels), output where sorted_result names it.
// r != nullptr: also the runs (find_runs' outputs) from the row scan.
static mlStatus counting_sort(const int32_t* keys_in, int64_t n, int bits, int64_t key_limit,
                              SortBufs& b, RunBufs* r, int32_t* rows_out, int32_t* U,
                              int32_t** keys, int32_t** vals, cudaStream_t s,
                              int64_t order_limit = -1) {
  const int fin = (sort_passes(bits) - 1) & 1;
  int32_t* kout = b.k[fin];
  int32_t* vout = b.v[fin];
  int32_t* spare_k = b.k[fin ^ 1];
  int32_t* spare_v = b.v[fin ^ 1];
  const uint32_t lim = uint32_t(key_limit);
  int32_t* n_long = b.ghist;
  ML_CUDA_TRY(cudaMemsetAsync(b.counts, 0, sizeof(int32_t) * size_t(lim), s));
  ML_CUDA_TRY(cudaMemsetAsync(n_long, 0, 2 * sizeof(int32_t), s));   // CTA runs, warp runs
  const unsigned g = unsigned(std::min<int64_t>((n + 255) / 256, int64_t(num_sms()) * 8));
  csort_hist_kernel<<<g, 256, 0, s>>>(keys_in, n, lim, b.counts, index_flag_ptr());
  ML_LAUNCH_CHECK("csort_hist");
  int32_t* uid = nullptr;
  if (r) {
    uid = b.counts + (int64_t(1) << bits);
    const int64_t nt = (int64_t(lim) + kScanTile - 1) / kScanTile;
    const int64_t ts = nt + 1;
    int32_t* tot = b.ghist + 4;
    rowscan_reduce_kernel<<<unsigned(nt), kScanThreads, 0, s>>>(b.counts, lim, b.scan_tmp, ts);
    ML_LAUNCH_CHECK("csort_rowscan");
    for (int j = 0; j < 3; ++j) {
      scan_blocks_kernel<<<1, 1024, 0, s>>>(b.scan_tmp + j * ts, nt, tot + j);
      ML_LAUNCH_CHECK("csort_rowscan");
    }
    rowscan_down_kernel<<<unsigned(nt), kScanThreads, 0, s>>>(
        b.counts, lim, n, b.scan_tmp, ts, tot, uid, r->run_begin, rows_out, r->piece_base,
        U ? U : r->lb, r->n_slots);
    ML_LAUNCH_CHECK("csort_rowscan");
  } else {
    ML_TRY(scan_exclusive(b.counts, b.counts, lim, b.scan_tmp, nullptr, s));
  }
  csort_scatter_kernel<<<g, 256, 0, s>>>(keys_in, n, lim, b.counts, kout, vout, uid,
                                         r ? r->rid : nullptr);
  ML_LAUNCH_CHECK("csort_scatter");
  const uint32_t ol = (order_limit >= 0 && order_limit < int64_t(lim)) ? uint32_t(order_limit) : lim;
  // the run lists share spare_k: runs > kFixShort number at most n / 33 each
  const int64_t med_off = n / 2;
  csort_fix_kernel<<<g, 256, 0, s>>>(kout, vout, b.counts, n, spare_k, n_long, ol, med_off);
  ML_LAUNCH_CHECK("csort_fix");
  csort_med_kernel<<<unsigned(num_sms()) * 2, 256, 0, s>>>(kout, vout, b.counts, spare_k + med_off,
                                                           n_long + 1);
  ML_LAUNCH_CHECK("csort_med");
  csort_long_kernel<<<unsigned(num_sms()), 256, 0, s>>>(kout, vout, spare_v, b.counts, spare_k,
                                                        n_long);
  ML_LAUNCH_CHECK("csort_long");
  *keys = kout;
  *vals = vout;
  return ML_OK;
}

mlStatus sorted_result(int64_t n, int bits, SortBufs& b, int32_t** keys, int32_t** vals) {
  if (n <= 0) {
    *keys = b.k[0];
    *vals = b.v[0];
    return ML_OK;
  }
  if (bits < 1) bits = 1;
  const int passes = sort_passes(bits);
  *keys = b.k[(passes - 1) & 1];
  *vals = b.v[(passes - 1) & 1];
  return ML_OK;
}

mlStatus sort_pairs(const int32_t* keys_in, int64_t n, int bits, SortBufs& b, int32_t** keys,
                    int32_t** vals, cudaStream_t s, int64_t key_limit, int64_t order_limit) {
  if (n <= 0) {
    *keys = b.k[0];
    *vals = b.v[0];
    return ML_OK;
  }
  if (bits < 1) bits = 1;
  if (bits > 31) return fail(ML_ERR_CONFIG, "sort: keys must fit in 31 bits");
  const int passes = sort_passes(bits);
  const int dbits = (bits + passes - 1) / passes;
  const int nbins = 1 << dbits;
  const int nb = sort_nblocks(n);
  if (counting_applies(n, bits, key_limit))
    return counting_sort(keys_in, n, bits, key_limit, b, nullptr, nullptr, nullptr, keys, vals, s,
                         order_limit);
  static bool attr = false;
  if (!attr) {
    const int max_smem = int(sizeof(int)) * ((kSortWarps + 2) * (1 << kMaxDigitBits) + 2 * kSortTile);
    ML_CUDA_TRY(cudaFuncSetAttribute(sort_hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     max_smem));
    ML_CUDA_TRY(cudaFuncSetAttribute(sort_scatter_kernel<false>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, max_smem));
    attr = true;
  }
  const size_t smem_hist = sizeof(int) * size_t(kSortWarps) * nbins;
  const size_t smem_scatter = sizeof(int) * (size_t(kSortWarps + 2) * nbins + 2 * kSortTile);
  SortPassParams p;
  p.n = n;
  p.nblocks = nb;
  p.dbits = dbits;
  p.key_limit = (key_limit > 0 && key_limit < (int64_t(1) << bits)) ? uint32_t(key_limit)
                                                                   : uint32_t(1) << bits;
  p.counts = b.counts;
  p.flag = index_flag_ptr();
  const int64_t ncounts = int64_t(nb) << dbits;
  const int32_t* kin = keys_in;
  const int32_t* vin = nullptr;
  int cur = 0;
  static const bool onesweep = [] {
    const char* e = std::getenv("ML_SORT_ONESWEEP");
    return !(e && e[0] == '0');
  }();
  if (onesweep && passes <= 3 && n < (int64_t(1) << 30)) {
    // one read of the keys for all passes' global histograms, then one
    // decoupled-look-back scatter kernel per pass
    ML_CUDA_TRY(cudaMemsetAsync(b.ghist, 0, sizeof(int32_t) * size_t(passes) * nbins, s));
    const unsigned gh = unsigned(std::min<int64_t>((n + 255) / 256, int64_t(num_sms()) * 8));
    sort_ghist_kernel<<<gh, 256, sizeof(int) * size_t(passes) * nbins, s>>>(
        keys_in, n, p.key_limit, passes, dbits, b.ghist, p.flag);
    ML_LAUNCH_CHECK("sort_hist");
    sort_gscan_kernel<<<1, 1024, 0, s>>>(b.ghist, passes, nbins);
    ML_LAUNCH_CHECK("scan_blocks");
    static bool attr1 = false;
    if (!attr1) {
      const int max_smem = int(sizeof(int)) * ((kSortWarps + 2) * (1 << kMaxDigitBits) + 2 * kSortTile);
      ML_CUDA_TRY(cudaFuncSetAttribute(sort_scatter_kernel<true>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, max_smem));
      attr1 = true;
    }
    p.status = reinterpret_cast<uint32_t*>(b.counts);
    for (int pass = 0; pass < passes; ++pass) {
      p.kin = kin;
      p.vin = vin;
      p.kout = b.k[cur];
      p.vout = b.v[cur];
      p.shift = pass * dbits;
      p.goff = b.ghist + pass * nbins;
      p.tile_ctr = b.ghist + passes * nbins + pass;
      ML_CUDA_TRY(cudaMemsetAsync(b.counts, 0, sizeof(uint32_t) * size_t(ncounts), s));
      sort_scatter_kernel<true><<<nb, 256, smem_scatter, s>>>(p, pass == 0);
      ML_LAUNCH_CHECK("sort_scatter");
      kin = b.k[cur];
      vin = b.v[cur];
      cur ^= 1;
    }
    *keys = const_cast<int32_t*>(kin);
    *vals = const_cast<int32_t*>(vin);
    return ML_OK;
  }
  for (int pass = 0; pass < passes; ++pass) {
    p.kin = kin;
    p.vin = vin;
    p.kout = b.k[cur];
    p.vout = b.v[cur];
    p.shift = pass * dbits;
    const bool first = pass == 0;
    sort_hist_kernel<<<nb, 256, smem_hist, s>>>(p, first);
    ML_LAUNCH_CHECK("sort_hist");
    ML_TRY(scan_exclusive(b.counts, b.counts, ncounts, b.scan_tmp, nullptr, s));
    sort_scatter_kernel<false><<<nb, 256, smem_scatter, s>>>(p, first);
    ML_LAUNCH_CHECK("sort_scatter");
    kin = b.k[cur];
    vin = b.v[cur];
    cur ^= 1;
  }
  *keys = const_cast<int32_t*>(kin);
  *vals = const_cast<int32_t*>(vin);
  return ML_OK;
}

void runs_carve(Carver& c, int64_t n, RunBufs& r) {
  r.rid = c.take<int32_t>(n);
  r.run_begin = c.take<int32_t>(n + 1);
  r.piece_base = c.take<int32_t>(n);
  r.n_slots = c.take<int32_t>(1);
  r.lb = c.take<int32_t>(4 * ((n + 2047) / 2048) + 8);   // 2 x tiles 64-bit status + tickets
}

mlStatus find_runs(const int32_t* skey, int64_t n, RunBufs& r, int32_t* rows_out, int32_t* U,
                   cudaStream_t s) {
  if (n <= 0) {
    if (U) ML_CUDA_TRY(cudaMemsetAsync(U, 0, sizeof(int32_t), s));
    return ML_OK;
  }
  if (n >= (int64_t(1) << 31)) return fail(ML_ERR_CONFIG, "runs: n must be < 2^31");
  const int64_t nt = (n + kRunTile - 1) / kRunTile;
  uint64_t* st1 = reinterpret_cast<uint64_t*>(r.lb);   // r.lb is 8-byte aligned (carver)
  uint64_t* st2 = st1 + nt;
  int32_t* tickets = r.lb + 4 * nt;     // [0], [1]: tile tickets; [2]: U when the caller passes none
  int32_t* u = U ? U : tickets + 2;
  ML_CUDA_TRY(cudaMemsetAsync(r.lb, 0, sizeof(int32_t) * size_t(4 * nt + 2), s));
  run_scan1_kernel<<<unsigned(nt), kScanThreads, 0, s>>>(skey, n, r.rid, r.run_begin, rows_out, u,
                                                         st1, tickets);
  ML_LAUNCH_CHECK("run_flags");
  run_scan2_kernel<<<unsigned(nt), kScanThreads, 0, s>>>(r.run_begin, u, r.piece_base, r.n_slots,
                                                         int(nt), st2, tickets + 1);
  ML_LAUNCH_CHECK("run_pieces");
  return ML_OK;
}

mlStatus sort_pairs_runs(const int32_t* keys_in, int64_t n, int bits, int64_t key_limit,
                         SortBufs& b, RunBufs& r, int32_t* rows_out, int32_t* U, int32_t** keys,
                         int32_t** vals, cudaStream_t s) {
  // opt-in (ML_RUNS_ROWSCAN=1): bit-identical, and the state is ready ~0.1 ms
  // sooner at C2, but the gate GEMMs that filled the segmented pass's wait
  // then land after it: step 5.178 vs 5.143 ms (scripts/rowscan_check.sh)
  static const bool rowscan = [] {
    const char* e = std::getenv("ML_RUNS_ROWSCAN");
    return e && e[0] == '1';
  }();
  if (n > 0 && rowscan && counting_applies(n, bits, key_limit))
    return counting_sort(keys_in, n, bits < 1 ? 1 : bits, key_limit, b, &r, rows_out, U, keys, vals, s);
  ML_TRY(sort_pairs(keys_in, n, bits, b, keys, vals, s, key_limit));
  return find_runs(*keys, n, r, rows_out, U, s);
}

}  // namespace ml
