// Product-key top-k (§3.1.1) and its backward.
//
//  scores:   S_half[t,h,half,a] = q[t,h,half*Dk/2 : ...] . K_half[h,a,:]   (fp32 FMA)
//  half top-k: per (t,h,half) the k best of S (score desc, ties -> lower a)
//  combine:  the k best of the k*k sums s1[i] + s2[j] (ties -> lower flat
//            index a*S+b), then w = softmax (Eq. 1)
//  softmax bwd: ds = w (dw - sum_j w_j dw_j)
//
// Selection is exact: every candidate gets a unique 64-bit key
// (ord(score) << 32 | ~id) whose order is the paper's order plus the
// tie-break; a warp-cooperative MSB radix select (8-bit digits, shared-memory
// histogram, early exit once the boundary bin is exactly filled) finds the k
// largest keys, which are then bitonic-sorted across the warp.
#include "internal.cuh"

namespace ml {
namespace {

constexpr unsigned FULL = 0xffffffffu;

// ------------------------------------------------ SIMT fp32 scoring GEMM
// Tile: 64 tokens x 64 keys, K-chunks of 32; 256 threads, 4x4 per thread.
template <typename T>
__global__ void __launch_bounds__(256) pkm_scores_kernel(const T* q, const T* K1, const T* K2,
                                                         float* scores, int T_, int H, int S,
                                                         int Dk) {
  __shared__ float As[32][64 + 4];
  __shared__ float Bs[32][64 + 4];
  const int Dh = Dk / 2;
  const int hh = blockIdx.z;  // h*2 + half
  const int h = hh >> 1, half = hh & 1;
  const T* K = half ? K2 : K1;
  const int t0 = blockIdx.x * 64, a0 = blockIdx.y * 64;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < Dh; k0 += 32) {
    for (int e = threadIdx.x; e < 64 * 32; e += 256) {
      const int m = e >> 5, kk = e & 31;
      const int t = t0 + m, a = a0 + m, kc = k0 + kk;
      float av = 0.f, bv = 0.f;
      if (t < T_ && kc < Dh) av = to_f(q[(int64_t(t) * H + h) * Dk + half * Dh + kc]);
      if (a < S && kc < Dh) bv = to_f(K[(int64_t(h) * S + a) * Dh + kc]);
      As[kk][m] = av;
      Bs[kk][m] = bv;
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < 32; ++kk) {
      float ar[4], br[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) ar[i] = As[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) br[j] = Bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(ar[i], br[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int t = t0 + ty + 16 * i;
    if (t >= T_) continue;
    float* row = scores + ((int64_t(t) * H + h) * 2 + half) * S;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int a = a0 + tx + 16 * j;
      if (a < S) row[a] = acc[i][j];
    }
  }
}

// ------------------------------------------------ warp top-k machinery
__device__ __forceinline__ uint64_t make_key(float score, uint32_t id) {
  return (uint64_t(ord_f32(score)) << 32) | uint64_t(0xFFFFFFFFu - id);
}
__device__ __forceinline__ uint32_t key_id(uint64_t k) { return 0xFFFFFFFFu - uint32_t(k); }
__device__ __forceinline__ float key_score(uint64_t k) { return unord_f32(uint32_t(k >> 32)); }

// Bitonic sort of one u64 per lane, descending across lanes 0..31.
__device__ __forceinline__ uint64_t warp_sort_desc(uint64_t x) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      const uint64_t y = __shfl_xor_sync(FULL, x, stride);
      const bool up = ((lane & size) == 0);          // this block sorted descending?
      const bool lower = ((lane & stride) == 0);
      const bool take_max = (up == lower);
      x = take_max ? (x > y ? x : y) : (x < y ? x : y);
    }
  }
  return x;
}

// k largest of n unique keys gen(e), e < n; lane j < k returns the j-th
// largest (descending); lanes >= k return 0.  hist: 256 u32 of warp-private
// smem; buf: 32 u64 of warp-private smem.
template <class Gen>
__device__ uint64_t warp_topk(const Gen& gen, int n, int k, uint32_t* hist, uint64_t* buf) {
  const int lane = threadIdx.x & 31;
  uint64_t prefix = 0;
  int shift = 64;
  int need = k;
  while (shift > 0) {
    shift -= 8;
    for (int b = lane; b < 256; b += 32) hist[b] = 0;
    __syncwarp();
    const int hs = shift + 8;
    for (int e = lane; e < n; e += 32) {
      const uint64_t key = gen(e);
      const bool match = (hs >= 64) || ((key >> hs) == (prefix >> hs));
      if (match) atomicAdd(&hist[(key >> shift) & 255u], 1u);
    }
    __syncwarp();
    uint32_t c[8], tot = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      c[j] = hist[lane * 8 + j];
      tot += c[j];
    }
    uint32_t incl = tot;  // suffix sum over lanes >= lane
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_down_sync(FULL, incl, o);
      if (lane + o < 32) incl += v;
    }
    uint32_t cum = incl - tot;  // keys in bins of higher lanes
    int found = -1;
    uint32_t above = 0, cnt = 0;
#pragma unroll
    for (int j = 7; j >= 0; --j) {
      if (found < 0 && cum < uint32_t(need) && cum + c[j] >= uint32_t(need)) {
        found = lane * 8 + j;
        above = cum;
        cnt = c[j];
      }
      cum += c[j];
    }
    const unsigned fm = __ballot_sync(FULL, found >= 0);
    const int srcl = __ffs(fm) - 1;
    found = __shfl_sync(FULL, found, srcl);
    above = __shfl_sync(FULL, above, srcl);
    cnt = __shfl_sync(FULL, cnt, srcl);
    need -= int(above);
    prefix |= uint64_t(found) << shift;
    __syncwarp();
    if (int(cnt) == need) break;
  }
  // selected: (key >> shift) >= (prefix >> shift); exactly k of them
  const uint64_t thr = prefix >> shift;
  int base = 0;
  const unsigned lt = (1u << lane) - 1u;
  for (int e0 = 0; e0 < n; e0 += 32) {
    const int e = e0 + lane;
    uint64_t key = 0;
    bool sel = false;
    if (e < n) {
      key = gen(e);
      sel = (key >> shift) >= thr;
    }
    const unsigned sm = __ballot_sync(FULL, sel);
    if (sel) buf[base + __popc(sm & lt)] = key;
    base += __popc(sm);
  }
  __syncwarp();
  uint64_t x = lane < k ? buf[lane] : 0ull;
  __syncwarp();
  return warp_sort_desc(x);
}

// ---- fast exact top-k: threshold filter + exact select on the survivors.
// theta = k-th largest of the union of every lane's 4 largest keys is a lower
// bound of the true k-th largest key (the union is a subset of all keys), so
// {keys >= theta} contains the top-k; it is typically ~k + a few elements.

__device__ __forceinline__ void insert4(uint64_t key, uint64_t& t0, uint64_t& t1, uint64_t& t2,
                                        uint64_t& t3) {
  if (key > t3) {
    if (key > t1) {
      t3 = t2;
      t2 = t1;
      if (key > t0) { t1 = t0; t0 = key; } else { t1 = key; }
    } else {
      if (key > t2) { t3 = t2; t2 = key; } else { t3 = key; }
    }
  }
}

constexpr int kCandCap = 256;

struct alignas(16) TopkSmem {   // per warp
  uint32_t hist[256];
  uint64_t sel[32];
  uint64_t u128[128];
  uint64_t cand[kCandCap];
};

// theta from the per-lane top-4 lists (t0 >= t1 >= t2 >= t3; 0 = empty)
__device__ __forceinline__ uint64_t warp_theta(uint64_t t0, uint64_t t1, uint64_t t2, uint64_t t3,
                                               int k, TopkSmem& sm) {
  const int lane = threadIdx.x & 31;
  sm.u128[lane * 4 + 0] = t0;
  sm.u128[lane * 4 + 1] = t1;
  sm.u128[lane * 4 + 2] = t2;
  sm.u128[lane * 4 + 3] = t3;
  __syncwarp();
  const uint64_t* u = sm.u128;
  auto gen = [u](int e) { return u[e]; };
  const uint64_t top = warp_topk(gen, 128, k, sm.hist, sm.sel);
  return __shfl_sync(FULL, top, k - 1);
}

// append the keys >= theta of this round (one candidate per lane) to sm.cand
__device__ __forceinline__ void append_cand(uint64_t key, bool sel, int& count, TopkSmem& sm) {
  const int lane = threadIdx.x & 31;
  const unsigned m = __ballot_sync(FULL, sel);
  const int pos = count + __popc(m & ((1u << lane) - 1u));
  if (sel && pos < kCandCap) sm.cand[pos] = key;
  count += __popc(m);
}

__device__ __forceinline__ uint64_t select_cand(int count, int k, TopkSmem& sm) {
  __syncwarp();
  const uint64_t* c = sm.cand;
  auto gen = [c](int e) { return c[e]; };
  return warp_topk(gen, count, k, sm.hist, sm.sel);
}

// theta from every lane's maximum: the k largest lane maxima are k distinct
// keys, so the k-th largest of them bounds the true k-th largest from below.
__device__ __forceinline__ uint64_t warp_theta_max(uint64_t lane_max, int k) {
  const uint64_t sorted = warp_sort_desc(lane_max);
  return __shfl_sync(FULL, sorted, k - 1);
}

// Bitonic sort of one float per lane, descending across lanes 0..31.
__device__ __forceinline__ float warp_sort_desc_f(float x) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      const float y = __shfl_xor_sync(FULL, x, stride);
      const bool take_max = (((lane & size) == 0) == ((lane & stride) == 0));
      x = take_max ? fmaxf(x, y) : fminf(x, y);
    }
  }
  return x;
}

// Fast exact path for rows of raw scores with S % 128 == 0 and k <= 32.
//  1. every lane keeps the two largest of its S/32 values;
//  2. theta = the k-th largest of those 64 values (two 32-lane sorts + the
//     merge-path identity kth(A u B) = max_i min(A[i-1], B[k-1-i])) is a
//     lower bound of the row's k-th largest value (64 distinct elements);
//  3. survivors v >= theta (~k + 4 on continuous data) go to shared memory;
//  4. each survivor's rank in (score desc, index asc) order is counted
//     against all survivors and ranks < k are written directly.
// Returns false (nothing written) when more than 64 values survive (ties).
// FULL: S == 1024 (all R rounds present: no padding of absent rounds)
template <bool FULL>
__device__ __forceinline__ bool row_topk_fast(const float* sr, int S, int k, TopkSmem& sm,
                                              int64_t row, int32_t* hI, float* hs, int* count_out) {
  constexpr int R = 8;                         // float4 rounds held in registers (S <= 1024)
  const int lane = threadIdx.x & 31;
  const int rounds = FULL ? R : S / 128;
  float4 v[R];
#pragma unroll
  for (int r = 0; r < R; ++r)
    v[r] = r < rounds ? *reinterpret_cast<const float4*>(sr + r * 128 + lane * 4)
                      : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
  float m0 = -INFINITY, m1 = -INFINITY;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const float vs[4] = {v[r].x, v[r].y, v[r].z, v[r].w};
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const float lo = fminf(m0, vs[c]);
      m0 = fmaxf(m0, vs[c]);
      m1 = fmaxf(m1, lo);
    }
  }
  const float A = warp_sort_desc_f(m0), B = warp_sort_desc_f(m1);
  // k-th largest of A u B (both descending): max over i = 0..k of min(A[i-1], B[k-1-i])
  float c = -INFINITY;
  {
    const int i = lane;
    const float a = __shfl_sync(FULL, A, (i + 31) & 31);
    const float b = __shfl_sync(FULL, B, (k - 1 - i) & 31);
    if (i <= k - 1) c = fminf(i == 0 ? INFINITY : a, b);
  }
  const float ak = __shfl_sync(FULL, A, k - 1);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c = fmaxf(c, __shfl_xor_sync(FULL, c, o));
  const float theta = fmaxf(c, ak);
  // survivors v >= theta: one lane-order scan per row, keys to shared memory
  uint32_t mask = 0;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    mask |= (v[r].x >= theta ? 1u : 0u) << (4 * r);
    mask |= (v[r].y >= theta ? 2u : 0u) << (4 * r);
    mask |= (v[r].z >= theta ? 4u : 0u) << (4 * r);
    mask |= (v[r].w >= theta ? 8u : 0u) << (4 * r);
  }
  const int cnt = __popc(mask);
  int incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(FULL, incl, o);
    if (lane >= o) incl += y;
  }
  const int count = __shfl_sync(FULL, incl, 31);
  *count_out = count;
  int pos = incl - cnt;
  uint64_t* ck = sm.cand;
  // the lane's survivors (~1 per lane) are re-read from the row (L1/L2 hits):
  // bit 4r + c of mask <-> element r*128 + lane*4 + c
  for (uint32_t bits = mask; bits; bits &= bits - 1) {
    const int b = __ffs(bits) - 1;
    const int e = (b >> 2) * 128 + lane * 4 + (b & 3);
    if (pos < kCandCap) ck[pos] = make_key(sr[e], uint32_t(e));
    ++pos;
  }
  if (count > 64) return false;
  __syncwarp();
  // rank of the keys at lane and lane + 32 among all survivors (keys unique),
  // two survivors per shared-memory load
  const bool h0 = lane < count, h1 = lane + 32 < count;
  const uint64_t k0 = h0 ? ck[lane] : ~0ull, k1 = h1 ? ck[lane + 32] : ~0ull;
  int r0 = 0, r1 = 0;
  if ((count & 1) != 0) ck[count] = 0ull;   // pad: ranks nothing
  __syncwarp();
  const int pairs = (count + 1) >> 1;
  if (count <= 32) {
    for (int l = 0; l < pairs; ++l) {
      const ulonglong2 kk = reinterpret_cast<const ulonglong2*>(ck)[l];
      r0 += (kk.x > k0 ? 1 : 0) + (kk.y > k0 ? 1 : 0);
    }
  } else {
    for (int l = 0; l < pairs; ++l) {
      const ulonglong2 kk = reinterpret_cast<const ulonglong2*>(ck)[l];
      r0 += (kk.x > k0 ? 1 : 0) + (kk.y > k0 ? 1 : 0);
      r1 += (kk.x > k1 ? 1 : 0) + (kk.y > k1 ? 1 : 0);
    }
  }
  if (h0 && r0 < k) { hI[row * k + r0] = int32_t(key_id(k0)); hs[row * k + r0] = key_score(k0); }
  if (h1 && r1 < k) { hI[row * k + r1] = int32_t(key_id(k1)); hs[row * k + r1] = key_score(k1); }
  return true;
}

// Streaming variant for long rows (S % 128 == 0, S > 1024: the 16m / 64m
// memories): the same bound-then-rank selection without holding the
// row in registers.
//  1. every lane streams its S/32 values (float4 rounds) keeping its two
//     largest; theta = the k-th largest of those 64 values (a lower bound of
//     the row's k-th largest: 64 distinct elements);
//  2. the row is streamed again (L2-hot) and the survivors v >= theta
//     (typically k + ~15) are appended to shared memory in lane order;
//  3. survivors are ranked by counting on unique keys (ranks < k written).
// Returns false (nothing written) when more than 64 values survive.
__device__ __forceinline__ bool row_topk_stream(const float* sr, int S, int k, TopkSmem& sm,
                                                int64_t row, int32_t* hI, float* hs,
                                                int* count_out) {
  const int lane = threadIdx.x & 31;
  const int rounds = S / 128;
  float m0 = -INFINITY, m1 = -INFINITY;
#pragma unroll 4
  for (int r = 0; r < rounds; ++r) {
    const float4 v = *reinterpret_cast<const float4*>(sr + r * 128 + lane * 4);
    const float vs[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const float lo = fminf(m0, vs[c]);
      m0 = fmaxf(m0, vs[c]);
      m1 = fmaxf(m1, lo);
    }
  }
  const float A = warp_sort_desc_f(m0), B = warp_sort_desc_f(m1);
  float c = -INFINITY;
  {
    const int i = lane;
    const float a = __shfl_sync(FULL, A, (i + 31) & 31);
    const float b = __shfl_sync(FULL, B, (k - 1 - i) & 31);
    if (i <= k - 1) c = fminf(i == 0 ? INFINITY : a, b);
  }
  const float ak = __shfl_sync(FULL, A, k - 1);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c = fmaxf(c, __shfl_xor_sync(FULL, c, o));
  const float theta = fmaxf(c, ak);
  int count = 0;
  uint64_t* ck = sm.cand;
#pragma unroll 4
  for (int r = 0; r < rounds; ++r) {
    const float4 v = *reinterpret_cast<const float4*>(sr + r * 128 + lane * 4);
    const uint32_t mk = (v.x >= theta ? 1u : 0u) | (v.y >= theta ? 2u : 0u) |
                        (v.z >= theta ? 4u : 0u) | (v.w >= theta ? 8u : 0u);
    if (__any_sync(FULL, mk != 0u)) {
      const int cnt = __popc(mk);
      int incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += y;
      }
      int pos = count + incl - cnt;
      const float vs[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if ((mk >> q) & 1u) {
          if (pos < kCandCap) ck[pos] = make_key(vs[q], uint32_t(r * 128 + lane * 4 + q));
          ++pos;
        }
      }
      count += __shfl_sync(FULL, incl, 31);
    }
  }
  *count_out = count;
  if (count > 64) return false;
  __syncwarp();
  const bool h0 = lane < count, h1 = lane + 32 < count;
  const uint64_t k0 = h0 ? ck[lane] : ~0ull, k1 = h1 ? ck[lane + 32] : ~0ull;
  int r0 = 0, r1 = 0;
  if ((count & 1) != 0) ck[count] = 0ull;   // pad: ranks nothing
  __syncwarp();
  const int pairs = (count + 1) >> 1;
  for (int l = 0; l < pairs; ++l) {
    const ulonglong2 kk = reinterpret_cast<const ulonglong2*>(ck)[l];
    r0 += (kk.x > k0 ? 1 : 0) + (kk.y > k0 ? 1 : 0);
    r1 += (kk.x > k1 ? 1 : 0) + (kk.y > k1 ? 1 : 0);
  }
  if (h0 && r0 < k) { hI[row * k + r0] = int32_t(key_id(k0)); hs[row * k + r0] = key_score(k0); }
  if (h1 && r1 < k) { hI[row * k + r1] = int32_t(key_id(k1)); hs[row * k + r1] = key_score(k1); }
  return true;
}

// Chunk-filtered variant for long rows (S % 1024 == 0, S >= 2048) when the
// scoring epilogue wrote cm = the maxima of the row's S/32 chunks of 32
// consecutive scores:
//  1. every lane keeps the two largest of its S/1024 chunk maxima; theta =
//     the k-th largest of those 64 values (distinct elements of the row, so a
//     lower bound of its k-th largest score);
//  2. only the chunks whose maximum reaches theta (typically ~k of S/32) are
//     read, one coalesced 128-byte row segment each, and their scores
//     v >= theta appended to shared memory;
//  3. survivors ranked by counting as in row_topk_stream.
// Reads ~k * 128 B of scores per row instead of streaming the row twice.
__device__ __forceinline__ bool row_topk_chunks(const float* sr, const float* cm, int S, int k,
                                                TopkSmem& sm, int64_t row, int32_t* hI, float* hs,
                                                int* count_out) {
  constexpr int NJ = 8;                        // chunk maxima per lane held in registers (S <= 8192)
  const int lane = threadIdx.x & 31;
  const int nj = S >> 10;
  float x[NJ];
  float m0 = -INFINITY, m1 = -INFINITY;
#pragma unroll
  for (int j = 0; j < NJ; ++j) {
    x[j] = j < nj ? cm[j * 32 + lane] : -INFINITY;
    const float lo = fminf(m0, x[j]);
    m0 = fmaxf(m0, x[j]);
    m1 = fmaxf(m1, lo);
  }
  for (int j = NJ; j < nj; ++j) {              // S > 8192
    const float v = cm[j * 32 + lane];
    const float lo = fminf(m0, v);
    m0 = fmaxf(m0, v);
    m1 = fmaxf(m1, lo);
  }
  const float A = warp_sort_desc_f(m0), B = warp_sort_desc_f(m1);
  float c = -INFINITY;
  {
    const int i = lane;
    const float a = __shfl_sync(FULL, A, (i + 31) & 31);
    const float b = __shfl_sync(FULL, B, (k - 1 - i) & 31);
    if (i <= k - 1) c = fminf(i == 0 ? INFINITY : a, b);
  }
  const float ak = __shfl_sync(FULL, A, k - 1);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c = fmaxf(c, __shfl_xor_sync(FULL, c, o));
  const float theta = fmaxf(c, ak);
  // qualifying chunk ids (max >= theta) -> sm.hist, in chunk order
  uint32_t* qlist = sm.hist;
  int nq = 0;
  auto list_chunks = [&](float xm, int j) {
    const unsigned qm = __ballot_sync(FULL, xm >= theta);
    if (xm >= theta) {
      const int pos = nq + __popc(qm & ((1u << lane) - 1u));
      if (pos < 256) qlist[pos] = uint32_t(j * 32 + lane);
    }
    nq += __popc(qm);
  };
#pragma unroll
  for (int j = 0; j < NJ; ++j)
    if (j < nj) list_chunks(x[j], j);
  for (int j = NJ; j < nj; ++j) list_chunks(cm[j * 32 + lane], j);
  if (nq > 256) {           // heavy ties at theta: leave it to the exact fallback
    *count_out = kCandCap + 1;
    return false;
  }
  __syncwarp();
  // four chunks per warp load (lane: chunk l/8, scores 4(l%8)..+3), two loads in flight
  int count = 0;
  uint64_t* ckw = sm.cand;
  auto take = [&](float4 v, int ci) {
    const int base = ci < nq ? int(qlist[ci]) * 32 + (lane & 7) * 4 : 0;
    const float vs[4] = {v.x, v.y, v.z, v.w};
    uint32_t mk = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) mk |= (ci < nq && vs[q] >= theta ? 1u : 0u) << q;
    const int cnt = __popc(mk);
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += y;
    }
    int pos = count + incl - cnt;
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if ((mk >> q) & 1u) {
        if (pos < kCandCap) ckw[pos] = make_key(vs[q], uint32_t(base + q));
        ++pos;
      }
    count += __shfl_sync(FULL, incl, 31);
  };
  const float4 ninf = make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
  for (int g = 0; g < nq; g += 8) {
    const int ca = g + (lane >> 3), cb = g + 4 + (lane >> 3);
    const float4 va = ca < nq ? *reinterpret_cast<const float4*>(sr + qlist[ca] * 32 + (lane & 7) * 4) : ninf;
    const float4 vb = cb < nq ? *reinterpret_cast<const float4*>(sr + qlist[cb] * 32 + (lane & 7) * 4) : ninf;
    take(va, ca);
    if (g + 4 < nq) take(vb, cb);
  }
  *count_out = count;
  if (count > 64) return false;
  __syncwarp();
  uint64_t* ck = sm.cand;
  const bool h0 = lane < count, h1 = lane + 32 < count;
  const uint64_t k0 = h0 ? ck[lane] : ~0ull, k1 = h1 ? ck[lane + 32] : ~0ull;
  int r0 = 0, r1 = 0;
  if ((count & 1) != 0) ck[count] = 0ull;   // pad: ranks nothing
  __syncwarp();
  const int pairs = (count + 1) >> 1;
  for (int l = 0; l < pairs; ++l) {
    const ulonglong2 kk = reinterpret_cast<const ulonglong2*>(ck)[l];
    r0 += (kk.x > k0 ? 1 : 0) + (kk.y > k0 ? 1 : 0);
    r1 += (kk.x > k1 ? 1 : 0) + (kk.y > k1 ? 1 : 0);
  }
  if (h0 && r0 < k) { hI[row * k + r0] = int32_t(key_id(k0)); hs[row * k + r0] = key_score(k0); }
  if (h1 && r1 < k) { hI[row * k + r1] = int32_t(key_id(k1)); hs[row * k + r1] = key_score(k1); }
  return true;
}

// one warp per (t, h, half) row of S scores
__global__ void __launch_bounds__(256) half_topk_kernel(const float* scores, int64_t rows, int S,
                                                        int k, int32_t* hI, float* hs, QkNorm qn,
                                                        int H, const float* cmax) {
  __shared__ TopkSmem s_sm[8];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row = int64_t(blockIdx.x) * 8 + wid;
  if (row >= rows) return;
  TopkSmem& sm = s_sm[wid];
  const float* sr = scores + row * S;
  // qk-norm: s = (q.k) * inv|q| * inv|k| (scores stay raw tensor-core products)
  const float qi = qn.qinv ? qn.qinv[row] : 1.f;
  const float* ki = qn.qinv ? ((row & 1) ? qn.kinv2 : qn.kinv1) + int64_t((row >> 1) % H) * S : nullptr;
  auto score_at = [=](int e) { return ki ? (sr[e] * qi) * ki[e] : sr[e]; };
  if ((S % 128) == 0 && ki == nullptr && k <= 32) {
    int count = 0;
    if (cmax ? row_topk_chunks(sr, cmax + row * (S >> 5), S, k, sm, row, hI, hs, &count)
        : S > 1024 ? row_topk_stream(sr, S, k, sm, row, hI, hs, &count)
                 : (S == 1024 ? row_topk_fast<true>(sr, S, k, sm, row, hI, hs, &count)
                              : row_topk_fast<false>(sr, S, k, sm, row, hI, hs, &count)))
      return;
    uint64_t key;
    if (count <= kCandCap) {     // many ties: exact select over the survivors
      key = select_cand(count, k, sm);
    } else {
      auto gen = [=](int e) { return make_key(sr[e], uint32_t(e)); };
      key = warp_topk(gen, S, k, sm.hist, sm.sel);
    }
    if (lane < k) {
      hI[row * k + lane] = int32_t(key_id(key));
      hs[row * k + lane] = key_score(key);
    }
    return;
  }
  // phase 1: each lane's maximum (float compares; the first index of a tied
  // maximum is kept, which is the larger 64-bit key)
  float ms = -INFINITY;
  int mi = 0x7fffffff;
  const bool vec4 = (S % 128) == 0 && ki == nullptr;
  if (vec4) {     // lane owns 4 consecutive scores per 512-B round
    for (int e0 = lane * 4; e0 < S; e0 += 128) {
      const float4 v = *reinterpret_cast<const float4*>(sr + e0);
      if (v.x > ms) { ms = v.x; mi = e0; }
      if (v.y > ms) { ms = v.y; mi = e0 + 1; }
      if (v.z > ms) { ms = v.z; mi = e0 + 2; }
      if (v.w > ms) { ms = v.w; mi = e0 + 3; }
    }
  } else {
    for (int e = lane; e < S; e += 32) {
      const float v = score_at(e);
      if (v > ms) { ms = v; mi = e; }
    }
  }
  const uint64_t lane_key = mi == 0x7fffffff ? 0ull : make_key(ms, uint32_t(mi));
  const uint64_t theta = warp_theta_max(lane_key, k);
  const float ts = key_score(theta);
  const int ti = int(key_id(theta));
  // phase 3: survivors key >= theta <=> s > ts or (s == ts and e <= ti)
  int count = 0;
  if (vec4) {
    for (int e0 = 0; e0 < S; e0 += 128) {
      const int eb = e0 + lane * 4;
      const float4 v = *reinterpret_cast<const float4*>(sr + eb);
      const float vs[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int e = eb + c;
        const bool sel = vs[c] > ts || (vs[c] == ts && e <= ti);
        append_cand(sel ? make_key(vs[c], uint32_t(e)) : 0ull, sel, count, sm);
      }
    }
  } else {
    for (int e0 = 0; e0 < S; e0 += 32) {
      const int e = e0 + lane;
      const float v = e < S ? score_at(e) : -INFINITY;
      const bool sel = e < S && (v > ts || (v == ts && e <= ti));
      append_cand(sel ? make_key(v, uint32_t(e)) : 0ull, sel, count, sm);
    }
  }
  uint64_t key;
  if (count <= kCandCap) {
    key = select_cand(count, k, sm);
  } else {  // pathological ties: exact select over the whole row
    auto gen = [=](int e) { return make_key(score_at(e), uint32_t(e)); };
    key = warp_topk(gen, S, k, sm.hist, sm.sel);
  }
  if (lane < k) {
    hI[row * k + lane] = int32_t(key_id(key));
    hs[row * k + lane] = key_score(key);
  }
}

// Top-32 (descending, one per lane) of the union of two descending lists
// a, b held one per lane: the elementwise max of a and reversed b is bitonic
// and holds the 32 largest; a 5-stage half-cleaner network sorts it.
__device__ __forceinline__ float merge_top_desc(float a, float b) {
  const int lane = threadIdx.x & 31;
  float x = fmaxf(a, __shfl_sync(FULL, b, 31 - lane));
#pragma unroll
  for (int stride = 16; stride > 0; stride >>= 1) {
    const float y = __shfl_xor_sync(FULL, x, stride);
    x = ((lane & stride) == 0) ? fmaxf(x, y) : fminf(x, y);
  }
  return x;
}

// Fast exact combine for k <= 32 using the sortedness of the grid
// c[i][j] = s1[i] + s2[j] (s1, s2 descending, fp32 addition is monotone):
//  theta = the k-th largest value of rows 0..15 (a merge tree of the sorted
//  rows) bounds the k-th largest cell from below; in every column the cells
//  >= theta are a prefix; their keys (score, flat index) are ranked by
//  counting and ranks < k written out.  Returns false (nothing written) when
//  more than 64 cells survive.
__device__ __forceinline__ bool combine_fast(const float* s1p, const int32_t* i1p, float s2,
                                             uint32_t i2, int S, int k, uint64_t* cand,
                                             uint64_t* sel, int64_t th, int32_t* idx, float* w,
                                             float* score) {
  const int lane = threadIdx.x & 31;
  constexpr int R = 16;
  float L[R];
#pragma unroll
  for (int r = 0; r < R; ++r) L[r] = (lane < k && r < k) ? s1p[r] + s2 : -INFINITY;
#pragma unroll
  for (int n = R; n > 2; n >>= 1) {
#pragma unroll
    for (int r = 0; r < n / 2; ++r) L[r] = merge_top_desc(L[2 * r], L[2 * r + 1]);
  }
  // k-th largest of L[0] u L[1] (descending): max over i = 0..k of min(A[i-1], B[k-1-i])
  float c = -INFINITY;
  {
    const float a = __shfl_sync(FULL, L[0], (lane + 31) & 31);
    const float b = __shfl_sync(FULL, L[1], (k - 1 - lane) & 31);
    if (lane <= k - 1) c = fminf(lane == 0 ? INFINITY : a, b);
  }
  const float ak = __shfl_sync(FULL, L[0], k - 1);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c = fmaxf(c, __shfl_xor_sync(FULL, c, o));
  const float theta = fmaxf(c, ak);
  // column prefix of survivors
  int n = 0;
  if (lane < k)
    while (n < k && s1p[n] + s2 >= theta) ++n;
  int incl = n;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(FULL, incl, o);
    if (lane >= o) incl += y;
  }
  const int count = __shfl_sync(FULL, incl, 31);
  if (count > 64) return false;
  int pos = incl - n;
  for (int i = 0; i < n; ++i)
    cand[pos + i] = make_key(s1p[i] + s2, uint32_t(i1p[i]) * uint32_t(S) + i2);
  if ((count & 1) != 0) cand[count] = 0ull;   // pad: ranks nothing
  __syncwarp();
  const bool h0 = lane < count, h1 = lane + 32 < count;
  const uint64_t k0 = h0 ? cand[lane] : ~0ull, k1 = h1 ? cand[lane + 32] : ~0ull;
  int r0 = 0, r1 = 0;
  const int pairs = (count + 1) >> 1;   // two survivors per shared-memory load
  if (count <= 32) {
    for (int l = 0; l < pairs; ++l) {
      const ulonglong2 kk = reinterpret_cast<const ulonglong2*>(cand)[l];
      r0 += (kk.x > k0 ? 1 : 0) + (kk.y > k0 ? 1 : 0);
    }
  } else {
    for (int l = 0; l < pairs; ++l) {
      const ulonglong2 kk = reinterpret_cast<const ulonglong2*>(cand)[l];
      r0 += (kk.x > k0 ? 1 : 0) + (kk.y > k0 ? 1 : 0);
      r1 += (kk.x > k1 ? 1 : 0) + (kk.y > k1 ? 1 : 0);
    }
  }
  if (h0 && r0 < k) sel[r0] = k0;
  if (h1 && r1 < k) sel[r1] = k1;
  __syncwarp();
  const uint64_t key = lane < k ? sel[lane] : 0ull;
  const float sc = key_score(key);
  const float m = __shfl_sync(FULL, sc, 0);
  const float ex = lane < k ? expf(sc - m) : 0.f;
  float sum = ex;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(FULL, sum, o);
  if (lane < k) {
    idx[th * k + lane] = int32_t(key_id(key));
    w[th * k + lane] = ex / sum;
    if (score) score[th * k + lane] = sc;
  }
  return true;
}

// The combine of one (t, h) given its two half lists: s1/i1 (descending, in
// this warp's shared memory) and this lane's entry of the second list
// (lane j < k: s2[j], i2[j]); k*k Cartesian sums, exact top-k, softmax.
__device__ __forceinline__ void combine_lists(float* s1p, int32_t* i1p, float* s2p, int32_t* i2p,
                                              float s2, uint32_t i2, int S, int k, TopkSmem& sm,
                                              int64_t th, int32_t* idx, float* w, float* score) {
  const int lane = threadIdx.x & 31;
  // lane j owns column j of the k x k grid: c[i][j] = s1[i] + s2[j]
  if (combine_fast(s1p, i1p, s2, i2, S, k, sm.cand, sm.sel, th, idx, w, score)) return;
  __syncwarp();
  auto key_of = [&](int i) {
    return make_key(s1p[i] + s2, uint32_t(i1p[i]) * uint32_t(S) + i2);
  };
  uint64_t t0 = 0, t1 = 0, t2 = 0, t3 = 0;
  if (lane < k)
    for (int i = 0; i < k; ++i) insert4(key_of(i), t0, t1, t2, t3);
  const uint64_t theta = warp_theta(t0, t1, t2, t3, k, sm);
  int count = 0;
  for (int i = 0; i < k; ++i) {
    uint64_t key = 0;
    if (lane < k) key = key_of(i);
    append_cand(key, lane < k && key >= theta, count, sm);
  }
  uint64_t key;
  if (count <= kCandCap) {
    key = select_cand(count, k, sm);
  } else {
    s2p[lane] = s2;
    i2p[lane] = int32_t(i2);
    __syncwarp();
    auto gen = [=](int e) {
      const int i = e / k, j = e - (e / k) * k;
      return make_key(s1p[i] + s2p[j], uint32_t(i1p[i]) * uint32_t(S) + uint32_t(i2p[j]));
    };
    key = warp_topk(gen, k * k, k, sm.hist, sm.sel);
  }
  const float sc = key_score(key);
  const float m = __shfl_sync(FULL, sc, 0);
  float ex = lane < k ? expf(sc - m) : 0.f;
  float sum = ex;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(FULL, sum, o);
  if (lane < k) {
    idx[th * k + lane] = int32_t(key_id(key));
    w[th * k + lane] = ex / sum;
    if (score) score[th * k + lane] = sc;
  }
}

// one warp per (t, h): combine the two half lists (k*k Cartesian sums), softmax
__global__ void __launch_bounds__(256) combine_kernel(const int32_t* hI, const float* hs,
                                                      int64_t TH, int S, int k, int32_t* idx,
                                                      float* w, float* score) {
  __shared__ TopkSmem s_sm[8];
  __shared__ float s_s1[8][32], s_s2[8][32];
  __shared__ int32_t s_i1[8][32], s_i2[8][32];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t th = int64_t(blockIdx.x) * 8 + wid;
  if (th >= TH) return;
  float s2 = 0.f;
  uint32_t i2 = 0;
  if (lane < k) {
    s_s1[wid][lane] = hs[(th * 2 + 0) * k + lane];
    s_i1[wid][lane] = hI[(th * 2 + 0) * k + lane];
    s2 = hs[(th * 2 + 1) * k + lane];
    i2 = uint32_t(hI[(th * 2 + 1) * k + lane]);
  }
  __syncwarp();
  combine_lists(s_s1[wid], s_i1[wid], s_s2[wid], s_i2[wid], s2, i2, S, k, s_sm[wid], th, idx, w,
                score);
}

// The k best (descending) of a row's n <= 96 unique candidate keys, by
// counting ranks: lane j < k returns the j-th largest.
__device__ __forceinline__ uint64_t cand_topk(const uint64_t* keys, int n, int k, TopkSmem& sm) {
  const int lane = threadIdx.x & 31;
  uint64_t* c = sm.cand;
  for (int e = lane; e < n; e += 32) c[e] = keys[e];
  if ((n & 1) != 0 && lane == 0) c[n] = 0ull;    // pad: ranks nothing
  __syncwarp();
  uint64_t mk[3];
  int rk[3] = {0, 0, 0};
#pragma unroll
  for (int r = 0; r < 3; ++r) mk[r] = (lane + 32 * r < n) ? c[lane + 32 * r] : ~0ull;
  const int pairs = (n + 1) >> 1;
  for (int l = 0; l < pairs; ++l) {
    const ulonglong2 kk = reinterpret_cast<const ulonglong2*>(c)[l];
#pragma unroll
    for (int r = 0; r < 3; ++r) rk[r] += (kk.x > mk[r] ? 1 : 0) + (kk.y > mk[r] ? 1 : 0);
  }
#pragma unroll
  for (int r = 0; r < 3; ++r)
    if (lane + 32 * r < n && rk[r] < k) sm.sel[rk[r]] = mk[r];
  __syncwarp();
  const uint64_t key = lane < k ? sm.sel[lane] : 0ull;
  __syncwarp();
  return key;
}

// one warp per (t, h): exact half top-k of each half row's candidates (the
// fused scoring kernel's lists), then the combine + softmax
__global__ void __launch_bounds__(256) combine_cand_kernel(const uint64_t* cand, const int32_t* cnt,
                                                           int cap, int64_t TH, int S, int k,
                                                           int32_t* idx, float* w, float* score) {
  __shared__ TopkSmem s_sm[8];
  __shared__ float s_s1[8][32], s_s2[8][32];
  __shared__ int32_t s_i1[8][32], s_i2[8][32];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t th = int64_t(blockIdx.x) * 8 + wid;
  if (th >= TH) return;
  TopkSmem& sm = s_sm[wid];
  const int n1 = cnt[th * 2 + 0], n2 = cnt[th * 2 + 1];
  const uint64_t k1 = cand_topk(cand + (th * 2 + 0) * cap, n1, k, sm);
  const uint64_t k2 = cand_topk(cand + (th * 2 + 1) * cap, n2, k, sm);
  if (lane < k) {
    s_s1[wid][lane] = key_score(k1);
    s_i1[wid][lane] = int32_t(key_id(k1));
  }
  __syncwarp();
  combine_lists(s_s1[wid], s_i1[wid], s_s2[wid], s_i2[wid], lane < k ? key_score(k2) : 0.f,
                lane < k ? key_id(k2) : 0u, S, k, sm, th, idx, w, score);
}

// Exact fallback for rows whose candidate list overflowed (heavy ties): one
// warp recomputes the row's S scores (fp32 FMA over the bf16 inputs) into
// shared memory and selects its k best with the radix select.
__global__ void __launch_bounds__(32) cand_fallback_kernel(const __nv_bfloat16* q,
                                                           const __nv_bfloat16* K1,
                                                           const __nv_bfloat16* K2, int H, int S,
                                                           int Dk, int k, uint64_t* cand,
                                                           int32_t* cnt, int cap,
                                                           const int32_t* fail_rows,
                                                           const int32_t* fail_n) {
  extern __shared__ float s_row[];      // [S]
  __shared__ TopkSmem sm;
  const int lane = threadIdx.x & 31;
  const int Dh = Dk / 2;
  const int nf = *fail_n;
  for (int f = blockIdx.x; f < nf; f += gridDim.x) {
    const int64_t row = fail_rows[f];
    const int64_t th = row >> 1;
    const int half = int(row & 1);
    const int h = int(th % H);
    const __nv_bfloat16* qh = q + th * Dk + half * Dh;
    const __nv_bfloat16* K = (half ? K2 : K1) + int64_t(h) * S * Dh;
    for (int a = 0; a < S; ++a) {
      float part = 0.f;
      for (int i = lane; i < Dh; i += 32)
        part = fmaf(__bfloat162float(qh[i]), __bfloat162float(K[int64_t(a) * Dh + i]), part);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(FULL, part, o);
      if (lane == 0) s_row[a] = part;
    }
    __syncwarp();
    auto gen = [](int e) { return make_key(s_row[e], uint32_t(e)); };
    const uint64_t key = warp_topk(gen, S, k, sm.hist, sm.sel);
    if (lane < k) cand[row * cap + lane] = key;
    if (lane == 0) cnt[row] = k;
    __syncwarp();
  }
}

// bound[0] = max_o |dw_o| (dw = sum of the ns partials), bound[3] = max_o |w_o|
// over the P = T*H*k positions (elementwise, coalesced; one atomic per block)
__global__ void __launch_bounds__(256) ds_bound_kernel(const float* __restrict__ w,
                                                       const float* __restrict__ dw_part, int ns,
                                                       int64_t sstride, int64_t P, float* bound) {
  float mdw = 0.f, mw = 0.f;
  for (int64_t o = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; o < P;
       o += int64_t(gridDim.x) * blockDim.x) {
    float dwv = 0.f;
    for (int s = 0; s < ns; ++s) dwv += dw_part[int64_t(s) * sstride + o];
    mdw = fmaxf(mdw, fabsf(dwv));
    mw = fmaxf(mw, fabsf(w[o]));
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    mdw = fmaxf(mdw, __shfl_xor_sync(FULL, mdw, off));
    mw = fmaxf(mw, __shfl_xor_sync(FULL, mw, off));
  }
  __shared__ float s_m[2][8];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    s_m[0][wid] = mdw;
    s_m[1][wid] = mw;
  }
  __syncthreads();
  if (threadIdx.x == 0) {      // values >= 0 order as ints
    for (int i = 1; i < 8; ++i) {
      mdw = fmaxf(mdw, s_m[0][i]);
      mw = fmaxf(mw, s_m[1][i]);
    }
    atomicMax(reinterpret_cast<int*>(bound), __float_as_int(mdw));
    atomicMax(reinterpret_cast<int*>(bound + 3), __float_as_int(mw));
  }
}

// one warp per (t, h)
__global__ void __launch_bounds__(256) softmax_bwd_kernel(const int32_t* idx, const float* w,
                                                          const float* dw_part, int ns,
                                                          int64_t sstride, int64_t TH, int H,
                                                          int S, int k, float* ds, int32_t* key1,
                                                          int32_t* key2, __nv_bfloat16* ds_dense,
                                                          QkNorm qn, float* ds1w, float* ds2w,
                                                          int full_rows, __nv_bfloat16* ds_lo,
                                                          const float* f16_bound) {
  __shared__ int s_sub[8][2][32];
  __shared__ float s_ds[8][32];
  __shared__ float s_sc[8][2][32];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t th = int64_t(blockIdx.x) * 8 + wid;
  if (th >= TH) return;
  const int h = int(th % H);
  const int64_t o = th * k + lane;
  float wv = 0.f, dwv = 0.f;
  int32_t ix = 0;
  if (lane < k) {
    wv = w[o];
    ix = idx[o];
    for (int s = 0; s < ns; ++s) dwv += dw_part[int64_t(s) * sstride + o];
  }
  float dot = wv * dwv;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) dot += __shfl_xor_sync(FULL, dot, off);
  const float dsv = wv * (dwv - dot);
  // qk-norm: the half scores were (q_half.k) * inv_q * inv_k, so the raw
  // products receive ds * inv_q * inv_k (projection done after the GEMMs)
  float sc1 = 1.f, sc2 = 1.f;
  if (qn.qinv && lane < k) {
    sc1 = qn.qinv[th * 2 + 0] * qn.kinv1[int64_t(h) * S + ix / S];
    sc2 = qn.qinv[th * 2 + 1] * qn.kinv2[int64_t(h) * S + ix % S];
  }
  if (lane < k) ds[o] = dsv;
  if (!ds_dense) {
    // sparse form: per half, the lanes selecting the same sub-key are summed
    // by the lowest one (lane order: deterministic); the others get the
    // sentinel key H*S and weight 0 (sorted last, skipped by the reduction)
    const int sub1 = lane < k ? ix / S : -1 - lane, sub2 = lane < k ? ix % S : -1 - lane;
    const float v1 = dsv * sc1, v2 = dsv * sc2;
    const unsigned g1 = __match_any_sync(FULL, sub1), g2 = __match_any_sync(FULL, sub2);
    float s1 = 0.f, s2 = 0.f;
    for (unsigned m = g1; m; m &= m - 1) s1 += __shfl_sync(g1, v1, __ffs(m) - 1);
    for (unsigned m = g2; m; m &= m - 1) s2 += __shfl_sync(g2, v2, __ffs(m) - 1);
    const bool l1 = (__ffs(g1) - 1) == lane, l2 = (__ffs(g2) - 1) == lane;
    if (lane < k) {
      key1[o] = l1 ? h * S + sub1 : H * S;
      key2[o] = l2 ? h * S + sub2 : H * S;
      ds1w[o] = l1 ? s1 : 0.f;
      ds2w[o] = l2 ? s2 : 0.f;
    }
  }
  if (ds_dense) {
    // dense half-key gradients of this (t, h); a sub-key selected by several
    // of the k pairs is summed in lane order (deterministic, no atomics).
    // full_rows: the two rows [2][S] are assembled in shared memory (zeros
    // included) and written with coalesced 16-byte stores, so ds_dense needs
    // no separate memset; otherwise the sums are scattered into a zeroed matrix.
    s_sub[wid][0][lane] = lane < k ? ix / S : -1;
    s_sub[wid][1][lane] = lane < k ? ix % S : -1;
    s_ds[wid][lane] = dsv;
    s_sc[wid][0][lane] = sc1;
    s_sc[wid][1][lane] = sc2;
    extern __shared__ __align__(16) __nv_bfloat16 s_rows[];   // [8 warps][2][S] when full_rows
    __nv_bfloat16* rows = s_rows + int64_t(wid) * 2 * S;
    // split form (ds_lo != NULL, full rows only): ds = hi + lo, both bf16,
    // hi = RN(ds), lo = RN(ds - hi): the pair carries ~16 significant bits
    __nv_bfloat16* rows_lo = s_rows + int64_t(8 + wid) * 2 * S;
    if (full_rows) {
      const uint4 z = make_uint4(0, 0, 0, 0);
      for (int c = lane; c < (2 * S) / 8; c += 32) reinterpret_cast<uint4*>(rows)[c] = z;
      if (ds_lo)
        for (int c = lane; c < (2 * S) / 8; c += 32) reinterpret_cast<uint4*>(rows_lo)[c] = z;
    }
    __syncwarp();
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const int a = s_sub[wid][half][lane];
      // lanes selecting the same sub-key: the lowest one sums the group in lane order
      const unsigned grp = __match_any_sync(FULL, a);
      const bool leader = lane < k && (__ffs(grp) - 1) == lane;
      float sum = 0.f;
      if (leader) {
        for (unsigned m = grp; m; m &= m - 1) {
          const int l = __ffs(m) - 1;
          sum += s_ds[wid][l] * s_sc[wid][half][l];
        }
      }
      if (leader) {
        // fp16 form (f16_bound, full rows only): fp16(ds * 2^e) in the same
        // 2-byte slots, read by the mixed-type MMA (pkm_tc_bwd.cu)
        const __nv_bfloat16 hi = f16_bound
            ? __ushort_as_bfloat16(__half_as_ushort(__float2half_rn(ldexpf(sum, ds_f16_exp_ds(f16_bound, k)))))
            : __float2bfloat16_rn(sum);
        if (full_rows) {
          rows[half * S + a] = hi;
          if (ds_lo) rows_lo[half * S + a] = __float2bfloat16_rn(sum - __bfloat162float(hi));
        } else {
          ds_dense[(th * 2 + half) * S + a] = hi;
        }
      }
    }
    if (full_rows) {
      __syncwarp();
      uint4* dst = reinterpret_cast<uint4*>(ds_dense + th * 2 * S);
      for (int c = lane; c < (2 * S) / 8; c += 32) dst[c] = reinterpret_cast<const uint4*>(rows)[c];
      if (ds_lo) {
        uint4* dl = reinterpret_cast<uint4*>(ds_lo + th * 2 * S);
        for (int c = lane; c < (2 * S) / 8; c += 32) dl[c] = reinterpret_cast<const uint4*>(rows_lo)[c];
      }
    }
  }
}

// dq[t, h, half] = sum over the distinct selected sub-keys a of
// ds_half[t,h,a] * K_half[h, a, :] (the deduplicated slots of softmax_bwd:
// sentinel slots skipped), one warp per (t, h), fp32 accumulation in slot
// order.  Lane l owns the 16-byte column vectors l, l + 32, ... (NV of them);
// 8 key rows are loaded per batch (8 * NV vectors in flight per lane).
template <typename T, int NV>
__global__ void __launch_bounds__(256) pkm_dq_kernel(const int32_t* key1, const int32_t* key2,
                                                     const float* ds1, const float* ds2,
                                                     const T* K1, const T* K2, int64_t TH, int HS,
                                                     int Dh, int k, float* dq) {
  constexpr int VEC = Vec<T>::N;
  constexpr int BATCH = 8;
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t th = int64_t(blockIdx.x) * 8 + wid;
  if (th >= TH) return;
  const int nv = Dh / VEC;                 // 16-byte vectors per key row
#pragma unroll 1
  for (int half = 0; half < 2; ++half) {
    const int32_t* key = half ? key2 : key1;
    const float* dsw = half ? ds2 : ds1;
    const T* K = half ? K2 : K1;
    int32_t kk = HS;
    float wv = 0.f;
    if (lane < k) {
      kk = key[th * k + lane];
      wv = dsw[th * k + lane];
    }
    unsigned m = __ballot_sync(FULL, kk < HS);
    float acc[NV][VEC];
#pragma unroll
    for (int c = 0; c < NV; ++c)
#pragma unroll
      for (int e = 0; e < VEC; ++e) acc[c][e] = 0.f;
    while (m) {
      int32_t row[BATCH];
      float wg[BATCH];
      int n = 0;
#pragma unroll
      for (int u = 0; u < BATCH; ++u) {
        const int src = m ? __ffs(m) - 1 : 0;
        row[u] = __shfl_sync(FULL, kk, src);
        wg[u] = __shfl_sync(FULL, wv, src);
        if (m) { m &= m - 1; ++n; }
      }
      uint4 raw[BATCH][NV];
#pragma unroll
      for (int u = 0; u < BATCH; ++u)
#pragma unroll
        for (int c = 0; c < NV; ++c) {
          const int v = lane + 32 * c;
          raw[u][c] = (u < n && v < nv) ? ldg_nc_v4(K + int64_t(row[u]) * Dh + int64_t(v) * VEC)
                                        : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
      for (int u = 0; u < BATCH; ++u) {
        if (u >= n) break;
#pragma unroll
        for (int c = 0; c < NV; ++c) {
          float f[VEC];
          Vec<T>::load(raw[u][c], f);
#pragma unroll
          for (int e = 0; e < VEC; ++e) acc[c][e] = fmaf(wg[u], f[e], acc[c][e]);
        }
      }
    }
    float* out = dq + (th * 2 + half) * int64_t(Dh);
#pragma unroll
    for (int c = 0; c < NV; ++c) {
      const int v = lane + 32 * c;
      if (v >= nv) continue;
      float4* o4 = reinterpret_cast<float4*>(out + int64_t(v) * VEC);
#pragma unroll
      for (int e = 0; e < VEC; e += 4)
        o4[e / 4] = make_float4(acc[c][e], acc[c][e + 1], acc[c][e + 2], acc[c][e + 3]);
    }
  }
}

}  // namespace

bool half_topk_chunked(const mlPkmShape& sh) {
  static int off = -1;
  if (off < 0) {
    const char* e = std::getenv("ML_TOPK_CHUNKS");
    off = (e && e[0] == '0') ? 1 : 0;
  }
  return !off && pkm_scores_tc_eligible(sh) && !sh.qk_norm && sh.S >= 2048 && sh.S % 1024 == 0 &&
         sh.k <= 32;
}

mlStatus launch_pkm_scores(const mlPkmShape& sh, const void* q, const void* K1, const void* K2,
                           float* scores, cudaStream_t s, float* cmax) {
  if (sh.T <= 0) return ML_OK;
  if (pkm_scores_tc_eligible(sh)) return launch_pkm_scores_tc(sh, q, K1, K2, scores, s, cmax);
  if (cmax) return fail(ML_ERR_UNSUPPORTED, "chunk maxima need the tcgen05 scoring path");
  dim3 grid{unsigned((sh.T + 63) / 64), unsigned((sh.S + 63) / 64), unsigned(sh.H * 2)};
  if (sh.dtype == ML_BF16)
    pkm_scores_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>(
        static_cast<const __nv_bfloat16*>(q), static_cast<const __nv_bfloat16*>(K1),
        static_cast<const __nv_bfloat16*>(K2), scores, sh.T, sh.H, sh.S, sh.Dk);
  else
    pkm_scores_kernel<float><<<grid, 256, 0, s>>>(static_cast<const float*>(q),
                                                  static_cast<const float*>(K1),
                                                  static_cast<const float*>(K2), scores, sh.T,
                                                  sh.H, sh.S, sh.Dk);
  ML_LAUNCH_CHECK("pkm_scores_simt");
  return ML_OK;
}

mlStatus launch_half_topk(const mlPkmShape& sh, const float* scores, int32_t* hI, float* hs,
                          const QkNorm& qn, cudaStream_t s, const float* cmax) {
  const int64_t rows = int64_t(sh.T) * sh.H * 2;
  if (rows <= 0) return ML_OK;
  half_topk_kernel<<<unsigned((rows + 7) / 8), 256, 0, s>>>(scores, rows, sh.S, sh.k, hI, hs, qn,
                                                            sh.H, cmax);
  ML_LAUNCH_CHECK("half_topk");
  return ML_OK;
}

mlStatus launch_combine_softmax(const mlPkmShape& sh, const int32_t* hI, const float* hs,
                                int32_t* idx, float* w, float* score, cudaStream_t s) {
  const int64_t TH = int64_t(sh.T) * sh.H;
  if (TH <= 0) return ML_OK;
  combine_kernel<<<unsigned((TH + 7) / 8), 256, 0, s>>>(hI, hs, TH, sh.S, sh.k, idx, w, score);
  ML_LAUNCH_CHECK("combine_softmax");
  return ML_OK;
}

mlStatus launch_cand_fallback(const mlPkmShape& sh, const void* q, const void* K1, const void* K2,
                              uint64_t* cand, int32_t* cnt, const int32_t* fail_rows,
                              const int32_t* fail_n, cudaStream_t s) {
  const size_t smem = size_t(sh.S) * sizeof(float);
  static bool attr = false;
  if (!attr) {
    ML_CUDA_TRY(cudaFuncSetAttribute(cand_fallback_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(16384 * sizeof(float))));
    attr = true;
  }
  if (sh.S > 16384) return fail(ML_ERR_UNSUPPORTED, "cand_fallback: S > 16384");
  cand_fallback_kernel<<<unsigned(num_sms() * 4), 32, smem, s>>>(
      static_cast<const __nv_bfloat16*>(q), static_cast<const __nv_bfloat16*>(K1),
      static_cast<const __nv_bfloat16*>(K2), sh.H, sh.S, sh.Dk, sh.k, cand, cnt,
      pkm_select_cap(), fail_rows, fail_n);
  ML_LAUNCH_CHECK("pkm_cand_fallback");
  return ML_OK;
}

mlStatus launch_combine_cand(const mlPkmShape& sh, const uint64_t* cand, const int32_t* cnt,
                             int32_t* idx, float* w, float* score, cudaStream_t s) {
  const int64_t TH = int64_t(sh.T) * sh.H;
  if (TH <= 0) return ML_OK;
  combine_cand_kernel<<<unsigned((TH + 7) / 8), 256, 0, s>>>(cand, cnt, pkm_select_cap(), TH, sh.S,
                                                             sh.k, idx, w, score);
  ML_LAUNCH_CHECK("combine_softmax");
  return ML_OK;
}

bool softmax_bwd_full_rows(const mlPkmShape& sh) { return sh.S % 8 == 0 && sh.S <= 2048; }

mlStatus launch_softmax_bwd(const mlPkmShape& sh, const int32_t* idx, const float* w,
                            const float* dw_part, int nslices, int64_t slice_stride, float* ds,
                            int32_t* key1, int32_t* key2, __nv_bfloat16* ds_dense,
                            const QkNorm& qn, float* ds1w, float* ds2w, cudaStream_t s,
                            __nv_bfloat16* ds_lo, const float* f16_bound) {
  const int64_t TH = int64_t(sh.T) * sh.H;
  if (TH <= 0) return ML_OK;
  const bool full = ds_dense && softmax_bwd_full_rows(sh);
  if (ds_lo && !full) return fail(ML_ERR_UNSUPPORTED, "softmax_bwd: the split ds needs full rows");
  if (f16_bound && (!full || ds_lo || qn.qinv))
    return fail(ML_ERR_UNSUPPORTED, "softmax_bwd: the fp16 ds needs full rows, no split, no qk-norm");
  const size_t smem = full ? size_t(ds_lo ? 16 : 8) * 2 * sh.S * sizeof(__nv_bfloat16) : 0;
  static bool attr = false;
  if (full && !attr) {
    ML_CUDA_TRY(cudaFuncSetAttribute(softmax_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(16 * 2 * 2048 * sizeof(__nv_bfloat16))));
    attr = true;
  }
  softmax_bwd_kernel<<<unsigned((TH + 7) / 8), 256, smem, s>>>(
      idx, w, dw_part, nslices, slice_stride, TH, sh.H, sh.S, sh.k, ds, key1, key2, ds_dense, qn,
      ds1w, ds2w, full ? 1 : 0, ds_lo, f16_bound);
  ML_LAUNCH_CHECK("softmax_bwd");
  return ML_OK;
}

mlStatus launch_ds_bound(const mlPkmShape& sh, const float* w, const float* dw_part, int nslices,
                         int64_t slice_stride, float* bound, cudaStream_t s) {
  const int64_t P = int64_t(sh.T) * sh.H * sh.k;
  ML_CUDA_TRY(cudaMemsetAsync(bound, 0, sizeof(float), s));
  ML_CUDA_TRY(cudaMemsetAsync(bound + 3, 0, sizeof(float), s));
  if (P <= 0) return ML_OK;
  const unsigned grid = unsigned(std::min<int64_t>((P + 255) / 256, int64_t(num_sms()) * 8));
  ds_bound_kernel<<<grid, 256, 0, s>>>(w, dw_part, nslices, slice_stride, P, bound);
  ML_LAUNCH_CHECK("ds_bound");
  return ML_OK;
}

}  // namespace ml

namespace ml {
mlStatus launch_pkm_dq(const mlPkmShape& sh, const int32_t* key1, const int32_t* key2,
                       const float* ds1, const float* ds2, const void* K1, const void* K2,
                       float* dq, cudaStream_t s) {
  const int64_t TH = int64_t(sh.T) * sh.H;
  if (TH <= 0) return ML_OK;
  const int Dh = sh.Dk / 2;
  const int HS = sh.H * sh.S;
  const unsigned grid = unsigned((TH + 7) / 8);
  if (sh.dtype == ML_BF16) {
    const auto* k1 = static_cast<const __nv_bfloat16*>(K1);
    const auto* k2 = static_cast<const __nv_bfloat16*>(K2);
    const int nvl = (Dh / 8 + 31) / 32;
    if (nvl <= 1) pkm_dq_kernel<__nv_bfloat16, 1><<<grid, 256, 0, s>>>(key1, key2, ds1, ds2, k1, k2, TH, HS, Dh, sh.k, dq);
    else if (nvl <= 2) pkm_dq_kernel<__nv_bfloat16, 2><<<grid, 256, 0, s>>>(key1, key2, ds1, ds2, k1, k2, TH, HS, Dh, sh.k, dq);
    else if (nvl <= 4) pkm_dq_kernel<__nv_bfloat16, 4><<<grid, 256, 0, s>>>(key1, key2, ds1, ds2, k1, k2, TH, HS, Dh, sh.k, dq);
    else return fail(ML_ERR_UNSUPPORTED, "pkm_dq: Dk/2 > 1024");
  } else {
    const auto* k1 = static_cast<const float*>(K1);
    const auto* k2 = static_cast<const float*>(K2);
    const int nvl = (Dh / 4 + 31) / 32;
    if (nvl <= 1) pkm_dq_kernel<float, 1><<<grid, 256, 0, s>>>(key1, key2, ds1, ds2, k1, k2, TH, HS, Dh, sh.k, dq);
    else if (nvl <= 2) pkm_dq_kernel<float, 2><<<grid, 256, 0, s>>>(key1, key2, ds1, ds2, k1, k2, TH, HS, Dh, sh.k, dq);
    else if (nvl <= 4) pkm_dq_kernel<float, 4><<<grid, 256, 0, s>>>(key1, key2, ds1, ds2, k1, k2, TH, HS, Dh, sh.k, dq);
    else return fail(ML_ERR_UNSUPPORTED, "pkm_dq: Dk/2 > 512 (fp32)");
  }
  ML_LAUNCH_CHECK("pkm_dq");
  return ML_OK;
}
}  // namespace ml
