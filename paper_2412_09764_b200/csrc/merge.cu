// The memory group's inverse index map, built once per group instead of
// once per rank (every rank of the group
// looks up ALL G*T_loc gathered tokens in its [N, dv/G] slice, so every rank
// needs the same sorted (row, position) map of all of them).
//
// Each rank stably sorts only its own T_loc*B positions by value row
// (sort_pairs) and tags them with their global position (rank*P_loc + p);
// the G sorted lists are all-gathered and merged here.  Because list g holds
// exactly the positions [g*P_loc, (g+1)*P_loc), merging with ties going to
// the left list gives the stable sort of all G*P_loc positions -- the very
// array one sort of the gathered indices produces (bit-identical state).
//
// Merge path: each 2048-output tile finds its split of the two inputs by a
// binary search on its first output's diagonal (A[i] goes before B[j] iff
// A[i] <= B[j]), stages the two input runs in shared memory, and each thread
// merges 8 consecutive outputs from its own diagonal.
#include "internal.cuh"

#include <algorithm>
#include <vector>

namespace ml {
namespace {

constexpr int kMergeThreads = 256;
constexpr int kMergeItems = 8;
constexpr int kMergeTile = kMergeThreads * kMergeItems;
constexpr int kMaxPairs = 32;

// number of A elements among the first d outputs (ties to A): the first i
// with NOT (a[i] <= b[d-i-1]), by a 32-ary search (one warp, ~5 dependent
// rounds of loads instead of ~21)
__device__ __forceinline__ int64_t co_rank_warp(const int32_t* a, int64_t na, const int32_t* b,
                                                int64_t nb, int64_t d, int lane) {
  int64_t lo = d > nb ? d - nb : 0, hi = d < na ? d : na;
  while (hi - lo > 32) {
    const int64_t step = (hi - lo + 31) >> 5;
    const int64_t m = lo + lane * step;
    const bool pred = m < hi && a[m] <= b[d - m - 1];
    const int c = __popc(__ballot_sync(0xffffffffu, pred));
    const int64_t nlo = c ? lo + (c - 1) * step + 1 : lo;
    const int64_t nhi = lo + c * step < hi ? lo + c * step : hi;
    lo = nlo;
    hi = nhi;
  }
  const int64_t m = lo + lane;
  const bool pred = m < hi && a[m] <= b[d - m - 1];
  return lo + __popc(__ballot_sync(0xffffffffu, pred));
}

// one merge round: pair p merges (a, b) into out; tiles of all pairs in one grid
struct MergePair { const int32_t* ka; const int32_t* pa; const int32_t* kb; const int32_t* pb;
                   int32_t* ko; int32_t* po; int64_t na, nb; int64_t first_tile; };
struct MergeRound { MergePair p[kMaxPairs]; int npairs; };

__global__ void __launch_bounds__(kMergeThreads) merge_round_kernel(const __grid_constant__ MergeRound R) {
  __shared__ int32_t sk[kMergeTile], sp[kMergeTile], ok[kMergeTile], op[kMergeTile];
  __shared__ int64_t s_i[2];
  int pi = 0;
  while (pi + 1 < R.npairs && int64_t(blockIdx.x) >= R.p[pi + 1].first_tile) ++pi;
  const MergePair& P = R.p[pi];
  const int64_t n = P.na + P.nb;
  const int64_t d0 = (int64_t(blockIdx.x) - P.first_tile) * kMergeTile;
  const int64_t d1 = d0 + kMergeTile < n ? d0 + kMergeTile : n;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp < 2) {
    const int64_t i = co_rank_warp(P.ka, P.na, P.kb, P.nb, warp ? d1 : d0, lane);
    if (lane == 0) s_i[warp] = i;
  }
  __syncthreads();
  const int64_t i0 = s_i[0], i1 = s_i[1], j0 = d0 - i0, j1 = d1 - i1;
  const int la = int(i1 - i0), lb = int(j1 - j0), len = la + lb;
  for (int x = threadIdx.x; x < len; x += kMergeThreads) {
    if (x < la) {
      sk[x] = P.ka[i0 + x];
      sp[x] = P.pa[i0 + x];
    } else {
      sk[x] = P.kb[j0 + x - la];
      sp[x] = P.pb[j0 + x - la];
    }
  }
  __syncthreads();
  const int d = min(int(threadIdx.x) * kMergeItems, len);
  int lo = d > lb ? d - lb : 0, hi = d < la ? d : la;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (sk[mid] <= sk[la + d - mid - 1]) lo = mid + 1;
    else hi = mid;
  }
  int i = lo, j = d - lo;
#pragma unroll
  for (int it = 0; it < kMergeItems; ++it) {
    const int o = d + it;
    if (o >= len) break;
    const bool take_a = i < la && (j >= lb || sk[i] <= sk[la + j]);
    const int src = take_a ? i++ : la + j++;
    ok[o] = sk[src];
    op[o] = sp[src];
  }
  __syncthreads();
  for (int x = threadIdx.x; x < len; x += kMergeThreads) {   // coalesced stores
    P.ko[d0 + x] = ok[x];
    P.po[d0 + x] = op[x];
  }
}

// own sorted positions -> global positions (clamp flag kept)
__global__ void tag_global_kernel(const int32_t* __restrict__ sk, const int32_t* __restrict__ sp,
                                  int64_t n, int32_t offset, int32_t* __restrict__ list) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int32_t p = sp[i];
    list[i] = sk[i];
    list[n + i] = ((p & ~kClampedPos) + offset) | (p & kClampedPos);
  }
}

}  // namespace

mlStatus tag_global_positions(const int32_t* sk, const int32_t* sp, int64_t n, int64_t offset,
                              int32_t* list, cudaStream_t s) {
  if (n <= 0) return ML_OK;
  const unsigned grid = unsigned(std::min<int64_t>((n + 255) / 256, int64_t(num_sms()) * 8));
  tag_global_kernel<<<grid, 256, 0, s>>>(sk, sp, n, int32_t(offset), list);
  ML_LAUNCH_CHECK("group_sort_tag");
  return ML_OK;
}

mlStatus merge_sorted_lists(const int32_t* lists, int G, int64_t n_each, int32_t* out_k,
                            int32_t* out_p, int32_t* scratch_k, int32_t* scratch_p, cudaStream_t s) {
  struct L { const int32_t* k; const int32_t* p; int64_t n; };
  std::vector<L> cur;
  for (int g = 0; g < G; ++g)
    cur.push_back({lists + int64_t(g) * 2 * n_each, lists + int64_t(g) * 2 * n_each + n_each, n_each});
  if (G == 1) {
    ML_CUDA_TRY(cudaMemcpyAsync(out_k, cur[0].k, sizeof(int32_t) * size_t(n_each), cudaMemcpyDeviceToDevice, s));
    ML_CUDA_TRY(cudaMemcpyAsync(out_p, cur[0].p, sizeof(int32_t) * size_t(n_each), cudaMemcpyDeviceToDevice, s));
    return ML_OK;
  }
  if (G > 2 * kMaxPairs) return fail(ML_ERR_CONFIG, "group merge: G > 64");
  int rounds = 0;
  while ((1 << rounds) < G) ++rounds;
  for (int r = 1; r <= rounds; ++r) {
    // the last round lands in out, earlier ones alternate so that it does
    const bool to_out = ((rounds - r) & 1) == 0;
    int32_t* dk = to_out ? out_k : scratch_k;
    int32_t* dp = to_out ? out_p : scratch_p;
    MergeRound R{};
    std::vector<L> next;
    int64_t off = 0, tiles = 0;
    for (size_t m = 0; m < cur.size(); m += 2) {
      const L& a = cur[m];
      const L b = m + 1 < cur.size() ? cur[m + 1] : L{a.k, a.p, 0};   // odd one out: moves as is
      MergePair& P = R.p[R.npairs++];
      P = MergePair{a.k, a.p, b.k, b.p, dk + off, dp + off, a.n, b.n, tiles};
      tiles += (a.n + b.n + kMergeTile - 1) / kMergeTile;
      next.push_back({dk + off, dp + off, a.n + b.n});
      off += a.n + b.n;
    }
    if (tiles > 0) {
      merge_round_kernel<<<unsigned(tiles), kMergeThreads, 0, s>>>(R);
      ML_LAUNCH_CHECK("group_merge");
    }
    cur.swap(next);
  }
  return ML_OK;
}

}  // namespace ml
