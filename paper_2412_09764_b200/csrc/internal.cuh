// Internal launchers shared by the C-ABI entry points (not exported).
#pragma once
#include "common.cuh"

namespace ml {

// ml_set_serial(1) in force: every library stream is the caller's stream
bool serial_mode();

// ------------------------------------------------------------ bag forward
// out[b, out_col0 + c] = sum_{j<B} w[b,j] * V[idx[b,j], c]   for c < dv
// (optionally gated: out = y * silu(gate[b, c]); y_ungated gets y).
constexpr int kMaxOutBlocks = 64;
struct BagFwdArgs {
  const void* V = nullptr; int64_t ldv = 0; int64_t N = 0;
  const int32_t* idx = nullptr; const float* w = nullptr;
  int32_t B = 0; int32_t nbags = 0; int32_t dv = 0;
  void* out = nullptr; int64_t ldo = 0; int32_t out_col0 = 0; bool out_f32 = false;
  const void* gate = nullptr; void* y_ungated = nullptr;
  mlDtype dtype = ML_BF16;
  const char* name = "bag_fwd";   // timing / profiling label
  // blocked output (nullable host array of ceil(nbags / block_rows) bases):
  // bag b -> out_blocks[b / block_rows] row b % block_rows
  void* const* out_blocks = nullptr; int32_t block_rows = 0;
};
mlStatus check_cols(int32_t dv, mlDtype dt, const char* what);
mlStatus launch_bag_fwd(const BagFwdArgs& a, cudaStream_t s);

// ------------------------------------------------------------ PEER (f4)
// h_part[slice][t*B+j] = U[idx[t,j]] . x[t] over the slice's columns
int peer_dot_slices(int32_t D, mlDtype dt);
mlStatus launch_peer_dot(const void* Ut, int64_t N, int32_t D, const int32_t* idx, int32_t T,
                         int32_t B, const void* x, mlDtype dt, float* h_part, cudaStream_t s);
// h = sum of slices, a = w * silu(h)
mlStatus launch_peer_act(const float* h_part, int ns, int64_t P, const float* w, float* h, float* a,
                         cudaStream_t s);
// da = sum of slices; dh = da * w * silu'(h), dwr = da * silu(h)
mlStatus launch_peer_dact(const float* da_part, int ns, int64_t P, const float* w, const float* h,
                          float* dh, float* dwr, cudaStream_t s);

// --------------------------------------------------------------- scan
// Exclusive prefix sum of n int32 values; total (device int, nullable) gets
// the sum.  tmp needs scan_tmp_elems(n) ints.
int64_t scan_tmp_elems(int64_t n);
mlStatus scan_exclusive(const int32_t* in, int32_t* out, int64_t n, int32_t* tmp,
                        int32_t* total, cudaStream_t s);

// --------------------------------------------------------------- sort
// Stable LSD radix sort of (key, position) pairs, keys < 2^bits.  The
// values are the original positions 0..n-1.
struct SortBufs {
  int32_t* k[2] = {nullptr, nullptr};
  int32_t* v[2] = {nullptr, nullptr};
  int32_t* counts = nullptr;
  int32_t* scan_tmp = nullptr;
  int32_t* ghist = nullptr;     // single-pass mode: per-pass digit offsets + tile tickets
};
void sort_carve(Carver& c, int64_t n, int bits, SortBufs& b);
// On return *keys / *vals point at the sorted arrays (inside b).  Values are
// the input positions; a key outside [0, key_limit) (default 2^bits) is sorted
// as 0 and its position carries kClampedPos (the segmented pass gives it
// weight 0).
constexpr int32_t kClampedPos = int32_t(0x80000000u);
// order_limit (>= 0): positions of keys >= order_limit may come in any order
// (the caller skips them; the counting sort then leaves such runs unsorted)
mlStatus sort_pairs(const int32_t* keys_in, int64_t n, int bits, SortBufs& b,
                    int32_t** keys, int32_t** vals, cudaStream_t s, int64_t key_limit = -1,
                    int64_t order_limit = -1);
// Where sort_pairs(n, bits) leaves its result inside b (without sorting).
mlStatus sorted_result(int64_t n, int bits, SortBufs& b, int32_t** keys, int32_t** vals);

// --------------------------------------------------- runs of sorted keys
constexpr int kPieceLen = 32;  // positions per reduction piece (L)
struct RunBufs {
  int32_t* rid = nullptr;        // [n] run id of each position
  int32_t* run_begin = nullptr;  // [U+1] first position of each run, then n
  int32_t* piece_base = nullptr; // [n] at the first position of each run longer than
                                 //     kPieceLen: exclusive scan of those runs' pieces
  int32_t* n_slots = nullptr;    // device scalar: total pieces
  int32_t* lb = nullptr;         // look-back status words + tile tickets
};
void runs_carve(Carver& c, int64_t n, RunBufs& r);
// rows_out (nullable) [n]: distinct keys ascending; U (device int) count.
// ---- group state (merge.cu): list [2][n] = sorted keys | global positions
// (pos + offset, kClampedPos kept); merge_sorted_lists merges G such lists
// (lists + g*2*n_each) stably (ties to the lower list) into out_k / out_p,
// using scratch_k / scratch_p (n_each*G each) between rounds.
mlStatus tag_global_positions(const int32_t* sk, const int32_t* sp, int64_t n, int64_t offset,
                              int32_t* list, cudaStream_t s);
mlStatus merge_sorted_lists(const int32_t* lists, int G, int64_t n_each, int32_t* out_k,
                            int32_t* out_p, int32_t* scratch_k, int32_t* scratch_p, cudaStream_t s);
mlStatus find_runs(const int32_t* skey, int64_t n, RunBufs& r, int32_t* rows_out,
                   int32_t* U, cudaStream_t s);
// sort_pairs + find_runs in one; opt-in ML_RUNS_ROWSCAN=1: where the
// counting sort applies, the runs come from its per-row counts (no pass over
// the sorted positions)
mlStatus sort_pairs_runs(const int32_t* keys_in, int64_t n, int bits, int64_t key_limit,
                         SortBufs& b, RunBufs& r, int32_t* rows_out, int32_t* U, int32_t** keys,
                         int32_t** vals, cudaStream_t s);

// ------------------------------------------------ segmented reduction
// For every run of equal sorted keys (one output row per run):
//   out[row, c] (=|+=) sum_{p in run} w[pos_p] * src[pos_p / B, src_col0 + c]
// and, if V != nullptr, partial dot products of <src row, V[key]>:
// dw[p] = sum_{s < *dw_slices_out} dw_part[s*P + p] (the pipelined kernel
// writes one partial per consumer warp: seg_slices * kDwWarps slices).
struct SegArgs {
  const int32_t* skey = nullptr; const int32_t* spos = nullptr; int64_t P = 0;
  const RunBufs* runs = nullptr;
  const float* w = nullptr;
  const void* src = nullptr; int64_t lds = 0; int32_t src_col0 = 0; int32_t B = 1;
  const void* V = nullptr; int64_t ldv = 0; int32_t v_col0 = 0;
  float* dw_part = nullptr;
  float* out = nullptr; int64_t ldo = 0; bool dense_accumulate = false;
  bool out_bf16 = false;             // out holds bf16 rows (grad_dtype ML_BF16)
  int32_t row_limit = INT32_MAX;     // dense form: keys >= row_limit are sentinels (skipped)
  float* partial = nullptr; int32_t* counters = nullptr;
  int32_t dv = 0; mlDtype dtype = ML_BF16;
  const char* name = "segreduce";  // timing / profiling label
  int* dw_slices_out = nullptr;      // set: number of dw_part slices written
};
constexpr int kDwWarps = 4;          // dw partial slices per column slice (capacity)
int seg_slices(int32_t dv, mlDtype dt);
void seg_carve(Carver& c, int64_t P, int32_t dv, mlDtype dt, float** partial, int32_t** counters);
mlStatus launch_segreduce(const SegArgs& a, cudaStream_t s);
// dw[p] = sum_s dw_part[s*P + p]
mlStatus launch_sum_slices(const float* part, int nslices, int64_t P, float* dw, cudaStream_t s);

// ------------------------------------------------------ product keys
// qk-normalisation factors (all null when off): qinv [T*H*2] per query half,
// kinv1 / kinv2 [H*S] per half-key row, each 1 / max(||x||, 1e-6)
struct QkNorm { const float* qinv = nullptr; const float* kinv1 = nullptr; const float* kinv2 = nullptr; };
mlStatus launch_row_inv_norm(const void* x, int64_t rows, int Dh, mlDtype dt, float* inv,
                             cudaStream_t s);
// out (=|+=) G - x_hat (x_hat . G) per row (or G where ||x|| <= eps)
mlStatus launch_qk_proj(const void* x, int64_t rows, int Dh, mlDtype dt, const float* G, float* out,
                        bool accumulate, cudaStream_t s);
// cmax (nullable; tcgen05 path): [T*H*2][S/32] maxima of every 32 consecutive
// scores, written by the scoring epilogue for the half top-k's chunk filter
mlStatus launch_pkm_scores(const mlPkmShape& sh, const void* q, const void* K1,
                           const void* K2, float* scores, cudaStream_t s, float* cmax = nullptr);
// the chunk-filtered half top-k applies (and the scoring should write cmax)
bool half_topk_chunked(const mlPkmShape& sh);
// tcgen05 path (bf16, Dk/2 % 64 == 0, S = 32..256 power of two or multiple of 256)
bool pkm_scores_tc_eligible(const mlPkmShape& sh);
mlStatus launch_pkm_scores_tc(const mlPkmShape& sh, const void* q, const void* K1, const void* K2,
                              float* scores, cudaStream_t s, float* cmax = nullptr);
// fused scoring + half top-k filter (bf16, no qk-norm, S % 256 == 0, S >= 512):
// per (t, h, half) row a candidate list cand[row][pkm_select_cap()] of 64-bit
// keys (ord(score) << 32 | ~a) holding the row's k best, cnt[row] its length
// or -1; rows with -1 are listed in fail_rows[0 .. *fail_n) for the exact
// fallback (launch_cand_fallback).
bool pkm_select_tc_eligible(const mlPkmShape& sh);
int pkm_select_cap();
mlStatus launch_pkm_select_tc(const mlPkmShape& sh, const void* q, const void* K1, const void* K2,
                              uint64_t* cand, int32_t* cnt, int32_t* fail_rows, int32_t* fail_n,
                              cudaStream_t s);
// exact top-k of the listed rows (scores recomputed in fp32), written as k
// candidates (cnt = k)
mlStatus launch_cand_fallback(const mlPkmShape& sh, const void* q, const void* K1, const void* K2,
                              uint64_t* cand, int32_t* cnt, const int32_t* fail_rows,
                              const int32_t* fail_n, cudaStream_t s);
// key / query backward contractions on tcgen05 (pkm_tc_bwd.cu): dq = ds K
// (overwrite), dK1/dK2 += ds^T q, ds the bf16 [T, H, 2, S] matrix
bool pkm_bwd_tc_eligible(const mlPkmShape& sh);
// opt-in (ML_PKM_BWD_SPLIT=1): ds carried as a bf16 hi/lo pair into the
// tcgen05 key backward (needs the tcgen05 path and whole ds rows)
bool pkm_bwd_split(const mlPkmShape& sh);
// opt-in (ML_PKM_BWD_F16=1) for the tcgen05 key backward with whole ds rows
// and no qk-norm: the three operands go to the tensor cores
// as fp16 (11 significant bits; ds in bf16 would keep 8), each scaled by a
// power of two 2^e from a bound on its magnitude so that it stays inside
// fp16's range; the GEMM epilogues multiply by 2^-(e_ds + e_op) (exact).
// bf16 q / keys convert exactly (8 <= 11 bits) inside fp16's normal range.
bool pkm_bwd_f16(const mlPkmShape& sh);
struct PkmBwdF16 {
  float* bound;      // [4]: max|dw|, max|q|, max|K1|,|K2|, max|w|
  __half* q16;       // [T, H, Dk]: fp16(q * 2^e_q)
  __half* K16;       // [2][H, S, Dk/2]: fp16(K * 2^e_K)
  cudaEvent_t keys_ready;  // nullable: the dq contraction waits for it (K16 made on another stream)
  cudaEvent_t q16_ready;   // nullable: the dK contraction waits for it (q16 likewise)
};
// bound[0] = max |dw|, bound[3] = max |w| over the T*H*k positions (overwritten);
// ds_f16_exp_ds turns them into a bound on every ds element
mlStatus launch_ds_bound(const mlPkmShape& sh, const float* w, const float* dw_part, int nslices,
                         int64_t slice_stride, float* bound, cudaStream_t s);
// bound[2] + the fp16 copies of K1, K2 / bound[1] + the fp16 copy of q
mlStatus launch_pkm_bwd_f16_keys(const mlPkmShape& sh, const void* K1, const void* K2,
                                 const PkmBwdF16& f, cudaStream_t s);
mlStatus launch_pkm_bwd_f16_query(const mlPkmShape& sh, const void* q, const PkmBwdF16& f,
                                  cudaStream_t s);
// the exponent e of an fp16 operand's scale: bound * 2^e < 2^14 (fp16 max 65504)
__device__ __forceinline__ int ds_f16_exp(const float* bound) {
  const float b = *bound;
  if (!(b > 0.f) || !(b < 3.0e38f)) return 0;
  int e;
  frexpf(b, &e);                 // b < 2^e
  e = 14 - e;
  return e > 100 ? 100 : (e < -100 ? -100 : e);
}
// ds's exponent: ds_j = w_j (dw_j - sum_l w_l dw_l) gives |ds_j| <= W M (1 + k W)
// (M = max|dw|, W = max|w|), and a sub-key's entry sums <= k of them
__device__ __forceinline__ int ds_f16_exp_ds(const float* bound, int k) {
  const float W = bound[3], kw = float(k) * W;
  const float b = bound[0] * kw * (1.f + kw);
  return ds_f16_exp(&b);
}
mlStatus launch_pkm_bwd_tc(const mlPkmShape& sh, const __nv_bfloat16* ds, const __nv_bfloat16* ds_lo,
                           const void* q,
                           const void* K1, const void* K2, float* dq, float* dK1, float* dK2,
                           cudaStream_t s, const PkmBwdF16* f16 = nullptr);
// dq from the deduplicated (key, ds) slots of softmax_bwd's sparse form
mlStatus launch_pkm_dq(const mlPkmShape& sh, const int32_t* key1, const int32_t* key2,
                       const float* ds1, const float* ds2, const void* K1, const void* K2,
                       float* dq, cudaStream_t s);
// exact half top-k of each row's candidates, then the combine + softmax
mlStatus launch_combine_cand(const mlPkmShape& sh, const uint64_t* cand, const int32_t* cnt,
                             int32_t* idx, float* w, float* score, cudaStream_t s);
mlStatus launch_half_topk(const mlPkmShape& sh, const float* scores, int32_t* hI,
                          float* hs, const QkNorm& qn, cudaStream_t s, const float* cmax = nullptr);
mlStatus launch_combine_softmax(const mlPkmShape& sh, const int32_t* hI, const float* hs,
                                int32_t* idx, float* w, float* score, cudaStream_t s);
// ds = w (dw - sum w dw) with dw = sum over nslices partials; also writes the
// half-key row ids key1 = h*S + idx/S, key2 = h*S + idx%S per position.
// If ds_dense != nullptr (bf16 [T*H, 2, S], pre-zeroed) the selected
// half-key score gradients are also scattered densely (duplicates of one
// (t,h) summed in lane order): ds_dense[th][0][a_j] += ds_j, [1][b_j] += ds_j.
// true when softmax_bwd writes whole rows of ds_dense (no memset needed)
bool softmax_bwd_full_rows(const mlPkmShape& sh);
mlStatus launch_softmax_bwd(const mlPkmShape& sh, const int32_t* idx, const float* w,
                            const float* dw_part, int nslices, int64_t slice_stride,
                            float* ds, int32_t* key1, int32_t* key2, __nv_bfloat16* ds_dense,
                            const QkNorm& qn, float* ds1w, float* ds2w, cudaStream_t s,
                            __nv_bfloat16* ds_lo = nullptr, const float* f16_bound = nullptr);

// ------------------------------------------------------------ gate
// z = y*silu(g); dy = dz*silu(g); dg = dz*y*silu'(g)   (elementwise, n elems)
mlStatus launch_gate_bwd(const void* dz, const void* g, const void* y, void* z, void* dy,
                         void* dg, int64_t n, mlDtype dt, cudaStream_t s);
mlStatus launch_scatter_rows(const int32_t* rows, const void* dV, mlDtype gdt, const int32_t* U,
                             int64_t cap, int32_t dv, float* dense, cudaStream_t s);

// Row-major GEMM on cuBLASLt: C[M,N] = op(A) op(B), fp32 accumulation.
mlStatus gemm_rm(bool transA, bool transB, int64_t M, int64_t N, int64_t K,
                 const void* A, int64_t lda, const void* B, int64_t ldb,
                 void* C, int64_t ldc, mlDtype ab, bool c_f32,
                 void* ws, size_t ws_bytes, cudaStream_t s, float beta = 0.f);
// Strided-batched variant (element strides between consecutive batch items).
mlStatus gemm_rm_batched(bool transA, bool transB, int64_t M, int64_t N, int64_t K,
                         const void* A, int64_t lda, int64_t strideA, const void* B, int64_t ldb,
                         int64_t strideB, void* C, int64_t ldc, int64_t strideC, int batch,
                         mlDtype ab, bool c_f32, void* ws, size_t ws_bytes, cudaStream_t s,
                         float beta = 0.f);
constexpr size_t kGemmWs = size_t(32) << 20;

// ------------------------------------------------ backward controls (f3)
// strategy 0 = "atomics", 1 = "lock" (§3.1.4); dense fp32 dV, accumulate
mlStatus launch_bag_bwd_ctrl(int strategy, const mlBagShape& sh, const int32_t* idx, const float* w,
                             const void* dy, float* dV, int* locks, cudaStream_t s);

// ------------------------------------------------ sparse optimizer (f1)
mlStatus launch_sparse_adam(const int32_t* rows, const void* dV, mlDtype gdt, const int32_t* U, int64_t cap,
                            int32_t dv, void* V, mlDtype dt, float* Vm, float* m, float* v,
                            int32_t* steps, const mlAdamParams& hp, cudaStream_t s);

// ------------------------------------------------------------ group layout
// fused exchange (peer memory): pack block g straight into dst[g]; the
// owner's deterministic sum of G rank slots
mlStatus launch_group_pack_peers(const void* src, int G, int64_t T_loc, int32_t dv_slice,
                                 void* const* dst, mlDtype dt, cudaStream_t s);
mlStatus launch_sum_ranks(const float* slots, int G, int64_t n, float* out, cudaStream_t s);
mlStatus launch_group_unpack(const void* recv, int G, int64_t T_loc, int32_t dv_slice,
                             const void* gate, void* y, void* z, mlDtype dt, cudaStream_t s);
mlStatus launch_group_pack(const void* src, int G, int64_t T_loc, int32_t dv_slice, void* dst,
                           mlDtype dt, cudaStream_t s);

// ------------------------------------------------------------ synth
mlStatus launch_synth(void* out, int64_t n_rows, int64_t n_cols, int64_t row0, uint64_t seed,
                      uint32_t tag, float scale, int cls, mlDtype dt, int64_t modulus,
                      cudaStream_t s);

int num_sms();
bool check_indices_enabled();
mlStatus check_index_flag(cudaStream_t s);

}  // namespace ml
