/* libmemlayer — C ABI of the B200-native (sm_100a) memory-layer hot path of
 * "Memory Layers at Scale" (arXiv 2412.09764).
 *
 * Paper passages (PAPER.md line numbers, "P:n"):
 *   Eq. 1  I = SelectTopkIndices(Kq), s = Softmax(K_I q), y = s V_I
 *   §3.1.1     product keys: K1, K2 in R^{sqrt(N) x n/2}; split q into
 *                      q1, q2; top-k per half; argmax over s1[i1] + s2[i2]
 *   §3.1.2     values sharded along the embedding dim (
 *                      the group exchange is driven from Python, NCCL)
 *   §3.1.4     EmbeddingBag: bandwidth-bound weighted gather-sum; the
 *                      backward with an inverted token->row map ("reverse_indices")
 *   Eq. 2      output = (y ⊙ silu(x^T W1))^T W2
 *
 * Conventions (all calls):
 *  - Every data pointer is a DEVICE pointer owned by the caller, pointing to a
 *    dense row-major array with the stated shape; 16-byte aligned.  The
 *    library never allocates device memory inside a call and never
 *    synchronises the host, except (a) under ML_CHECK_INDICES=1 (see below)
 *    and (b) once per GEMM shape: the first call that runs a cuBLASLt GEMM of
 *    a new shape (the gated layer, the key/query backward, ml_gemm) times the
 *    top heuristic candidates with events on `stream` and caches the fastest.
 *    Set ML_GEMM_TUNE=0 to disable (e.g. before capturing a CUDA graph).
 *  - `stream` is a cudaStream_t passed as void*; all work is enqueued on it in
 *    order.  NULL means the legacy default stream.
 *  - Scratch comes from a caller workspace `ws` of at least the size returned
 *    by the matching *_workspace() query for the same shape.
 *  - Outputs are overwritten unless documented "accumulate".
 *  - idx are int32, weights / scores / gradients of scores, of keys, of
 *    queries and of values are fp32 regardless of mlDtype; q, K1, K2, V, x,
 *    W1, W2, y, g, out, dout, dx are of mlDtype.
 *  - Errors: every call returns mlStatus and, on failure, leaves a message in
 *    ml_last_error() (thread-local).  Shape/config validation happens on the
 *    host before any launch.  No C++ exception crosses this boundary.
 *  - Indices outside [0, N) are clamped to row 0 with weight 0 (no fault); the
 *    kernels raise a device flag.  With the environment variable
 *    ML_CHECK_INDICES=1 each bag call synchronises its stream, reads the flag
 *    and returns ML_ERR_INDEX if it was raised ("index error").
 */
#ifndef MEMLAYER_H_
#define MEMLAYER_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  ML_OK = 0,
  ML_ERR_ARG = 1,          /* null / misaligned pointer, negative size          */
  ML_ERR_CONFIG = 2,       /* shape rules violated (k > S, odd Dk, N != S^2 ...) */
  ML_ERR_INDEX = 3,        /* out-of-range index seen (ML_CHECK_INDICES=1)      */
  ML_ERR_WORKSPACE = 4,    /* workspace smaller than the *_workspace() size     */
  ML_ERR_CUDA = 5,         /* CUDA runtime / launch error (text in last_error)  */
  ML_ERR_NCCL = 6,         /* NCCL error or libnccl.so.2 missing (group calls)  */
  ML_ERR_UNSUPPORTED = 7   /* legal per the paper but not supported by v1       */
} mlStatus;

typedef enum { ML_F32 = 0, ML_BF16 = 1 } mlDtype;

/* ---------------------------------------------------------------- misc */
const char* ml_last_error(void);
int ml_version(void);
/* Number of kernels this library has launched since load (all calls). */
uint64_t ml_launch_count(void);
/* Number of SMs / compute capability of the current device (host query). */
int ml_device_info(int* sm_count, int* cc_major, int* cc_minor);

/* Optional per-launch timing: when enabled, the library records a CUDA event
 * on the launch stream after every kernel / GEMM / memset it issues (and a
 * start marker at each entry point).  ml_timing_report() synchronises on the
 * recorded events and writes "name count total_ms" lines aggregated per
 * kernel name into buf (len bytes); returns the bytes needed incl. NUL.
 * Not thread-safe against concurrent calls on different streams' reports. */
void ml_timing_enable(int on);
void ml_timing_reset(void);
size_t ml_timing_report(char* buf, size_t len);
/* Serial mode (measurement only): with on != 0, the layer calls issue every
 * kernel on the caller's stream instead of forking independent parts onto the
 * library's auxiliary streams, so the timing events above bracket one kernel
 * each (bench.py's per-kernel pass).  Results are bit-identical either way. */
void ml_set_serial(int on);

/* Counter-based synthetic generator (not method arithmetic).
 * Fills out[r - row0][c] for rows r in [row0, row0 + n_rows), c < n_cols of a
 * logical [*, n_cols] tensor with
 *   u = splitmix64(seed*0x9E3779B97F4A7C15 + tag*0xD1B54A32D192ED03 + r*n_cols + c)
 * cls 0 (continuous): f = ((u>>40) - 2^23) / 2^23;  cls 1 (exact):
 * f = (((u>>60)&15) - 8)/8;  cls 2 (dyadic): f = ((u>>58)&63)/64;
 * value = RN_fp32(f * scale) then RNE to `dtype`.  cls 3 (index): int32
 * (u mod modulus) (out is int32, scale/dtype ignored). */
mlStatus ml_synth_fill(void* out, int64_t n_rows, int64_t n_cols, int64_t row0,
                       uint64_t seed, uint32_t tag, float scale, int cls,
                       mlDtype dtype, int64_t modulus, void* stream);

/* ------------------------------------------------ product-key top-k (a1-a4)
 * Per token t and head h (reading Q1: H independent heads):
 *   q1 = q[t,h,0:Dk/2], q2 = q[t,h,Dk/2:Dk]
 *   s1[a] = q1 . K1[h,a,:], s2[b] = q2 . K2[h,b,:] for a, b < S
 *   I1, I2 = top-k of s1, s2 (score desc, ties -> lower sub-index)
 *   keep the k best of the k*k sums s1[i]+s2[j] (score desc, ties -> lower
 *   flat index a*S+b)
 *   w = softmax of the k kept scores (fp32, max-subtracted)        (Eq. 1)
 * Arithmetic: fp32 products/accumulation of the mlDtype inputs.
 * Shapes: q [T,H,Dk]; K1, K2 [H,S,Dk/2];  outputs idx [T,H,k] (flat a*S+b,
 * sorted by descending score), w [T,H,k], score [T,H,k] pre-softmax
 * (nullable).  Rules: 1 <= k <= min(S, 32); Dk even; S*S < 2^31; T >= 0
 * (T == 0 is a no-op).  Scratch: [T,H,2,S] fp32 scores + half top-k lists.
 * qk_norm != 0: qk-normalisation ("We use qk-normalization when
 * needed"; reading Q12): every query half and half-key row is L2-normalised,
 * x / max(||x||_2, 1e-6), before scoring (applied as fp32 scale factors of
 * the raw products; the backward chains through the normalisation). */
typedef struct { int32_t T, H, S, Dk, k; mlDtype dtype; int32_t qk_norm; } mlPkmShape;

mlStatus pkm_topk_workspace(const mlPkmShape* shape, size_t* bytes);
mlStatus pkm_topk(const mlPkmShape* shape, const void* q, const void* K1, const void* K2,
                  int32_t* idx, float* w, float* score,
                  void* ws, size_t ws_bytes, void* stream);

/* Backward of the lookup into the query and the half keys ("keys ...
 * are trainable"; reading Q8: no gradient through the selection):
 *   ds = w ⊙ (dw - sum_j w_j dw_j);  with a_j = idx/S, b_j = idx%S:
 *   dq[t,h,0:Dk/2]  = sum_j ds_j K1[h,a_j,:],   dq[t,h,Dk/2:] = sum_j ds_j K2[h,b_j,:]
 *   dK1[h,a,:] += sum_{(t,j): a_j = a} ds_j q1[t,h,:]   (likewise dK2)
 * dw [T,H,k] fp32 (the bag's weight gradient).  dq [T,H,Dk] fp32 overwrite;
 * dK1, dK2 [H,S,Dk/2] fp32 ACCUMULATE (deterministic: sorted segments, fixed
 * order, no float atomics). */
mlStatus pkm_topk_bwd_workspace(const mlPkmShape* shape, size_t* bytes);
mlStatus pkm_topk_bwd(const mlPkmShape* shape, const void* q, const void* K1, const void* K2,
                      const int32_t* idx, const float* w, const float* dw,
                      float* dq, float* dK1, float* dK2,
                      void* ws, size_t ws_bytes, void* stream);

/* ------------------------------------------------- EmbeddingBag (a5, a9)
 * One bag per token of B (index, weight) pairs (B = H*k in the layer):
 *   y[t,:] = sum_{j<B} w[t,j] * V[idx[t,j],:]            (Eq. 1 y = s V_I)
 * fp32 accumulation in j order, stored as dtype.  If gate_pre != NULL
 * (Eq. 2): y_out = y ⊙ silu(gate_pre) and, if y_ungated != NULL, y is
 * stored there too.  V [N,dv], idx/w [T,B], gate_pre/y/y_ungated [T,dv].
 * Rules: dv*e a multiple of 16 B; dv/(16/e) a power of two <= 256 or a
 * multiple of 256; 1 <= B <= 1024. */
/* grad_dtype: storage type of the compact value gradient dV of the backward
 * calls (ML_F32, the default of a zero-initialised shape; or ML_BF16, only
 * with a bf16 table: each element is accumulated in fp32 and rounded once,
 * half the dV bytes -- the table's own dtype, as a bf16 framework's
 * EmbeddingBag gradient).  The forward ignores it. */
typedef struct { int64_t N; int32_t dv; int32_t T; int32_t B; mlDtype dtype; mlDtype grad_dtype; } mlBagShape;

mlStatus embbag_fwd(const mlBagShape* shape, const void* V, const int32_t* idx, const float* w,
                    const void* gate_pre, void* y, void* y_ungated, void* stream);

/* Backward, "reverse_indices" strategy: the P = T*B (idx, position)
 * pairs are stably radix-sorted by idx (the inverted token->row map); each
 * distinct row r is reduced by one owner in position order:
 *   dV[r,:] = sum_{p: idx[p]=r} w[p] * dy[t(p),:]   (fp32 sums; V[r] read once per row)
 *   dw[p]   = <dy[t(p),:], V[idx[p],:]>
 * Outputs: rows[0..U) ascending distinct indices, dV[0..U) their gradient
 * rows in shape->grad_dtype (compact SparseGrad), *U (device
 * int32), dw [T,B] fp32.  An index outside [0, N) is treated as row 0 with
 * weight 0 (as the forward; ML_ERR_INDEX under ML_CHECK_INDICES=1).  rows / dV need capacity T*B rows.  Deterministic: bitwise equal
 * across runs (no float atomics; runs longer than 32 positions are split into
 * fixed pieces combined in piece order). */
mlStatus embbag_bwd_workspace(const mlBagShape* shape, size_t* bytes);
mlStatus embbag_bwd(const mlBagShape* shape, const void* V, const int32_t* idx, const float* w,
                    const void* dy, int32_t* rows, void* dV, int32_t* U, float* dw,
                    void* ws, size_t ws_bytes, void* stream);

/* With V == NULL and dw == NULL only the value gradient is computed (rows /
 * dV / U), as in the strategy comparison below. */

/* The inverse index map of embbag_bwd as a separate, caller-owned state
 * ("preprocessing to inverse the token_id to embedding_id mapping"): it
 * depends only on idx, so a caller can build it early on another stream
 * (the memory group builds it during its forward).  embbag_bwd_state then
 * runs only the segmented reduction; results are bit-identical to embbag_bwd
 * with the same idx.  state [embbag_bwd_state_bytes(shape)] must not change
 * in between.  Errors: ML_ERR_WORKSPACE when too small; others as embbag_bwd. */
mlStatus embbag_bwd_state_bytes(const mlBagShape* shape, size_t* bytes);
mlStatus embbag_bwd_prepare(const mlBagShape* shape, const int32_t* idx, void* state,
                            size_t state_bytes, void* stream);
mlStatus embbag_bwd_state(const mlBagShape* shape, const void* V, const float* w, const void* dy,
                          const void* state, size_t state_bytes, int32_t* rows, void* dV,
                          int32_t* U, float* dw, void* ws, size_t ws_bytes, void* stream);

/* Controls: the other two backward strategies of PAPER.md §3.1.4,
 * for the strategy benchmark.  Both ACCUMULATE
 * dV_dense[idx[p],:] += w[p] * dy[t(p),:] into a dense fp32 [N,dv] table the
 * caller zeroed; neither is bitwise deterministic (order of the adds).
 *   embbag_bwd_atomics: "accumulation via atomic additions" (vector float
 *     atomics, one team of threads per token).
 *   embbag_bwd_lock: "row-level atomic lock where we amortize the cost of
 *     memory lock over the embedding dimension": one CTA per token acquires a
 *     spin lock on each destination row, adds the whole row, releases.
 *     locks: int32 [embbag_bwd_lock_count(shape)] zero-initialised; left zero. */
mlStatus embbag_bwd_atomics(const mlBagShape* shape, const int32_t* idx, const float* w,
                            const void* dy, float* dV_dense, void* stream);
mlStatus embbag_bwd_lock(const mlBagShape* shape, const int32_t* idx, const float* w, const void* dy,
                         float* dV_dense, int32_t* locks, void* stream);
int64_t embbag_bwd_lock_count(const mlBagShape* shape);

/* dV_dense[rows[i],:] += dV[i,:] for i < *U (unique rows: no atomics).
 * dV in shape->grad_dtype; dV_dense [N,dv] fp32. */
mlStatus embbag_grad_apply(const mlBagShape* shape, const int32_t* rows, const void* dV,
                           const int32_t* U, float* dV_dense, void* stream);

/* Sparse (lazy, row-wise) Adam(W) for the memory values (SPEC.md
 * S:506-514; "associated optimizer states"): consumes the
 * compact (rows, dV, *U) of embbag_bwd / memory_layer_bwd directly.  For
 * i < *U, r = rows[i], g = dV[i] (rows distinct):
 *   c = ++steps[r]; m[r] = b1 m[r] + (1-b1) g; v[r] = b2 v[r] + (1-b2) g^2
 *   V[r] -= lr * ( m[r]/(1-b1^c) / (sqrt(v[r]/(1-b2^c)) + eps) + wd * V[r] )
 * Untouched rows (and their moments / counters) are unchanged.  V [N,dv] of
 * shape->dtype; V_master [N,dv] fp32 (nullable: if given, the update is done
 * on it and V receives its rounding); m, v [N,dv] fp32; steps [N] int32.
 * shape->T * shape->B = capacity of rows / dV; dV in shape->grad_dtype. */
typedef struct { float lr, beta1, beta2, eps, weight_decay; } mlAdamParams;
mlStatus ml_sparse_adam(const mlBagShape* shape, const int32_t* rows, const void* dV,
                        const int32_t* U, void* V, float* V_master, float* m, float* v,
                        int32_t* steps, const mlAdamParams* hp, void* stream);

/* ------------------------------------------------ memory layer (a1-a11)
 * Forward: pkm_topk -> g = x W1 -> z = embbag(V; idx, w) ⊙ silu(g) ->
 * out = z W2 (Eq. 1 + Eq. 2).  With gated == 0 (vanilla Memory) out = y and
 * D must equal dv; x, W1, W2, g_saved are unused.
 * x [T,D], q [T,H,Dk], K1/K2 [H,S,Dk/2], V [N,dv], W1 [D,dv], W2 [dv,D],
 * out [T,D].  Saved for the backward (caller-owned): idx_saved [T,H,k] i32,
 * w_saved [T,H,k] f32, g_saved [T,dv] (dtype, gated only), y_saved [T,dv]
 * (dtype).  N must equal S*S.  W1/W2 products run on cuBLASLt (library GEMM,
 * fp32 accumulation). */
typedef struct { mlPkmShape pkm; int64_t N; int32_t dv; int32_t D; int32_t gated;
                 mlDtype grad_dtype; /* dV storage, as mlBagShape.grad_dtype */ } mlLayerShape;

mlStatus memory_layer_fwd_workspace(const mlLayerShape* shape, size_t* bytes);
mlStatus memory_layer_fwd(const mlLayerShape* shape, const void* x, const void* q,
                          const void* K1, const void* K2, const void* V,
                          const void* W1, const void* W2, void* out,
                          int32_t* idx_saved, float* w_saved, void* g_saved, void* y_saved,
                          void* ws, size_t ws_bytes, void* stream);

/* Backward of memory_layer_fwd given dout [T,D]:
 *   gate (Eq. 2): dz = dout W2^T, dW2 = z^T dout, dy = dz ⊙ silu(g),
 *   dg = dz ⊙ y ⊙ silu'(g), dW1 = x^T dg, dx = dg W1^T     (dx: gate path only)
 *   bag: rows/dV/U compact as embbag_bwd; dw_out [T,H,k] (nullable)
 *   keys: dq [T,H,Dk] overwrite, dK1/dK2 ACCUMULATE as pkm_topk_bwd.
 * dW1 [D,dv], dW2 [dv,D] fp32 overwrite; dx [T,D] dtype. */
mlStatus memory_layer_bwd_workspace(const mlLayerShape* shape, size_t* bytes);
mlStatus memory_layer_bwd(const mlLayerShape* shape, const void* dout, const void* x,
                          const void* q, const void* K1, const void* K2, const void* V,
                          const void* W1, const void* W2,
                          const int32_t* idx_saved, const float* w_saved,
                          const void* g_saved, const void* y_saved,
                          void* dx, float* dq, float* dK1, float* dK2,
                          int32_t* dV_rows, void* dV, int32_t* U,
                          float* dW1, float* dW2, float* dw_out,
                          void* ws, size_t ws_bytes, void* stream);

/* Forward/backward pair with a precomputed backward state.  The bag
 * backward's inverse index map ("reverse_indices" preprocessing, PAPER.md
 * §3.1.4: sort of (idx, position) + runs) depends only on idx_saved,
 * so memory_layer_fwd_state builds it into the caller-owned `state` buffer
 * (memory_layer_state_bytes) on a library side stream, concurrent with the
 * HBM-bound bag forward, and memory_layer_bwd_state consumes it instead of
 * sorting.  state must not be modified between the two calls.  The state is
 * built asynchronously on a library stream (it fills the SMs the bag forward's
 * tail and the gate GEMMs leave idle); memory_layer_bwd_state orders its
 * segmented pass after it, and memory_layer_state_wait(state, stream) makes
 * any other stream wait for it (e.g. before the buffer is freed or reused).
 * Results are bit-identical to memory_layer_fwd / memory_layer_bwd (same
 * kernels, same order).  Errors: ML_ERR_WORKSPACE when state_bytes is too
 * small. */
mlStatus memory_layer_state_bytes(const mlLayerShape* shape, size_t* bytes);
mlStatus memory_layer_state_wait(const void* state, void* stream);
mlStatus memory_layer_fwd_state(const mlLayerShape* shape, const void* x, const void* q,
                                const void* K1, const void* K2, const void* V, const void* W1,
                                const void* W2, void* out, int32_t* idx_saved, float* w_saved,
                                void* g_saved, void* y_saved, void* state, size_t state_bytes,
                                void* ws, size_t ws_bytes, void* stream);
mlStatus memory_layer_bwd_state(const mlLayerShape* shape, const void* dout, const void* x,
                                const void* q, const void* K1, const void* K2, const void* V,
                                const void* W1, const void* W2, const int32_t* idx_saved,
                                const float* w_saved, const void* g_saved, const void* y_saved,
                                const void* state, size_t state_bytes, void* dx, float* dq,
                                float* dK1, float* dK2, int32_t* dV_rows, void* dV, int32_t* U,
                                float* dW1, float* dW2, float* dw_out, void* ws, size_t ws_bytes,
                                void* stream);

/* ------------------------------------------------ PEER
 * Product-key retrieval of rank-1 experts ("replacing vector
 * values with rank-one matrices"; "it retrieves a pair of embeddings,
 * which combine into a rank-1 matrix.  Several of these are assembled
 * together into a dynamic feed-forward layer").  Reading Q21:
 * key i owns U[i], V[i] in R^D; with idx, w from pkm_topk (B = H*k per token)
 *   h[t,j] = U[idx[t,j]] . x[t],  a = w * silu(h),  y[t] = sum_j a[t,j] V[idx[t,j]].
 * x, y [T,D]; U, V [N,D] (dtype); saved: idx_saved [T,H,k] i32, w_saved,
 * h_saved [T,H,k] f32.  N must equal S*S; D*e a multiple of 16 bytes and
 * (D*e/16) a power of two or a multiple of 256 (as embbag).
 * Backward given dy [T,D]: dV/dU compact over the same rows (rows [U] ascending,
 * dU, dV [P,D] fp32 capacity, *Ucount = U), dx [T,D] dtype (expert path only),
 * dq overwrite, dK1/dK2 ACCUMULATE (as pkm_topk_bwd), dwr_out [T,H,k] (nullable)
 * = dL/dw of the router weights.  Errors as the other entry points. */
typedef struct { mlPkmShape pkm; int64_t N; int32_t D; } mlPeerShape;
mlStatus peer_fwd_workspace(const mlPeerShape* shape, size_t* bytes);
mlStatus peer_fwd(const mlPeerShape* shape, const void* x, const void* q, const void* K1,
                  const void* K2, const void* U, const void* V, void* y, int32_t* idx_saved,
                  float* w_saved, float* h_saved, void* ws, size_t ws_bytes, void* stream);
mlStatus peer_bwd_workspace(const mlPeerShape* shape, size_t* bytes);
mlStatus peer_bwd(const mlPeerShape* shape, const void* dy, const void* x, const void* q,
                  const void* K1, const void* K2, const void* U, const void* V,
                  const int32_t* idx_saved, const float* w_saved, const float* h_saved, void* dx,
                  float* dq, float* dK1, float* dK2, int32_t* rows, float* dU, float* dV,
                  int32_t* Ucount, float* dwr_out, void* ws, size_t ws_bytes, void* stream);

/* ------------------------------------------- memory group pieces (a7, a12)
 * Parallel memory (§3.1.2, Fig. 2): the value table is
 * sharded along the embedding dim over the G ranks of a memory group; the
 * exchange (all-gather of (idx, w), all-to-all of the partial embeddings,
 * reverse all-to-all of dy, reduce-scatter of the partial dw) is issued by
 * the group entry points below (or by a caller running its own exchange).
 * These calls do the on-device layout work around it:
 *   ml_group_unpack: recv [G][T_loc][dv/G] (rank g's slice of this rank's
 *     tokens) -> y [T_loc][dv], y[t][g*dv/G + c] = recv[g][t][c]; if gate !=
 *     NULL also z = y ⊙ silu(gate) (Eq. 2) into z [T_loc][dv] (y nullable then).
 *   ml_group_pack: src [T_loc][dv] -> dst [G][T_loc][dv/G] (the reverse).
 * Rules: G | dv, (dv/G)*e a multiple of 16 bytes (SPEC S:401 config error). */
mlStatus ml_group_unpack(const void* recv, int32_t G, int32_t T_loc, int32_t dv, const void* gate,
                         void* y, void* z, mlDtype dtype, void* stream);
mlStatus ml_group_pack(const void* src, int32_t G, int32_t T_loc, int32_t dv, void* dst,
                       mlDtype dtype, void* stream);

/* Eq. 2 backward, elementwise over n elements (n*e a multiple of 16 B):
 * z = y ⊙ silu(g), dy = dz ⊙ silu(g), dg = dz ⊙ y ⊙ sigmoid(g)(1 + g(1 - sigmoid(g))). */
mlStatus ml_gate_bwd(const void* dz, const void* g, const void* y, void* z, void* dy, void* dg,
                     int64_t n, mlDtype dtype, void* stream);

/* Library GEMM (cuBLASLt, fp32 accumulation) for the dense gate projections:
 * row-major C[M,N] = op(A)[M,K] op(B)[K,N], op = transpose if trans*; A/B of
 * dtype `ab`, C fp32 if c_f32 else `ab`.  ws: >= 32 MiB device scratch. */
mlStatus ml_gemm(int transA, int transB, int64_t M, int64_t N, int64_t K, const void* A, int64_t lda,
                 const void* B, int64_t ldb, void* C, int64_t ldc, mlDtype ab, int c_f32, void* ws,
                 size_t ws_bytes, void* stream);

/* ------------------------------------------------ memory group (a7, a12)
 * The dim-sharded memory group of PAPER.md §3.1.2 (Fig. 2)
 * behind the C ABI: rank g of G owns V[:, g*dv/G : (g+1)*dv/G] as a
 * contiguous [N, dv/G] table; tokens are data-parallel (T_loc per rank, equal
 * on every rank: reading Q19).
 *
 * A group owns its transport and its streams (one outstanding forward /
 * backward pair at a time per group; calls on one group are not
 * thread-safe).  ml_group_init: NCCL on the current device -- one rank of an
 * ncclUniqueId (128 bytes) that the caller creates on one rank with
 * ml_group_unique_id and broadcasts (torch.distributed).  NCCL is resolved
 * at run time (libnccl.so.2); without it these two return ML_ERR_NCCL and
 * the rest of the library is unaffected.  ml_group_init_hub: G ranks as host
 * threads of one process on one device sharing a hub (ml_group_hub_create);
 * collectives are host-synchronised device copies (test harness of the same
 * protocol on one GPU; no kernel waits on another).
 *
 * Output modes (reading Q13): ML_OUT_ALLTOALL (the paper: "each
 * worker gathers the partial embeddings corresponding to its own portion of
 * the indices": y [T_loc, dv] of the rank's own tokens) and ML_OUT_ALLGATHER
 * (north-star wording: every rank receives y [G*T_loc, dv] of all tokens). */
typedef struct mlGroup_* mlGroup;
typedef enum { ML_OUT_ALLTOALL = 0, ML_OUT_ALLGATHER = 1 } mlOutMode;
mlStatus ml_group_unique_id(void* id128);
mlStatus ml_group_init(const void* id128, int G, int rank, mlGroup* out);
mlStatus ml_group_hub_create(int G, void** hub);
mlStatus ml_group_hub_destroy(void* hub);
mlStatus ml_group_init_hub(void* hub, int rank, mlGroup* out);
/* ml_group_init_loopback: rank `rank` of a G-rank group with the network
 * removed (SURVEY §8(e) t_ref(G): this rank's work, collectives replaced by
 * local copies), running the group's own code path on one GPU.  All-gathers
 * copy this rank's chunk into place and the other ranks' chunks from the
 * caller's captures (device buffers, not copied: they must outlive the
 * group): the next capture, cyclically, whose size is G x the chunk -- in a
 * layer step the packed (idx, w) [G][T_loc][2B] int32 (w as bits) and the
 * sorted lists [G][2][T_loc*B] of embbag_bwd_group_sort_local; without a
 * match the own chunk is replicated.  Other exchanges move this rank's own
 * data. */
mlStatus ml_group_init_loopback(int G, int rank, const void* const* sources, const size_t* bytes,
                                int n_sources, mlGroup* out);
mlStatus ml_group_destroy(mlGroup g);
mlStatus ml_group_info(mlGroup g, int* G, int* rank);
/* Fused forward exchange (mode ML_OUT_ALLTOALL; "each worker gathers
 * the partial embeddings corresponding to its own portion of the indices"):
 * on = 1 makes the bag forward of every token block store its output rows
 * straight into the owning rank's exchange region over peer memory (NCCL
 * transport: a cudaMalloc'd region per rank mapped into the others with CUDA
 * IPC, which needs peer access between the group's GPUs -- NVLink/NVSwitch;
 * hub transport: plain device pointers) instead of point-to-point sends,
 * followed by one flag barrier (epoch flags stored with release semantics at
 * system scope, waited on with acquire).  The region (2 x G x T_loc x dv/G
 * elements + 4 KiB of flags per rank) is allocated by the group on first use
 * -- a collective: every rank must make the same calls.  Default off, or on
 * when the environment sets ML_GROUP_P2P=1 at group creation. */
mlStatus ml_group_set_p2p(mlGroup g, int on);

/* Bag level.  shape: N, dv = the FULL value dim, T = T_loc, B, dtype
 * (grad_dtype for dV_shard).  Forward: idx_local/w_local [T_loc, B] ->
 * idx_all/w_all [G*T_loc, B] (outputs: one packed all-gather; keep them for
 * the backward), the bag over all G*T_loc tokens on V_shard [N, dv/G] (block
 * by block, each block sent to its owner while the next is computed), then
 * y: ML_OUT_ALLTOALL [T_loc, dv], ML_OUT_ALLGATHER [G*T_loc, dv].
 * Backward: dy ML_OUT_ALLTOALL [T_loc, dv] (this rank's tokens; the dv/G
 * slices go back by one all-to-all) or ML_OUT_ALLGATHER [G*T_loc, dv]
 * (replicated; the rank reads its column slice, no exchange); the sorted
 * segmented reduction on the slice gives rows [<= G*T_loc*B] ascending,
 * dV_shard [cap G*T_loc*B, dv/G] (dV never leaves the rank), *U; the partial
 * dw (a dot over dv/G columns) is reduce-scattered: dw_local [T_loc, B] =
 * the full dw of this rank's tokens.  state (nullable): the inverse index
 * map of idx_all built early by embbag_bwd_group_prepare (group stream; the
 * backward waits for it), embbag_bwd_group_state_bytes bytes.
 * embbag_bwd_group_prepare is a COLLECTIVE (every rank calls it, in the same
 * order relative to the other group calls): the inverse map is built once per
 * group, not G times -- each rank stably sorts only its own T_loc*B positions
 * (embbag_bwd_group_sort_local), the G sorted lists are all-gathered and
 * merged (embbag_bwd_group_merge); the result is bit-identical to
 * embbag_bwd_prepare of idx_all on the shard shape. */
mlStatus embbag_fwd_group_workspace(mlGroup g, const mlBagShape* shape, mlOutMode mode, size_t* bytes);
mlStatus embbag_fwd_group(mlGroup g, const mlBagShape* shape, const void* V_shard,
                          const int32_t* idx_local, const float* w_local, int32_t* idx_all,
                          float* w_all, mlOutMode mode, void* y, void* ws, size_t ws_bytes,
                          void* stream);
mlStatus embbag_bwd_group_state_bytes(mlGroup g, const mlBagShape* shape, size_t* bytes);
mlStatus embbag_bwd_group_prepare(mlGroup g, const mlBagShape* shape, const int32_t* idx_all,
                                  void* state, size_t state_bytes, void* stream);
/* The two local halves of embbag_bwd_group_prepare, usable with any
 * transport (every rank needs the inverse map of all gathered
 * indices).  sort_local: local = this rank's bag shape [T_loc, B]; idx_local
 * its [T_loc, B] indices; list [2][T_loc*B] int32 (device) receives the
 * positions sorted stably by row: list[0..P) the rows (an index outside
 * [0, N) sorts as row 0 and sets the sticky index flag), list[P..2P) the
 * GLOBAL positions rank*T_loc*B + p (bit 31 set on an out-of-range index,
 * which the backward then ignores); needs (rank+1)*T_loc*B < 2^31; idx_local
 * and list 4-byte aligned, ws 16-byte aligned, of
 * embbag_bwd_group_sort_local_workspace bytes.  merge: shard = the bag shape
 * over all group tokens (T = G*T_loc, dv = dv/G); lists [G][2][T_loc*B] the
 * G ranks' lists in rank order; state of embbag_bwd_state_bytes(shard) bytes
 * receives the merged map (ties to the lower rank: the stable order) and its
 * run table, for embbag_bwd_state. */
mlStatus embbag_bwd_group_sort_local_workspace(const mlBagShape* local, size_t* bytes);
mlStatus embbag_bwd_group_sort_local(const mlBagShape* local, int rank, const int32_t* idx_local,
                                     int32_t* list, void* ws, size_t ws_bytes, void* stream);
mlStatus embbag_bwd_group_merge(const mlBagShape* shard, int G, const int32_t* lists, void* state,
                                size_t state_bytes, void* stream);
mlStatus embbag_bwd_group_workspace(mlGroup g, const mlBagShape* shape, mlOutMode mode, size_t* bytes);
mlStatus embbag_bwd_group(mlGroup g, const mlBagShape* shape, const void* V_shard,
                          const int32_t* idx_all, const float* w_all, const void* dy,
                          mlOutMode mode, const void* state, size_t state_bytes, int32_t* rows,
                          void* dV_shard, int32_t* U, float* dw_local, void* ws, size_t ws_bytes,
                          void* stream);

/* Layer level (the gated Memory+ layer, Eq. 1 + Eq. 2, over the group).
 * shape: pkm.T = T_loc, N, dv = FULL value dim, D, gated = 1.  Forward: own
 * tokens' pkm_topk -> idx_saved/w_saved [T_loc,H,k]; g_saved = x W1 (library
 * side stream); the bag forward of embbag_fwd_group (idx_all/w_all
 * [G*T_loc,H,k] outputs); own rows y_saved [T_loc, dv] and z = y ⊙ silu(g)
 * in the unpack; out = z W2 [T_loc, D].  ML_OUT_ALLGATHER also fills y_all
 * [G*T_loc, dv].  state (nullable, embbag_bwd_group_state_bytes of the bag
 * shape [T_loc, H*k]): the backward's inverse map, built during the forward.
 * Backward (gate on own tokens, then embbag_bwd_group in the all-to-all form
 * -- the layer's dy exists for own tokens only -- then pkm_topk_bwd on own
 * tokens with the reduce-scattered dw): dx [T_loc, D] (gate path), dq
 * [T_loc,H,Dk], dK1/dK2 ACCUMULATE (this rank's tokens' part; the caller
 * all-reduces them like any replicated weight gradient), dV_rows / dV_shard /
 * U as embbag_bwd_group, dW1/dW2 fp32 (this rank's part), dw_out
 * [T_loc,H,k] nullable. */
mlStatus memory_layer_fwd_group_workspace(mlGroup g, const mlLayerShape* shape, mlOutMode mode,
                                          size_t* bytes);
mlStatus memory_layer_fwd_group(mlGroup g, const mlLayerShape* shape, mlOutMode mode, const void* x,
                                const void* q, const void* K1, const void* K2, const void* V_shard,
                                const void* W1, const void* W2, void* out, int32_t* idx_saved,
                                float* w_saved, int32_t* idx_all, float* w_all, void* g_saved,
                                void* y_saved, void* y_all, void* state, size_t state_bytes,
                                void* ws, size_t ws_bytes, void* stream);
mlStatus memory_layer_bwd_group_workspace(mlGroup g, const mlLayerShape* shape, size_t* bytes);
mlStatus memory_layer_bwd_group(mlGroup g, const mlLayerShape* shape, const void* dout,
                                const void* x, const void* q, const void* K1, const void* K2,
                                const void* V_shard, const void* W1, const void* W2,
                                const int32_t* idx_saved, const float* w_saved,
                                const int32_t* idx_all, const float* w_all, const void* g_saved,
                                const void* y_saved, const void* state, size_t state_bytes, void* dx,
                                float* dq, float* dK1, float* dK2, int32_t* dV_rows, void* dV_shard,
                                int32_t* U, float* dW1, float* dW2, float* dw_out, void* ws,
                                size_t ws_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* MEMLAYER_H_ */
