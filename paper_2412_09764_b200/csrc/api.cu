// C-ABI entry points of libmemlayer (declared and documented in
// include/memlayer.h): host-side validation, workspace planning, and the
// stream-ordered composition of the kernels.  No C++ exception crosses the
// boundary; every failure is an mlStatus plus ml_last_error() text.
#include "internal.cuh"

#include <atomic>
#include <map>
#include <mutex>
#include <cstdlib>
#include <cstdio>
#include <exception>

namespace ml {

static thread_local std::string t_last_error;
static std::atomic<uint64_t> g_launches{0};

void set_error(const std::string& msg) { t_last_error = msg; }
mlStatus fail(mlStatus st, const std::string& msg) {
  t_last_error = msg;
  return st;
}
void count_launch(int n) { g_launches.fetch_add(uint64_t(n), std::memory_order_relaxed); }

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
      n = 148;
  }
  return n;
}

// ---- auxiliary streams: independent parts of a layer call (the value-row
// sort, the gate weight-gradient GEMMs, the gate projection) run on
// library-owned streams forked from / joined into the caller's stream with
// events, so tensor-core GEMMs overlap the HBM-bound bag kernels.  One set
// per caller stream (calls on different streams never share them).
struct Aux {
  // 3: the sparse key backward's dq gather (beside the dK sort); 4 (normal
  // priority): the layer backward's gate weight-gradient GEMMs
  cudaStream_t s[5];
  cudaEvent_t ev[10];   // 8, 9: the fp16 key / query copies of the key backward
};

// Completion event of the backward state a forward built into a caller buffer
// (keyed by the buffer): memory_layer_bwd_state orders its segmented pass after
// it, so the forward need not wait for the sort.
static mlStatus state_event(const void* state, cudaEvent_t* ev) {
  static std::mutex mu;
  static std::map<const void*, cudaEvent_t> m;
  std::lock_guard<std::mutex> lk(mu);
  auto it = m.find(state);
  if (it == m.end()) {
    cudaEvent_t e;
    ML_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    it = m.emplace(state, e).first;
  }
  *ev = it->second;
  return ML_OK;
}
// ml_set_serial(1): every auxiliary stream is the caller's stream (one
// in-order queue), so per-launch timing events bracket each kernel alone --
// the per-kernel measurement pass of bench.py; the headline timing runs with
// the concurrent streams.
static std::atomic<int> g_serial{0};
bool serial_mode() { return g_serial.load() != 0; }
static mlStatus aux_for(cudaStream_t caller, Aux** out) {
  static std::mutex mu;
  static std::map<cudaStream_t, Aux*> m, m_serial;
  std::lock_guard<std::mutex> lk(mu);
  if (g_serial.load()) {
    auto it = m_serial.find(caller);
    if (it != m_serial.end()) {
      *out = it->second;
      return ML_OK;
    }
    Aux* a = new Aux();
    for (auto& x : a->s) x = caller;
    for (auto& e : a->ev) ML_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    m_serial[caller] = a;
    *out = a;
    return ML_OK;
  }
  auto it = m.find(caller);
  if (it != m.end()) {
    *out = it->second;
    return ML_OK;
  }
  Aux* a = new Aux();
  // aux 1 runs at the highest priority: the inverse-map sort it carries
  // during the forward interleaves with the (long, HBM-bound) bag forward
  // instead of waiting for its CTAs to drain
  int lo = 0, hi = 0;
  ML_CUDA_TRY(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  ML_CUDA_TRY(cudaStreamCreateWithFlags(&a->s[0], cudaStreamNonBlocking));
  ML_CUDA_TRY(cudaStreamCreateWithPriority(&a->s[1], cudaStreamNonBlocking, hi));
  ML_CUDA_TRY(cudaStreamCreateWithFlags(&a->s[2], cudaStreamNonBlocking));
  ML_CUDA_TRY(cudaStreamCreateWithFlags(&a->s[3], cudaStreamNonBlocking));
  ML_CUDA_TRY(cudaStreamCreateWithFlags(&a->s[4], cudaStreamNonBlocking));
  for (auto& e : a->ev) ML_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  m[caller] = a;
  *out = a;
  return ML_OK;
}
// The layer backward's gate weight-gradient GEMMs: aux 4 (normal priority),
// so the value-row state build (the forward's aux 2, which the segmented pass
// waits for) is not starved of SMs by them; ML_BWD_GEMM_STREAM=1 puts them on
// the high-priority aux 1 (the earlier layout, for A/B runs)
static cudaStream_t bwd_gemm_stream(const Aux* a) {
  static const int gs = [] {
    const char* e = std::getenv("ML_BWD_GEMM_STREAM");
    return (e && e[0] == '1') ? 1 : 4;
  }();
  return a->s[gs];
}
// make `to` wait for all work enqueued so far on `from`
static mlStatus stream_dep(cudaStream_t from, cudaStream_t to, cudaEvent_t ev) {
  ML_CUDA_TRY(cudaEventRecord(ev, from));
  ML_CUDA_TRY(cudaStreamWaitEvent(to, ev, 0));
  timing_mark(nullptr, to);
  return ML_OK;
}

static int ceil_log2(int64_t n) {
  int b = 0;
  while ((int64_t(1) << b) < n) ++b;
  return b;
}

// ------------------------------------------------------------ validation
static mlStatus check_pkm(const mlPkmShape* s) {
  if (!s) return fail(ML_ERR_ARG, "null shape");
  if (s->dtype != ML_F32 && s->dtype != ML_BF16) return fail(ML_ERR_ARG, "unknown dtype");
  if (s->T < 0 || s->H < 1 || s->S < 1 || s->Dk < 2)
    return fail(ML_ERR_CONFIG, "pkm: need T >= 0, H >= 1, S >= 1, Dk >= 2");
  if (s->Dk % 2) return fail(ML_ERR_CONFIG, "pkm: odd key dimension Dk (SPEC S:143)");
  if (s->k < 1 || s->k > s->S) return fail(ML_ERR_CONFIG, "pkm: need 1 <= k <= S (SPEC S:150)");
  if (s->k > 32) return fail(ML_ERR_UNSUPPORTED, "pkm: k > 32 not supported by the warp select");
  if (s->qk_norm != 0 && s->qk_norm != 1) return fail(ML_ERR_ARG, "pkm: qk_norm must be 0 or 1");
  if (int64_t(s->S) * s->S >= (int64_t(1) << 31)) return fail(ML_ERR_CONFIG, "pkm: N = S^2 must be < 2^31");
  if (int64_t(s->H) * s->S >= (int64_t(1) << 30)) return fail(ML_ERR_CONFIG, "pkm: H*S too large");
  ML_TRY(check_cols(s->Dk / 2, s->dtype, "pkm half-key row"));
  return ML_OK;
}

static mlStatus check_bag(const mlBagShape* s) {
  if (!s) return fail(ML_ERR_ARG, "null shape");
  if (s->dtype != ML_F32 && s->dtype != ML_BF16) return fail(ML_ERR_ARG, "unknown dtype");
  if (s->grad_dtype != ML_F32 && s->grad_dtype != ML_BF16) return fail(ML_ERR_ARG, "unknown grad_dtype");
  if (s->grad_dtype == ML_BF16 && s->dtype != ML_BF16)
    return fail(ML_ERR_UNSUPPORTED, "bag: a bf16 value gradient needs a bf16 value table");
  if (s->N < 1 || s->N >= (int64_t(1) << 31)) return fail(ML_ERR_CONFIG, "bag: need 1 <= N < 2^31");
  if (s->T < 0) return fail(ML_ERR_CONFIG, "bag: T < 0");
  if (s->B < 1 || s->B > 1024) return fail(ML_ERR_CONFIG, "bag: need 1 <= B <= 1024");
  if (int64_t(s->T) * s->B >= (int64_t(1) << 31)) return fail(ML_ERR_CONFIG, "bag: T*B must be < 2^31");
  ML_TRY(check_cols(s->dv, s->dtype, "value row"));
  return ML_OK;
}

static mlStatus check_ptrs(std::initializer_list<const void*> ps) {
  for (const void* p : ps) {
    if (!p) return fail(ML_ERR_ARG, "null pointer argument");
    if (reinterpret_cast<uintptr_t>(p) % 16) return fail(ML_ERR_ARG, "pointer not 16-byte aligned");
  }
  return ML_OK;
}

// ------------------------------------------------------------ plans
// qk-normalisation scale factors (shape.qk_norm): 1/max(||x||, eps) per query
// half [T*H*2] and per half-key row [2][H*S]
struct QkBufs { float* qinv = nullptr; float* kinv = nullptr; };
static void qk_carve(Carver& c, const mlPkmShape& s, QkBufs& b) {
  if (!s.qk_norm) return;
  b.qinv = c.take<float>(int64_t(s.T) * s.H * 2);
  b.kinv = c.take<float>(int64_t(2) * s.H * s.S);
}
static mlStatus qk_compute(const mlPkmShape& s, const void* q, const void* K1, const void* K2,
                           QkBufs& b, QkNorm* qn, cudaStream_t st) {
  *qn = QkNorm{};
  if (!s.qk_norm) return ML_OK;
  const int Dh = s.Dk / 2;
  const int64_t HS = int64_t(s.H) * s.S;
  ML_TRY(launch_row_inv_norm(q, int64_t(s.T) * s.H * 2, Dh, s.dtype, b.qinv, st));
  ML_TRY(launch_row_inv_norm(K1, HS, Dh, s.dtype, b.kinv, st));
  ML_TRY(launch_row_inv_norm(K2, HS, Dh, s.dtype, b.kinv + HS, st));
  qn->qinv = b.qinv;
  qn->kinv1 = b.kinv;
  qn->kinv2 = b.kinv + HS;
  return ML_OK;
}

struct PkmFwdBufs {
  float* scores = nullptr; int32_t* hI = nullptr; float* hs = nullptr; QkBufs qk;
  float* cmax = nullptr;   // chunk maxima for the chunk-filtered half top-k (long rows)
  // fused scoring + filter: candidate lists, their lengths, fallback row list
  uint64_t* cand = nullptr; int32_t* cnt = nullptr; int32_t* fail_rows = nullptr;
  int32_t* fail_n = nullptr;
};
static void pkm_fwd_carve(Carver& c, const mlPkmShape& s, PkmFwdBufs& b) {
  const int64_t TH = int64_t(s.T) * s.H;
  if (pkm_select_tc_eligible(s)) {
    b.cand = c.take<uint64_t>(TH * 2 * pkm_select_cap());
    b.cnt = c.take<int32_t>(TH * 2);
    b.fail_rows = c.take<int32_t>(TH * 2);
    b.fail_n = c.take<int32_t>(1);
    return;
  }
  b.scores = c.take<float>(TH * 2 * s.S);
  if (half_topk_chunked(s)) b.cmax = c.take<float>(TH * 2 * (s.S / 32));
  b.hI = c.take<int32_t>(TH * 2 * s.k);
  b.hs = c.take<float>(TH * 2 * s.k);
  qk_carve(c, s, b.qk);
}

// Key/query backward strategy.  dense: the k selected score gradients per
// (t, h, half) are scattered into a bf16 [T*H, 2, S] matrix and dq = ds K,
// dK += ds^T q run as tensor-core GEMMs (cuBLASLt) -- cheaper than the sparse
// gathers while S / k is small (the dense FLOPs grow with S).  sparse: dq as a
// k-row bag over the half-key table, dK by the sorted segmented reduction
// (fp32 end to end; used for fp32 inputs and large S).
static bool pkm_bwd_dense(const mlPkmShape& s) {
  static int force_sparse = -1;
  if (force_sparse < 0) {
    const char* e = std::getenv("ML_PKM_BWD_SPARSE");
    force_sparse = (e && e[0] == '1') ? 1 : 0;
  }
  return !force_sparse && s.dtype == ML_BF16 && s.S <= 2048 && (s.S % 8) == 0 &&
         ((s.Dk / 2) % 8) == 0;
}

struct PkmBwdBufs {
  float* ds; int32_t* key1; int32_t* key2;
  SortBufs sort; RunBufs runs; float* partial; int32_t* counters;
  __nv_bfloat16* ds_dense; __nv_bfloat16* ds_lo; void* gemm_ws;
  QkBufs qk; float* dK_tmp; float* ds1w; float* ds2w;
  PkmBwdF16 f16; bool use_f16;   // fp16 operands of the tcgen05 key backward (pkm_bwd_f16)
};
static void pkm_bwd_carve(Carver& c, const mlPkmShape& s, PkmBwdBufs& b) {
  const int64_t P = int64_t(s.T) * s.H * s.k;
  b.ds = c.take<float>(P);
  b.key1 = c.take<int32_t>(P);
  b.key2 = c.take<int32_t>(P);
  b.ds_dense = b.ds_lo = nullptr;
  b.gemm_ws = nullptr;
  b.dK_tmp = b.ds1w = b.ds2w = nullptr;
  b.f16 = PkmBwdF16{nullptr, nullptr, nullptr, nullptr, nullptr};
  b.use_f16 = false;
  qk_carve(c, s, b.qk);
  if (s.qk_norm) b.dK_tmp = c.take<float>(int64_t(2) * s.H * s.S * (s.Dk / 2));
  if (pkm_bwd_dense(s)) {
    b.ds_dense = c.take<__nv_bfloat16>(int64_t(s.T) * s.H * 2 * s.S);
    b.gemm_ws = c.take<char>(kGemmWs);
    if (pkm_bwd_split(s)) b.ds_lo = c.take<__nv_bfloat16>(int64_t(s.T) * s.H * 2 * s.S);
    if (pkm_bwd_f16(s)) {
      b.use_f16 = true;
      b.f16.bound = c.take<float>(4);
      b.f16.q16 = c.take<__half>(int64_t(s.T) * s.H * s.Dk);
      b.f16.K16 = c.take<__half>(int64_t(2) * s.H * s.S * (s.Dk / 2));
    }
    if (!c.base) {   // measuring: mark dense / split
      b.ds_dense = reinterpret_cast<__nv_bfloat16*>(1);
      if (b.ds_lo) b.ds_lo = b.ds_dense;
    }
    return;
  }
  b.ds1w = c.take<float>(P);
  b.ds2w = c.take<float>(P);
  sort_carve(c, P, ceil_log2(int64_t(s.H) * s.S + 1), b.sort);
  runs_carve(c, P, b.runs);
  seg_carve(c, P, s.Dk / 2, s.dtype, &b.partial, &b.counters);
}

struct BagBwdBufs { SortBufs sort; RunBufs runs; float* partial; int32_t* counters; float* dw_part; };
static void bag_bwd_carve(Carver& c, const mlBagShape& s, BagBwdBufs& b) {
  const int64_t P = int64_t(s.T) * s.B;
  sort_carve(c, P, ceil_log2(s.N), b.sort);
  runs_carve(c, P, b.runs);
  seg_carve(c, P, s.dv, s.dtype, &b.partial, &b.counters);
  b.dw_part = c.take<float>(int64_t(seg_slices(s.dv, s.dtype)) * kDwWarps * P);
}

// ------------------------------------------------------------ cores
static mlStatus pkm_fwd_core(const mlPkmShape& s, const void* q, const void* K1, const void* K2,
                             int32_t* idx, float* w, float* score, PkmFwdBufs& b, cudaStream_t st) {
  if (s.T == 0) return ML_OK;
  if (b.cand) {   // fused: scores never leave the SM (pkm_tc.cu)
    ML_TRY(launch_pkm_select_tc(s, q, K1, K2, b.cand, b.cnt, b.fail_rows, b.fail_n, st));
    ML_TRY(launch_cand_fallback(s, q, K1, K2, b.cand, b.cnt, b.fail_rows, b.fail_n, st));
    return launch_combine_cand(s, b.cand, b.cnt, idx, w, score, st);
  }
  QkNorm qn;
  ML_TRY(qk_compute(s, q, K1, K2, b.qk, &qn, st));
  ML_TRY(launch_pkm_scores(s, q, K1, K2, b.scores, st, b.cmax));
  ML_TRY(launch_half_topk(s, b.scores, b.hI, b.hs, qn, st, b.cmax));
  ML_TRY(launch_combine_softmax(s, b.hI, b.hs, idx, w, score, st));
  return ML_OK;
}

static mlStatus pkm_bwd_core(const mlPkmShape& s, const void* q, const void* K1, const void* K2,
                             const int32_t* idx, const float* w, const float* dw_part, int ns,
                             int64_t sstride, float* dq, float* dK1, float* dK2, PkmBwdBufs& b,
                             cudaStream_t st) {
  if (s.T == 0) return ML_OK;
  const int64_t P = int64_t(s.T) * s.H * s.k;
  const int Dh = s.Dk / 2;
  const int64_t HS = int64_t(s.H) * s.S;
  QkNorm qn;
  ML_TRY(qk_compute(s, q, K1, K2, b.qk, &qn, st));
  // with qk-norm the products below give G = inv * d(x_hat); the half-key
  // part goes to a temporary and is projected into dK (accumulate)
  float* dKo1 = s.qk_norm ? b.dK_tmp : dK1;
  float* dKo2 = s.qk_norm ? b.dK_tmp + HS * Dh : dK2;
  if (s.qk_norm) {
    timing_mark(nullptr, st);
    ML_CUDA_TRY(cudaMemsetAsync(b.dK_tmp, 0, sizeof(float) * size_t(2 * HS * Dh), st));
    timing_mark("memset", st);
  }
  if (b.ds_dense) {
    if (!softmax_bwd_full_rows(s)) {
      timing_mark(nullptr, st);
      ML_CUDA_TRY(cudaMemsetAsync(b.ds_dense, 0, sizeof(__nv_bfloat16) * size_t(s.T) * s.H * 2 * s.S, st));
      timing_mark("memset", st);
    }
    if (b.use_f16) {
      // the fp16 query / key copies on aux 3 / aux 2, beside ds_bound and
      // softmax_bwd (before the persistent contractions take every SM); the
      // dq contraction waits for the keys (ev[8]), the dK contraction for q (ev[9])
      Aux* aux = nullptr;
      ML_TRY(aux_for(st, &aux));
      ML_TRY(stream_dep(st, aux->s[3], aux->ev[6]));
      ML_TRY(launch_pkm_bwd_f16_query(s, q, b.f16, aux->s[3]));
      ML_CUDA_TRY(cudaEventRecord(aux->ev[9], aux->s[3]));
      ML_TRY(stream_dep(st, aux->s[2], aux->ev[7]));
      ML_TRY(launch_pkm_bwd_f16_keys(s, K1, K2, b.f16, aux->s[2]));
      ML_CUDA_TRY(cudaEventRecord(aux->ev[8], aux->s[2]));
      b.f16.keys_ready = aux->ev[8];
      b.f16.q16_ready = aux->ev[9];
      ML_TRY(launch_ds_bound(s, w, dw_part, ns, sstride, b.f16.bound, st));
    }
    ML_TRY(launch_softmax_bwd(s, idx, w, dw_part, ns, sstride, b.ds, b.key1, b.key2, b.ds_dense, qn,
                              nullptr, nullptr, st, b.ds_lo, b.use_f16 ? b.f16.bound : nullptr));
    if (pkm_bwd_tc_eligible(s)) {
      // hand-written tcgen05 contractions (pkm_tc_bwd.cu); with ds_lo the
      // operand is the bf16 pair hi + lo (two MMAs per k-step); with
      // use_f16 all three operands are scaled fp16 copies
      ML_TRY(launch_pkm_bwd_tc(s, b.ds_dense, b.ds_lo, q, K1, K2, dq, dKo1, dKo2, st,
                               b.use_f16 ? &b.f16 : nullptr));
    } else {
    const int64_t lds = int64_t(s.H) * 2 * s.S;  // row pitch of ds_dense per token
    for (int half = 0; half < 2; ++half) {        // one strided-batched GEMM over heads each
      const __nv_bfloat16* A = b.ds_dense + int64_t(half) * s.S;
      const void* Kh = half ? K2 : K1;
      const char* qh = static_cast<const char*>(q) + int64_t(half) * Dh * 2;
      float* dKh = half ? dKo2 : dKo1;
      // dq[t, h, half] = ds[t, h, half, :] K_half[h]          [T, Dh] per head
      ML_TRY(gemm_rm_batched(false, false, s.T, Dh, s.S, A, lds, 2 * int64_t(s.S), Kh, Dh,
                             int64_t(s.S) * Dh, dq + int64_t(half) * Dh, int64_t(s.H) * s.Dk, s.Dk,
                             s.H, ML_BF16, true, b.gemm_ws, kGemmWs, st));
      // dK_half[h] += ds[:, h, half, :]^T q_half[:, h]        [S, Dh] per head
      ML_TRY(gemm_rm_batched(true, false, s.S, Dh, s.T, A, lds, 2 * int64_t(s.S), qh,
                             int64_t(s.H) * s.Dk, s.Dk, dKh, Dh, int64_t(s.S) * Dh, s.H, ML_BF16,
                             true, b.gemm_ws, kGemmWs, st, 1.f));
    }
    }
  } else {
    // sparse: per (t, h, half) the selected sub-keys deduplicated (ds summed
    // per distinct sub-key, the other slots get the sentinel key H*S)
    ML_TRY(launch_softmax_bwd(s, idx, w, dw_part, ns, sstride, b.ds, b.key1, b.key2, nullptr, qn,
                              b.ds1w, b.ds2w, st));
    // dq_half[t,h] = sum_a ds_half[a] K_half[h, a]   (one warp per (t, h)),
    // on its own stream beside the dK sorts and segmented passes (both only
    // read what softmax_bwd wrote; the gather is L2/HBM-bound, the sorts
    // latency-bound)
    Aux* aux = nullptr;
    ML_TRY(aux_for(st, &aux));
    cudaStream_t qs = aux->s[3];
    ML_TRY(stream_dep(st, qs, aux->ev[6]));
    ML_TRY(launch_pkm_dq(s, b.key1, b.key2, b.ds1w, b.ds2w, K1, K2, dq, qs));
    const int bits = ceil_log2(HS + 1);
    for (int half = 0; half < 2; ++half) {
      const int32_t* key = half ? b.key2 : b.key1;
      const float* wts = half ? b.ds2w : b.ds1w;
      // dK_half[h, a] += sum ds * q_half[t,h]  (sorted segments, dense
      // accumulate; the sentinel slots sort last and are skipped, so their
      // order is free: order_limit = H*S)
      int32_t *skey, *spos;
      ML_TRY(sort_pairs(key, P, bits, b.sort, &skey, &spos, st, HS + 1, HS));
      ML_TRY(find_runs(skey, P, b.runs, nullptr, nullptr, st));
      SegArgs g;
      g.skey = skey; g.spos = spos; g.P = P; g.runs = &b.runs; g.w = wts;
      g.src = q; g.lds = s.Dk; g.src_col0 = half * Dh; g.B = s.k;
      g.out = half ? dKo2 : dKo1; g.ldo = Dh; g.dense_accumulate = true;
      g.row_limit = int32_t(HS);
      g.partial = b.partial; g.counters = b.counters; g.dv = Dh; g.dtype = s.dtype;
      g.name = "pkm_dK_segreduce";
      ML_TRY(launch_segreduce(g, st));
    }
    ML_TRY(stream_dep(qs, st, aux->ev[7]));   // join the dq gather
  }
  if (s.qk_norm) {  // chain through x_hat = x / max(||x||, eps)
    ML_TRY(launch_qk_proj(q, int64_t(s.T) * s.H * 2, Dh, s.dtype, dq, dq, false, st));
    ML_TRY(launch_qk_proj(K1, HS, Dh, s.dtype, b.dK_tmp, dK1, true, st));
    ML_TRY(launch_qk_proj(K2, HS, Dh, s.dtype, b.dK_tmp + HS * Dh, dK2, true, st));
  }
  return ML_OK;
}

// the "inverse token_id -> embedding_id map": sort + runs (needs idx only)
static mlStatus bag_bwd_prepare(const mlBagShape& s, const int32_t* idx, int32_t* rows, int32_t* U,
                                BagBwdBufs& b, int32_t** skey, int32_t** spos, cudaStream_t st) {
  const int64_t P = int64_t(s.T) * s.B;
  if (P == 0) {
    ML_CUDA_TRY(cudaMemsetAsync(U, 0, sizeof(int32_t), st));
    return ML_OK;
  }
  return sort_pairs_runs(idx, P, ceil_log2(s.N), s.N, b.sort, b.runs, rows, U, skey, spos, st);
}

// *nsw (nullable): number of dw partial slices written to b.dw_part
static mlStatus bag_bwd_reduce(const mlBagShape& s, const void* V, const float* w, const void* dy,
                               void* dV, BagBwdBufs& b, int32_t* skey, int32_t* spos,
                               cudaStream_t st, int* nsw = nullptr) {
  const int64_t P = int64_t(s.T) * s.B;
  if (nsw) *nsw = seg_slices(s.dv, s.dtype);
  if (P == 0) return ML_OK;
  SegArgs g;
  g.skey = skey; g.spos = spos; g.P = P; g.runs = &b.runs; g.w = w;
  g.src = dy; g.lds = s.dv; g.src_col0 = 0; g.B = s.B;
  g.V = V; g.ldv = s.dv; g.v_col0 = 0; g.dw_part = b.dw_part;
  g.out = static_cast<float*>(dV); g.ldo = s.dv; g.dense_accumulate = false;
  g.out_bf16 = s.grad_dtype == ML_BF16;
  g.partial = b.partial; g.counters = b.counters; g.dv = s.dv; g.dtype = s.dtype;
  g.name = "embbag_bwd_segreduce";
  g.dw_slices_out = nsw;
  ML_TRY(launch_segreduce(g, st));
  return ML_OK;
}

static mlStatus bag_bwd_core(const mlBagShape& s, const void* V, const int32_t* idx, const float* w,
                             const void* dy, int32_t* rows, void* dV, int32_t* U, BagBwdBufs& b,
                             cudaStream_t st, int* nsw = nullptr) {
  int32_t *skey = nullptr, *spos = nullptr;
  ML_TRY(bag_bwd_prepare(s, idx, rows, U, b, &skey, &spos, st));
  return bag_bwd_reduce(s, V, w, dy, dV, b, skey, spos, st, nsw);
}

}  // namespace ml

using namespace ml;

#define ML_API_BEGIN try {
#define ML_API_END                                                        \
  }                                                                       \
  catch (const std::exception& e) {                                       \
    return fail(ML_ERR_CUDA, std::string("internal exception: ") + e.what()); \
  }                                                                       \
  catch (...) {                                                           \
    return fail(ML_ERR_CUDA, "internal exception");                       \
  }

static cudaStream_t S(void* p) { return static_cast<cudaStream_t>(p); }

extern "C" {

const char* ml_last_error(void) { return t_last_error.c_str(); }
int ml_version(void) { return 100; }

void ml_set_serial(int on) { g_serial.store(on ? 1 : 0); }
uint64_t ml_launch_count(void) { return g_launches.load(); }

int ml_device_info(int* sm_count, int* cc_major, int* cc_minor) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  if (sm_count) cudaDeviceGetAttribute(sm_count, cudaDevAttrMultiProcessorCount, dev);
  if (cc_major) cudaDeviceGetAttribute(cc_major, cudaDevAttrComputeCapabilityMajor, dev);
  if (cc_minor) cudaDeviceGetAttribute(cc_minor, cudaDevAttrComputeCapabilityMinor, dev);
  return 0;
}

mlStatus ml_synth_fill(void* out, int64_t n_rows, int64_t n_cols, int64_t row0, uint64_t seed,
                       uint32_t tag, float scale, int cls, mlDtype dtype, int64_t modulus,
                       void* stream) {
  ML_API_BEGIN
  if (!out) return fail(ML_ERR_ARG, "null output");
  if (n_rows < 0 || n_cols < 0 || row0 < 0) return fail(ML_ERR_ARG, "negative size");
  timing_mark(nullptr, S(stream));
  return launch_synth(out, n_rows, n_cols, row0, seed, tag, scale, cls, dtype, modulus, S(stream));
  ML_API_END
}

mlStatus pkm_topk_workspace(const mlPkmShape* shape, size_t* bytes) {
  ML_API_BEGIN
  ML_TRY(check_pkm(shape));
  if (!bytes) return fail(ML_ERR_ARG, "null bytes");
  Carver c(nullptr);
  PkmFwdBufs b;
  pkm_fwd_carve(c, *shape, b);
  *bytes = c.used;
  return ML_OK;
  ML_API_END
}

mlStatus pkm_topk(const mlPkmShape* shape, const void* q, const void* K1, const void* K2,
                  int32_t* idx, float* w, float* score, void* ws, size_t ws_bytes, void* stream) {
  ML_API_BEGIN
  ML_TRY(check_pkm(shape));
  if (shape->T == 0) return ML_OK;
  ML_TRY(check_ptrs({q, K1, K2, idx, w, ws}));
  if (score) ML_TRY(check_ptrs({score}));
  size_t need = 0;
  ML_TRY(pkm_topk_workspace(shape, &need));
  if (ws_bytes < need) return fail(ML_ERR_WORKSPACE, "pkm_topk: workspace too small");
  Carver c(ws);
  PkmFwdBufs b;
  pkm_fwd_carve(c, *shape, b);
  timing_mark(nullptr, S(stream));
  return pkm_fwd_core(*shape, q, K1, K2, idx, w, score, b, S(stream));
  ML_API_END
}

mlStatus pkm_topk_bwd_workspace(const mlPkmShape* shape, size_t* bytes) {
  ML_API_BEGIN
  ML_TRY(check_pkm(shape));
  if (!bytes) return fail(ML_ERR_ARG, "null bytes");
  Carver c(nullptr);
  PkmBwdBufs b;
  pkm_bwd_carve(c, *shape, b);
  *bytes = c.used;
  return ML_OK;
  ML_API_END
}

mlStatus pkm_topk_bwd(const mlPkmShape* shape, const void* q, const void* K1, const void* K2,
                      const int32_t* idx, const float* w, const float* dw, float* dq, float* dK1,
                      float* dK2, void* ws, size_t ws_bytes, void* stream) {
  ML_API_BEGIN
  ML_TRY(check_pkm(shape));
  if (shape->T == 0) return ML_OK;
  ML_TRY(check_ptrs({q, K1, K2, idx, w, dw, dq, dK1, dK2, ws}));
  size_t need = 0;
  ML_TRY(pkm_topk_bwd_workspace(shape, &need));
  if (ws_bytes < need) return fail(ML_ERR_WORKSPACE, "pkm_topk_bwd: workspace too small");
  Carver c(ws);
  PkmBwdBufs b;
  pkm_bwd_carve(c, *shape, b);
  const int64_t P = int64_t(shape->T) * shape->H * shape->k;
  timing_mark(nullptr, S(stream));
  return pkm_bwd_core(*shape, q, K1, K2, idx, w, dw, 1, P, dq, dK1, dK2, b, S(stream));
  ML_API_END
}

mlStatus embbag_fwd(const mlBagShape* shape, const void* V, const int32_t* idx, const float* w,
                    const void* gate_pre, void* y, void* y_ungated, void* stream) {
  ML_API_BEGIN
  ML_TRY(check_bag(shape));
  if (shape->T == 0) return ML_OK;
  ML_TRY(check_ptrs({V, idx, w, y}));
  if (gate_pre) ML_TRY(check_ptrs({gate_pre}));
  if (y_ungated) ML_TRY(check_ptrs({y_ungated}));
  BagFwdArgs a;
  a.V = V; a.ldv = shape->dv; a.N = shape->N;
  a.idx = idx; a.w = w; a.B = shape->B; a.nbags = shape->T; a.dv = shape->dv;
  a.out = y; a.ldo = shape->dv; a.out_col0 = 0; a.out_f32 = false;
  a.gate = gate_pre; a.y_ungated = y_ungated; a.dtype = shape->dtype;
  a.name = gate_pre ? "embbag_fwd_gate" : "embbag_fwd";
  timing_mark(nullptr, S(stream));
  ML_TRY(launch_bag_fwd(a, S(stream)));
  return check_index_flag(S(stream));
  ML_API_END
}

mlStatus embbag_bwd_workspace(const mlBagShape* shape, size_t* bytes) {
  ML_API_BEGIN
  ML_TRY(check_bag(shape));
  if (!bytes) return fail(ML_ERR_ARG, "null bytes");
  Carver c(nullptr);
  BagBwdBufs b;
  bag_bwd_carve(c, *shape, b);
  *bytes = c.used;
  return ML_OK;
  ML_API_END
}

mlStatus embbag_bwd(const mlBagShape* shape, const void* V, const int32_t* idx, const float* w,
                    const void* dy, int32_t* rows, void* dV, int32_t* U, float* dw, void* ws,
                    size_t ws_bytes, void* stream) {
  ML_API_BEGIN
  ML_TRY(check_bag(shape));
  if (!U) return fail(ML_ERR_ARG, "null U");
  if (shape->T == 0) {
    ML_CUDA_TRY(cudaMemsetAsync(U, 0, sizeof(int32_t), S(stream)));
    return ML_OK;
  }
  ML_TRY(check_ptrs({idx, w, dy, rows, dV, ws}));
  if ((V == nullptr) != (dw == nullptr)) return fail(ML_ERR_ARG, "embbag_bwd: V and dw are both set or both NULL");
  if (V) ML_TRY(check_ptrs({V, dw}));
  size_t need = 0;
  ML_TRY(embbag_bwd_workspace(shape, &need));
  if (ws_bytes < need) return fail(ML_ERR_WORKSPACE, "embbag_bwd: workspace too small");
  Carver c(ws);
  BagBwdBufs b;
  bag_bwd_carve(c, *shape, b);
  timing_mark(nullptr, S(stream));
  int nsw = 0;
  ML_TRY(bag_bwd_core(*shape, V, idx, w, dy, rows, dV, U, b, S(stream), &nsw));
  const int64_t P = int64_t(shape->T) * shape->B;
  if (dw) ML_TRY(launch_sum_slices(b.dw_part, nsw, P, dw, S(stream)));
  return check_index_flag(S(stream));
  ML_API_END
}

mlStatus embbag_bwd_atomics(const mlBagShape* shape, const int32_t* idx, const float* w,
                            const void* dy, float* dV_dense, void* stream) {
  ML_API_BEGIN
  ML_TRY(check_bag(shape));
  if (shape->T == 0) return ML_OK;
  ML_TRY(check_ptrs({idx, w, dy, dV_dense}));
  timing_mark(nullptr, S(stream));
  ML_TRY(launch_bag_bwd_ctrl(0, *shape, idx, w, dy, dV_dense, nullptr, S(stream)));
  return check_index_flag(S(stream));
  ML_API_END
}

int64_t embbag_bwd_lock_count(const mlBagShape* shape) {
  if (!shape || shape->N < 1) return -1;
  const int64_t vu = int64_t(shape->dv) * int64_t(dtype_size(shape->dtype)) / 16;
  return (vu > 256 ? vu / 256 : 1) * shape->N;
}

mlStatus embbag_bwd_lock(const mlBagShape* shape, const int32_t* idx, const float* w, const void* dy,
                         float* dV_dense, int32_t* locks, void* stream) {
  ML_API_BEGIN
  ML_TRY(check_bag(shape));
  if (shape->T == 0) return ML_OK;
  ML_TRY(check_ptrs({idx, w, dy, dV_dense, locks}));
  timing_mark(nullptr, S(stream));
  ML_TRY(launch_bag_bwd_ctrl(1, *shape, idx, w, dy, dV_dense, locks, S(stream)));
  return check_index_flag(S(stream));
  ML_API_END
}

mlStatus ml_sparse_adam(const mlBagShape* shape, const int32_t* rows, const void* dV,
                        const int32_t* U, void* V, float* V_master, float* m, float* v,
                        int32_t* steps, const mlAdamParams* hp, void* stream) {
  ML_API_BEGIN
  ML_TRY(check_bag(shape));
  if (!hp) return fail(ML_ERR_ARG, "sparse_adam: null hyper-parameters");
  if (shape->T == 0) return ML_OK;
  ML_TRY(check_ptrs({rows, dV, U, V, m, v, steps}));
  if (V_master) ML_TRY(check_ptrs({V_master}));
  timing_mark(nullptr, S(stream));
  return launch_sparse_adam(rows, dV, shape->grad_dtype, U, int64_t(shape->T) * shape->B, shape->dv, V, shape->dtype,
                            V_master, m, v, steps, *hp, S(stream));
  ML_API_END
}

mlStatus embbag_grad_apply(const mlBagShape* shape, const int32_t* rows, const void* dV,
                           const int32_t* U, float* dV_dense, void* stream) {
  ML_API_BEGIN
  ML_TRY(check_bag(shape));
  if (shape->T == 0) return ML_OK;
  ML_TRY(check_ptrs({rows, dV, U, dV_dense}));
  timing_mark(nullptr, S(stream));
  return launch_scatter_rows(rows, dV, shape->grad_dtype, U, int64_t(shape->T) * shape->B, shape->dv, dV_dense,
                             S(stream));
  ML_API_END
}

// ------------------------------------------------------------ layer
static mlStatus check_layer(const mlLayerShape* s) {
  if (!s) return fail(ML_ERR_ARG, "null shape");
  ML_TRY(check_pkm(&s->pkm));
  if (s->N != int64_t(s->pkm.S) * s->pkm.S) return fail(ML_ERR_CONFIG, "layer: N must equal S*S");
  mlBagShape bs{s->N, s->dv, s->pkm.T, s->pkm.H * s->pkm.k, s->pkm.dtype, s->grad_dtype};
  ML_TRY(check_bag(&bs));
  if (s->gated) {
    if (s->D < 1) return fail(ML_ERR_CONFIG, "layer: D < 1");
    if ((int64_t(s->D) * int64_t(dtype_size(s->pkm.dtype))) % 16)
      return fail(ML_ERR_CONFIG, "layer: D*e must be a multiple of 16 bytes");
  } else if (s->D != s->dv) {
    return fail(ML_ERR_CONFIG, "layer: ungated Memory needs D == dv");
  }
  return ML_OK;
}

static mlBagShape bag_of(const mlLayerShape& s) {
  return mlBagShape{s.N, s.dv, s.pkm.T, s.pkm.H * s.pkm.k, s.pkm.dtype, s.grad_dtype};
}

struct LayerFwdBufs { PkmFwdBufs pkm; void* z; void* gemm_ws; };
static void layer_fwd_carve(Carver& c, const mlLayerShape& s, LayerFwdBufs& b) {
  pkm_fwd_carve(c, s.pkm, b.pkm);
  b.z = c.take<char>(int64_t(s.pkm.T) * s.dv * int64_t(dtype_size(s.pkm.dtype)));
  b.gemm_ws = c.take<char>(kGemmWs);
}

struct LayerBwdBufs {
  BagBwdBufs bag; PkmBwdBufs pkm; void *dz, *z, *dy, *dg, *gemm_ws, *gemm_ws2;
};
static void layer_bwd_carve(Carver& c, const mlLayerShape& s, LayerBwdBufs& b) {
  const int64_t act = int64_t(s.pkm.T) * s.dv * int64_t(dtype_size(s.pkm.dtype));
  bag_bwd_carve(c, bag_of(s), b.bag);
  pkm_bwd_carve(c, s.pkm, b.pkm);
  b.dz = c.take<char>(act);
  b.z = c.take<char>(act);
  b.dy = c.take<char>(act);
  b.dg = c.take<char>(act);
  b.gemm_ws = c.take<char>(kGemmWs);
  b.gemm_ws2 = c.take<char>(kGemmWs);
}

// Backward state built by the forward: the sorted inverse index map of the
// bag backward depends only on the indices, so the forward can compute it on
// a side stream while the bag forward streams V (HBM-bound).
struct BagPrepState { SortBufs sort; RunBufs runs; int32_t* rows; int32_t* U; };
static void state_carve(Carver& c, const mlBagShape& s, BagPrepState& st) {
  const int64_t P = int64_t(s.T) * s.B;
  sort_carve(c, P, ceil_log2(s.N), st.sort);
  runs_carve(c, P, st.runs);
  st.rows = c.take<int32_t>(std::max<int64_t>(P, 1));
  st.U = c.take<int32_t>(1);
}

mlStatus memory_layer_state_bytes(const mlLayerShape* shape, size_t* bytes) {
  ML_API_BEGIN
  ML_TRY(check_layer(shape));
  if (!bytes) return fail(ML_ERR_ARG, "null bytes");
  Carver c(nullptr);
  BagPrepState b;
  state_carve(c, bag_of(*shape), b);
  *bytes = c.used;
  return ML_OK;
  ML_API_END
}

// bag-level state (the memory group builds it during its forward)
mlStatus embbag_bwd_state_bytes(const mlBagShape* shape, size_t* bytes) {
  ML_API_BEGIN
  ML_TRY(check_bag(shape));
  if (!bytes) return fail(ML_ERR_ARG, "null bytes");
  Carver c(nullptr);
  BagPrepState b;
  state_carve(c, *shape, b);
  *bytes = c.used;
  return ML_OK;
  ML_API_END
}

mlStatus embbag_bwd_prepare(const mlBagShape* shape, const int32_t* idx, void* state,
                            size_t state_bytes, void* stream) {
  ML_API_BEGIN
  ML_TRY(check_bag(shape));
  size_t need = 0;
  ML_TRY(embbag_bwd_state_bytes(shape, &need));
  if (state_bytes < need) return fail(ML_ERR_WORKSPACE, "embbag_bwd_prepare: state too small");
  ML_TRY(check_ptrs({state}));
  if (shape->T > 0) ML_TRY(check_ptrs({idx}));
  Carver sc(state);
  BagPrepState ps;
  state_carve(sc, *shape, ps);
  BagBwdBufs pb{};
  pb.sort = ps.sort;
  pb.runs = ps.runs;
  int32_t *sk = nullptr, *sp = nullptr;
  timing_mark(nullptr, S(stream));
  ML_TRY(bag_bwd_prepare(*shape, idx, ps.rows, ps.U, pb, &sk, &sp, S(stream)));
  return check_index_flag(S(stream));
  ML_API_END
}

// ---- the memory group's state, built once per group (merge.cu)
mlStatus embbag_bwd_group_sort_local_workspace(const mlBagShape* local, size_t* bytes) {
  ML_API_BEGIN
  ML_TRY(check_bag(local));
  if (!bytes) return fail(ML_ERR_ARG, "null bytes");
  Carver c(nullptr);
  SortBufs sb;
  sort_carve(c, int64_t(local->T) * local->B, ceil_log2(local->N), sb);
  *bytes = c.used;
  return ML_OK;
  ML_API_END
}

mlStatus embbag_bwd_group_sort_local(const mlBagShape* local, int rank, const int32_t* idx_local,
                                     int32_t* list, void* ws, size_t ws_bytes, void* stream) {
  ML_API_BEGIN
  ML_TRY(check_bag(local));
  const int64_t P = int64_t(local->T) * local->B;
  if (rank < 0) return fail(ML_ERR_ARG, "embbag_bwd_group_sort_local: rank < 0");
  if (int64_t(rank + 1) * P >= (int64_t(1) << 31))
    return fail(ML_ERR_CONFIG, "embbag_bwd_group_sort_local: (rank+1)*T*B must be < 2^31");
  if (P == 0) return ML_OK;
  ML_TRY(check_ptrs({ws}));
  // element-wise int32 access: 4-byte alignment suffices (a rank's chunk of
  // a gathered index array need not start on 16 bytes)
  if (!idx_local || !list) return fail(ML_ERR_ARG, "null pointer argument");
  if ((reinterpret_cast<uintptr_t>(idx_local) | reinterpret_cast<uintptr_t>(list)) % 4)
    return fail(ML_ERR_ARG, "pointer not 4-byte aligned");
  size_t need = 0;
  ML_TRY(embbag_bwd_group_sort_local_workspace(local, &need));
  if (ws_bytes < need) return fail(ML_ERR_WORKSPACE, "embbag_bwd_group_sort_local: workspace too small");
  Carver c(ws);
  SortBufs sb;
  sort_carve(c, P, ceil_log2(local->N), sb);
  int32_t *sk = nullptr, *sp = nullptr;
  timing_mark(nullptr, S(stream));
  ML_TRY(sort_pairs(idx_local, P, ceil_log2(local->N), sb, &sk, &sp, S(stream), local->N));
  ML_TRY(tag_global_positions(sk, sp, P, int64_t(rank) * P, list, S(stream)));
  return check_index_flag(S(stream));
  ML_API_END
}

mlStatus embbag_bwd_group_merge(const mlBagShape* shard, int G, const int32_t* lists, void* state,
                                size_t state_bytes, void* stream) {
  ML_API_BEGIN
  ML_TRY(check_bag(shard));
  if (G < 1) return fail(ML_ERR_ARG, "embbag_bwd_group_merge: G < 1");
  if (shard->T % G) return fail(ML_ERR_CONFIG, "embbag_bwd_group_merge: G must divide shard T");
  size_t need = 0;
  ML_TRY(embbag_bwd_state_bytes(shard, &need));
  if (state_bytes < need) return fail(ML_ERR_WORKSPACE, "embbag_bwd_group_merge: state too small");
  ML_TRY(check_ptrs({state}));
  cudaStream_t st = S(stream);
  const int64_t P = int64_t(shard->T) * shard->B;
  Carver sc(state);
  BagPrepState ps;
  state_carve(sc, *shard, ps);
  if (P == 0) {
    ML_CUDA_TRY(cudaMemsetAsync(ps.U, 0, sizeof(int32_t), st));
    return ML_OK;
  }
  if (!lists || reinterpret_cast<uintptr_t>(lists) % 4) return fail(ML_ERR_ARG, "lists: null or not 4-byte aligned");
  const int bits = ceil_log2(shard->N);
  int32_t *fk = nullptr, *fp = nullptr;
  ML_TRY(sorted_result(P, bits, ps.sort, &fk, &fp));
  const int other = fk == ps.sort.k[0] ? 1 : 0;
  timing_mark(nullptr, st);
  ML_TRY(merge_sorted_lists(lists, G, P / G, fk, fp, ps.sort.k[other], ps.sort.v[other], st));
  ML_TRY(find_runs(fk, P, ps.runs, ps.rows, ps.U, st));
  return ML_OK;
  ML_API_END
}

mlStatus embbag_bwd_state(const mlBagShape* shape, const void* V, const float* w, const void* dy,
                          const void* state, size_t state_bytes, int32_t* rows, void* dV,
                          int32_t* U, float* dw, void* ws, size_t ws_bytes, void* stream) {
  ML_API_BEGIN
  ML_TRY(check_bag(shape));
  if (!U) return fail(ML_ERR_ARG, "null U");
  cudaStream_t st = S(stream);
  const int64_t P = int64_t(shape->T) * shape->B;
  if (P == 0) {
    ML_CUDA_TRY(cudaMemsetAsync(U, 0, sizeof(int32_t), st));
    return ML_OK;
  }
  ML_TRY(check_ptrs({w, dy, rows, dV, ws, state}));
  if ((V == nullptr) != (dw == nullptr)) return fail(ML_ERR_ARG, "embbag_bwd_state: V and dw are both set or both NULL");
  if (V) ML_TRY(check_ptrs({V, dw}));
  size_t need = 0, sneed = 0;
  ML_TRY(embbag_bwd_workspace(shape, &need));
  if (ws_bytes < need) return fail(ML_ERR_WORKSPACE, "embbag_bwd_state: workspace too small");
  ML_TRY(embbag_bwd_state_bytes(shape, &sneed));
  if (state_bytes < sneed) return fail(ML_ERR_WORKSPACE, "embbag_bwd_state: state too small");
  Carver c(ws);
  BagBwdBufs b;
  bag_bwd_carve(c, *shape, b);
  Carver sc(const_cast<void*>(state));
  BagPrepState ps;
  state_carve(sc, *shape, ps);
  b.sort = ps.sort;
  b.runs = ps.runs;
  int32_t *skey = nullptr, *spos = nullptr;
  ML_TRY(sorted_result(P, ceil_log2(shape->N), ps.sort, &skey, &spos));
  timing_mark(nullptr, st);
  ML_CUDA_TRY(cudaMemcpyAsync(rows, ps.rows, sizeof(int32_t) * size_t(P), cudaMemcpyDeviceToDevice, st));
  ML_CUDA_TRY(cudaMemcpyAsync(U, ps.U, sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
  int nsw = 0;
  ML_TRY(bag_bwd_reduce(*shape, V, w, dy, dV, b, skey, spos, st, &nsw));
  if (dw) ML_TRY(launch_sum_slices(b.dw_part, nsw, P, dw, st));
  return check_index_flag(st);
  ML_API_END
}

mlStatus memory_layer_state_wait(const void* state, void* stream) {
  ML_API_BEGIN
  ML_TRY(check_ptrs({state}));
  cudaEvent_t done;
  ML_TRY(state_event(state, &done));
  ML_CUDA_TRY(cudaStreamWaitEvent(S(stream), done, 0));
  return ML_OK;
  ML_API_END
}

mlStatus memory_layer_fwd_workspace(const mlLayerShape* shape, size_t* bytes) {
  ML_API_BEGIN
  ML_TRY(check_layer(shape));
  if (!bytes) return fail(ML_ERR_ARG, "null bytes");
  Carver c(nullptr);
  LayerFwdBufs b;
  layer_fwd_carve(c, *shape, b);
  *bytes = c.used;
  return ML_OK;
  ML_API_END
}

mlStatus memory_layer_fwd(const mlLayerShape* shape, const void* x, const void* q, const void* K1,
                          const void* K2, const void* V, const void* W1, const void* W2, void* out,
                          int32_t* idx_saved, float* w_saved, void* g_saved, void* y_saved,
                          void* ws, size_t ws_bytes, void* stream) {
  return memory_layer_fwd_state(shape, x, q, K1, K2, V, W1, W2, out, idx_saved, w_saved, g_saved,
                                y_saved, nullptr, 0, ws, ws_bytes, stream);
}

mlStatus memory_layer_fwd_state(const mlLayerShape* shape, const void* x, const void* q,
                                const void* K1, const void* K2, const void* V, const void* W1,
                                const void* W2, void* out, int32_t* idx_saved, float* w_saved,
                                void* g_saved, void* y_saved, void* state, size_t state_bytes,
                                void* ws, size_t ws_bytes, void* stream) {
  ML_API_BEGIN
  ML_TRY(check_layer(shape));
  const mlLayerShape& s = *shape;
  if (s.pkm.T == 0) return ML_OK;
  ML_TRY(check_ptrs({q, K1, K2, V, out, idx_saved, w_saved, ws}));
  if (s.gated) ML_TRY(check_ptrs({x, W1, W2, g_saved, y_saved}));
  size_t need = 0;
  ML_TRY(memory_layer_fwd_workspace(shape, &need));
  if (ws_bytes < need) return fail(ML_ERR_WORKSPACE, "memory_layer_fwd: workspace too small");
  Carver c(ws);
  LayerFwdBufs b;
  layer_fwd_carve(c, s, b);
  cudaStream_t st = S(stream);
  const int T = s.pkm.T;
  timing_mark(nullptr, st);
  Aux* aux = nullptr;
  if (s.gated) {
    // g = x W1 [T, dv] on an auxiliary stream, concurrent with the lookup
    ML_TRY(aux_for(st, &aux));
    ML_TRY(stream_dep(st, aux->s[0], aux->ev[0]));
    ML_TRY(gemm_rm(false, false, T, s.dv, s.D, x, s.D, W1, s.dv, g_saved, s.dv, s.pkm.dtype, false,
                   b.gemm_ws, kGemmWs, aux->s[0]));
  }
  if (state) {
    size_t sneed = 0;
    ML_TRY(memory_layer_state_bytes(shape, &sneed));
    if (state_bytes < sneed) return fail(ML_ERR_WORKSPACE, "memory_layer_fwd_state: state too small");
  }
  ML_TRY(pkm_fwd_core(s.pkm, q, K1, K2, idx_saved, w_saved, nullptr, b.pkm, st));
  if (state) {
    // the backward's sort + runs on aux 2 (normal priority): it fills the SMs
    // the bag forward's tail and the gate GEMMs leave idle; the backward's
    // segmented pass waits for its completion event (no join here)
    if (!aux) ML_TRY(aux_for(st, &aux));
    Carver sc(state);
    BagPrepState ps;
    state_carve(sc, bag_of(s), ps);
    BagBwdBufs pb{};
    pb.sort = ps.sort;
    pb.runs = ps.runs;
    int32_t *sk = nullptr, *sp = nullptr;
    cudaEvent_t done;
    ML_TRY(state_event(state, &done));
    // (on the high-priority aux 1 it finished during the bag forward but
    // slowed it by 0.11 ms: step 5.21 vs 5.15 ms, scripts/state_stream_ab.sh)
    ML_TRY(stream_dep(st, aux->s[2], aux->ev[4]));
    ML_TRY(bag_bwd_prepare(bag_of(s), idx_saved, ps.rows, ps.U, pb, &sk, &sp, aux->s[2]));
    ML_CUDA_TRY(cudaEventRecord(done, aux->s[2]));
  }
  BagFwdArgs a;
  a.V = V; a.ldv = s.dv; a.N = s.N;
  a.idx = idx_saved; a.w = w_saved; a.B = s.pkm.H * s.pkm.k; a.nbags = T; a.dv = s.dv;
  a.ldo = s.dv; a.dtype = s.pkm.dtype;
  a.name = s.gated ? "embbag_fwd_gate" : "embbag_fwd";
  if (!s.gated) {
    a.out = out;
    ML_TRY(launch_bag_fwd(a, st));
    if (y_saved && y_saved != out)
      ML_CUDA_TRY(cudaMemcpyAsync(y_saved, out, size_t(T) * s.dv * dtype_size(s.pkm.dtype),
                                  cudaMemcpyDeviceToDevice, st));
    return check_index_flag(st);
  }
  ML_TRY(stream_dep(aux->s[0], st, aux->ev[1]));   // join: g ready
  // z = (sum_j w_j V[idx_j]) * silu(g); y saved
  a.out = b.z; a.gate = g_saved; a.y_ungated = y_saved;
  ML_TRY(launch_bag_fwd(a, st));
  // out = z W2  [T, D]
  ML_TRY(gemm_rm(false, false, T, s.D, s.dv, b.z, s.dv, W2, s.D, out, s.D, s.pkm.dtype, false,
                 b.gemm_ws, kGemmWs, st));
  return check_index_flag(st);
  ML_API_END
}

mlStatus memory_layer_bwd_workspace(const mlLayerShape* shape, size_t* bytes) {
  ML_API_BEGIN
  ML_TRY(check_layer(shape));
  if (!bytes) return fail(ML_ERR_ARG, "null bytes");
  Carver c(nullptr);
  LayerBwdBufs b;
  layer_bwd_carve(c, *shape, b);
  *bytes = c.used;
  return ML_OK;
  ML_API_END
}

mlStatus memory_layer_bwd(const mlLayerShape* shape, const void* dout, const void* x,
                          const void* q, const void* K1, const void* K2, const void* V,
                          const void* W1, const void* W2, const int32_t* idx_saved,
                          const float* w_saved, const void* g_saved, const void* y_saved,
                          void* dx, float* dq, float* dK1, float* dK2, int32_t* dV_rows,
                          void* dV, int32_t* U, float* dW1, float* dW2, float* dw_out, void* ws,
                          size_t ws_bytes, void* stream) {
  return memory_layer_bwd_state(shape, dout, x, q, K1, K2, V, W1, W2, idx_saved, w_saved, g_saved,
                                y_saved, nullptr, 0, dx, dq, dK1, dK2, dV_rows, dV, U, dW1, dW2,
                                dw_out, ws, ws_bytes, stream);
}

mlStatus memory_layer_bwd_state(const mlLayerShape* shape, const void* dout, const void* x,
                                const void* q, const void* K1, const void* K2, const void* V,
                                const void* W1, const void* W2, const int32_t* idx_saved,
                                const float* w_saved, const void* g_saved, const void* y_saved,
                                const void* state, size_t state_bytes, void* dx, float* dq,
                                float* dK1, float* dK2, int32_t* dV_rows, void* dV, int32_t* U,
                                float* dW1, float* dW2, float* dw_out, void* ws, size_t ws_bytes,
                                void* stream) {
  ML_API_BEGIN
  ML_TRY(check_layer(shape));
  const mlLayerShape& s = *shape;
  if (!U) return fail(ML_ERR_ARG, "null U");
  cudaStream_t st = S(stream);
  if (s.pkm.T == 0) {
    ML_CUDA_TRY(cudaMemsetAsync(U, 0, sizeof(int32_t), st));
    return ML_OK;
  }
  ML_TRY(check_ptrs({dout, q, K1, K2, V, idx_saved, w_saved, dq, dK1, dK2, dV_rows, dV, ws}));
  if (s.gated) ML_TRY(check_ptrs({x, W1, W2, g_saved, y_saved, dx, dW1, dW2}));
  if (dw_out) ML_TRY(check_ptrs({dw_out}));
  size_t need = 0;
  ML_TRY(memory_layer_bwd_workspace(shape, &need));
  if (ws_bytes < need) return fail(ML_ERR_WORKSPACE, "memory_layer_bwd: workspace too small");
  Carver c(ws);
  LayerBwdBufs b;
  layer_bwd_carve(c, s, b);
  const int T = s.pkm.T;
  const mlDtype dt = s.pkm.dtype;
  const void* dy = dout;
  const mlBagShape bs = bag_of(s);
  timing_mark(nullptr, st);
  Aux* aux = nullptr;
  ML_TRY(aux_for(st, &aux));
  int32_t *skey = nullptr, *spos = nullptr;
  const int32_t *state_rows = nullptr, *state_U = nullptr;
  if (state) {
    // sorted map from the forward (memory_layer_fwd_state)
    size_t sneed = 0;
    ML_TRY(memory_layer_state_bytes(shape, &sneed));
    if (state_bytes < sneed) return fail(ML_ERR_WORKSPACE, "memory_layer_bwd_state: state too small");
    Carver sc(const_cast<void*>(state));
    BagPrepState ps;
    state_carve(sc, bs, ps);
    b.bag.sort = ps.sort;
    b.bag.runs = ps.runs;
    const int64_t P = int64_t(bs.T) * bs.B;
    ML_TRY(sorted_result(P, ceil_log2(bs.N), ps.sort, &skey, &spos));
    state_rows = ps.rows;
    state_U = ps.U;
    ML_TRY(stream_dep(st, aux->s[0], aux->ev[0]));
  } else {
    // aux 0: the value-row sort + runs need only the saved indices
    ML_TRY(stream_dep(st, aux->s[0], aux->ev[0]));
    ML_TRY(bag_bwd_prepare(bs, idx_saved, dV_rows, U, b.bag, &skey, &spos, aux->s[0]));
  }
  if (s.gated) {
    // dz = dout W2^T ; elementwise gate backward -> z, dy, dg
    ML_TRY(gemm_rm(false, true, T, s.dv, s.D, dout, s.D, W2, s.D, b.dz, s.dv, dt, false, b.gemm_ws,
                   kGemmWs, st));
    ML_TRY(launch_gate_bwd(b.dz, g_saved, y_saved, b.z, b.dy, b.dg, int64_t(T) * s.dv, dt, st));
    // aux 4: dW2 = z^T dout ; dW1 = x^T dg ; dx = dg W1^T  (overlap the bag backward)
    cudaStream_t gst = bwd_gemm_stream(aux);
    ML_TRY(stream_dep(st, gst, aux->ev[1]));
    ML_TRY(gemm_rm(true, false, s.dv, s.D, T, b.z, s.dv, dout, s.D, dW2, s.D, dt, true, b.gemm_ws2,
                   kGemmWs, gst));
    ML_TRY(gemm_rm(true, false, s.D, s.dv, T, x, s.D, b.dg, s.dv, dW1, s.dv, dt, true, b.gemm_ws2,
                   kGemmWs, gst));
    ML_TRY(gemm_rm(false, true, T, s.D, s.dv, b.dg, s.dv, W1, s.dv, dx, s.D, dt, false, b.gemm_ws2,
                   kGemmWs, gst));
    dy = b.dy;
  }
  ML_TRY(stream_dep(aux->s[0], st, aux->ev[2]));     // sorted runs ready
  if (state) {   // the forward's state build (its own stream) must be complete
    cudaEvent_t done;
    ML_TRY(state_event(state, &done));
    ML_CUDA_TRY(cudaStreamWaitEvent(st, done, 0));
    // the row list / count copies run on aux 0, beside the segmented pass
    ML_CUDA_TRY(cudaStreamWaitEvent(aux->s[0], done, 0));
    const int64_t P = int64_t(bs.T) * bs.B;
    if (P == 0) {
      ML_CUDA_TRY(cudaMemsetAsync(U, 0, sizeof(int32_t), aux->s[0]));
    } else {
      ML_CUDA_TRY(cudaMemcpyAsync(dV_rows, state_rows, sizeof(int32_t) * size_t(P),
                                  cudaMemcpyDeviceToDevice, aux->s[0]));
      ML_CUDA_TRY(cudaMemcpyAsync(U, state_U, sizeof(int32_t), cudaMemcpyDeviceToDevice, aux->s[0]));
    }
  }
  int ns = 0;   // dw partial slices
  ML_TRY(bag_bwd_reduce(bs, V, w_saved, dy, dV, b.bag, skey, spos, st, &ns));
  if (state) ML_TRY(stream_dep(aux->s[0], st, aux->ev[5]));   // join the copies
  const int64_t P = int64_t(T) * bs.B;
  ML_TRY(pkm_bwd_core(s.pkm, q, K1, K2, idx_saved, w_saved, b.bag.dw_part, ns, P, dq, dK1, dK2,
                      b.pkm, st));
  if (s.gated) ML_TRY(stream_dep(bwd_gemm_stream(aux), st, aux->ev[3]));   // join the gate GEMMs
  if (dw_out) ML_TRY(launch_sum_slices(b.bag.dw_part, ns, P, dw_out, st));
  return check_index_flag(st);
  ML_API_END
}

// ------------------------------------------------------------ group pieces
static mlStatus check_group(int32_t G, int32_t T_loc, int32_t dv, mlDtype dt) {
  if (G < 1 || T_loc < 0 || dv < 1) return fail(ML_ERR_CONFIG, "group: need G >= 1, T_loc >= 0, dv >= 1");
  if (dv % G) return fail(ML_ERR_CONFIG, "group: G must divide dv (SPEC S:401)");
  if ((int64_t(dv / G) * int64_t(dtype_size(dt))) % 16)
    return fail(ML_ERR_CONFIG, "group: (dv/G)*e must be a multiple of 16 bytes");
  return ML_OK;
}

mlStatus ml_group_unpack(const void* recv, int32_t G, int32_t T_loc, int32_t dv, const void* gate,
                         void* y, void* z, mlDtype dtype, void* stream) {
  ML_API_BEGIN
  ML_TRY(check_group(G, T_loc, dv, dtype));
  if (T_loc == 0) return ML_OK;
  ML_TRY(check_ptrs({recv}));
  if (gate) ML_TRY(check_ptrs({gate, z}));
  if (y) ML_TRY(check_ptrs({y}));
  if (!y && !gate) return fail(ML_ERR_ARG, "group_unpack: nothing to write");
  timing_mark(nullptr, S(stream));
  return launch_group_unpack(recv, G, T_loc, dv / G, gate, y, z, dtype, S(stream));
  ML_API_END
}

mlStatus ml_group_pack(const void* src, int32_t G, int32_t T_loc, int32_t dv, void* dst,
                       mlDtype dtype, void* stream) {
  ML_API_BEGIN
  ML_TRY(check_group(G, T_loc, dv, dtype));
  if (T_loc == 0) return ML_OK;
  ML_TRY(check_ptrs({src, dst}));
  timing_mark(nullptr, S(stream));
  return launch_group_pack(src, G, T_loc, dv / G, dst, dtype, S(stream));
  ML_API_END
}

mlStatus ml_gate_bwd(const void* dz, const void* g, const void* y, void* z, void* dy, void* dg,
                     int64_t n, mlDtype dtype, void* stream) {
  ML_API_BEGIN
  if (n < 0) return fail(ML_ERR_ARG, "gate_bwd: n < 0");
  if (n == 0) return ML_OK;
  if ((n * int64_t(dtype_size(dtype))) % 16) return fail(ML_ERR_CONFIG, "gate_bwd: n*e must be a multiple of 16");
  ML_TRY(check_ptrs({dz, g, y, z, dy, dg}));
  timing_mark(nullptr, S(stream));
  return launch_gate_bwd(dz, g, y, z, dy, dg, n, dtype, S(stream));
  ML_API_END
}

// ------------------------------------------------------------ PEER (f4)
static mlStatus check_peer(const mlPeerShape* s) {
  if (!s) return fail(ML_ERR_ARG, "null shape");
  ML_TRY(check_pkm(&s->pkm));
  if (s->N != int64_t(s->pkm.S) * s->pkm.S) return fail(ML_ERR_CONFIG, "peer: N must equal S*S");
  mlBagShape bs{s->N, s->D, s->pkm.T, s->pkm.H * s->pkm.k, s->pkm.dtype};
  ML_TRY(check_bag(&bs));
  return ML_OK;
}
static mlBagShape peer_bag_of(const mlPeerShape& s) {
  return mlBagShape{s.N, s.D, s.pkm.T, s.pkm.H * s.pkm.k, s.pkm.dtype};
}

struct PeerFwdBufs { PkmFwdBufs pkm; float* h_part; float* a; };
static void peer_fwd_carve(Carver& c, const mlPeerShape& s, PeerFwdBufs& b) {
  const int64_t P = int64_t(s.pkm.T) * s.pkm.H * s.pkm.k;
  pkm_fwd_carve(c, s.pkm, b.pkm);
  b.h_part = c.take<float>(int64_t(peer_dot_slices(s.D, s.pkm.dtype)) * std::max<int64_t>(P, 1));
  b.a = c.take<float>(std::max<int64_t>(P, 1));
}

mlStatus peer_fwd_workspace(const mlPeerShape* shape, size_t* bytes) {
  ML_API_BEGIN
  ML_TRY(check_peer(shape));
  if (!bytes) return fail(ML_ERR_ARG, "null bytes");
  Carver c(nullptr);
  PeerFwdBufs b;
  peer_fwd_carve(c, *shape, b);
  *bytes = c.used;
  return ML_OK;
  ML_API_END
}

mlStatus peer_fwd(const mlPeerShape* shape, const void* x, const void* q, const void* K1,
                  const void* K2, const void* Ut, const void* V, void* y, int32_t* idx_saved,
                  float* w_saved, float* h_saved, void* ws, size_t ws_bytes, void* stream) {
  ML_API_BEGIN
  ML_TRY(check_peer(shape));
  const mlPeerShape& s = *shape;
  if (s.pkm.T == 0) return ML_OK;
  ML_TRY(check_ptrs({x, q, K1, K2, Ut, V, y, idx_saved, w_saved, h_saved, ws}));
  size_t need = 0;
  ML_TRY(peer_fwd_workspace(shape, &need));
  if (ws_bytes < need) return fail(ML_ERR_WORKSPACE, "peer_fwd: workspace too small");
  Carver c(ws);
  PeerFwdBufs b;
  peer_fwd_carve(c, s, b);
  cudaStream_t st = S(stream);
  const int T = s.pkm.T, B = s.pkm.H * s.pkm.k;
  const int64_t P = int64_t(T) * B;
  timing_mark(nullptr, st);
  ML_TRY(pkm_fwd_core(s.pkm, q, K1, K2, idx_saved, w_saved, nullptr, b.pkm, st));
  ML_TRY(launch_peer_dot(Ut, s.N, s.D, idx_saved, T, B, x, s.pkm.dtype, b.h_part, st));
  ML_TRY(launch_peer_act(b.h_part, peer_dot_slices(s.D, s.pkm.dtype), P, w_saved, h_saved, b.a, st));
  BagFwdArgs a;
  a.V = V; a.ldv = s.D; a.N = s.N;
  a.idx = idx_saved; a.w = b.a; a.B = B; a.nbags = T; a.dv = s.D;
  a.out = y; a.ldo = s.D; a.dtype = s.pkm.dtype;
  a.name = "peer_bag_fwd";
  ML_TRY(launch_bag_fwd(a, st));
  return check_index_flag(st);
  ML_API_END
}

struct PeerBwdBufs { BagBwdBufs bag; PkmBwdBufs pkm; float *h, *a, *dh, *dwr; };
static void peer_bwd_carve(Carver& c, const mlPeerShape& s, PeerBwdBufs& b) {
  const int64_t P = std::max<int64_t>(int64_t(s.pkm.T) * s.pkm.H * s.pkm.k, 1);
  bag_bwd_carve(c, peer_bag_of(s), b.bag);
  pkm_bwd_carve(c, s.pkm, b.pkm);
  b.h = c.take<float>(P);
  b.a = c.take<float>(P);
  b.dh = c.take<float>(P);
  b.dwr = c.take<float>(P);
}

mlStatus peer_bwd_workspace(const mlPeerShape* shape, size_t* bytes) {
  ML_API_BEGIN
  ML_TRY(check_peer(shape));
  if (!bytes) return fail(ML_ERR_ARG, "null bytes");
  Carver c(nullptr);
  PeerBwdBufs b;
  peer_bwd_carve(c, *shape, b);
  *bytes = c.used;
  return ML_OK;
  ML_API_END
}

mlStatus peer_bwd(const mlPeerShape* shape, const void* dy, const void* x, const void* q,
                  const void* K1, const void* K2, const void* Ut, const void* V,
                  const int32_t* idx_saved, const float* w_saved, const float* h_saved, void* dx,
                  float* dq, float* dK1, float* dK2, int32_t* rows, float* dU, float* dV,
                  int32_t* Ucount, float* dwr_out, void* ws, size_t ws_bytes, void* stream) {
  ML_API_BEGIN
  ML_TRY(check_peer(shape));
  const mlPeerShape& s = *shape;
  if (!Ucount) return fail(ML_ERR_ARG, "null U");
  cudaStream_t st = S(stream);
  if (s.pkm.T == 0) {
    ML_CUDA_TRY(cudaMemsetAsync(Ucount, 0, sizeof(int32_t), st));
    return ML_OK;
  }
  ML_TRY(check_ptrs({dy, x, q, K1, K2, Ut, V, idx_saved, w_saved, h_saved, dx, dq, dK1, dK2, rows,
                     dU, dV, ws}));
  size_t need = 0;
  ML_TRY(peer_bwd_workspace(shape, &need));
  if (ws_bytes < need) return fail(ML_ERR_WORKSPACE, "peer_bwd: workspace too small");
  Carver c(ws);
  PeerBwdBufs b;
  peer_bwd_carve(c, s, b);
  const mlBagShape bs = peer_bag_of(s);
  const int T = s.pkm.T, B = bs.B;
  const int64_t P = int64_t(T) * B;
  timing_mark(nullptr, st);
  // a = w * silu(h) (recomputed), then the bag backward over V with weights a:
  // dV rows and da = <dy, V[idx]> (its score gradient)
  ML_TRY(launch_peer_act(h_saved, 1, P, w_saved, b.h, b.a, st));
  int32_t *skey = nullptr, *spos = nullptr;
  ML_TRY(bag_bwd_prepare(bs, idx_saved, rows, Ucount, b.bag, &skey, &spos, st));
  int nsw = 0;
  ML_TRY(bag_bwd_reduce(bs, V, b.a, dy, dV, b.bag, skey, spos, st, &nsw));
  ML_TRY(launch_peer_dact(b.bag.dw_part, nsw, P, w_saved, h_saved, b.dh,
                          b.dwr, st));
  // dU[r] = sum_{p: idx = r} dh[p] x[t(p)]: the same sorted segments, source x
  SegArgs g;
  g.skey = skey; g.spos = spos; g.P = P; g.runs = &b.bag.runs; g.w = b.dh;
  g.src = x; g.lds = s.D; g.src_col0 = 0; g.B = B;
  g.out = dU; g.ldo = s.D; g.dense_accumulate = false;
  g.partial = b.bag.partial; g.counters = b.bag.counters; g.dv = s.D; g.dtype = s.pkm.dtype;
  g.name = "peer_dU_segreduce";
  ML_TRY(launch_segreduce(g, st));
  // dx[t] = sum_j dh[t,j] U[idx[t,j]]
  BagFwdArgs a;
  a.V = Ut; a.ldv = s.D; a.N = s.N;
  a.idx = idx_saved; a.w = b.dh; a.B = B; a.nbags = T; a.dv = s.D;
  a.out = dx; a.ldo = s.D; a.dtype = s.pkm.dtype;
  a.name = "peer_dx_bag";
  ML_TRY(launch_bag_fwd(a, st));
  // router: the product-key backward with dw = dwr
  ML_TRY(pkm_bwd_core(s.pkm, q, K1, K2, idx_saved, w_saved, b.dwr, 1, P, dq, dK1, dK2, b.pkm, st));
  if (dwr_out)
    ML_CUDA_TRY(cudaMemcpyAsync(dwr_out, b.dwr, sizeof(float) * size_t(P), cudaMemcpyDeviceToDevice, st));
  return check_index_flag(st);
  ML_API_END
}

mlStatus ml_gemm(int transA, int transB, int64_t M, int64_t N, int64_t K, const void* A, int64_t lda,
                 const void* B, int64_t ldb, void* C, int64_t ldc, mlDtype ab, int c_f32, void* ws,
                 size_t ws_bytes, void* stream) {
  ML_API_BEGIN
  if (M < 0 || N < 0 || K < 1) return fail(ML_ERR_ARG, "gemm: bad sizes");
  if (M == 0 || N == 0) return ML_OK;
  ML_TRY(check_ptrs({A, B, C}));
  timing_mark(nullptr, S(stream));
  return gemm_rm(transA != 0, transB != 0, M, N, K, A, lda, B, ldb, C, ldc, ab, c_f32 != 0, ws, ws_bytes,
                 S(stream));
  ML_API_END
}

}  // extern "C"
