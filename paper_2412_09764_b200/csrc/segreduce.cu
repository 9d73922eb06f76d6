// Segmented reduction over sorted (key, position) runs: the atomic-free
// "reverse_indices" EmbeddingBag backward (§3.1.4):
//   dV[r, :] = sum_{p: idx[p] = r} w[p] * dy[t(p), :]        (one owner per row)
//   dw[p]    = <dy[t(p), :], V[r, :]>                          (fused: V[r] read once)
// The same kernel (without dw, dense-accumulating) produces the half-key
// gradients dK[h, a] = sum ds * q_half (pkm backward).
//
// Work split (load balance under skew, determinism): one CTA ("team") per
// chunk of 64 sorted positions; it reduces every "piece" that STARTS in its
// chunk.  A piece is a whole run, or a 32-position piece of a run longer than
// 32.  Whole runs are written directly (rows are unique: no atomics); pieces
// of long runs go to a partial buffer and the last piece to arrive (counter)
// sums all pieces of its run in piece order -> bitwise deterministic.
// The team's threads each own one 16-byte vector of the row (blockDim =
// row vectors, up to 256 = 2048 bf16 columns; wider rows use column slices,
// blockIdx.y).  Per-position metadata is decoded once into shared memory and
// read as broadcasts; the position range is walked in full batches of NB
// positions regardless of piece boundaries: all source-row and value-row
// loads of a batch are issued at once (value rows repeat inside a piece and
// hit L1), then the batch is accumulated, flushing each piece at its end.
// The fused dw dot products are reduced per batch: warp butterfly, then one
// shared-memory exchange and one barrier per batch.
// Columns: lane l owns 16-byte vector l of a 32-vector (512 B) column slice
// (blockIdx.y); every load is a coalesced 512 B row segment.
// Per chunk the warp loads all position metadata in one round (lane <->
// position), so each piece costs one memory round trip (V row + dy rows).
//
// Two kernels implement this contract:
//  * seg_kernel: one CTA per 64-position chunk, register batches (above).
//    Used for row slices < 2 KiB (e.g. the 4-/8-way dim-sharded group) and
//    for the dense-accumulating key gradients.
//  * seg_pipe_kernel (further below): persistent and warp-specialised (chunks
//    drawn from a global work ticket), rows staged in shared memory by
//    cp.async.bulk; used for the bag backward when
//    a row slice spans >= 2 KiB (C2: 4 KiB rows).  Same pieces and the same
//    position order inside each dV row (identical dV); the dw dot products
//    group their partial sums by thread width (equal up to rounding).
#include "internal.cuh"

#include <type_traits>

#include <algorithm>
#include <cstdlib>

namespace ml {
namespace {

struct SegParams {
  const int32_t* skey; const int32_t* spos; int64_t P;
  const int32_t* rid; const int32_t* run_begin; const int32_t* piece_base;
  const float* w;
  const char* src; int64_t lds_bytes; int32_t src_col0; int32_t B;
  const char* V; int64_t ldv_bytes; int32_t v_col0;
  float* dw_part;
  float* out; int64_t ldo; int dense;
  int out_bf16;      // dV rows stored as bf16 (fp32 accumulation, one rounding per element)
  float* partial; int32_t* counters; int64_t nslots_cap;
  int32_t* ticket;   // work-item counter of the persistent kernel (zeroed)
  int32_t vec_units;  // 16-byte vectors per row (whole dv)
  int32_t row_limit;  // keys >= row_limit (sorted last) are skipped (sentinels)
};

constexpr int kChunk = 64;                   // positions whose pieces a team owns
constexpr int kMeta = kChunk + kPieceLen;    // positions a team may touch

// Butterfly "transpose" reduction of N per-lane values across the warp:
// after it, lane l holds in a[0] the warp total of value index
// (l >> (5 - log2 N)) & (N - 1).  N - 1 + 5 - log2 N shuffles instead of 5 N.
template <int N, int O>
struct TransposeReduce {
  __device__ __forceinline__ static void run(float* a, int lane) {
    const bool up = (lane & O) != 0;
#pragma unroll
    for (int i = 0; i < N / 2; ++i) {
      const float lo = a[i], hi = a[i + N / 2];
      const float keep = up ? hi : lo;
      const float send = up ? lo : hi;
      a[i] = keep + __shfl_xor_sync(0xffffffffu, send, O);
    }
    TransposeReduce<N / 2, O / 2>::run(a, lane);
  }
};
template <int O>
struct TransposeReduce<1, O> {
  __device__ __forceinline__ static void run(float* a, int) {
#pragma unroll
    for (int o = O; o > 0; o >>= 1) a[0] += __shfl_xor_sync(0xffffffffu, a[0], o);
  }
};

__device__ __forceinline__ void st_v8(float* o, const float* a) {
  asm volatile(
      "{\n .reg .b64 pol;\n createpolicy.fractional.L2::evict_first.b64 pol, 1.0;\n"
      " st.global.L2::cache_hint.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8}, pol;\n}" ::"l"(o),
               "r"(__float_as_uint(a[0])), "r"(__float_as_uint(a[1])), "r"(__float_as_uint(a[2])),
               "r"(__float_as_uint(a[3])), "r"(__float_as_uint(a[4])), "r"(__float_as_uint(a[5])),
               "r"(__float_as_uint(a[6])), "r"(__float_as_uint(a[7]))
               : "memory");
}
// Write (or add into) this thread's VEC fp32 outputs; with bf16 sources each
// thread owns 32 contiguous bytes: one 256-bit store (full sectors).
template <int VEC, bool WIDE = true>
__device__ __forceinline__ void store_vec(float* o, const float* acc, bool dense) {
  if constexpr (VEC % 8 == 0 && WIDE) {
#pragma unroll
    for (int h = 0; h < VEC; h += 8) {
      if (dense) {
        const float4 b0 = *reinterpret_cast<const float4*>(o + h);
        const float4 b1 = *reinterpret_cast<const float4*>(o + h + 4);
        float c[8] = {acc[h] + b0.x, acc[h + 1] + b0.y, acc[h + 2] + b0.z, acc[h + 3] + b0.w,
                      acc[h + 4] + b1.x, acc[h + 5] + b1.y, acc[h + 6] + b1.z, acc[h + 7] + b1.w};
        st_v8(o + h, c);
      } else {
        st_v8(o + h, acc + h);
      }
    }
  } else {
#pragma unroll
    for (int v = 0; v < VEC; v += 4) {
      float4 a = make_float4(acc[v], acc[v + 1], acc[v + 2], acc[v + 3]);
      if (dense) {
        const float4 b = *reinterpret_cast<const float4*>(o + v);
        a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
      }
      *reinterpret_cast<float4*>(o + v) = a;
    }
  }
}

// One finished output row slice: fp32 (optionally added into a dense table),
// or rounded once to bf16 (grad_dtype = ML_BF16; half the dV bytes).
template <int VEC, bool WIDE = true, bool OBF = false, bool MAYBE_DENSE = true>
__device__ __forceinline__ void store_out(const SegParams& p, int64_t row, int64_t col,
                                          const float* acc) {
  // MAYBE_DENSE = false (the pipelined kernel, never launched in dense mode):
  // the dense read-add-write path is compiled out (with a runtime p.dense the
  // 1-2 KiB-row kernel measured 1.66 vs 1.35 ms)
  // OBF is a template parameter: the fp32 kernels carry no trace of the bf16
  // path (a runtime branch cost the 1-2 KiB-row pipelined kernel 27 %: spills)
  static_assert(!OBF || VEC % 8 == 0, "bf16 rows are stored 8 elements at a time");
  if constexpr (OBF) {
    {
      __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(p.out) + row * p.ldo + col;
#pragma unroll
      for (int h = 0; h < VEC; h += 8) {
        const uint4 u = make_uint4(f2_to_bf2(acc[h], acc[h + 1]), f2_to_bf2(acc[h + 2], acc[h + 3]),
                                   f2_to_bf2(acc[h + 4], acc[h + 5]), f2_to_bf2(acc[h + 6], acc[h + 7]));
        asm volatile(
            "{\n .reg .b64 pol;\n createpolicy.fractional.L2::evict_first.b64 pol, 1.0;\n"
            " st.global.L2::cache_hint.v4.b32 [%0], {%1,%2,%3,%4}, pol;\n}" ::"l"(o + h),
            "r"(u.x), "r"(u.y), "r"(u.z), "r"(u.w)
            : "memory");
      }
      return;
    }
  }
  store_vec<VEC, WIDE>(p.out + row * p.ldo + col, acc, MAYBE_DENSE && p.dense != 0);
}

// Piece of a run longer than kPieceLen: park the partial; pieces are combined
// in two fixed-order levels so a hot row (e.g. 50 % of all positions) is not
// summed by one CTA: the last piece to arrive in each group of 32 pieces sums
// the group, the last group to finish sums the group partials.  Fixed order ->
// bitwise deterministic.  counters: [2][nslots_cap] per slice, zeroed.
template <int VEC>
struct FVec { float v[VEC]; };

template <int VEC>
__device__ __forceinline__ void sum_slots(const SegParams& p, int slice, int64_t slice_w,
                                          int32_t first, int32_t count, int32_t stride,
                                          bool act, float* tot, int ttid) {
#pragma unroll
  for (int v = 0; v < VEC; ++v) tot[v] = 0.f;
  if (!act) return;
  for (int32_t q = 0; q < count; ++q) {
    const float* srcp = p.partial + (int64_t(slice) * p.nslots_cap + first + q * stride) * slice_w +
                        ttid * VEC;
#pragma unroll
    for (int v = 0; v < VEC; v += 4) {
      const float4 a = __ldcg(reinterpret_cast<const float4*>(srcp + v));
      tot[v] += a.x; tot[v + 1] += a.y; tot[v + 2] += a.z; tot[v + 3] += a.w;
    }
  }
}

// Barrier over the reducing threads: the whole CTA (SYNC 0), the consumer
// warps of the pipelined kernel (SYNC 1: named barrier 1, the producer warps
// never join), or one warp (SYNC 2: the warp-per-chunk kernel).
template <int SYNC>
__device__ __forceinline__ void team_sync(int team) {
  if constexpr (SYNC == 1) asm volatile("bar.sync 1, %0;" ::"r"(team) : "memory");
  else if constexpr (SYNC == 2) __syncwarp();
  else __syncthreads();
}
template <int SYNC>
__device__ __forceinline__ int team_tid() {
  if constexpr (SYNC == 2) return int(threadIdx.x & 31);
  else return int(threadIdx.x);
}

template <int VEC, int SYNC = 0, bool OBF = false, bool MAYBE_DENSE = true>
__device__ __forceinline__ void finish_long_piece(const SegParams& p, const FVec<VEC> accv, bool act,
                                               int64_t col, int slice, int32_t row, int32_t rbb,
                                               int32_t re, int32_t ps, int* s_flag, int team) {
  constexpr int L = kPieceLen;
  constexpr int GRP = 32;
  const float* acc = accv.v;
  const int64_t slice_w = int64_t(team) * VEC;
  const int32_t base = p.piece_base[rbb];
  const int32_t piece = (ps - rbb) / L;
  const int32_t npieces = (re - rbb + L - 1) / L;
  const int32_t ngroups = (npieces + GRP - 1) / GRP;
  const int32_t grp = piece / GRP;
  const int32_t g0 = grp * GRP;
  const int32_t gn = min(GRP, npieces - g0);
  int32_t* cnt1 = p.counters + int64_t(slice) * 2 * p.nslots_cap;
  int32_t* cnt2 = cnt1 + p.nslots_cap;
  const int ttid = team_tid<SYNC>();
  float* pp = p.partial + (int64_t(slice) * p.nslots_cap + base + piece) * slice_w + ttid * VEC;
  if (act) {
#pragma unroll
    for (int v = 0; v < VEC; v += 4)
      __stcg(reinterpret_cast<float4*>(pp + v), make_float4(acc[v], acc[v + 1], acc[v + 2], acc[v + 3]));
  }
  __threadfence();
  team_sync<SYNC>(team);
  if (ttid == 0) *s_flag = atomicAdd(cnt1 + base + g0, 1) == gn - 1;
  team_sync<SYNC>(team);
  if (*s_flag) {                       // last piece of its group: sum the group
    __threadfence();
    float tot[VEC];
    sum_slots<VEC>(p, slice, slice_w, base + g0, gn, 1, act, tot, ttid);
    if (ngroups == 1) {
      if (act) store_out<VEC, false, OBF, MAYBE_DENSE>(p, row, col, tot);
    } else {
      team_sync<SYNC>(team);                 // every thread has read the group's slots
      float* gp = p.partial + (int64_t(slice) * p.nslots_cap + base + g0) * slice_w + ttid * VEC;
      if (act) {
#pragma unroll
        for (int v = 0; v < VEC; v += 4)
          __stcg(reinterpret_cast<float4*>(gp + v), make_float4(tot[v], tot[v + 1], tot[v + 2], tot[v + 3]));
      }
      __threadfence();
      team_sync<SYNC>(team);
      if (ttid == 0) *s_flag = atomicAdd(cnt2 + base, 1) == ngroups - 1;
      team_sync<SYNC>(team);
      if (*s_flag) {                   // last group: sum the group partials in order
        __threadfence();
        sum_slots<VEC>(p, slice, slice_w, base, ngroups, GRP, act, tot, ttid);
        if (act) store_out<VEC, false, OBF, MAYBE_DENSE>(p, row, col, tot);
      }
    }
  }
  team_sync<SYNC>(team);
}

// Out-of-line copy for the pipelined kernel: keeping the rare long-run path
// out of its hot loop leaves the consumer's registers to the batch (measured:
// 2.50 ms out of line vs 2.58 ms inlined at C2); the one-CTA-per-chunk kernel
// inlines it (2.65 vs 2.81 ms at the 8-way group shape).
template <typename T, int VEC, int SYNC, bool OBF = false>
__device__ __noinline__ void finish_long_piece_ool(const SegParams& p, const FVec<VEC> accv,
                                                   bool act, int64_t col, int slice, int32_t row,
                                                   int32_t rbb, int32_t re, int32_t ps, int* s_flag,
                                                   int team) {
  finish_long_piece<VEC, SYNC, OBF, false>(p, accv, act, col, slice, row, rbb, re, ps, s_flag, team);
}

// blockDim.x = row vectors of one column slice (32..256); one CTA per chunk.
// DENSE: rows added into a dense table (the key gradient, sentinel keys
// >= row_limit skipped); else compact rows (the value gradient) -- a compile-
// time split so the value path carries neither the dense nor the sentinel code
template <typename T, bool DW, bool OBF = false, bool DENSE = false>
__global__ void __launch_bounds__(256, 2) seg_kernel(SegParams p) {
  constexpr int VEC = Vec<T>::N;
  constexpr int NB = 8;                  // positions per batch
  constexpr int L = kPieceLen;
  __shared__ int s_t[kMeta], s_key[kMeta], s_fl[kMeta], s_pos[kMeta];
  __shared__ float s_w[kMeta];
  __shared__ int s_rr[kMeta], s_rb[kMeta], s_re[kMeta];
  __shared__ int s_range[2];
  __shared__ int s_flag;
  __shared__ float s_red[2][8][NB];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const int slice = blockIdx.y;
  const int64_t c0 = int64_t(blockIdx.x) * kChunk;
  // sentinel keys sort last: a chunk that starts on one has nothing to do
  if (DENSE && c0 < p.P && p.skey[c0] >= p.row_limit) return;
  if (tid == 0) {
    s_range[0] = 0x7fffffff;
    s_range[1] = -1;
  }
  __syncthreads();
  // ---- decode the metadata of positions [c0, c0 + kMeta) once
  for (int k = tid; k < kMeta; k += blockDim.x) {
    const int64_t i = c0 + k;
    int fl = 0, t = 0, key = 0, pos = 0, r = 0, rb = 0, re = 0;
    float w = 0.f;
    if (i < p.P && (!DENSE || p.skey[i] < p.row_limit)) {
      pos = p.spos[i];
      const bool clamped = pos < 0;   // index outside [0, N): row 0, weight 0
      pos &= ~kClampedPos;
      key = p.skey[i];
      r = p.rid[i];
      w = clamped ? 0.f : p.w[pos];
      t = pos / p.B;
      rb = p.run_begin[r];
      re = p.run_begin[r + 1];
      const int32_t ps = rb + ((int32_t(i) - rb) / L) * L;
      const int32_t pe = min(re, ps + L);
      fl = (int32_t(i) == ps ? 1 : 0) | (int32_t(i) == pe - 1 ? 2 : 0);
      if ((fl & 1) && k < kChunk) {   // a piece starting in this chunk
        atomicMin(&s_range[0], k);
        atomicMax(&s_range[1], int(pe - c0));
      }
    }
    s_t[k] = t; s_key[k] = key; s_fl[k] = fl; s_pos[k] = pos; s_w[k] = w;
    s_rr[k] = r; s_rb[k] = rb; s_re[k] = re;
  }
  __syncthreads();
  const int k_first = s_range[0], k_end = s_range[1];
  if (k_end < 0) return;  // the whole chunk continues a piece begun earlier

  const int u = slice * blockDim.x + tid;
  const bool act = u < p.vec_units;
  const int64_t col = int64_t(u) * VEC;
  const char* srcb = p.src + (int64_t(p.src_col0) + col) * int64_t(sizeof(T));
  const char* vb = DW ? p.V + (int64_t(p.v_col0) + col) * int64_t(sizeof(T)) : nullptr;
  const uint32_t lds = uint32_t(p.lds_bytes);
  const uint64_t ldv = uint64_t(p.ldv_bytes);

  constexpr int V2 = VEC / 2;
  // dy (bag backward) is re-read ~B times: keep it in L2; the query rows of the
  // key backward are not (default policy)
  const uint64_t pol_keep = DW ? l2_evict_last_policy() : 0;
  const uint64_t pol_stream = l2_evict_first_policy();  // V: read once per piece
  float2 acc[V2], g[V2];
#pragma unroll
  for (int v = 0; v < V2; ++v) acc[v] = g[v] = make_float2(0.f, 0.f);
  int buf = 0;

  for (int kb = k_first; kb < k_end; kb += NB) {
    uint4 d[NB];
    uint4 vr[DW ? NB : 1];
    int fl[NB];
#pragma unroll
    for (int j = 0; j < NB; ++j) {  // all loads of the batch first (clamped past the end)
      const int k = min(kb + j, k_end - 1);
      fl[j] = s_fl[k];
      const char* sp = srcb + uint64_t(uint32_t(s_t[k])) * lds;
      d[j] = make_uint4(0, 0, 0, 0);
      if (act) d[j] = DW ? ldg_nc_v4_hint(sp, pol_keep) : __ldg(reinterpret_cast<const uint4*>(sp));
      if constexpr (DW) {
        vr[j] = make_uint4(0, 0, 0, 0);
        if (act && (fl[j] & 1))     // value row: only at piece starts
          vr[j] = ldg_nc_v4_hint(vb + uint64_t(uint32_t(s_key[k])) * ldv, pol_stream);
      }
    }
    float part[NB];
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      part[j] = 0.f;
      const int k = kb + j;
      if (k >= k_end) continue;              // uniform across the team
      if (fl[j] & 1) {                       // piece start: reset, unpack its value row
#pragma unroll
        for (int v = 0; v < V2; ++v) acc[v] = make_float2(0.f, 0.f);
        if constexpr (DW) Vec<T>::load(vr[j], reinterpret_cast<float*>(g));
      }
      float2 f[V2];
      Vec<T>::load(d[j], reinterpret_cast<float*>(f));
      const float wv = s_w[k];
      const float2 w2 = make_float2(wv, wv);
      if constexpr (DW) {
        float2 pr = make_float2(0.f, 0.f);
#pragma unroll
        for (int v = 0; v < V2; ++v) pr = ffma2(f[v], g[v], pr);
        part[j] = pr.x + pr.y;
      }
#pragma unroll
      for (int v = 0; v < V2; ++v) acc[v] = ffma2(w2, f[v], acc[v]);
      if (fl[j] & 2) {                       // last position of a piece
        const int32_t rr = s_rr[k], rb = s_rb[k], re = s_re[k];
        const int32_t row = DENSE ? s_key[k] : rr;
        const float* accf = reinterpret_cast<const float*>(acc);
        if (re - rb <= L) {
          if (act) store_out<VEC, true, OBF, DENSE>(p, row, col, accf);
        } else {
          const int32_t i = int32_t(c0) + k;
          const int32_t ps = rb + ((i - rb) / L) * L;
          FVec<VEC> av;
#pragma unroll
          for (int v = 0; v < VEC; ++v) av.v[v] = accf[v];
          finish_long_piece<VEC, 0, OBF, DENSE>(p, av, act, col, slice, row, rb, re, ps, &s_flag, blockDim.x);
        }
      }
    }
    if constexpr (DW) {
      TransposeReduce<NB, 16>::run(part, lane);   // lane l: warp sum of slot (l >> 2) & 7
      if ((lane & 3) == 0) s_red[buf][warp][lane >> 2] = part[0];
      __syncthreads();
      if (tid < NB && kb + tid < k_end) {
        float t = 0.f;
        for (int w2 = 0; w2 < nwarps; ++w2) t += s_red[buf][w2][tid];
        p.dw_part[int64_t(slice) * p.P + s_pos[kb + tid]] = t;
      }
      buf ^= 1;
    }
  }
}

// ---------------------------------------------------------------------------
// Pipelined variant (bag backward, dense_accumulate == false): a persistent CTA
// per SM walks work items (slice-major: all chunks of column slice 0, then
// slice 1, ... so the GPU-wide working set of dy stays one slice wide).  One
// producer warp decodes each chunk's metadata into a 2-stage shared ring and
// issues one bulk copy (cp.async.bulk, 1-D TMA) per position for the dy row
// slice, plus the value row slice at piece starts, into a ring of nslots
// shared-memory row slots completed by mbarrier transaction counts.  The
// consumer warps (one 16-byte vector per thread, as in seg_kernel) read rows
// from shared memory: the copies of the next ~nslots positions are in flight
// while a batch is reduced, instead of one register batch per round trip.
constexpr uint32_t kSegSpin = 1u << 28;   // bounded waits: trap instead of hanging
constexpr int kMetaStages = 3;

struct SegMeta { int t, key, fl, pos, rr, rb, re; float w; };

__device__ __forceinline__ uint32_t sm_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sm_addr(b)), "r"(n));
}
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sm_addr(b)) : "memory");
}
__device__ __forceinline__ void bar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sm_addr(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t parity) {
  const uint32_t a = sm_addr(b);
  uint32_t ok = 0, n = 0;
  while (true) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
    if (ok) return;
    if (++n > kSegSpin) __trap();
  }
}
// waits of the metadata / copy-issue warps: back off so their spinning does
// not take issue slots from the consumer warps
__device__ __forceinline__ void bar_wait_sleep(uint64_t* b, uint32_t parity) {
  const uint32_t a = sm_addr(b);
  uint32_t ok = 0, n = 0;
  while (true) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
    if (ok) return;
    if (++n > kSegSpin) __trap();
    __nanosleep(64);
  }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b,
                                         uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], "
      "%2, [%3], %4;" ::"r"(sm_addr(dst)),
      "l"(src), "r"(bytes), "r"(sm_addr(b)), "l"(pol)
      : "memory");
}

// dynamic smem: [2*nslots] mbarriers (full, empty), pad to 128, nslots x (dy, V) row slots.
// UPT = 16-byte row vectors per consumer thread, NB = positions per batch / stage.
template <typename T, bool DW, int UPT, int NB, int CT, int TEAM, bool OBF = false>
__global__ void __launch_bounds__(TEAM + 64, CT)
    seg_pipe_kernel(SegParams p, int nslots, int64_t nchunks, int nslices) {
  constexpr int VEC = Vec<T>::N;
  constexpr int TV = VEC * UPT;                 // elements per consumer thread
  constexpr int L = kPieceLen;
  constexpr int MS = kMetaStages;
  __shared__ SegMeta s_meta[MS][kMeta];
  __shared__ int s_rng[MS][2];
  __shared__ int s_item[MS];                    // work item of each metadata stage, -1 = done
  __shared__ uint64_t s_mfull[MS], s_mempty[MS];
  __shared__ int s_flag;
  extern __shared__ __align__(128) unsigned char dsm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(dsm);
  uint64_t* empty = full + nslots;
  const int team = blockDim.x - 64;             // consumer threads (+ issue warp + metadata warp)
  const int cwarps = team >> 5;
  const int slice_units = min(team * UPT, p.vec_units);
  const uint32_t RB = uint32_t(slice_units) * 16u;   // bytes of one row slice
  // nslots = stages of NB positions: [NB dy row slices][NB value row slices]
  unsigned char* rows = dsm + ((2 * nslots * 8 + 127) / 128) * 128;
  auto slot_dy = [&](int sl, int j) { return rows + (size_t(sl) * 2 * NB + j) * RB; };
  auto slot_v = [&](int sl, int j) { return rows + (size_t(sl) * 2 * NB + NB + j) * RB; };

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int i = 0; i < nslots; ++i) { bar_init(&full[i], 1); bar_init(&empty[i], cwarps); }
    for (int i = 0; i < MS; ++i) { bar_init(&s_mfull[i], 32); bar_init(&s_mempty[i], cwarps + 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t items = nchunks * nslices;

  if (warp == cwarps + 1) {
    // --------------------------------------------- metadata warp (runs ahead)
    // Work items are taken from a global ticket (dynamic: CTAs that start late
    // behind a concurrent kernel, or draw cheap chunks, take more items).
    for (int it = 0;; ++it) {
      int64_t w = 0;
      if (lane == 0) w = atomicAdd(p.ticket, 1);
      w = __shfl_sync(0xffffffffu, w, 0);
      const int ms = it % MS;
      const uint32_t mu = uint32_t(it / MS);
      if (mu > 0) bar_wait_sleep(&s_mempty[ms], (mu - 1) & 1);
      if (w >= items) {
        if (lane == 0) s_item[ms] = -1;
        __syncwarp();
        bar_arrive(&s_mfull[ms]);
        break;
      }
      const int64_t c0 = (w % nchunks) * kChunk;
      int kmin = 0x7fffffff, kmax = -1;
#pragma unroll
      for (int r = 0; r < (kMeta + 31) / 32; ++r) {
        const int k = lane + 32 * r;
        if (k >= kMeta) break;
        const int64_t i = c0 + k;
        SegMeta m{0, 0, 0, 0, 0, 0, 0, 0.f};
        if (i < p.P) {
          m.pos = p.spos[i];
          const bool clamped = m.pos < 0;   // index outside [0, N): row 0, weight 0
          m.pos &= ~kClampedPos;
          m.key = p.skey[i];
          m.rr = p.rid[i];
          m.w = clamped ? 0.f : p.w[m.pos];
          m.t = m.pos / p.B;
          m.rb = p.run_begin[m.rr];
          m.re = p.run_begin[m.rr + 1];
          const int32_t ps = m.rb + ((int32_t(i) - m.rb) / L) * L;
          const int32_t pe = min(m.re, ps + L);
          m.fl = (int32_t(i) == ps ? 1 : 0) | (int32_t(i) == pe - 1 ? 2 : 0);
          if ((m.fl & 1) && k < kChunk) {
            kmin = min(kmin, k);
            kmax = max(kmax, int(pe - c0));
          }
        }
        s_meta[ms][k] = m;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        kmin = min(kmin, __shfl_xor_sync(0xffffffffu, kmin, o));
        kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
      }
      if (lane == 0) { s_rng[ms][0] = kmin; s_rng[ms][1] = kmax; s_item[ms] = int(w); }
      __syncwarp();
      bar_arrive(&s_mfull[ms]);                 // 32 arrivals: every lane's writes released
    }
    return;
  }
  if (warp == cwarps) {
    // ------------------------------------------------ copy-issue warp: lane 0
    // arms each stage's barrier, lane j issues position j's copies
    const uint64_t pol_keep = l2_evict_last_policy();     // dy: re-read ~B times
    const uint64_t pol_stream = l2_evict_first_policy();  // V: once per piece
    const uint32_t lds = uint32_t(p.lds_bytes);
    const uint64_t ldv = uint64_t(p.ldv_bytes);
    int ps_slot = 0;            // next stage, its phase, whether the ring has wrapped once
    uint32_t ps_phase = 0;
    bool ps_used = false;
    for (int it = 0;; ++it) {
      const int ms = it % MS;
      bar_wait_sleep(&s_mfull[ms], uint32_t(it / MS) & 1);
      const int w = s_item[ms];
      if (w < 0) break;
      const int slice = int(w / nchunks);
      const int kmin = s_rng[ms][0], kmax = s_rng[ms][1];
      const char* srcb = p.src + (int64_t(p.src_col0) + int64_t(slice) * team * TV) * int64_t(sizeof(T));
      const char* vb = DW ? p.V + (int64_t(p.v_col0) + int64_t(slice) * team * TV) * int64_t(sizeof(T))
                          : nullptr;
      for (int kb = kmin; kb < kmax; kb += NB) {   // one stage per consumer batch
        const int sl = ps_slot;
        if (ps_used) bar_wait_sleep(&empty[sl], ps_phase ^ 1u);
        if (++ps_slot == nslots) { ps_slot = 0; ps_phase ^= 1u; ps_used = true; }
        const int nb = min(NB, kmax - kb);
        uint32_t rows_in = uint32_t(nb);
        if constexpr (DW) {
          for (int j = 0; j < nb; ++j) rows_in += uint32_t(s_meta[ms][kb + j].fl & 1);
        }
        if (lane == 0) bar_expect_tx(&full[sl], rows_in * RB);
        __syncwarp();
        if (lane < nb) {
          const SegMeta& m = s_meta[ms][kb + lane];
          bulk_g2s(slot_dy(sl, lane), srcb + uint64_t(uint32_t(m.t)) * lds, RB, &full[sl], pol_keep);
          if (DW && (m.fl & 1))
            bulk_g2s(slot_v(sl, lane), vb + uint64_t(uint32_t(m.key)) * ldv, RB, &full[sl], pol_stream);
        }
      }
      __syncwarp();
      if (lane == 0) bar_arrive(&s_mempty[ms]);   // done reading this chunk's metadata
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  const bool act = tid * UPT < slice_units;
  constexpr int V2 = TV / 2;
  constexpr int LG = NB == 8 ? 3 : (NB == 4 ? 2 : 1);
  static_assert(NB == (1 << LG), "NB must be 2, 4 or 8");
  float2 acc[V2], g[V2];
#pragma unroll
  for (int v = 0; v < V2; ++v) acc[v] = g[v] = make_float2(0.f, 0.f);
  int cs_slot = 0;               // stage of the next batch and its full-barrier phase
  uint32_t cs_phase = 0;
  for (int it = 0;; ++it) {
    const int ms = it % MS;
    bar_wait(&s_mfull[ms], uint32_t(it / MS) & 1);
    const int w = s_item[ms];
    if (w < 0) break;
    const int slice = int(w / nchunks);
    const int64_t c0 = (w % nchunks) * kChunk;
    const SegMeta* M = s_meta[ms];
    const int k_first = s_rng[ms][0], k_end = s_rng[ms][1];
    const int64_t col = int64_t(slice) * team * TV + int64_t(tid) * TV;
    for (int kb = k_first; kb < k_end; kb += NB) {
      const int nb = min(NB, k_end - kb);
      bar_wait(&full[cs_slot], cs_phase);
      // every thread reads its UPT x 16 bytes of each row slot at use (value
      // slots not filled this batch hold stale data that is never selected;
      // threads past a narrow slice read the padding after the ring).  The
      // per-position work is branch-free except for long-run pieces, so the
      // unrolled batch schedules as one block.
      const unsigned char* sd = slot_dy(cs_slot, 0) + tid * 16 * UPT;
      const unsigned char* sv = slot_v(cs_slot, 0) + tid * 16 * UPT;
      float part[NB];
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        part[j] = 0.f;
        if (j >= nb) continue;
        const int k = kb + j;
        const int flj = M[k].fl;
        const float wv = M[k].w;
        const bool st = (flj & 1) != 0;
        float2 f[V2];
#pragma unroll
        for (int u = 0; u < UPT; ++u)
          Vec<T>::load(*reinterpret_cast<const uint4*>(sd + size_t(j) * RB + u * 16),
                       reinterpret_cast<float*>(f) + u * VEC);
        if constexpr (DW) {
          float2 gn[V2];
#pragma unroll
          for (int u = 0; u < UPT; ++u)
            Vec<T>::load(*reinterpret_cast<const uint4*>(sv + size_t(j) * RB + u * 16),
                         reinterpret_cast<float*>(gn) + u * VEC);
#pragma unroll
          for (int v = 0; v < V2; ++v) {
            g[v].x = st ? gn[v].x : g[v].x;
            g[v].y = st ? gn[v].y : g[v].y;
          }
          float2 pr = make_float2(0.f, 0.f);
#pragma unroll
          for (int v = 0; v < V2; ++v) pr = ffma2(f[v], g[v], pr);
          part[j] = act ? pr.x + pr.y : 0.f;   // threads past the slice read padding
        }
        // acc is zero at every piece start: it is cleared after each piece's
        // flush below (pieces are contiguous and every chunk starts on one)
        const float2 w2 = make_float2(wv, wv);
#pragma unroll
        for (int v = 0; v < V2; ++v) acc[v] = ffma2(w2, f[v], acc[v]);
        if (flj & 2) {
          const int32_t rr = M[k].rr, rb = M[k].rb, re = M[k].re;
          const float* accf = reinterpret_cast<const float*>(acc);
          if (re - rb <= L) {
            if (act) store_out<TV, true, OBF, false>(p, rr, col, accf);
          } else {
            const int32_t i = int32_t(c0) + k;
            const int32_t ps = rb + ((i - rb) / L) * L;
            FVec<TV> av;
#pragma unroll
            for (int v = 0; v < TV; ++v) av.v[v] = accf[v];
            finish_long_piece_ool<T, TV, 1, OBF>(p, av, act, col, slice, rr, rb, re, ps, &s_flag, team);
          }
#pragma unroll
          for (int v = 0; v < V2; ++v) acc[v] = make_float2(0.f, 0.f);
        }
      }
      __syncwarp();
      if (lane == 0) bar_arrive(&empty[cs_slot]);
      if (++cs_slot == nslots) { cs_slot = 0; cs_phase ^= 1u; }
      if constexpr (DW) {
        // each consumer warp writes its own partial dot products (dw part
        // slice * kDwWarps + warp): no cross-warp exchange or barrier per batch
        TransposeReduce<NB, 16>::run(part, lane);   // lane l: warp sum of slot l >> (5 - LG)
        const int jj = lane >> (5 - LG);
        if ((lane & ((32 >> LG) - 1)) == 0 && jj < nb)
          p.dw_part[(int64_t(slice) * kDwWarps + warp) * p.P + M[kb + jj].pos] = part[0];
      }
    }
    __syncwarp();
    if (lane == 0) bar_arrive(&s_mempty[ms]);
  }
}

__global__ void sum_slices_kernel(const float* part, int ns, int64_t P, float* dw) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= P) return;
  float t = 0.f;
  for (int s = 0; s < ns; ++s) t += part[int64_t(s) * P + i];
  dw[i] = t;
}

// team size: one thread per 16-byte row vector, 32..256 threads
static int team_cap() {
  static const int v = [] {
    const char* e = std::getenv("ML_SEG_TEAM");
    const int c = e ? std::atoi(e) : 256;
    return (c == 32 || c == 64 || c == 128) ? c : 256;
  }();
  return v;
}
int team_threads(int64_t vu) {
  const int cap = team_cap();
  return vu <= 32 ? 32 : (vu >= cap ? cap : int(vu));
}

template <typename T>
mlStatus dispatch_seg(int threads, bool dw, dim3 grid, const SegParams& p, cudaStream_t s,
                      const char* name) {
  if constexpr (std::is_same<T, __nv_bfloat16>::value) {
    if (p.out_bf16) {
      if (dw) seg_kernel<T, true, true><<<grid, threads, 0, s>>>(p);
      else seg_kernel<T, false, true><<<grid, threads, 0, s>>>(p);
      ML_LAUNCH_CHECK(name);
      return ML_OK;
    }
  }
  if (p.dense) {
    if (dw) seg_kernel<T, true, false, true><<<grid, threads, 0, s>>>(p);
    else seg_kernel<T, false, false, true><<<grid, threads, 0, s>>>(p);
  } else {
    if (dw) seg_kernel<T, true><<<grid, threads, 0, s>>>(p);
    else seg_kernel<T, false><<<grid, threads, 0, s>>>(p);
  }
  ML_LAUNCH_CHECK(name);
  return ML_OK;
}

static int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e ? std::atoi(e) : dflt;
}

// pipelined kernel. cfg 2 (default): 2 CTAs per SM, 32 bytes per consumer
// thread, batches of 4; cfg 1: 1 CTA per SM, 16 bytes per thread, batches of 8.
template <typename T, bool DW, int UPT, int NB, int CT, int TEAM, bool OBF = false>
mlStatus launch_pipe(int threads, int ns, int64_t nchunks, const SegParams& p, cudaStream_t s,
                     const char* name, int ctas, size_t budget) {
  const int team = threads / UPT;
  const int slice_units = int(std::min<int64_t>(int64_t(team) * UPT, p.vec_units));
  const size_t rb = size_t(slice_units) * 16;
  const size_t stage = 2 * size_t(NB) * rb;   // NB dy + NB value row slices
  const size_t pad = (size_t(team) * UPT - size_t(slice_units)) * 16;
  int nslots = int((budget - 128 - pad) / (stage + 16));
  nslots = std::max(2, std::min(nslots, env_int("ML_SEG_SLOTS", 64)));
  const size_t smem = ((2 * size_t(nslots) * 8 + 127) / 128) * 128 + size_t(nslots) * stage + pad;
  static bool attr = false;
  if (!attr) {
    ML_CUDA_TRY(cudaFuncSetAttribute(seg_pipe_kernel<T, DW, UPT, NB, CT, TEAM, OBF>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, int(210 * 1024)));
    attr = true;
  }
  const int64_t items = nchunks * ns;
  const unsigned grid = unsigned(std::min<int64_t>(items, int64_t(num_sms()) * ctas));
  seg_pipe_kernel<T, DW, UPT, NB, CT, TEAM, OBF><<<grid, team + 64, smem, s>>>(p, nslots, nchunks, ns);
  ML_LAUNCH_CHECK(name);
  return ML_OK;
}

template <typename T, bool DW>
mlStatus dispatch_pipe(int threads, int ns, int64_t nchunks, const SegParams& p, cudaStream_t s,
                       const char* name) {
  // 4 KiB row slices: 4 consumer warps of 32-byte threads, 2 CTAs/SM;
  // 1-2 KiB rows: 16-byte threads, 3 CTAs/SM (more rows in flight per SM)
  // both configurations run kDwWarps = 4 consumer warps (one dw partial each)
  if constexpr (std::is_same<T, __nv_bfloat16>::value) {
    if (p.out_bf16) {
      if (threads >= 256)
        return launch_pipe<T, DW, 2, 4, 2, 128, true>(threads, ns, nchunks, p, s, name, 2, 100 * 1024);
      return launch_pipe<T, DW, 1, 4, 3, 128, true>(threads, ns, nchunks, p, s, name, 3, 62 * 1024);
    }
  }
  if (threads >= 256)
    return launch_pipe<T, DW, 2, 4, 2, 128>(threads, ns, nchunks, p, s, name, 2, 100 * 1024);
  return launch_pipe<T, DW, 1, 4, 3, 128>(threads, ns, nchunks, p, s, name, 3, 62 * 1024);
}

}  // namespace

int seg_slices(int32_t dv, mlDtype dt) {
  const int64_t vu = int64_t(dv) * int64_t(dtype_size(dt)) / 16;
  return vu <= team_cap() ? 1 : int(vu / team_cap());
}

static int64_t nslots_cap(int64_t P) { return 2 * (P / kPieceLen) + 2; }

void seg_carve(Carver& c, int64_t P, int32_t dv, mlDtype dt, float** partial, int32_t** counters) {
  const int64_t vu = int64_t(dv) * int64_t(dtype_size(dt)) / 16;
  const int ns = seg_slices(dv, dt);
  const int64_t slice_w = int64_t(team_threads(vu)) * (16 / int64_t(dtype_size(dt)));
  *partial = c.take<float>(ns * nslots_cap(P) * slice_w);
  *counters = c.take<int32_t>(ns * 2 * nslots_cap(P) + 1);   // + the work ticket
}

mlStatus launch_segreduce(const SegArgs& a, cudaStream_t s) {
  if (a.P <= 0) return ML_OK;
  ML_TRY(check_cols(a.dv, a.dtype, "segreduce"));
  const int64_t vu = int64_t(a.dv) * int64_t(dtype_size(a.dtype)) / 16;
  const int threads = team_threads(vu);
  const int ns = seg_slices(a.dv, a.dtype);
  if (vu > team_cap() && vu % team_cap()) return fail(ML_ERR_CONFIG, "segreduce: row vectors must divide into slices of 256");
  if (a.P >= (int64_t(1) << 31)) return fail(ML_ERR_CONFIG, "segreduce: too many positions");
  if (a.lds * int64_t(dtype_size(a.dtype)) >= (int64_t(1) << 32))
    return fail(ML_ERR_UNSUPPORTED, "segreduce: source row pitch too large");
  SegParams p;
  p.skey = a.skey; p.spos = a.spos; p.P = a.P;
  p.rid = a.runs->rid; p.run_begin = a.runs->run_begin;
  p.piece_base = a.runs->piece_base;
  p.w = a.w;
  const int64_t es = int64_t(dtype_size(a.dtype));
  p.src = static_cast<const char*>(a.src); p.lds_bytes = a.lds * es; p.src_col0 = a.src_col0; p.B = a.B;
  p.V = static_cast<const char*>(a.V); p.ldv_bytes = a.ldv * es; p.v_col0 = a.v_col0;
  p.dw_part = a.dw_part;
  p.out = a.out; p.ldo = a.ldo; p.dense = a.dense_accumulate ? 1 : 0;
  p.out_bf16 = a.out_bf16 ? 1 : 0;
  if (a.out_bf16 && (a.dense_accumulate || a.dtype != ML_BF16))
    return fail(ML_ERR_UNSUPPORTED, "segreduce: bf16 output needs bf16 sources, no dense accumulate");
  p.partial = a.partial; p.counters = a.counters; p.nslots_cap = nslots_cap(a.P);
  p.ticket = a.counters + 2 * int64_t(ns) * p.nslots_cap;
  p.vec_units = int32_t(vu);
  p.row_limit = a.row_limit;
  if (a.row_limit != INT32_MAX && !a.dense_accumulate)
    return fail(ML_ERR_UNSUPPORTED, "segreduce: sentinel keys need the dense-accumulating form");
  timing_mark(nullptr, s);
  ML_CUDA_TRY(cudaMemsetAsync(a.counters, 0, sizeof(int32_t) * (2 * size_t(ns) * size_t(p.nslots_cap) + 1), s));
  timing_mark("memset", s);
  const int64_t nchunks = (a.P + kChunk - 1) / kChunk;
  dim3 grid{unsigned(nchunks), unsigned(ns), 1u};
  const bool dw = a.V != nullptr;
  // bulk copies need 16-byte aligned row slices (row pitches and column offsets)
  const bool aligned = p.lds_bytes % 16 == 0 && (a.src_col0 * es) % 16 == 0 &&
                       reinterpret_cast<uintptr_t>(a.src) % 16 == 0 &&
                       (!dw || (p.ldv_bytes % 16 == 0 && (a.v_col0 * es) % 16 == 0 &&
                                reinterpret_cast<uintptr_t>(a.V) % 16 == 0));
  // the pipelined kernel pays off once a row slice spans >= 4 warps (2 KiB,
  // measured); narrower slices (the 4- and 8-way dim-sharded group) keep one
  // CTA per chunk
  static const bool pipe = env_int("ML_SEG_PIPE", 1) != 0;
  const bool use_pipe = pipe && !a.dense_accumulate && aligned && threads >= 128;
  if (a.dw_slices_out) *a.dw_slices_out = use_pipe ? ns * kDwWarps : ns;
  if (use_pipe) {
    if (a.dtype == ML_BF16)
      return dw ? dispatch_pipe<__nv_bfloat16, true>(threads, ns, nchunks, p, s, a.name)
                : dispatch_pipe<__nv_bfloat16, false>(threads, ns, nchunks, p, s, a.name);
    return dw ? dispatch_pipe<float, true>(threads, ns, nchunks, p, s, a.name)
              : dispatch_pipe<float, false>(threads, ns, nchunks, p, s, a.name);
  }
  if (a.dtype == ML_BF16) return dispatch_seg<__nv_bfloat16>(threads, dw, grid, p, s, a.name);
  return dispatch_seg<float>(threads, dw, grid, p, s, a.name);
}

mlStatus launch_sum_slices(const float* part, int nslices, int64_t P, float* dw, cudaStream_t s) {
  if (P <= 0) return ML_OK;
  sum_slices_kernel<<<unsigned((P + 255) / 256), 256, 0, s>>>(part, nslices, P, dw);
  ML_LAUNCH_CHECK("sum_slices");
  return ML_OK;
}

}  // namespace ml
