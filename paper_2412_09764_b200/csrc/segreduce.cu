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
#include "internal.cuh"

namespace ml {
namespace {

struct SegParams {
  const int32_t* skey; const int32_t* spos; int64_t P;
  const int32_t* flags; const int32_t* excl; const int32_t* run_begin; const int32_t* piece_base;
  const float* w;
  const char* src; int64_t lds_bytes; int32_t src_col0; int32_t B;
  const char* V; int64_t ldv_bytes; int32_t v_col0;
  float* dw_part;
  float* out; int64_t ldo; int dense;
  float* partial; int32_t* counters; int64_t nslots_cap;
  int32_t vec_units;  // 16-byte vectors per row (whole dv)
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
  if constexpr (VEC == 8 && WIDE) {
    if (dense) {
      const float4 b0 = *reinterpret_cast<const float4*>(o);
      const float4 b1 = *reinterpret_cast<const float4*>(o + 4);
      float c[8] = {acc[0] + b0.x, acc[1] + b0.y, acc[2] + b0.z, acc[3] + b0.w,
                    acc[4] + b1.x, acc[5] + b1.y, acc[6] + b1.z, acc[7] + b1.w};
      st_v8(o, c);
    } else {
      st_v8(o, acc);
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
                                          bool act, float* tot) {
#pragma unroll
  for (int v = 0; v < VEC; ++v) tot[v] = 0.f;
  if (!act) return;
  for (int32_t q = 0; q < count; ++q) {
    const float* srcp = p.partial + (int64_t(slice) * p.nslots_cap + first + q * stride) * slice_w +
                        threadIdx.x * VEC;
#pragma unroll
    for (int v = 0; v < VEC; v += 4) {
      const float4 a = __ldcg(reinterpret_cast<const float4*>(srcp + v));
      tot[v] += a.x; tot[v + 1] += a.y; tot[v + 2] += a.z; tot[v + 3] += a.w;
    }
  }
}

template <int VEC>
__device__ __noinline__ void finish_long_piece(const SegParams& p, const FVec<VEC> accv, bool act,
                                               int64_t col, int slice, int32_t row, int32_t rbb,
                                               int32_t re, int32_t ps, int* s_flag) {
  constexpr int L = kPieceLen;
  constexpr int GRP = 32;
  const float* acc = accv.v;
  const int64_t slice_w = int64_t(blockDim.x) * VEC;
  const int32_t base = p.piece_base[rbb];
  const int32_t piece = (ps - rbb) / L;
  const int32_t npieces = (re - rbb + L - 1) / L;
  const int32_t ngroups = (npieces + GRP - 1) / GRP;
  const int32_t grp = piece / GRP;
  const int32_t g0 = grp * GRP;
  const int32_t gn = min(GRP, npieces - g0);
  int32_t* cnt1 = p.counters + int64_t(slice) * 2 * p.nslots_cap;
  int32_t* cnt2 = cnt1 + p.nslots_cap;
  float* pp = p.partial + (int64_t(slice) * p.nslots_cap + base + piece) * slice_w + threadIdx.x * VEC;
  if (act) {
#pragma unroll
    for (int v = 0; v < VEC; v += 4)
      __stcg(reinterpret_cast<float4*>(pp + v), make_float4(acc[v], acc[v + 1], acc[v + 2], acc[v + 3]));
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) *s_flag = atomicAdd(cnt1 + base + g0, 1) == gn - 1;
  __syncthreads();
  if (*s_flag) {                       // last piece of its group: sum the group
    __threadfence();
    float tot[VEC];
    sum_slots<VEC>(p, slice, slice_w, base + g0, gn, 1, act, tot);
    if (ngroups == 1) {
      if (act) store_vec<VEC, false>(p.out + int64_t(row) * p.ldo + col, tot, p.dense != 0);
    } else {
      __syncthreads();                 // every thread has read the group's slots
      float* gp = p.partial + (int64_t(slice) * p.nslots_cap + base + g0) * slice_w + threadIdx.x * VEC;
      if (act) {
#pragma unroll
        for (int v = 0; v < VEC; v += 4)
          __stcg(reinterpret_cast<float4*>(gp + v), make_float4(tot[v], tot[v + 1], tot[v + 2], tot[v + 3]));
      }
      __threadfence();
      __syncthreads();
      if (threadIdx.x == 0) *s_flag = atomicAdd(cnt2 + base, 1) == ngroups - 1;
      __syncthreads();
      if (*s_flag) {                   // last group: sum the group partials in order
        __threadfence();
        sum_slots<VEC>(p, slice, slice_w, base, ngroups, GRP, act, tot);
        if (act) store_vec<VEC, false>(p.out + int64_t(row) * p.ldo + col, tot, p.dense != 0);
      }
    }
  }
  __syncthreads();
}

// blockDim.x = row vectors of one column slice (32..256); one CTA per chunk.
template <typename T, bool DW>
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
    if (i < p.P) {
      pos = p.spos[i];
      key = p.skey[i];
      r = p.excl[i] - 1 + p.flags[i];
      w = p.w[pos];
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
        const int32_t row = p.dense ? s_key[k] : rr;
        const float* accf = reinterpret_cast<const float*>(acc);
        if (re - rb <= L) {
          if (act) store_vec<VEC>(p.out + int64_t(row) * p.ldo + col, accf, p.dense != 0);
        } else {
          const int32_t i = int32_t(c0) + k;
          const int32_t ps = rb + ((i - rb) / L) * L;
          FVec<VEC> av;
#pragma unroll
          for (int v = 0; v < VEC; ++v) av.v[v] = accf[v];
          finish_long_piece<VEC>(p, av, act, col, slice, row, rb, re, ps, &s_flag);
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

__global__ void sum_slices_kernel(const float* part, int ns, int64_t P, float* dw) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= P) return;
  float t = 0.f;
  for (int s = 0; s < ns; ++s) t += part[int64_t(s) * P + i];
  dw[i] = t;
}

// team size: one thread per 16-byte row vector, 32..256 threads
int team_threads(int64_t vu) { return vu <= 32 ? 32 : (vu >= 256 ? 256 : int(vu)); }

template <typename T>
mlStatus dispatch_seg(int threads, bool dw, dim3 grid, const SegParams& p, cudaStream_t s,
                      const char* name) {
  if (dw) seg_kernel<T, true><<<grid, threads, 0, s>>>(p);
  else seg_kernel<T, false><<<grid, threads, 0, s>>>(p);
  ML_LAUNCH_CHECK(name);
  return ML_OK;
}

}  // namespace

int seg_slices(int32_t dv, mlDtype dt) {
  const int64_t vu = int64_t(dv) * int64_t(dtype_size(dt)) / 16;
  return vu <= 256 ? 1 : int(vu / 256);
}

static int64_t nslots_cap(int64_t P) { return 2 * (P / kPieceLen) + 2; }

void seg_carve(Carver& c, int64_t P, int32_t dv, mlDtype dt, float** partial, int32_t** counters) {
  const int64_t vu = int64_t(dv) * int64_t(dtype_size(dt)) / 16;
  const int ns = seg_slices(dv, dt);
  const int64_t slice_w = int64_t(team_threads(vu)) * (16 / int64_t(dtype_size(dt)));
  *partial = c.take<float>(ns * nslots_cap(P) * slice_w);
  *counters = c.take<int32_t>(ns * 2 * nslots_cap(P));
}

mlStatus launch_segreduce(const SegArgs& a, cudaStream_t s) {
  if (a.P <= 0) return ML_OK;
  ML_TRY(check_cols(a.dv, a.dtype, "segreduce"));
  const int64_t vu = int64_t(a.dv) * int64_t(dtype_size(a.dtype)) / 16;
  const int threads = team_threads(vu);
  const int ns = seg_slices(a.dv, a.dtype);
  if (vu > 256 && vu % 256) return fail(ML_ERR_CONFIG, "segreduce: row vectors must divide into slices of 256");
  if (a.P >= (int64_t(1) << 31)) return fail(ML_ERR_CONFIG, "segreduce: too many positions");
  if (a.lds * int64_t(dtype_size(a.dtype)) >= (int64_t(1) << 32))
    return fail(ML_ERR_UNSUPPORTED, "segreduce: source row pitch too large");
  SegParams p;
  p.skey = a.skey; p.spos = a.spos; p.P = a.P;
  p.flags = a.runs->flags; p.excl = a.runs->excl; p.run_begin = a.runs->run_begin;
  p.piece_base = a.runs->piece_base;
  p.w = a.w;
  const int64_t es = int64_t(dtype_size(a.dtype));
  p.src = static_cast<const char*>(a.src); p.lds_bytes = a.lds * es; p.src_col0 = a.src_col0; p.B = a.B;
  p.V = static_cast<const char*>(a.V); p.ldv_bytes = a.ldv * es; p.v_col0 = a.v_col0;
  p.dw_part = a.dw_part;
  p.out = a.out; p.ldo = a.ldo; p.dense = a.dense_accumulate ? 1 : 0;
  p.partial = a.partial; p.counters = a.counters; p.nslots_cap = nslots_cap(a.P);
  p.vec_units = int32_t(vu);
  timing_mark(nullptr, s);
  ML_CUDA_TRY(cudaMemsetAsync(a.counters, 0, sizeof(int32_t) * 2 * size_t(ns) * size_t(p.nslots_cap), s));
  timing_mark("memset", s);
  const int64_t nchunks = (a.P + kChunk - 1) / kChunk;
  dim3 grid{unsigned(nchunks), unsigned(ns), 1u};
  const bool dw = a.V != nullptr;
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
