// Segmented reduction over sorted (key, position) runs: the atomic-free
// "reverse_indices" EmbeddingBag backward (§3.1.4):
//   dV[r, :] = sum_{p: idx[p] = r} w[p] * dy[t(p), :]        (one owner per row)
//   dw[p]    = <dy[t(p), :], V[r, :]>                          (fused: V[r] read once)
// The same kernel (without dw, dense-accumulating) produces the half-key
// gradients dK[h, a] = sum ds * q_half (pkm backward).
//
// Work split (load balance under skew, determinism): one warp per chunk of
// 32 sorted positions; it reduces every "piece" that STARTS in its chunk.  A
// piece is a whole run, or a 32-position piece of a run longer than 32.
// Whole runs are written directly (rows are unique: no atomics); pieces of
// long runs go to a partial buffer and the last piece to arrive (counter)
// sums all pieces of its run in piece order -> bitwise deterministic.
// Columns: lane l owns 16-byte vectors l, l+32 (CPL <= 2 of them) of a
// 32*CPL-vector column slice (blockIdx.y); loads are coalesced 512 B rows.
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

template <typename T, int CPL>
__device__ __forceinline__ void write_row(const SegParams& p, int64_t row, const float* acc,
                                          int slice, int lane, const bool* act) {
  constexpr int VEC = Vec<T>::N;
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    if (!act[c]) continue;
    const int64_t col = (int64_t(slice) * 32 * CPL + c * 32 + lane) * VEC;
    float* o = p.out + row * p.ldo + col;
#pragma unroll
    for (int v = 0; v < VEC; v += 4) {
      float4 a = make_float4(acc[c * VEC + v], acc[c * VEC + v + 1], acc[c * VEC + v + 2],
                             acc[c * VEC + v + 3]);
      if (p.dense) {
        float4 b = *reinterpret_cast<float4*>(o + v);
        a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
      }
      *reinterpret_cast<float4*>(o + v) = a;
    }
  }
}

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
template <int N> struct Log2 { static constexpr int v = 1 + Log2<N / 2>::v; };
template <> struct Log2<1> { static constexpr int v = 0; };

template <typename T, int CPL, bool DW>
__global__ void __launch_bounds__(256, 2) seg_kernel(SegParams p) {
  constexpr int VEC = Vec<T>::N;
  constexpr int NB = 8 / CPL;             // positions per batch of loads
  constexpr int L = kPieceLen;
  constexpr unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int64_t chunk = int64_t(blockIdx.x) * 8 + (threadIdx.x >> 5);
  const int slice = blockIdx.y;
  const int64_t c0 = chunk * 32;
  if (c0 >= p.P) return;
  const int64_t c1 = min(c0 + 32, p.P);

  // ---- per-lane metadata of position c0 + lane (one round of loads)
  const int64_t iA = c0 + lane;
  int posA = 0, keyA = 0, rA = 0, rbA = 0, reA = 0;
  float wA = 0.f;
  bool stA = false;
  if (iA < c1) {
    posA = p.spos[iA];
    keyA = p.skey[iA];
    rA = p.excl[iA] - 1 + p.flags[iA];
    wA = p.w[posA];
    rbA = p.run_begin[rA];
    reA = p.run_begin[rA + 1];
    stA = ((int32_t(iA) - rbA) % L) == 0;
  }
  unsigned starts = __ballot_sync(FULL, stA);
  if (!starts) return;  // the whole chunk continues a piece begun earlier
  // the last piece may run up to 31 positions past the chunk: prefetch those
  const int last = 31 - __clz(starts);
  const int32_t e_last = min(__shfl_sync(FULL, reA, last), int32_t(c0) + last + L);
  int posB = 0;
  float wB = 0.f;
  if (e_last > c1) {
    const int64_t iB = c1 + lane;
    if (iB < e_last) {
      posB = p.spos[iB];
      wB = p.w[posB];
    }
  }

  bool act[CPL];
  int64_t colb[CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    const int u = slice * 32 * CPL + c * 32 + lane;
    act[c] = u < p.vec_units;
    colb[c] = int64_t(u) * 16;
  }
  const int64_t slice_w = int64_t(32) * CPL * VEC;
  const int64_t src_off = int64_t(p.src_col0) * int64_t(sizeof(T));

  while (starts) {
    const int b = __ffs(starts) - 1;
    starts &= starts - 1;
    const int32_t s = int32_t(c0) + b;
    const int32_t rr = __shfl_sync(FULL, rA, b);
    const int32_t rbb = __shfl_sync(FULL, rbA, b);
    const int32_t re = __shfl_sync(FULL, reA, b);
    const int32_t key = __shfl_sync(FULL, keyA, b);
    const int32_t e = min(re, s + L);
    const bool lng = (re - rbb) > L;

    uint4 vv[CPL];
    if constexpr (DW) {
#pragma unroll
      for (int c = 0; c < CPL; ++c)
        if (act[c]) vv[c] = ldg_nc_v4(p.V + int64_t(key) * p.ldv_bytes +
                                      int64_t(p.v_col0) * int64_t(sizeof(T)) + colb[c]);
    }
    float acc[CPL * VEC];
#pragma unroll
    for (int v = 0; v < CPL * VEC; ++v) acc[v] = 0.f;

    for (int32_t pb = s; pb < e; pb += NB) {
      const int n = min(NB, e - pb);
      int posb[NB];
      float wb[NB];
      uint4 d[NB][CPL];
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        const int off = pb + j - int32_t(c0);  // 0..62
        const int src = off & 31;
        const int pa = __shfl_sync(FULL, posA, src);
        const float wa = __shfl_sync(FULL, wA, src);
        const int pbv = __shfl_sync(FULL, posB, src);
        const float wbv = __shfl_sync(FULL, wB, src);
        posb[j] = off < 32 ? pa : pbv;
        wb[j] = off < 32 ? wa : wbv;
        if (j < n) {
          const char* row = p.src + int64_t(posb[j] / p.B) * p.lds_bytes + src_off;
#pragma unroll
          for (int c = 0; c < CPL; ++c)
            if (act[c]) d[j][c] = ldg_v4(row + colb[c]);
        }
      }
      float part[NB];
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        part[j] = 0.f;
        if (j < n) {
#pragma unroll
          for (int c = 0; c < CPL; ++c) {
            if (!act[c]) continue;
            float f[VEC];
            Vec<T>::load(d[j][c], f);
            if constexpr (DW) {
              float g[VEC];
              Vec<T>::load(vv[c], g);
#pragma unroll
              for (int v = 0; v < VEC; ++v) part[j] = fmaf(f[v], g[v], part[j]);
            }
#pragma unroll
            for (int v = 0; v < VEC; ++v) acc[c * VEC + v] = fmaf(wb[j], f[v], acc[c * VEC + v]);
          }
        }
      }
      if constexpr (DW) {
        TransposeReduce<NB, 16>::run(part, lane);
        constexpr int SH = 5 - Log2<NB>::v;
        const int jj = (lane >> SH) & (NB - 1);
        int pos_mine = posb[0];
#pragma unroll
        for (int j = 1; j < NB; ++j)
          if (jj == j) pos_mine = posb[j];
        if ((lane & ((1 << SH) - 1)) == 0 && jj < n)
          p.dw_part[int64_t(slice) * p.P + pos_mine] = part[0];
      }
    }

    if (!lng) {
      write_row<T, CPL>(p, p.dense ? int64_t(key) : int64_t(rr), acc, slice, lane, act);
    } else {
      const int32_t base = p.piece_base[rbb];
      const int32_t slot = base + (s - rbb) / L;
      const int32_t npieces = (re - rbb + L - 1) / L;
      float* pp = p.partial + (int64_t(slice) * p.nslots_cap + slot) * slice_w;
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        if (!act[c]) continue;
#pragma unroll
        for (int v = 0; v < VEC; v += 4)
          __stcg(reinterpret_cast<float4*>(pp + (c * 32 + lane) * VEC + v),
                 make_float4(acc[c * VEC + v], acc[c * VEC + v + 1], acc[c * VEC + v + 2],
                             acc[c * VEC + v + 3]));
      }
      __threadfence();
      __syncwarp();
      int old = 0;
      if (lane == 0) old = atomicAdd(p.counters + int64_t(slice) * p.nslots_cap + base, 1);
      old = __shfl_sync(FULL, old, 0);
      if (old == npieces - 1) {  // last piece of this run: combine in piece order
        __threadfence();
#pragma unroll
        for (int v = 0; v < CPL * VEC; ++v) acc[v] = 0.f;
        for (int32_t q = 0; q < npieces; ++q) {
          const float* src = p.partial + (int64_t(slice) * p.nslots_cap + base + q) * slice_w;
#pragma unroll
          for (int c = 0; c < CPL; ++c) {
            if (!act[c]) continue;
#pragma unroll
            for (int v = 0; v < VEC; v += 4) {
              const float4 a = __ldcg(reinterpret_cast<const float4*>(src + (c * 32 + lane) * VEC + v));
              acc[c * VEC + v] += a.x;
              acc[c * VEC + v + 1] += a.y;
              acc[c * VEC + v + 2] += a.z;
              acc[c * VEC + v + 3] += a.w;
            }
          }
        }
        write_row<T, CPL>(p, p.dense ? int64_t(key) : int64_t(rr), acc, slice, lane, act);
      }
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

int cpl_for(int64_t vu) { return vu <= 32 ? 1 : 2; }

template <typename T>
mlStatus dispatch_seg(int cpl, bool dw, dim3 grid, const SegParams& p, cudaStream_t s,
                      const char* name) {
#define ML_SEG(C, D) seg_kernel<T, C, D><<<grid, 256, 0, s>>>(p)
  if (dw) {
    if (cpl == 1) ML_SEG(1, true); else ML_SEG(2, true);
  } else {
    if (cpl == 1) ML_SEG(1, false); else ML_SEG(2, false);
  }
#undef ML_SEG
  ML_LAUNCH_CHECK(name);
  return ML_OK;
}

}  // namespace

int seg_slices(int32_t dv, mlDtype dt) {
  const int64_t vu = int64_t(dv) * int64_t(dtype_size(dt)) / 16;
  return vu <= 64 ? 1 : int(vu / 64);
}

static int64_t nslots_cap(int64_t P) { return 2 * (P / kPieceLen) + 2; }

void seg_carve(Carver& c, int64_t P, int32_t dv, mlDtype dt, float** partial, int32_t** counters) {
  const int64_t vu = int64_t(dv) * int64_t(dtype_size(dt)) / 16;
  const int cpl = cpl_for(vu);
  const int ns = seg_slices(dv, dt);
  const int64_t slice_w = int64_t(32) * cpl * (16 / int64_t(dtype_size(dt)));
  *partial = c.take<float>(ns * nslots_cap(P) * slice_w);
  *counters = c.take<int32_t>(ns * nslots_cap(P));
}

mlStatus launch_segreduce(const SegArgs& a, cudaStream_t s) {
  if (a.P <= 0) return ML_OK;
  ML_TRY(check_cols(a.dv, a.dtype, "segreduce"));
  const int64_t vu = int64_t(a.dv) * int64_t(dtype_size(a.dtype)) / 16;
  const int cpl = cpl_for(vu);
  const int ns = seg_slices(a.dv, a.dtype);
  if (vu > 64 && vu % 64) return fail(ML_ERR_CONFIG, "segreduce: row vectors must divide into slices of 64");
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
  ML_CUDA_TRY(cudaMemsetAsync(a.counters, 0, sizeof(int32_t) * size_t(ns) * size_t(p.nslots_cap), s));
  timing_mark("memset", s);
  const int64_t nchunks = (a.P + 31) / 32;
  dim3 grid(unsigned((nchunks + 7) / 8), unsigned(ns));
  const bool dw = a.V != nullptr;
  if (a.dtype == ML_BF16) return dispatch_seg<__nv_bfloat16>(cpl, dw, grid, p, s, a.name);
  return dispatch_seg<float>(cpl, dw, grid, p, s, a.name);
}

mlStatus launch_sum_slices(const float* part, int nslices, int64_t P, float* dw, cudaStream_t s) {
  if (P <= 0) return ML_OK;
  sum_slices_kernel<<<unsigned((P + 255) / 256), 256, 0, s>>>(part, nslices, P, dw);
  ML_LAUNCH_CHECK("sum_slices");
  return ML_OK;
}

}  // namespace ml
