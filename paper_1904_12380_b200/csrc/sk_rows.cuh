// sk_rows.cuh -- K1: short rows held in registers, LPR lanes per row.
//
// Replaces, for C <= 1024, the three reference phase loops
//   _maxsub_rows_scalar  kernels.py:136-151
//   _exp_rows_scalar     kernels.py:171-174
//   _sumscale_rows_scalar kernels.py:177-189
// with one pass: each row is read from HBM once (128-bit streaming loads when
// the row pitch allows, else 64-bit for even rows on 8-B pitches, else 32-bit
// coalesced loads), reduced with
// __shfl_xor inside an aligned group of LPR lanes, and written once.
//
// Work unit: one warp owns U * (32/LPR) consecutive rows per iteration; lane
// `sl` of a row group holds vectors j*LPR+sl, j < NV, of VEC floats each, so a
// warp-wide load instruction touches (32/LPR) rows * LPR*VEC*4 contiguous bytes.
#pragma once
#include "sk_common.cuh"

namespace sk {

constexpr int kRowsThreads = 256;

template <int VEC, int LPR, int NV, int U>
struct RowBatch {
  float v[U][NV * VEC];  // element e of lane-row u sits at column col<>(e)
};

template <int VEC, int LPR>
__device__ __forceinline__ int k1_col(int e, int sl) {
  return ((e / VEC) * LPR + sl) * VEC + (e % VEC);
}

template <int VEC, int LPR, int NV, int U>
__device__ __forceinline__ void k1_load(RowBatch<VEC, LPR, NV, U>& B, const float* __restrict__ x,
                                        int64_t base, int64_t rows, int cols, int64_t ldx,
                                        int sub, int sl) {
  constexpr int RPW = 32 / LPR;
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int64_t r = base + u * RPW + sub;
    const bool rv = r < rows;
    const float* xr = x + (rv ? r : 0) * ldx;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const int c = (j * LPR + sl) * VEC;
      if (rv && c < cols) {
        if constexpr (VEC == 8) {
          float t[8];
          ld_stream8(xr + c, t);
#pragma unroll
          for (int k = 0; k < 8; ++k) B.v[u][8 * j + k] = t[k];
        } else if constexpr (VEC == 4) {
          const float4 t = ld_stream4(xr + c);
          B.v[u][4 * j] = t.x; B.v[u][4 * j + 1] = t.y;
          B.v[u][4 * j + 2] = t.z; B.v[u][4 * j + 3] = t.w;
        } else if constexpr (VEC == 2) {
          const float2 t = ld_stream2(xr + c);
          B.v[u][2 * j] = t.x; B.v[u][2 * j + 1] = t.y;
        } else {
          B.v[u][j] = ld_stream1(xr + c);
        }
      } else {
#pragma unroll
        for (int k = 0; k < VEC; ++k) B.v[u][j * VEC + k] = kPadLogit;
      }
    }
  }
}

// One batch: max -> exp -> sum -> scale -> store, all in registers.
// FULL: cols == LPR*NV*VEC, so no lane holds padding and the sum needs no mask.
template <int MODE, bool FULL, int VEC, int LPR, int NV, int U>
__device__ __forceinline__ void k1_process(RowBatch<VEC, LPR, NV, U>& B, float* __restrict__ y,
                                           int64_t base, int64_t rows, int cols, int64_t ldy,
                                           int sub, int sl, unsigned long long* bad_row,
                                           float shift_scale) {
  constexpr int RPW = 32 / LPR;
  constexpr int E = NV * VEC;
  // ---- row max (== the strict-'>' scan for finite data) + finite check
  float m[U];
  bool bad[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    float mu = kPadLogit;
    u64 z = f2pk(0.0f, 0.0f);
#pragma unroll
    for (int e = 0; e + 1 < E; e += 2) {
      mu = fmaxf(mu, fmaxf(B.v[u][e], B.v[u][e + 1]));
      z = nf_acc2(z, B.v[u][e], B.v[u][e + 1]);
    }
    if constexpr (E % 2) {
      mu = fmaxf(mu, B.v[u][E - 1]);
      z = nf_acc2(z, B.v[u][E - 1], 0.0f);
    }
    bad[u] = nf_bad(z);
    m[u] = group_max<LPR>(mu) * shift_scale;  // shift_scale = 0: fault hook
  }
  // ---- shift, clip, exp (kept in registers), row sum
  float rcp[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const bool rv = base + u * RPW + sub < rows;
    u64 acc = f2pk(0.0f, 0.0f);
#pragma unroll
    for (int e = 0; e + 1 < E; e += 2) {
      float2 ex = sexp2<MODE>(B.v[u][e], B.v[u][e + 1], m[u]);
      B.v[u][e] = ex.x;
      B.v[u][e + 1] = ex.y;
      if constexpr (!FULL) {
        if (!(rv && k1_col<VEC, LPR>(e, sl) < cols)) ex.x = 0.0f;
        if (!(rv && k1_col<VEC, LPR>(e + 1, sl) < cols)) ex.y = 0.0f;
      }
      acc = f2add(acc, f2pk(ex.x, ex.y));
    }
    float s;
    {
      const float2 a = f2up(acc);
      s = a.x + a.y;
    }
    if constexpr (E % 2) {
      float ex = sexp1<MODE>(B.v[u][E - 1], m[u]);
      B.v[u][E - 1] = ex;
      if (!FULL && !(rv && k1_col<VEC, LPR>(E - 1, sl) < cols)) ex = 0.0f;
      s += ex;
    }
    rcp[u] = recip_of_sum(group_sum<LPR>(static_cast<double>(s)));
  }
  // ---- scale (+ flush), write once
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int64_t r = base + u * RPW + sub;
    if (r >= rows) continue;
    float* yr = y + r * ldy;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const int c = (j * LPR + sl) * VEC;
      if (FULL || c < cols) {
        if constexpr (VEC == 8) {
          float o[8];
#pragma unroll
          for (int k = 0; k < 8; k += 2) {
            const float2 a = scale2<MODE>(make_float2(B.v[u][8 * j + k], B.v[u][8 * j + k + 1]),
                                          rcp[u]);
            o[k] = a.x;
            o[k + 1] = a.y;
          }
          st_stream8(yr + c, o);
        } else if constexpr (VEC == 4) {
          const float2 a = scale2<MODE>(make_float2(B.v[u][4 * j], B.v[u][4 * j + 1]), rcp[u]);
          const float2 b =
              scale2<MODE>(make_float2(B.v[u][4 * j + 2], B.v[u][4 * j + 3]), rcp[u]);
          st_stream4(yr + c, make_float4(a.x, a.y, b.x, b.y));
        } else if constexpr (VEC == 2) {
          st_stream2(yr + c, scale2<MODE>(make_float2(B.v[u][2 * j], B.v[u][2 * j + 1]), rcp[u]));
        } else {
          st_stream1(yr + c, scale1<MODE>(B.v[u][j], rcp[u]));
        }
      }
    }
  }
  // ---- non-finite input: report the smallest offending row (kernels.py:342-347)
#pragma unroll
  for (int u = 0; u < U; ++u)
    if (bad[u]) atomicMin(bad_row, static_cast<unsigned long long>(base + u * RPW + sub));
}

template <int MODE, int VEC, int LPR, int NV, int U>
__device__ __forceinline__ void k1_process_any(RowBatch<VEC, LPR, NV, U>& B,
                                               float* __restrict__ y, int64_t base,
                                               int64_t rows, int cols, int64_t ldy, int sub,
                                               int sl, unsigned long long* bad_row,
                                               float shift_scale) {
  if (cols == LPR * NV * VEC)
    k1_process<MODE, true>(B, y, base, rows, cols, ldy, sub, sl, bad_row, shift_scale);
  else
    k1_process<MODE, false>(B, y, base, rows, cols, ldy, sub, sl, bad_row, shift_scale);
}

// PF = 1: software-pipelined -- the next batch's loads are issued before the
// current batch is reduced, so each lane keeps 2*U*NV requests in flight.
// Occupancy floor: >= 3 CTAs (24 warps) per SM for the register-heavy shapes,
// >= 4 otherwise, so there are always enough warps to cover HBM latency.
template <int VEC, int NV, int U, int PF>
constexpr int k1_min_blocks() {
  return NV * VEC * U * (PF ? 2 : 1) >= 128 ? 1
         : NV * VEC * U * (PF ? 2 : 1) >= 64 ? 2
         : NV * VEC * U * (PF ? 2 : 1) >= 32 ? 3 : 4;
}

template <int MODE, int VEC, int LPR, int NV, int U, int PF>
__global__ void __launch_bounds__(kRowsThreads, (k1_min_blocks<VEC, NV, U, PF>()))
    k1_rows(const float* __restrict__ x, float* __restrict__ y, int64_t rows, int cols,
            int64_t ldx, int64_t ldy, unsigned long long* __restrict__ bad_row,
            float shift_scale) {
  static_assert(VEC == 1 || VEC == 2 || VEC == 4 || VEC == 8, "VEC");
  static_assert(LPR >= 1 && LPR <= 32 && (LPR & (LPR - 1)) == 0, "LPR");
  constexpr int ROWS_ITER = U * (32 / LPR);
  const int lane = threadIdx.x & 31;
  const int sub = lane / LPR;
  const int sl = lane % LPR;
  const int64_t gwarp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t stride = ((int64_t(gridDim.x) * blockDim.x) >> 5) * ROWS_ITER;
  pdl_wait();
  pdl_launch_dependents();

  int64_t base = gwarp * ROWS_ITER;
  if constexpr (PF) {
    if (base >= rows) return;
    RowBatch<VEC, LPR, NV, U> cur;
    k1_load(cur, x, base, rows, cols, ldx, sub, sl);
    for (; base < rows; base += stride) {
      RowBatch<VEC, LPR, NV, U> nxt;
      const bool more = base + stride < rows;
      if (more) k1_load(nxt, x, base + stride, rows, cols, ldx, sub, sl);
      k1_process_any<MODE>(cur, y, base, rows, cols, ldy, sub, sl, bad_row, shift_scale);
      if (more) cur = nxt;
    }
  } else {
    for (; base < rows; base += stride) {
      RowBatch<VEC, LPR, NV, U> cur;
      k1_load(cur, x, base, rows, cols, ldx, sub, sl);
      k1_process_any<MODE>(cur, y, base, rows, cols, ldy, sub, sl, bad_row, shift_scale);
    }
  }
}

}  // namespace sk
