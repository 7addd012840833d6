// sk_rows_mw.cuh -- K1m: medium rows (3 K .. 8 K floats) in the registers of
// WPR warps.
//
// K1 (sk_rows.cuh) gives a row to LPR lanes of one warp; past ~3 K floats a
// warp's registers run out.  K1m spreads a row over WPR warps of a 256-thread
// block (8/WPR rows per block iteration), each thread holding NV float4 of it:
// one 128-bit streaming read and one streaming write per element, like K1, and
// the row max / row sum cross warps through 32 B of shared memory and one
// __syncthreads each.  No shared-memory staging of the data (the TMA
// block-per-row K2 it replaces pays a smem round trip per element and two
// block-wide barriers per row with a quarter of the warps).
//
// Same operation order as K1 (kernels.py:136-189): row max, exp(clip(x - m))
// kept in registers, f64 row sum (lane fp32 pairs -> f64 butterfly -> WPR warp
// partials in fixed order), y = e * (1/(float)S) with the reference's flush.
// The result depends only on (WPR, NV), never on the grid, so row blocks keep
// their bits.
#pragma once
#include "sk_common.cuh"
#include "sk_rows.cuh"

namespace sk {

template <int MODE, int WPR, int NV>
__global__ void __launch_bounds__(kRowsThreads, 2)
    k1m_rows(const float* __restrict__ x, float* __restrict__ y, int64_t rows, int cols,
             int64_t ldx, int64_t ldy, unsigned long long* __restrict__ bad_row,
             float shift_scale) {
  static_assert(WPR == 2 || WPR == 4 || WPR == 8, "WPR");
  constexpr int T = WPR * 32;  // threads per row
  __shared__ float red_m[kRowsThreads / 32];
  __shared__ double red_s[kRowsThreads / 32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rw = warp / WPR;  // row slot of this warp in the block
  const int t = (warp % WPR) * 32 + lane;
  const int rpc = static_cast<int>(blockDim.x >> 5) / WPR;
  const int nvec = cols >> 2;  // 128-bit path: cols % 4 == 0
  pdl_wait();
  pdl_launch_dependents();

  for (int64_t r0 = int64_t(blockIdx.x) * rpc; r0 < rows; r0 += int64_t(gridDim.x) * rpc) {
    const int64_t r = r0 + rw;
    const bool rv = r < rows;
    const float* xr = x + (rv ? r : 0) * ldx;
    float4 v[NV];
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const int q = j * T + t;
      v[j] = (rv && q < nvec) ? ld_stream4(xr + 4 * q)
                              : make_float4(kPadLogit, kPadLogit, kPadLogit, kPadLogit);
    }
    // ---- row max + finite check
    float mu = kPadLogit;
    u64 z = f2pk(0.0f, 0.0f);
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      mu = fmaxf(mu, fmaxf(fmaxf(v[j].x, v[j].y), fmaxf(v[j].z, v[j].w)));
      z = nf_acc2(nf_acc2(z, v[j].x, v[j].y), v[j].z, v[j].w);
    }
    const bool bad = rv && nf_bad(z);
    mu = group_max<32>(mu);
    if (lane == 0) red_m[warp] = mu;
    __syncthreads();
    float m = red_m[rw * WPR];
#pragma unroll
    for (int k = 1; k < WPR; ++k) m = fmaxf(m, red_m[rw * WPR + k]);
    m *= shift_scale;  // shift_scale = 0: fault hook
    // ---- exp(clip(x - m)) kept in registers, row sum
    u64 acc = f2pk(0.0f, 0.0f);
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const float2 a = sexp2<MODE>(v[j].x, v[j].y, m);
      const float2 b = sexp2<MODE>(v[j].z, v[j].w, m);
      v[j] = make_float4(a.x, a.y, b.x, b.y);
      if (j * T + t < nvec) acc = f2add(f2add(acc, f2pk(a.x, a.y)), f2pk(b.x, b.y));
    }
    const float2 a2 = f2up(acc);
    const double sw = group_sum<32>(static_cast<double>(a2.x + a2.y));
    if (lane == 0) red_s[warp] = sw;
    __syncthreads();
    double S = red_s[rw * WPR];
#pragma unroll
    for (int k = 1; k < WPR; ++k) S += red_s[rw * WPR + k];  // fixed order
    const float rcp = recip_of_sum(S);
    // ---- scale (+ flush), write once
    if (rv) {
      float* yr = y + r * ldy;
#pragma unroll
      for (int j = 0; j < NV; ++j) {
        const int q = j * T + t;
        if (q < nvec) {
          const float2 p = scale2<MODE>(make_float2(v[j].x, v[j].y), rcp);
          const float2 o = scale2<MODE>(make_float2(v[j].z, v[j].w), rcp);
          st_stream4(yr + 4 * q, make_float4(p.x, p.y, o.x, o.y));
        }
      }
    }
    if (bad) atomicMin(bad_row, static_cast<unsigned long long>(r));
  }
}

}  // namespace sk
