// sk_rows_mw.cuh -- K1m: medium rows (128-bit rows of 3 K .. 8 K floats, and
// rows of any length / alignment from 1 K to 8 K floats with 32-bit accesses)
// in the registers of WPR warps.
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
// The result depends only on (VEC, WPR, NV), never on the grid, so row blocks
// keep their bits.
#pragma once
#include "sk_common.cuh"
#include "sk_rows.cuh"

namespace sk {

// VEC = 4: 128-bit accesses (cols % 4 == 0, 16-B aligned rows); VEC = 1:
// 32-bit coalesced accesses for rows of any length / alignment.  Thread t of
// a row holds vectors j*T + t, j < NV (T = 32*WPR threads per row).
template <int MODE, int WPR, int NV, int VEC>
__global__ void __launch_bounds__(kRowsThreads, 2)
    k1m_rows(const float* __restrict__ x, float* __restrict__ y, int64_t rows, int cols,
             int64_t ldx, int64_t ldy, unsigned long long* __restrict__ bad_row,
             float shift_scale) {
  static_assert(WPR == 2 || WPR == 4 || WPR == 8, "WPR");
  static_assert(VEC == 1 || VEC == 4, "VEC");
  static_assert((NV * VEC) % 2 == 0, "packed pairs");
  constexpr int T = WPR * 32;  // threads per row
  constexpr int E = NV * VEC;  // floats per thread
  __shared__ float red_m[kRowsThreads / 32];
  __shared__ double red_s[kRowsThreads / 32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rw = warp / WPR;  // row slot of this warp in the block
  const int t = (warp % WPR) * 32 + lane;
  const int rpc = static_cast<int>(blockDim.x >> 5) / WPR;
  const int nvec = VEC == 4 ? cols >> 2 : cols;
  pdl_wait();
  pdl_launch_dependents();

  for (int64_t r0 = int64_t(blockIdx.x) * rpc; r0 < rows; r0 += int64_t(gridDim.x) * rpc) {
    const int64_t r = r0 + rw;
    const bool rv = r < rows;
    const float* xr = x + (rv ? r : 0) * ldx;
    float v[E];
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const int q = j * T + t;
      if (rv && q < nvec) {
        if constexpr (VEC == 4) {
          const float4 a = ld_stream4(xr + 4 * q);
          v[4 * j] = a.x; v[4 * j + 1] = a.y; v[4 * j + 2] = a.z; v[4 * j + 3] = a.w;
        } else {
          v[j] = ld_stream1(xr + q);
        }
      } else {
#pragma unroll
        for (int k = 0; k < VEC; ++k) v[VEC * j + k] = kPadLogit;
      }
    }
    // ---- row max + finite check
    float mu = kPadLogit;
    u64 z = f2pk(0.0f, 0.0f);
#pragma unroll
    for (int e = 0; e < E; e += 2) {
      mu = fmaxf(mu, fmaxf(v[e], v[e + 1]));
      z = nf_acc2(z, v[e], v[e + 1]);
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
    for (int e = 0; e < E; e += 2) {
      float2 a = sexp2<MODE>(v[e], v[e + 1], m);
      v[e] = a.x;
      v[e + 1] = a.y;
      if ((e / VEC) * T + t >= nvec) a.x = 0.0f;  // padding contributes nothing
      if (((e + 1) / VEC) * T + t >= nvec) a.y = 0.0f;
      acc = f2add(acc, f2pk(a.x, a.y));
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
          if constexpr (VEC == 4) {
            const float2 p = scale2<MODE>(make_float2(v[4 * j], v[4 * j + 1]), rcp);
            const float2 o = scale2<MODE>(make_float2(v[4 * j + 2], v[4 * j + 3]), rcp);
            st_stream4(yr + 4 * q, make_float4(p.x, p.y, o.x, o.y));
          } else {
            st_stream1(yr + q, scale1<MODE>(v[j], rcp));
          }
        }
      }
    }
    if (bad) atomicMin(bad_row, static_cast<unsigned long long>(r));
  }
}

}  // namespace sk
