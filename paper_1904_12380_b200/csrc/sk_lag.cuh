// sk_lag.cuh -- K3: long rows, online two-pass with a lag (L2 re-read).
//
// Rows too long for one CTA (C > 8192) are cut into nseg segments of
// `seglen` floats; work item w = (row, seg) = (w / nseg, w % nseg).  A
// cooperative (all-resident) grid of G CTAs walks the items in rounds: in
// iteration j, CTA b
//
//   1. STATS item a = b + j*G: streams the segment from HBM into registers
//      (128-bit loads, L2 evict_last so the re-read below hits L2), reduces
//      m_l = max and s_l = sum exp(clip(x - m_l)) over the CTA and publishes
//      (m_l, s_l) for its row (release add on the row counter);
//   2. NORMALIZE item b' = b + (j - lag)*G, published `lag` rounds earlier:
//      by now every segment of its row has been published (the counter is
//      checked; a short spin only if a row-mate is late), so it merges
//         M = max_k m_k,   S = sum_k s_k * exp(m_k - M)    (f64, fixed order)
//      re-reads the segment (from L2: it was read lag*G segments ago, well
//      inside the 126 MB L2) and writes y = exp(clip(x - M)) * (1/(float)S)
//      -- the reference's operation order (kernels.py:144-189) for every
//      output element.
//
// The lag hides the cross-CTA exchange latency behind a full round of
// streaming; HBM sees one read and one write per element (8 B/element), the
// second read is served by L2.  No deadlock: a normalize only waits for
// stats of items at most one round ahead of it, and every CTA publishes the
// stats of round j before it can block in round j (needs nseg <= G and a
// co-resident grid, guaranteed by the cooperative launch).
#pragma once
#include "sk_common.cuh"
#include "sk_seg.cuh"

namespace sk {

__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ float4 ld_hint4(const float* p, uint64_t pol) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p), "l"(pol));
  return v;
}

template <int NWARPS_MAX = 32>
struct BlockRed {
  float f[NWARPS_MAX + 1];
  double d[NWARPS_MAX + 1];
  float M;
  double S;
};

template <int MODE, int NV>
__global__ void __launch_bounds__(256)
    k3_lag(const float* __restrict__ x, float* __restrict__ y, int64_t rows, int64_t cols,
           int64_t ldx, int64_t ldy, int nseg, int seglen, int lag,
           unsigned* __restrict__ row_cnt, RowPartial* __restrict__ partials,
           unsigned long long* __restrict__ bad_row, float shift_scale) {
  __shared__ BlockRed<8> red;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const int64_t items = rows * nseg;
  const int64_t G = gridDim.x;
  const uint64_t keep = policy_evict_last();
  const uint64_t drop = policy_evict_first();
  pdl_wait();
  pdl_launch_dependents();

  for (int64_t j = 0;; ++j) {
    const int64_t a = blockIdx.x + j * G;
    const int64_t b = blockIdx.x + (j - lag) * G;
    const bool do_stats = a < items;
    const bool do_norm = j >= lag && b < items;
    if (!do_stats && !do_norm) break;

    if (do_stats) {
      const int64_t row = a / nseg;
      const int seg = static_cast<int>(a - row * nseg);
      const int64_t c0 = int64_t(seg) * seglen;
      const int64_t rem = cols - c0;
      const int nvec = static_cast<int>((rem < seglen ? rem : seglen) >> 2);
      const float* xs = x + row * ldx + c0;
      float v[NV][4];
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        const int q = tid + i * blockDim.x;
        if (q < nvec) {
          const float4 t = ld_hint4(xs + 4 * q, keep);
          v[i][0] = t.x; v[i][1] = t.y; v[i][2] = t.z; v[i][3] = t.w;
        } else {
          v[i][0] = v[i][1] = v[i][2] = v[i][3] = kPadLogit;
        }
      }
      float mt = kPadLogit;
      bool bad = false;
#pragma unroll
      for (int i = 0; i < NV; ++i)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          mt = fmaxf(mt, v[i][c]);
          bad |= not_finite(v[i][c]);
        }
      if (bad) atomicMin(bad_row, static_cast<unsigned long long>(row));
      mt = group_max<32>(mt);
      if (lane == 0) red.f[warp] = mt;
      __syncthreads();
      if (warp == 0) {
        float t = lane < nwarps ? red.f[lane] : kPadLogit;
        t = group_max<32>(t);
        if (lane == 0) red.f[8] = t;
      }
      __syncthreads();
      const float m_l = red.f[8] * shift_scale;
      float st = 0.0f;
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        const bool ok = tid + i * static_cast<int>(blockDim.x) < nvec;
#pragma unroll
        for (int c = 0; c < 4; ++c) st += ok ? shifted_exp<MODE>(v[i][c], m_l) : 0.0f;
      }
      double sd = group_sum<32>(static_cast<double>(st));
      if (lane == 0) red.d[warp] = sd;
      __syncthreads();
      if (tid == 0) {
        double t = 0.0;
        for (int w = 0; w < nwarps; ++w) t += red.d[w];
        RowPartial p;
        p.m = m_l;
        p.pad = 0.0f;
        p.s = t;
        partials[a] = p;
        red_release_add_gpu(&row_cnt[row], 1u);
      }
    }

    if (do_norm) {
      const int64_t row = b / nseg;
      const int seg = static_cast<int>(b - row * nseg);
      if (warp == 0) {
        if (lane == 0) {
          unsigned ns = 32;
          while (ld_acquire_gpu(&row_cnt[row]) < static_cast<unsigned>(nseg)) {
            __nanosleep(ns);
            if (ns < 256) ns <<= 1;
          }
        }
        __syncwarp();
        const RowPartial* rp = partials + row * nseg;
        float Mw = kPadLogit;
        for (int q = lane; q < nseg; q += 32) Mw = fmaxf(Mw, __ldcg(&rp[q].m));
        Mw = group_max<32>(Mw);
        double S = 0.0;
        for (int q = lane; q < nseg; q += 32) {
          const float mq = __ldcg(&rp[q].m);
          S += __ldcg(&rp[q].s) * static_cast<double>(mq == Mw ? 1.0f : expf(mq - Mw));
        }
        S = group_sum<32>(S);
        if (lane == 0) {
          red.M = Mw;
          red.S = S;
        }
      }
      __syncthreads();
      const float M = red.M;
      const float rcp = recip_of_sum(red.S);
      const int64_t c0 = int64_t(seg) * seglen;
      const int64_t rem = cols - c0;
      const int nvec = static_cast<int>((rem < seglen ? rem : seglen) >> 2);
      const float* xs = x + row * ldx + c0;
      float* ys = y + row * ldy + c0;
      float4 t[NV];
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        const int q = tid + i * blockDim.x;
        if (q < nvec) t[i] = ld_hint4(xs + 4 * q, drop);
      }
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        const int q = tid + i * blockDim.x;
        if (q < nvec)
          st_stream4(ys + 4 * q, make_float4(scale_flush(shifted_exp<MODE>(t[i].x, M), rcp),
                                             scale_flush(shifted_exp<MODE>(t[i].y, M), rcp),
                                             scale_flush(shifted_exp<MODE>(t[i].z, M), rcp),
                                             scale_flush(shifted_exp<MODE>(t[i].w, M), rcp)));
      }
    }
    __syncthreads();  // red reuse
  }
}

}  // namespace sk
