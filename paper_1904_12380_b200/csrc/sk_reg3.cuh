// sk_reg3.cuh -- K3: long rows held in REGISTERS across the row exchange.
//
// Why: on B200 the L2 slices' throughput, not DRAM, bounds a streaming kernel
// (~6.5 TB/s for 8 B/element).  Two-pass schemes that re-read a segment --
// even from L2 -- push 12 B/element through L2 and cap out at ~8/12 of that.
// Here a segment never leaves the SM between its two passes:
//
//   task t (static round-robin: warp w runs t = w, w+W, ...; row-major order,
//   so the nseg segments of a row run on nseg neighbouring warps at once):
//     1. (already prefetched) segment t in registers: 32 lanes x NV float4
//     2. m = max, s = sum exp(clip(x - m)) -> warp shuffles; lane 0 stores the
//        partial and arrives on the row counter (atom.acq_rel); the last
//        arrival merges the row  M = max m_k, S = sum s_k exp(m_k - M)  (f64,
//        fixed order) and release-stores the row's ready flag
//     3. issue the loads of task t+W into the second register buffer
//     4. wait for the row's ready flag (normally already set or imminent --
//        the row's segments were loaded together), then write
//        y = exp(clip(x - M)) * (1/(float)S) straight from registers: the
//        reference's operation order (kernels.py:144-189) for every element.
//
// HBM and L2 see one read and one write per element.  The launch is
// cooperative (all warps resident): a warp only waits for segments of its
// own row, which neighbouring warps reach without waiting on anything of a
// later task, so the waits cannot deadlock.
#pragma once
#include "sk_common.cuh"
#include "sk_seg.cuh"
#include "sk_chunk.cuh"
#include "sk_warp3.cuh"

namespace sk {

constexpr int kReg3Threads = 256;

template <int NV>
__device__ __forceinline__ void r3_load(float4 (&v)[NV], const float* __restrict__ x, int64_t t,
                                        int64_t ns, int64_t cols, int64_t ldx, int lane) {
  constexpr int SEG = 32 * NV * 4;
  const int64_t row = t / ns;
  const int64_t c0 = (t - row * ns) * SEG;
  const int64_t rem = cols - c0;
  const int nvec = static_cast<int>((rem < SEG ? rem : SEG) >> 2);
  const float* xs = x + row * ldx + c0;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int q = lane + 32 * i;
    v[i] = q < nvec ? ld_stream4(xs + 4 * q)
                    : make_float4(kPadLogit, kPadLogit, kPadLogit, kPadLogit);
  }
}

template <int MODE, int NV>
__global__ void __launch_bounds__(kReg3Threads)
    k3_reg(const float* __restrict__ x, float* __restrict__ y, int64_t rows, int64_t cols,
           int64_t ldx, int64_t ldy, int nseg, unsigned* __restrict__ row_cnt,
           unsigned* __restrict__ row_ready, RowPartial* __restrict__ partials,
           float* __restrict__ row_max, double* __restrict__ row_sum,
           unsigned long long* __restrict__ bad_row, float shift_scale) {
  constexpr int SEG = 32 * NV * 4;
  const int lane = threadIdx.x & 31;
  pdl_wait();
  pdl_launch_dependents();
  const int64_t ns = nseg;
  const int64_t total = rows * ns;
  const int64_t W = (int64_t(gridDim.x) * blockDim.x) >> 5;
  int64_t t = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;

  float4 cur[NV], nxt[NV];
  if (t < total) r3_load<NV>(cur, x, t, ns, cols, ldx, lane);
  for (; t < total; t += W) {
    const int64_t row = t / ns;
    const int seg = static_cast<int>(t - row * ns);
    const int64_t c0 = int64_t(seg) * SEG;
    const int64_t rem = cols - c0;
    const int nvec = static_cast<int>((rem < SEG ? rem : SEG) >> 2);

    // ---- local statistics of this segment
    float mt = kPadLogit;
    u64 z = f2pk(0.0f, 0.0f);
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      mt = fmaxf(mt, fmaxf(fmaxf(cur[i].x, cur[i].y), fmaxf(cur[i].z, cur[i].w)));
      z = nf_acc2(nf_acc2(z, cur[i].x, cur[i].y), cur[i].z, cur[i].w);
    }
    if (nf_bad(z)) atomicMin(bad_row, static_cast<unsigned long long>(row));
    const float m_l = group_max<32>(mt) * shift_scale;  // shift_scale = 0: fault hook
    u64 acc = f2pk(0.0f, 0.0f);
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      float2 a = sexp2<MODE>(cur[i].x, cur[i].y, m_l);
      float2 b = sexp2<MODE>(cur[i].z, cur[i].w, m_l);
      if (!(lane + 32 * i < nvec)) a = b = make_float2(0.0f, 0.0f);
      acc = f2add(f2add(acc, f2pk(a.x, a.y)), f2pk(b.x, b.y));
    }
    const float2 acc2 = f2up(acc);
    const double s_l = group_sum<32>(static_cast<double>(acc2.x + acc2.y));

    // ---- publish; the last arrival merges the row
    unsigned last = 0;
    if (lane == 0) {
      RowPartial p;
      p.m = m_l;
      p.pad = 0.0f;
      p.s = s_l;
      partials[row * ns + seg] = p;
      last = atom_add_acq_rel_gpu(&row_cnt[row], 1u) == static_cast<unsigned>(nseg) - 1u;
    }
    last = __shfl_sync(0xffffffffu, last, 0);
    if (last) {
      __syncwarp();
      const RowPartial* rp = partials + row * ns;
      float mq = kPadLogit;
      for (int q = lane; q < nseg; q += 32) mq = fmaxf(mq, __ldcg(&rp[q].m));
      const float M = group_max<32>(mq);
      double sq = 0.0;
      for (int q = lane; q < nseg; q += 32) {
        const float m = __ldcg(&rp[q].m);
        sq += __ldcg(&rp[q].s) * static_cast<double>(m == M ? 1.0f : expf(m - M));
      }
      const double S = group_sum<32>(sq);
      if (lane == 0) {
        row_max[row] = M;
        row_sum[row] = S;
        st_release_gpu_u32(&row_ready[row], 1u);
      }
    }

    // ---- prefetch the next segment while the row completes
    const int64_t tn = t + W;
    if (tn < total) r3_load<NV>(nxt, x, tn, ns, cols, ldx, lane);

    // ---- wait for the row, normalize from registers
    if (lane == 0) {
      unsigned sleep = 16;
      while (ld_acquire_gpu(&row_ready[row]) == 0u) {
        __nanosleep(sleep);
        if (sleep < 256) sleep <<= 1;
      }
    }
    __syncwarp();
    const float M = __ldcg(&row_max[row]);
    const float rcp = recip_of_sum(__ldcg(&row_sum[row]));
    float* ys = y + row * ldy + c0;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int q = lane + 32 * i;
      if (q < nvec) {
        const float2 a = scale2<MODE>(sexp2<MODE>(cur[i].x, cur[i].y, M), rcp);
        const float2 b = scale2<MODE>(sexp2<MODE>(cur[i].z, cur[i].w, M), rcp);
        st_stream4(ys + 4 * q, make_float4(a.x, a.y, b.x, b.y));
      }
    }
#pragma unroll
    for (int i = 0; i < NV; ++i) cur[i] = nxt[i];
  }
}

}  // namespace sk
