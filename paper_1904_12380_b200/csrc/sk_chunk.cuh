// sk_chunk.cuh -- K3: long rows as an L2-chunked two-pass pipeline.
//
// Rows longer than one CTA can hold (C > 8192) are cut into nseg segments
// of `seglen` floats, and the matrix into row chunks of ~24 MB (a fraction of
// the 126 MB L2).  Launch k of a softmax call does two independent phases:
//
//   STATS(chunk k):  every (row, segment) item streams its segment from HBM
//      (128-bit loads, L2 evict_last so it stays for the normalize re-read),
//      reduces m = max and s = sum exp(clip(x - m)) over the CTA and stores
//      the partial.  The CTA whose atomic arrival on the row counter is the
//      last one merges the row (threadfence-reduction pattern, no waiting):
//          M = max_k m_k,  S = sum_k s_k * exp(m_k - M)   (f64, fixed order)
//      and stores (M, S) for the row.
//   NORMALIZE(chunk k-1):  after griddepcontrol.wait (launch k-1, which merged
//      chunk k-1, is complete), every item re-reads its segment -- from L2 --
//      and writes y = exp(clip(x - M)) * (1/(float)S): the reference's own
//      operation order (kernels.py:144-189) for every output element.
//
// Launch k calls launch_dependents only after its wait, so with programmatic
// dependent launch the STATS phase of launch k+1 streams chunk k+1 from HBM
// while launch k normalizes chunk k out of L2, and at most ~3 chunks are L2
// resident.  HBM traffic: one read + one write per element (8 B/element).
// STATS reads x, which no launch of this call writes, so launch k+1 may read
// it before launch k completes; the first launch waits before touching x.
// Replaces kernels.py:136-189 for long rows (and row_stats, kernels.py:272-276).
#pragma once
#include "sk_common.cuh"
#include "sk_seg.cuh"

namespace sk {

constexpr int kChunkThreads = 256;

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

struct ChunkRed {
  float f[kChunkThreads / 32 + 1];
  double d[kChunkThreads / 32 + 1];
  int last;
};

__device__ __forceinline__ float cta_max(float v, ChunkRed& r) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = group_max<32>(v);
  if (lane == 0) r.f[warp] = v;
  __syncthreads();
  float m = r.f[0];
#pragma unroll
  for (int w = 1; w < kChunkThreads / 32; ++w) m = fmaxf(m, r.f[w]);
  __syncthreads();
  return m;
}
__device__ __forceinline__ double cta_sum(double v, ChunkRed& r) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = group_sum<32>(v);
  if (lane == 0) r.d[warp] = v;
  __syncthreads();
  double s = r.d[0];
#pragma unroll
  for (int w = 1; w < kChunkThreads / 32; ++w) s += r.d[w];
  __syncthreads();
  return s;
}

template <int MODE, int NV>
__global__ void __launch_bounds__(kChunkThreads)
    k3_chunk(const float* __restrict__ x, float* __restrict__ y, int64_t cols, int64_t ldx,
             int64_t ldy, int nseg, int seglen, int64_t s_row0, int64_t s_rows, int64_t n_row0,
             int64_t n_rows, int wait_first, unsigned* __restrict__ row_cnt,
             RowPartial* __restrict__ partials, float* __restrict__ row_max,
             double* __restrict__ row_sum, unsigned long long* __restrict__ bad_row,
             float shift_scale) {
  __shared__ ChunkRed red;
  const int tid = threadIdx.x;
  if (wait_first) pdl_wait();

  // ---------------------------------------------------------------- STATS
  if (s_rows > 0) {
    const uint64_t keep = policy_evict_last();
    const int64_t n_items = s_rows * nseg;
    for (int64_t w = blockIdx.x; w < n_items; w += gridDim.x) {
      const int64_t row = s_row0 + w / nseg;
      const int seg = static_cast<int>(w % nseg);
      const int64_t c0 = int64_t(seg) * seglen;
      const int64_t rem = cols - c0;
      const int nvec = static_cast<int>((rem < seglen ? rem : seglen) >> 2);
      const float* xs = x + row * ldx + c0;
      float v[NV][4];
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        const int q = tid + i * kChunkThreads;
        if (q < nvec) {
          const float4 t = ld_hint4(xs + 4 * q, keep);
          v[i][0] = t.x; v[i][1] = t.y; v[i][2] = t.z; v[i][3] = t.w;
        } else {
          v[i][0] = v[i][1] = v[i][2] = v[i][3] = kPadLogit;
        }
      }
      float mt = kPadLogit;
      u64 z = f2pk(0.0f, 0.0f);
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        mt = fmaxf(mt, fmaxf(fmaxf(v[i][0], v[i][1]), fmaxf(v[i][2], v[i][3])));
        z = nf_acc2(nf_acc2(z, v[i][0], v[i][1]), v[i][2], v[i][3]);
      }
      if (nf_bad(z)) atomicMin(bad_row, static_cast<unsigned long long>(row));
      const float m_l = cta_max(mt, red) * shift_scale;  // shift_scale = 0: fault hook
      u64 acc = f2pk(0.0f, 0.0f);
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        float2 a = sexp2<MODE>(v[i][0], v[i][1], m_l);
        float2 b = sexp2<MODE>(v[i][2], v[i][3], m_l);
        if (!(tid + i * kChunkThreads < nvec)) a = b = make_float2(0.0f, 0.0f);
        acc = f2add(f2add(acc, f2pk(a.x, a.y)), f2pk(b.x, b.y));
      }
      const float2 acc2 = f2up(acc);
      const double s_l = cta_sum(static_cast<double>(acc2.x + acc2.y), red);
      if (tid == 0) {
        RowPartial p;
        p.m = m_l;
        p.pad = 0.0f;
        p.s = s_l;
        partials[row * nseg + seg] = p;
        __threadfence();
        const unsigned old = atomicAdd(&row_cnt[row], 1u);
        red.last = (old == static_cast<unsigned>(nseg) - 1u);
      }
      __syncthreads();
      if (red.last) {  // last arrival merges the row (fixed order: deterministic)
        __threadfence();
        const RowPartial* rp = partials + row * nseg;
        float mq = kPadLogit;
        for (int q = tid; q < nseg; q += kChunkThreads) mq = fmaxf(mq, __ldcg(&rp[q].m));
        const float M = cta_max(mq, red);
        double sq = 0.0;
        for (int q = tid; q < nseg; q += kChunkThreads) {
          const float m = __ldcg(&rp[q].m);
          sq += __ldcg(&rp[q].s) * static_cast<double>(m == M ? 1.0f : expf(m - M));
        }
        const double S = cta_sum(sq, red);
        if (tid == 0) {
          row_max[row] = M;
          row_sum[row] = S;
          row_cnt[row] = 0u;  // clean for the next call
        }
      }
    }
  }

  // ------------------------------------------------------------ NORMALIZE
  pdl_wait();  // launch k-1 merged chunk k-1 and is complete
  pdl_launch_dependents();
  if (n_rows > 0) {
    const uint64_t drop = policy_evict_first();
    const int64_t n_items = n_rows * nseg;
    for (int64_t w = blockIdx.x; w < n_items; w += gridDim.x) {
      const int64_t row = n_row0 + w / nseg;
      const int seg = static_cast<int>(w % nseg);
      const int64_t c0 = int64_t(seg) * seglen;
      const int64_t rem = cols - c0;
      const int nvec = static_cast<int>((rem < seglen ? rem : seglen) >> 2);
      const float* xs = x + row * ldx + c0;
      float* ys = y + row * ldy + c0;
      const float M = __ldcg(&row_max[row]);
      const float rcp = recip_of_sum(__ldcg(&row_sum[row]));
      float4 t[NV];
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        const int q = tid + i * kChunkThreads;
        if (q < nvec) t[i] = ld_hint4(xs + 4 * q, drop);
      }
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        const int q = tid + i * kChunkThreads;
        if (q < nvec) {
          const float2 a = scale2<MODE>(sexp2<MODE>(t[i].x, t[i].y, M), rcp);
          const float2 b = scale2<MODE>(sexp2<MODE>(t[i].z, t[i].w, M), rcp);
          st_stream4(ys + 4 * q, make_float4(a.x, a.y, b.x, b.y));
        }
      }
    }
  }
}

}  // namespace sk
