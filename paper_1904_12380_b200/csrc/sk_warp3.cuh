// sk_warp3.cuh -- K3: long rows, one launch, ordered queue of WARP tasks.
//
// Same dataflow as k3_dyn (sk_dyn.cuh) -- tasks S(row r+lag) then N(row r),
// claimed in order from a global counter; the last-arriving S of a row
// merges it and release-stores its ready flag; N tasks re-read their segment
// from L2 -- but every task belongs to ONE WARP: a segment is 32 lanes x NV
// float4 (1024 floats at NV = 8), reductions are warp shuffles only, and no
// __syncthreads exists in the kernel.  Every warp is an independent dependency
// chain, so an SM overlaps dozens of them; each warp also claims its next
// task index while working on the current one, and an N task issues its
// segment loads before it checks the row's ready flag.  Deadlock-free without
// co-residency: S tasks never wait, and an N task waits only for S tasks with
// smaller indices, which running warps have already claimed.
//
// Replaces kernels.py:136-189 for long rows; outputs are rounded exactly as
// the reference rounds them: y = exp(clip(x - M)) * (1/(float)S).
#pragma once
#include "sk_common.cuh"
#include "sk_seg.cuh"
#include "sk_chunk.cuh"

namespace sk {

constexpr int kWarp3Threads = 256;

__device__ __forceinline__ unsigned atom_add_acq_rel_gpu(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v)
               : "memory");
  return old;
}
__device__ __forceinline__ void st_release_gpu_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int NV>
__device__ __forceinline__ void w3_decode(int64_t t, int64_t rows, int64_t ns, int64_t lag,
                                          bool& stats, int64_t& row, int& seg) {
  const int64_t head = lag * ns;
  const int64_t pairs = (rows - lag) * 2 * ns;
  if (t < head) {
    stats = true;
    row = t / ns;
    seg = static_cast<int>(t % ns);
  } else if (t - head < pairs) {
    const int64_t u = t - head;
    const int64_t r = u / (2 * ns);
    const int64_t w = u % (2 * ns);
    stats = w < ns;
    row = stats ? r + lag : r;
    seg = static_cast<int>(stats ? w : w - ns);
  } else {
    const int64_t u = t - head - pairs;
    stats = false;
    row = rows - lag + u / ns;
    seg = static_cast<int>(u % ns);
  }
}

template <int MODE, int NV>
__global__ void __launch_bounds__(kWarp3Threads)
    k3_warp(const float* __restrict__ x, float* __restrict__ y, int64_t rows, int64_t cols,
            int64_t ldx, int64_t ldy, int nseg, int64_t lag, int batch,
            unsigned long long* __restrict__ task_ctr, unsigned* __restrict__ row_cnt,
            unsigned* __restrict__ row_ready, RowPartial* __restrict__ partials,
            float* __restrict__ row_max, double* __restrict__ row_sum,
            unsigned long long* __restrict__ bad_row, float shift_scale) {
  constexpr int SEG = 32 * NV * 4;
  const int lane = threadIdx.x & 31;
  pdl_wait();
  pdl_launch_dependents();
  const uint64_t keep = policy_evict_last();
  const uint64_t drop = policy_evict_first();
  const int64_t ns = nseg;
  const int64_t total = 2 * rows * ns;

  // batch == 0: static round-robin -- warp w runs tasks w, w+W, w+2W, ... (no
  //   atomics; the in-flight window is exactly one task per warp; the launch is
  //   cooperative so every warp is resident, which keeps the waits deadlock-free).
  // batch >= 1: tasks claimed `batch` at a time from the global counter (one
  //   atomic per batch: a single counter sustains only ~0.5 G atomics/s).
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const int64_t gwarp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  unsigned long long cur = 0, next = 0;
  if (batch > 0) {
    if (lane == 0) cur = atomicAdd(task_ctr, static_cast<unsigned long long>(batch));
    cur = __shfl_sync(0xffffffffu, cur, 0);
  }
  int k = 0;
  for (int64_t it = 0;; ++it) {
    const int64_t t = batch > 0 ? static_cast<int64_t>(cur) + k : gwarp + it * nwarps;
    if (t >= total) break;
    if (batch > 0 && k == batch - 1 && lane == 0)
      next = atomicAdd(task_ctr, static_cast<unsigned long long>(batch));
    bool stats;
    int64_t row;
    int seg;
    w3_decode<NV>(t, rows, ns, lag, stats, row, seg);
    const int64_t c0 = int64_t(seg) * SEG;
    const int64_t rem = cols - c0;
    const int nvec = static_cast<int>((rem < SEG ? rem : SEG) >> 2);
    const float* xs = x + row * ldx + c0;
    float4 v[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int q = lane + 32 * i;
      v[i] = q < nvec ? ld_hint4(xs + 4 * q, stats ? keep : drop)
                      : make_float4(kPadLogit, kPadLogit, kPadLogit, kPadLogit);
    }

    if (stats) {
      float mt = kPadLogit;
      u64 z = f2pk(0.0f, 0.0f);
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        mt = fmaxf(mt, fmaxf(fmaxf(v[i].x, v[i].y), fmaxf(v[i].z, v[i].w)));
        z = nf_acc2(nf_acc2(z, v[i].x, v[i].y), v[i].z, v[i].w);
      }
      if (nf_bad(z)) atomicMin(bad_row, static_cast<unsigned long long>(row));
      const float m_l = group_max<32>(mt) * shift_scale;  // shift_scale = 0: fault hook
      u64 acc = f2pk(0.0f, 0.0f);
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        float2 a = sexp2<MODE>(v[i].x, v[i].y, m_l);
        float2 b = sexp2<MODE>(v[i].z, v[i].w, m_l);
        if (!(lane + 32 * i < nvec)) a = b = make_float2(0.0f, 0.0f);
        acc = f2add(f2add(acc, f2pk(a.x, a.y)), f2pk(b.x, b.y));
      }
      const float2 acc2 = f2up(acc);
      const double s_l = group_sum<32>(static_cast<double>(acc2.x + acc2.y));
      unsigned last = 0;
      if (lane == 0) {
        RowPartial p;
        p.m = m_l;
        p.pad = 0.0f;
        p.s = s_l;
        partials[row * ns + seg] = p;
        // release our partial / acquire everyone else's if we are last
        last = atom_add_acq_rel_gpu(&row_cnt[row], 1u) == static_cast<unsigned>(nseg) - 1u;
      }
      last = __shfl_sync(0xffffffffu, last, 0);
      if (last) {  // merge the row (fixed order: deterministic)
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
    } else {
      if (lane == 0) {
        unsigned sleep = 20;
        while (ld_acquire_gpu(&row_ready[row]) == 0u) {
          __nanosleep(sleep);
          if (sleep < 320) sleep <<= 1;
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
          const float2 a = scale2<MODE>(sexp2<MODE>(v[i].x, v[i].y, M), rcp);
          const float2 b = scale2<MODE>(sexp2<MODE>(v[i].z, v[i].w, M), rcp);
          st_stream4(ys + 4 * q, make_float4(a.x, a.y, b.x, b.y));
        }
      }
    }
    if (batch > 0 && ++k == batch) {
      cur = __shfl_sync(0xffffffffu, next, 0);
      k = 0;
    }
  }
}

}  // namespace sk
