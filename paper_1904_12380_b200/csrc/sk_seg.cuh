// sk_seg.cuh -- K2/K3: TMA-staged row segments, one CTA per segment.
//
// A row of C floats is cut into nseg segments of `seglen` floats (seglen % 4
// == 0, last one shorter).  Work item w = (row, seg) = (w / nseg, w % nseg).
// Each CTA walks items blockIdx.x, +gridDim.x, ... and for each one:
//
//   1. waits for the segment to land in shared memory (cp.async.bulk 1-D TMA,
//      issued NS items ahead on an mbarrier ring, L2 evict-first),
//   2. copies it into registers (NV float4 per thread) and immediately re-arms
//      the freed stage with the item NS steps ahead -- HBM keeps streaming while
//      this item computes,
//   3. block-reduces the local max m_l and the local sum s_l of
//      e = exp(clip(x - m_l)), keeping e in registers (exp computed once),
//   4. K2 (nseg == 1): M = m_l, S = s_l -- exactly the reference order.
//      K3 (nseg > 1): publishes (m_l, s_l) for its row, waits until all nseg
//      segments of the row have published (cooperative launch: every CTA is
//      resident and items are taken in increasing order, so the wait cannot
//      deadlock while nseg <= gridDim.x), then merges
//         M = max_k m_k,   S = sum_k s_k * exp(m_k - M)      (f64, fixed order)
//   5. writes y = exp(clip(x - M)) * (1/S) from the registers (K2 reuses e;
//      K3 recomputes exp against the merged M so every output is rounded as
//      the reference rounds it) -- HBM is read once and written once:
//      8 B/element.  Row counters are zeroed by the launcher before a K3 launch.
//
// Replaces kernels.py:136-189 for C > 1024 (and row_stats, kernels.py:272-276,
// whose (max, sum) pair is exactly what step 4 exchanges).
#pragma once
#include "sk_common.cuh"

namespace sk {

struct RowPartial {  // one (row, segment) statistic, 16 B
  float m;
  float pad;
  double s;
};

constexpr int kSegStages = 2;

template <int MODE, int NV>
__global__ void __launch_bounds__(1024)
    k_seg(const float* __restrict__ x, float* __restrict__ y, int64_t rows, int64_t cols,
          int64_t ldx, int64_t ldy, int nseg, int seglen, unsigned* __restrict__ row_cnt,
          RowPartial* __restrict__ partials, unsigned long long* __restrict__ bad_row,
          float shift_scale) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* stage_buf = reinterpret_cast<float*>(smem_raw);
  const int seg_floats = blockDim.x * NV * 4;  // stage capacity in floats
  __shared__ uint64_t bars[kSegStages];
  __shared__ float red_f[33];
  __shared__ double red_d[33];
  __shared__ float bc_M;
  __shared__ double bc_S;

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const int64_t items = rows * nseg;

  auto item_ptr = [&](int64_t w, int64_t& row, int& seg, int& len) {
    row = w / nseg;
    seg = static_cast<int>(w - row * nseg);
    const int64_t c0 = int64_t(seg) * seglen;
    const int64_t rem = cols - c0;
    len = static_cast<int>(rem < seglen ? rem : seglen);
    return x + row * ldx + c0;
  };
  auto issue = [&](int64_t w, int stage) {
    int64_t row;
    int seg, len;
    const float* src = item_ptr(w, row, seg, len);
    mbar_arrive_expect_tx(&bars[stage], static_cast<uint32_t>(len) * 4u);
    tma_load_1d(stage_buf + stage * seg_floats, src, static_cast<uint32_t>(len) * 4u,
                &bars[stage]);
  };

  pdl_wait();
  pdl_launch_dependents();
  if (tid == 0) {
    for (int s = 0; s < kSegStages; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) {
    for (int s = 0; s < kSegStages; ++s) {
      const int64_t w = blockIdx.x + int64_t(s) * gridDim.x;
      if (w < items) issue(w, s);
    }
  }

  int k = 0;
  for (int64_t w = blockIdx.x; w < items; w += gridDim.x, ++k) {
    const int stage = k % kSegStages;
    const uint32_t parity = (k / kSegStages) & 1;
    int64_t row;
    int seg, len;
    item_ptr(w, row, seg, len);
    const int nvec = len >> 2;

    mbar_wait(&bars[stage], parity);
    float v[NV][4];
    const float4* sb = reinterpret_cast<const float4*>(stage_buf + stage * seg_floats);
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int q = tid + i * blockDim.x;
      if (q < nvec) {
        const float4 t = sb[q];
        v[i][0] = t.x; v[i][1] = t.y; v[i][2] = t.z; v[i][3] = t.w;
      } else {
        v[i][0] = v[i][1] = v[i][2] = v[i][3] = kPadLogit;
      }
    }
    __syncthreads();  // every thread is done with this stage
    if (tid == 0) {
      const int64_t wn = w + int64_t(kSegStages) * gridDim.x;
      if (wn < items) {
        fence_proxy_async_smem();
        issue(wn, stage);
      }
    }

    // ---- local max + finite check
    float mt = kPadLogit;
    u64 z = f2pk(0.0f, 0.0f);
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      mt = fmaxf(mt, fmaxf(fmaxf(v[i][0], v[i][1]), fmaxf(v[i][2], v[i][3])));
      z = nf_acc2(nf_acc2(z, v[i][0], v[i][1]), v[i][2], v[i][3]);
    }
    if (nf_bad(z)) atomicMin(bad_row, static_cast<unsigned long long>(row));
    mt = group_max<32>(mt);
    if (lane == 0) red_f[warp] = mt;
    __syncthreads();
    if (warp == 0) {
      float t = lane < nwarps ? red_f[lane] : kPadLogit;
      t = group_max<32>(t);
      if (lane == 0) red_f[32] = t;
    }
    __syncthreads();
    const float m_l = red_f[32] * shift_scale;  // shift_scale = 0: fault hook

    // ---- local sum of e = exp(clip(x - m_l)).  K2 keeps e in registers (one
    // exp per element, reference order); K3 keeps x and recomputes exp(x - M)
    // against the merged row max below, so every output is rounded exactly as
    // the reference rounds it (s = x - M in fp32, clip, expf, * 1/S).
    const bool single = (nseg == 1);
    u64 acc = f2pk(0.0f, 0.0f);
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const bool ok = tid + i * static_cast<int>(blockDim.x) < nvec;
      float2 a = sexp2<MODE>(v[i][0], v[i][1], m_l);
      float2 b = sexp2<MODE>(v[i][2], v[i][3], m_l);
      if (single) {
        v[i][0] = a.x; v[i][1] = a.y; v[i][2] = b.x; v[i][3] = b.y;
      }
      if (!ok) a = b = make_float2(0.0f, 0.0f);
      acc = f2add(f2add(acc, f2pk(a.x, a.y)), f2pk(b.x, b.y));
    }
    const float2 acc2 = f2up(acc);
    const float st = acc2.x + acc2.y;
    double sd = group_sum<32>(static_cast<double>(st));
    if (lane == 0) red_d[warp] = sd;
    __syncthreads();
    if (warp == 0) {
      double t = lane < nwarps ? red_d[lane] : 0.0;
      t = group_sum<32>(t);
      if (lane == 0) red_d[32] = t;
    }
    __syncthreads();
    const double s_l = red_d[32];

    float M = m_l, rcp;
    if (single) {
      rcp = recip_of_sum(s_l);
    } else {
      // ---- publish, wait for the row, merge (warp 0)
      if (warp == 0) {
        if (lane == 0) {
          RowPartial p;
          p.m = m_l;
          p.pad = 0.0f;
          p.s = s_l;
          partials[row * nseg + seg] = p;
          red_release_add_gpu(&row_cnt[row], 1u);
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
          bc_M = Mw;
          bc_S = S;
        }
      }
      __syncthreads();
      M = bc_M;
      rcp = recip_of_sum(bc_S);
    }

    // ---- y = exp(clip(x - M)) * r, flush, streaming store straight from registers
    float* yr = y + row * ldy + int64_t(seg) * seglen;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int q = tid + i * blockDim.x;
      if (q < nvec) {
        float2 a, b;
        if (single) {
          a = make_float2(v[i][0], v[i][1]);
          b = make_float2(v[i][2], v[i][3]);
        } else {
          a = sexp2<MODE>(v[i][0], v[i][1], M);
          b = sexp2<MODE>(v[i][2], v[i][3], M);
        }
        a = scale2<MODE>(a, rcp);
        b = scale2<MODE>(b, rcp);
        st_stream4(yr + 4 * q, make_float4(a.x, a.y, b.x, b.y));
      }
    }
    __syncthreads();  // red_* / bc_* reuse in the next item
  }
}

}  // namespace sk
