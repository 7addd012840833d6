// sk_split.cuh -- K4: split softmax = row statistics pass + normalize pass.
//
// Used for (a) column-sharded softmax across GPUs (the per-row (max, sum)
// pair is all that crosses NVLink; see sharding.py) and (b) long rows whose
// pitch or base is not 16-B aligned (no TMA), at 12 B/element.
//
//   k4_stats:   item (row, chunk) -> partial (m_k, s_k), s_k = sum exp(clip(x - m_k))
//   k4_combine: per row M = max m_k, S = sum s_k * exp(m_k - M)      (f64, fixed order)
//   k4_rescale: s *= exp(m_local - M_global)   (between the two all-reduces)
//   k4_normalize: y = exp(clip(x - M)) * (1/(float)S), flush  -- the reference's
//               own operation order (kernels.py:144-189) given the row stats.
//
// RowStats / row_stats (kernels.py:108-112, 272-276) is the (max, sum) pair.
#pragma once
#include "sk_common.cuh"
#include "sk_seg.cuh"

namespace sk {

constexpr int kSplitThreads = 256;
constexpr int kSplitPerThread = 16;
constexpr int kSplitChunk = kSplitThreads * kSplitPerThread;  // 4096 floats

__device__ __forceinline__ float block_max_256(float v, float* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = group_max<32>(v);
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (warp == 0) {
    float t = lane < (kSplitThreads / 32) ? red[lane] : kPadLogit;
    t = group_max<32>(t);
    if (lane == 0) red[32] = t;
  }
  __syncthreads();
  const float r = red[32];
  __syncthreads();
  return r;
}
__device__ __forceinline__ double block_sum_256(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = group_sum<32>(v);
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (warp == 0) {
    double t = lane < (kSplitThreads / 32) ? red[lane] : 0.0;
    t = group_sum<32>(t);
    if (lane == 0) red[32] = t;
  }
  __syncthreads();
  const double r = red[32];
  __syncthreads();
  return r;
}

template <int MODE, int VEC>
__global__ void __launch_bounds__(kSplitThreads)
    k4_stats(const float* __restrict__ x, int64_t rows, int64_t cols, int64_t ldx, int nch,
             RowPartial* __restrict__ partials, unsigned long long* __restrict__ bad_row,
             float shift_scale) {
  __shared__ float red_f[33];
  __shared__ double red_d[33];
  pdl_wait();
  pdl_launch_dependents();
  const int64_t w = blockIdx.x;
  const int64_t row = w / nch;
  const int ch = static_cast<int>(w - row * nch);
  const int64_t c0 = int64_t(ch) * kSplitChunk;
  const float* xr = x + row * ldx + c0;
  const int64_t rem = cols - c0;
  const int len = static_cast<int>(rem < kSplitChunk ? rem : kSplitChunk);
  float v[kSplitPerThread];
  // element i of this thread sits at column col(i): strided scalars, or
  // 128-bit vectors (thread-strided) when VEC == 4
  auto col = [&](int i) {
    return VEC == 4 ? 4 * (static_cast<int>(threadIdx.x) + (i / 4) * kSplitThreads) + (i % 4)
                    : static_cast<int>(threadIdx.x) + i * kSplitThreads;
  };
  if constexpr (VEC == 4) {
#pragma unroll
    for (int i = 0; i < kSplitPerThread; i += 4) {
      const int c = col(i);
      if (c < len) {
        const float4 t = ld_stream4(xr + c);
        v[i] = t.x; v[i + 1] = t.y; v[i + 2] = t.z; v[i + 3] = t.w;
      } else {
        v[i] = v[i + 1] = v[i + 2] = v[i + 3] = kPadLogit;
      }
    }
  } else {
#pragma unroll
    for (int i = 0; i < kSplitPerThread; ++i) {
      const int c = col(i);
      v[i] = c < len ? ld_stream1(xr + c) : kPadLogit;
    }
  }
  float mt = kPadLogit;
  u64 z = f2pk(0.0f, 0.0f);
#pragma unroll
  for (int i = 0; i < kSplitPerThread; i += 2) {
    mt = fmaxf(mt, fmaxf(v[i], v[i + 1]));
    z = nf_acc2(z, v[i], v[i + 1]);
  }
  if (nf_bad(z)) atomicMin(bad_row, static_cast<unsigned long long>(row));
  const float m = block_max_256(mt, red_f) * shift_scale;
  u64 acc = f2pk(0.0f, 0.0f);
#pragma unroll
  for (int i = 0; i < kSplitPerThread; i += 2) {
    float2 e = sexp2<MODE>(v[i], v[i + 1], m);
    if (!(col(i) < len)) e.x = 0.0f;
    if (!(col(i + 1) < len)) e.y = 0.0f;
    acc = f2add(acc, f2pk(e.x, e.y));
  }
  const float2 acc2 = f2up(acc);
  const double s = block_sum_256(static_cast<double>(acc2.x + acc2.y), red_d);
  if (threadIdx.x == 0) {
    RowPartial p;
    p.m = m;
    p.pad = 0.0f;
    p.s = s;
    partials[w] = p;
  }
}

// a row's (M, S) from its nch partials, by one warp in a fixed order (every
// caller -- k4_combine, k4_normalize_rows -- gets the same bits)
__device__ __forceinline__ void k4_combine_row(const RowPartial* __restrict__ rp, int nch, int lane,
                                               float& M, double& S) {
  M = kPadLogit;
  for (int q = lane; q < nch; q += 32) M = fmaxf(M, rp[q].m);
  M = group_max<32>(M);
  S = 0.0;
  for (int q = lane; q < nch; q += 32)
    S += rp[q].s * static_cast<double>(rp[q].m == M ? 1.0f : expf(rp[q].m - M));
  S = group_sum<32>(S);
}

// one warp per row
__global__ void k4_combine(const RowPartial* __restrict__ partials, int64_t rows, int nch,
                           float* __restrict__ row_max, double* __restrict__ row_sum) {
  pdl_wait();
  pdl_launch_dependents();
  const int64_t row = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  float M;
  double S;
  k4_combine_row(partials + row * nch, nch, lane, M, S);
  if (lane == 0) {
    row_max[row] = M;
    row_sum[row] = S;
  }
}

__global__ void k4_rescale(const float* __restrict__ local_max,
                           const float* __restrict__ global_max, double* __restrict__ sum,
                           int64_t rows) {
  pdl_wait();
  pdl_launch_dependents();
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= rows) return;
  const float d = local_max[i] - global_max[i];
  sum[i] *= static_cast<double>(d == 0.0f ? 1.0f : expf(d));
}

// y of item w = (row, chunk) given the row's M and 1/S
template <int MODE, int VEC>
__device__ __forceinline__ void k4_normalize_item(const float* __restrict__ x, float* __restrict__ y,
                                                  int64_t cols, int64_t ldx, int64_t ldy, int nch,
                                                  int64_t w, float M, float r) {
  const int64_t row = w / nch;
  const int ch = static_cast<int>(w - row * nch);
  const int64_t c0 = int64_t(ch) * kSplitChunk;
  const float* xr = x + row * ldx + c0;
  float* yr = y + row * ldy + c0;
  const int64_t rem = cols - c0;
  const int len = static_cast<int>(rem < kSplitChunk ? rem : kSplitChunk);
  if constexpr (VEC == 4) {
#pragma unroll
    for (int i = 0; i < kSplitPerThread / 4; ++i) {
      const int c = 4 * (threadIdx.x + i * kSplitThreads);
      if (c < len) {
        const float4 t = ld_stream4(xr + c);
        const float2 a = scale2<MODE>(sexp2<MODE>(t.x, t.y, M), r);
        const float2 b = scale2<MODE>(sexp2<MODE>(t.z, t.w, M), r);
        st_stream4(yr + c, make_float4(a.x, a.y, b.x, b.y));
      }
    }
  } else {
#pragma unroll
    for (int i = 0; i < kSplitPerThread; ++i) {
      const int c = threadIdx.x + i * kSplitThreads;
      if (c < len) st_stream1(yr + c, scale1<MODE>(sexp1<MODE>(ld_stream1(xr + c), M), r));
    }
  }
}

template <int MODE, int VEC>
__global__ void __launch_bounds__(kSplitThreads)
    k4_normalize(const float* __restrict__ x, float* __restrict__ y, int64_t rows, int64_t cols,
                 int64_t ldx, int64_t ldy, int nch, const float* __restrict__ row_max,
                 const double* __restrict__ row_sum) {
  pdl_wait();
  pdl_launch_dependents();
  const int64_t row = blockIdx.x / nch;
  k4_normalize_item<MODE, VEC>(x, y, cols, ldx, ldy, nch, blockIdx.x, row_max[row],
                               recip_of_sum(row_sum[row]));
}

// combine + normalize in one launch: warp 0 of every item merges its row's
// partials (k4_combine_row: the three-kernel path's bits), the block
// normalizes the item -- the split path as two launches
template <int MODE, int VEC>
__global__ void __launch_bounds__(kSplitThreads)
    k4_normalize_rows(const float* __restrict__ x, float* __restrict__ y, int64_t rows,
                      int64_t cols, int64_t ldx, int64_t ldy, int nch,
                      const RowPartial* __restrict__ partials) {
  __shared__ float M_s;
  __shared__ double S_s;
  pdl_wait();
  pdl_launch_dependents();
  const int64_t row = blockIdx.x / nch;
  if (threadIdx.x < 32) {
    float M;
    double S;
    k4_combine_row(partials + row * nch, nch, threadIdx.x, M, S);
    if (threadIdx.x == 0) {
      M_s = M;
      S_s = S;
    }
  }
  __syncthreads();
  k4_normalize_item<MODE, VEC>(x, y, cols, ldx, ldy, nch, blockIdx.x, M_s, recip_of_sum(S_s));
}

}  // namespace sk
