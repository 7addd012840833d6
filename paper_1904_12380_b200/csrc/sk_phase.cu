// sk_phase.cu -- the reference's three softmax phases as separate kernels.
//
// Not the hot path: the fused kernels (K1-K4) are.  These exist so the GPU
// can reproduce the reference's phase structure -- variant_pipeline /
// PhasePipeline (kernels.py:283-339) and the Fig. 2 phase profile
// (profiler.py:96-133) -- with the same per-phase semantics:
//
//   sk_maxsub_f32    kernels.py:136-151  y = x - rowmax (ValueClip at -64 if clip)
//   sk_exp_f32       kernels.py:171-174  buf = exp(buf), elementwise, in place
//   sk_sumscale_f32  kernels.py:177-189  S = sum(row) (f64), r = 1/(float)S,
//                                        y = e*r, y < FLT_MIN -> +0, in place
//
// and the reference's 1-D component operations (kernels.py:229-276), which
// compose into the same phases:
//
//   sk_row_sum_f32      kernels.py:258-260  S = sum(row) accumulated in f64
//   sk_shift_scale_f32  kernels.py:234-236  y = x - v        (scale 1: exact)
//                       kernels.py:263-269  y = x * (1/s)    (shift 0: exact)
//
// One CTA per row, grid-stride over columns, any row pitch / alignment.
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/softmax_b200.h"
#include "sk_common.cuh"

namespace sk {
namespace {

constexpr int kPhaseThreads = 256;

__device__ __forceinline__ float cta_reduce_max(float v, float* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = group_max<32>(v);
  if (lane == 0) red[warp] = v;
  __syncthreads();
  float m = red[0];
  for (int w = 1; w < kPhaseThreads / 32; ++w) m = fmaxf(m, red[w]);
  __syncthreads();
  return m;
}
__device__ __forceinline__ double cta_reduce_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = group_sum<32>(v);
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = red[0];
  for (int w = 1; w < kPhaseThreads / 32; ++w) s += red[w];
  __syncthreads();
  return s;
}

__global__ void __launch_bounds__(kPhaseThreads)
    k_maxsub(const float* __restrict__ x, float* __restrict__ y, int64_t cols, int64_t ldx,
             int64_t ldy, int clip, float shift_scale) {
  __shared__ float red[kPhaseThreads / 32];
  const float* xr = x + int64_t(blockIdx.x) * ldx;
  float* yr = y + int64_t(blockIdx.x) * ldy;
  float m = kPadLogit;
  for (int64_t c = threadIdx.x; c < cols; c += kPhaseThreads) m = fmaxf(m, xr[c]);
  m = cta_reduce_max(m, red) * shift_scale;
  for (int64_t c = threadIdx.x; c < cols; c += kPhaseThreads) {
    const float s = xr[c] - m;
    yr[c] = clip ? (s > kClipFloor ? s : kClipFloor) : s;
  }
}

// exp over the whole float range for the unclipped modes: like sexp1, but a
// result below FLT_MIN comes out subnormal (as np.exp / glibc expf give it,
// exp_batch kernels.py:245-255) instead of flushed: ex2 of t + 32 (exact for
// these t), then an exact scale by 2^-32 that rounds once into the subnormal
// range.  Not on the fused path, which flushes such outputs anyway.
__device__ __forceinline__ float exp_subnormal(float s) {
  s = fmaxf(s, -104.0f);  // exp(-104) < 2^-150 (rounds to 0); keeps t finite
  const float t = s * kLog2eHi;
  const float d = fmaf(fmaf(s, kLog2eHi, -t), kLn2, s * kLog2eLoLn2);
  const float p = ex2_ftz(t + 32.0f);
  return __fmul_rn(fmaf(p, d, p), 2.3283064365386963e-10f);  // 2^-32
}

template <int MODE>
__global__ void k_exp(float* __restrict__ buf, int64_t n) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const float v = buf[i];
    buf[i] = (MODE == kAccurate && v < -87.0f) ? exp_subnormal(v) : sexp1<MODE>(v, 0.0f);
  }
}

__global__ void __launch_bounds__(kPhaseThreads)
    k_sumscale(float* __restrict__ buf, int64_t cols, int64_t ld) {
  __shared__ double red[kPhaseThreads / 32];
  float* r = buf + int64_t(blockIdx.x) * ld;
  double s = 0.0;
  for (int64_t c = threadIdx.x; c < cols; c += kPhaseThreads) s += static_cast<double>(r[c]);
  s = cta_reduce_sum(s, red);
  const float rcp = recip_of_sum(s);
  for (int64_t c = threadIdx.x; c < cols; c += kPhaseThreads) r[c] = scale_flush(r[c], rcp);
}

__global__ void __launch_bounds__(kPhaseThreads)
    k_rowsum(const float* __restrict__ x, int64_t cols, int64_t ldx, double* __restrict__ out) {
  __shared__ double red[kPhaseThreads / 32];
  const float* r = x + int64_t(blockIdx.x) * ldx;
  double s = 0.0;
  for (int64_t c = threadIdx.x; c < cols; c += kPhaseThreads) s += static_cast<double>(r[c]);
  s = cta_reduce_sum(s, red);
  if (threadIdx.x == 0) out[blockIdx.x] = s;
}

// y = (x - shift) * scale: IEEE subtract then multiply, so shift = v, scale = 1
// is exactly x - v and shift = 0, scale = r exactly x * r (NaN/Inf propagate)
__global__ void k_shift_scale(const float* __restrict__ x, float* __restrict__ y, int64_t n,
                              float shift, float scale) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    y[i] = __fmul_rn(__fsub_rn(x[i], shift), scale);
}

// row_max_scalar / row_stats of ONE row with the reference's semantics for
// ANY input (kernels.py:119-126 strict '>' scan from a[0]; kernels.py:272-276
// sum of np.exp(row - max) in f64): max = NaN if a[0] is NaN, else the largest
// non-NaN value (-inf for an all -inf row); sum = sum of expf(a - max) with
// IEEE propagation (NaN / inf in, NaN / inf out).  The component ops take it
// for rows the fast stats kernel flagged as non-finite.
__global__ void __launch_bounds__(kPhaseThreads)
    k_row_stats_ref(const float* __restrict__ x, int64_t n, float* __restrict__ out_max,
                    double* __restrict__ out_sum) {
  __shared__ float redf[kPhaseThreads / 32];
  __shared__ double red[kPhaseThreads / 32];
  __shared__ float mb;
  float m = -INFINITY;
  for (int64_t i = threadIdx.x; i < n; i += kPhaseThreads) m = fmaxf(m, x[i]);  // NaN ignored
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) redf[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    float v = redf[0];
    for (int w = 1; w < kPhaseThreads / 32; ++w) v = fmaxf(v, redf[w]);
    mb = isnan(x[0]) ? x[0] : v;
  }
  __syncthreads();
  const float M = mb;
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += kPhaseThreads)
    s += static_cast<double>(expf(__fsub_rn(x[i], M)));
  s = cta_reduce_sum(s, red);
  if (threadIdx.x == 0) {
    *out_max = M;
    *out_sum = s;
  }
}

unsigned elementwise_grid(int64_t n) {
  int sms = 148;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (n + 255) / 256;
  return static_cast<unsigned>(want < int64_t(sms) * 16 ? want : int64_t(sms) * 16);
}

bool bad_shape(const void* a, const void* b, int64_t rows, int64_t cols, int64_t ld1,
               int64_t ld2) {
  return rows < 0 || cols < 1 || ld1 < cols || ld2 < cols || rows > INT32_MAX ||
         (rows > 0 && (!a || !b));
}

}  // namespace
}  // namespace sk

extern "C" {

int sk_maxsub_f32(const float* x, float* y, int64_t rows, int64_t cols, int64_t ldx,
                  int64_t ldy, int clip, void* stream) {
  if (sk::bad_shape(x, y, rows, cols, ldx, ldy)) return SK_ERR_ARGUMENT;
  if (rows == 0) return SK_OK;
  sk::k_maxsub<<<static_cast<unsigned>(rows), sk::kPhaseThreads, 0,
                 static_cast<cudaStream_t>(stream)>>>(x, y, cols, ldx, ldy, clip ? 1 : 0, 1.0f);
  return cudaGetLastError() == cudaSuccess ? SK_OK : SK_ERR_CUDA;
}

int sk_exp_f32(float* buf, int64_t n, int mode, void* stream) {
  if (n < 0 || (n > 0 && !buf) || mode < 0 || mode > 2) return SK_ERR_ARGUMENT;
  if (n == 0) return SK_OK;
  const unsigned grid = sk::elementwise_grid(n);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  switch (mode) {
    case 0: sk::k_exp<sk::kClipAccurate><<<grid, 256, 0, s>>>(buf, n); break;
    case 1: sk::k_exp<sk::kAccurate><<<grid, 256, 0, s>>>(buf, n); break;
    default: sk::k_exp<sk::kApprox><<<grid, 256, 0, s>>>(buf, n); break;
  }
  return cudaGetLastError() == cudaSuccess ? SK_OK : SK_ERR_CUDA;
}

int sk_sumscale_f32(float* buf, int64_t rows, int64_t cols, int64_t ld, void* stream) {
  if (sk::bad_shape(buf, buf, rows, cols, ld, ld)) return SK_ERR_ARGUMENT;
  if (rows == 0) return SK_OK;
  sk::k_sumscale<<<static_cast<unsigned>(rows), sk::kPhaseThreads, 0,
                   static_cast<cudaStream_t>(stream)>>>(buf, cols, ld);
  return cudaGetLastError() == cudaSuccess ? SK_OK : SK_ERR_CUDA;
}

int sk_row_sum_f32(const float* x, int64_t rows, int64_t cols, int64_t ldx, double* row_sum,
                   void* stream) {
  if (sk::bad_shape(x, row_sum, rows, cols, ldx, cols)) return SK_ERR_ARGUMENT;
  if (rows == 0) return SK_OK;
  sk::k_rowsum<<<static_cast<unsigned>(rows), sk::kPhaseThreads, 0,
                 static_cast<cudaStream_t>(stream)>>>(x, cols, ldx, row_sum);
  return cudaGetLastError() == cudaSuccess ? SK_OK : SK_ERR_CUDA;
}

int sk_row_stats_ref_f32(const float* x, int64_t n, float* row_max, double* row_sum,
                         void* stream) {
  if (n < 1 || !x || !row_max || !row_sum) return SK_ERR_ARGUMENT;
  sk::k_row_stats_ref<<<1, sk::kPhaseThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      x, n, row_max, row_sum);
  return cudaGetLastError() == cudaSuccess ? SK_OK : SK_ERR_CUDA;
}

int sk_shift_scale_f32(const float* x, float* y, int64_t n, float shift, float scale,
                       void* stream) {
  if (n < 0 || (n > 0 && (!x || !y))) return SK_ERR_ARGUMENT;
  if (n == 0) return SK_OK;
  sk::k_shift_scale<<<sk::elementwise_grid(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      x, y, n, shift, scale);
  return cudaGetLastError() == cudaSuccess ? SK_OK : SK_ERR_CUDA;
}

}  // extern "C"
