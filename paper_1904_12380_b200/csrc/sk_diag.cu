// sk_diag.cu -- accuracy diagnostics for the hot-path exponential.
//
// sk_exp_accuracy sweeps EVERY fp32 value in [lo, hi] (hi <= 0) through the
// kernels' exponential (sexp2 packed path and sexp1 scalar path, as used by
// the softmax kernels with m = 0) and compares it with the double-precision
// exp, reporting the worst error in units of the fp32 ulp of the true result
// and the worst relative error.  The reference's own exp (glibc expf via
// numba, kernels.py:171-174) is within 0.5 ulp of the true value, so the
// difference to the reference is bounded by max_ulp + 0.5.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstring>

#include "../../include/softmax_b200.h"
#include "sk_common.cuh"

namespace sk {
namespace {

__device__ __forceinline__ double ulp_of(double v) {
  // fp32 ulp of the magnitude v (normal range; subnormal spacing below)
  int e;
  frexp(v, &e);  // v = f * 2^e, f in [0.5, 1)
  const int ee = e - 1;
  return ee < -126 ? ldexp(1.0, -149) : ldexp(1.0, ee - 23);
}

template <int MODE>
__global__ void exp_sweep(uint32_t bits_lo, uint64_t n, unsigned long long* max_ulp_bits,
                          unsigned long long* max_rel_bits) {
  double worst_ulp = 0.0, worst_rel = 0.0;
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < (n + 1) / 2;
       i += stride) {
    const uint64_t i0 = 2 * i, i1 = (2 * i + 1 < n) ? 2 * i + 1 : 2 * i;
    const float x0 = __uint_as_float(bits_lo + static_cast<uint32_t>(i0));
    const float x1 = __uint_as_float(bits_lo + static_cast<uint32_t>(i1));
    const float2 p = sexp2<MODE>(x0, x1, 0.0f);
    const float q0 = sexp1<MODE>(x0, 0.0f);
    const float xs[2] = {x0, x1};
    const float ys[3] = {p.x, p.y, q0};
    for (int k = 0; k < 3; ++k) {
      const float xv = xs[k == 1 ? 1 : 0];
      const double ref = exp(static_cast<double>(fmaxf(xv, exp_floor<MODE>())));
      const double err = fabs(static_cast<double>(ys[k]) - ref);
      worst_ulp = fmax(worst_ulp, err / ulp_of(ref));
      worst_rel = fmax(worst_rel, err / ref);
    }
  }
  atomicMax(max_ulp_bits, static_cast<unsigned long long>(__double_as_longlong(worst_ulp)));
  atomicMax(max_rel_bits, static_cast<unsigned long long>(__double_as_longlong(worst_rel)));
}

}  // namespace
}  // namespace sk

extern "C" int sk_exp_accuracy(int mode, float lo, float hi, double* max_ulp, double* max_rel,
                               int device) {
  if (!(lo <= hi) || hi > 0.0f || mode < 0 || mode > 2 || !max_ulp || !max_rel)
    return SK_ERR_ARGUMENT;
  if (cudaSetDevice(device) != cudaSuccess) return SK_ERR_CUDA;
  // negative floats: magnitude grows with the bit pattern; [lo, hi] <-> [bits(hi), bits(lo)]
  uint32_t bhi, blo;
  float h = hi == 0.0f ? -0.0f : hi;
  std::memcpy(&bhi, &h, 4);
  std::memcpy(&blo, &lo, 4);
  if (!(bhi & 0x80000000u)) bhi = 0x80000000u;
  const uint64_t n = uint64_t(blo) - uint64_t(bhi) + 1;
  unsigned long long* d = nullptr;
  if (cudaMalloc(&d, 16) != cudaSuccess) return SK_ERR_RESOURCE;
  cudaMemset(d, 0, 16);
  const int threads = 256, blocks = 148 * 16;
  switch (mode) {
    case 0: sk::exp_sweep<sk::kClipAccurate><<<blocks, threads>>>(bhi, n, d, d + 1); break;
    case 1: sk::exp_sweep<sk::kAccurate><<<blocks, threads>>>(bhi, n, d, d + 1); break;
    default: sk::exp_sweep<sk::kApprox><<<blocks, threads>>>(bhi, n, d, d + 1); break;
  }
  unsigned long long h2[2] = {0, 0};
  cudaError_t e = cudaMemcpy(h2, d, 16, cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e != cudaSuccess) return SK_ERR_CUDA;
  std::memcpy(max_ulp, &h2[0], 8);
  std::memcpy(max_rel, &h2[1], 8);
  return SK_OK;
}

// ---------------------------------------------------------------------------
// Diagnostic streaming copy with the softmax kernels' access pattern
// (128-bit no-allocate loads, streaming stores, PDL): the same-run floor for a
// kernel that moves 8 B/element, used by scripts/sweep.py and the bound probe.
namespace sk {
namespace {
__global__ void __launch_bounds__(256) k_copy4(const float4* __restrict__ x, float4* __restrict__ y,
                                               int64_t n4) {
  pdl_wait();
  pdl_launch_dependents();
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n4; i += 4 * stride) {
    const float4 a = ld_stream4(reinterpret_cast<const float*>(x + i));
    const float4 b = ld_stream4(reinterpret_cast<const float*>(x + i + stride));
    const float4 c = ld_stream4(reinterpret_cast<const float*>(x + i + 2 * stride));
    const float4 d = ld_stream4(reinterpret_cast<const float*>(x + i + 3 * stride));
    st_stream4(reinterpret_cast<float*>(y + i), a);
    st_stream4(reinterpret_cast<float*>(y + i + stride), b);
    st_stream4(reinterpret_cast<float*>(y + i + 2 * stride), c);
    st_stream4(reinterpret_cast<float*>(y + i + 3 * stride), d);
  }
  for (; i < n4; i += stride)
    st_stream4(reinterpret_cast<float*>(y + i), ld_stream4(reinterpret_cast<const float*>(x + i)));
}
}  // namespace
}  // namespace sk

extern "C" int sk_copy_f32(const float* x, float* y, int64_t n, int blocks, void* stream) {
  if (n < 0 || (n % 4) || (n > 0 && (!x || !y)) ||
      (reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) % 16)
    return SK_ERR_ARGUMENT;
  if (n == 0) return SK_OK;
  const int64_t n4 = n / 4;
  int64_t g = blocks > 0 ? blocks : (n4 + 1023) / 1024;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(g < 1 ? 1 : g));
  cfg.blockDim = dim3(256);
  cfg.stream = static_cast<cudaStream_t>(stream);
  cudaLaunchAttribute a[1];
  a[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  a[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = a;
  cfg.numAttrs = 1;
  const float4* xs = reinterpret_cast<const float4*>(x);
  float4* ys = reinterpret_cast<float4*>(y);
  return cudaLaunchKernelEx(&cfg, sk::k_copy4, xs, ys, n4) == cudaSuccess ? SK_OK : SK_ERR_CUDA;
}
