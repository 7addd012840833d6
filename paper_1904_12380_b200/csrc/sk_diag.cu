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
