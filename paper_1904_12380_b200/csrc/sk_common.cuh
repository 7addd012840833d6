// sk_common.cuh -- device helpers shared by every softmax kernel (sm_100a).
//
// Numeric contract (reference /root/reference/pkg/src/softmax_kit/kernels.py):
//   s = x - m                    kernels.py:146 (fp32 subtract)
//   s = s > -64 ? s : -64        kernels.py:147 (ValueClip, CLIP_FLOOR kernels.py:99)
//   e = exp(s)                   kernels.py:171-174
//   S = sum(e) (wide accumulate) kernels.py:181-183 (f64 there; here fp32 chains of
//                                <= 64 terms, combined in f64 -- see DESIGN.md §4)
//   r = 1.0f / (float)S          kernels.py:184 (IEEE reciprocal, never a divide per element)
//   y = e * r; y < FLT_MIN -> +0 kernels.py:185-188
#pragma once
#include <cstdint>
#include <cfloat>
#include <cuda_runtime.h>

namespace sk {

// Exp modes: the variant ladder maps onto these (kernels.py:76-96).
enum ExpMode : int {
  kClipAccurate = 0,   // ReferenceClipped
  kAccurate = 1,       // ReferenceInference / MklStyleScalar / VectorizedSum / FullVectorized
  kApprox = 2,         // FullVectorizedApproxExp (ex2.approx based, tol 1e-5: bench.py:52)
};

constexpr float kClipFloor = -64.0f;                  // kernels.py:99
constexpr float kFltMinNormal = 1.1754943508222875e-38f;  // kernels.py:101
constexpr float kPadLogit = -FLT_MAX;                 // padding for max (finite!)

template <int MODE>
__device__ __forceinline__ float shifted_exp(float x, float m) {
  float s = x - m;
  if (MODE == kClipAccurate) s = s > kClipFloor ? s : kClipFloor;
  if (MODE == kApprox) {
    float r;
    // ex2.approx.ftz: 2^(s*log2e); rel. error ~2^-22 + |s|*log2e*2^-24
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(s * 1.4426950408889634f));
    return r;
  }
  return expf(s);  // CUDA libdevice expf, <= 2 ulp (compiled without fast-math)
}

// Output scale with the reference's flush-to-zero of sub-normal results.
__device__ __forceinline__ float scale_flush(float e, float r) {
  float y = e * r;
  return y < kFltMinNormal ? 0.0f : y;
}

// IEEE round-to-nearest reciprocal of the fp32-rounded sum (kernels.py:184).
__device__ __forceinline__ float recip_of_sum(double s) {
  return __frcp_rn(__double2float_rn(s));
}

// Non-finite detector: true iff |x| is Inf or x is NaN.  One FSETP per element.
__device__ __forceinline__ bool not_finite(float x) { return !(fabsf(x) <= FLT_MAX); }

// ---- warp reductions over aligned groups of G lanes (G power of two) -----
template <int G>
__device__ __forceinline__ float group_max(float v) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
template <int G>
__device__ __forceinline__ double group_sum(double v) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
template <int G>
__device__ __forceinline__ bool group_any(bool b) {
  if (G == 1) return b;
  return __any_sync(0xffffffffu, b);  // conservative: any lane of the warp
}

// ---- streaming global memory access ----------------------------------------
// Inputs are read exactly once: bypass L1 allocation.
__device__ __forceinline__ float4 ld_stream4(const float* p) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ float ld_stream1(const float* p) {
  float v;
  asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}
// Outputs are written once and not re-read by this kernel: streaming store.
__device__ __forceinline__ void st_stream4(float* p, float4 v) {
  asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y),
               "f"(v.z), "f"(v.w)
               : "memory");
}
__device__ __forceinline__ void st_stream1(float* p, float v) {
  asm volatile("st.global.cs.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}

// ---- mbarrier + TMA 1-D bulk copy (cp.async.bulk) ---------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile(
      "{\n\t.reg .b64 st;\n\t"
      "mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(smem_u32(bar)),
      "r"(bytes)
      : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
// global -> shared bulk copy; bytes % 16 == 0, both addresses 16-B aligned.
__device__ __forceinline__ void tma_load_1d(void* smem_dst, const void* gmem_src, uint32_t bytes,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(smem_dst)),
      "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar)), "l"(0x12F0000000000000ull)  // EVICT_FIRST
      : "memory");
}

// ---- programmatic dependent launch (PDL) -----------------------------------
// Every kernel waits for its stream predecessor's memory to be visible before
// touching global memory, then immediately lets its own successor be
// scheduled, so back-to-back launches overlap launch latency and tail.  Both
// are no-ops when the launch did not carry the PDL attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ---- global-scope acquire/release for cross-CTA row statistics --------------
__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add_gpu(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

}  // namespace sk
