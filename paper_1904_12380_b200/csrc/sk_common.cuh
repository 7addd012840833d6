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

// ---- packed fp32x2 arithmetic (sm_100a FADD2/FMUL2/FFMA2) -----------------
typedef unsigned long long u64;
__device__ __forceinline__ u64 f2pk(float a, float b) {
  u64 r;
  asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float2 f2up(u64 r) {
  float2 v;
  asm("mov.b64 {%0,%1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(r));
  return v;
}
__device__ __forceinline__ u64 f2add(u64 a, u64 b) {
  u64 d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ u64 f2sub(u64 a, u64 b) {
  u64 d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ u64 f2mul(u64 a, u64 b) {
  u64 d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ u64 f2mul_ftz(u64 a, u64 b) {
  u64 d;
  asm("mul.rn.ftz.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ u64 f2fma(u64 a, u64 b, u64 c) {
  u64 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ float ex2_ftz(float t) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(t));
  return r;
}

// ---- the exponential used on the hot path -----------------------------------
// exp(s) for a shifted logit s <= 0, clamped first at the mode's floor:
//   clip mode  : -64 (the reference's ValueClip, kernels.py:147 -- exactly
//                `s > -64 ? s : -64`, since fmaxf(s, -64) is that for non-NaN s)
//   other modes: -104 (every exp below FLT_MIN flushes to 0 in the output
//                anyway, kernels.py:186-188; the floor keeps the arithmetic finite)
// Accurate modes: with L = log2(e) = L_hi + L_lo,
//   t  = fl(s * L_hi)                     (MUFU argument)
//   d  = (s*L_hi - t) * ln2 + s*(L_lo*ln2)  (the rounding error of t, exact via FMA)
//   e  = ex2(t) * (1 + d)                 (one MUFU.EX2 per element)
// so the MUFU sees one rounded argument and the lost low bits are put back by
// a first-order correction (|d| < 4e-6).  Measured accuracy is reported by
// sk_exp_accuracy() and tests/test_gpu_parity.py::test_exp_accuracy_exhaustive.
// Everything except the clamp and the MUFU runs as packed fp32x2 (FFMA2 etc.),
// ~5 issue slots per element instead of ~10 for libdevice expf.
constexpr float kLog2eHi = 1.44269502162933349609375f;            // fp32(log2 e)
constexpr float kLog2eLoLn2 = 1.925963033500011079e-08f * 0.69314718055994530942f;
constexpr float kLn2 = 0.69314718055994530942f;
constexpr float kLog2e = 1.4426950408889634f;

template <int MODE>
__device__ __forceinline__ constexpr float exp_floor() {
  return MODE == kClipAccurate ? kClipFloor : -104.0f;
}

// (x0, x1) -> (exp(clamp(x0 - m)), exp(clamp(x1 - m)))
template <int MODE>
__device__ __forceinline__ float2 sexp2(float x0, float x1, float m) {
  const float2 s = f2up(f2sub(f2pk(x0, x1), f2pk(m, m)));
  const float s0 = fmaxf(s.x, exp_floor<MODE>()), s1 = fmaxf(s.y, exp_floor<MODE>());
  const u64 S = f2pk(s0, s1);
  if (MODE == kApprox) {
    const float2 t = f2up(f2mul(S, f2pk(kLog2e, kLog2e)));
    return make_float2(ex2_ftz(t.x), ex2_ftz(t.y));
  }
  const u64 tn = f2mul(S, f2pk(-kLog2eHi, -kLog2eHi));      // -t
  const u64 d1 = f2fma(S, f2pk(kLog2eHi, kLog2eHi), tn);    // s*L_hi - t (exact)
  const u64 d = f2fma(d1, f2pk(kLn2, kLn2), f2mul(S, f2pk(kLog2eLoLn2, kLog2eLoLn2)));
  const float2 t = f2up(tn);
  const u64 p = f2pk(ex2_ftz(-t.x), ex2_ftz(-t.y));
  return f2up(f2fma(p, d, p));
}

template <int MODE>
__device__ __forceinline__ float sexp1(float x, float m) {
  const float s = fmaxf(x - m, exp_floor<MODE>());
  if (MODE == kApprox) return ex2_ftz(s * kLog2e);
  const float t = s * kLog2eHi;
  const float d = fmaf(fmaf(s, kLog2eHi, -t), kLn2, s * kLog2eLoLn2);
  const float p = ex2_ftz(t);
  return fmaf(p, d, p);
}

// Backwards-compatible scalar name used by the split kernels.
template <int MODE>
__device__ __forceinline__ float shifted_exp(float x, float m) {
  return sexp1<MODE>(x, m);
}

// Output scale y = e * r with the reference's flush of sub-normal results to
// +0 (kernels.py:186-188).  In clip mode every output is >= e^-64 / C, which is
// normal for C < 1.3e10 (checked by the launcher), so the flush cannot fire and
// a plain multiply is bit-identical; otherwise the ftz multiply flushes exactly
// the results below FLT_MIN.
template <int MODE>
__device__ __forceinline__ float2 scale2(float2 e, float r) {
  const u64 E = f2pk(e.x, e.y), R = f2pk(r, r);
  return f2up(MODE == kClipAccurate ? f2mul(E, R) : f2mul_ftz(E, R));
}
template <int MODE>
__device__ __forceinline__ float scale1(float e, float r) {
  const float y = e * r;
  return (MODE != kClipAccurate && y < kFltMinNormal) ? 0.0f : y;
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

// Non-finite accumulator: z += x * 0 stays +-0 for finite x and turns NaN for
// any +-Inf/NaN; packed, half an issue slot per element.
__device__ __forceinline__ u64 nf_acc2(u64 z, float a, float b) {
  return f2fma(f2pk(a, b), f2pk(0.0f, 0.0f), z);
}
__device__ __forceinline__ bool nf_bad(u64 z) {
  const float2 v = f2up(z);
  return !(v.x == 0.0f && v.y == 0.0f);
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
// 256-bit variants (sm_100): one request moves 32 B; needs 32-B alignment.
__device__ __forceinline__ void ld_stream8(const float* p, float (&v)[8]) {
  asm volatile(
      "ld.global.nc.L1::no_allocate.L2::evict_first.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]),
        "=f"(v[7])
      : "l"(p));
}
__device__ __forceinline__ void st_stream8(float* p, const float (&v)[8]) {
  asm volatile("st.global.cs.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(v[0]),
               "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
               : "memory");
}
// Outputs are written once and not re-read by this kernel: streaming store.
__device__ __forceinline__ void st_stream4(float* p, float4 v) {
  asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y),
               "f"(v.z), "f"(v.w)
               : "memory");
}
__device__ __forceinline__ float2 ld_stream2(const float* p) {
  float2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f32 {%0,%1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ void st_stream2(float* p, float2 v) {
  asm volatile("st.global.cs.v2.f32 [%0], {%1,%2};" ::"l"(p), "f"(v.x), "f"(v.y) : "memory");
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

// ---- timing chaos for the barrier-heavy kernels (K3g, K3c) ------------------
// Timing chaos (gres_diag bit 6; bits 8.. seed it): pseudo-random per-warp
// delays of up to ~4 us at every hand-off point -- before waiting for a stage,
// arriving at a named barrier, publishing, refilling, polling, writing out --
// so the tests can shake the schedule the barriers, mbarriers and tagged slots
// must hold under (the pool's GPUs refuse compute-sanitizer's racecheck).
// Results must not change by a bit; a missed dependency shows as wrong output
// or as the exchange timing out.
__device__ __forceinline__ void timing_chaos(int diag, unsigned point, unsigned k) {
  if (diag & 64) {
    unsigned h = (blockIdx.x * 2654435761u) ^ ((threadIdx.x >> 5) * 0x9E3779B1u) ^
                 (point * 0x85EBCA6Bu) ^ (k * 0xC2B2AE35u) ^ (static_cast<unsigned>(diag) >> 8);
    h ^= h >> 15;
    h *= 0x2C1B3C6Du;
    h ^= h >> 12;
    h *= 0x297A2D39u;
    h ^= h >> 15;
    if ((h & 3u) == 0u) __nanosleep(100u + ((h >> 8) & 4095u));
  }
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
