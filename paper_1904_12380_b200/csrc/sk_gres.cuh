// sk_gres.cuh -- K3g: a long row resident across P CTAs anywhere on the chip.
//
// K3c (sk_cluster.cuh) keeps a row in the shared memory of one thread-block
// cluster, but a cluster must fit inside one GPC, so the cluster sizes a 1 MB
// row needs (10-12 CTAs at 2 ring stages) pack only ~110 of the 148 SMs.  K3g
// drops the GPC constraint: a cooperative, persistent grid of one CTA per SM
// is cut into G = SMs / P groups of P CTAs; group g owns rows g, g+G, ... and
// CTA `rank` of the group holds columns [rank*L, (rank+1)*L) of the row in
// shared memory (TMA ring of NS stages, like K3c).
//
// The two row statistics are exchanged through global memory: every CTA
// publishes its partial (max, then f64 sum of exp) into a per-group slot array
// and bumps the group's monotonic counter with red.release.gpu; the group
// waits for counter == (exchange+1) * P with ld.acquire.gpu and reduces the P
// slots in fixed order, so M and S are bit-identical in every CTA of the row.
// Slots alternate by row parity: a CTA can be at most one exchange ahead.
//
// Warp specialisation keeps the handshake off the data path: warps 0..15
// compute (max pass, exp pass in place, normalise + streaming stores); warp
// 16 only issues the TMA loads and does the exchanges.  Its release fence thus
// never waits for the compute warps' output stores to drain (the stall that a
// single-role CTA pays at every global handshake), and named barriers hand the
// statistics between the roles:
//   bar 1  compute -> exchange  "CTA partials of this exchange are in smem"
//   bar 2  exchange -> compute  "row statistic broadcast in smem"
//   bar 3  compute -> exchange  "ring stage consumed (proxy-fenced): refill it"
// Traffic is 8 B/element in both HBM and L2 (the row never leaves the chip
// between its passes); kernels.py:144-188 is the operation order followed.
#pragma once
#include "sk_common.cuh"

namespace sk {

constexpr int kGresCompute = 512;                   // 16 compute warps
constexpr int kGresThreads = kGresCompute + 32;     // + 1 exchange/TMA warp
constexpr int kGresStages = 3;                      // maximum ring depth
constexpr unsigned kGresSpinLimit = 1u << 24;       // ~10 s of polling: abort, never hang

__device__ __forceinline__ void bar_sync_n(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_arrive_n(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ float ld_relaxed_f32(const float* p) {
  float v;
  asm volatile("ld.relaxed.gpu.global.f32 %0, [%1];" : "=f"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ double ld_relaxed_f64(const double* p) {
  double v;
  asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_f32(float* p, float v) {
  asm volatile("st.relaxed.gpu.global.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_f64(double* p, double v) {
  asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Exchange warp: all lanes poll the group counter (one broadcast load).  A
// stuck peer (impossible under a cooperative launch, but a hung GPU costs more
// than a wrong answer) raises the kernel-wide abort flag instead of spinning.
__device__ __forceinline__ void gres_wait(const unsigned* cnt, unsigned target, unsigned* abort_flag) {
  unsigned spins = 0;
  while (ld_acquire_gpu(cnt) < target) {
    if ((++spins & 0xFFFu) == 0) {
      if (ld_relaxed_u32(abort_flag)) return;
      if (spins >= kGresSpinLimit) {
        atomicExch(abort_flag, 1u);
        return;
      }
    }
  }
}

template <int MODE>
__global__ void __launch_bounds__(kGresThreads, 1)
    k3_gres(const float* __restrict__ x, float* __restrict__ y, int64_t rows, int64_t cols,
            int64_t ldx, int64_t ldy, int P, int slice, int nstages, unsigned* __restrict__ cnt_base,
            float* __restrict__ pmax, double* __restrict__ psum, unsigned* __restrict__ abort_flag,
            unsigned long long* __restrict__ bad_row, float shift_scale) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* stage_buf = reinterpret_cast<float*>(smem_raw);
  __shared__ uint64_t bars[kGresStages];
  __shared__ float red_f[kGresCompute / 32];
  __shared__ double red_d[kGresCompute / 32];
  __shared__ float bc_m;
  __shared__ double bc_s;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int G = static_cast<int>(gridDim.x) / P;
  const int g = static_cast<int>(blockIdx.x) / P, rank = static_cast<int>(blockIdx.x) % P;
  if (g >= G) return;  // whole CTA: no barrier below is shared with it
  const int64_t c0 = int64_t(rank) * slice;
  const int64_t rem = cols - c0;
  const int len = rem <= 0 ? 0 : static_cast<int>(rem < slice ? rem : slice);  // % 4 == 0
  const int nvec = len >> 2;

  if (tid == 0) {
    for (int s = 0; s < nstages; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  pdl_wait();

  if (warp == kGresCompute / 32) {
    // ------------------------------------------------ exchange + TMA warp
    unsigned* cnt = cnt_base + size_t(g) * 32;  // own 128-B line per group
    auto issue = [&](int64_t row, int stage) {
      mbar_arrive_expect_tx(&bars[stage], static_cast<uint32_t>(len) * 4u);
      if (len > 0)
        tma_load_1d(stage_buf + size_t(stage) * slice, x + row * ldx + c0,
                    static_cast<uint32_t>(len) * 4u, &bars[stage]);
    };
    if (lane == 0)
      for (int s = 0; s < nstages; ++s) {
        const int64_t row = g + int64_t(s) * G;
        if (row < rows) issue(row, s);
      }
    unsigned k = 0;
    for (int64_t row = g; row < rows; row += G, ++k) {
      const int par = k & 1;
      float* pm = pmax + (size_t(g) * 2 + par) * P;
      double* ps = psum + (size_t(g) * 2 + par) * P;
      // max exchange
      bar_sync_n(1, kGresThreads);
      float m = lane < kGresCompute / 32 ? red_f[lane] : kPadLogit;
      m = group_max<32>(m);
      if (lane == 0) {
        st_relaxed_f32(pm + rank, m);
        red_release_add_gpu(cnt, 1u);
      }
      gres_wait(cnt, (2u * k + 1u) * unsigned(P), abort_flag);
      float M = kPadLogit;
      for (int j = lane; j < P; j += 32) M = fmaxf(M, ld_relaxed_f32(pm + j));
      M = group_max<32>(M);
      if (lane == 0) bc_m = M * shift_scale;  // shift_scale = 0: fault hook
      bar_arrive_n(2, kGresThreads);
      // sum exchange
      bar_sync_n(1, kGresThreads);
      double t = lane < kGresCompute / 32 ? red_d[lane] : 0.0;
      t = group_sum<32>(t);
      if (lane == 0) {
        st_relaxed_f64(ps + rank, t);
        red_release_add_gpu(cnt, 1u);
      }
      gres_wait(cnt, (2u * k + 2u) * unsigned(P), abort_flag);
      double S = 0.0;
      for (int j = lane; j < P; j += 32) S += ld_relaxed_f64(ps + j);  // fixed order
      S = group_sum<32>(S);  // same butterfly in every CTA: identical S group-wide
      if (lane == 0) bc_s = S;
      bar_arrive_n(2, kGresThreads);
      // refill the consumed stage with the row NS steps ahead
      bar_sync_n(3, kGresThreads);
      const int64_t rn = row + int64_t(nstages) * G;
      if (lane == 0 && rn < rows) issue(rn, static_cast<int>(k % unsigned(nstages)));
    }
    return;
  }

  // ---------------------------------------------------------- compute warps
  unsigned k = 0;
  for (int64_t row = g; row < rows; row += G, ++k) {
    const int stage = static_cast<int>(k % unsigned(nstages));
    mbar_wait(&bars[stage], (k / unsigned(nstages)) & 1u);
    float4* sb = reinterpret_cast<float4*>(stage_buf + size_t(stage) * slice);

    float mt = kPadLogit;
    u64 z = f2pk(0.0f, 0.0f);
#pragma unroll 4
    for (int q = tid; q < nvec; q += kGresCompute) {
      const float4 v = sb[q];
      mt = fmaxf(mt, fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w)));
      z = nf_acc2(nf_acc2(z, v.x, v.y), v.z, v.w);
    }
    if (nf_bad(z)) atomicMin(bad_row, static_cast<unsigned long long>(row));
    mt = group_max<32>(mt);
    if (lane == 0) red_f[warp] = mt;
    bar_arrive_n(1, kGresThreads);
    bar_sync_n(2, kGresThreads);
    const float M = bc_m;

    u64 acc = f2pk(0.0f, 0.0f);
#pragma unroll 4
    for (int q = tid; q < nvec; q += kGresCompute) {
      const float4 v = sb[q];
      const float2 a = sexp2<MODE>(v.x, v.y, M);
      const float2 b = sexp2<MODE>(v.z, v.w, M);
      sb[q] = make_float4(a.x, a.y, b.x, b.y);
      acc = f2add(f2add(acc, f2pk(a.x, a.y)), f2pk(b.x, b.y));
    }
    const float2 acc2 = f2up(acc);
    const double sd = group_sum<32>(static_cast<double>(acc2.x + acc2.y));
    if (lane == 0) red_d[warp] = sd;
    bar_arrive_n(1, kGresThreads);
    bar_sync_n(2, kGresThreads);
    const float rcp = recip_of_sum(bc_s);

    float* yr = y + row * ldy + c0;
#pragma unroll 4
    for (int q = tid; q < nvec; q += kGresCompute) {
      const float4 e = sb[q];
      const float2 a = scale2<MODE>(make_float2(e.x, e.y), rcp);
      const float2 b = scale2<MODE>(make_float2(e.z, e.w), rcp);
      st_stream4(yr + 4 * q, make_float4(a.x, a.y, b.x, b.y));
    }
    fence_proxy_async_smem();  // generic smem accesses before the TMA refill
    bar_arrive_n(3, kGresThreads);
  }
}

}  // namespace sk
