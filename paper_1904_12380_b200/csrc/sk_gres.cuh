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
// One exchange per row, overlapped with the next row.  Each compute warp
// reduces its share of the slice to a pair (m_w, s_w = sum exp(clip(x - m_w)))
// without any CTA barrier; the exchange warp merges the 16 pairs into the CTA
// pair (fixed order, s_w scaled by exp(m_w - m)), publishes it into the
// group's slot array and bumps the group's monotonic counter with
// red.release.gpu, then waits for counter == (k+1) * P with ld.acquire.gpu and
// merges the P pairs in rank order -- so M and S are bit-identical in every CTA
// of the row.  Meanwhile the compute warps already run row k+1's local pass;
// only then do they write row k: y = exp(clip(x - M)) * (1/(float)S), the exp
// recomputed against the GLOBAL max from the untouched slice (reference order,
// kernels.py:144-188).  The group round trip (~1.5 us through L2) therefore
// hides behind a full row step instead of stalling it.  Slots alternate by
// row parity (a CTA can run at most one exchange ahead of its group).
//
// Warp specialisation keeps the handshake off the data path: warp 16 only
// issues the TMA loads and does the exchanges, so its release fence never
// waits for the compute warps' output stores to drain.  Named barriers:
//   bar 1/4  compute -> exchange  "warp pairs of row k in smem" (by row parity)
//   bar 2    exchange -> compute  "(M, S) of row k in smem"
//   bar 3    compute -> exchange  "row k's stage consumed (proxy-fenced): refill"
// HBM and L2 each see 8 B/element: the row never leaves the chip between its
// three shared-memory passes (ring depth NS >= 3 keeps one row loading, one
// in its local pass and one awaiting its statistics).
#pragma once
#include "sk_common.cuh"

namespace sk {

constexpr int kGresCompute = 512;                   // 16 compute warps
constexpr int kGresThreads = kGresCompute + 32;     // + 1 exchange/TMA warp
constexpr int kGresStages = 4;                      // maximum ring depth
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
  constexpr int NW = kGresCompute / 32;
  __shared__ uint64_t bars[kGresStages];
  __shared__ float red_f[2][NW];   // [row parity][warp]: warp-local max
  __shared__ double red_d[2][NW];  //                     warp-local sum vs that max
  __shared__ float bc_m[2];        // [row parity] merged row max / sum
  __shared__ double bc_s[2];

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

  if (warp == NW) {
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
      // CTA pair (m, s) of row k from the 16 warp pairs, fixed order
      bar_sync_n(1 + 3 * par, kGresThreads);
      const float mw = lane < NW ? red_f[par][lane] : kPadLogit;
      const float mc = group_max<32>(mw);
      double sw = lane < NW ? red_d[par][lane] : 0.0;
      if (lane < NW && mw != mc) sw *= static_cast<double>(expf(mw - mc));
      const double sc = group_sum<32>(sw);
      float* pm = pmax + (size_t(g) * 2 + par) * P;
      double* ps = psum + (size_t(g) * 2 + par) * P;
      if (lane == 0) {
        st_relaxed_f32(pm + rank, mc);
        st_relaxed_f64(ps + rank, sc);
        red_release_add_gpu(cnt, 1u);
      }
      // while the group's pairs arrive: refill the stage row k-1 released
      if (k > 0) {
        bar_sync_n(3, kGresThreads);
        const int64_t rn = row - G + int64_t(nstages) * G;
        if (lane == 0 && rn < rows) issue(rn, static_cast<int>((k - 1) % unsigned(nstages)));
      }
      gres_wait(cnt, (k + 1u) * unsigned(P), abort_flag);
      // merge the P pairs in rank order: identical (M, S) in every CTA of the row
      float Mg = kPadLogit;
      for (int j = lane; j < P; j += 32) Mg = fmaxf(Mg, ld_relaxed_f32(pm + j));
      Mg = group_max<32>(Mg);
      double S = 0.0;
      for (int j = lane; j < P; j += 32) {
        const float mj = ld_relaxed_f32(pm + j);
        double sj = ld_relaxed_f64(ps + j);
        if (mj != Mg) sj *= static_cast<double>(expf(mj - Mg));
        S += sj;
      }
      S = group_sum<32>(S);
      if (lane == 0) {
        bc_m[par] = Mg * shift_scale;  // shift_scale = 0: fault hook
        bc_s[par] = S;
      }
      bar_arrive_n(2, kGresThreads);
    }
    if (k > 0) bar_sync_n(3, kGresThreads);  // last row's output pass done
    return;
  }

  // ---------------------------------------------------------- compute warps
  // row k's output pass runs after row k+1's local pass, so the group
  // exchange of row k overlaps a full row of streaming work.
  auto output = [&](unsigned j, int64_t orow) {
    bar_sync_n(2, kGresThreads);
    const float M = bc_m[j & 1];
    const float rcp = recip_of_sum(bc_s[j & 1]);
    const float4* sb = reinterpret_cast<const float4*>(stage_buf + size_t(j % unsigned(nstages)) * slice);
    float* yr = y + orow * ldy + c0;
#pragma unroll 4
    for (int q = tid; q < nvec; q += kGresCompute) {
      const float4 v = sb[q];
      const float2 a = scale2<MODE>(sexp2<MODE>(v.x, v.y, M), rcp);
      const float2 b = scale2<MODE>(sexp2<MODE>(v.z, v.w, M), rcp);
      st_stream4(yr + 4 * q, make_float4(a.x, a.y, b.x, b.y));
    }
    fence_proxy_async_smem();  // generic smem reads before the TMA refill
    bar_arrive_n(3, kGresThreads);
  };

  unsigned k = 0;
  int64_t prow = 0;
  for (int64_t row = g; row < rows; row += G, ++k) {
    const int stage = static_cast<int>(k % unsigned(nstages));
    mbar_wait(&bars[stage], (k / unsigned(nstages)) & 1u);
    const float4* sb = reinterpret_cast<const float4*>(stage_buf + size_t(stage) * slice);

    float mt = kPadLogit;
    u64 z = f2pk(0.0f, 0.0f);
#pragma unroll 4
    for (int q = tid; q < nvec; q += kGresCompute) {
      const float4 v = sb[q];
      mt = fmaxf(mt, fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w)));
      z = nf_acc2(nf_acc2(z, v.x, v.y), v.z, v.w);
    }
    if (nf_bad(z)) atomicMin(bad_row, static_cast<unsigned long long>(row));
    const float mw = group_max<32>(mt);  // warp-local max: no CTA barrier
    u64 acc = f2pk(0.0f, 0.0f);
#pragma unroll 4
    for (int q = tid; q < nvec; q += kGresCompute) {
      const float4 v = sb[q];
      const float2 a = sexp2<MODE>(v.x, v.y, mw);
      const float2 b = sexp2<MODE>(v.z, v.w, mw);
      acc = f2add(f2add(acc, f2pk(a.x, a.y)), f2pk(b.x, b.y));
    }
    const float2 acc2 = f2up(acc);
    const double sw = group_sum<32>(static_cast<double>(acc2.x + acc2.y));
    if (lane == 0) {
      red_f[k & 1][warp] = mw;
      red_d[k & 1][warp] = sw;
    }
    bar_arrive_n(1 + 3 * (k & 1), kGresThreads);
    if (k > 0) output(k - 1, prow);
    prow = row;
  }
  if (k > 0) output(k - 1, prow);
}

}  // namespace sk
