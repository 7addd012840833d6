// sk_cluster.cuh -- K3c: a long row resident in one thread-block CLUSTER.
//
// A cluster of CS CTAs (one per SM; CS chosen by the launcher to cover the most
// SMs given the GPC layout) owns a row at a time; CTA
// `rank` holds columns [rank*L, (rank+1)*L) of it in shared memory.  Per row:
//
//   1. the slice lands in smem by cp.async.bulk (1-D TMA) on an mbarrier; the
//      ring has NS stages, so the slices of the next NS-1 rows are in flight
//      while this one is computed (HBM keeps streaming)
//   2. local max -> pushed into slot [rank] of every peer's smem with
//      st.async (DSMEM store that completes a transaction count on the peer's
//      mbarrier); each CTA waits on its own mbarrier for all CS slots, then
//      reduces them -> the row max M, identical in every CTA (fixed order).
//      No cluster barrier and no fence: nothing waits for the previous row's
//      global stores to drain.  Slots/barriers alternate by row parity (a
//      peer can be at most one exchange ahead).
//   3. e = exp(clip(x - M)) computed against the GLOBAL max -- the reference's
//      exact operation order, kernels.py:144-174 -- written back in place;
//      local f64 sum -> pushed the same way; S = sum of the CS slots (fixed order)
//   4. y = e * (1/(float)S) (flush as the reference, kernels.py:184-188),
//      streaming 128-bit stores; the stage is then re-armed with the slice of
//      the row NS steps ahead
//
// The row never leaves the chip between its passes, so HBM *and* L2 each see
// one read and one write per element (8 B/element) -- unlike two-pass schemes
// whose re-read costs L2 bandwidth -- and the row exchange is two cluster
// DSMEM pushes per row, not a global-memory handshake.
#pragma once
#include "sk_common.cuh"

namespace sk {

constexpr int kClusterThreads = 512;
constexpr int kClusterStages = 3;  // maximum ring depth (runtime nstages <= this)

__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned cluster_nrank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned cluster_id_x() {
  unsigned r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned ncluster_x() {
  unsigned r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\t"
               "barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t dsmem_addr(const void* local, unsigned rank) {
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(local)), "r"(rank));
  return ra;
}
__device__ __forceinline__ float ld_dsmem_f32(uint32_t a) {
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ double ld_dsmem_f64(uint32_t a) {
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
  return v;
}
// remote smem store that completes `bytes` of transaction on the peer's mbarrier
__device__ __forceinline__ void st_async_f32(uint32_t raddr, float v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f32 [%0], %1, [%2];"
               ::"r"(raddr), "f"(v), "r"(rbar) : "memory");
}
__device__ __forceinline__ void st_async_f64(uint32_t raddr, double v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];"
               ::"r"(raddr), "d"(v), "r"(rbar) : "memory");
}

// ONEX = true: one exchange per row -- each CTA reduces its slice to
// (m_l, s_l = sum exp(clip(x - m_l))) locally and pushes the pair once; every
// CTA merges M = max m_j, S = sum s_j exp(m_j - M) (fixed order) and the output
// pass recomputes exp(clip(x - M)) from the untouched slice (reference order).
// Trades one exp per element for one fewer cluster round trip per row.
template <int MODE, bool ONEX, int TPB = kClusterThreads>
__global__ void __launch_bounds__(TPB, 1)
    k3_cluster(const float* __restrict__ x, float* __restrict__ y, int64_t rows, int64_t cols,
               int64_t ldx, int64_t ldy, int slice, int nstages,
               unsigned long long* __restrict__ bad_row, float shift_scale, int diag) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* stage_buf = reinterpret_cast<float*>(smem_raw);
  __shared__ uint64_t bars[kClusterStages];
  __shared__ float red_f[TPB / 32];
  __shared__ double red_d[TPB / 32];
  __shared__ float slot_max[2][16];   // [row parity][sender rank], pushed by peers
  __shared__ double slot_sum[2][16];
  __shared__ float bc_m;
  __shared__ uint64_t xbar_max[2], xbar_sum[2];  // exchange barriers per row parity

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = TPB / 32;
  const unsigned rank = cluster_rank(), cs = cluster_nrank();
  const int64_t cid = cluster_id_x(), ncl = ncluster_x();
  const int64_t c0 = int64_t(rank) * slice;
  const int64_t rem = cols - c0;
  const int len = rem <= 0 ? 0 : static_cast<int>(rem < slice ? rem : slice);  // floats, % 4 == 0
  const int nvec = len >> 2;

  auto issue = [&](int64_t row, int stage) {
    mbar_arrive_expect_tx(&bars[stage], static_cast<uint32_t>(len) * 4u);
    if (len > 0)
      tma_load_1d(stage_buf + size_t(stage) * slice, x + row * ldx + c0,
                  static_cast<uint32_t>(len) * 4u, &bars[stage]);
  };

  if (tid == 0) {
    for (int s = 0; s < nstages; ++s) mbar_init(&bars[s], 1);
    for (int p = 0; p < 2; ++p) {
      mbar_init(&xbar_max[p], 1);
      mbar_init(&xbar_sum[p], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  cluster_sync_all();  // peers' exchange barriers are initialised before any push
  pdl_wait();
  pdl_launch_dependents();
  if (tid == 0)
    for (int s = 0; s < nstages; ++s) {
      const int64_t row = cid + int64_t(s) * ncl;
      if (row < rows) issue(row, s);
    }

  int k = 0;
  for (int64_t row = cid; row < rows; row += ncl, ++k) {
    const int stage = k % nstages;
    timing_chaos(diag, 8, k);  // diag bit 6: timing chaos (sk_common.cuh), results unchanged
    mbar_wait(&bars[stage], (k / nstages) & 1);
    float4* sb = reinterpret_cast<float4*>(stage_buf + size_t(stage) * slice);

    // ---- local max + finite check -> DSMEM exchange -> row max
    float mt = kPadLogit;
    u64 z = f2pk(0.0f, 0.0f);
#pragma unroll 4
    for (int q = tid; q < nvec; q += TPB) {
      const float4 v = sb[q];
      mt = fmaxf(mt, fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w)));
      z = nf_acc2(nf_acc2(z, v.x, v.y), v.z, v.w);
    }
    if (nf_bad(z)) atomicMin(bad_row, static_cast<unsigned long long>(row));
    mt = group_max<32>(mt);
    if (lane == 0) red_f[warp] = mt;
    __syncthreads();
    const int par = k & 1;
    const uint32_t xpar = (k >> 1) & 1;  // phase of this parity's barrier
    float M;
    if constexpr (ONEX) {
      if (tid == 0) {
        float m = red_f[0];
        for (int w = 1; w < NW; ++w) m = fmaxf(m, red_f[w]);
        bc_m = m * shift_scale;  // shift_scale = 0: fault hook
      }
      __syncthreads();
      M = bc_m;  // local max of this slice for now
    } else {
      if (tid == 0) mbar_arrive_expect_tx(&xbar_max[par], cs * 4u);
      timing_chaos(diag, 2, k);
      if (warp == 0) {
        float m = lane < NW ? red_f[lane] : kPadLogit;
        m = group_max<32>(m);
        if (lane < static_cast<int>(cs))  // push to rank `lane`
          st_async_f32(dsmem_addr(&slot_max[par][rank], lane), m,
                       dsmem_addr(&xbar_max[par], lane));
      }
      mbar_wait(&xbar_max[par], xpar);
      M = lane < static_cast<int>(cs) ? slot_max[par][lane] : kPadLogit;
      M = group_max<32>(M) * shift_scale;  // shift_scale = 0: fault hook
    }

    // ---- e = exp(clip(x - M)) (in place unless ONEX), local sum -> exchange
    u64 acc = f2pk(0.0f, 0.0f);
#pragma unroll 4
    for (int q = tid; q < nvec; q += TPB) {
      const float4 v = sb[q];
      const float2 a = sexp2<MODE>(v.x, v.y, M);
      const float2 b = sexp2<MODE>(v.z, v.w, M);
      if constexpr (!ONEX) sb[q] = make_float4(a.x, a.y, b.x, b.y);
      acc = f2add(f2add(acc, f2pk(a.x, a.y)), f2pk(b.x, b.y));
    }
    const float2 acc2 = f2up(acc);
    const double sd = group_sum<32>(static_cast<double>(acc2.x + acc2.y));
    if (lane == 0) red_d[warp] = sd;
    __syncthreads();
    if (tid == 0) {
      if (ONEX) mbar_arrive_expect_tx(&xbar_max[par], cs * 4u);
      mbar_arrive_expect_tx(&xbar_sum[par], cs * 8u);
    }
    timing_chaos(diag, 3, k);
    if (warp == 0) {
      double t = lane < NW ? red_d[lane] : 0.0;
      t = group_sum<32>(t);
      if (lane < static_cast<int>(cs)) {
        if (ONEX)
          st_async_f32(dsmem_addr(&slot_max[par][rank], lane), M,
                       dsmem_addr(&xbar_max[par], lane));
        st_async_f64(dsmem_addr(&slot_sum[par][rank], lane), t,
                     dsmem_addr(&xbar_sum[par], lane));
      }
    }
    timing_chaos(diag, 4, k);
    if (ONEX) mbar_wait(&xbar_max[par], xpar);
    mbar_wait(&xbar_sum[par], xpar);
    double S;
    if constexpr (ONEX) {
      const float mj = lane < static_cast<int>(cs) ? slot_max[par][lane] : kPadLogit;
      const float Mg = group_max<32>(mj);
      double sj = lane < static_cast<int>(cs) ? slot_sum[par][lane] : 0.0;
      if (lane < static_cast<int>(cs) && mj != Mg) sj *= static_cast<double>(expf(mj - Mg));
      S = group_sum<32>(sj);  // same butterfly in every CTA: identical S cluster-wide
      M = Mg;
    } else {
      S = lane < static_cast<int>(cs) ? slot_sum[par][lane] : 0.0;
      S = group_sum<32>(S);  // same butterfly in every CTA: identical S cluster-wide
    }
    const float rcp = recip_of_sum(S);

    // ---- y = e * r, streaming stores
    timing_chaos(diag, 6, k);
    float* yr = y + row * ldy + c0;
#pragma unroll 4
    for (int q = tid; q < nvec; q += TPB) {
      const float4 e = sb[q];
      float2 a, b;
      if constexpr (ONEX) {
        a = scale2<MODE>(sexp2<MODE>(e.x, e.y, M), rcp);
        b = scale2<MODE>(sexp2<MODE>(e.z, e.w, M), rcp);
      } else {
        a = scale2<MODE>(make_float2(e.x, e.y), rcp);
        b = scale2<MODE>(make_float2(e.z, e.w), rcp);
      }
      st_stream4(yr + 4 * q, make_float4(a.x, a.y, b.x, b.y));
    }
    timing_chaos(diag, 7, k);
    __syncthreads();  // stage fully consumed
    if (tid == 0) {
      const int64_t rn = row + int64_t(nstages) * ncl;
      if (rn < rows) {
        fence_proxy_async_smem();
        issue(rn, stage);
      }
    }
  }
  // no CTA leaves while a peer's push into it may still be in flight
  cluster_sync_all();
}

}  // namespace sk
