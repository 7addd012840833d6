// sk_gres.cuh -- K3g: a long row resident across P CTAs anywhere on the chip.
//
// K3c (sk_cluster.cuh) keeps a row in the shared memory of one thread-block
// cluster, but a cluster must fit inside one GPC, so the cluster sizes a 1 MB
// row needs (10-12 CTAs at 2 ring stages) pack only ~110 of the 148 SMs.  K3g
// drops the GPC constraint: a cooperative, persistent grid of one CTA per SM
// is cut into G = SMs / P groups of P CTAs; group g owns rows g, g+G, ... and
// CTA `rank` of the group holds columns [rank*W, (rank+1)*W) of the row in
// shared memory (TMA ring of NS stages, like K3c).
//
// One exchange per row, overlapped with the next rows.  Each compute warp
// reduces its share of the slice to a pair (m_w, s_w = sum exp(clip(x - m_w)))
// without any CTA barrier; the publisher warp merges the 16 pairs into the
// CTA pair (fixed order, s_w scaled by exp(m_w - m)) and stores it as one
// epoch-tagged 16-B slot of the group's slot array (one relaxed store: no
// counter, no release fence, no per-launch memset); a poller polls the P slots
// -- the poll returns the data itself -- and merges them in rank order, so M
// and S are bit-identical in every CTA of the row.  Meanwhile the compute
// warps run the local passes of the next rows; row k is written L rows later,
// y = exp(clip(x - M)) * (1/(float)S), the exp recomputed against the GLOBAL
// max from the untouched slice (reference order, kernels.py:144-188).
//
// Timing diagnostics (gres_diag, results wrong): bit 0 waits for the CTA's
// own slot only (no group exchange), bit 1 skips the math (the ring as a copy).
// Bit 6 (results unchanged): random delays at every hand-off, see gres_chaos.
//
// Roles: warps 0-15 compute; warp 16 publishes and issues the TMA refills; at
// lag 1 (ring depth 2-3) warp 16 also polls right after publishing, at lag >= 2
// (depth 4-5) warp 17 polls, so a slow poll never delays the next publication
// (which would chain the group into a per-row convoy).  No fence ever waits on
// the compute warps' output stores.  Named barriers:
//   bar1  compute -> publisher  "warp pairs of row k in smem"
//   bar2  poller -> compute     "(M, S) of row k in smem"
//   bar3  compute -> publisher  "row k's stage consumed (proxy-fenced): refill"
// With a ring of NS >= L+2 stages the output pass of row k runs after the
// local pass of row k+L: L+1 rows resident awaiting statistics, NS-L-1 rows
// loading ahead.  The group round trip hides behind L row steps; the loads in
// flight per SM (NS-L-1 slices) set the streaming rate for short slices.  HBM and L2 each see
// 8 B/element: the row never leaves the chip between its three smem passes.
#pragma once
#include "sk_common.cuh"

namespace sk {

constexpr int kGresCompute = 512;                   // 16 compute warps
constexpr int kGresThreads = kGresCompute + 32;     // compute + one hand-off warp per barrier
constexpr int kGresBlock = kGresCompute + 64;       // + publisher/TMA warp + poller warp
constexpr int kGresStages = 8;                      // maximum ring depth (lag <= 3, + loads ahead)
constexpr unsigned kGresSpinLimit = 1u << 24;       // ~10 s of polling: abort, never hang

__device__ __forceinline__ void bar_sync_n(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_arrive_n(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Slot stores/loads: .gpu scope on one device, .sys scope when the slot arrays
// are peer memory (column shards across GPUs).  Each 64-bit element is
// single-copy atomic; the pair is not, hence a tag in every word.
__device__ __forceinline__ void st_slot2(unsigned long long* p, unsigned long long a,
                                         unsigned long long b, bool sys) {
  if (sys)
    asm volatile("st.relaxed.sys.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
  else
    asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ void ld_slot2(const unsigned long long* p, unsigned long long& a,
                                         unsigned long long& b, bool sys) {
  if (sys)
    asm volatile("ld.relaxed.sys.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
  else
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}

constexpr int kGresMaxSlots = 160;  // pairs merged per row (world x P), 5 per poller lane
constexpr int kGresMaxWorld = 8;

// Where a group's pairs go.  dst[r] is rank r's slot array -- a peer pointer
// for a real column shard on another GPU, or one of `world` arrays on this GPU
// when the launch emulates all ranks (one cooperative kernel over every
// rank's data).  This launch covers ranks rank0 .. rank0+nvr-1; virtual rank
// v reads x + v*shard_stride.  ctl: [0] launch epoch, [1] finished-CTA count,
// [2] abort flag -- in the LOCAL workspace, advanced by the launch's last CTA.
struct GresComm {
  unsigned long long* dst[kGresMaxWorld];
  unsigned* ctl;
  int64_t shard_stride;
  int world, rank0, nvr, sys;
  unsigned spin_limit;  // polls before a missing peer aborts the exchange
  // Device-side epoch reset (blocks no other process writes: the library's
  // per-stream block, a world-1 or emulated column shard): every
  // reset_period launches the launch's last CTA zeroes reset_words 64-bit
  // words of slots in each of the launch's blocks and restarts the epoch at
  // 0, so the 23-bit slot epoch never wraps -- CUDA-graph replays included.
  // 0: the host resets the block (cross-GPU column shards, sk_xchg_reset).
  unsigned long long reset_words;
  unsigned reset_period;
};

// comm.dst[i] without dynamic indexing of the parameter array (which would
// copy the whole descriptor to local memory)
__device__ __forceinline__ unsigned long long* gres_dst(const GresComm& c, int i) {
  unsigned long long* d = c.dst[0];
#pragma unroll
  for (int r = 1; r < kGresMaxWorld; ++r)
    if (i == r) d = c.dst[r];
  return d;
}

// A CTA's row pair as one 16-B slot of two independently tagged 64-bit words:
// tag << 32 | bits(m) and tag << 32 | bits(s) -- the CTA's partial sum rounded
// to fp32 (2^-24 relative; the row sum S itself is still accumulated in f64
// over the pairs).  tag = 0x80000000 | (epoch mod 2^23) << 8 | (k mod 256):
// never 0 (zeroed memory is "not yet"); the row bits only have to tell k from
// the slot set's previous row in this launch, k - (2L+2) with 2L+2 <= 8; the
// 23 epoch bits tell this launch from every earlier one, because the host
// zeroes an exchange block (epoch back to 0, every slot "not yet") at least
// every kGresEpochReset < 2^23 launches -- so the epoch never wraps and a slot
// left over from an older launch can never carry a matching tag.  The data IS
// the flag -- no counter, no fence, no per-launch memset for a peer to race.
// One store, one load.
constexpr unsigned kGresEpochBits = 23;
constexpr unsigned long long kGresEpochReset = 1ull << 22;  // default reset period (launches)
static_assert(kGresEpochReset < (1ull << kGresEpochBits), "the epoch must never wrap");
__device__ __forceinline__ unsigned gres_tag(unsigned epoch, unsigned k) {
  return 0x80000000u | ((epoch & ((1u << kGresEpochBits) - 1u)) << 8) | (k & 0xFFu);
}
static_assert(2 * 3 + 2 <= 256, "row tag bits must cover the slot-set rotation");
__device__ __forceinline__ void gres_publish(unsigned long long* slot, float m, double s,
                                             unsigned tag, bool sys) {
  const unsigned long long t = static_cast<unsigned long long>(tag) << 32;
  st_slot2(slot, t | __float_as_uint(m), t | __float_as_uint(static_cast<float>(s)), sys);
}

// Global slot sets per group.  A publisher can run ahead of a REMOTE poller:
// CTA A publishing row k needs its own row k-1-L merged (all of the group
// published k-1-L), so every CTA B has finished its local pass of k-1-L and
// hence its output -- and its poller's read -- of row k-2-2L.  Rows
// k-1-2L .. k may be live: 2L+2 sets.
__host__ __device__ constexpr int gres_slot_sets(int L) { return 2 * L + 2; }
constexpr unsigned long long kExchangeAborted = 0xFFFFFFFFFFFFFFFEull;  // in *bad_row

// Named barrier ids for lag L (stages - 2, 1..3): a hand-off can have at most
// L+1 (bars 1 and 2) or L (bar 3) phases outstanding, so each rotates over
// that many ids.  Id 0 is __syncthreads.
template <int L>
__device__ __forceinline__ int gres_bar1(unsigned k) { return 1 + int(k % unsigned(L + 1)); }
template <int L>
__device__ __forceinline__ int gres_bar2(unsigned k) { return 2 + L + int(k % unsigned(L + 1)); }
template <int L>
__device__ __forceinline__ int gres_bar3(unsigned k) { return 3 + 2 * L + int(k % unsigned(L)); }

// UNAL: rows of any length / alignment.  Each row's slices are cut at x's
// 16-B boundaries, which shift per row: with h = floats before the row's first
// boundary, CTA 0 owns columns [0, h + W), CTA r > 0 owns [h + rW, h + (r+1)W)
// (the last one up to C).  A CTA stages the aligned middle of its range by TMA;
// the <= 3 head floats (CTA 0) and <= 3 tail floats (last CTA) are read from
// global memory.  The compute keeps 128-bit smem accesses, and stores stay
// 128-bit when y has x's 16-B phase (equal pitches and bases' phases, the usual
// case); otherwise 32-bit.  Bits depend on the row's phase (deterministic for a
// given buffer).
struct SliceGeom {
  int64_t a;  // first column of the staged middle (16-B aligned in x)
  int hd;     // head floats before a (CTA 0 only)
  int nmid;   // staged floats (% 4 == 0)
  int tl;     // tail floats after the middle (last CTA only)
};
__device__ __forceinline__ SliceGeom unal_geom(const float* xrow, int64_t cols, int prank, int P,
                                               int slice) {
  const int h = static_cast<int>(((16u - (reinterpret_cast<uintptr_t>(xrow) & 15u)) & 15u) >> 2);
  int64_t c_start = prank == 0 ? 0 : int64_t(h) + int64_t(prank) * slice;
  int64_t c_end = prank == P - 1 ? cols : int64_t(h) + int64_t(prank + 1) * slice;
  if (c_end > cols) c_end = cols;
  if (c_start > c_end) c_start = c_end;
  SliceGeom sg;
  sg.hd = prank == 0 ? static_cast<int>(c_end < h ? c_end : h) : 0;
  sg.a = c_start + sg.hd;
  sg.nmid = static_cast<int>(((c_end - sg.a) >> 2) << 2);
  sg.tl = static_cast<int>(c_end - sg.a - sg.nmid);
  return sg;
}

// L: rows between a row's local pass and its output pass (ring depth L + 2).
// SPLIT: a separate poller warp (block 576) vs the publisher warp polling
// after each publication (block 544).
template <int MODE, int L, bool SPLIT, bool UNAL = false>
__global__ void __launch_bounds__(kGresBlock, 1)
    k3_gres(const float* __restrict__ x, float* __restrict__ y, int64_t rows, int64_t cols,
            int64_t ldx, int64_t ldy, int P, int slice, int nstages, const GresComm comm,
            unsigned long long* __restrict__ bad_row, float shift_scale, int poll_ns, int diag) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* stage_buf = reinterpret_cast<float*>(smem_raw);
  constexpr int NW = kGresCompute / 32;
  constexpr int NB = L + 1;              // smem broadcast slots
  constexpr int NS = gres_slot_sets(L);  // global slot sets
  __shared__ uint64_t bars[kGresStages];
  __shared__ float red_f[NB][NW];   // [row % (L+1)][warp]: warp-local max
  __shared__ double red_d[NB][NW];  //                      warp-local sum vs that max
  __shared__ float bc_m[NB];        // [row % (L+1)] merged row max / sum
  __shared__ double bc_s[NB];
  __shared__ unsigned epoch_s;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int per_rank = static_cast<int>(gridDim.x) / comm.nvr;  // CTAs of one rank's shard
  const int G = per_rank / P;
  const int v = static_cast<int>(blockIdx.x) / per_rank;        // virtual rank in this launch
  const int cta = static_cast<int>(blockIdx.x) % per_rank;
  const int g = cta / P, prank = cta % P;
  const int myr = comm.rank0 + v;                                // global rank of this shard
  const int WP = comm.world * P;                                 // pairs per row
  const int gi = myr * P + prank;                                // this CTA's slot index
  const bool sys = comm.sys != 0;
  x += v * comm.shard_stride;
  y += v * comm.shard_stride;
  const int64_t c0 = int64_t(prank) * slice;
  const int64_t rem = cols - c0;
  const int len = rem <= 0 ? 0 : static_cast<int>(rem < slice ? rem : slice);
  const int nvec = len >> 2;  // aligned rows: % 4 == 0
  if (tid == 0) {
    for (int s = 0; s < nstages; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  pdl_wait();  // (PDL only) the previous launch's epoch advance is visible after this
  if (tid == 0) epoch_s = ld_relaxed_u32(comm.ctl);
  __syncthreads();
  pdl_launch_dependents();
  const unsigned epoch = epoch_s;

  // slot array layout: [epoch parity][group][NS sets][WP] x 16 B.  The epoch
  // parity matters across GPUs: a rank can start its next launch (and publish
  // into its peers' arrays) while a peer still polls this launch's last rows;
  // it cannot get two launches ahead (its next launch waits for that peer).
  auto slot_set = [&](unsigned long long* base, unsigned k) {  // row k of group g
    return base + ((size_t(epoch & 1u) * G + g) * NS + k % unsigned(NS)) * size_t(WP) * 2;
  };


  // Row k's pairs in this rank's slot array: lane l loads slots l, l+32, ...;
  // true (warp-uniform) once every word carries row k's tag.  diag & 1 (timing
  // only): this CTA's own slot instead of the group's.
  constexpr int NI = kGresMaxSlots / 32;
  const int pp = (diag & 1) ? 1 : WP;
  unsigned long long* const mine = gres_dst(comm, myr);
  auto poll_load = [&](unsigned k, unsigned long long (&wa)[NI], unsigned long long (&wb)[NI]) {
    const unsigned long long* sl = slot_set(mine, k);
#pragma unroll
    for (int i = 0; i < NI; ++i)
      if (lane + 32 * i < pp) ld_slot2(sl + 2 * ((diag & 1) ? gi : lane + 32 * i), wa[i], wb[i], sys);
  };
  auto poll_ok = [&](unsigned k, const unsigned long long (&wa)[NI], const unsigned long long (&wb)[NI]) {
    const unsigned tag = gres_tag(epoch, k);
    bool ok = true;
#pragma unroll
    for (int i = 0; i < NI; ++i)
      if (lane + 32 * i < pp)
        ok = ok && static_cast<unsigned>(wa[i] >> 32) == tag && static_cast<unsigned>(wb[i] >> 32) == tag;
    return __all_sync(0xffffffffu, ok);
  };
  // a stuck peer raises abort: never hang the GPU (checked every 4096 polls)
  auto poll_abort = [&](unsigned& spins) {
    if ((++spins & 0xFFFu) == 0 && (ld_relaxed_u32(comm.ctl + 2) || spins >= comm.spin_limit)) {
      if (lane == 0) atomicExch(comm.ctl + 2, 1u);
      return true;
    }
    return false;
  };
  // merge the pairs in slot order (identical (M, S) on every CTA of the row,
  // on every rank) and broadcast through smem slot k % NB
  auto merge_bcast = [&](unsigned k, const unsigned long long (&wa)[NI], const unsigned long long (&wb)[NI]) {
    float Mg = kPadLogit;
#pragma unroll
    for (int i = 0; i < NI; ++i)
      if (lane + 32 * i < pp) Mg = fmaxf(Mg, __uint_as_float(static_cast<unsigned>(wa[i])));
    Mg = group_max<32>(Mg);
    double S = 0.0;
#pragma unroll
    for (int i = 0; i < NI; ++i)
      if (lane + 32 * i < pp) {
        const float mj = __uint_as_float(static_cast<unsigned>(wa[i]));
        double sj = static_cast<double>(__uint_as_float(static_cast<unsigned>(wb[i])));
        if (mj != Mg) sj *= static_cast<double>(expf(mj - Mg));
        S += sj;
      }
    S = group_sum<32>(S);
    if (lane == 0) {
      const int b = static_cast<int>(k % unsigned(NB));
      bc_m[b] = Mg * shift_scale;  // shift_scale = 0: fault hook
      bc_s[b] = S;
    }
  };
  // wait for row k's pairs and merge them (the poller warp, or the publisher at lag 1)
  auto poll_merge = [&](unsigned k) {
    unsigned long long wa[NI], wb[NI];
    unsigned spins = 0;
    while (true) {
      poll_load(k, wa, wb);
      if (poll_ok(k, wa, wb)) break;
      // back off: a spinning poller steals issue slots from its sub-partition's
      // compute warps, and its loads queue behind the publishers' stores
      if (SPLIT && poll_ns > 0) __nanosleep(static_cast<unsigned>(poll_ns));
      if (poll_abort(spins)) break;
    }
    merge_bcast(k, wa, wb);
  };

  if (g >= G) {
    // idle CTA (the grid is a whole multiple of neither P nor ranks): tail only
  } else if (warp == NW) {
    // ------------------------------------------------ publisher + TMA warp
    auto issue = [&](int64_t row, int stage) {
      const float* src = x + row * ldx + c0;
      int n = len;
      if constexpr (UNAL) {
        const float* xrow = x + row * ldx;
        const SliceGeom sg = unal_geom(xrow, cols, prank, P, slice);
        src = xrow + sg.a;
        n = sg.nmid;
      }
      mbar_arrive_expect_tx(&bars[stage], static_cast<uint32_t>(n) * 4u);
      if (n > 0)
        tma_load_1d(stage_buf + size_t(stage) * slice, src, static_cast<uint32_t>(n) * 4u,
                    &bars[stage]);
    };
    if (lane == 0)
      for (int s = 0; s < nstages; ++s) {
        const int64_t row = g + int64_t(s) * G;
        if (row < rows) issue(row, s);
      }
    unsigned k = 0;
    for (int64_t row = g; row < rows; row += G, ++k) {
      const int b = static_cast<int>(k % unsigned(NB));
      // CTA pair (m, s) of row k from the 16 warp pairs, fixed order
      timing_chaos(diag, 1, k);
      bar_sync_n(gres_bar1<L>(k), kGresThreads);
      const float mw = lane < NW ? red_f[b][lane] : kPadLogit;
      const float mc = group_max<32>(mw);
      double sw = lane < NW ? red_d[b][lane] : 0.0;
      if (lane < NW && mw != mc) sw *= static_cast<double>(expf(mw - mc));
      const double sc = group_sum<32>(sw);
      // lane r stores the pair into rank r's slot array (a peer's, over NVLink)
      timing_chaos(diag, 2, k);
      if (lane < comm.world)
        gres_publish(slot_set(gres_dst(comm, lane), k) + 2 * gi, mc, sc, gres_tag(epoch, k), sys);
      // refill the stage row k-L released
      if (k >= unsigned(L)) {
        const unsigned j = k - unsigned(L);
        bar_sync_n(gres_bar3<L>(j), kGresThreads);
        timing_chaos(diag, 3, k);
        const int64_t rn = row - int64_t(L) * G + int64_t(nstages) * G;
        if (lane == 0 && rn < rows) issue(rn, static_cast<int>(j % unsigned(nstages)));
      }
      if (!SPLIT) {
        timing_chaos(diag, 4, k);
        poll_merge(k);
        timing_chaos(diag, 5, k);
        bar_arrive_n(gres_bar2<L>(k), kGresThreads);
      }
    }
    for (unsigned j = k >= unsigned(L) ? k - unsigned(L) : 0u; j < k; ++j)
      bar_sync_n(gres_bar3<L>(j), kGresThreads);  // the last L output passes
  } else if (warp == NW + 1) {
    // ------------------------------------------------ poller warp
    if (SPLIT) {
      unsigned k = 0;
      for (int64_t row = g; row < rows; row += G, ++k) {
        timing_chaos(diag, 4, k);
        poll_merge(k);
        timing_chaos(diag, 5, k);
        bar_arrive_n(gres_bar2<L>(k), kGresThreads);
      }
    }
  } else {
    // ------------------------------------------------ compute warps
    // row k's output pass runs after row k+L's local pass, so the group
    // exchange of row k overlaps L full rows of streaming work.
    auto output = [&](unsigned j) {
      timing_chaos(diag, 6, j);
      bar_sync_n(gres_bar2<L>(j), kGresThreads);
      const int b = static_cast<int>(j % unsigned(NB));
      const float M = bc_m[b];
      const float rcp = recip_of_sum(bc_s[b]);
      const float* sm = stage_buf + size_t(j % unsigned(nstages)) * slice;
      const float4* sb = reinterpret_cast<const float4*>(sm);
      const int64_t orow = g + int64_t(j) * G;
      float* yr = y + orow * ldy + c0;
      if constexpr (UNAL) {
        const float* xrow = x + orow * ldx;
        float* yrow = y + orow * ldy;
        const SliceGeom sg = unal_geom(xrow, cols, prank, P, slice);
        float* ym = yrow + sg.a;
        const bool yv = (reinterpret_cast<uintptr_t>(ym) & 15u) == 0;
        const int nq = sg.nmid >> 2;
#pragma unroll 4
        for (int q = tid; q < nq; q += kGresCompute) {
          const float4 v4 = sb[q];
          const float2 a = scale2<MODE>(sexp2<MODE>(v4.x, v4.y, M), rcp);
          const float2 c = scale2<MODE>(sexp2<MODE>(v4.z, v4.w, M), rcp);
          if (yv) {
            st_stream4(ym + 4 * q, make_float4(a.x, a.y, c.x, c.y));
          } else {
            st_stream1(ym + 4 * q, a.x);
            st_stream1(ym + 4 * q + 1, a.y);
            st_stream1(ym + 4 * q + 2, c.x);
            st_stream1(ym + 4 * q + 3, c.y);
          }
        }
        // head (CTA 0) and tail (last CTA): <= 3 floats each, from global
        if (tid < sg.hd) {
          const int64_t col = sg.a - sg.hd + tid;
          st_stream1(yrow + col, scale1<MODE>(sexp1<MODE>(__ldg(xrow + col), M), rcp));
        } else if (tid >= 32 && tid < 32 + sg.tl) {
          const int64_t col = sg.a + sg.nmid + (tid - 32);
          st_stream1(yrow + col, scale1<MODE>(sexp1<MODE>(__ldg(xrow + col), M), rcp));
        }
      } else if (diag & 2) {  // timing only: the ring as a plain copy (no math)
        for (int q = tid; q < nvec; q += kGresCompute) st_stream4(yr + 4 * q, sb[q]);
      } else {
#pragma unroll 4
        for (int q = tid; q < nvec; q += kGresCompute) {
          const float4 v4 = sb[q];
          const float2 a = scale2<MODE>(sexp2<MODE>(v4.x, v4.y, M), rcp);
          const float2 c = scale2<MODE>(sexp2<MODE>(v4.z, v4.w, M), rcp);
          st_stream4(yr + 4 * q, make_float4(a.x, a.y, c.x, c.y));
        }
      }
      fence_proxy_async_smem();  // generic smem reads before the TMA refill
      timing_chaos(diag, 7, j);
      bar_arrive_n(gres_bar3<L>(j), kGresThreads);
    };

    unsigned k = 0;
    for (int64_t row = g; row < rows; row += G, ++k) {
      const int stage = static_cast<int>(k % unsigned(nstages));
      timing_chaos(diag, 8, k);
      mbar_wait(&bars[stage], (k / unsigned(nstages)) & 1u);
      const float4* sb = reinterpret_cast<const float4*>(stage_buf + size_t(stage) * slice);
      int nq = nvec;  // staged float4 groups
      SliceGeom sg{0, 0, 0, 0};
      const float* xrow = x + row * ldx;
      if constexpr (UNAL) {
        sg = unal_geom(xrow, cols, prank, P, slice);
        nq = sg.nmid >> 2;
      }
      // head / tail floats (UNAL): threads 0..2 (head) and 32..34 (tail)
      const bool edge = UNAL && ((tid < sg.hd) || (tid >= 32 && tid < 32 + sg.tl));
      const float xe = edge ? __ldg(xrow + (tid < 32 ? sg.a - sg.hd + tid : sg.a + sg.nmid + (tid - 32)))
                            : kPadLogit;

      float mt = xe;
      u64 z = f2pk(0.0f, 0.0f);
      if (edge) z = nf_acc2(z, xe, 0.0f);
      if (!UNAL && (diag & 2)) nq = 0;  // timing only: skip the local pass
#pragma unroll 4
      for (int q = tid; q < nq; q += kGresCompute) {
        const float4 v4 = sb[q];
        mt = fmaxf(mt, fmaxf(fmaxf(v4.x, v4.y), fmaxf(v4.z, v4.w)));
        z = nf_acc2(nf_acc2(z, v4.x, v4.y), v4.z, v4.w);
      }
      if (nf_bad(z)) atomicMin(bad_row, static_cast<unsigned long long>(row));
      const float mw = group_max<32>(mt);  // warp-local max: no CTA barrier
      u64 acc = f2pk(edge ? sexp1<MODE>(xe, mw) : 0.0f, 0.0f);
#pragma unroll 4
      for (int q = tid; q < nq; q += kGresCompute) {
        const float4 v4 = sb[q];
        const float2 a = sexp2<MODE>(v4.x, v4.y, mw);
        const float2 c = sexp2<MODE>(v4.z, v4.w, mw);
        acc = f2add(f2add(acc, f2pk(a.x, a.y)), f2pk(c.x, c.y));
      }
      const float2 acc2 = f2up(acc);
      const double sw = group_sum<32>(static_cast<double>(acc2.x + acc2.y));
      if (lane == 0) {
        const int b = static_cast<int>(k % unsigned(NB));
        red_f[b][warp] = mw;
        red_d[b][warp] = sw;
      }
      timing_chaos(diag, 9, k);
      bar_arrive_n(gres_bar1<L>(k), kGresThreads);
      if (k >= unsigned(L)) output(k - unsigned(L));
    }
    for (unsigned j = k >= unsigned(L) ? k - unsigned(L) : 0u; j < k; ++j) output(j);
  }

  // ------------------------------------------------------------------ tail
  // The launch's last CTA advances the epoch (every CTA has read it by now)
  // and turns an exchange timeout into a status the host can see.
  __syncthreads();
  __shared__ int last_s;
  if (tid == 0) {
    __threadfence();
    last_s = atomicAdd(comm.ctl + 1, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last_s) {
    // every other CTA of the launch is done with the slots; the next launch
    // reads them only after griddepcontrol.wait, i.e. after this grid completes
    const bool wipe = comm.reset_words != 0 && comm.reset_period != 0 &&
                      (epoch + 1u) % comm.reset_period == 0u;
    if (wipe) {
      const int nb = comm.nvr == comm.world ? comm.world : 1;
      for (int r = 0; r < nb; ++r) {
        unsigned long long* d = comm.nvr == comm.world ? gres_dst(comm, r) : gres_dst(comm, comm.rank0);
        for (unsigned long long i = tid; i < comm.reset_words; i += blockDim.x) d[i] = 0ull;
      }
      __threadfence();
      __syncthreads();
    }
    if (tid == 0) {
      if (atomicExch(comm.ctl + 2, 0u)) atomicMin(bad_row, kExchangeAborted);
      comm.ctl[1] = 0;
      comm.ctl[0] = wipe ? 0u : epoch + 1u;
    }
  }
}

}  // namespace sk
