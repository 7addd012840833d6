// sk_api.cu -- C ABI (include/softmax_b200.h) for device buffers: launch
// planning, workspaces, tuning, the row-statistics building blocks.  The
// host-buffer pipeline lives in sk_host.cu, the fused column shard in
// sk_colshard.cu (shared internals: sk_internal.h).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <atomic>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/softmax_b200.h"
#include "sk_rows.cuh"
#include "sk_seg.cuh"
#include "sk_split.cuh"
#include "sk_cluster.cuh"
#include "sk_gres.cuh"
#include "sk_rows_mw.cuh"
#include "sk_internal.h"

namespace sk {
namespace detail {

thread_local std::string g_last_error;

int cuda_fail(cudaError_t e, const char* what) {
  g_last_error = std::string(what) + ": " + cudaGetErrorString(e);
  (void)cudaGetLastError();
  if (e == cudaErrorMemoryAllocation) return SK_ERR_RESOURCE;
  return SK_ERR_CUDA;
}

int arg_fail(const std::string& msg) {
  g_last_error = msg;
  return SK_ERR_ARGUMENT;
}

// ---------------------------------------------------------------- device info
DevInfo dev_info(int dev) {
  static std::mutex mu;
  static std::map<int, DevInfo> cache;
  std::lock_guard<std::mutex> g(mu);
  auto it = cache.find(dev);
  if (it != cache.end()) return it->second;
  DevInfo d;
  cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev);
  int coop = 0;
  cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
  d.coop = coop != 0;
  cache[dev] = d;
  return d;
}

// ------------------------------------------------------------ tuning overrides
std::atomic<int> g_force_path{-1};  // -1 auto, 0 k1, 1 seg, 2 split, 3 k1m
// fault hook mirroring kernels._SKIP_MAX_SHIFT (kernels.py:103-105): when set the
// kernels shift by 0 instead of the row max, so large logits overflow exp.
std::atomic<int> g_skip_max_shift{0};
float shift_scale() { return g_skip_max_shift.load() ? 0.0f : 1.0f; }

// Raise (never lower) a kernel's dynamic shared-memory limit.
void ensure_smem_attr(const void* fn, size_t smem) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> set;
  // any dynamic request: static + dynamic must fit the opt-in limit (the
  // default 48 KB cap counts the static arrays too -- K2 at 6144 columns asks
  // for exactly 48 KB of dynamic smem and failed to launch without this)
  if (smem == 0) return;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> g(mu);
  size_t& cur = set[{fn, dev}];
  if (smem > cur) {
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    cur = smem;
  }
}
// Tuning knobs (sk_set_tuning); defaults are the measured-best settings.
// K1
std::atomic<int> g_k1_lpr{0}, g_k1_nv{0}, g_k1_u{0};  // force a K1 shape (0 = table default)
std::atomic<int> g_k1_pf{-1};      // -1: table default, 0/1 force register prefetch
std::atomic<int> g_grid_mult{0};   // K1 grid = SMs x occupancy x mult (0 = one batch per warp)
std::atomic<int> g_vec8{0};        // 256-bit K1 path (measured no faster: off by default)
std::atomic<int> g_vec2_max{128};  // widest even row the 64-bit K1 path takes (0: off)
std::atomic<int> g_pdl{1};         // programmatic dependent launch on every kernel
std::atomic<int> g_coop_pdl{1};    // ... also on cooperative launches (K3g; measured -0.6..1.3 us/launch)
// long rows: 3 = K3g, else K3c (default); 5 = K3c only
std::atomic<int> g_k3_impl{3};
// K3c (cluster-resident rows)
std::atomic<int> g_cluster_k3{1};    // allow the cluster kernel (fallback to K3g)
std::atomic<int> g_cluster_size{0};  // force a K3c cluster size (0 = auto)
// K3g (grid-resident rows)
std::atomic<int> g_gres{1};        // 0 off, 1 auto, 2 force
std::atomic<int> g_gres_p{0};      // force CTAs per row (0 = planner)
std::atomic<int> g_gres_st{0};     // force ring depth (0 = planner)
std::atomic<int> g_gres_lag{0};    // force the lag (rows between local and output pass; 0 = planner)
std::atomic<int> g_gres_split{-1};  // separate poller warp: -1 auto (lag >= 2), 0 off, 1 on
std::atomic<int> g_gres_sleep{128};  // poller back-off between polls (ns)
std::atomic<int> g_latency_steps{3};  // K3g row steps per group up to which the latency path is taken
std::atomic<int> g_gres_diag{0};     // timing diagnostics (1: wait only for the own slot -- wrong results)
std::atomic<unsigned> g_gres_spins{kGresSpinLimit};  // exchange timeout (polls), tests shorten it
std::atomic<int> g_colshard_sys{0};  // 1: the emulated column shard uses the cross-GPU (.sys) slot accesses
bool gres_split(int lag) {
  const int v = g_gres_split.load();
  return v < 0 ? lag >= 2 : v != 0;
}

// ------------------------------------------------------------------ K1 table
using K1Fn = void (*)(const float*, float*, int64_t, int, int64_t, int64_t,
                      unsigned long long*, float);
struct K1Entry {
  int vec, lpr, nv, u, pf;
  K1Fn fn[3];
};
#define SK_K1(VEC, LPR, NV, U, PF)                                                         \
  K1Entry {                                                                                \
    VEC, LPR, NV, U, PF, {                                                                 \
      &k1_rows<kClipAccurate, VEC, LPR, NV, U, PF>, &k1_rows<kAccurate, VEC, LPR, NV, U, PF>, \
          &k1_rows<kApprox, VEC, LPR, NV, U, PF>                                           \
    }                                                                                      \
  }
const K1Entry kK1Table[] = {
    // 128-bit path (cols % 4 == 0, 16-B aligned rows)
    SK_K1(4, 4, 1, 4, 0), SK_K1(4, 8, 1, 4, 0), SK_K1(4, 16, 1, 4, 0), SK_K1(4, 8, 2, 2, 0),
    SK_K1(4, 8, 4, 1, 0), SK_K1(4, 8, 4, 2, 0), SK_K1(4, 16, 2, 2, 0), SK_K1(4, 16, 2, 1, 0),
    SK_K1(4, 16, 4, 1, 0), SK_K1(4, 16, 4, 2, 0), SK_K1(4, 32, 1, 4, 0), SK_K1(4, 32, 2, 2, 0),
    SK_K1(4, 32, 4, 1, 0), SK_K1(4, 32, 8, 1, 0), SK_K1(4, 32, 1, 2, 0), SK_K1(4, 32, 2, 1, 0),
    SK_K1(4, 8, 4, 1, 1), SK_K1(4, 16, 2, 1, 1), SK_K1(4, 16, 4, 1, 1), SK_K1(4, 32, 2, 1, 1),
    SK_K1(4, 32, 4, 1, 1), SK_K1(4, 32, 8, 1, 1), SK_K1(4, 16, 1, 4, 1), SK_K1(4, 8, 1, 4, 1),
    SK_K1(4, 4, 1, 8, 0), SK_K1(4, 8, 1, 8, 0), SK_K1(4, 16, 1, 8, 0), SK_K1(4, 16, 1, 8, 1),
    SK_K1(4, 4, 2, 4, 0), SK_K1(4, 4, 2, 2, 0), SK_K1(4, 4, 4, 2, 0), SK_K1(4, 4, 4, 1, 0),
    SK_K1(4, 4, 8, 1, 0), SK_K1(4, 4, 4, 1, 1), SK_K1(4, 4, 8, 1, 1), SK_K1(4, 8, 8, 1, 0),
    SK_K1(4, 8, 8, 2, 0), SK_K1(4, 4, 16, 1, 0),
    // exact-fit vectors per lane (kK1Fit): no padded slots for C just above 2^k
    SK_K1(4, 4, 3, 1, 0), SK_K1(4, 8, 3, 1, 0), SK_K1(4, 16, 3, 1, 0), SK_K1(4, 16, 3, 2, 0),
    SK_K1(4, 32, 3, 1, 0), SK_K1(4, 32, 5, 1, 0), SK_K1(4, 32, 6, 1, 0), SK_K1(4, 32, 7, 1, 0),
    SK_K1(4, 32, 12, 1, 0), SK_K1(4, 32, 20, 1, 0), SK_K1(4, 32, 9, 1, 0), SK_K1(4, 32, 10, 1, 0),
    SK_K1(4, 32, 11, 1, 0), SK_K1(4, 32, 13, 1, 0), SK_K1(4, 32, 14, 1, 0), SK_K1(4, 32, 15, 1, 0),
    SK_K1(4, 32, 17, 1, 0), SK_K1(4, 32, 18, 1, 0), SK_K1(4, 32, 19, 1, 0), SK_K1(4, 32, 21, 1, 0),
    SK_K1(4, 32, 22, 1, 0), SK_K1(4, 32, 23, 1, 0),
    SK_K1(2, 8, 3, 2, 0), SK_K1(2, 8, 3, 1, 1), SK_K1(2, 16, 3, 2, 0), SK_K1(2, 16, 3, 1, 1),
    SK_K1(1, 2, 3, 4, 0), SK_K1(1, 2, 3, 1, 1), SK_K1(1, 4, 3, 4, 0), SK_K1(1, 4, 3, 1, 1),
    SK_K1(1, 8, 3, 4, 0), SK_K1(1, 8, 3, 2, 0), SK_K1(1, 8, 5, 2, 0), SK_K1(1, 8, 5, 1, 1),
    SK_K1(1, 8, 6, 2, 0), SK_K1(1, 8, 6, 1, 1), SK_K1(1, 8, 7, 2, 0), SK_K1(1, 8, 7, 1, 1),
    SK_K1(1, 16, 5, 2, 0), SK_K1(1, 16, 5, 1, 1), SK_K1(1, 16, 6, 2, 0), SK_K1(1, 16, 6, 1, 1),
    SK_K1(1, 16, 7, 2, 0), SK_K1(1, 16, 7, 1, 1), SK_K1(1, 32, 5, 1, 0), SK_K1(1, 32, 6, 1, 0),
    SK_K1(1, 32, 7, 1, 0), SK_K1(1, 32, 9, 1, 0), SK_K1(1, 32, 10, 1, 0), SK_K1(1, 32, 11, 1, 0),
    SK_K1(1, 32, 12, 1, 0), SK_K1(1, 32, 13, 1, 0), SK_K1(1, 32, 14, 1, 0), SK_K1(1, 32, 15, 1, 0),
    SK_K1(1, 32, 17, 1, 0), SK_K1(1, 32, 18, 1, 0), SK_K1(1, 32, 19, 1, 0), SK_K1(1, 32, 20, 1, 0),
    SK_K1(1, 32, 21, 1, 0), SK_K1(1, 32, 22, 1, 0), SK_K1(1, 32, 23, 1, 0), SK_K1(1, 32, 24, 1, 0),
    SK_K1(1, 32, 36, 1, 0), SK_K1(1, 32, 40, 1, 0),

    // medium rows: a warp holds up to 2048 / 3072 floats in registers
    SK_K1(4, 32, 16, 1, 0), SK_K1(4, 32, 24, 1, 0),
    // 256-bit path (cols % 8 == 0, 32-B aligned rows)
    SK_K1(8, 8, 1, 4, 0), SK_K1(8, 16, 1, 2, 0), SK_K1(8, 16, 1, 4, 0), SK_K1(8, 8, 2, 1, 0),
    SK_K1(8, 8, 2, 2, 0), SK_K1(8, 16, 2, 1, 0), SK_K1(8, 32, 1, 1, 0), SK_K1(8, 32, 1, 2, 0),
    SK_K1(8, 32, 2, 1, 0), SK_K1(8, 32, 4, 1, 0), SK_K1(8, 16, 1, 1, 0),
    // 64-bit path (even cols, 8-B aligned rows)
    SK_K1(2, 8, 4, 1, 0), SK_K1(2, 8, 4, 2, 0), SK_K1(2, 8, 4, 1, 1), SK_K1(2, 16, 2, 1, 0),
    SK_K1(2, 16, 2, 2, 0), SK_K1(2, 16, 2, 1, 1), SK_K1(2, 4, 8, 1, 0), SK_K1(2, 4, 8, 2, 0),
    SK_K1(2, 8, 2, 2, 0), SK_K1(2, 8, 2, 4, 0), SK_K1(2, 16, 4, 1, 0), SK_K1(2, 32, 2, 1, 0), SK_K1(2, 32, 4, 1, 0),
    SK_K1(2, 8, 8, 1, 0), SK_K1(2, 16, 1, 4, 0), SK_K1(2, 8, 1, 4, 0), SK_K1(2, 4, 2, 4, 0),
    SK_K1(2, 4, 2, 8, 0), SK_K1(2, 4, 4, 4, 0), SK_K1(2, 8, 8, 2, 0), SK_K1(2, 16, 4, 2, 0), SK_K1(2, 8, 2, 1, 1), SK_K1(2, 4, 2, 1, 1), SK_K1(2, 4, 2, 2, 0), SK_K1(2, 16, 4, 1, 1),
    // 32-bit path (any pitch / alignment)
    SK_K1(1, 8, 1, 4, 0), SK_K1(1, 16, 1, 4, 0), SK_K1(1, 32, 1, 4, 0), SK_K1(1, 16, 4, 2, 0),
    SK_K1(1, 32, 2, 2, 0), SK_K1(1, 32, 4, 1, 0), SK_K1(1, 32, 8, 1, 0), SK_K1(1, 32, 16, 1, 0),
    SK_K1(1, 32, 32, 1, 0), SK_K1(1, 16, 4, 2, 1), SK_K1(1, 16, 4, 1, 1), SK_K1(1, 16, 4, 4, 0),
    SK_K1(1, 16, 4, 4, 1), SK_K1(1, 16, 4, 8, 0), SK_K1(1, 8, 8, 1, 0), SK_K1(1, 8, 8, 2, 0),
    SK_K1(1, 4, 16, 1, 0), SK_K1(1, 4, 8, 2, 0), SK_K1(1, 8, 4, 2, 0), SK_K1(1, 8, 4, 4, 0),
    SK_K1(1, 16, 8, 1, 0), SK_K1(1, 16, 8, 2, 0), SK_K1(1, 8, 16, 1, 0), SK_K1(1, 4, 4, 4, 0),
    SK_K1(1, 8, 2, 4, 0), SK_K1(1, 4, 4, 1, 1), SK_K1(1, 4, 4, 2, 0), SK_K1(1, 8, 4, 1, 1),
    SK_K1(1, 8, 8, 1, 1), SK_K1(1, 16, 8, 1, 1), SK_K1(1, 4, 2, 4, 0), SK_K1(1, 2, 4, 4, 0),
    SK_K1(1, 2, 4, 8, 0), SK_K1(1, 4, 2, 8, 0), SK_K1(1, 2, 4, 1, 1), SK_K1(1, 2, 4, 2, 0),
};
#undef SK_K1

const K1Entry* k1_find(int vec, int lpr, int nv, int u, int pf) {
  for (const auto& e : kK1Table)
    if (e.vec == vec && e.lpr == lpr && e.nv == nv && e.u == u && e.pf == pf) return &e;
  return nullptr;
}

// (VEC, LPR, NV) shapes the planner may shrink NV to -- the fewest vectors per
// lane that cover the row -- for every rows-per-group / prefetch variant the
// job-size policy of k1_default picks, so the shape (hence the bits) stays a
// function of C alone.
struct K1Fit {
  int vec, lpr, nv;
};
constexpr K1Fit kK1Fit[] = {{4, 4, 3},  {4, 8, 3},  {4, 16, 3}, {4, 32, 3},  {4, 32, 5},
                            {4, 32, 6}, {4, 32, 7}, {4, 32, 9},  {4, 32, 10}, {4, 32, 11},
                            {4, 32, 12}, {4, 32, 13}, {4, 32, 14}, {4, 32, 15}, {4, 32, 17},
                            {4, 32, 18}, {4, 32, 19}, {4, 32, 20}, {4, 32, 21}, {4, 32, 22},
                            {4, 32, 23}, {2, 8, 3},
                            {2, 16, 3}, {1, 2, 3},  {1, 4, 3},  {1, 8, 3},   {1, 8, 5},
                            {1, 8, 6},  {1, 8, 7},  {1, 16, 5}, {1, 16, 6},  {1, 16, 7},
                            {1, 32, 5}, {1, 32, 6}, {1, 32, 7},  {1, 32, 9},  {1, 32, 10},
                            {1, 32, 11}, {1, 32, 12}, {1, 32, 13}, {1, 32, 14}, {1, 32, 15},
                            {1, 32, 17}, {1, 32, 18}, {1, 32, 19}, {1, 32, 20}, {1, 32, 21},
                            {1, 32, 22}, {1, 32, 23}, {1, 32, 24}};  // 25-31: measured slower
std::atomic<int> g_k1_fit{1};
// K1 block size, shrunk to 64 for small jobs: 128 measured 0.5-2.5 % faster
// than 256 (c2 11.57 vs 11.61-11.66 us, c3 11.77 vs 12.05-12.11,
// profiles/r1d_k1_block_size_ab.jsonl); the bits do not depend on it
std::atomic<int> g_k1_threads{128};
std::atomic<int> g_k1_wide32{1280};  // 32-bit rows up to here take K1 (one warp per row), not K1m
int k1_fit_nv(int vec, int lpr, int nv, int64_t cols) {
  if (!g_k1_fit.load()) return nv;
  const int fit = static_cast<int>((cols + int64_t(lpr) * vec - 1) / (int64_t(lpr) * vec));
  if (fit >= nv) return nv;
  for (const auto& f : kK1Fit)
    if (f.vec == vec && f.lpr == lpr && f.nv == fit) return fit;
  return nv;
}

constexpr int64_t kK1MaxCols = 3072;  // 128-bit rows up to here take K1

// default K1 shape per row length (covers cols <= 1024; 128-bit rows <= 3072).  gm: grid multiplier
// over SMs x occupancy; 0 = non-persistent (one row batch per warp, grid = rows /
// rows-per-CTA), which measured fastest for every shape (c5a: 7.0 TB/s).
// The (VEC, LPR, NV) shape -- hence the bits -- is a function of C alone;
// only U (rows per lane group), PF and the grid follow the job size.  Rows of
// <= 64 floats in a large job (>= 4 Mi elements) stream with a persistent
// grid (2 waves, grid-stride) and, when a row group would otherwise carry one
// row, two rows per lane group: measured at 64 MiB (profiles/
// r1c_k1_small_rows_sweep2.jsonl) C = 48 / 52 25.7 / 25.3 us vs 33.3 / 31.3,
// C = 50 (32-bit) 33.3 vs 41.7, C = 8 / 20 -4 / -4 %.
constexpr int64_t kK1LargeJob = int64_t(1) << 22;
void k1_default(int vec, int64_t cols, int& lpr, int& nv, int& u, int& pf, int& gm,
                int64_t elems = 0) {
  pf = 0;
  gm = 0;
  const bool large = elems >= kK1LargeJob;
  if (vec == 8) {
    if (cols <= 64) { lpr = 8; nv = 1; u = 4; }
    else if (cols <= 128) { lpr = 16; nv = 1; u = 2; }
    else if (cols <= 256) { lpr = 16; nv = 2; u = 1; }
    else if (cols <= 512) { lpr = 32; nv = 2; u = 1; }
    else { lpr = 32; nv = 4; u = 1; }
  } else if (vec == 4) {
    if (cols <= 16) { lpr = 4; nv = 1; u = 4; gm = large ? 2 : 0; }
    // 17-64 floats: 4 lanes per row (profiles/r1d_k1_vec4_sweep.jsonl: 1.07-1.25x
    // the 8-lane shapes at 8-64 MiB); 129-256: one row per group unless large
    else if (cols <= 32) { lpr = 4; nv = 2; u = 2; gm = large ? 2 : 0; }
    else if (cols <= 64) { lpr = 4; nv = 4; u = 1; gm = large ? 2 : 0; }
    else if (cols <= 128) { lpr = 8; nv = 4; u = 1; }
    else if (cols <= 256) { lpr = 16; nv = 4; u = large ? 2 : 1; }
    else if (cols <= 512) { lpr = 32; nv = 4; u = 1; }
    else if (cols <= 1024) { lpr = 32; nv = 8; u = 1; }
    // medium rows: a whole warp holds the row in registers -- measured
    // 1.1-1.3x faster than the TMA block-per-row K2 from 1536 to 3072 columns
    else if (cols <= 2048) { lpr = 32; nv = 16; u = 1; }
    else { lpr = 32; nv = 24; u = 1; }
  } else if (vec == 2) {
    // 64-bit rows (even C, not a multiple of 4, 8-B pitch): half the memory
    // instructions of the 32-bit shapes and fewer lanes per row (fewer
    // shuffle levels), which is what bounds short rows.  Measured at 64 MiB
    // (profiles/r1d_k1_vec2_*.jsonl): 1.19-1.32x over the 32-bit plan for
    // C = 34..126, 2.6-2.9x for C = 10..30; rows per lane group follow the
    // job size (>= 1 Mi elements: 2-4) without changing the bits.
    const bool mid = elems >= (int64_t(1) << 20);
    if (cols <= 16) {
      lpr = 4; nv = 2;
      if (elems >= (int64_t(1) << 21)) u = 4;
      else if (elems >= (int64_t(1) << 18)) u = 2;
      else { u = 1; pf = 1; }
    }
    else if (cols <= 32) {
      lpr = 8; nv = 2;
      if (mid) u = 4; else { u = 1; pf = 1; }
    }
    else if (cols <= 64) {
      lpr = 8; nv = 4;
      if (mid) u = 2; else { u = 1; pf = 1; }
    }
    else if (cols <= 128) {
      lpr = 16; nv = 4;
      if (mid) u = 2; else { u = 1; pf = 1; }
    }
    else { lpr = 32; nv = 4; u = 1; }
  } else {
    // 32-bit rows: few lanes per row (2 / 4 / 8 / 8 / 16 for C <= 8 / 16 /
    // 32 / 64 / 128) -- short rows are bound by instructions per element
    // (memory instructions, shuffle levels), not by sectors.  Measured at
    // 64 MiB (profiles/r1d_k1_odd_*.jsonl): 1.1-2.7x the former 8-32-lane
    // shapes; small jobs take one row per group with prefetch.
    const bool mid = elems >= (int64_t(1) << 20);
    if (cols <= 8) {
      lpr = 2; nv = 4;
      if (elems >= (int64_t(1) << 21)) u = 4; else { u = 1; pf = 1; }
    }
    else if (cols <= 16) {
      lpr = 4; nv = 4;
      if (large) u = 4; else { u = 1; pf = 1; }
    }
    else if (cols <= 32) { lpr = 8; nv = 4; u = large ? 4 : 2; }
    else if (cols <= 64) {
      lpr = 8; nv = 8;
      if (large) { u = 2; gm = 2; } else if (mid) u = 2; else { u = 1; pf = 1; }
    }
    else if (cols <= 128) {
      lpr = 16; nv = 8;
      if (mid) u = 2; else { u = 1; pf = 1; }
    }
    else if (cols <= 256) { lpr = 32; nv = 8; u = 1; }
    else if (cols <= 512) { lpr = 32; nv = 16; u = 1; }
    else if (cols <= 1024) { lpr = 32; nv = 32; u = 1; }
    else if (cols <= 1152) { lpr = 32; nv = 36; u = 1; }  // one warp per row (g_k1_wide32)
    else { lpr = 32; nv = 40; u = 1; }
  }
}

// --------------------------------------------------------------- seg table
using SegFn = void (*)(const float*, float*, int64_t, int64_t, int64_t, int64_t, int, int,
                       unsigned*, RowPartial*, unsigned long long*, float);
template <int NV>
SegFn seg_fn(int mode) {
  switch (mode) {
    case kClipAccurate: return &k_seg<kClipAccurate, NV>;
    case kAccurate: return &k_seg<kAccurate, NV>;
    default: return &k_seg<kApprox, NV>;
  }
}
std::atomic<int> g_cluster_onex{0};  // K3c: one (m, s) exchange per row (measured slower)
std::atomic<int> g_cluster_tpb{512};  // K3c threads per CTA (512 or 1024)
template <int TPB>
const void* cluster_fn_t(int mode, bool one) {
  switch (mode) {
    case kClipAccurate:
      return one ? reinterpret_cast<const void*>(&k3_cluster<kClipAccurate, true, TPB>)
                 : reinterpret_cast<const void*>(&k3_cluster<kClipAccurate, false, TPB>);
    case kAccurate:
      return one ? reinterpret_cast<const void*>(&k3_cluster<kAccurate, true, TPB>)
                 : reinterpret_cast<const void*>(&k3_cluster<kAccurate, false, TPB>);
    default:
      return one ? reinterpret_cast<const void*>(&k3_cluster<kApprox, true, TPB>)
                 : reinterpret_cast<const void*>(&k3_cluster<kApprox, false, TPB>);
  }
}
const void* cluster_fn(int mode) {
  const bool one = g_cluster_onex.load() != 0;
  return g_cluster_tpb.load() == 1024 ? cluster_fn_t<1024>(mode, one)
                                      : cluster_fn_t<512>(mode, one);
}
int cluster_tpb() { return g_cluster_tpb.load() == 1024 ? 1024 : 512; }
constexpr int64_t kClusterSmemMax = 220 * 1024;  // ring bytes per CTA (227 KB minus statics)
constexpr int64_t kClusterSliceMaxAny = kClusterSmemMax / (2 * 4);  // 2-stage ring

// Clusters of `cs` CTAs that can be co-resident (0 if the shape cannot launch).
int max_active_clusters(const void* fn, int cs, size_t smem) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, int, size_t, int>, int> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_tuple(fn, cs, smem, dev);
  {
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
  }
  cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  ensure_smem_attr(fn, smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cs * 148);
  cfg.blockDim = dim3(cluster_tpb());
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute a[1];
  a[0].id = cudaLaunchAttributeClusterDimension;
  a[0].val.clusterDim.x = cs;
  a[0].val.clusterDim.y = 1;
  a[0].val.clusterDim.z = 1;
  cfg.attrs = a;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, fn, &cfg) != cudaSuccess) {
    (void)cudaGetLastError();
    n = 0;
  }
  std::lock_guard<std::mutex> g(mu);
  cache[key] = n;
  return n;
}

bool gres_split(int lag);
constexpr int64_t kGresSmemMax = 225 * 1024;  // ring bytes per K3g CTA (227 KB opt-in minus statics)
template <int L, bool SPLIT, bool UNAL = false>
const void* gres_fn_l(int mode) {
  switch (mode) {
    case kClipAccurate: return reinterpret_cast<const void*>(&k3_gres<kClipAccurate, L, SPLIT, UNAL>);
    case kAccurate: return reinterpret_cast<const void*>(&k3_gres<kAccurate, L, SPLIT, UNAL>);
    default: return reinterpret_cast<const void*>(&k3_gres<kApprox, L, SPLIT, UNAL>);
  }
}
// lag 1..3 (the ring depth is a launch argument >= lag + 2, or 2 at lag 1)
const void* gres_fn(int mode, int lag, bool split);
// rows of any alignment: the two schedules the planner uses (lag 1 with the
// publisher polling, lag 2 with a poller warp); nullptr otherwise
const void* gres_fn_unal(int mode, int lag, bool split) {
  if (lag == 1 && !split) return gres_fn_l<1, false, true>(mode);
  if (lag == 2 && split) return gres_fn_l<2, true, true>(mode);
  return nullptr;
}
const void* gres_fn(int mode, int lag, bool split, bool unal) {
  if (unal) return gres_fn_unal(mode, lag, split);
  return gres_fn(mode, lag, split);
}
const void* gres_fn(int mode, int lag, bool split) {
  if (split)
    return lag >= 3 ? gres_fn_l<3, true>(mode)
           : lag == 2 ? gres_fn_l<2, true>(mode) : gres_fn_l<1, true>(mode);
  return lag >= 3 ? gres_fn_l<3, false>(mode)
         : lag == 2 ? gres_fn_l<2, false>(mode) : gres_fn_l<1, false>(mode);
}

constexpr int kSegNV = 4;
constexpr int kSegMaxThreads = 512;
constexpr int64_t kSegCap = int64_t(kSegMaxThreads) * kSegNV * 4;  // 8192 floats / CTA

// Occupancy per (kernel, block, smem, device), cached: the query is not free
// and sk_softmax_f32 is called once per softmax.

int occupancy(const void* fn, int threads, size_t smem) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, int, size_t, int>, int> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_tuple(fn, threads, smem, dev);
  {
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
  }
  ensure_smem_attr(fn, smem);
  int nb = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, threads, smem) != cudaSuccess) {
    (void)cudaGetLastError();
    nb = 0;
  }
  std::lock_guard<std::mutex> g(mu);
  cache[key] = nb;
  return nb;
}

// --------------------------------------------------------------- planning
enum PathKind { kPathK1 = 0, kPathSeg = 1, kPathSplit = 2, kPathK1m = 3 };

// ------------------------------------------------------------ K1m table
using K1mFn = K1Fn;
struct K1mEntry {
  int vec, wpr, nv;
  K1mFn fn[3];
};
#define SK_K1M(VEC, WPR, NV)                                                             \
  K1mEntry {                                                                             \
    VEC, WPR, NV, {                                                                      \
      &k1m_rows<kClipAccurate, WPR, NV, VEC>, &k1m_rows<kAccurate, WPR, NV, VEC>,        \
          &k1m_rows<kApprox, WPR, NV, VEC>                                               \
    }                                                                                    \
  }
const K1mEntry kK1mTable[] = {
    // 128-bit rows
    SK_K1M(4, 2, 16), SK_K1M(4, 4, 8), SK_K1M(4, 4, 12), SK_K1M(4, 4, 16), SK_K1M(4, 8, 8),
    SK_K1M(4, 8, 12), SK_K1M(4, 8, 16),
    // exact fit (fewest float4 per thread covering the row, k1m_fit_nv)
    SK_K1M(4, 2, 13), SK_K1M(4, 2, 14), SK_K1M(4, 2, 15), SK_K1M(4, 4, 9), SK_K1M(4, 4, 10),
    SK_K1M(4, 4, 11), SK_K1M(4, 4, 13), SK_K1M(4, 4, 14), SK_K1M(4, 4, 15), SK_K1M(4, 8, 9),
    SK_K1M(4, 8, 10), SK_K1M(4, 8, 11), SK_K1M(4, 8, 13), SK_K1M(4, 8, 14), SK_K1M(4, 8, 15),
    SK_K1M(1, 2, 18), SK_K1M(1, 2, 20), SK_K1M(1, 2, 28), SK_K1M(1, 2, 36), SK_K1M(1, 2, 40),
    SK_K1M(1, 4, 28), SK_K1M(1, 4, 36), SK_K1M(1, 4, 40), SK_K1M(1, 8, 28), SK_K1M(1, 8, 36),
    SK_K1M(1, 8, 40), SK_K1M(1, 8, 52), SK_K1M(1, 8, 56),
    // 32-bit rows (any length / alignment): 1025..16384 floats
    SK_K1M(1, 2, 24), SK_K1M(1, 2, 32), SK_K1M(1, 2, 48), SK_K1M(1, 4, 32), SK_K1M(1, 4, 48),
    SK_K1M(1, 8, 32), SK_K1M(1, 8, 48), SK_K1M(1, 8, 64)};
#undef SK_K1M
const K1mEntry* k1m_find(int vec, int wpr, int nv) {
  for (const auto& e : kK1mTable)
    if (e.vec == vec && e.wpr == wpr && e.nv == nv) return &e;
  return nullptr;
}
constexpr int64_t kK1mCap = 16384;  // widest row a K1m instantiation holds
std::atomic<int> g_k1m{1}, g_k1m_wpr{0}, g_k1m_nv{0};
std::atomic<int> g_k1m_threads{0};  // K1m threads per block (0: one row, 32 * WPR)
// widest row the planner gives K1m.  Measured (scripts/wide_k1m.py,
// profiles/r1c_wide_k1m.jsonl): a 256-thread block holding a 12288 / 16384-float
// row beats K3g's one-CTA rows by 2-16% (1024x16384 26.1 vs 30.3 us)
std::atomic<int> g_k1m_max{16384};
// measured (scripts/medium_rows.py): 16384x4096 80.5 us with (2,16) vs 101.5
// for K2; 8192x6144 62.4 (4,12); 8192x8192 80.1 (4,16) vs 88.6 for K2
void k1m_default(int vec, int64_t cols, int& wpr, int& nv) {
  if (vec == 4) {
    if (cols <= 4096) { wpr = 2; nv = 16; }
    else if (cols <= 6144) { wpr = 4; nv = 12; }
    else if (cols <= 8192) { wpr = 4; nv = 16; }
    else if (cols <= 12288) { wpr = 8; nv = 12; }  // a 256-thread block per row
    else { wpr = 8; nv = 16; }
  } else {  // 32-bit accesses
    if (cols <= 1536) { wpr = 2; nv = 24; }
    else if (cols <= 2048) { wpr = 2; nv = 32; }
    else if (cols <= 3072) { wpr = 2; nv = 48; }
    else if (cols <= 4096) { wpr = 4; nv = 32; }
    else if (cols <= 6144) { wpr = 4; nv = 48; }
    else if (cols <= 8192) { wpr = 8; nv = 32; }
    else if (cols <= 12288) { wpr = 8; nv = 48; }
    else { wpr = 8; nv = 64; }
  }
}

struct Plan {
  PathKind kind = kPathK1;
  // K1
  const K1Entry* k1 = nullptr;
  const K1mEntry* k1m = nullptr;
  bool unal = false;  // K3g over rows of any alignment
  // seg (K2: nseg == 1; K3: nseg > 1)
  int nseg = 1, seglen = 0, threads = 0, lag = 0;  // lag: ring depth (K2/K3c/K3g)
  int glag = 0;                                     // K3g: rows between local and output pass
  int k3 = 0;  // 0 K2, 6 K3c (cluster), 7 K3g (grid-resident)
  int64_t chunk_rows = 0;
  size_t smem = 0;
  // split
  int nch = 0;
  int64_t grid = 0;
  bool vec = false;
};

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// [0] bad-row flag (8 B) | [8] task counter (8 B) | row counters | row ready
// flags | partials | row max | row sum.  [8, part) is zeroed before a K3 launch.
struct WsLayout {
  size_t bad = 0, ctrl = 8, cnt = 0, ready = 0, part = 0, rmax = 0, rsum = 0, total = 0;
};
WsLayout ws_layout(int64_t rows, int64_t parts_per_row) {
  WsLayout l;
  l.bad = 0;
  l.ctrl = 8;
  l.cnt = 256;
  l.ready = align_up(l.cnt + size_t(rows) * 4, 256);
  l.part = align_up(l.ready + size_t(rows) * 4, 256);
  l.rmax = align_up(l.part + size_t(rows) * size_t(parts_per_row) * sizeof(RowPartial), 256);
  l.rsum = align_up(l.rmax + size_t(rows) * 4, 256);
  l.total = align_up(l.rsum + size_t(rows) * 8, 256);
  return l;
}

int plan_split(int64_t rows, int64_t cols, Plan& p) {
  p.kind = kPathSplit;
  p.nch = static_cast<int>((cols + kSplitChunk - 1) / kSplitChunk);
  p.grid = rows * p.nch;
  if (p.grid > int64_t(INT32_MAX)) return arg_fail("matrix too large for the split path");
  return SK_OK;
}

// K3g shape: P CTAs per row (per rank), ring depth st, `groups` row groups
// per rank.  world ranks each hold a [rows, cols] column shard (world*P pairs
// merged per row); nvr of them run in this launch (nvr = world when one GPU
// emulates all ranks, 1 on a real rank).  Deterministic in its inputs, so
// every rank of a column shard derives the same plan.
// Step-time model, fitted to a (P, stages) grid measured on B200 (c4, c5b;
// profiles/r1_gres_grid.jsonl) and checked against the best measured plan of
// ten other long-row shapes (it picks it, within ~5%, on all of them):
//   step   = streaming of 8 B x slice at the SM's share of HBM (<= 55 GB/s)
//          + X, the part of the exchange round trip the ring does not hide:
//   RTT    = 1.6 us (+16 ns per merged pair beyond 32, at most 2.3 us)
//   hide   = 0.0775 us per 1000 floats of slice per lag step
//   X      = RTT (depth 2) | RTT - hide (depth 3, lag 1) |
//            RTT - 2 hide + 0.3 us (depth 4, lag 2: the poller warp's cost)
//   time   = (ceil(rows / groups) + 1) x step     (one CTA per SM)
double gres_time_us(int64_t rows, int P, int st, int64_t slice, int groups, int world, int nvr) {
  const double active = double(std::min<int64_t>(groups, rows)) * P * nvr;
  const double ts = double(slice) * 8.0 / std::min(6.47e12 / std::max(1.0, active), 55e9) * 1e6;
  const double rtt = std::min(2.3, 1.6 + 0.016 * std::max(0, world * P - 32));
  const double hide = 0.0775 * double(slice) / 1000.0;
  const double x = st == 2 ? rtt : st == 3 ? std::max(0.1, rtt - hide)
                                           : std::max(0.1, rtt - 2.0 * hide) + 0.3;
  return double((rows + groups - 1) / groups + 1) * (ts + x);
}

// The plan is a function of the row LENGTH only (modelled at a fixed row
// count), so a row block computed alone takes the same plan -- and gives the
// same bits -- as the whole matrix: row sharding stays communication-free and
// bit-identical.  At 2048 rows the choice equals the per-shape best on every
// measured long-row shape.

GresChoice plan_gres(int64_t rows, int64_t cols, int mode, const DevInfo& di, int world, int nvr,
                     bool unal) {
  GresChoice best;
  double best_t = 0.0;
  for (int P = 1; P * world <= kGresMaxSlots && P * nvr <= di.sms; ++P) {
    if (g_gres_p.load() > 0 && P != g_gres_p.load()) continue;
    const int64_t slice = align_up((cols + P - 1) / P, 4);
    if ((P - 1) * slice >= cols) continue;
    // depth 5 (lag 3) measured no better than 4: only when forced
    const int st_cap = g_gres_st.load() >= 2 ? kGresStages : 4;
    const int st_max = static_cast<int>(std::min<int64_t>(
        st_cap, kGresSmemMax / (slice * int64_t(sizeof(float)))));
    const int groups = di.sms / (P * nvr);  // one CTA per SM
    if (groups < 1 || (rows + groups - 1) / groups >= (int64_t(1) << 31)) continue;
    for (int st = 2; st <= st_max; ++st) {
      if (g_gres_st.load() >= 2 && st != g_gres_st.load()) continue;
      // lag: the forced one, else the classic schedule (depth 2-3 lag 1, 4 lag 2, 5 lag 3)
      const int lag = g_gres_lag.load() > 0 ? g_gres_lag.load() : std::max(1, std::min(3, st - 2));
      if (lag > 3 || (st < lag + 2 && !(st == 2 && lag == 1))) continue;
      const size_t smem = size_t(st) * slice * sizeof(float);
      const bool split = gres_split(lag);
      const void* fn = gres_fn(mode, lag, split, unal);
      if (!fn || occupancy(fn, split ? kGresBlock : kGresThreads, smem) < 1) continue;
      const double t = gres_time_us(rows, P, st, slice, groups, world, nvr);
      if (best.P == 0 || t < best_t) {
        best_t = t;
        best.P = P;
        best.st = st;
        best.lag = lag;
        best.groups = groups;
        best.slice = slice;
        best.score = 1.0 / t;
      }
    }
  }
  return best;
}

// Single-device K3g plan: a function of the row length alone, so row blocks
// keep their bits.  K3g's per-CTA pipeline needs a few row steps to amortise
// its fill (first slice in flight), its exchange round trip and its launch
// (cooperative, no PDL): with <= 3 row steps per group (decode-sized batches
// over wide rows) the caller is told to take the latency path instead --
// measured: 1 x 32000 K3c 3.45 us vs K3g 6.18; 32 x 151936 split 14.3 vs
// K3g 15.6; 8 x 50257 split 7.0 vs 8.3.  Larger jobs (c4 row-sharded 8 ways:
// 64 rows, 7 steps) keep the C-only plan.
GresChoice plan_gres_for(int64_t rows, int64_t cols, int mode, const DevInfo& di, bool unal,
                         bool* latency) {
  const GresChoice gc = plan_gres(kGresPlanRows, cols, mode, di, 1, 1, unal);
  *latency = gc.P > 0 && g_gres.load() != 2 &&
             (rows + gc.groups - 1) / gc.groups <= g_latency_steps.load();
  return gc;
}

int make_plan(int64_t rows, int64_t cols, int64_t ldx, int64_t ldy, uint64_t xa, uint64_t ya,
              int mode, int dev, Plan& p, bool bulk = false) {
  const DevInfo di = dev_info(dev);
  const bool vec = (cols % 4 == 0) && (ldx % 4 == 0) && (ldy % 4 == 0) && (xa % 16 == 0) &&
                   (ya % 16 == 0);
  const bool vec8 = vec && (cols % 8 == 0) && (ldx % 8 == 0) && (ldy % 8 == 0) &&
                    (xa % 32 == 0) && (ya % 32 == 0) && g_vec8.load();
  // 64-bit K1 rows: even rows on 8-B pitches / bases that rule out 128-bit ones
  const bool vec2 = !vec && cols > 8 && (cols % 2 == 0) && (ldx % 2 == 0) && (ldy % 2 == 0) &&
                    (xa % 8 == 0) && (ya % 8 == 0) && cols <= g_vec2_max.load();
  p.vec = vec;
  const int force = g_force_path.load();
  const int64_t k1m_max = std::min<int64_t>(g_k1m_max.load(), kK1mCap);
  PathKind kind;
  if (force >= 0) kind = static_cast<PathKind>(force);
  else if (cols <= 1024 || (vec && cols <= kK1MaxCols) || (!vec && cols <= g_k1_wide32.load()))
    kind = kPathK1;
  else if (cols <= k1m_max && g_k1m.load()) kind = kPathK1m;
  else if (vec) kind = kPathSeg;
  else kind = kPathSplit;
  if (kind == kPathK1 && cols > kK1MaxCols) return arg_fail("k1 path needs cols <= 3072");
  if (kind == kPathSeg && !vec) return arg_fail("seg path needs 16-B aligned rows");

  if (kind == kPathSplit && force < 0 && !vec && cols > k1m_max && g_gres.load() != 0 &&
      di.coop) {
    // rows of any alignment too long for one CTA: K3g with TMA on each slice's
    // aligned middle (1.7x the split path's 12 B/element on a 50257-wide vocab)
    bool latency = false;
    const GresChoice gc = plan_gres_for(rows, cols, mode, di, true, &latency);
    if (bulk) latency = false;
    if (gc.P > 0 && !latency) {
      p.kind = kPathSeg;
      p.k3 = 7;
      p.unal = true;
      p.nseg = gc.P;
      p.seglen = static_cast<int>(gc.slice);
      p.lag = gc.st;
      p.glag = gc.lag;
      p.threads = gres_split(gc.lag) ? kGresBlock : kGresThreads;
      p.smem = size_t(gc.st) * gc.slice * sizeof(float);
      p.grid = int64_t(gc.groups) * gc.P;
      return SK_OK;
    }
  }
  if (kind == kPathK1m) {
    const int vw = vec ? 4 : 1;
    int wpr, nv;
    k1m_default(vw, cols, wpr, nv);
    if (g_k1_fit.load()) {  // fit: the fewest instantiated vectors per thread covering the row
      const int need = static_cast<int>((cols + int64_t(wpr) * 32 * vw - 1) / (int64_t(wpr) * 32 * vw));
      for (const auto& f : kK1mTable)
        if (f.vec == vw && f.wpr == wpr && f.nv >= need && f.nv < nv) nv = f.nv;
    }
    if (g_k1m_wpr.load() > 0) { wpr = g_k1m_wpr; nv = g_k1m_nv; }
    const K1mEntry* e = k1m_find(vw, wpr, nv);
    if (!e) return arg_fail("no K1m instantiation for the requested shape");
    if (int64_t(wpr) * 32 * nv * vw < cols) return arg_fail("K1m shape does not cover cols");
    p.kind = kPathK1m;
    p.k1m = e;
    // block: one row (32 * WPR threads) -- 1.10-1.25x over 256-thread blocks
    // holding 2-4 rows (4096 floats 23.9 -> 21.5 us, 1501 44.2 -> 35.4,
    // profiles/r1d_k1m_block_size_ab.jsonl; same bits); the k1m_threads knob
    // forces a size that still holds a whole row
    const int kt = g_k1m_threads.load();
    // whole rows per block: a multiple of 32 * WPR threads (a partial row would
    // read reduction slots no warp wrote)
    p.threads = (kt >= 32 * wpr && kt <= kRowsThreads) ? kt / (32 * wpr) * (32 * wpr) : 32 * wpr;
    const int64_t rpc = p.threads / 32 / wpr;
    p.grid = std::max<int64_t>(1, std::min<int64_t>((rows + rpc - 1) / rpc, INT32_MAX));
    return SK_OK;
  }
  if (kind == kPathK1) {
    int lpr, nv, u, pf, gm;
    const int vw = vec8 ? 8 : vec ? 4 : vec2 ? 2 : 1;
    k1_default(vw, cols, lpr, nv, u, pf, gm, rows * cols);
    nv = k1_fit_nv(vw, lpr, nv, cols);
    if (g_k1_lpr.load() > 0) { lpr = g_k1_lpr; nv = g_k1_nv; u = g_k1_u; }
    if (g_k1_pf.load() >= 0) pf = g_k1_pf.load();
    if (g_grid_mult.load() > 0) gm = g_grid_mult.load();
    const K1Entry* e = k1_find(vw, lpr, nv, u, pf);
    if (!e) return arg_fail("no K1 instantiation for the requested shape");
    if (int64_t(lpr) * nv * e->vec < cols) return arg_fail("K1 shape does not cover cols");
    p.kind = kPathK1;
    p.k1 = e;
    // block size: 256 threads, halved (to 64) while the job would occupy fewer
    // CTAs than SMs -- a small job then spreads over the chip.  Each row is one
    // warp's work whatever the block size, so the bits do not change.
    // a whole number of warps (K1 numbers warps as (blockIdx*blockDim+tid)>>5)
    int threads = std::max(32, std::min(g_k1_threads.load(), kRowsThreads) / 32 * 32);
    auto rows_per = [&](int t) { return int64_t(t / 32) * u * (32 / lpr); };
    while (threads > 64 && (rows + rows_per(threads) - 1) / rows_per(threads) < di.sms) threads /= 2;
    p.threads = threads;
    const int64_t rows_per_cta = rows_per(threads);
    const int64_t need = (rows + rows_per_cta - 1) / rows_per_cta;
    const int occ = occupancy(reinterpret_cast<const void*>(e->fn[mode]), threads, 0);
    const int64_t cap = gm > 0 ? int64_t(di.sms) * std::max(occ, 1) * gm : need;
    p.grid = std::max<int64_t>(1, std::min({need, cap, int64_t(INT32_MAX)}));
    return SK_OK;
  }
  if (kind == kPathSeg) {
    const int impl0 = g_k3_impl.load();
    // Resident rows: K3g (P CTAs anywhere on the chip, global-memory
    // exchange; plan from the measured step-time model) -- measured 1.1-1.4x
    // faster than K3c on every long-row shape tried -- else K3c (one
    // thread-block cluster per row) when K3g is off or cannot launch.
    const int gres = g_gres.load();
    if ((cols > kSegCap || gres == 2) && (impl0 == 5 || impl0 == 3)) {
      GresChoice gc;
      bool latency = false;
      if (gres != 0 && impl0 != 5 && di.coop) gc = plan_gres_for(rows, cols, mode, di, false, &latency);
      if (bulk) latency = false;
      if (latency && rows > 2) return plan_split(rows, cols, p);
      if (gc.P > 0 && !latency) {
        p.kind = kPathSeg;
        p.k3 = 7;
        p.nseg = gc.P;
        p.seglen = static_cast<int>(gc.slice);
        p.lag = gc.st;
        p.glag = gc.lag;
        p.threads = gres_split(gc.lag) ? kGresBlock : kGresThreads;
        p.smem = size_t(gc.st) * gc.slice * sizeof(float);
        p.grid = int64_t(gc.groups) * gc.P;
        return SK_OK;
      }
      if (gres == 2) return arg_fail("K3g cannot launch this row length on this device");
      double best_c = 0.0;
      int c_cs = 0, c_st = 0, c_n = 0;
      int64_t c_slice = 0;
      if (g_cluster_k3.load() && cols <= 16 * kClusterSliceMaxAny) {
        // K3c: the cluster size that keeps the most SMs busy (GPC packing), with
        // a ring of >= 2 stages of the row slice in shared memory
        const void* fn = cluster_fn(mode);
        for (int cs = 16; cs >= 1; --cs) {
          if (g_cluster_size.load() > 0 && cs != g_cluster_size.load()) continue;
          const int64_t slice = align_up((cols + cs - 1) / cs, 4);
          if ((cs - 1) * slice >= cols) continue;  // every rank needs a non-empty slice
          const int st = static_cast<int>(std::min<int64_t>(
              kClusterStages, kClusterSmemMax / (slice * int64_t(sizeof(float)))));
          if (st < 2) continue;
          const size_t smem = size_t(st) * slice * sizeof(float);
          const int n = max_active_clusters(fn, cs, smem);
          // each row step costs ~8192 floats' worth of time in its two exchanges
          const double score = double(std::min<int64_t>(n, rows)) * cs * double(slice) /
                               double(slice + 8192);
          if (n > 0 && score > best_c) {
            best_c = score;
            c_cs = cs;
            c_st = st;
            c_n = n;
            c_slice = slice;
          }
        }
      }
      if (c_n > 0) {
        p.kind = kPathSeg;
        p.k3 = 6;
        p.nseg = c_cs;
        p.seglen = static_cast<int>(c_slice);
        p.lag = c_st;
        p.threads = cluster_tpb();
        p.smem = size_t(c_st) * c_slice * sizeof(float);
        p.grid = int64_t(c_n) * c_cs;
        return SK_OK;
      }
      if (impl0 == 5) return arg_fail("cluster K3 cannot launch on this device");
    }
    if (cols > kSegCap) {
      if (force >= 0 && impl0 == 5) return arg_fail("cluster K3 cannot launch on this device");
      return plan_split(rows, cols, p);  // beyond on-chip residency: K4
    }
    // K2: one CTA per row, TMA into a 2-stage shared-memory ring (the fallback
    // for rows <= 8192 when K1/K1m are switched off)
    p.kind = kPathSeg;
    p.nseg = 1;
    p.seglen = static_cast<int>(align_up(cols, 4));
    int threads = static_cast<int>(align_up((p.seglen / 4 + kSegNV - 1) / kSegNV, 32));
    threads = std::max(threads, 64);
    p.threads = threads;
    p.smem = size_t(kSegStages) * threads * kSegNV * 4 * sizeof(float);
    const int occ = occupancy(reinterpret_cast<const void*>(seg_fn<kSegNV>(mode)), threads, p.smem);
    p.grid = std::min(rows, int64_t(di.sms) * std::max(occ, 1));
    return SK_OK;
  }
  return plan_split(rows, cols, p);
}

// K3g control block: ctl words (epoch, finished CTAs, abort) | slot sets
// [epoch parity][group][2L+2][P] x 16 B.  Slots are epoch-tagged, so a block that persists
// across launches (the library's, below) is never cleared; a caller-supplied
// workspace is cleared before every launch instead (epoch restarts at 0).
struct GresWs {
  size_t ctl = 0, slots = 256, total = 0;
};
GresWs gres_ws(const Plan& p) {
  GresWs w;
  const size_t groups = size_t(p.grid / p.nseg);
  const int lag = p.glag;
  w.total = align_up(w.slots + 2 * groups * gres_slot_sets(lag) * p.nseg * 16, 256);
  return w;
}
constexpr size_t kGresWsMax = size_t(1) << 20;  // >= any single-device plan (<= 444 CTAs x 8 sets x 32 B)

// Library-owned K3g control block per (device, stream): zeroed once, then
// only ever advanced by the kernels themselves (other paths never touch it).
// The kernels zero this block themselves every gres_reset_period() launches
// (GresComm::reset_words, sk_gres.cuh), so its 23-bit slot epoch never wraps,
// CUDA-graph replays included.
std::mutex g_gres_mu;
std::map<std::pair<int, cudaStream_t>, void*> g_gres_blk;
std::atomic<unsigned long long> g_gres_epoch_reset{kGresEpochReset};
unsigned long long gres_reset_period() {
  const unsigned long long v = g_gres_epoch_reset.load();
  return (v == 0 || v > kGresEpochReset) ? kGresEpochReset : v;
}
int get_gres_block(int dev, cudaStream_t s, char** out) {
  std::lock_guard<std::mutex> g(g_gres_mu);
  void*& b = g_gres_blk[{dev, s}];
  if (!b) {
    SK_CUDA(cudaMallocAsync(&b, kGresWsMax, s));
    SK_CUDA(cudaMemsetAsync(b, 0, kGresWsMax, s));
  }
  *out = static_cast<char*>(b);
  return SK_OK;
}

size_t plan_ws_bytes(const Plan& p, int64_t rows) {
  if (p.kind == kPathSeg && p.k3 == 6) return ws_layout(0, 0).total;
  if (p.kind == kPathSeg && p.k3 == 7) return 256 + gres_ws(p).total;  // at ws + 256
  if (p.kind == kPathSeg && p.nseg > 1) return ws_layout(rows, p.nseg).total;
  if (p.kind == kPathSplit) return ws_layout(rows, p.nch).total;
  return ws_layout(0, 0).total;
}

// ------------------------------------------------- library-managed workspace
struct Ws {
  void* ptr = nullptr;
  size_t bytes = 0;
};
std::mutex g_ws_mu;
std::map<std::pair<int, cudaStream_t>, Ws> g_ws;

int get_ws(int dev, cudaStream_t s, size_t need, void** out) {
  std::lock_guard<std::mutex> g(g_ws_mu);
  Ws& w = g_ws[{dev, s}];
  if (w.bytes < need) {
    size_t nb = std::max(need, size_t(1) << 20);
    if (w.ptr) SK_CUDA(cudaFreeAsync(w.ptr, s));
    w.ptr = nullptr;
    w.bytes = 0;
    SK_CUDA(cudaMallocAsync(&w.ptr, nb, s));
    SK_CUDA(cudaMemsetAsync(w.ptr, 0, nb, s));
    // bad-row flag lives at offset 0: "no bad row"
    SK_CUDA(cudaMemsetAsync(w.ptr, 0xFF, 8, s));
    w.bytes = nb;
  }
  *out = w.ptr;
  return SK_OK;
}

int check_common(const float* x, const void* y, int64_t rows, int64_t cols, int64_t ldx,
                 int64_t ldy, int mode) {
  if (rows < 0 || cols < 1) return arg_fail("need rows >= 0 and cols >= 1");
  if (ldx < cols || ldy < cols) return arg_fail("row pitch must be >= cols");
  if (mode < 0 || mode > 2) return arg_fail("mode must be SK_MODE_CLIPPED/EXACT/APPROX");
  if (rows > 0 && (!x || !y)) return arg_fail("null buffer");
  if (cols > (int64_t(1) << 40)) return arg_fail("cols too large");
  // clip mode skips the sub-normal flush: every output >= e^-64 / cols is normal
  if (mode == 0 && cols > int64_t(13000000000)) return arg_fail("cols too large for clip mode");
  return SK_OK;
}

std::atomic<int> g_k4_fuse_combine{1};  // split path: merge the row stats inside normalize
int launch_split(const float* x, float* y, int64_t rows, int64_t cols, int64_t ldx,
                 int64_t ldy, int mode, bool v4, unsigned long long* bad, char* ws, int nch,
                 bool normalize, float* rmax_out, double* rsum_out, cudaStream_t s) {
  const WsLayout l = ws_layout(rows, nch);
  RowPartial* part = reinterpret_cast<RowPartial*>(ws + l.part);
  float* rmax = rmax_out ? rmax_out : reinterpret_cast<float*>(ws + l.rmax);
  double* rsum = rsum_out ? rsum_out : reinterpret_cast<double*>(ws + l.rsum);
  const dim3 g(static_cast<unsigned>(rows * nch));
  const float sh = shift_scale();
  const bool sv4 = (cols % 4 == 0) && (ldx % 4 == 0) && (reinterpret_cast<uintptr_t>(x) % 16 == 0);
  const void* stats =
      mode == kClipAccurate
          ? (sv4 ? reinterpret_cast<const void*>(&k4_stats<kClipAccurate, 4>)
                 : reinterpret_cast<const void*>(&k4_stats<kClipAccurate, 1>))
      : mode == kAccurate ? (sv4 ? reinterpret_cast<const void*>(&k4_stats<kAccurate, 4>)
                                 : reinterpret_cast<const void*>(&k4_stats<kAccurate, 1>))
                          : (sv4 ? reinterpret_cast<const void*>(&k4_stats<kApprox, 4>)
                                 : reinterpret_cast<const void*>(&k4_stats<kApprox, 1>));
  SK_CUDA(launch_k(stats, g, dim3(kSplitThreads), 0, s, false, x, rows, cols, ldx, nch, part,
                   bad, sh));
  if (normalize && !rmax_out && !rsum_out && g_k4_fuse_combine.load() &&
      (rows * nch <= 4096 || g_k4_fuse_combine.load() == 2)) {
    // two launches: the row statistics are merged inside the normalize pass --
    // for decode-sized jobs, where the third launch is a visible share
    // (8x50257 6.90 -> 6.53 us, 32x151936 15.6 -> 14.7, 64x128256 21.6 -> 19.9);
    // with many items every item re-merging its row's partials costs more
    // (1024x50257: 118 -> 125 us), profiles/r1d_split_fused_combine.jsonl
    const void* nr;
    switch (mode) {
      case kClipAccurate:
        nr = v4 ? reinterpret_cast<const void*>(&k4_normalize_rows<kClipAccurate, 4>)
                : reinterpret_cast<const void*>(&k4_normalize_rows<kClipAccurate, 1>);
        break;
      case kAccurate:
        nr = v4 ? reinterpret_cast<const void*>(&k4_normalize_rows<kAccurate, 4>)
                : reinterpret_cast<const void*>(&k4_normalize_rows<kAccurate, 1>);
        break;
      default:
        nr = v4 ? reinterpret_cast<const void*>(&k4_normalize_rows<kApprox, 4>)
                : reinterpret_cast<const void*>(&k4_normalize_rows<kApprox, 1>);
    }
    SK_CUDA(launch_k(nr, g, dim3(kSplitThreads), 0, s, false, x, y, rows, cols, ldx, ldy, nch,
                     static_cast<const RowPartial*>(part)));
    return SK_OK;
  }
  SK_CUDA(launch_k(reinterpret_cast<const void*>(&k4_combine),
                   dim3(static_cast<unsigned>((rows * 32 + 255) / 256)), dim3(256), 0, s, false,
                   static_cast<const RowPartial*>(part), rows, nch, rmax, rsum));
  if (!normalize) return SK_OK;
  const void* norm;
  switch (mode) {
    case kClipAccurate:
      norm = v4 ? reinterpret_cast<const void*>(&k4_normalize<kClipAccurate, 4>)
                : reinterpret_cast<const void*>(&k4_normalize<kClipAccurate, 1>);
      break;
    case kAccurate:
      norm = v4 ? reinterpret_cast<const void*>(&k4_normalize<kAccurate, 4>)
                : reinterpret_cast<const void*>(&k4_normalize<kAccurate, 1>);
      break;
    default:
      norm = v4 ? reinterpret_cast<const void*>(&k4_normalize<kApprox, 4>)
                : reinterpret_cast<const void*>(&k4_normalize<kApprox, 1>);
  }
  SK_CUDA(launch_k(norm, g, dim3(kSplitThreads), 0, s, false, x, y, rows, cols, ldx, ldy, nch,
                   static_cast<const float*>(rmax), static_cast<const double*>(rsum)));
  return SK_OK;
}

int launch_plan(const Plan& p, const float* x, float* y, int64_t rows, int64_t cols,
                int64_t ldx, int64_t ldy, int mode, unsigned long long* bad, char* ws,
                cudaStream_t s, bool user_ws) {
  const float sh = shift_scale();
  if (p.kind == kPathK1m) {
    SK_CUDA(launch_k(reinterpret_cast<const void*>(p.k1m->fn[mode]),
                     dim3(static_cast<unsigned>(p.grid)), dim3(p.threads), 0, s, false, x, y,
                     rows, static_cast<int>(cols), ldx, ldy, bad, sh));
    return SK_OK;
  }
  if (p.kind == kPathK1) {
    SK_CUDA(launch_k(reinterpret_cast<const void*>(p.k1->fn[mode]),
                     dim3(static_cast<unsigned>(p.grid)), dim3(p.threads), 0, s, false, x, y,
                     rows, static_cast<int>(cols), ldx, ldy, bad, sh));
    return SK_OK;
  }
  if (p.kind == kPathSeg) {
    const WsLayout l = ws_layout(rows, p.nseg);
    unsigned* cnt = reinterpret_cast<unsigned*>(ws + l.cnt);
    RowPartial* part = reinterpret_cast<RowPartial*>(ws + l.part);
    const int nseg = p.nseg, seglen = p.seglen;
    if (p.k3 == 6) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(static_cast<unsigned>(p.grid));
      cfg.blockDim = dim3(p.threads);
      cfg.dynamicSmemBytes = p.smem;
      cfg.stream = s;
      cudaLaunchAttribute a[2];
      a[0].id = cudaLaunchAttributeClusterDimension;
      a[0].val.clusterDim.x = static_cast<unsigned>(p.nseg);
      a[0].val.clusterDim.y = 1;
      a[0].val.clusterDim.z = 1;
      int na = 1;
      if (g_pdl.load()) {
        a[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        a[1].val.programmaticStreamSerializationAllowed = 1;
        na = 2;
      }
      cfg.attrs = a;
      cfg.numAttrs = na;
      int slice = p.seglen, nst = p.lag, dg = g_gres_diag.load();
      float shv = sh;
      void* args[] = {(void*)&x, (void*)&y, (void*)&rows, (void*)&cols, (void*)&ldx,
                      (void*)&ldy, (void*)&slice, (void*)&nst, (void*)&bad, (void*)&shv,
                      (void*)&dg};
      SK_CUDA(cudaLaunchKernelExC(&cfg, cluster_fn(mode), args));
    } else if (p.k3 == 7) {
      const GresWs w = gres_ws(p);
      char* blk = nullptr;
      if (user_ws) {
        blk = ws + 256;
        SK_CUDA(cudaMemsetAsync(blk, 0, w.total, s));
      } else {
        int dev = 0;
        SK_CUDA(cudaGetDevice(&dev));
        const int st = get_gres_block(dev, s, &blk);
        if (st) return st;
      }
      GresComm comm = {};
      comm.dst[0] = reinterpret_cast<unsigned long long*>(blk + w.slots);
      comm.ctl = reinterpret_cast<unsigned*>(blk + w.ctl);
      comm.shard_stride = 0;
      comm.world = 1;
      comm.rank0 = 0;
      comm.nvr = 1;
      comm.sys = 0;
      comm.spin_limit = g_gres_spins.load();
      // the library block: self-reset by the kernel; a caller's workspace is
      // cleared before every launch (above)
      comm.reset_words = user_ws ? 0ull : (kGresWsMax - w.slots) / 8;
      comm.reset_period = static_cast<unsigned>(gres_reset_period());
      int P = p.nseg, slice = p.seglen, nst = p.lag;
      SK_CUDA(launch_k(gres_fn(mode, p.glag, p.threads == kGresBlock, p.unal), dim3(static_cast<unsigned>(p.grid)),
                       dim3(p.threads), p.smem, s, true, x, y, rows, cols, ldx, ldy, P, slice, nst, comm,
                       bad, sh, g_gres_sleep.load(), g_gres_diag.load()));
    } else {
      SK_CUDA(launch_k(reinterpret_cast<const void*>(seg_fn<kSegNV>(mode)),
                       dim3(static_cast<unsigned>(p.grid)), dim3(p.threads), p.smem, s, nseg > 1,
                       x, y, rows, cols, ldx, ldy, nseg, seglen, cnt, part, bad, sh));
    }
    return SK_OK;
  }
  return launch_split(x, y, rows, cols, ldx, ldy, mode, p.vec, bad, ws, p.nch, true, nullptr,
                      nullptr, s);
}

int softmax_dev(const float* x, float* y, int64_t rows, int64_t cols, int64_t ldx, int64_t ldy,
                int mode, unsigned long long* bad, void* workspace, size_t ws_bytes,
                cudaStream_t s, bool bulk) {
  int st = check_common(x, y, rows, cols, ldx, ldy, mode);
  if (st) return st;
  if (rows == 0) return SK_OK;
  if (reinterpret_cast<const char*>(x) < reinterpret_cast<const char*>(y) + rows * ldy * 4 &&
      reinterpret_cast<const char*>(y) < reinterpret_cast<const char*>(x) + rows * ldx * 4)
    return arg_fail("x and y must not alias");
  int dev = 0;
  SK_CUDA(cudaGetDevice(&dev));
  Plan p;
  st = make_plan(rows, cols, ldx, ldy, reinterpret_cast<uint64_t>(x),
                 reinterpret_cast<uint64_t>(y), mode, dev, p, bulk);
  if (st) return st;
  const size_t need = plan_ws_bytes(p, rows);
  char* ws = static_cast<char*>(workspace);
  if (ws && ws_bytes < need) return arg_fail("workspace too small");
  if (!ws) {
    void* w = nullptr;
    st = get_ws(dev, s, need, &w);
    if (st) return st;
    ws = static_cast<char*>(w);
  }
  if (!bad) bad = reinterpret_cast<unsigned long long*>(ws);  // library flag at offset 0
  return launch_plan(p, x, y, rows, cols, ldx, ldy, mode, bad, ws, s, workspace != nullptr);
}

}  // namespace detail
}  // namespace sk

using namespace sk;
using namespace sk::detail;

extern "C" {

int sk_abi_version(void) { return SK_ABI_VERSION; }

const char* sk_status_string(int status) {
  switch (status) {
    case SK_OK: return "ok";
    case SK_ERR_ARGUMENT: return "invalid argument";
    case SK_ERR_NONFINITE: return "non-finite logits";
    case SK_ERR_CUDA: return "cuda error";
    case SK_ERR_RESOURCE: return "allocation failed";
    default: return "unknown status";
  }
}

const char* sk_last_error(void) { return g_last_error.c_str(); }

int sk_set_tuning(const char* key, int value) {
  if (!key) return SK_ERR_ARGUMENT;
  std::string k(key);
  if (k == "path") g_force_path = value;
  else if (k == "k1_lpr") g_k1_lpr = value;
  else if (k == "k1_nv") g_k1_nv = value;
  else if (k == "k1_u") g_k1_u = value;
  else if (k == "grid_mult") g_grid_mult = value;
  else if (k == "skip_max_shift") g_skip_max_shift = value;
  else if (k == "k1_pf") g_k1_pf = value;
  else if (k == "pdl") g_pdl = value;
  else if (k == "host_chunk_kb") g_host_chunk_kb = value;
  else if (k == "host_threads") g_host_threads = value;
  else if (k == "host_nt") g_host_nt = value;
  else if (k == "host_zero_copy") g_host_zero_copy = value;
  else if (k == "cluster_k3") g_cluster_k3 = value;
  else if (k == "cluster_size") g_cluster_size = value;
  else if (k == "vec8") g_vec8 = value;
  else if (k == "vec2_max") g_vec2_max = value;
  else if (k == "cluster_onex") g_cluster_onex = value;
  else if (k == "cluster_tpb") g_cluster_tpb = value;
  else if (k == "k3_impl") {
    if (value != 3 && value != 5) return arg_fail("k3_impl: 3 (K3g, then K3c) or 5 (K3c only)");
    g_k3_impl = value;
  }
  else if (k == "gres") g_gres = value;
  else if (k == "gres_p") g_gres_p = value;
  else if (k == "colshard_sys") g_colshard_sys = value;
  else if (k == "gres_st") g_gres_st = value;
  else if (k == "gres_diag") g_gres_diag = value;
  else if (k == "gres_sleep") g_gres_sleep = value;
  else if (k == "gres_split") g_gres_split = value;
  else if (k == "gres_lag") g_gres_lag = value;
  else if (k == "gres_epoch_reset") {
    if (value < 0) return arg_fail("gres_epoch_reset: launches between exchange-block resets (0 = default)");
    g_gres_epoch_reset = static_cast<unsigned long long>(value);
  }
  else if (k == "k1m") g_k1m = value;
  else if (k == "k1_fit") g_k1_fit = value;
  else if (k == "k1_threads") g_k1_threads = value;
  else if (k == "k1m_threads") g_k1m_threads = value;
  else if (k == "k1_wide32") g_k1_wide32 = value;
  else if (k == "k4_fuse_combine") g_k4_fuse_combine = value;
  else if (k == "latency_steps") g_latency_steps = value;
  else if (k == "coop_pdl") g_coop_pdl = value;
  else if (k == "k1m_wpr") g_k1m_wpr = value;
  else if (k == "k1m_nv") g_k1m_nv = value;
  else if (k == "k1m_max_cols") g_k1m_max = value > 0 ? value : 16384;
  else if (k == "gres_timeout_spins") g_gres_spins = value > 0 ? unsigned(value) : kGresSpinLimit;
  else return arg_fail("unknown tuning key " + k);
  return SK_OK;
}

size_t sk_softmax_workspace_bytes(int64_t rows, int64_t cols) {
  if (rows <= 0 || cols <= 0) return ws_layout(0, 0).total;
  const int64_t nseg = (cols + 512 - 1) / 512;  // smallest K3 segment
  const int64_t nch = (cols + kSplitChunk - 1) / kSplitChunk;
  const size_t gres_max = 256 + kGresWsMax;  // K3g control block at ws + 256
  return std::max({ws_layout(rows, nseg).total, ws_layout(rows, nch).total, gres_max});
}

int sk_softmax_f32(const float* x, float* y, int64_t rows, int64_t cols, int64_t ldx,
                   int64_t ldy, int mode, unsigned long long* bad_row, void* workspace,
                   size_t workspace_bytes, void* stream) {
  return softmax_dev(x, y, rows, cols, ldx, ldy, mode, bad_row, workspace, workspace_bytes,
                     static_cast<cudaStream_t>(stream));
}

int sk_describe_plan(int64_t rows, int64_t cols, int64_t ldx, int64_t ldy, uint64_t x_addr,
                     uint64_t y_addr, int device, char* buf, int buflen) {
  if (!buf || buflen < 1) return arg_fail("null buffer");
  int st = check_common(reinterpret_cast<const float*>(1), reinterpret_cast<const void*>(1),
                        rows, cols, ldx, ldy, 0);
  if (st) return st;
  Plan p;
  st = make_plan(rows, cols, ldx, ldy, x_addr, y_addr, 0, device, p);
  if (st) return st;
  if (p.kind == kPathK1m)
    snprintf(buf, buflen, "k1m vec=%d wpr=%d nv=%d threads=%d grid=%lld", p.k1m->vec,
             p.k1m->wpr, p.k1m->nv, p.threads, (long long)p.grid);
  else if (p.kind == kPathK1)
    snprintf(buf, buflen, "k1 vec=%d lpr=%d nv=%d u=%d pf=%d threads=%d grid=%lld", p.k1->vec,
             p.k1->lpr, p.k1->nv, p.k1->u, p.k1->pf, p.threads, (long long)p.grid);
  else if (p.kind == kPathSeg)
    snprintf(buf, buflen, "%s nseg=%d seglen=%d threads=%d smem=%zu chunk_rows=%lld stages=%d grid=%lld",
             p.k3 == 6 ? "k3_cluster"
             : p.k3 == 7 ? (p.unal ? "k3_gres_unal" : "k3_gres")
             : "k2_tma",
             p.nseg, p.seglen,
             p.threads, p.smem, (long long)p.chunk_rows, p.lag, (long long)p.grid);
  else
    snprintf(buf, buflen, "k4_split vec=%d nch=%d grid=%lld", p.vec ? 4 : 1, p.nch,
             (long long)p.grid);
  if (p.kind == kPathSeg && p.k3 == 7) {
    const size_t n = strlen(buf);
    if (n < size_t(buflen)) snprintf(buf + n, size_t(buflen) - n, " lag=%d", p.glag);
  }
  return SK_OK;
}

int sk_device_flag(int device, unsigned long long** flag) {
  if (!flag) return arg_fail("null output pointer");
  static std::mutex mu;
  static std::map<int, unsigned long long*> flags;
  std::lock_guard<std::mutex> g(mu);
  unsigned long long*& f = flags[device];
  if (!f) {
    int prev = 0;
    SK_CUDA(cudaGetDevice(&prev));
    SK_CUDA(cudaSetDevice(device));
    cudaError_t e = cudaMalloc(&f, sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMemset(f, 0xFF, sizeof(unsigned long long));  // SK_NO_BAD_ROW
    cudaSetDevice(prev);
    if (e != cudaSuccess) {
      f = nullptr;
      return cuda_fail(e, "sk_device_flag");
    }
  }
  *flag = f;
  return SK_OK;
}

int sk_flag_read(unsigned long long* flag, void* stream, int reset, unsigned long long* value) {
  if (!flag || !value) return arg_fail("null pointer");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  unsigned long long v = SK_NO_BAD_ROW;
  SK_CUDA(cudaMemcpyAsync(&v, flag, sizeof(v), cudaMemcpyDeviceToHost, s));
  SK_CUDA(cudaStreamSynchronize(s));
  if (reset && v != SK_NO_BAD_ROW) {
    SK_CUDA(cudaMemsetAsync(flag, 0xFF, sizeof(v), s));
    SK_CUDA(cudaStreamSynchronize(s));
  }
  *value = v;
  return SK_OK;
}

size_t sk_row_stats_workspace_bytes(int64_t rows, int64_t cols) {
  const int64_t nch = (cols + kSplitChunk - 1) / kSplitChunk;
  return ws_layout(std::max<int64_t>(rows, 0), nch).total;
}

int sk_row_stats_f32(const float* x, int64_t rows, int64_t cols, int64_t ldx, int mode,
                     float* row_max, double* row_sum, unsigned long long* bad_row,
                     void* workspace, size_t workspace_bytes, void* stream) {
  int st = check_common(x, row_max, rows, cols, ldx, ldx, mode);
  if (st) return st;
  if (rows == 0) return SK_OK;
  if (!row_sum) return arg_fail("null row_sum");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int dev = 0;
  SK_CUDA(cudaGetDevice(&dev));
  const int nch = static_cast<int>((cols + kSplitChunk - 1) / kSplitChunk);
  const WsLayout l = ws_layout(rows, nch);
  char* ws = static_cast<char*>(workspace);
  if (ws && workspace_bytes < l.total) return arg_fail("workspace too small");
  if (!ws) {
    void* w = nullptr;
    st = get_ws(dev, s, l.total, &w);
    if (st) return st;
    ws = static_cast<char*>(w);
  }
  if (!bad_row) bad_row = reinterpret_cast<unsigned long long*>(ws);
  return launch_split(x, nullptr, rows, cols, ldx, ldx, mode, false, bad_row, ws, nch, false,
                      row_max, row_sum, s);
}

int sk_rescale_sumexp(const float* local_max, const float* global_max, double* row_sum,
                      int64_t rows, void* stream) {
  if (rows < 0) return arg_fail("rows < 0");
  if (rows == 0) return SK_OK;
  if (!local_max || !global_max || !row_sum) return arg_fail("null buffer");
  SK_CUDA(launch_k(reinterpret_cast<const void*>(&k4_rescale),
                   dim3(static_cast<unsigned>((rows + 255) / 256)), dim3(256), 0,
                   static_cast<cudaStream_t>(stream), false, local_max, global_max, row_sum,
                   rows));
  return SK_OK;
}

int sk_normalize_f32(const float* x, float* y, int64_t rows, int64_t cols, int64_t ldx,
                     int64_t ldy, int mode, const float* row_max, const double* row_sum,
                     void* stream) {
  int st = check_common(x, y, rows, cols, ldx, ldy, mode);
  if (st) return st;
  if (rows == 0) return SK_OK;
  if (!row_max || !row_sum) return arg_fail("null row statistics");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int nch = static_cast<int>((cols + kSplitChunk - 1) / kSplitChunk);
  const unsigned g = static_cast<unsigned>(rows * nch);
  const bool v4 = (cols % 4 == 0) && (ldx % 4 == 0) && (ldy % 4 == 0) &&
                  (reinterpret_cast<uintptr_t>(x) % 16 == 0) &&
                  (reinterpret_cast<uintptr_t>(y) % 16 == 0);
  const void* norm;
  switch (mode) {
    case kClipAccurate:
      norm = v4 ? reinterpret_cast<const void*>(&k4_normalize<kClipAccurate, 4>)
                : reinterpret_cast<const void*>(&k4_normalize<kClipAccurate, 1>);
      break;
    case kAccurate:
      norm = v4 ? reinterpret_cast<const void*>(&k4_normalize<kAccurate, 4>)
                : reinterpret_cast<const void*>(&k4_normalize<kAccurate, 1>);
      break;
    default:
      norm = v4 ? reinterpret_cast<const void*>(&k4_normalize<kApprox, 4>)
                : reinterpret_cast<const void*>(&k4_normalize<kApprox, 1>);
  }
  SK_CUDA(launch_k(norm, dim3(g), dim3(kSplitThreads), 0, s, false, x, y, rows, cols, ldx, ldy,
                   nch, row_max, row_sum));
  return SK_OK;
}

}  // extern "C"
