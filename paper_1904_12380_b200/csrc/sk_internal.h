// sk_internal.h -- internals shared by the C ABI translation units
// (sk_api.cu: planning + device entry points; sk_host.cu: host-buffer
// pipeline; sk_colshard.cu: fused column shard).  Not part of the ABI.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <string>

#include "../../include/softmax_b200.h"

namespace sk {
namespace detail {

extern thread_local std::string g_last_error;
int cuda_fail(cudaError_t e, const char* what);
int arg_fail(const std::string& msg);
#define SK_CUDA(call)                                   \
  do {                                                  \
    cudaError_t _e = (call);                            \
    if (_e != cudaSuccess) return cuda_fail(_e, #call); \
  } while (0)

struct DevInfo {
  int sms = 0;
  bool coop = false;
};
DevInfo dev_info(int dev);
float shift_scale();
int occupancy(const void* fn, int threads, size_t smem);
int check_common(const float* x, const void* y, int64_t rows, int64_t cols, int64_t ldx,
                 int64_t ldy, int mode);
// rows up to this many floats are processed by one CTA (K1 / K1m / K2)
inline constexpr int64_t kOneCtaRowMax = 8192;

// tuning knobs read outside sk_api.cu (sk_set_tuning writes them)
extern std::atomic<int> g_pdl, g_coop_pdl, g_gres_sleep, g_gres_diag, g_host_chunk_kb,
    g_host_zero_copy, g_host_threads, g_host_nt;
extern std::atomic<unsigned> g_gres_spins;
extern std::atomic<int> g_colshard_sys;  // test hook: .sys-scope slot accesses in the one-GPU emulation too

// Launch helper: cudaLaunchKernelExC with PDL (and cooperative) attributes.
template <typename... Args>
cudaError_t launch_k(const void* fn, dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                     bool coop, Args... args) {
  void* argv[] = {static_cast<void*>(&args)...};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  int n = 0;
  if (coop) {
    attr[n].id = cudaLaunchAttributeCooperative;
    attr[n].val.cooperative = 1;
    ++n;
  }
  if ((!coop || g_coop_pdl.load()) && g_pdl.load()) {
    attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  return cudaLaunchKernelExC(&cfg, fn, argv);
}


// the device-buffer softmax (plan + launch), as sk_softmax_f32.  bulk: the
// rows are one chunk of a larger pipelined job (the host-buffer path), so the
// plan is the throughput plan of the row length -- never the latency path a
// small standalone call would take -- and chunks keep the whole job's bits.
int softmax_dev(const float* x, float* y, int64_t rows, int64_t cols, int64_t ldx, int64_t ldy,
                int mode, unsigned long long* bad, void* workspace, size_t ws_bytes,
                cudaStream_t s, bool bulk = false);

// K3g planning and kernels (sk_api.cu), used by the fused column shard
struct GresChoice {
  int P = 0, st = 0, lag = 0, groups = 0;  // ring depth st >= lag + 2
  int64_t slice = 0;
  double score = 0.0;
};

GresChoice plan_gres(int64_t rows, int64_t cols, int mode, const DevInfo& di, int world, int nvr,
                     bool unal);
const void* gres_fn(int mode, int lag, bool split);
bool gres_split(int lag);
// exchange blocks are zeroed every gres_reset_period() launches (<= 2^22) so the
// slot tags' 23-bit epoch never wraps (sk_gres.cuh, gres_tag)
unsigned long long gres_reset_period();
// the K3g plan is modelled at this row count: plans (hence bits) depend on C only
inline constexpr int64_t kGresPlanRows = 2048;

}  // namespace detail
}  // namespace sk
