// sk_colshard.cu -- the fused column-sharded softmax: K3g (sk_gres.cuh) with
// its row-statistics exchange spanning GPUs through peer-mapped exchange
// blocks (cudaIpc over NVLink), and the single-GPU all-ranks emulation.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>

#include "sk_gres.cuh"
#include "sk_internal.h"

namespace sk {
namespace detail {

// ------------------------------------------------ fused column shard (K3g)
// Every rank holds a [rows, cols] column shard and one exchange block:
// [0, 256) ctl words (epoch, finished CTAs, abort) | [256, ...) slot arrays
// [2][groups][2L+2][world*P] x 16 B.  Rank r's K3g CTAs store their row pairs
// into EVERY rank's block (peer pointers over NVLink) and poll only their
// own, so the per-row (max, sum) all-reduce of the column shard happens inside
// the kernel, overlapped with the streaming -- no NCCL call on the data path.
constexpr size_t kXBlockBytes = size_t(2) << 20;
constexpr size_t kXSlots = 256;

// Cross-GPU blocks (peers in other processes write into them) are reset by
// their owner through sk_xchg_reset with every rank quiescent
// (sharding.FusedColumnShard does it every gres_reset_period() calls between
// two barriers); this counts launches per owned block and refuses one past
// the period rather than risk a wrapped epoch.  Blocks no other process
// writes (world 1, emulation) are reset by the kernel itself
// (GresComm::reset_words), CUDA-graph replays included.
std::mutex g_xchg_mu;
std::map<const void*, unsigned long long> g_xchg_launches;

int colshard_launch(const float* x, float* y, int64_t rows, int64_t cols, int64_t ldx,
                    int64_t ldy, int mode, int rank, int world, int nvr, void* const* blocks,
                    unsigned long long* bad, cudaStream_t s, char* desc, int desc_len) {
  if (world < 1 || world > kGresMaxWorld) return arg_fail("world must be 1..8");
  if (nvr != 1 && nvr != world) return arg_fail("bad virtual rank count");
  if (rank < 0 || rank >= world) return arg_fail("rank out of range");
  if (rows < 0 || cols < 1 || ldx < cols || ldy < cols) return arg_fail("bad shard shape");
  if (mode < 0 || mode > 2) return arg_fail("mode must be SK_MODE_CLIPPED/EXACT/APPROX");
  if (!blocks) return arg_fail("null exchange blocks");
  for (int r = 0; r < world; ++r)
    if (!blocks[r]) return arg_fail("null exchange block");
  const bool aligned = cols % 4 == 0 && ldx % 4 == 0 && ldy % 4 == 0 &&
                       reinterpret_cast<uintptr_t>(x) % 16 == 0 &&
                       reinterpret_cast<uintptr_t>(y) % 16 == 0;
  if (!desc && rows > 0 && (!x || !y)) return arg_fail("null buffer");
  if (!desc && !aligned) return arg_fail("fused column shard needs cols % 4 == 0 and 16-B aligned rows");
  int dev = 0;
  SK_CUDA(cudaGetDevice(&dev));
  const DevInfo di = dev_info(dev);
  if (!di.coop) return arg_fail("device cannot co-schedule the fused column shard");
  const GresChoice gc = plan_gres(kGresPlanRows, cols, mode, di, world, nvr, false);
  if (gc.P == 0) return arg_fail("shard row too long for the fused column shard (use the split path)");
  const bool split = gres_split(gc.lag);
  const int lag = gc.lag;
  const size_t need = kXSlots + 2 * size_t(gc.groups) * gres_slot_sets(lag) * world * gc.P * 16;
  if (need > kXBlockBytes) return arg_fail("exchange block too small for this plan");
  if (desc) {
    snprintf(desc, desc_len, "k3_gres_colshard world=%d nvr=%d nseg=%d seglen=%lld stages=%d lag=%d groups=%d threads=%d",
             world, nvr, gc.P, (long long)gc.slice, gc.st, gc.lag, gc.groups, split ? kGresBlock : kGresThreads);
    return SK_OK;
  }
  if (rows == 0) return SK_OK;
  const bool cross_gpu = world > 1 && nvr == 1;
  if (cross_gpu) {
    std::lock_guard<std::mutex> g(g_xchg_mu);
    unsigned long long& n = g_xchg_launches[blocks[rank]];
    const unsigned long long period = gres_reset_period();
    if (n >= period)
      return arg_fail("exchange block needs sk_xchg_reset: " + std::to_string(n) +
                      " launches since the last reset (limit " + std::to_string(period) + ")");
    ++n;
  }
  GresComm comm = {};
  for (int r = 0; r < world; ++r)
    comm.dst[r] = reinterpret_cast<unsigned long long*>(static_cast<char*>(blocks[r]) + kXSlots);
  comm.ctl = reinterpret_cast<unsigned*>(blocks[nvr == 1 ? rank : 0]);
  comm.shard_stride = nvr == 1 ? 0 : cols;
  comm.world = world;
  comm.rank0 = nvr == 1 ? rank : 0;
  comm.nvr = nvr;
  // peers are other GPUs (or the test hook asks the emulation for the same
  // st / ld.relaxed.sys slot accesses the cross-GPU launch uses)
  comm.sys = (world > 1 && (nvr == 1 || g_colshard_sys.load())) ? 1 : 0;
  comm.spin_limit = g_gres_spins.load();
  comm.reset_words = cross_gpu ? 0ull : (kXBlockBytes - kXSlots) / 8;
  comm.reset_period = static_cast<unsigned>(gres_reset_period());
  const size_t smem = size_t(gc.st) * gc.slice * sizeof(float);
  int P = gc.P, slice = static_cast<int>(gc.slice), nst = gc.st;
  const int grid = gc.groups * gc.P * nvr;
  SK_CUDA(launch_k(gres_fn(mode, gc.lag, split), dim3(static_cast<unsigned>(grid)),
                   dim3(split ? kGresBlock : kGresThreads), smem, s, true, x, y, rows, cols, ldx,
                   ldy, P, slice, nst, comm, bad, shift_scale(), g_gres_sleep.load(),
                   g_gres_diag.load()));
  return SK_OK;
}

}  // namespace detail
}  // namespace sk

using namespace sk;
using namespace sk::detail;

extern "C" {

size_t sk_xchg_block_bytes(void) { return kXBlockBytes; }

int sk_xchg_alloc(int device, void** block) {
  if (!block) return arg_fail("null output pointer");
  int prev = 0;
  SK_CUDA(cudaGetDevice(&prev));
  SK_CUDA(cudaSetDevice(device));
  void* b = nullptr;
  cudaError_t e = cudaMalloc(&b, kXBlockBytes);  // plain cudaMalloc: IPC-exportable
  if (e == cudaSuccess) e = cudaMemset(b, 0, kXBlockBytes);
  cudaSetDevice(prev);
  if (e != cudaSuccess) return cuda_fail(e, "sk_xchg_alloc");
  *block = b;
  return SK_OK;
}

int sk_xchg_free(void* block) {
  if (block) {
    {
      std::lock_guard<std::mutex> g(g_xchg_mu);
      g_xchg_launches.erase(block);
    }
    SK_CUDA(cudaFree(block));
  }
  return SK_OK;
}

int sk_xchg_reset(void* block, void* stream) {
  if (!block) return arg_fail("null exchange block");
  SK_CUDA(cudaMemsetAsync(block, 0, kXBlockBytes, static_cast<cudaStream_t>(stream)));
  std::lock_guard<std::mutex> g(g_xchg_mu);
  g_xchg_launches[block] = 0;
  return SK_OK;
}

unsigned long long sk_xchg_reset_period(void) { return gres_reset_period(); }

int sk_ipc_handle(const void* dev_ptr, void* handle) {
  if (!dev_ptr || !handle) return arg_fail("null pointer");
  cudaIpcMemHandle_t h;
  SK_CUDA(cudaIpcGetMemHandle(&h, const_cast<void*>(dev_ptr)));
  std::memcpy(handle, &h, sizeof(h));
  return SK_OK;
}

int sk_ipc_open(const void* handle, void** dev_ptr) {
  if (!handle || !dev_ptr) return arg_fail("null pointer");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  SK_CUDA(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return SK_OK;
}

int sk_ipc_close(void* dev_ptr) {
  if (dev_ptr) SK_CUDA(cudaIpcCloseMemHandle(dev_ptr));
  return SK_OK;
}

int sk_colshard_softmax_f32(const float* x, float* y, int64_t rows, int64_t cols, int64_t ldx,
                            int64_t ldy, int mode, int rank, int world, void* const* blocks,
                            unsigned long long* bad_row, void* stream) {
  if (!bad_row) return arg_fail("bad_row flag required");
  return colshard_launch(x, y, rows, cols, ldx, ldy, mode, rank, world, 1, blocks, bad_row,
                         static_cast<cudaStream_t>(stream), nullptr, 0);
}

int sk_colshard_emulate_f32(const float* x, float* y, int64_t rows, int64_t cols, int64_t ldx,
                            int64_t ldy, int mode, int world, void* const* blocks,
                            unsigned long long* bad_row, void* stream) {
  if (!bad_row) return arg_fail("bad_row flag required");
  if (world < 1 || cols % world) return arg_fail("cols must split evenly over world");
  return colshard_launch(x, y, rows, cols / world, ldx, ldy, mode, 0, world, world, blocks,
                         bad_row, static_cast<cudaStream_t>(stream), nullptr, 0);
}

int sk_describe_colshard_plan(int64_t rows, int64_t cols, int world, int emulate, int device,
                              char* buf, int buflen) {
  if (!buf || buflen < 1) return arg_fail("null buffer");
  int prev = 0;
  SK_CUDA(cudaGetDevice(&prev));
  SK_CUDA(cudaSetDevice(device));
  void* fake[kGresMaxWorld];
  for (auto& f : fake) f = reinterpret_cast<void*>(256);
  const int st = colshard_launch(nullptr, nullptr, rows, cols, cols, cols, 0, 0, world,
                                 emulate ? world : 1, fake, nullptr, nullptr, buf, buflen);
  cudaSetDevice(prev);
  return st;
}

}  // extern "C"
