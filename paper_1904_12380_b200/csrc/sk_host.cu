// sk_host.cu -- sk_softmax_f32_host: the reference-facing call on HOST
// buffers (kernels.softmax(Matrix2D), kernels.py:350-362) as a pipelined
// H2D -> kernel -> D2H over three streams, plus page-locked allocation.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include <emmintrin.h>

#include "sk_internal.h"

namespace sk {
namespace detail {

// ------------------------------------------------ pipelined host-buffer path
// Three streams (H2D copy engine, compute, D2H copy engine) over a ring of
// kRing device buffer pairs, ordered by events: chunk k's kernel waits for its
// H2D, its D2H waits for its kernel, and slot reuse waits for the kernel / D2H
// that last used the slot.  H2D of chunk k+1, compute of chunk k and D2H of
// chunk k-1 run concurrently, so a call costs ~max(H2D, D2H) + one chunk.
constexpr int kRing = 4;
struct HostCtx {
  std::mutex mu;
  bool init = false;
  cudaStream_t s_h2d = nullptr, s_comp = nullptr, s_d2h = nullptr;
  cudaEvent_t ev_h2d[kRing] = {}, ev_k[kRing] = {}, ev_d2h[kRing] = {};
  float* dx[kRing] = {};
  float* dy[kRing] = {};
  unsigned long long* dbad = nullptr;  // one bad-row flag per chunk
  unsigned long long* hbad = nullptr;  // pinned mirror
  int64_t flag_cap = 0;
  size_t cap_bytes = 0;
  float* pin_in[kRing] = {};   // page-locked staging (pageable caller buffers)
  float* pin_out[kRing] = {};
  size_t pin_bytes = 0;
};
std::mutex g_host_mu;
std::map<int, HostCtx*> g_host;
std::atomic<int> g_host_chunk_kb{0};  // 0: auto
std::atomic<int> g_host_zero_copy{0};  // K1/K2 rows read/write pinned host memory directly

// Device-visible address of a page-locked (cudaHostAlloc / registered) host
// buffer, or nullptr for pageable memory.
const void* mapped_device_ptr(const void* h) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, h) != cudaSuccess) {
    (void)cudaGetLastError();
    return nullptr;
  }
  if (a.type != cudaMemoryTypeHost || !a.devicePointer) return nullptr;
  return a.devicePointer;
}

// Ranges page-locked in place through sk_host_register (start -> bytes).  One
// cudaMemcpyAsync may not span two registrations (invalid argument).  The
// Python mirror registers one range per buffer (hostpin.py), but a C caller
// may register a buffer in adjacent pieces, so direct copies are cut at the
// range boundaries found here.
std::mutex g_reg_mu;
std::map<uintptr_t, size_t> g_reg;

// [p, p + bytes) as pieces that each lie inside one registered range; false
// when some byte is in none of the library's registrations.
bool reg_pieces(const void* p, size_t bytes, std::vector<std::pair<size_t, size_t>>* pieces) {
  std::lock_guard<std::mutex> g(g_reg_mu);
  uintptr_t cur = reinterpret_cast<uintptr_t>(p);
  const uintptr_t base = cur, end = cur + bytes;
  while (cur < end) {
    auto it = g_reg.upper_bound(cur);
    if (it == g_reg.begin()) return false;
    --it;
    if (cur >= it->first + it->second) return false;
    const uintptr_t next = std::min<uintptr_t>(end, it->first + it->second);
    if (pieces) pieces->emplace_back(size_t(cur - base), size_t(next - cur));
    cur = next;
  }
  return true;
}

// ------------------------------------------- host copy pool (pageable buffers)
// A drop-in caller hands over pageable numpy memory (the reference's
// alloc_matrix is np.zeros, tensor.py:90-103).  cudaMemcpyAsync from pageable
// memory is synchronous and goes through the driver's small bounce buffer, so
// the staged path below copies each chunk between the caller's buffer and a
// page-locked staging slot with this pool of persistent host threads (a
// memcpy split into page-aligned pieces), and the DMA engines only ever see
// page-locked memory.
std::atomic<int> g_host_threads{0};  // 0: auto (min(16, hardware threads))
std::atomic<int> g_host_nt{1};       // non-temporal stores in the staging copies

// dst[0, n) = src[0, n) with 16-B non-temporal stores: the destination is
// written once and read next by a DMA engine (staging slot) or by the caller
// much later (output), so skipping the read-for-ownership of every
// destination line cuts the host memory traffic of a copy from 3 to 2 passes.
void stream_copy(char* d, const char* s, size_t n) {
  size_t head = (16 - (reinterpret_cast<uintptr_t>(d) & 15)) & 15;
  if (head > n) head = n;
  std::memcpy(d, s, head);
  d += head;
  s += head;
  n -= head;
  const size_t blocks = n / 64;
  for (size_t i = 0; i < blocks; ++i, d += 64, s += 64) {
    const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s));
    const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + 16));
    const __m128i c = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + 32));
    const __m128i e = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + 48));
    _mm_stream_si128(reinterpret_cast<__m128i*>(d), a);
    _mm_stream_si128(reinterpret_cast<__m128i*>(d + 16), b);
    _mm_stream_si128(reinterpret_cast<__m128i*>(d + 32), c);
    _mm_stream_si128(reinterpret_cast<__m128i*>(d + 48), e);
  }
  _mm_sfence();
  std::memcpy(d, s, n % 64);
}
void piece_copy(void* dst, const void* src, size_t n) {
  if (g_host_nt.load(std::memory_order_relaxed) && n >= (size_t(64) << 10))
    stream_copy(static_cast<char*>(dst), static_cast<const char*>(src), n);
  else
    std::memcpy(dst, src, n);
}
class CopyPool {
 public:
  static CopyPool& get() {
    static CopyPool* p = new CopyPool();  // never destroyed: threads live with the process
    return *p;
  }
  // dst[0, bytes) = src[0, bytes) using up to n threads (the caller is one of them)
  void copy(void* dst, const void* src, size_t bytes) {
    int n = g_host_threads.load();
    if (n <= 0) n = std::min(16, std::max(1, static_cast<int>(std::thread::hardware_concurrency())));
    const size_t piece = std::max<size_t>(size_t(1) << 20, ((bytes / n) + 4095) / 4096 * 4096);
    const int parts = static_cast<int>(std::min<size_t>(n, (bytes + piece - 1) / piece));
    if (parts <= 1) {
      piece_copy(dst, src, bytes);
      return;
    }
    ensure(parts - 1);
    std::unique_lock<std::mutex> lk(mu_);
    job_ = [=](int i) {
      const size_t a = size_t(i) * piece, b = std::min(bytes, a + piece);
      if (a < b) piece_copy(static_cast<char*>(dst) + a, static_cast<const char*>(src) + a, b - a);
    };
    parts_ = parts;
    next_ = 1;  // part 0 is done by the caller
    pending_ = parts - 1;
    ++gen_;
    cv_.notify_all();
    lk.unlock();
    job_(0);
    lk.lock();
    done_.wait(lk, [&] { return pending_ == 0; });
  }

 private:
  void ensure(int n) {
    std::lock_guard<std::mutex> g(mu_);
    while (static_cast<int>(th_.size()) < n) th_.emplace_back([this] { loop(); });
  }
  void loop() {
    uint64_t seen = 0;
    std::unique_lock<std::mutex> lk(mu_);
    for (;;) {
      cv_.wait(lk, [&] { return gen_ != seen; });
      seen = gen_;
      while (next_ < parts_) {
        const int i = next_++;
        auto fn = job_;
        lk.unlock();
        fn(i);
        lk.lock();
        if (--pending_ == 0) done_.notify_all();
      }
    }
  }
  std::mutex mu_;
  std::condition_variable cv_, done_;
  std::vector<std::thread> th_;
  std::function<void(int)> job_;
  int parts_ = 0, next_ = 0, pending_ = 0;
  uint64_t gen_ = 0;
};

HostCtx* host_ctx(int dev) {
  std::lock_guard<std::mutex> g(g_host_mu);
  HostCtx*& c = g_host[dev];
  if (!c) c = new HostCtx();
  return c;
}

}  // namespace detail
}  // namespace sk

using namespace sk;
using namespace sk::detail;

extern "C" {

void* sk_alloc_pinned(size_t bytes) {
  void* p = nullptr;
  if (cudaHostAlloc(&p, bytes ? bytes : 1, cudaHostAllocPortable) != cudaSuccess) {
    g_last_error = "cudaHostAlloc failed";
    (void)cudaGetLastError();
    return nullptr;
  }
  return p;
}

void sk_free_pinned(void* p) {
  if (p) cudaFreeHost(p);
}

int sk_host_register(void* p, size_t bytes) {
  if (!p || !bytes) return arg_fail("host_register: empty range");
  if (mapped_device_ptr(p)) {
    g_last_error = "host_register: the range is already page-locked";
    return SK_ERR_CUDA;
  }
  if (cudaHostRegister(p, bytes, cudaHostRegisterPortable) != cudaSuccess) {
    g_last_error = std::string("cudaHostRegister failed: ") + cudaGetErrorString(cudaGetLastError());
    return SK_ERR_CUDA;
  }
  std::lock_guard<std::mutex> g(g_reg_mu);
  g_reg[reinterpret_cast<uintptr_t>(p)] = bytes;
  return SK_OK;
}

int sk_host_unregister(void* p) {
  if (!p) return arg_fail("host_unregister: null");
  {
    std::lock_guard<std::mutex> g(g_reg_mu);
    g_reg.erase(reinterpret_cast<uintptr_t>(p));
  }
  if (cudaHostUnregister(p) != cudaSuccess) {
    g_last_error = std::string("cudaHostUnregister failed: ") + cudaGetErrorString(cudaGetLastError());
    return SK_ERR_CUDA;
  }
  return SK_OK;
}

int sk_softmax_f32_host(const float* x_host, float* y_host, int64_t rows, int64_t cols,
                        int mode, int device, int64_t* bad_row_out) {
  if (bad_row_out) *bad_row_out = -1;
  int st = check_common(x_host, y_host, rows, cols, cols, cols, mode);
  if (st) return st;
  if (rows == 0) return SK_OK;
  SK_CUDA(cudaSetDevice(device));
  HostCtx* c = host_ctx(device);
  std::lock_guard<std::mutex> g(c->mu);
  if (!c->init) {
    SK_CUDA(cudaStreamCreateWithFlags(&c->s_h2d, cudaStreamNonBlocking));
    SK_CUDA(cudaStreamCreateWithFlags(&c->s_comp, cudaStreamNonBlocking));
    SK_CUDA(cudaStreamCreateWithFlags(&c->s_d2h, cudaStreamNonBlocking));
    for (int i = 0; i < kRing; ++i) {
      SK_CUDA(cudaEventCreateWithFlags(&c->ev_h2d[i], cudaEventDisableTiming));
      SK_CUDA(cudaEventCreateWithFlags(&c->ev_k[i], cudaEventDisableTiming));
      SK_CUDA(cudaEventCreateWithFlags(&c->ev_d2h[i], cudaEventDisableTiming));
    }
    c->init = true;
  }
  // Zero-copy: a row that fits one CTA (K1/K2) is read from and written to
  // pinned host memory directly by the kernel -- PCIe reads and (posted) writes
  // proceed concurrently inside one launch, with no staging copies, events or
  // chunk pipeline.  Long rows (K3/K4 re-read segments) keep the staged path.
  if (g_host_zero_copy.load() && cols <= kOneCtaRowMax) {
    const float* xd = static_cast<const float*>(mapped_device_ptr(x_host));
    float* yd = static_cast<float*>(const_cast<void*>(mapped_device_ptr(y_host)));
    if (xd && yd) {
      if (c->flag_cap < 1) {
        SK_CUDA(cudaMalloc(&c->dbad, 64 * sizeof(unsigned long long)));
        SK_CUDA(cudaMemset(c->dbad, 0xFF, 64 * sizeof(unsigned long long)));
        SK_CUDA(cudaMallocHost(&c->hbad, 64 * sizeof(unsigned long long)));
        c->flag_cap = 64;
      }
      st = softmax_dev(xd, yd, rows, cols, cols, cols, mode, c->dbad, nullptr, 0, c->s_comp);
      if (st) return st;
      SK_CUDA(cudaMemcpyAsync(c->hbad, c->dbad, sizeof(unsigned long long),
                              cudaMemcpyDeviceToHost, c->s_comp));
      SK_CUDA(cudaStreamSynchronize(c->s_comp));
      if (c->hbad[0] == SK_EXCHANGE_ABORTED) {
        SK_CUDA(cudaMemset(c->dbad, 0xFF, sizeof(unsigned long long)));
        g_last_error = "row-statistics exchange timed out";
        return SK_ERR_CUDA;
      }
      if (c->hbad[0] != SK_NO_BAD_ROW) {
        const int64_t row = static_cast<int64_t>(c->hbad[0]);
        SK_CUDA(cudaMemset(c->dbad, 0xFF, sizeof(unsigned long long)));
        if (bad_row_out) *bad_row_out = row;
        g_last_error = "non-finite logits in row " + std::to_string(row);
        return SK_ERR_NONFINITE;
      }
      return SK_OK;
    }
  }
  const int64_t row_bytes = cols * 4;
  const int64_t total = rows * row_bytes;
  // Chunk schedule: steady chunks of ~1/4 of the job (4..16 MiB; tunable),
  // ramped 1/8, 1/4, 1/2 at both ends: the first H2D and the last D2H are
  // the only transfers that cannot overlap the other direction, so they are
  // made small (each ramp chunk costs ~10 us of issue + DMA setup, paid once).
  // Whole rows.
  // (32 MiB steady chunks for jobs of >= 256 MiB: c5a 91.6 -> 95.1 GB/s,
  // profiles/r1b_e2e_probe.jsonl -- fewer per-chunk DMA setups, same overlap)
  const int64_t cap = total >= (int64_t(256) << 20) ? (int64_t(32) << 20) : (int64_t(16) << 20);
  int64_t chunk_bytes = std::min<int64_t>(std::max<int64_t>(total / 4, 4 << 20), cap);
  if (g_host_chunk_kb.load() > 0) chunk_bytes = int64_t(g_host_chunk_kb.load()) << 10;
  const int64_t big = std::min(rows, std::max<int64_t>(1, chunk_bytes / row_bytes));
  std::vector<int64_t> sched;  // rows per chunk
  {
    std::vector<int64_t> head;
    for (int64_t r = big / 8; r >= 1 && r < big; r *= 2) head.push_back(r);
    int64_t left = rows;
    std::vector<int64_t> tail;
    for (int64_t r : head) {  // ramp up at the start and down at the end
      if (left >= 2 * r + 2 * big && r * row_bytes >= (int64_t(512) << 10)) {
        sched.push_back(r);
        tail.push_back(r);
        left -= 2 * r;
      }
    }
    while (left > 0) {
      const int64_t r = std::min(big, left);
      sched.push_back(r);
      left -= r;
    }
    for (auto it = tail.rbegin(); it != tail.rend(); ++it) sched.push_back(*it);
  }
  const size_t need = size_t(big * row_bytes);
  if (c->cap_bytes < need) {
    SK_CUDA(cudaDeviceSynchronize());
    for (int i = 0; i < kRing; ++i) {
      if (c->dx[i]) cudaFree(c->dx[i]);
      if (c->dy[i]) cudaFree(c->dy[i]);
      c->dx[i] = c->dy[i] = nullptr;
    }
    c->cap_bytes = 0;
    for (int i = 0; i < kRing; ++i) {
      SK_CUDA(cudaMalloc(&c->dx[i], need));
      SK_CUDA(cudaMalloc(&c->dy[i], need));
    }
    c->cap_bytes = need;
  }
  const int64_t nchunks = static_cast<int64_t>(sched.size());
  if (c->flag_cap < nchunks) {
    SK_CUDA(cudaDeviceSynchronize());
    if (c->dbad) cudaFree(c->dbad);
    if (c->hbad) cudaFreeHost(c->hbad);
    c->dbad = nullptr;
    c->hbad = nullptr;
    c->flag_cap = 0;
    const int64_t cap = std::max<int64_t>(nchunks, 64);
    SK_CUDA(cudaMalloc(&c->dbad, cap * sizeof(unsigned long long)));
    SK_CUDA(cudaMemset(c->dbad, 0xFF, cap * sizeof(unsigned long long)));
    SK_CUDA(cudaMallocHost(&c->hbad, cap * sizeof(unsigned long long)));
    c->flag_cap = cap;
  }
  std::vector<int64_t> start(nchunks + 1, 0);
  for (int64_t k = 0; k < nchunks; ++k) start[k + 1] = start[k] + sched[k];
  // Pageable caller memory is staged through page-locked slots, decided per
  // chunk: a caller may have page-locked only part of a buffer (e.g. its
  // 2 MiB-aligned inside, which registers 4x faster), so the chunks at either
  // end can reach into pageable memory while every other chunk is DMA-ed
  // directly.
  auto locked = [](const float* p, size_t bytes) {
    if (reg_pieces(p, bytes, nullptr)) return true;
    // page-locked by someone else (cudaHostAlloc, the caller's own registration):
    // taken as one range when both ends are locked
    return !reg_pieces(p, 1, nullptr) && !reg_pieces(reinterpret_cast<const char*>(p) + bytes - 1, 1, nullptr) &&
           mapped_device_ptr(p) != nullptr &&
           mapped_device_ptr(reinterpret_cast<const char*>(p) + bytes - 1) != nullptr;
  };
  // one cudaMemcpyAsync per registered range the host side of a direct copy touches
  auto copy_direct = [](void* dst, const void* src, size_t bytes, cudaMemcpyKind kind,
                        const void* host, cudaStream_t s) -> cudaError_t {
    std::vector<std::pair<size_t, size_t>> pc;
    if (!reg_pieces(host, bytes, &pc) || pc.size() <= 1)
      return cudaMemcpyAsync(dst, src, bytes, kind, s);
    for (const auto& q : pc) {
      const cudaError_t e = cudaMemcpyAsync(static_cast<char*>(dst) + q.first,
                                            static_cast<const char*>(src) + q.first, q.second, kind, s);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  };
  std::vector<char> stage_in(nchunks), stage_out(nchunks);
  bool staged_in = false, staged_out = false;
  {
    // whole buffer locked (the common cases: cudaHostAlloc'd or fully pageable)
    const bool all_in = locked(x_host, size_t(total)), all_out = locked(y_host, size_t(total));
    const bool mid_in = mapped_device_ptr(x_host + (rows / 2) * cols) != nullptr;
    const bool mid_out = mapped_device_ptr(y_host + (rows / 2) * cols) != nullptr;
    for (int64_t k = 0; k < nchunks; ++k) {
      const size_t b = size_t(sched[k] * row_bytes);
      stage_in[k] = all_in ? 0 : (!mid_in || !locked(x_host + start[k] * cols, b));
      stage_out[k] = all_out ? 0 : (!mid_out || !locked(y_host + start[k] * cols, b));
      staged_in |= stage_in[k] != 0;
      staged_out |= stage_out[k] != 0;
    }
  }
  if ((staged_in || staged_out) && c->pin_bytes < need) {
    SK_CUDA(cudaDeviceSynchronize());
    for (int i = 0; i < kRing; ++i) {
      if (c->pin_in[i]) cudaFreeHost(c->pin_in[i]);
      if (c->pin_out[i]) cudaFreeHost(c->pin_out[i]);
      c->pin_in[i] = c->pin_out[i] = nullptr;
    }
    c->pin_bytes = 0;
    for (int i = 0; i < kRing; ++i) {
      SK_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&c->pin_in[i]), need, cudaHostAllocPortable));
      SK_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&c->pin_out[i]), need, cudaHostAllocPortable));
    }
    c->pin_bytes = need;
  }
  CopyPool& pool = CopyPool::get();
  // copy chunk j's staged output back into the caller's buffer once its D2H is done
  auto drain = [&](int64_t j) -> int {
    if (!stage_out[j]) return SK_OK;
    const int i = static_cast<int>(j % kRing);
    SK_CUDA(cudaEventSynchronize(c->ev_d2h[i]));
    pool.copy(y_host + start[j] * cols, c->pin_out[i], size_t(sched[j] * row_bytes));
    return SK_OK;
  };
  for (int64_t k = 0; k < nchunks; ++k) {
    const int i = static_cast<int>(k % kRing);
    const int64_t r0 = start[k];
    const int64_t nr = sched[k];
    const size_t bytes = size_t(nr * row_bytes);
    if (staged_out && k >= kRing) {  // slot i's staged output must be copied out first
      st = drain(k - kRing);
      if (st) return st;
    }
    // input slot free once the kernel that last read it is done
    if (k >= kRing) SK_CUDA(cudaStreamWaitEvent(c->s_h2d, c->ev_k[i], 0));
    const float* src = x_host + r0 * cols;
    // (placing the chunk at the host address's phase within a 4 KiB page on
    // the device side does not speed the DMA up: profiles/r2_hostpin_ab.jsonl)
    float* const dxk = c->dx[i];
    float* const dyk = c->dy[i];
    if (stage_in[k]) {
      // the staging slot is free once the H2D that last read it is done
      if (k >= kRing) SK_CUDA(cudaEventSynchronize(c->ev_h2d[i]));
      pool.copy(c->pin_in[i], src, bytes);
      src = c->pin_in[i];
    }
    SK_CUDA(copy_direct(dxk, src, bytes, cudaMemcpyHostToDevice, src, c->s_h2d));
    SK_CUDA(cudaEventRecord(c->ev_h2d[i], c->s_h2d));
    SK_CUDA(cudaStreamWaitEvent(c->s_comp, c->ev_h2d[i], 0));
    // output slot free once the D2H that last read it is done
    if (k >= kRing) SK_CUDA(cudaStreamWaitEvent(c->s_comp, c->ev_d2h[i], 0));
    // a chunk of this job: the job's throughput plan (never the latency path a
    // small standalone call would take), so every chunk keeps the whole job's bits
    const bool whole = nr == rows;
    st = softmax_dev(dxk, dyk, nr, cols, cols, cols, mode, c->dbad + k, nullptr, 0, c->s_comp,
                     !whole);
    if (st) return st;
    SK_CUDA(cudaEventRecord(c->ev_k[i], c->s_comp));
    SK_CUDA(cudaStreamWaitEvent(c->s_d2h, c->ev_k[i], 0));
    float* const dsty = stage_out[k] ? c->pin_out[i] : y_host + r0 * cols;
    SK_CUDA(copy_direct(dsty, dyk, bytes, cudaMemcpyDeviceToHost, dsty, c->s_d2h));
    SK_CUDA(cudaEventRecord(c->ev_d2h[i], c->s_d2h));
  }
  if (staged_out)
    for (int64_t j = std::max<int64_t>(0, nchunks - kRing); j < nchunks; ++j) {
      st = drain(j);
      if (st) return st;
    }
  // every chunk's non-finite flag in one small copy after the last kernel
  // (one DMA instead of one per chunk between the bulk transfers)
  SK_CUDA(cudaMemcpyAsync(c->hbad, c->dbad, size_t(nchunks) * sizeof(unsigned long long),
                          cudaMemcpyDeviceToHost, c->s_d2h));
  SK_CUDA(cudaStreamSynchronize(c->s_d2h));
  for (int64_t k = 0; k < nchunks; ++k) {
    if (c->hbad[k] == SK_EXCHANGE_ABORTED) {
      SK_CUDA(cudaMemset(c->dbad, 0xFF, nchunks * sizeof(unsigned long long)));
      g_last_error = "row-statistics exchange timed out";
      return SK_ERR_CUDA;
    }
    if (c->hbad[k] != SK_NO_BAD_ROW) {
      const int64_t row = start[k] + static_cast<int64_t>(c->hbad[k]);
      SK_CUDA(cudaMemset(c->dbad, 0xFF, nchunks * sizeof(unsigned long long)));
      if (bad_row_out) *bad_row_out = row;
      g_last_error = "non-finite logits in row " + std::to_string(row);
      return SK_ERR_NONFINITE;
    }
  }
  return SK_OK;
}

}  // extern "C"
