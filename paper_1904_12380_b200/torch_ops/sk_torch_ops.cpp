// sk_torch_ops.cpp -- torch.ops.softmax_b200.* (TORCH_LIBRARY) over the C ABI.
//
// The op surface SURVEY.md §8(b).2 asks for, so the kernels compose with other
// torch code (current CUDA stream, CUDA graphs, torch.compile graphs) without
// the Python wrapper.  Every op is a thin launcher: argument checks
// (TORCH_CHECK), then the C entry point of libsoftmax_b200.so on the current
// stream; no torch types cross the C ABI.  Reference interface each follows:
//   softmax_fwd / softmax_fwd_out   kernels.softmax, kernels.py:350-362
//                                   (clip = variant is REFERENCE_CLIPPED)
//   row_max / row_sumexp / normalize_   RowStats pieces, kernels.py:108-112,
//                                   272-276 (the column-shard building blocks)
// Non-finite rows (and a timed-out row-statistics exchange) are recorded in
// the library's per-device flag (sk_device_flag) -- the flag the Python
// wrappers use too -- because the ops are asynchronous;
// kernels.check_device_flag() raises NumericDomainError / SoftmaxKitError
// for them.
#include <ATen/ATen.h>
#include <c10/cuda/CUDAGuard.h>
#include <c10/cuda/CUDAStream.h>
#include <torch/library.h>

#include "softmax_b200.h"

namespace {

void check_status(int st, const char* what) {
  TORCH_CHECK(st == SK_OK, what, ": ", sk_status_string(st), ": ", sk_last_error());
}

void check_matrix(const at::Tensor& x, const char* name) {
  TORCH_CHECK(x.is_cuda(), name, " must be a CUDA tensor");
  TORCH_CHECK(x.scalar_type() == at::kFloat, name, " must be float32");
  TORCH_CHECK(x.dim() == 2, name, " must be 2-D [rows, cols]");
  TORCH_CHECK(x.size(1) >= 1, name, " needs cols >= 1");
  TORCH_CHECK(x.stride(1) == 1, name, " rows must be contiguous (stride(1) == 1)");
}

int64_t pitch(const at::Tensor& x) { return x.size(0) > 1 ? x.stride(0) : x.size(1); }

void* stream_of(const at::Tensor& x) {
  return static_cast<void*>(c10::cuda::getCurrentCUDAStream(x.device().index()).stream());
}

unsigned long long* flag_of(const at::Tensor& x) {
  unsigned long long* f = nullptr;
  check_status(sk_device_flag(x.device().index(), &f), "device_flag");
  return f;
}

void softmax_fwd_out(const at::Tensor& x, at::Tensor& y, bool clip) {
  check_matrix(x, "x");
  check_matrix(y, "y");
  TORCH_CHECK(x.sizes() == y.sizes(), "x and y must have the same shape");
  TORCH_CHECK(x.device() == y.device(), "x and y must be on the same device");
  c10::cuda::CUDAGuard g(x.device());
  if (x.size(0) == 0) return;
  check_status(sk_softmax_f32(x.data_ptr<float>(), y.data_ptr<float>(), x.size(0), x.size(1),
                              pitch(x), pitch(y), clip ? SK_MODE_CLIPPED : SK_MODE_EXACT,
                              flag_of(x), nullptr, 0, stream_of(x)),
               "softmax_fwd");
}

at::Tensor softmax_fwd(const at::Tensor& x, bool clip) {
  check_matrix(x, "x");
  at::Tensor y = at::empty({x.size(0), x.size(1)}, x.options());
  softmax_fwd_out(x, y, clip);
  return y;
}

// local (max, sum exp(clip(x - max))) -- the stats half of the K4 split
std::tuple<at::Tensor, at::Tensor> stats(const at::Tensor& x, bool clip) {
  check_matrix(x, "x");
  c10::cuda::CUDAGuard g(x.device());
  at::Tensor m = at::empty({x.size(0)}, x.options());
  at::Tensor s = at::empty({x.size(0)}, x.options().dtype(at::kDouble));
  if (x.size(0) > 0)
    check_status(sk_row_stats_f32(x.data_ptr<float>(), x.size(0), x.size(1), pitch(x),
                                  clip ? SK_MODE_CLIPPED : SK_MODE_EXACT, m.data_ptr<float>(),
                                  s.data_ptr<double>(), flag_of(x), nullptr, 0, stream_of(x)),
                 "row_stats");
  return {m, s};
}

at::Tensor row_max(const at::Tensor& x) { return std::get<0>(stats(x, true)); }

// sum_c exp(clip(x[r,c] - gmax[r])) in f64, as (local sum) * exp(local max - gmax)
at::Tensor row_sumexp(const at::Tensor& x, const at::Tensor& gmax, bool clip) {
  TORCH_CHECK(gmax.is_cuda() && gmax.scalar_type() == at::kFloat && gmax.dim() == 1 &&
                  gmax.size(0) == x.size(0) && gmax.is_contiguous(),
              "gmax must be a contiguous CUDA float32 [rows] tensor");
  auto [m, s] = stats(x, clip);
  c10::cuda::CUDAGuard g(x.device());
  if (x.size(0) > 0)
    check_status(sk_rescale_sumexp(m.data_ptr<float>(), gmax.data_ptr<float>(),
                                   s.data_ptr<double>(), x.size(0), stream_of(x)),
                 "row_sumexp");
  return s;
}

void normalize_(const at::Tensor& x, const at::Tensor& gmax, const at::Tensor& gsum,
                at::Tensor& y, bool clip) {
  check_matrix(x, "x");
  check_matrix(y, "y");
  TORCH_CHECK(x.sizes() == y.sizes(), "x and y must have the same shape");
  TORCH_CHECK(gmax.is_cuda() && gmax.scalar_type() == at::kFloat && gmax.dim() == 1 &&
                  gmax.size(0) == x.size(0) && gmax.is_contiguous(),
              "gmax must be a contiguous CUDA float32 [rows] tensor");
  TORCH_CHECK(gsum.is_cuda() && gsum.scalar_type() == at::kDouble && gsum.dim() == 1 &&
                  gsum.size(0) == x.size(0) && gsum.is_contiguous(),
              "gsum must be a contiguous CUDA float64 [rows] tensor");
  c10::cuda::CUDAGuard g(x.device());
  if (x.size(0) == 0) return;
  check_status(sk_normalize_f32(x.data_ptr<float>(), y.data_ptr<float>(), x.size(0), x.size(1),
                                pitch(x), pitch(y), clip ? SK_MODE_CLIPPED : SK_MODE_EXACT,
                                gmax.data_ptr<float>(), gsum.data_ptr<double>(), stream_of(x)),
               "normalize_");
}

}  // namespace

TORCH_LIBRARY(softmax_b200, m) {
  m.def("softmax_fwd(Tensor x, bool clip) -> Tensor");
  m.def("softmax_fwd_out(Tensor x, Tensor(a!) y, bool clip) -> ()");
  m.def("row_max(Tensor x) -> Tensor");
  m.def("row_sumexp(Tensor x, Tensor gmax, bool clip) -> Tensor");
  m.def("normalize_(Tensor x, Tensor gmax, Tensor gsum, Tensor(a!) y, bool clip) -> ()");
}

TORCH_LIBRARY_IMPL(softmax_b200, CUDA, m) {
  m.impl("softmax_fwd", &softmax_fwd);
  m.impl("softmax_fwd_out", &softmax_fwd_out);
  m.impl("row_max", &row_max);
  m.impl("row_sumexp", &row_sumexp);
  m.impl("normalize_", &normalize_);
}
