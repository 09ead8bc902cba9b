// fastbind.cpp -- the default gemm_f16 call from torch tensors with the fewest host steps:
// argument marshalling only (dtypes, device, row-major strides, torch's current stream), then
// the library's C-ABI entry point gemm_f16, whose address the Python binding hands over once
// (set_entry).  Anything unusual is declined (-1) and the Python general path handles the call
// and raises the precise error; a non-zero status is returned for Python to raise GemmError.
// Built in-tree by paper_2108_13191_b200/_build.py (build_fastbind); the ctypes path in
// __init__.py is used when this module is absent.  No arithmetic of the method lives here.
#include <torch/extension.h>
#include <ATen/cuda/CUDAContext.h>
#include <c10/cuda/CUDAFunctions.h>
#include <cstdint>
#include <cstring>
#include "../../include/gemm_f16.h"   // gemm_options_t (the C ABI's plain-C struct)

namespace {

using GemmFn = int (*)(int64_t, int64_t, int64_t, const void*, int64_t, const void*, int64_t, void*, int64_t, int,
                       void*);
using GemmExFn = int (*)(int64_t, int64_t, int64_t, const void*, int64_t, const void*, int64_t, void*, int64_t, int,
                         void*, const gemm_options_t*);
GemmFn g_gemm = nullptr;
GemmExFn g_gemm_ex = nullptr;

void set_entry(int64_t addr) { g_gemm = reinterpret_cast<GemmFn>(static_cast<intptr_t>(addr)); }
void set_entry_ex(int64_t addr) { g_gemm_ex = reinterpret_cast<GemmExFn>(static_cast<intptr_t>(addr)); }

// shared checks of both entry points: -1 = decline (the Python path handles it), else acc type
int check_common(const at::Tensor& A, const at::Tensor& B, const at::Tensor& C, bool allow_bf16) {
  const auto at_ = A.scalar_type();
  if (!(at_ == at::kHalf || (allow_bf16 && at_ == at::kBFloat16)) || B.scalar_type() != at_) return -1;
  const auto ct = C.scalar_type();
  const int acc = ct == at::kFloat ? 0 : (ct == at::kHalf ? 1 : -1);
  if (acc < 0) return -1;
  if (!C.is_cuda() || !A.is_cuda() || !B.is_cuda()) return -1;
  const auto dev = C.get_device();
  if (A.get_device() != dev || B.get_device() != dev || dev != c10::cuda::current_device()) return -1;
  if (A.dim() != 2 || B.dim() != 2 || C.dim() != 2) return -1;
  const int64_t M = A.size(0), K = A.size(1), N = B.size(1);
  if (B.size(0) != K || C.size(0) != M || C.size(1) != N || M < 2 || N < 2 || K < 2) return -1;
  if (A.stride(1) != 1 || B.stride(1) != 1 || C.stride(1) != 1) return -1;
  return acc;
}

int64_t gemm_options(const at::Tensor& A, const at::Tensor& B, const at::Tensor& C, int64_t config, int64_t beta0,
                     int64_t relu, const c10::optional<at::Tensor>& bias);

int64_t gemm_default(const at::Tensor& A, const at::Tensor& B, const at::Tensor& C) {
  if (g_gemm == nullptr) return -1;
  if (A.scalar_type() == at::kBFloat16) return gemm_options(A, B, C, 0, 0, 0, c10::nullopt);   // (in_type BF16)
  const int acc = check_common(A, B, C, false);
  if (acc < 0) return -1;
  cudaStream_t s = at::cuda::getCurrentCUDAStream(C.get_device()).stream();
  return g_gemm(A.size(0), B.size(1), A.size(1), A.data_ptr(), A.stride(0), B.data_ptr(), B.stride(0), C.data_ptr(),
                C.stride(0), acc, static_cast<void*>(s));
}

// the common user options (configuration, beta = 0, ReLU, a bias vector; BF16 inputs follow A's
// dtype); every other gemm_options_t field stays 0 (= default).  bias: an undefined tensor = none
int64_t gemm_options(const at::Tensor& A, const at::Tensor& B, const at::Tensor& C, int64_t config, int64_t beta0,
                     int64_t relu, const c10::optional<at::Tensor>& bias) {
  if (g_gemm_ex == nullptr) return -1;
  const int acc = check_common(A, B, C, true);
  if (acc < 0) return -1;
  gemm_options_t o;
  std::memset(&o, 0, sizeof(o));
  o.config = static_cast<int>(config);
  o.in_type = A.scalar_type() == at::kBFloat16 ? GEMM_IN_BF16 : GEMM_IN_F16;
  o.beta0 = static_cast<int>(beta0);
  o.relu = static_cast<int>(relu);
  if (bias.has_value() && bias->defined()) {
    const at::Tensor& b = *bias;
    if (b.scalar_type() != at::kFloat || b.dim() != 1 || b.numel() != B.size(1) || !b.is_cuda() ||
        b.get_device() != C.get_device() || (b.numel() > 1 && b.stride(0) != 1))
      return -1;
    o.bias = b.data_ptr();
  }
  cudaStream_t s = at::cuda::getCurrentCUDAStream(C.get_device()).stream();
  return g_gemm_ex(A.size(0), B.size(1), A.size(1), A.data_ptr(), A.stride(0), B.data_ptr(), B.stride(0),
                   C.data_ptr(), C.stride(0), acc, static_cast<void*>(s), &o);
}

}  // namespace

PYBIND11_MODULE(TORCH_EXTENSION_NAME, m) {
  m.def("set_entry", &set_entry, "address of the library's gemm_f16");
  m.def("set_entry_ex", &set_entry_ex, "address of the library's gemm_f16_ex");
  m.def("gemm_default", &gemm_default, "C += A @ B (default options); -1 = declined, else the gemm_status_t");
  m.def("gemm_options", &gemm_options, "C <- relu?(beta C + A @ B + bias) with a configuration; -1 = declined");
}
