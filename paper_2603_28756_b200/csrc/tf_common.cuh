// Shared host/device helpers for the tomoforge-b200 C-ABI library.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <string>

#include "tf_fft.cuh"

namespace tf {

// Error codes returned by every extern "C" entry point (include/tomoforge_b200.h).
enum : int { TF_OK = 0, TF_EARG = -1, TF_ECUDA = -2, TF_EUNSUPPORTED = -3 };

void set_error(const std::string& msg);
int fail_arg(const char* fmt, ...);
int check_cuda(cudaError_t e, const char* what);
int check_launch(const char* what);
int ensure_init();
int num_sms();

// Optional per-kernel CUDA-event timing (bench.py's roofline numbers): when
// enabled, launch sites bracket each kernel with events on its own stream.
struct KernelTimer {
  cudaEvent_t a = nullptr, b = nullptr;
  cudaStream_t st = nullptr;
  int slot = -1;
};
void timer_begin(KernelTimer& t, int slot, cudaStream_t st);
void timer_end(KernelTimer& t);

inline bool is_pow2(long long v) { return v > 0 && (v & (v - 1)) == 0; }

// opt a kernel into more than 48 KB of dynamic shared memory
template <typename K>
inline int prep_kernel(K kern, size_t smem) {
  if (smem > 48 * 1024) {
    return check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smem),
                      "cudaFuncSetAttribute");
  }
  return TF_OK;
}

}  // namespace tf

#define TF_TRY(expr)                 \
  do {                               \
    int _rc = (expr);                \
    if (_rc != ::tf::TF_OK) return _rc; \
  } while (0)
