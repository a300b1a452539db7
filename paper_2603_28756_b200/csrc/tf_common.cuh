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

// M = 5Q FFT sides (toeplitz5.cu): Toeplitz apply and PSF build
bool is_side5(int M);
int toeplitz_apply5(const float* x, float* out, const float* aux, float alpha, float beta,
                    long long nslices, int n, int M, const void* PQ, const float* Bi, bool flip,
                    void* ws, size_t ws_bytes, cudaStream_t st);
int psf_build5(int n, int M, const double* cs, int n_angles, int nd, void* PQ, float* Bi,
               void* ws, cudaStream_t st);
// K6 lag kernels on the M x M grid (toeplitz.cu)
int psf_lags_launch(float* lags, int n, int M, const double* cs, int n_angles, int nd,
                    cudaStream_t st);

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
