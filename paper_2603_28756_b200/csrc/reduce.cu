// Deterministic fp64 reductions of fp32 products (objective terms, norms).
//
// Fixed grid (2 x SMs blocks) -> per-block fp64 partials -> one-block final
// sum: the summation order depends only on n, so results are bitwise
// reproducible run to run (the reference asserts bitwise determinism,
// tests/test_solver.py:168-179).
#include "tf_common.cuh"

namespace tf {

constexpr int RED_THREADS = 256;

template <int NT>
__device__ __forceinline__ double block_sum(double v, double* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x < 32) {
    r = threadIdx.x < NT / 32 ? sh[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) r += __shfl_down_sync(0xffffffffu, r, o);
  }
  return r;  // valid in thread 0
}

// partial[b*2 + {0,1}] = sum x*a, sum x*b over block b's grid-stride share
__global__ void __launch_bounds__(RED_THREADS)
k_dot2_partial(const float* __restrict__ x, const float* __restrict__ a,
               const float* __restrict__ b, long long n, double* __restrict__ partial) {
  __shared__ double sh[RED_THREADS / 32];
  double s0 = 0.0, s1 = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride) {
    const float xv = x[i];
    s0 += (double)xv * (double)a[i];
    if (b) s1 += (double)xv * (double)b[i];
  }
  const double r0 = block_sum<RED_THREADS>(s0, sh);
  const double r1 = block_sum<RED_THREADS>(s1, sh);
  if (threadIdx.x == 0) {
    partial[2 * blockIdx.x] = r0;
    partial[2 * blockIdx.x + 1] = r1;
  }
}

// out[j] = sum_b partial[b*nv + j]
__global__ void __launch_bounds__(RED_THREADS)
k_final_sum(const double* __restrict__ partial, int nblocks, int nv, double* __restrict__ out) {
  __shared__ double sh[RED_THREADS / 32];
  for (int j = 0; j < nv; ++j) {
    double s = 0.0;
    for (int b = threadIdx.x; b < nblocks; b += blockDim.x) s += partial[(long long)b * nv + j];
    const double r = block_sum<RED_THREADS>(s, sh);
    if (threadIdx.x == 0) out[j] = r;
  }
}

int reduce_blocks() { return 2 * num_sms(); }

int dot2(const float* x, const float* a, const float* b, long long n, double* out, double* ws,
         cudaStream_t st) {
  const int nb = reduce_blocks();
  k_dot2_partial<<<nb, RED_THREADS, 0, st>>>(x, a, b, n, ws);
  TF_TRY(check_launch("k_dot2_partial"));
  k_final_sum<<<1, RED_THREADS, 0, st>>>(ws, nb, 2, out);
  return check_launch("k_final_sum");
}

}  // namespace tf
