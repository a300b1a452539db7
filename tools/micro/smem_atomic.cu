// Shared-memory accumulation throughput on sm_100a, for the K7 design choice
// (DESIGN.md §5): fp32 atomicAdd to shared memory compiles to a CAS spin loop
// (ATOMS.CAST.SPIN), int32 atomicAdd to a native ATOMS.ADD.  Each warp adds a
// 7 x 7 Kaiser-Bessel-like window of 49 contributions per "sample" into a 64 x 64
// smem tile, windows of consecutive lanes overlapping as on a polar trajectory
// (lane l's window starts at column (base + l) % 58: neighbouring lanes hit
// neighbouring cells), or spread out (lane l at column (base + 7 l) % 58).
// Reports G adds/s per GPU.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>  // 0: fp32 atomicAdd, 1: int32 atomicAdd, 2: fp32 plain add (racy, bound)
__global__ void k(float* out, int iters, int spread) {
  __shared__ float tile[64 * 64];
  for (int i = threadIdx.x; i < 64 * 64; i += blockDim.x) tile[i] = 0.f;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float w = 1e-3f * (lane + 1);
  for (int it = 0; it < iters; ++it) {
    const int base = it * 3 + warp * 5;
    const int a0 = spread ? (base + 7 * lane) % 58 : (base + lane) % 58;
    const int b0 = (base / 7 + warp * 9) % 58;
#pragma unroll
    for (int u = 0; u < 7; ++u)
#pragma unroll
      for (int t = 0; t < 7; ++t) {
        float* p = &tile[(b0 + u) * 64 + a0 + t];
        if constexpr (MODE == 0) atomicAdd(p, w);
        else if constexpr (MODE == 1) atomicAdd(reinterpret_cast<int*>(p), 3);
        else *p += w;
      }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 64 * 64; i += blockDim.x) out[blockIdx.x * 4096 + i] = tile[i];
}

template <int MODE>
float run(float* out, int blocks, int iters, int spread) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k<MODE><<<blocks, 256>>>(out, iters, spread);
  cudaEventRecord(a);
  k<MODE><<<blocks, 256>>>(out, iters, spread);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 4, iters = 200;
  float* out;
  cudaMalloc(&out, (size_t)blocks * 4096 * sizeof(float));
  const double adds = (double)blocks * 256 * iters * 49;
  const char* names[3] = {"fp32 atomicAdd (ATOMS.CAST.SPIN loop)", "int32 atomicAdd (ATOMS.ADD)",
                          "fp32 plain read-add-write (no atomicity, bound)"};
  for (int spread = 0; spread < 2; ++spread) {
    float ms[3] = {run<0>(out, blocks, iters, spread), run<1>(out, blocks, iters, spread),
                   run<2>(out, blocks, iters, spread)};
    for (int m = 0; m < 3; ++m)
      printf("%-48s %-22s %8.3f ms  %8.1f G adds/s\n", names[m],
             spread ? "lanes 7 cells apart" : "lanes 1 cell apart", ms[m], adds / ms[m] / 1e6);
  }
  return 0;
}
