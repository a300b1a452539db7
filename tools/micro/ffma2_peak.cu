// FFMA2 / FADD2 issue-rate microbenchmark: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp ffma2_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int ACC, int MODE>
__global__ void k(float2* out, int iters, float2 a, float2 b) {
  float2 acc[ACC];
#pragma unroll
  for (int i = 0; i < ACC; ++i) acc[i] = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ACC; ++i) {
      if (MODE == 0) acc[i] = __ffma2_rn(acc[i], a, b);                 // FFMA2 3 regs
      else if (MODE == 1) acc[i] = __fadd2_rn(acc[i], b);                // FADD2
      else if (MODE == 2) acc[i] = __ffma2_rn(acc[(i + 1) % ACC], a, acc[i]);  // FFMA2, 2 live operands
      else if (MODE == 3) {                                              // scalar FFMA
        acc[i].x = __fmaf_rn(acc[i].x, a.x, b.x);
        acc[i].y = __fmaf_rn(acc[i].y, a.y, b.y);
      } else if (MODE == 4) {  // scalar FFMA, register operands (3-reg form)
        acc[i].x = __fmaf_rn(acc[i].x, acc[(i + 1) % ACC].y, acc[(i + 2) % ACC].x);
        acc[i].y = __fmaf_rn(acc[i].y, acc[(i + 1) % ACC].x, acc[(i + 3) % ACC].y);
      } else if (MODE == 5) {  // FFMA2 (reg) on even i, two imm-form scalar FFMA on odd i
        if (i % 2 == 0) acc[i] = __ffma2_rn(acc[i], a, b);
        else { acc[i].x = __fmaf_rn(acc[i].x, 1.0001f, -2.5f); acc[i].y = __fmaf_rn(acc[i].y, 0.9999f, 3.5f); }
      } else if (MODE == 6) {  // imm-form scalar only
        acc[i].x = __fmaf_rn(acc[i].x, 1.0001f, -2.5f); acc[i].y = __fmaf_rn(acc[i].y, 0.9999f, 3.5f);
      } else {  // FADD2 on even i, imm-form FFMA pairs on odd i
        if (i % 2 == 0) acc[i] = __fadd2_rn(acc[i], b);
        else { acc[i].x = __fmaf_rn(acc[i].x, 1.0001f, -2.5f); acc[i].y = __fmaf_rn(acc[i].y, 0.9999f, 3.5f); }
      }
    }
  }
  float2 s = make_float2(0.f, 0.f);
#pragma unroll
  for (int i = 0; i < ACC; ++i) s = __fadd2_rn(s, acc[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int ACC, int MODE>
void run(const char* name, int threads, int blocks_per_sm) {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * blocks_per_sm, iters = 4096;
  float2* out;
  cudaMalloc(&out, sizeof(float2) * blocks * threads);
  k<ACC, MODE><<<blocks, threads>>>(out, 16, make_float2(1.0001f, 0.9999f), make_float2(1e-7f, 2e-7f));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<ACC, MODE><<<blocks, threads>>>(out, iters, make_float2(1.0001f, 0.9999f), make_float2(1e-7f, 2e-7f));
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  // lane-FMA (or add) count per warp, in units of FFMA2-equivalents (64 lane-ops)
  const double warp_instr = (double)blocks * threads / 32 * iters * ACC;
  const double cycles = ms * 1e-3 * clk * 1e3;
  printf("%-28s warps/SMSP %2d ACC %2d: %.3f ms  FFMA2-equiv per SMSP-cycle %.3f\n", name,
         threads * blocks_per_sm / 32 / 4, ACC, ms, warp_instr / (sms * 4) / cycles);
  cudaFree(out);
}

int main() {
  for (int w : {4, 8}) {
    run<8, 0>("FFMA2 reg", 128 * w, 1);
    run<8, 3>("FFMA scalar const-bank", 128 * w, 1);
    run<8, 4>("FFMA scalar 3-reg", 128 * w, 1);
    run<8, 6>("FFMA scalar imm", 128 * w, 1);
    run<8, 5>("FFMA2 reg + FFMA imm mix", 128 * w, 1);
    run<8, 7>("FADD2 + FFMA imm mix", 128 * w, 1);
  }
  return 0;
}
