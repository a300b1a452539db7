// Separable Lanczos-3 resampling (K9) for the coarse-to-fine schedule
// (SURVEY.md §8 row a23).
//
// Reference: tomoforge/multires.py:145-195 builds, per axis, a dense
// (n_tgt x n_src) interpolation matrix (Lanczos-3 taps, edge-clamped, rows
// normalised to 1) and applies it with einsum along z, then y, then x.  The
// matrix is banded: at most 2a+1 = 7 consecutive source samples per target row.
// The host extracts the band in float64 (same construction as the reference)
// and this kernel applies one axis:
//   out[o][t][i] = sum_k w[t][k] in[o][s0[t] + k][i]
// with `inner` the product of the dimensions after the axis.  Threads run over
// the output with the inner index fastest, so every load and store is
// coalesced for the z and y passes; the x pass (inner = 1) reads each source
// row segment through L1.  HBM-bound: one read of the source, one write of the
// target per pass.
#include "tf_common.cuh"

namespace tf {

template <int K>
__global__ void __launch_bounds__(256)
k_resample_axis(const float* __restrict__ in, float* __restrict__ out, long long outer, int n_src,
                int n_tgt, long long inner, const int* __restrict__ s0,
                const float* __restrict__ w) {
  const long long total = outer * n_tgt * inner;
  for (long long id = blockIdx.x * (long long)blockDim.x + threadIdx.x; id < total;
       id += (long long)gridDim.x * blockDim.x) {
    const long long i = id % inner;
    const long long ot = id / inner;
    const int t = (int)(ot % n_tgt);
    const long long o = ot / n_tgt;
    const int s = __ldg(s0 + t);
    const float* src = in + (o * n_src + s) * inner + i;
    const float* wt = w + (long long)t * K;
    float acc = 0.f;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const float wk = __ldg(wt + k);
      if (wk != 0.f) acc = fmaf(wk, __ldg(src + (long long)k * inner), acc);
    }
    out[id] = acc;
  }
}

int resample_axis(const float* in, float* out, long long outer, int n_src, int n_tgt,
                  long long inner, const int* s0, const float* w, int K, cudaStream_t st) {
  const long long total = outer * n_tgt * inner;
  if (total == 0) return TF_OK;
  const int threads = 256;
  const long long want = (total + threads - 1) / threads;
  const int blocks = (int)std::min<long long>(want, (long long)num_sms() * 16);
  switch (K) {
#define TF_K(KK) \
  case KK: k_resample_axis<KK><<<blocks, threads, 0, st>>>(in, out, outer, n_src, n_tgt, inner, s0, w); break;
    TF_K(1) TF_K(2) TF_K(3) TF_K(4) TF_K(5) TF_K(6) TF_K(7) TF_K(8)
#undef TF_K
    default: return fail_arg("resampling band %d exceeds 8 taps", K);
  }
  return check_launch("k_resample_axis");
}

}  // namespace tf
