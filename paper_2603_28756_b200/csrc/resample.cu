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
// with `inner` the product of the dimensions after the axis.  For the z and y
// passes threads run along the inner dimension (coalesced loads and stores);
// the x pass (inner = 1) maps 256 consecutive targets of a row to a block, whose
// source window is a short contiguous run read through L1.  HBM-bound: one read
// of the source, one write of the target per pass.
#include <algorithm>

#include "tf_common.cuh"

namespace tf {

// inner > 1: grid (ceil(inner / 256), n_tgt, outer) -- 32-bit index math only,
// loads and stores coalesced along the inner dimension
template <int K>
__global__ void __launch_bounds__(256)
k_resample_axis(const float* __restrict__ in, float* __restrict__ out, int n_src, int n_tgt,
                long long inner, const int* __restrict__ s0, const float* __restrict__ w) {
  const long long i = blockIdx.x * 256LL + threadIdx.x;
  if (i >= inner) return;
  const int t = blockIdx.y;
  const long long o = blockIdx.z;
  const float* src = in + (o * n_src + __ldg(s0 + t)) * inner + i;
  const float* wt = w + t * K;
  float acc = 0.f;
#pragma unroll
  for (int k = 0; k < K; ++k) acc = fmaf(__ldg(wt + k), __ldg(src + k * inner), acc);
  out[(o * n_tgt + t) * inner + i] = acc;
}

// inner == 1 (the contiguous axis): block b covers targets [tb * 256, +256) of row
// o = b / nblk; the source window of a block is a contiguous run read through L1
template <int K>
__global__ void __launch_bounds__(256)
k_resample_rows(const float* __restrict__ in, float* __restrict__ out, int n_src, int n_tgt,
                int nblk, const int* __restrict__ s0, const float* __restrict__ w) {
  const long long o = blockIdx.x / nblk;
  const int t = (blockIdx.x - (int)o * nblk) * 256 + threadIdx.x;
  if (t >= n_tgt) return;
  const float* src = in + o * n_src + __ldg(s0 + t);
  const float* wt = w + t * K;
  float acc = 0.f;
#pragma unroll
  for (int k = 0; k < K; ++k) acc = fmaf(__ldg(wt + k), __ldg(src + k), acc);
  out[o * n_tgt + t] = acc;
}

template <int K>
int launch_resample(const float* in, float* out, long long outer, int n_src, int n_tgt,
                    long long inner, const int* s0, const float* w, cudaStream_t st) {
  if (inner == 1) {
    const int nblk = (n_tgt + 255) / 256;
    for (long long o0 = 0; o0 < outer; o0 += (1LL << 30) / nblk) {
      const long long no = std::min<long long>(outer - o0, (1LL << 30) / nblk);
      k_resample_rows<K><<<(unsigned)(no * nblk), 256, 0, st>>>(in + o0 * n_src, out + o0 * n_tgt,
                                                                n_src, n_tgt, nblk, s0, w);
    }
  } else {
    for (long long o0 = 0; o0 < outer; o0 += 65535) {
      const long long no = std::min<long long>(outer - o0, 65535);
      const dim3 g((unsigned)((inner + 255) / 256), (unsigned)n_tgt, (unsigned)no);
      k_resample_axis<K><<<g, 256, 0, st>>>(in + o0 * n_src * inner, out + o0 * n_tgt * inner,
                                            n_src, n_tgt, inner, s0, w);
    }
  }
  return check_launch("k_resample");
}

int resample_axis(const float* in, float* out, long long outer, int n_src, int n_tgt,
                  long long inner, const int* s0, const float* w, int K, cudaStream_t st) {
  if (outer * n_tgt * inner == 0) return TF_OK;
  if (n_tgt > 65535 && inner > 1) return fail_arg("resampling target %d too long", n_tgt);
  switch (K) {
#define TF_K(KK) \
  case KK: return launch_resample<KK>(in, out, outer, n_src, n_tgt, inner, s0, w, st);
    TF_K(1) TF_K(2) TF_K(3) TF_K(4) TF_K(5) TF_K(6) TF_K(7) TF_K(8)
#undef TF_K
    default: return fail_arg("resampling band %d exceeds 8 taps", K);
  }
}

}  // namespace tf
