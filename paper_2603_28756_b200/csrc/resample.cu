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

// ---------------------------------------------------------------- fused 3-axis
// All three axes in one pass (multires.py:186-191).  A CTA owns a 32 (x) x 128
// (y) target tile and walks its run of target planes t.  The tile's source
// window (nr x nc cells per coarse plane) of every coarse plane it needs is
// copied into a shared-memory ring (cp.async, one copy per cell) exactly once;
// the plane the next target needs is in flight while the current target is
// interpolated: z from the ring into t1, x into t2, y on the way out.  HBM
// traffic: the source read once (plus the window halo) and the target written
// once -- ~4.5 B per fine voxel at ratio 2.  Upsampling only: consecutive target
// planes advance the z band by at most one coarse plane, so kz + 1 ring slots
// suffice.
constexpr int UP_TX = 128, UP_TY = 32;  // target tile (y contiguous, x rows)

__device__ __forceinline__ void cp_async4(float* dst, const float* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(
                   static_cast<unsigned>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// KT > 0: every axis has KT taps (compile time: 6 for the Lanczos-3 doubling of the
// schedule); KT == 0: per-axis tap counts <= 8 at run time
template <int KT>
__global__ void __launch_bounds__(256)
k_upsample3(const float* __restrict__ src, float* __restrict__ out, int hs, int ws, int t_begin,
            int nzt, int zper, int ht, int wt, const int* __restrict__ sz,
            const float* __restrict__ wz, int kz_rt, const int* __restrict__ sx,
            const float* __restrict__ wx, int kx_rt, const int* __restrict__ sy,
            const float* __restrict__ wy, int ky_rt, int nrm, int ncm) {
  constexpr int KM = KT > 0 ? KT : 8;  // unrolled tap loops
  const int kz = KT > 0 ? KT : kz_rt, kx = KT > 0 ? KT : kx_rt, ky = KT > 0 ? KT : ky_rt;
  extern __shared__ __align__(16) float up_sm[];
  const int ring_n = kz + 1;
  const int pw = nrm * ncm;                 // words per ring plane
  float* ring = up_sm;                      // [ring_n][nrm][ncm]
  float* t1 = ring + ring_n * pw;           // z-interpolated window [nrm][ncm]
  float* t2 = t1 + pw;                      // then x-interpolated [UP_TY][ncm]
  float* wxs = t2 + UP_TY * ncm;            // x taps of the tile rows [UP_TY][8]
  int* rss = reinterpret_cast<int*>(wxs + UP_TY * 8);  // their window rows [UP_TY]
  const int j0 = blockIdx.x * UP_TX, i0 = blockIdx.y * UP_TY;
  const int jn = min(UP_TX, wt - j0), in_ = min(UP_TY, ht - i0);
  const int r0 = __ldg(sx + i0), c0 = __ldg(sy + j0);
  const int nr = __ldg(sx + i0 + in_ - 1) + kx - r0;
  const int nc = __ldg(sy + j0 + jn - 1) + ky - c0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x < UP_TY) {
    const int i = threadIdx.x;
    rss[i] = i < in_ ? __ldg(sx + i0 + i) - r0 : 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) wxs[i * 8 + k] = (i < in_ && k < kx) ? __ldg(wx + (i0 + i) * kx + k) : 0.f;
  }
  // y taps of this thread's target column (fixed for the whole CTA)
  const int j = threadIdx.x % UP_TX, ib = threadIdx.x / UP_TX;
  float wyr[KM];
  int ys = 0;
#pragma unroll
  for (int k = 0; k < KM; ++k) wyr[k] = 0.f;
  if (j < jn) {
    ys = __ldg(sy + j0 + j) - c0;
#pragma unroll
    for (int k = 0; k < KM; ++k) wyr[k] = k < ky ? __ldg(wy + (j0 + j) * ky + k) : 0.f;
  }
  const long long plane = (long long)hs * ws;
  auto load_plane = [&](int s) {  // coarse plane s -> its ring slot
    const float* sp = src + (long long)s * plane + (long long)r0 * ws + c0;
    float* dst = ring + (s % ring_n) * pw;
    for (int r = warp; r < nr; r += 8)
      for (int c = lane; c < nc; c += 32) cp_async4(dst + r * ncm + c, sp + (long long)r * ws + c);
  };
  const int z_lo = blockIdx.z * zper, z_hi = min(nzt, z_lo + zper);
  if (z_lo >= z_hi) return;
  int hi = __ldg(sz + t_begin + z_lo);
  for (int k = 0; k < kz; ++k) load_plane(hi++);
  cp_async_commit();
  for (int tz = z_lo; tz < z_hi; ++tz) {
    const int t = t_begin + tz;
    const int s_lo = __ldg(sz + t);
    // the coarse plane the next target adds (at most one when upsampling)
    if (tz + 1 < z_hi && __ldg(sz + t + 1) + kz > hi) load_plane(hi++);
    cp_async_commit();
    cp_async_wait<1>();  // everything but the plane just issued
    __syncthreads();
    const float* wzt = wz + (long long)t * kz;
    float wzr[KM];
    const float* pl[KM];  // ring slots of the band's planes (no modulo in the cell loop)
    int slot = s_lo % ring_n;
#pragma unroll
    for (int k = 0; k < KM; ++k) {
      wzr[k] = k < kz ? __ldg(wzt + k) : 0.f;
      pl[k] = ring + slot * pw;
      slot = slot + 1 == ring_n ? 0 : slot + 1;
    }
    for (int r = warp; r < nr; r += 8)
      for (int c = lane; c < nc; c += 32) {
        const int off = r * ncm + c;
        float a = 0.f;
#pragma unroll
        for (int k = 0; k < KM; ++k)
          if (k < kz) a = fmaf(wzr[k], pl[k][off], a);
        t1[off] = a;
      }
    __syncthreads();
    for (int i = warp; i < in_; i += 8) {
      const float* src_r = t1 + rss[i] * ncm;
      float w8[KM];
#pragma unroll
      for (int k = 0; k < KM; ++k) w8[k] = wxs[i * 8 + k];
      for (int c = lane; c < nc; c += 32) {
        float a = 0.f;
#pragma unroll
        for (int k = 0; k < KM; ++k)
          if (k < kx) a = fmaf(w8[k], src_r[k * ncm + c], a);
        t2[i * ncm + c] = a;
      }
    }
    __syncthreads();
    if (j < jn) {
      float* op = out + ((long long)tz * ht + i0) * wt + j0 + j;
      for (int i = ib; i < in_; i += 256 / UP_TX) {
        const float* row = t2 + i * ncm + ys;
        float a = 0.f;
#pragma unroll
        for (int k = 0; k < KM; ++k)
          if (k < ky) a = fmaf(wyr[k], row[k], a);
        op[(long long)i * wt] = a;
      }
    }
  }
  cp_async_wait<0>();
}

int upsample3(const float* src, int zs, int hs, int ws, float* out, int t_begin, int nzt, int ht,
              int wt, const int* sz, const float* wz, int kz, const int* sx, const float* wx, int kx,
              const int* sy, const float* wy, int ky, int nrm, int ncm, cudaStream_t st) {
  if ((long long)nzt * ht * wt == 0) return TF_OK;
  if (kz < 1 || kz > 8 || kx < 1 || kx > 8 || ky < 1 || ky > 8)
    return fail_arg("upsample bands must have 1..8 taps (got %d, %d, %d)", kz, kx, ky);
  if (hs > ht || ws > wt) return fail_arg("upsample3 cannot reduce the grid");
  if (nrm < 1 || ncm < 1 || nrm > UP_TY + 8 || ncm > UP_TX + 8)
    return fail_arg("upsample3 window %d x %d out of range", nrm, ncm);
  (void)zs;
  const size_t smem = sizeof(float) * ((size_t)(kz + 3) * nrm * ncm + UP_TY * ncm + UP_TY * 9);
  auto kern = (kz == 6 && kx == 6 && ky == 6) ? k_upsample3<6> : k_upsample3<0>;
  TF_TRY(prep_kernel(kern, smem));
  int per_sm = 0;
  TF_TRY(check_cuda(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, smem),
                    "occupancy"));
  const int gx = (wt + UP_TX - 1) / UP_TX, gy = (ht + UP_TY - 1) / UP_TY;
  // split the target planes into z-runs so that the launch is ~16 waves of CTAs: with
  // one run per tile (1024 tiles at 2048^2) the last partial wave of long runs left
  // two thirds of the SMs idle for a third of the kernel; each extra run re-reads
  // only its first kz coarse window planes
  const long long tiles = (long long)gx * gy;
  const long long want = 16LL * std::max(1, per_sm) * num_sms();
  const int zch = (int)std::max<long long>(1, std::min<long long>(nzt, (want + tiles - 1) / tiles));
  const int zper = (nzt + zch - 1) / zch;
  const dim3 g(gx, gy, (nzt + zper - 1) / zper);
  kern<<<g, 256, smem, st>>>(src, out, hs, ws, t_begin, nzt, zper, ht, wt, sz, wz, kz, sx, wx, kx,
                             sy, wy, ky, nrm, ncm);
  return check_launch("k_upsample3");
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
