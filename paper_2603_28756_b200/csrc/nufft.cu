// Adjoint NUFFT (type 1) back-projection and ramp filtering on B200
// (SURVEY.md §8 rows a16-a20).
//
// Reference: tomoforge/radon.py:124-128 (_back_project_rows) Fourier-transforms
// every detector row, shifts it to signed frequency order, multiplies by the
// detector-centring phase / Nd and hands the polar samples to nufft.type1
// (nufft.py:203-223), which spreads them onto a 2x oversampled grid with a
// width-w Kaiser-Bessel kernel (np.bincount scatter), inverse-FFTs the grid,
// crops the N x N centre and divides by the kernel's Fourier transform.
// radon.py:137-160 (ramp_filter_apply, fbp) filters the rows with |w| first.
//
//   K8 k_detector_rows : one CTA per (slice, angle) row: mixed-radix DFT of
//                        length Nd = L * r (L a power of two, r odd) in shared
//                        memory -- r Stockham radix-2 FFTs of length L and an
//                        r-term recombination -- then either
//                        mode 0: the sample values c_m of the row (fftshift,
//                                detector phase, plan centring phase, 1/Nd,
//                                optional |w| ramp and scale folded into one
//                                complex factor per sample), or
//                        mode 1: the ramp-filtered row (x |w|, inverse DFT,
//                                real part) -- ramp_filter_apply.
//   K7 k_spread        : gridding without atomics.  The polar sampling is the
//                        same for every slice, so the plan bins samples once
//                        into 32 x 32 grid tiles (CSR, sample order kept).  A
//                        CTA owns one tile for NB slices: lane = grid column,
//                        each warp owns 4 grid rows, and every grid point is
//                        accumulated by exactly one thread in sample order --
//                        deterministic, no shared or global atomics.  Samples
//                        are staged 32 at a time per warp (one lane per
//                        sample's index chain) in shared memory.  The tile
//                        is stored with a per-index phase e^{-2 pi i a (N/2)/os} so
//                        the centred N x N crop of the inverse FFT becomes its
//                        first N outputs (pruned last pass).
//   k_nufft_rows       : inverse FFT along a (contiguous) of every grid row b,
//                        first os/2 outputs, written row-blocked [b/4][ix][b%4].
//   k_nufft_cols       : per output row ix < N: gather the 32-byte pieces of
//                        column ix, inverse FFT along b, keep iy < N, multiply
//                        by the deapodisation deapod[ix] deapod[iy] and scale,
//                        real (or complex) output, coalesced along iy.
//
// The GPU grid side os is the smallest power of two >= max(32, ceil(sigma N));
// at the reference's default sigma = 2 and power-of-two N it equals the
// reference grid (2N).  Kernel width and shape beta follow the reference's rule
// (nufft.py:54-57, :128-129), so the approximation error is the reference's or
// smaller.
#include <algorithm>

#include "tf_common.cuh"

namespace tf {

// ============================================================ K8: detector rows
// In-place Stockham radix-2 FFTs of length L on r interleaved sequences held as
// buf[s * L + n1] (s < r), ping-ponging with tmp; returns the buffer holding the
// result.  tw[q] = e^{-+2 pi i q / nd} (sign chosen by the caller's table).
__device__ c32* smem_fft_pow2(c32* buf, c32* tmp, const c32* tw, int L, int r, int nd) {
  const int half = L / 2;
  for (int ls = 1; ls < L; ls <<= 1) {
    const int tw_step = nd / (2 * ls);  // e^{-2 pi i k / (2 ls)} = tw[k * nd / (2 ls)]
    for (int id = threadIdx.x; id < r * half; id += blockDim.x) {
      const int s = id / half, j = id - s * half;
      const int k = j & (ls - 1);
      const c32 a = buf[s * L + j];
      const c32 b = cmul(buf[s * L + j + half], tw[k * tw_step]);
      const int o = s * L + ((j - k) << 1) + k;
      tmp[o] = cadd(a, b);
      tmp[o + ls] = csub(a, b);
    }
    __syncthreads();
    c32* t = buf;
    buf = tmp;
    tmp = t;
  }
  return buf;
}

// X[k] = sum_s tw[(s k) mod nd] F_s[k mod L] for k < nd (out may not alias F)
__device__ void smem_recombine(const c32* F, c32* out, const c32* tw, int L, int r, int nd) {
  for (int k = threadIdx.x; k < nd; k += blockDim.x) {
    const int k1 = k & (L - 1);
    c32 acc = F[k1];
    int q = 0;
    for (int s = 1; s < r; ++s) {
      q += k;
      if (q >= nd) q -= nd;
      const c32 f = F[s * L + k1];
      acc = cadd(acc, cmul(f, tw[q]));
    }
    out[k] = acc;
  }
}

// Full DFT of the nd values in a (natural order) -> returns buffer with X[k].
// a, b, c are nd-word buffers; tw the sign-appropriate twiddle table.
__device__ c32* smem_dft(c32* a, c32* b, c32* c, const c32* tw, int L, int r, int nd) {
  if (r > 1) {
    // decimate: b[s * L + n1] = a[r n1 + s]
    for (int i = threadIdx.x; i < nd; i += blockDim.x) {
      const int s = i % r, n1 = i / r;
      b[s * L + n1] = a[i];
    }
    __syncthreads();
    c32* F = smem_fft_pow2(b, c, tw, L, r, nd);
    smem_recombine(F, a, tw, L, r, nd);
    __syncthreads();
    return a;
  }
  c32* F = smem_fft_pow2(a, b, tw, L, 1, nd);
  return F;
}

// signed detector frequency index of FFT bin k (ifftshift of the signed range)
__device__ __forceinline__ int signed_bin(int k, int nd) { return k < (nd + 1) / 2 ? k : k - nd; }

// rows: [nrows][nd] fp32 (all (slice, angle) rows).  mode 0 -> out c32
// [nrows][nd] samples in signed order times sph[(row % n_angles) * nd + jj];
// mode 1 -> out fp32 [nrows][nd] ramp-filtered rows.
__global__ void k_detector_rows(const float* __restrict__ rows, int nd, int L, int r,
                                int n_angles, const c32* __restrict__ sph, int mode, int ramp,
                                float gain, void* __restrict__ out) {
  extern __shared__ __align__(16) c32 sm[];
  c32* a = sm;
  c32* b = a + nd;
  c32* c = b + nd;
  c32* tw = c + nd;
  const long long row = blockIdx.x;
  const float* x = rows + row * nd;
  for (int q = threadIdx.x; q < nd; q += blockDim.x) {
    float s, co;
    sincospif(-2.0f * (float)q / (float)nd, &s, &co);
    tw[q] = mk(co, s);
    a[q] = mk(__ldg(x + q), 0.f);
  }
  __syncthreads();
  c32* X = smem_dft(a, b, c, tw, L, r, nd);
  const float two_pi_nd = 6.283185307179586f / (float)nd;
  if (mode == 0) {
    c32* o = reinterpret_cast<c32*>(out) + row * nd;
    const c32* ph = sph + (row % n_angles) * nd;
    const int jlo = -(nd / 2);
    for (int jj = threadIdx.x; jj < nd; jj += blockDim.x) {
      const int j = jj + jlo;
      const int k = j < 0 ? j + nd : j;
      float f = gain;
      if (ramp) f *= fabsf(two_pi_nd * (float)j);
      o[jj] = scale(cmul(X[k], __ldg(ph + jj)), f);
    }
    return;
  }
  // mode 1: Y = X |w|, inverse DFT (conjugate twiddles), real part / nd
  c32* Y = (X == a) ? b : a;
  c32* s1 = (X == c) ? b : c;
  for (int k = threadIdx.x; k < nd; k += blockDim.x) {
    Y[k] = scale(X[k], fabsf(two_pi_nd * (float)signed_bin(k, nd)));
    tw[k] = conj(tw[k]);
  }
  __syncthreads();
  // smem_dft needs (a, b, c) distinct with the input in a
  c32* s2 = X;
  c32* R = smem_dft(Y, s1, s2, tw, L, r, nd);
  float* o = reinterpret_cast<float*>(out) + row * nd;
  const float inv = gain / (float)nd;
  for (int k = threadIdx.x; k < nd; k += blockDim.x) o[k] = R[k].x * inv;
}

// ============================================================ K7: gridding
// Tile of 32 (a, lanes) x 32 (b, 4 per warp) grid points for NB slices.
// ab[m] = (a0, b0): first grid index of sample m's window (mod os); wts[m] =
// (wx[0..W), wy[0..W)); c: [nslices][c_stride] samples.
//
// Each warp walks its band list (the samples whose window touches its 4 rows,
// sample order) in chunks of 32: lane l fetches the index chain tile_idx -> ab ->
// weights / values of sample base + l (32 independent chains in flight instead of
// one), the chunk is staged in the warp's shared-memory slot, and while the warp
// accumulates it sample by sample from shared memory (broadcast reads), the next
// chunk's fetches are already in flight.  Every grid point is still accumulated by
// one thread in sample order with the same arithmetic: deterministic, no atomics.
template <int W, int NB>
struct SpreadStage {
  int2 ab[32];
  float w[32][2 * W + 1];  // +1: rows of odd stride (distinct banks per sample)
  c32 cv[32][NB];
};

template <int W, int NB>
__global__ void __launch_bounds__(256)
k_spread(const c32* __restrict__ c, long long c_stride, int nslices, int os, int ntile_a,
         const int* __restrict__ tile_ptr, const int* __restrict__ tile_idx,
         const int* __restrict__ tile_order, const int2* __restrict__ ab,
         const float* __restrict__ wts, const c32* __restrict__ preph, c32* __restrict__ grid) {
  __shared__ SpreadStage<W, NB> stage_all[8];
  // heaviest tiles first (longest-processing-time order): the polar sampling puts
  // most samples in the centre tiles, which otherwise finish last and leave a tail
  const int tile = tile_order ? __ldg(tile_order + blockIdx.x) : (int)blockIdx.x;
  const int ta = tile % ntile_a, tb = tile / ntile_a;
  const int z0 = blockIdx.y * NB;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  SpreadStage<W, NB>& st = stage_all[warp];
  const int a = ta * 32 + lane;
  const int bb = tb * 32 + warp * 4;
  c32 acc[4][NB];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < NB; ++j) acc[i][j] = mk(0.f, 0.f);
  // this warp's list: the samples whose window touches its 4-row band
  const int beg = __ldg(tile_ptr + tile * 8 + warp), end = __ldg(tile_ptr + tile * 8 + warp + 1);
  // registers of the chunk in flight (lane l: sample base + l)
  int2 r_ab = make_int2(0, 0);
  float r_w[2 * W];
  c32 r_cv[NB];
  auto fetch = [&](int base) {
    const int q = base + lane;
    if (q < end) {
      const int m = __ldg(tile_idx + q);
      r_ab = __ldg(ab + m);
      const float* wr = wts + (long long)m * (2 * W);
#pragma unroll
      for (int k = 0; k < 2 * W; ++k) r_w[k] = __ldg(wr + k);
#pragma unroll
      for (int j = 0; j < NB; ++j)
        r_cv[j] = (z0 + j < nslices) ? __ldg(c + (long long)(z0 + j) * c_stride + m) : mk(0.f, 0.f);
    }
  };
  if (beg < end) fetch(beg);
  for (int base = beg; base < end; base += 32) {
    const int cnt = min(32, end - base);
    __syncwarp();  // the previous chunk is consumed
    st.ab[lane] = r_ab;
#pragma unroll
    for (int k = 0; k < 2 * W; ++k) st.w[lane][k] = r_w[k];
#pragma unroll
    for (int j = 0; j < NB; ++j) st.cv[lane][j] = r_cv[j];
    __syncwarp();
    if (base + 32 < end) fetch(base + 32);
    for (int q = 0; q < cnt; ++q) {
      const int2 s = st.ab[q];
      int db = bb - s.y;
      if (db < 0) db += os;
      if (db >= W && db <= os - 4) continue;  // none of this warp's rows (warp-uniform)
      int da = a - s.x;
      if (da < 0) da += os;
      const float wx = da < W ? st.w[q][da] : 0.f;
      c32 cv[NB];
#pragma unroll
      for (int j = 0; j < NB; ++j) cv[j] = st.cv[q][j];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        int d = db + i;
        if (d >= os) d -= os;
        if (d < W) {
          const float w = wx * st.w[q][W + d];
#pragma unroll
          for (int j = 0; j < NB; ++j) acc[i][j] = pfma(cv[j], mk(w, w), acc[i][j]);
        }
      }
    }
  }
  const c32 pa = __ldg(preph + a);
  const long long plane = (long long)os * os;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int b = bb + i;
    const c32 p = cmul(pa, __ldg(preph + b));
#pragma unroll
    for (int j = 0; j < NB; ++j)
      if (z0 + j < nslices) grid[(z0 + j) * plane + (long long)b * os + a] = cmul(acc[i][j], p);
  }
}

// ============================================================ grid inverse FFT
// rows pass: grid [z][b][a] (b < os rows of length M = os), inverse FFT along a,
// first M/2 outputs -> Tn[z][b/4][ix][b%4] (ix < M/2).  Group g of a CTA
// transforms rows 2p, 2p+1 with p = blockIdx.x * G + g.
template <int M, int E, int G>
__global__ void __launch_bounds__(G*(M / E))
k_nufft_rows(const c32* __restrict__ grid, c32* __restrict__ Tn) {
  constexpr int TT = M / E;
  constexpr int SB = group_stride(M, 2 * G);
  constexpr int HC = M / 2;
  extern __shared__ __align__(16) c32 smem[];
  const int g = threadIdx.x / TT;
  const int t = threadIdx.x - g * TT;
  const int z = blockIdx.y;
  const int p = blockIdx.x * G + g;  // row pair, rows 2p, 2p+1 (M/2 pairs)
  const bool active = p < M / 2;       // surplus groups still join the barriers
  const c32* src = grid + ((long long)z * M + 2 * (active ? p : 0)) * M;
  c32 v[2][E];
#pragma unroll
  for (int m = 0; m < E; ++m)
#pragma unroll
    for (int b = 0; b < 2; ++b) v[b][m] = __ldg(src + b * M + t + TT * m);
  fftn<M, E, true, false, true, 2>(v, smem + g * 2 * SB, SB, t);
  if (!active) return;
  const int blk = p >> 1, r = (p & 1) * 2;
  float4* dst = reinterpret_cast<float4*>(Tn + ((long long)z * (M / 4) + blk) * HC * 4);
#pragma unroll
  for (int m = 0; m < E / 2; ++m) {
    const int ix = t + TT * m;
    dst[(ix * 4 + r) >> 1] = make_float4(v[0][m].x, v[0][m].y, v[1][m].x, v[1][m].y);
  }
}

// cols pass: for ix < n, gather column ix of Tn over b, inverse FFT, keep iy < n,
// out[z][ix][iy] = val * scale * deapod[ix] * deapod[iy] (real part unless CPLX).
template <int M, int E, int G, bool CPLX>
__global__ void __launch_bounds__(G*(M / E))
k_nufft_cols(const c32* __restrict__ Tn, const float* __restrict__ deapod, int n, float gain,
             void* __restrict__ out) {
  constexpr int TT = M / E;
  constexpr int SB = group_stride(M, G);
  constexpr int HC = M / 2;
  extern __shared__ __align__(16) c32 smem[];
  const int g = threadIdx.x / TT;
  const int t = threadIdx.x - g * TT;
  const int z = blockIdx.y;
  const int ix = blockIdx.x * G + g;
  const bool active = ix < n;
  const int ixc = active ? ix : 0;
  const c32* src = Tn + (long long)z * (M / 4) * HC * 4;
  c32 v[E];
#pragma unroll
  for (int m = 0; m < E; ++m) {
    const int b = t + TT * m;
    v[m] = __ldg(src + ((long long)(b >> 2) * HC + ixc) * 4 + (b & 3));
  }
  fft<M, E, true, false, true>(v, smem + g * SB, t);
  if (!active) return;
  const float dx = __ldg(deapod + ix) * gain;
#pragma unroll
  for (int m = 0; m < E / 2; ++m) {
    const int iy = t + TT * m;
    if (iy < n) {
      const float f = dx * __ldg(deapod + iy);
      const long long o = ((long long)z * n + ix) * n + iy;
      if constexpr (CPLX) reinterpret_cast<c32*>(out)[o] = scale(v[m], f);
      else reinterpret_cast<float*>(out)[o] = v[m].x * f;
    }
  }
}

// ============================================================ plan tables
// Per sample m and axis: first window index a0 = ceil(eta - w/2) mod os with
// eta = k os / (2 pi), and the w Kaiser-Bessel weights I0(beta sqrt(1 - (2x/w)^2))
// at x = a0 + t - eta, in fp64 (the reference tabulates the same kernel,
// nufft.py:80-87).  kxy: [S][2] fp64; ab: [S] int2; wts: [S][2w] fp32.
__global__ void k_plan_weights(const double* __restrict__ kxy, long long S, int os, int w,
                               double beta, int2* __restrict__ ab, float* __restrict__ wts) {
  const long long m = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (m >= S) return;
  int a0[2];
#pragma unroll
  for (int ax = 0; ax < 2; ++ax) {
    const double eta = kxy[2 * m + ax] * os / (2.0 * 3.14159265358979323846);
    const double start = ceil(eta - 0.5 * w);
    long long st = (long long)start % os;
    if (st < 0) st += os;
    a0[ax] = (int)st;
    for (int t = 0; t < w; ++t) {
      const double x = start + t - eta;
      const double arg = 1.0 - (2.0 * x / w) * (2.0 * x / w);
      wts[m * 2 * w + ax * w + t] = arg >= 0.0 ? (float)cyl_bessel_i0(beta * sqrt(arg)) : 0.f;
    }
  }
  ab[m] = make_int2(a0[0], a0[1]);
}

int nufft_plan_weights(const double* kxy, long long S, int os, int w, double beta, void* ab,
                       float* wts, cudaStream_t st) {
  if (S <= 0) return TF_OK;
  const int bs = 256;
  k_plan_weights<<<(unsigned)((S + bs - 1) / bs), bs, 0, st>>>(kxy, S, os, w, beta,
                                                               reinterpret_cast<int2*>(ab), wts);
  return check_launch("k_plan_weights");
}

// ============================================================ forward NUFFT (type 2)
// Reference: nufft.type2 (nufft.py:184-200): deapodise, embed centred, fft2,
// gather each sample's w x w window with the Kaiser-Bessel weights, x phase;
// radon.forward_project (radon.py:85-96): x detector phase, ifftshift, ifft
// along the bins, real part.  Here the image (x deapod) is transformed with the
// Toeplitz row kernel and a forward column pass into the half spectrum
// S[b][a] (b in [0, os/2]) of its offset-0 embedding; the centring is the
// conjugate pre-phase per grid index, and G(a, b) for b > os/2 is
// conj(G(-a, -b)) (real image).  One thread per (sample, slice) gathers its
// window from L2.

// x * deapod[ix] * deapod[iy] * gain  (fp32, same layout)
__global__ void k_scale_deapod(const float* __restrict__ x, float* __restrict__ out, long long total,
                               int n, const float* __restrict__ deapod, float gain) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int iy = (int)(i % n);
    const int ix = (int)((i / n) % n);
    out[i] = x[i] * __ldg(deapod + ix) * __ldg(deapod + iy) * gain;
  }
}

template <int W>
__global__ void __launch_bounds__(256)
k_interp(const c32* __restrict__ S, int os, long long n_samples, const int2* __restrict__ ab,
         const float* __restrict__ wts, const c32* __restrict__ preph,
         const c32* __restrict__ factor, c32* __restrict__ out) {
  const long long m = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (m >= n_samples) return;
  const int z = blockIdx.y;
  const int H = os / 2 + 1;
  const c32* Sz = S + (long long)z * H * os;
  const int2 s = __ldg(ab + m);
  const float* wr = wts + m * (2 * W);
  c32 wx[W];
  int ax[W];
#pragma unroll
  for (int t = 0; t < W; ++t) {
    int a = s.x + t;
    if (a >= os) a -= os;
    ax[t] = a;
    wx[t] = scale(conj(__ldg(preph + a)), __ldg(wr + t));
  }
  c32 acc = mk(0.f, 0.f);
#pragma unroll
  for (int u = 0; u < W; ++u) {
    int b = s.y + u;
    if (b >= os) b -= os;
    const c32 wy = scale(conj(__ldg(preph + b)), __ldg(wr + W + u));
    c32 row = mk(0.f, 0.f);
    if (b <= os / 2) {
      const c32* Sb = Sz + (long long)b * os;
#pragma unroll
      for (int t = 0; t < W; ++t) row = cadd(row, cmul(__ldg(Sb + ax[t]), wx[t]));
    } else {  // Hermitian mirror of a real image's spectrum
      const c32* Sb = Sz + (long long)(os - b) * os;
#pragma unroll
      for (int t = 0; t < W; ++t) {
        const int am = ax[t] == 0 ? 0 : os - ax[t];
        row = cadd(row, cmul(conj(__ldg(Sb + am)), wx[t]));
      }
    }
    acc = cadd(acc, cmul(row, wy));
  }
  if (factor) acc = cmul(acc, __ldg(factor + m));
  out[(long long)z * n_samples + m] = acc;
}

// rows[r][n] = Re(ifft(ifftshift(c[r][.])))[n] * gain: c in signed-frequency
// order (jj), complex; inverse mixed-radix DFT in shared memory (K8's engine)
__global__ void k_detector_rows_inv(const c32* __restrict__ c, int nd, int L, int r, float gain,
                                    float* __restrict__ out) {
  extern __shared__ __align__(16) c32 sm[];
  c32* a = sm;
  c32* b = a + nd;
  c32* cc = b + nd;
  c32* tw = cc + nd;
  const long long row = blockIdx.x;
  const c32* x = c + row * nd;
  const int jlo = -(nd / 2);
  for (int q = threadIdx.x; q < nd; q += blockDim.x) {
    float sn, co;
    sincospif(2.0f * (float)q / (float)nd, &sn, &co);  // inverse: e^{+2 pi i q / nd}
    tw[q] = mk(co, sn);
    const int j = q + jlo;                               // signed index of entry q
    a[j < 0 ? j + nd : j] = __ldg(x + q);                // ifftshift
  }
  __syncthreads();
  c32* X = smem_dft(a, b, cc, tw, L, r, nd);
  float* o = out + row * nd;
  const float g = gain / (float)nd;
  for (int k = threadIdx.x; k < nd; k += blockDim.x) o[k] = X[k].x * g;
}

// ============================================================ direct DFT (fp64)
// c_m = sum_{ix, iy} f[ix][iy] exp(-i (kx_m x + ky_m y)), x = ix - (N-1)/2: the
// brute-force type-2 oracle of nufft.direct_dft (nufft.py:230-249), one thread
// per sample, fp64 throughout (sincos per term; N <= 128 as in the reference).
__global__ void k_direct_dft(const double* __restrict__ img, int n, const double* __restrict__ kxy,
                             long long S, double2* __restrict__ out) {
  const long long m = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (m >= S) return;
  const double kx = kxy[2 * m], ky = kxy[2 * m + 1];
  const double c0 = 0.5 * (n - 1);
  double re = 0.0, im = 0.0;
  for (int ix = 0; ix < n; ++ix) {
    const double px = kx * (ix - c0);
    for (int iy = 0; iy < n; ++iy) {
      double sn, cs;
      sincos(px + ky * (iy - c0), &sn, &cs);
      const double f = __ldg(img + (long long)ix * n + iy);
      re = fma(f, cs, re);
      im = fma(-f, sn, im);
    }
  }
  out[m] = make_double2(re, im);
}

int direct_dft(const double* img, int n, const double* kxy, long long S, void* out,
               cudaStream_t st) {
  if (S <= 0) return TF_OK;
  k_direct_dft<<<(unsigned)((S + 127) / 128), 128, 0, st>>>(img, n, kxy, S,
                                                             reinterpret_cast<double2*>(out));
  return check_launch("k_direct_dft");
}

// ============================================================ host dispatch
namespace {

template <typename K>
int prep_nufft_kernel(K kern, size_t smem) {
  if (smem > 48 * 1024)
    return check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smem),
                      "cudaFuncSetAttribute");
  return TF_OK;
}

template <int M>
struct NufftFftFn {
  static constexpr int E = M < 16 ? M : 16;
  static constexpr int TT = M / E;
  static constexpr int GR = TT >= 128 ? 1 : 128 / TT;  // groups per CTA (rows pass)
  static constexpr int GC = TT >= 128 ? 1 : 128 / TT;  // groups per CTA (cols pass)
  static int run(const c32* grid, c32* Tn, long long nz, int n, const float* deapod, float scale,
                 bool cplx, void* out, cudaStream_t st) {
    {
      auto kern = k_nufft_rows<M, E, GR>;
      const size_t smem = sizeof(c32) * 2 * GR * group_stride(M, 2 * GR);
      TF_TRY(prep_nufft_kernel(kern, smem));
      const int pairs = M / 2;
      kern<<<dim3((pairs + GR - 1) / GR, (unsigned)nz), GR * TT, smem, st>>>(grid, Tn);
      TF_TRY(check_launch("k_nufft_rows"));
    }
    {
      const size_t smem = sizeof(c32) * GC * group_stride(M, GC);
      const dim3 g((n + GC - 1) / GC, (unsigned)nz);
      if (cplx) {
        auto kern = k_nufft_cols<M, E, GC, true>;
        TF_TRY(prep_nufft_kernel(kern, smem));
        kern<<<g, GC * TT, smem, st>>>(Tn, deapod, n, scale, out);
      } else {
        auto kern = k_nufft_cols<M, E, GC, false>;
        TF_TRY(prep_nufft_kernel(kern, smem));
        kern<<<g, GC * TT, smem, st>>>(Tn, deapod, n, scale, out);
      }
      TF_TRY(check_launch("k_nufft_cols"));
    }
    return TF_OK;
  }
};

template <int W>
int launch_spread(const c32* c, long long c_stride, long long nz, int os, const int* tile_ptr,
                  const int* tile_idx, const int* tile_order, const int2* ab, const float* wts,
                  const c32* preph, c32* grid, cudaStream_t st) {
#ifndef TF_SPREAD_NB
#define TF_SPREAD_NB 2
#endif
  constexpr int NB = TF_SPREAD_NB;  // slices per CTA: amortises each sample's index chain
  const int nta = os / 32;
  const dim3 g((unsigned)(nta * nta), (unsigned)((nz + NB - 1) / NB));
  k_spread<W, NB><<<g, 256, 0, st>>>(c, c_stride, (int)nz, os, nta, tile_ptr, tile_idx,
                                      tile_order, ab, wts, preph, grid);
  return check_launch("k_spread");
}

int dispatch_spread(int w, const c32* c, long long c_stride, long long nz, int os,
                    const int* tile_ptr, const int* tile_idx, const int* tile_order,
                    const int2* ab, const float* wts, const c32* preph, c32* grid,
                    cudaStream_t st) {
  switch (w) {
#define TF_W(W)                                                                              \
  case W:                                                                                    \
    return launch_spread<W>(c, c_stride, nz, os, tile_ptr, tile_idx, tile_order, ab, wts, preph, \
                            grid, st);
    TF_W(2) TF_W(3) TF_W(4) TF_W(5) TF_W(6) TF_W(7) TF_W(8) TF_W(9) TF_W(10) TF_W(11) TF_W(12)
    TF_W(13) TF_W(14) TF_W(15) TF_W(16)
#undef TF_W
    default: return fail_arg("unsupported kernel width %d", w);
  }
}

int dispatch_grid_fft(int os, const c32* grid, c32* Tn, long long nz, int n, const float* deapod,
                      float scale, bool cplx, void* out, cudaStream_t st) {
  switch (os) {
    case 32: return NufftFftFn<32>::run(grid, Tn, nz, n, deapod, scale, cplx, out, st);
    case 64: return NufftFftFn<64>::run(grid, Tn, nz, n, deapod, scale, cplx, out, st);
    case 128: return NufftFftFn<128>::run(grid, Tn, nz, n, deapod, scale, cplx, out, st);
    case 256: return NufftFftFn<256>::run(grid, Tn, nz, n, deapod, scale, cplx, out, st);
    case 512: return NufftFftFn<512>::run(grid, Tn, nz, n, deapod, scale, cplx, out, st);
    case 1024: return NufftFftFn<1024>::run(grid, Tn, nz, n, deapod, scale, cplx, out, st);
    case 2048: return NufftFftFn<2048>::run(grid, Tn, nz, n, deapod, scale, cplx, out, st);
    case 4096: return NufftFftFn<4096>::run(grid, Tn, nz, n, deapod, scale, cplx, out, st);
    case 8192: return NufftFftFn<8192>::run(grid, Tn, nz, n, deapod, scale, cplx, out, st);
    default: return fail_arg("unsupported NUFFT grid side %d", os);
  }
}

}  // namespace

size_t spectrum_workspace_bytes(int n, int M);
int real_spectrum(const float* img, long long nslices, int n, int M, void* T, void* S,
                  cudaStream_t st);

size_t type2_workspace_bytes(int n, int os, long long nslices) {
  const size_t spec = (size_t)(os / 2 + 1) * os * sizeof(c32);
  return (size_t)nslices * (spec + spectrum_workspace_bytes(n, os) + (size_t)n * n * sizeof(float));
}

template <int W>
int launch_interp(const c32* S, int os, long long ns, long long nz, const int2* ab,
                  const float* wts, const c32* preph, const c32* factor, c32* out,
                  cudaStream_t st) {
  const dim3 g((unsigned)((ns + 255) / 256), (unsigned)nz);
  k_interp<W><<<g, 256, 0, st>>>(S, os, ns, ab, wts, preph, factor, out);
  return check_launch("k_interp");
}

int nufft_type2(const float* img, long long nslices, int n, int os, int w, const void* ab,
                const float* wts, const void* preph, const float* deapod, const void* factor,
                long long n_samples, void* out, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (!is_pow2(os) || os < 32 || os > 8192 || 2 * n > os)
    return fail_arg("NUFFT grid side %d unsupported for N = %d", os, n);
  const size_t per = type2_workspace_bytes(n, os, 1);
  const long long chunk = (long long)(ws_bytes / per);
  if (chunk < 1) return fail_arg("type2 workspace too small: %zu < %zu", ws_bytes, per);
  const long long spec = (long long)(os / 2 + 1) * os;
  const long long nn = (long long)n * n;
  for (long long z0 = 0; z0 < nslices; z0 += chunk) {
    const long long nz = std::min(chunk, nslices - z0);
    c32* S = reinterpret_cast<c32*>(ws);
    c32* T = S + nz * spec;
    float* sc = reinterpret_cast<float*>(reinterpret_cast<char*>(T) +
                                         nz * spectrum_workspace_bytes(n, os));
    const long long tot = nz * nn;
    k_scale_deapod<<<(unsigned)std::min<long long>((tot + 255) / 256, 65535 * 8), 256, 0, st>>>(
        img + z0 * nn, sc, tot, n, deapod, 1.f);
    TF_TRY(check_launch("k_scale_deapod"));
    TF_TRY(real_spectrum(sc, nz, n, os, T, S, st));
    c32* o = reinterpret_cast<c32*>(out) + z0 * n_samples;
    const int2* ab2 = reinterpret_cast<const int2*>(ab);
    const c32* pp = reinterpret_cast<const c32*>(preph);
    const c32* fc = reinterpret_cast<const c32*>(factor);
    switch (w) {
#define TF_W(W) case W: TF_TRY(launch_interp<W>(S, os, n_samples, nz, ab2, wts, pp, fc, o, st)); break;
      TF_W(2) TF_W(3) TF_W(4) TF_W(5) TF_W(6) TF_W(7) TF_W(8) TF_W(9) TF_W(10) TF_W(11) TF_W(12)
      TF_W(13) TF_W(14) TF_W(15) TF_W(16)
#undef TF_W
      default: return fail_arg("unsupported kernel width %d", w);
    }
  }
  return TF_OK;
}

int detector_rows_inv(const void* c, long long nrows, int nd, float gain, float* out,
                      cudaStream_t st) {
  if (nd < 1 || nd > 8192) return fail_arg("detector bins %d outside [1, 8192]", nd);
  int L = 1;
  while ((nd % (2 * L)) == 0) L *= 2;
  const size_t smem = 4 * (size_t)nd * sizeof(c32);
  TF_TRY(prep_nufft_kernel(k_detector_rows_inv, smem));
  if (nrows == 0) return TF_OK;
  k_detector_rows_inv<<<(unsigned)nrows, 256, smem, st>>>(reinterpret_cast<const c32*>(c), nd, L,
                                                          nd / L, gain, out);
  return check_launch("k_detector_rows_inv");
}

int init_twiddles_nufft() { return check_cuda(init_twiddles_tu(), "twiddle init (nufft)"); }

size_t nufft_workspace_bytes(int os, long long nslices) {
  const size_t plane = (size_t)os * os * sizeof(c32);
  return (size_t)nslices * (plane + plane / 2);
}

int detector_rows(const float* rows, long long nrows, int nd, int n_angles, const void* sph,
                  int mode, int ramp, float scale, void* out, cudaStream_t st) {
  if (nd < 1 || nd > 8192) return fail_arg("detector bins %d outside [1, 8192]", nd);
  if (mode == 0 && (!sph || n_angles < 1)) return fail_arg("sample phases required");
  int L = 1;
  while ((nd % (2 * L)) == 0) L *= 2;
  const int r = nd / L;
  const size_t smem = 4 * (size_t)nd * sizeof(c32);
  TF_TRY(prep_nufft_kernel(k_detector_rows, smem));
  for (long long r0 = 0; r0 < nrows; r0 += 2147483647LL) {
    const long long nr = std::min<long long>(2147483647LL, nrows - r0);
    const size_t es = mode == 0 ? sizeof(c32) : sizeof(float);
    k_detector_rows<<<(unsigned)nr, 256, smem, st>>>(
        rows + r0 * nd, nd, L, r, n_angles, reinterpret_cast<const c32*>(sph), mode, ramp, scale,
        reinterpret_cast<char*>(out) + r0 * nd * es);
    TF_TRY(check_launch("k_detector_rows"));
  }
  return TF_OK;
}

int nufft_type1(const void* samples, long long s_stride, long long nslices, int n, int os, int w,
                const int* tile_ptr, const int* tile_idx, const int* tile_order, const void* ab,
                const float* wts,
                const void* preph, const float* deapod, float scale, int cplx, void* out,
                void* ws, size_t ws_bytes, cudaStream_t st) {
  if (!is_pow2(os) || os < 32 || os > 8192) return fail_arg("NUFFT grid side %d unsupported", os);
  if (2 * n > os) return fail_arg("NUFFT grid side %d < 2N = %d", os, 2 * n);
  const size_t per = nufft_workspace_bytes(os, 1);
  const long long chunk = (long long)(ws_bytes / per);
  if (chunk < 1) return fail_arg("NUFFT workspace too small: %zu < %zu", ws_bytes, per);
  const long long plane = (long long)os * os;
  for (long long z0 = 0; z0 < nslices; z0 += chunk) {
    const long long nz = std::min(chunk, nslices - z0);
    c32* grid = reinterpret_cast<c32*>(ws);
    c32* Tn = grid + nz * plane;
    TF_TRY(dispatch_spread(w, reinterpret_cast<const c32*>(samples) + z0 * s_stride, s_stride, nz,
                           os, tile_ptr, tile_idx, tile_order, reinterpret_cast<const int2*>(ab),
                           wts,
                           reinterpret_cast<const c32*>(preph), grid, st));
    const size_t osz = cplx ? sizeof(c32) : sizeof(float);
    TF_TRY(dispatch_grid_fft(os, grid, Tn, nz, n, deapod, scale, cplx != 0,
                             reinterpret_cast<char*>(out) + z0 * (long long)n * n * osz, st));
  }
  return TF_OK;
}

}  // namespace tf
