// Toeplitz normal operator K x = R*R x on B200.
//
// Reference: tomoforge/toeplitz.py:134-149 (_apply_batch) pads each N x N
// slice into an odd 7-smooth M x M grid, runs a complex fft2, multiplies by
// main (+ conj(F) * flip), and crops the real part of ifft2.  Here the lag
// kernels are re-embedded circularly on an even power-of-two grid M >= 2N-1
// with the image at offset 0 (exact: all lags |d| <= N-1 stay distinct mod M),
// and the flip term becomes B = spec(K_flip) * ph(kx) ph(ky),
// ph_k = e^{-2 pi i k (N-1)/M} (derivation in DESIGN.md §3).  Both lag kernels
// are real and even, so the transform is real-to-complex on the half spectrum:
//
//   K1 k_rows_fwd  : two image rows per complex FFT of length M (zero padded),
//                    split into two half spectra, stored frequency-major
//                    T[z][ky][ix] (column ix contiguous for K2).
//   K2 k_cols_conv : per half-spectrum column ky, length-M FFT over ix,
//                    Y = F*A + conj(F)*B with the PSF column held in registers
//                    for the whole slice loop, inverse FFT, keep ix < N.
//   K3 k_rows_inv  : two rows per complex inverse FFT (Hermitian packing),
//                    crop n < N, epilogue out = alpha*y + beta*aux.
//
// PSF (K6, toeplitz.py:85-131 compute_psf/build_psf): the NUFFT-of-ones kernel
// is replaced by its exact closed form, K(d) = sum_theta D(d . e_theta) with
// the Dirichlet sum D(u) = sum_j cos(2 pi j u / Nd) over the signed detector
// frequencies (geometry.py:196-201), K_nyq(d) = 1/2 sum_theta cos(pi d.e_theta)
// for even Nd (toeplitz.py:106-114); evaluated in fp64, transformed with the
// same K1 + forward column pass, and folded with 1/M^2 into
//   PQ = ((A + Re B)/M^2, (A - Re B)/M^2),  Bi = Im B / M^2
// so that Y = (Fr P + Fi Bi, Fi Q + Fr Bi): two paired-fp32 instructions.
#include <algorithm>

#include "tf_common.cuh"

namespace tf {

// ============================================================ K1: rows, forward
// x: [nslices][rows][row_stride] fp32, row r nonzero for n < n_in (zero beyond)
// T: [nslices][M/2+1][rows] c32
template <int M, int E, int F>
__global__ void __launch_bounds__(F*(M / E))
k_rows_fwd(const float* __restrict__ x, c32* __restrict__ T, int rows, int n_in,
           long long x_slice_stride, long long x_row_stride) {
  using S = FftShape<M, E>;
  constexpr int TT = S::T;
  extern __shared__ __align__(16) c32 smem[];
  const int f = threadIdx.x / TT;
  const int t = threadIdx.x - f * TT;
  const int z = blockIdx.y;
  const int row0 = blockIdx.x * (2 * F);
  c32* sm = smem + f * S::SB;

  const int ra = row0 + 2 * f, rb = ra + 1;
  const float* xa = x + z * x_slice_stride + (long long)ra * x_row_stride;
  const float* xb = xa + x_row_stride;
  const bool va = ra < rows, vb = rb < rows;
  c32 v[E];
#pragma unroll
  for (int m = 0; m < E; ++m) {
    const int j = t + TT * m;
    float a = 0.f, b = 0.f;
    if (j < n_in) {
      if (va) a = __ldg(xa + j);
      if (vb) b = __ldg(xb + j);
    }
    v[m] = mk(a, b);
  }
  fft<M, E, false>(v, sm, t);
#pragma unroll
  for (int m = 0; m < E; ++m) sm[pad_idx(t + TT * m)] = v[m];
  __syncthreads();

  // X_a(k) = (Z(k) + conj Z(-k))/2 ; X_b(k) = -i (Z(k) - conj Z(-k))/2
  constexpr int H = M / 2 + 1;
  c32* Tz = T + (long long)z * H * rows;
  for (int id = threadIdx.x; id < H * 2 * F; id += blockDim.x) {
    const int k = id / (2 * F);
    const int r = id - k * (2 * F);
    const int row = row0 + r;
    if (row >= rows) continue;
    const c32* s = smem + (r >> 1) * S::SB;
    const c32 zk = s[pad_idx(k)];
    const c32 zm = s[pad_idx((M - k) & (M - 1))];
    c32 o;
    if ((r & 1) == 0)
      o = scale(mk(zk.x + zm.x, zk.y - zm.y), 0.5f);
    else
      o = scale(mk(zk.y + zm.y, zm.x - zk.x), 0.5f);
    Tz[(long long)k * rows + row] = o;
  }
}

// ============================================================ K3: rows, inverse
// T: [nslices][M/2+1][rows] c32 half spectra; out: [nslices][rows][out_row_stride]
// out[n] = alpha * y[n] + beta * aux[n]  for n < n_out
template <int M, int E, int F>
__global__ void __launch_bounds__(F*(M / E))
k_rows_inv(const c32* __restrict__ T, float* __restrict__ out, const float* __restrict__ aux,
           int rows, int n_out, long long o_slice_stride, long long o_row_stride, float alpha,
           float beta) {
  using S = FftShape<M, E>;
  constexpr int TT = S::T;
  constexpr int H = M / 2 + 1;
  extern __shared__ __align__(16) c32 smem[];
  const int f = threadIdx.x / TT;
  const int t = threadIdx.x - f * TT;
  const int z = blockIdx.y;
  const int row0 = blockIdx.x * (2 * F);
  const c32* Tz = T + (long long)z * H * rows;

  // stage the 2F half-spectrum rows: group g holds Ya at [0,H) and Yb at [H,2H)
  for (int id = threadIdx.x; id < H * 2 * F; id += blockDim.x) {
    const int k = id / (2 * F);
    const int r = id - k * (2 * F);
    const int row = row0 + r;
    c32 val = mk(0.f, 0.f);
    if (row < rows) val = Tz[(long long)k * rows + row];
    if (k == 0 || k == M / 2) val.y = 0.f;  // irfft ignores Im of DC/Nyquist
    smem[(r >> 1) * S::SB + (r & 1) * H + k] = val;
  }
  __syncthreads();
  c32 v[E];
  {
    const c32* s = smem + f * S::SB;
#pragma unroll
    for (int m = 0; m < E; ++m) {
      const int j = t + TT * m;
      c32 za;
      if (j <= M / 2) {
        const c32 ya = s[j], yb = s[H + j];
        za = mk(ya.x - yb.y, ya.y + yb.x);  // Ya + i Yb
      } else {
        const c32 ya = s[M - j], yb = s[H + M - j];
        za = mk(ya.x + yb.y, yb.x - ya.y);  // conj(Ya) + i conj(Yb)
      }
      v[m] = za;
    }
  }
  __syncthreads();
  fft<M, E, true>(v, smem + f * S::SB, t);

  const int ra = row0 + 2 * f, rb = ra + 1;
  float* oa = out + z * o_slice_stride + (long long)ra * o_row_stride;
  float* ob = oa + o_row_stride;
  const float* aa = aux ? aux + z * o_slice_stride + (long long)ra * o_row_stride : nullptr;
  const float* ab = aux ? aa + o_row_stride : nullptr;
#pragma unroll
  for (int m = 0; m < E; ++m) {
    const int n = t + TT * m;
    if (n < n_out) {
      if (ra < rows) {
        float y = alpha * v[m].x;
        if (aa) y = fmaf(beta, __ldg(aa + n), y);
        oa[n] = y;
      }
      if (rb < rows) {
        float y = alpha * v[m].y;
        if (ab) y = fmaf(beta, __ldg(ab + n), y);
        ob[n] = y;
      }
    }
  }
}

// ============================================================ K2: column convolution
// T[z][c][0..col_len) in place; PSF columns PQ[c][kx], Bi[c][kx] (kx in [0,M))
template <int M, int E, int G, bool FLIP>
__global__ void __launch_bounds__(G*(M / E))
k_cols_conv(c32* __restrict__ T, const c32* __restrict__ PQ, const float* __restrict__ Bi,
            int ncols, int col_len, int nslices, long long slice_stride) {
  using S = FftShape<M, E>;
  constexpr int TT = S::T;
  extern __shared__ __align__(16) c32 smem[];
  const int g = threadIdx.x / TT;
  const int t = threadIdx.x - g * TT;
  c32* sm = smem + g * S::SB;
  const int nsteps = (ncols + G * gridDim.x - 1) / (G * gridDim.x);
  for (int step = 0; step < nsteps; ++step) {
    const int c = (step * gridDim.x + blockIdx.x) * G + g;
    const bool active = c < ncols;
    c32 pq[E];
    float bi[FLIP ? E : 1];
#pragma unroll
    for (int m = 0; m < E; ++m) {
      const int kx = t + TT * m;
      pq[m] = active ? PQ[(long long)c * M + kx] : mk(0.f, 0.f);
      if constexpr (FLIP) bi[m] = active ? Bi[(long long)c * M + kx] : 0.f;
    }
    c32* col = T + (long long)c * col_len;
    for (int z = 0; z < nslices; ++z) {
      c32* cz = col + z * slice_stride;
      c32 v[E];
#pragma unroll
      for (int m = 0; m < E; ++m) {
        const int j = t + TT * m;
        v[m] = (active && j < col_len) ? cz[j] : mk(0.f, 0.f);
      }
      fft<M, E, false>(v, sm, t);
#pragma unroll
      for (int m = 0; m < E; ++m) {
        if constexpr (FLIP) {
          // (Fr P + Fi Bi, Fi Q + Fr Bi)
          c32 p = pmul(v[m], pq[m]);
          v[m] = pfma(mk(v[m].y, v[m].x), mk(bi[m], bi[m]), p);
        } else {
          v[m] = pmul(v[m], pq[m]);
        }
      }
      // no barrier needed: the forward transform's last shared-memory read is
      // fenced by the barrier inside fft(), and its last pass is register-only
      fft<M, E, true>(v, sm, t);
#pragma unroll
      for (int m = 0; m < E; ++m) {
        const int j = t + TT * m;
        if (active && j < col_len) cz[j] = v[m];
      }
    }
  }
}

// forward-only column FFT (PSF spectra): S[z][c][kx] = FFT_ix(T[z][c][ix])
template <int M, int E, int G>
__global__ void __launch_bounds__(G*(M / E))
k_cols_fwd(const c32* __restrict__ T, c32* __restrict__ Sout, int ncols, int col_len,
           long long t_slice_stride, long long s_slice_stride) {
  using S = FftShape<M, E>;
  constexpr int TT = S::T;
  extern __shared__ __align__(16) c32 smem[];
  const int g = threadIdx.x / TT;
  const int t = threadIdx.x - g * TT;
  const int z = blockIdx.y;
  const int c = blockIdx.x * G + g;
  const bool active = c < ncols;
  const c32* col = T + z * t_slice_stride + (long long)c * col_len;
  c32 v[E];
#pragma unroll
  for (int m = 0; m < E; ++m) {
    const int j = t + TT * m;
    v[m] = (active && j < col_len) ? col[j] : mk(0.f, 0.f);
  }
  fft<M, E, false>(v, smem + g * S::SB, t);
  if (active) {
    c32* o = Sout + z * s_slice_stride + (long long)c * M;
#pragma unroll
    for (int m = 0; m < E; ++m) o[t + TT * m] = v[m];
  }
}

// ============================================================ K6: PSF lag kernels
// Dirichlet sum over the signed detector frequencies j in [jlo, jhi]
__device__ __forceinline__ double dirichlet(double u, int nd, int jlo, int jhi) {
  const double a = u / nd;
  const double den = sinpi(a);
  if (fabs(den) < 1e-12) {
    // u/nd within 1e-12 of an integer k: every cos(2 pi j k) = 1
    return (double)(jhi - jlo + 1);
  }
  return (sinpi((2.0 * jhi + 1.0) * a) - sinpi((2.0 * jlo - 1.0) * a)) / (2.0 * den);
}

// K_main and K_flip embedded circularly on the M x M grid (lag d at d mod M)
__global__ void k_psf_lags(float* __restrict__ kmain, float* __restrict__ kflip, int n, int M,
                           const double* __restrict__ cs, int n_angles, int nd) {
  const long long id = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (id >= (long long)M * M) return;
  const int i0 = (int)(id / M), i1 = (int)(id - (long long)i0 * M);
  const int d0 = i0 < n ? i0 : i0 - M;
  const int d1 = i1 < n ? i1 : i1 - M;
  float km = 0.f, kf = 0.f;
  if (d0 > -n && d1 > -n && (i0 < n || i0 > M - n) && (i1 < n || i1 > M - n)) {
    const int jlo = -(nd / 2), jhi = (nd + 1) / 2 - 1;
    const bool even = (nd % 2) == 0;
    double k = 0.0, kn = 0.0;
    for (int a = 0; a < n_angles; ++a) {
      const double u = d0 * cs[2 * a] + d1 * cs[2 * a + 1];
      k += dirichlet(u, nd, jlo, jhi);
      if (even) kn += cospi(u);
    }
    kn *= 0.5;
    km = (float)((k - kn) / nd);
    kf = (float)(-kn / nd);
  }
  kmain[id] = km;
  kflip[id] = kf;
}

// PQ/Bi from the two spectra S[2][c][kx] (c = ky in [0, M/2])
__global__ void k_psf_finish(const c32* __restrict__ spec, c32* __restrict__ PQ,
                             float* __restrict__ Bi, int n, int M, int flip) {
  const long long H = M / 2 + 1;
  const long long id = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (id >= H * M) return;
  const int c = (int)(id / M), kx = (int)(id - (long long)c * M);
  const double inv = 1.0 / ((double)M * (double)M);
  const double a = (double)spec[id].x * inv;
  double br = 0.0, bim = 0.0;
  if (flip) {
    const double sf = (double)spec[H * M + id].x * inv;
    // ph(kx) ph(ky) = e^{-2 pi i (kx + ky)(n-1)/M}
    const long long j = ((long long)(kx + c) * (n - 1)) % M;
    double s, co;
    sincospi(-2.0 * (double)j / M, &s, &co);
    br = sf * co;
    bim = sf * s;
  }
  PQ[id] = mk((float)(a + br), (float)(a - br));
  Bi[id] = (float)bim;
}

__global__ void k_twiddle_init(c32* tw) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= TW_MAX) return;
  double s, c;
  sincospi(-2.0 * (double)j / TW_MAX, &s, &c);
  tw[j] = mk((float)c, (float)s);
}


// ============================================================ host dispatch
namespace {

constexpr int E_DEFAULT = 16;

template <int M>
constexpr int eper() { return M < E_DEFAULT ? M : E_DEFAULT; }

template <int M>
constexpr int rows_f() {  // FFTs (row pairs) per CTA in K1/K3
  constexpr int T = M / eper<M>();
  constexpr int f = 512 / T;
  return f < 1 ? 1 : (f > 16 ? 16 : f);
}
template <int M>
constexpr int cols_g() {  // columns per CTA in K2
  constexpr int T = M / eper<M>();
  constexpr int g = 128 / T;
  return g < 1 ? 1 : g;
}

template <typename K>
int prep_kernel(K kern, size_t smem) {
  if (smem > 48 * 1024) {
    TF_TRY(check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smem),
                      "cudaFuncSetAttribute"));
  }
  return TF_OK;
}

template <int M>
int launch_rows_fwd(const float* x, c32* T, int rows, int n_in, long long xs, long long xr,
                    long long nslices, cudaStream_t st) {
  constexpr int E = eper<M>(), F = rows_f<M>();
  constexpr int TT = M / E;
  const size_t smem = sizeof(c32) * F * FftShape<M, E>::SB;
  auto kern = k_rows_fwd<M, E, F>;
  TF_TRY(prep_kernel(kern, smem));
  const int gx = (rows + 2 * F - 1) / (2 * F);
  KernelTimer tm;
  timer_begin(tm, 0, st);
  for (long long z0 = 0; z0 < nslices; z0 += 65535) {
    const int nz = (int)std::min<long long>(65535, nslices - z0);
    kern<<<dim3(gx, nz), F * TT, smem, st>>>(x + z0 * xs, T + z0 * (long long)(M / 2 + 1) * rows,
                                             rows, n_in, xs, xr);
  }
  timer_end(tm);
  return check_launch("k_rows_fwd");
}

template <int M>
int launch_rows_inv(const c32* T, float* out, const float* aux, int rows, int n_out,
                    long long os, long long orow, float alpha, float beta, long long nslices,
                    cudaStream_t st) {
  constexpr int E = eper<M>(), F = rows_f<M>();
  constexpr int TT = M / E;
  const size_t smem = sizeof(c32) * F * FftShape<M, E>::SB;
  auto kern = k_rows_inv<M, E, F>;
  TF_TRY(prep_kernel(kern, smem));
  const int gx = (rows + 2 * F - 1) / (2 * F);
  KernelTimer tm;
  timer_begin(tm, 2, st);
  for (long long z0 = 0; z0 < nslices; z0 += 65535) {
    const int nz = (int)std::min<long long>(65535, nslices - z0);
    kern<<<dim3(gx, nz), F * TT, smem, st>>>(T + z0 * (long long)(M / 2 + 1) * rows, out + z0 * os,
                                             aux ? aux + z0 * os : nullptr, rows, n_out, os, orow,
                                             alpha, beta);
  }
  timer_end(tm);
  return check_launch("k_rows_inv");
}

template <int M>
int launch_cols_conv(c32* T, const c32* PQ, const float* Bi, int col_len, long long nslices,
                     bool flip, cudaStream_t st) {
  constexpr int E = eper<M>(), G = cols_g<M>();
  constexpr int TT = M / E;
  const int ncols = M / 2 + 1;
  const size_t smem = sizeof(c32) * G * FftShape<M, E>::SB;
  int blocks_per_sm = 0;
  int grid = 0;
  const long long sstride = (long long)(M / 2 + 1) * col_len;
  KernelTimer tm;
  if (flip) {
    auto kern = k_cols_conv<M, E, G, true>;
    TF_TRY(prep_kernel(kern, smem));
    TF_TRY(check_cuda(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, kern, G * TT, smem),
                      "occupancy"));
    grid = std::max(1, std::min((ncols + G - 1) / G, blocks_per_sm * num_sms()));
    timer_begin(tm, 1, st);
    kern<<<grid, G * TT, smem, st>>>(T, PQ, Bi, ncols, col_len, (int)nslices, sstride);
  } else {
    auto kern = k_cols_conv<M, E, G, false>;
    TF_TRY(prep_kernel(kern, smem));
    TF_TRY(check_cuda(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, kern, G * TT, smem),
                      "occupancy"));
    grid = std::max(1, std::min((ncols + G - 1) / G, blocks_per_sm * num_sms()));
    timer_begin(tm, 1, st);
    kern<<<grid, G * TT, smem, st>>>(T, PQ, Bi, ncols, col_len, (int)nslices, sstride);
  }
  timer_end(tm);
  return check_launch("k_cols_conv");
}

template <int M>
int launch_cols_fwd(const c32* T, c32* Sout, int col_len, long long nslices, cudaStream_t st) {
  constexpr int E = eper<M>(), G = cols_g<M>();
  constexpr int TT = M / E;
  const int ncols = M / 2 + 1;
  const size_t smem = sizeof(c32) * G * FftShape<M, E>::SB;
  auto kern = k_cols_fwd<M, E, G>;
  TF_TRY(prep_kernel(kern, smem));
  kern<<<dim3((ncols + G - 1) / G, (unsigned)nslices), G * TT, smem, st>>>(
      T, Sout, ncols, col_len, (long long)ncols * col_len, (long long)ncols * M);
  return check_launch("k_cols_fwd");
}

// compile-time dispatch over the supported power-of-two sides
template <template <int> class Fn, typename... A>
int dispatch_m(int M, A... args) {
  switch (M) {
    case 8: return Fn<8>::run(args...);
    case 16: return Fn<16>::run(args...);
    case 32: return Fn<32>::run(args...);
    case 64: return Fn<64>::run(args...);
    case 128: return Fn<128>::run(args...);
    case 256: return Fn<256>::run(args...);
    case 512: return Fn<512>::run(args...);
    case 1024: return Fn<1024>::run(args...);
    case 2048: return Fn<2048>::run(args...);
    case 4096: return Fn<4096>::run(args...);
    case 8192: return Fn<8192>::run(args...);
    default: return fail_arg("unsupported FFT side %d", M);
  }
}

template <int M>
struct ApplyFn {
  static int run(const float* x, float* out, const float* aux, float alpha, float beta,
                 long long nslices, int n, const c32* PQ, const float* Bi, bool flip, c32* T,
                 long long chunk, cudaStream_t st) {
    const long long img = (long long)n * n;
    for (long long z0 = 0; z0 < nslices; z0 += chunk) {
      const long long nz = std::min(chunk, nslices - z0);
      TF_TRY(launch_rows_fwd<M>(x + z0 * img, T, n, n, img, n, nz, st));
      TF_TRY(launch_cols_conv<M>(T, PQ, Bi, n, nz, flip, st));
      TF_TRY(launch_rows_inv<M>(T, out + z0 * img, aux ? aux + z0 * img : nullptr, n, n, img, n,
                                alpha, beta, nz, st));
    }
    return TF_OK;
  }
};

template <int M>
struct PsfFn {
  static int run(int n, const double* cs, int n_angles, int nd, c32* PQ, float* Bi, char* ws,
                 cudaStream_t st) {
    // ws: lags [2][M][M] f32 | T [2][M/2+1][M] c32 | spec [2][M/2+1][M] c32
    const long long MM = (long long)M * M;
    const long long H = M / 2 + 1;
    float* lags = reinterpret_cast<float*>(ws);
    c32* T = reinterpret_cast<c32*>(ws + 2 * MM * sizeof(float));
    c32* spec = T + 2 * H * M;
    const bool flip = (nd % 2) == 0;
    {
      const int bs = 256;
      const long long nb = (MM + bs - 1) / bs;
      k_psf_lags<<<(unsigned)nb, bs, 0, st>>>(lags, lags + MM, n, M, cs, n_angles, nd);
      TF_TRY(check_launch("k_psf_lags"));
    }
    TF_TRY(launch_rows_fwd<M>(lags, T, M, M, MM, M, flip ? 2 : 1, st));
    TF_TRY(launch_cols_fwd<M>(T, spec, M, flip ? 2 : 1, st));
    {
      const int bs = 256;
      const long long nb = (H * M + bs - 1) / bs;
      k_psf_finish<<<(unsigned)nb, bs, 0, st>>>(spec, PQ, Bi, n, M, flip ? 1 : 0);
      TF_TRY(check_launch("k_psf_finish"));
    }
    return TF_OK;
  }
};

}  // namespace

int toeplitz_apply(const float* x, float* out, const float* aux, float alpha, float beta,
                   long long nslices, int n, int M, const void* PQ, const float* Bi, bool flip,
                   void* ws, size_t ws_bytes, cudaStream_t st) {
  const long long per = (long long)(M / 2 + 1) * n * (long long)sizeof(c32);
  const long long chunk = (long long)(ws_bytes / per);
  if (chunk < 1) return fail_arg("toeplitz workspace too small: %zu < %lld", ws_bytes, per);
  return dispatch_m<ApplyFn>(M, x, out, aux, alpha, beta, nslices, n,
                             reinterpret_cast<const c32*>(PQ), Bi, flip,
                             reinterpret_cast<c32*>(ws), chunk, st);
}

size_t psf_workspace_bytes(int M) {
  const size_t MM = (size_t)M * M, H = M / 2 + 1;
  return 2 * MM * sizeof(float) + 4 * H * M * sizeof(c32);
}

int psf_build(int n, int M, const double* cs, int n_angles, int nd, void* PQ, float* Bi,
              void* ws, size_t ws_bytes, cudaStream_t st) {
  if (ws_bytes < psf_workspace_bytes(M)) return fail_arg("psf workspace too small");
  return dispatch_m<PsfFn>(M, n, cs, n_angles, nd, reinterpret_cast<c32*>(PQ), Bi,
                           reinterpret_cast<char*>(ws), st);
}

int init_twiddles() {
  c32* p = nullptr;
  TF_TRY(check_cuda(cudaGetSymbolAddress((void**)&p, g_twiddle), "cudaGetSymbolAddress"));
  k_twiddle_init<<<(TW_MAX + 255) / 256, 256>>>(p);
  TF_TRY(check_launch("k_twiddle_init"));
  return check_cuda(cudaDeviceSynchronize(), "twiddle init sync");
}

}  // namespace tf
