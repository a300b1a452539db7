// Toeplitz apply and PSF build on M = 5Q grids (Q = 256, 512, 1024), the C5
// sides N = 640, 1280, 2560 (BASELINE configs[4]).
//
// Same algorithm and HBM layout as toeplitz.cu (row-blocked half spectrum
// T[z][rb][ky][r], PQ/Bi folded PSF); only the transform length
// changes: M = 5Q through tf_fft5.cuh (a radix-5 DIF step and five Q-point
// transforms of the power-of-two engine).  One transform per CTA of 5Q/16
// threads:
//   K1 k5_rows_fwd  : a row pair x_a + i x_b, forward 5Q FFT, Z(k) to shared
//                     memory in natural order, split into the two half spectra,
//                     16-byte stores (half a row block).
//   K2 k5_cols_conv : one column per CTA, PSF in registers (layout G) across all
//                     slices; gather, forward 5Q FFT, Y = F A + conj(F) B,
//                     inverse, keep ix < N, scatter back in place.
//   K3 k5_rows_inv  : a row pair's Hermitian spectrum gathered in layout G,
//                     inverse 5Q FFT, crop, out = alpha y + beta aux.
//   k5_cols_fwd     : forward column FFT of the PSF lag grids.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>

#include "tf_async.cuh"
#include "tf_common.cuh"
#include "tf_fft5.cuh"

namespace tf {

int encode_tmap(CUtensorMap* map, c32* T, int M, int nrb, long long nslices, int boxr);

namespace {

constexpr int RB5 = 4;  // rows per block of the half-spectrum layout (toeplitz.cu RB)
__host__ __device__ constexpr int nrb5(int rows) { return (rows + RB5 - 1) / RB5; }
__device__ __forceinline__ long long tidx5(int z, int ix, int c, int nrb, int H) {
  return (((long long)z * nrb + (ix >> 2)) * H + c) * RB5 + (ix & 3);
}

// K1: unit = row pair (blockIdx.x), slice blockIdx.y
template <int Q, bool ZIN>
__global__ void __launch_bounds__(Fft5Shape<Q>::T5)
k5_rows_fwd(const float* __restrict__ x, c32* __restrict__ T, int rows, int n_in,
            long long xs, long long xr) {
  using S = Fft5Shape<Q>;
  constexpr int M = S::M, H = M / 2 + 1, TP = S::TP;
  extern __shared__ __align__(16) c32 smem[];
  const int p = threadIdx.x;
  const int z = blockIdx.y;
  const int u = blockIdx.x, r0 = 2 * u, rb = u >> 1, b0 = u & 1;
  const int nrb = nrb5(rows);
  const float* xa = x + z * xs + (long long)r0 * xr;
  const bool has_b = r0 + 1 < rows;
  c32 xi[20];
#pragma unroll
  for (int m = 0; m < 20; ++m) {
    const int n = p + S::TI * m;
    float a = 0.f, c = 0.f;
    if (p < S::TI && n < n_in && (!ZIN || m < 10)) {
      a = __ldg(xa + n);
      if (has_b) c = __ldg(xa + xr + n);
    }
    xi[m] = mk(a, c);
  }
  c32 v[16];
  fft5_fwd<Q, ZIN>(xi, v, smem, p);
  const int g = p / TP, t = p - g * TP;
#pragma unroll
  for (int m = 0; m < 16; ++m) smem[5 * (t + TP * m) + g] = v[m];
  __syncthreads();
  float4* dst = reinterpret_cast<float4*>(T + ((long long)z * nrb + rb) * H * RB5);
  auto emit = [&](int k) {
    const c32 zk = smem[k];
    const c32 zm = smem[k == 0 ? 0 : M - k];
    const c32 a = scale(mk(zk.x + zm.x, zk.y - zm.y), 0.5f);
    const c32 b = scale(mk(zk.y + zm.y, zm.x - zk.x), 0.5f);
    dst[2 * k + b0] = make_float4(a.x, a.y, b.x, b.y);
  };
#pragma unroll
  for (int m = 0; m < 8; ++m) emit(p + S::T5 * m);  // k < M/2 = 8 T5
  if (p == 0) emit(M / 2);
}

// K3: unit = row pair (blockIdx.x), slice blockIdx.y
template <int Q>
__global__ void __launch_bounds__(Fft5Shape<Q>::T5)
k5_rows_inv(const c32* __restrict__ T, float* __restrict__ out, const float* __restrict__ aux,
            int rows, int n_out, long long os, long long orow, float alpha, float beta,
            int pf_dist) {
  using S = Fft5Shape<Q>;
  constexpr int M = S::M, H = M / 2 + 1, TP = S::TP;
  extern __shared__ __align__(16) c32 smem[];
  const int p = threadIdx.x;
  const int z = blockIdx.y;
  const int u = blockIdx.x, r0 = 2 * u, rb = u >> 1, b0 = u & 1;
  const int nrb = nrb5(rows);
  // L2 prefetch of the row block (both row pairs) and aux rows of the CTA pf_dist
  // blocks ahead, as K3 of the power-of-two path: the loads below are latency-bound
  // (long-scoreboard stalls) otherwise
  if (pf_dist > 0 && p == 32) {
    const long long lin = (long long)blockIdx.y * gridDim.x + blockIdx.x + pf_dist;
    if (lin < (long long)gridDim.x * gridDim.y) {
      const int zz = (int)(lin / gridDim.x), uu = (int)(lin - (long long)zz * gridDim.x);
      if ((uu & 1) == 0) {
        bulk_prefetch_l2(T + ((long long)zz * nrb + (uu >> 1)) * H * RB5,
                         (uint32_t)(H * RB5 * sizeof(c32)));
      }
      if (aux && (n_out * sizeof(float)) % 16 == 0 && (orow * sizeof(float)) % 16 == 0 &&
          (os * sizeof(float)) % 16 == 0 && reinterpret_cast<uintptr_t>(aux) % 16 == 0) {
        for (int q = 0; q < 2 && 2 * uu + q < rows; ++q)
          bulk_prefetch_l2(aux + zz * os + (long long)(2 * uu + q) * orow,
                           (uint32_t)(n_out * sizeof(float)));
      }
    }
  }
  const float4* src = reinterpret_cast<const float4*>(T + ((long long)z * nrb + rb) * H * RB5);
  const int g = p / TP, t = p - g * TP;
  // the row pair's half spectrum (Ya, Yb)(k), k <= M/2: coalesced loads into shared
  // memory in natural order, then gathered in layout G (16-byte words at stride 5:
  // conflict-free quarter warps)
  float4* stage = reinterpret_cast<float4*>(smem);
  static_assert(2 * (M / 2 + 1) <= S::SMEM_WORDS, "stage fits the exchange buffers");
#pragma unroll
  for (int m = 0; m < 8; ++m) {
    const int k = p + S::T5 * m;
    float4 y = __ldg(src + 2 * k + b0);
    if (k == 0) {  // irfft drops Im(DC, Nyquist)
      y.y = 0.f;
      y.w = 0.f;
    }
    stage[k] = y;
  }
  if (p == 0) {
    float4 y = __ldg(src + 2 * (M / 2) + b0);
    y.y = 0.f;
    y.w = 0.f;
    stage[M / 2] = y;
  }
  __syncthreads();
  c32 v[16];
#pragma unroll
  for (int m = 0; m < 16; ++m) {
    const int k = 5 * (t + TP * m) + g;
    const bool hi = k > M / 2;
    const float4 y = stage[hi ? M - k : k];
    v[m] = hi ? mk(y.x + y.w, y.z - y.y)   // conj(Ya) + i conj(Yb)
              : mk(y.x - y.w, y.y + y.z);  // Ya + i Yb
  }
  __syncthreads();  // the transform reuses the stage
  c32 xo[20];
  fft5_inv<Q, true>(v, xo, smem, p);
  if (p >= S::TI) return;
  const long long zo = z * os;
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int r = r0 + q;
    if (r >= rows) break;
    float* o = out + zo + (long long)r * orow;
    const float* a = aux ? aux + zo + (long long)r * orow : nullptr;
#pragma unroll
    for (int m = 0; m < 10; ++m) {
      const int n = p + S::TI * m;
      if (n < n_out) {
        float y = alpha * (q ? xo[m].y : xo[m].x);
        if (a) y = fmaf(beta, __ldg(a + n), y);
        o[n] = y;
      }
    }
  }
}

// K2: column c = blockIdx.x + i gridDim.x, all slices; col_len <= M/2
template <int Q, bool FLIP>
__global__ void __launch_bounds__(Fft5Shape<Q>::T5)
k5_cols_conv(c32* __restrict__ T, const c32* __restrict__ PQ, const float* __restrict__ Bi,
             int ncols, int col_len, int nslices) {
  using S = Fft5Shape<Q>;
  constexpr int M = S::M, H = M / 2 + 1, TP = S::TP;
  extern __shared__ __align__(16) c32 smem[];
  const int p = threadIdx.x;
  const int g = p / TP, t = p - g * TP;
  const int nrb = nrb5(col_len);
  for (int c = blockIdx.x; c < ncols; c += gridDim.x) {
    c32 pq[16];
    float bi[FLIP ? 16 : 1];
#pragma unroll
    for (int m = 0; m < 16; ++m) {
      const int kx = 5 * (t + TP * m) + g;
      pq[m] = __ldg(PQ + (long long)c * M + kx);
      if constexpr (FLIP) bi[m] = __ldg(Bi + (long long)c * M + kx);
    }
    // the next slice's column is loaded while this one is transformed
    c32 nxt[10];
    auto gather = [&](int z) {
#pragma unroll
      for (int m = 0; m < 10; ++m) {
        const int j = p + S::TI * m;
        nxt[m] = (p < S::TI && j < col_len) ? T[tidx5(z, j, c, nrb, H)] : mk(0.f, 0.f);
      }
    };
    gather(0);
    for (int z = 0; z < nslices; ++z) {
      c32 xi[20];
#pragma unroll
      for (int m = 0; m < 10; ++m) xi[m] = nxt[m];
      if (z + 1 < nslices) gather(z + 1);
      c32 v[16];
      fft5_fwd<Q, true>(xi, v, smem, p);
#pragma unroll
      for (int m = 0; m < 16; ++m) {
        if constexpr (FLIP) {
          v[m] = pfma(mk(v[m].y, v[m].x), mk(bi[m], bi[m]), pmul(v[m], pq[m]));
        } else {
          v[m] = pmul(v[m], pq[m]);
        }
      }
      c32 xo[20];
      fft5_inv<Q, true>(v, xo, smem, p);
      if (p < S::TI) {
#pragma unroll
        for (int m = 0; m < 10; ++m) {
          const int j = p + S::TI * m;
          if (j < col_len) T[tidx5(z, j, c, nrb, H)] = xo[m];
        }
      }
    }
  }
}

// K2 for M = 5120 (Q = 1024, the C5 finest level) in the style of k_cols_conv64:
// a group of five warps per (column, slice) item, three groups per CTA, one CTA per
// SM.  With n = n1 + Q n2 and k = 5 k1 + k2 (tf_fft5.cuh):
// * layout I (128 threads, eight n1 each): the radix-5 step over n2 with the
//   W_M^{n1 k2} twiddles, written to sub-buffer k2 at word n1 + n1/32;
// * layout G (warp k2 of the group, lane t): the Q-point transform of z_k2 as two
//   radix-32 passes (E = 32) whose one exchange stays inside the warp (__syncwarp);
//   it leaves X[5 (t + 32 m) + k2] in register m for the PSF product (the column's
//   PSF bulk-copied to shared memory once per column, shared by the groups);
// * the inverse runs the same way back, then the inverse radix-5 step in layout I
//   writes the kept outputs n < N straight to the half spectrum.
// Three group barriers per item instead of the ~10 CTA barriers and six exchanges
// of k5_cols_conv; the next item is TMA-gathered into the group's buffer as soon as
// the last exchange has been read.
template <bool FLIP, int G>
__global__ void __launch_bounds__(G * 160, 1)
k5_cols_conv_q1024(const __grid_constant__ CUtensorMap tmap, const c32* __restrict__ PQ,
                   const float* __restrict__ Bi, int ncols, int nrb, int nslices, int boxr,
                   c32* __restrict__ T) {
  constexpr int Q = 1024, M = 5 * Q, H = M / 2 + 1, E = 32, TQ = Q / E;
  constexpr int GT = 5 * TQ;          // 160 threads per group
  constexpr int TI = Q / 8;           // layout I: 128 threads x 8 n1
  constexpr int SW = Q + Q / TQ;      // sub-buffer words (pad 1 per 32)
  constexpr int XW = 5 * SW;          // group buffer words
  using S = FftShape<Q, E>;
  static_assert(S::NP == 2 && (1 << S::LFIRST) == TQ, "two radix-32 passes");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int g = threadIdx.x / GT, p = threadIdx.x - g * GT;
  const int k2 = p / TQ, t = p - k2 * TQ;  // layout G: warp k2, lane t
  c32* pq_s = reinterpret_cast<c32*>(smem_raw);
  float* bi_s = reinterpret_cast<float*>(pq_s + M);
  c32* xb = reinterpret_cast<c32*>(bi_s + M) + g * XW;
  c32* tw5s = reinterpret_cast<c32*>(bi_s + M) + G * XW;  // W_M^{n1}, n1 < Q
  uint64_t* bars = reinterpret_cast<uint64_t*>(tw5s + Q);
  uint64_t* full = bars + 2 * g;
  uint64_t* empty = full + 1;
  uint64_t* psf_full = bars + 2 * G;
  const int bar_id = 1 + g;
  // the radix-5 step's base twiddles, read 16 times per item: shared memory, not L1/L2
  for (int i = threadIdx.x; i < Q; i += G * GT) tw5s[i] = g_tw5[(Q - Q5_MIN) + i];
  if (threadIdx.x == 0) mbar_init(psf_full, 1);
  if (p == 0) {
    mbar_init(full, 1);
    mbar_init(empty, GT);
  }
  if (threadIdx.x == 0) fence_mbar_init();
  __syncthreads();
  if ((int)blockIdx.x >= ncols) return;
  const bool active = g < nslices;
  const int my_cols = (ncols - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
  const int nz_g = active ? (nslices - g + G - 1) / G : 0;
  const int nitems = my_cols * nz_g;
  const int nbox = (nrb + boxr - 1) / boxr;
  const uint32_t box_bytes = (uint32_t)boxr * RB5 * sizeof(c32);
  const int col_len = nrb * RB5;
  int p_col = blockIdx.x, p_z = g, issued = 0;
  auto issue = [&]() {
    mbar_expect_tx(full, nbox * box_bytes);
    for (int q = 0; q < nbox; ++q)
      tma_load_4d(xb + q * boxr * RB5, &tmap, 0, p_col, q * boxr, p_z, full);
    ++issued;
    p_z += G;
    if (p_z >= nslices) {
      p_z = g;
      p_col += gridDim.x;
    }
  };
  if (p == 0 && nitems > 0) {
    tma_prefetch_desc(&tmap);
    issue();
  }
  PassTw<Q, E, 1> tw;
  tw.from_table(t);
  c32* sub = xb + k2 * SW;  // this warp's sub-buffer
  // one radix-32 exchange inside the warp: pass-0 outputs of lane t are words t*32 + r
  // (padded t*33 + r), the canonical reads t + 32 m (padded t + 33 m)
  auto warp_exchange = [&](c32 (&v)[1][E]) {
    __syncwarp();
#pragma unroll
    for (int r = 0; r < E; ++r) sub[t * (TQ + 1) + r] = v[0][r];
    __syncwarp();
#pragma unroll
    for (int m = 0; m < E; ++m) v[0][m] = sub[t + (TQ + 1) * m];
  };
  const long long rb_stride = (long long)H * RB5;
  const long long slice_stride = (long long)nrb * rb_stride;
  int item = 0;
  for (int kc = 0; kc < my_cols; ++kc) {
    const int c = blockIdx.x + kc * gridDim.x;
    __syncthreads();  // every group is done with the previous column's PSF
    if (threadIdx.x == 0) {
      mbar_expect_tx(psf_full, M * (uint32_t)(sizeof(c32) + (FLIP ? sizeof(float) : 0)));
      bulk_g2s(pq_s, PQ + (long long)c * M, M * sizeof(c32), psf_full);
      if constexpr (FLIP) bulk_g2s(bi_s, Bi + (long long)c * M, M * sizeof(float), psf_full);
      if (kc + 1 < my_cols) {
        bulk_prefetch_l2(PQ + (long long)(c + gridDim.x) * M, M * sizeof(c32));
        if constexpr (FLIP) bulk_prefetch_l2(Bi + (long long)(c + gridDim.x) * M, M * sizeof(float));
      }
    }
    bool psf_ready = false;
    for (int z = g; active && z < nslices; z += G, ++item) {
      mbar_wait(full, (uint32_t)(item & 1));
      // ---- forward radix-5 step, layout I (the input sits in xb[0, col_len))
      c32 a5[8][3];
      if (p < TI) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int n1 = p + TI * j;
#pragma unroll
          for (int n2 = 0; n2 < 3; ++n2) {
            const int n = n1 + Q * n2;
            a5[j][n2] = n < col_len ? xb[n] : mk(0.f, 0.f);
          }
        }
      }
      named_bar_sync(bar_id, GT);  // the input has been read: xb takes the sub-buffers
      if (p < TI) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int n1 = p + TI * j;
          c32 a[5] = {a5[j][0], a5[j][1], a5[j][2], mk(0.f, 0.f), mk(0.f, 0.f)};
          dft5<false>(a);
          c32 w[5];
          w[1] = tw5s[n1];
          w[2] = cmul(w[1], w[1]);
          w[3] = cmul(w[2], w[1]);
          w[4] = cmul(w[2], w[2]);
          const int word = n1 + n1 / TQ;
          xb[word] = a[0];
#pragma unroll
          for (int kk = 1; kk < 5; ++kk) xb[kk * SW + word] = cmul(a[kk], w[kk]);
        }
      }
      named_bar_sync(bar_id, GT);
      // ---- forward Q-point transform of z_k2, layout G
      c32 v[1][E];
#pragma unroll
      for (int m = 0; m < E; ++m) v[0][m] = sub[t + (TQ + 1) * m];
      fft_pass<Q, E, 0, false, false, false, 1>(v, (const PassTw<Q, E, 0>*)nullptr);
      warp_exchange(v);
      fft_pass<Q, E, 1, false, false, false, 1>(v, &tw);
      if (!psf_ready) {
        mbar_wait(psf_full, (uint32_t)(kc & 1));
        psf_ready = true;
      }
#pragma unroll
      for (int m = 0; m < E; ++m) {
        const int kx = 5 * (t + TQ * m) + k2;
        const c32 pq = pq_s[kx];
        if constexpr (FLIP) {
          const float bi = bi_s[kx];
          v[0][m] = pfma(mk(v[0][m].y, v[0][m].x), mk(bi, bi), pmul(v[0][m], pq));
        } else {
          v[0][m] = pmul(v[0][m], pq);
        }
      }
      // ---- inverse Q-point transform, then back to layout I
      fft_pass<Q, E, 0, true, false, false, 1>(v, (const PassTw<Q, E, 0>*)nullptr);
      warp_exchange(v);
      fft_pass<Q, E, 1, true, false, false, 1>(v, &tw);
      __syncwarp();
#pragma unroll
      for (int m = 0; m < E; ++m) sub[t + (TQ + 1) * m] = v[0][m];
      named_bar_sync(bar_id, GT);
      if (p < TI) {
        c32* dst = T + z * slice_stride + (long long)c * RB5;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int n1 = p + TI * j;
          const int word = n1 + n1 / TQ;
          c32 w[5];
          w[1] = tw5s[n1];
          w[2] = cmul(w[1], w[1]);
          w[3] = cmul(w[2], w[1]);
          w[4] = cmul(w[2], w[2]);
          c32 a[5];
          a[0] = xb[word];
#pragma unroll
          for (int kk = 1; kk < 5; ++kk) a[kk] = cmulc(xb[kk * SW + word], w[kk]);
          dft5<true>(a);
#pragma unroll
          for (int n2 = 0; n2 < 3; ++n2) {
            const int n = n1 + Q * n2;
            if (n < col_len) dst[(long long)(n >> 2) * rb_stride + (n & 3)] = a[n2];
          }
        }
      }
      mbar_arrive(empty);  // this thread's reads of xb are done
      if (p == 0 && issued < nitems) {
        mbar_wait(empty, (uint32_t)(item & 1));
        issue();
      }
    }
  }
}

// forward column FFT of full-length columns (PSF spectra): S[z][c][kx]
template <int Q>
__global__ void __launch_bounds__(Fft5Shape<Q>::T5)
k5_cols_fwd(const c32* __restrict__ T, c32* __restrict__ Sout, int ncols, int col_len,
            long long s_slice_stride) {
  using S = Fft5Shape<Q>;
  constexpr int M = S::M, H = M / 2 + 1, TP = S::TP;
  extern __shared__ __align__(16) c32 smem[];
  const int p = threadIdx.x;
  const int z = blockIdx.y, c = blockIdx.x;
  const int nrb = nrb5(col_len);
  c32 xi[20];
#pragma unroll
  for (int m = 0; m < 20; ++m) {
    const int j = p + S::TI * m;
    xi[m] = (p < S::TI && j < col_len) ? T[tidx5(z, j, c, nrb, H)] : mk(0.f, 0.f);
  }
  c32 v[16];
  fft5_fwd<Q, false>(xi, v, smem, p);
  const int g = p / TP, t = p - g * TP;
  c32* o = Sout + z * s_slice_stride + (long long)c * M;
#pragma unroll
  for (int m = 0; m < 16; ++m) o[5 * (t + TP * m) + g] = v[m];
}

template <int Q>
size_t smem5() {
  return sizeof(c32) * (size_t)Fft5Shape<Q>::SMEM_WORDS;
}

template <int Q>
int rows_fwd5(const float* x, c32* T, int rows, int n_in, long long xs, long long xr,
              long long nslices, cudaStream_t st) {
  using S = Fft5Shape<Q>;
  const size_t sm = smem5<Q>();
  const bool zin = 2 * n_in <= S::M;
  auto kern = zin ? k5_rows_fwd<Q, true> : k5_rows_fwd<Q, false>;
  TF_TRY(prep_kernel(kern, sm));
  const int units = (rows + 1) / 2;
  KernelTimer tm;
  timer_begin(tm, 0, st);
  for (long long z0 = 0; z0 < nslices; z0 += 65535) {
    const int nz = (int)std::min<long long>(65535, nslices - z0);
    c32* Tz = T + z0 * (long long)(S::M / 2 + 1) * RB5 * nrb5(rows);
    kern<<<dim3(units, nz), S::T5, sm, st>>>(x + z0 * xs, Tz, rows, n_in, xs, xr);
  }
  timer_end(tm);
  return check_launch("k5_rows_fwd");
}

// L2 prefetch distance of k5_rows_inv in multiples of the SM count (0 = off)
#ifndef TF_K5_PF_MUL
#define TF_K5_PF_MUL 1
#endif
template <int Q>
int rows_inv5(const c32* T, float* out, const float* aux, int rows, int n_out, long long os,
              long long orow, float alpha, float beta, long long nslices, cudaStream_t st) {
  using S = Fft5Shape<Q>;
  if (2 * n_out > S::M) return fail_arg("k5_rows_inv: n_out %d exceeds M/2", n_out);
  const size_t sm = smem5<Q>();
  TF_TRY(prep_kernel(k5_rows_inv<Q>, sm));
  const int units = (rows + 1) / 2;
  KernelTimer tm;
  timer_begin(tm, 2, st);
  for (long long z0 = 0; z0 < nslices; z0 += 65535) {
    const int nz = (int)std::min<long long>(65535, nslices - z0);
    k5_rows_inv<Q><<<dim3(units, nz), S::T5, sm, st>>>(
        T + z0 * (long long)(S::M / 2 + 1) * RB5 * nrb5(rows), out + z0 * os,
        aux ? aux + z0 * os : nullptr, rows, n_out, os, orow, alpha, beta,
        TF_K5_PF_MUL * num_sms());
  }
  timer_end(tm);
  return check_launch("k5_rows_inv");
}

#ifndef TF_K5_GROUPS
#define TF_K5_GROUPS 3
#endif
template <bool FLIP>
int cols_conv5_q1024(c32* T, const c32* PQ, const float* Bi, int col_len, long long nslices,
                     cudaStream_t st) {
  constexpr int Q = 1024, M = 5 * Q, G = TF_K5_GROUPS;
  const int ncols = M / 2 + 1;
  const int nrb = nrb5(col_len);
  const int boxr = std::min(nrb, 256);
  CUtensorMap map;
  TF_TRY(encode_tmap(&map, T, M, nrb, nslices, boxr));
  const size_t smem = (sizeof(c32) + sizeof(float)) * M + sizeof(c32) * G * 5 * (Q + Q / 32) +
                      sizeof(c32) * Q + (2 * G + 1) * sizeof(uint64_t);
  auto kern = k5_cols_conv_q1024<FLIP, G>;
  TF_TRY(prep_kernel(kern, smem));
  const int grid = std::max(1, std::min(ncols, num_sms()));
  KernelTimer tm;
  timer_begin(tm, 1, st);
  kern<<<grid, G * 160, smem, st>>>(map, PQ, Bi, ncols, nrb, (int)nslices, boxr, T);
  timer_end(tm);
  return check_launch("k5_cols_conv_q1024");
}

#ifndef TF_K2_Q1024
#define TF_K2_Q1024 1
#endif

template <int Q>
int cols_conv5(c32* T, const c32* PQ, const float* Bi, int col_len, long long nslices, bool flip,
               cudaStream_t st) {
  using S = Fft5Shape<Q>;
  if (2 * col_len > S::M) return fail_arg("k5_cols_conv: column length %d exceeds M/2", col_len);
  if constexpr (TF_K2_Q1024 && Q == 1024) {
    return flip ? cols_conv5_q1024<true>(T, PQ, Bi, col_len, nslices, st)
                : cols_conv5_q1024<false>(T, PQ, Bi, col_len, nslices, st);
  }
  const size_t sm = smem5<Q>();
  auto kern = flip ? k5_cols_conv<Q, true> : k5_cols_conv<Q, false>;
  TF_TRY(prep_kernel(kern, sm));
  int per_sm = 0;
  TF_TRY(check_cuda(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, S::T5, sm),
                    "occupancy"));
  const int ncols = S::M / 2 + 1;
  const int grid = std::max(1, std::min(ncols, std::max(1, per_sm) * num_sms()));
  KernelTimer tm;
  timer_begin(tm, 1, st);
  kern<<<grid, S::T5, sm, st>>>(T, PQ, Bi, ncols, col_len, (int)nslices);
  timer_end(tm);
  return check_launch("k5_cols_conv");
}

template <int Q>
int apply5(const float* x, float* out, const float* aux, float alpha, float beta,
           long long nslices, int n, const c32* PQ, const float* Bi, bool flip, c32* T,
           long long chunk, cudaStream_t st) {
  const long long img = (long long)n * n;
  for (long long z0 = 0; z0 < nslices; z0 += chunk) {
    const long long nz = std::min(chunk, nslices - z0);
    TF_TRY(rows_fwd5<Q>(x + z0 * img, T, n, n, img, n, nz, st));
    TF_TRY(cols_conv5<Q>(T, PQ, Bi, n, nz, flip, st));
    TF_TRY(rows_inv5<Q>(T, out + z0 * img, aux ? aux + z0 * img : nullptr, n, n, img, n, alpha,
                        beta, nz, st));
  }
  return TF_OK;
}

__global__ void k5_psf_finish(const c32* __restrict__ spec, c32* __restrict__ PQ,
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
    const long long j = ((long long)(kx + c) * (n - 1)) % M;
    double s, co;
    sincospi(-2.0 * (double)j / M, &s, &co);
    br = sf * co;
    bim = sf * s;
  }
  PQ[id] = mk((float)(a + br), (float)(a - br));
  Bi[id] = (float)bim;
}

template <int Q>
int psf5(int n, const double* cs, int n_angles, int nd, c32* PQ, float* Bi, char* ws,
         cudaStream_t st) {
  using S = Fft5Shape<Q>;
  constexpr int M = S::M;
  const long long MM = (long long)M * M;
  const long long H = M / 2 + 1;
  float* lags = reinterpret_cast<float*>(ws);
  c32* T = reinterpret_cast<c32*>(ws + 2 * MM * sizeof(float));
  c32* spec = T + 2 * H * M;
  const bool flip = (nd % 2) == 0;
  TF_TRY(psf_lags_launch(lags, n, M, cs, n_angles, nd, st));
  TF_TRY(rows_fwd5<Q>(lags, T, M, M, MM, M, flip ? 2 : 1, st));
  const size_t sm = smem5<Q>();
  TF_TRY(prep_kernel(k5_cols_fwd<Q>, sm));
  k5_cols_fwd<Q><<<dim3((unsigned)H, flip ? 2 : 1), S::T5, sm, st>>>(T, spec, (int)H, M, H * M);
  TF_TRY(check_launch("k5_cols_fwd"));
  const int bs = 256;
  k5_psf_finish<<<(unsigned)((H * M + bs - 1) / bs), bs, 0, st>>>(spec, PQ, Bi, n, M, flip ? 1 : 0);
  return check_launch("k5_psf_finish");
}

template <template <int> class Fn, typename... A>
int dispatch_q(int M, A... args) {
  switch (M) {
    case 5 * 256: return Fn<256>::run(args...);
    case 5 * 512: return Fn<512>::run(args...);
    case 5 * 1024: return Fn<1024>::run(args...);
    default: return fail_arg("unsupported FFT side %d", M);
  }
}

template <int Q>
struct Apply5Fn {
  template <typename... A>
  static int run(A... a) { return apply5<Q>(a...); }
};
template <int Q>
struct Psf5Fn {
  template <typename... A>
  static int run(A... a) { return psf5<Q>(a...); }
};

}  // namespace

bool is_side5(int M) { return M == 5 * 256 || M == 5 * 512 || M == 5 * 1024; }

int toeplitz_apply5(const float* x, float* out, const float* aux, float alpha, float beta,
                    long long nslices, int n, int M, const void* PQ, const float* Bi, bool flip,
                    void* ws, size_t ws_bytes, cudaStream_t st) {
  const long long per = (long long)(M / 2 + 1) * RB5 * nrb5(n) * (long long)sizeof(c32);
  const long long chunk = (long long)(ws_bytes / per);
  if (chunk < 1) return fail_arg("toeplitz workspace too small: %zu < %lld", ws_bytes, per);
  return dispatch_q<Apply5Fn>(M, x, out, aux, alpha, beta, nslices, n,
                              reinterpret_cast<const c32*>(PQ), Bi, flip,
                              reinterpret_cast<c32*>(ws), chunk, st);
}

int psf_build5(int n, int M, const double* cs, int n_angles, int nd, void* PQ, float* Bi,
               void* ws, cudaStream_t st) {
  return dispatch_q<Psf5Fn>(M, n, cs, n_angles, nd, reinterpret_cast<c32*>(PQ), Bi,
                            reinterpret_cast<char*>(ws), st);
}

int init_twiddles_toeplitz5() {
  TF_TRY(check_cuda(init_twiddles_tu(), "twiddle init (toeplitz5)"));
  return check_cuda(init_twiddles5_tu(), "radix-5 twiddle init");
}

}  // namespace tf
