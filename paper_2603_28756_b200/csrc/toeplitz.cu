// Toeplitz normal operator K x = R*R x on B200.
//
// Reference: tomoforge/toeplitz.py:134-149 (_apply_batch) pads each N x N
// slice into an odd 7-smooth M x M grid, runs a complex fft2, multiplies by
// main (+ conj(F) * flip), and crops the real part of ifft2.  Here the lag
// kernels are re-embedded circularly on an even power-of-two grid M >= 2N-1
// with the image at offset 0 (exact: all lags |d| <= N-1 stay distinct mod M),
// and the flip term becomes B = spec(K_flip) * ph(kx) ph(ky),
// ph_k = e^{-2 pi i k (N-1)/M} (derivation in DESIGN.md §3).  Both lag kernels
// are real and even, so the transform is real-to-complex on the half spectrum.
//
// Half-spectrum layout in HBM ("row-blocked"): T[z][rb][ky][r], rb = ix / 4,
// r = ix % 4, ky in [0, M/2] -- the 4 rows of a block are 32 contiguous bytes
// per frequency, and one block's whole half spectrum is contiguous.
//
//   K1 k_rows_fwd  : each thread runs two complex FFTs (rows 4rb..4rb+3 packed
//                    pairwise as x_a + i x_b, zero padded to M), splits them
//                    into four half spectra and writes its block contiguously.
//   K2 k_cols_conv : per column ky, a TMA 4-D tensor copy gathers the 32-byte
//                    pieces of all row blocks into shared memory; length-M FFT
//                    over ix, Y = F*A + conj(F)*B with the PSF column held in
//                    registers across all slices, inverse FFT, keep ix < N,
//                    TMA tensor store back in place.
//   K3 k_rows_inv  : reads a block contiguously, two inverse complex FFTs
//                    (Hermitian packing), crop n < N, out = alpha*y + beta*aux.
//
// PSF (K6, toeplitz.py:85-131 compute_psf/build_psf): the NUFFT-of-ones kernel
// is replaced by its exact closed form, K(d) = sum_theta D(d . e_theta) with
// the Dirichlet sum D(u) = sum_j cos(2 pi j u / Nd) over the signed detector
// frequencies (geometry.py:196-201), K_nyq(d) = 1/2 sum_theta cos(pi d.e_theta)
// for even Nd (toeplitz.py:106-114); evaluated in fp64, transformed with the
// same K1 + a forward column pass, and folded with 1/M^2 into
//   PQ = ((A + Re B)/M^2, (A - Re B)/M^2),  Bi = Im B / M^2
// so that Y = (Fr P + Fi Bi, Fi Q + Fr Bi): two paired-fp32 instructions.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "tf_async.cuh"
#include "tf_common.cuh"

namespace tf {

constexpr int RB = 4;  // rows per block of the half-spectrum layout
__host__ __device__ constexpr int nrb_of(int rows) { return (rows + RB - 1) / RB; }

// ============================================================ K1: rows, forward
// x: [nslices][rows][x_row_stride] fp32, row r nonzero for n < n_in (zero beyond)
// T: [nslices][nrb][M/2+1][4] c32.  Thread t of group g transforms the block
// rb = blockIdx.x*G + g as two complex FFTs z_b = x_{4rb+2b} + i x_{4rb+2b+1}
// and splits them:  X_a(k) = (Z(k) + conj Z(M-k))/2,  X_b(k) = -i (Z(k) - conj Z(M-k))/2.
// Thread t owns k = t + T m (m < E/2); Z(M-k) sits in the upper half of partner
// thread T-t and is exchanged through shared memory.  Stores are 32 B per k,
// contiguous across the warp.  ZP: n_in <= M/2 (upper half of inputs is zero).
template <int M, int E, int G, bool ZP, int NB>
__global__ void __launch_bounds__(G*(M / E), (M >= 8192 ? 1 : 2))
k_rows_fwd(const float* __restrict__ x, c32* __restrict__ T, int rows, int n_in,
           long long x_slice_stride, long long x_row_stride) {
  constexpr int TT = M / E;
  constexpr int SB = group_stride(M, NB * G);
  constexpr int H = M / 2 + 1;
  constexpr int EL = ZP ? E / 2 : E;  // loaded elements
  extern __shared__ __align__(16) c32 smem[];
  const int g = threadIdx.x / TT;
  const int t = threadIdx.x - g * TT;
  const int z = blockIdx.y;
  const int nrb = nrb_of(rows);
  // NB == 2: a group owns a 4-row block; NB == 1: half a block (row pair b0)
  const int unit = blockIdx.x * G + g;
  const int rb = NB == 2 ? unit : unit >> 1;
  const int b0 = NB == 2 ? 0 : (unit & 1);
  const int r0 = rb * RB + 2 * b0;
  c32* sm = smem + g * NB * SB;

  const float* xr = x + z * x_slice_stride + (long long)r0 * x_row_stride;
  c32 v[NB][E];
#pragma unroll
  for (int m = 0; m < EL; ++m) {
    const int j = t + TT * m;
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      float a = 0.f, c = 0.f;
      if (j < n_in) {
        if (r0 + 2 * b < rows) a = __ldg(xr + (2 * b) * x_row_stride + j);
        if (r0 + 2 * b + 1 < rows) c = __ldg(xr + (2 * b + 1) * x_row_stride + j);
      }
      v[b][m] = mk(a, c);
    }
  }
  fftn<M, E, false, ZP, false, NB>(v, sm, SB, t);
  // upper half Z(M/2 + w) -> sm[b][w]; the buffers are free (last pass is register-only)
#pragma unroll
  for (int m = E / 2; m < E; ++m)
#pragma unroll
    for (int b = 0; b < NB; ++b) sm[b * SB + t + TT * m - M / 2] = v[b][m];
  __syncthreads();
  if (rb >= nrb) return;

  float4* dst = reinterpret_cast<float4*>(T + ((long long)z * nrb + rb) * H * RB);
  auto emit = [&](int k, int m, bool self) {
    float4 o[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const c32 zk = v[b][m];
      const c32 zm = self ? zk : sm[b * SB + M / 2 - k];
      const c32 xa = scale(mk(zk.x + zm.x, zk.y - zm.y), 0.5f);
      const c32 xb = scale(mk(zk.y + zm.y, zm.x - zk.x), 0.5f);
      o[b] = make_float4(xa.x, xa.y, xb.x, xb.y);
    }
    if constexpr (NB == 2) st_global_v8(dst + 2 * k, o[0], o[NB - 1]);  // 32 B: all 4 rows
    else dst[2 * k + b0] = o[0];
  };
#pragma unroll
  for (int m = 0; m < E / 2; ++m) {
    const int k = t + TT * m;
    emit(k, m, k == 0);
  }
  if (t == 0) emit(M / 2, E / 2, true);
}

#ifndef TF_K1_MIRROR
#define TF_K1_MIRROR 1
#endif
#ifndef TF_K3_MIRROR
#define TF_K3_MIRROR 1
#endif
// K1 (mirror path): the split outputs are staged in the freed exchange buffer and
// written by one bulk async copy per row block instead of per-thread stores
#ifndef TF_K1_BULKST
#define TF_K1_BULKST 1
#endif
// K3: output rows staged in the freed exchange buffer, one bulk async copy per row
#ifndef TF_K3_BULKST
#define TF_K3_BULKST 1
#endif
// Persistent K1 with a bulk-copied input stage.  Each CTA walks units u =
// blockIdx.x + i * gridDim.x (unit = (slice, 4-row block)); the four input rows
// of the next unit are fetched by the copy engine (cp.async.bulk, one 1-D copy
// per row) into the single shared stage as soon as the current unit has read
// it, so the load latency overlaps this unit's FFT.  Needs 16-byte aligned rows
// of n_in * 4 bytes.  Same transform and output as k_rows_fwd (NB = 2).
// TF_K1_MIRROR (default): the last pass runs in a mirror-pair mapping (thread
// t = 2s + b owns columns s and T - s of row pair b), so Z(k) and Z(M - k) meet
// in registers and the Hermitian split needs no shared-memory round trip; lane
// pairs b = 0, 1 write the two 16-byte halves of each 32-byte output word.
// TF_K1_BULKST (default): those words go to the (by then free) exchange buffer
// in the block's HBM layout, and one bulk async copy writes the 64 KB block --
// the LSU issues 16 shared stores per thread instead of 16 global ones, and the
// copy overlaps the next unit (K1 0.68 -> 0.62 ms).
template <int M, int E, bool ZP>
__global__ void __launch_bounds__(M / E, (M >= 8192 ? 1 : 2))
k_rows_fwd_pf(const float* __restrict__ x, c32* __restrict__ T, int rows, int n_in,
              long long x_slice_stride, long long x_row_stride, long long nunits) {
  constexpr int TT = M / E;
  constexpr int NB = 2;
  constexpr int SB = group_stride(M, NB);
  constexpr int H = M / 2 + 1;
  constexpr int EL = ZP ? E / 2 : E;
  extern __shared__ __align__(128) c32 smem[];
  c32* sm = smem;                                                   // exchange: NB * SB
  float* stage = reinterpret_cast<float*>(smem + NB * SB);          // [RB][n_in]
  uint64_t* full = reinterpret_cast<uint64_t*>(stage + RB * n_in);  // 8-byte aligned
  const int t = threadIdx.x;
  using S = FftShape<M, E>;
  constexpr bool MIR = TF_K1_MIRROR && TT % 32 == 0 && S::NP >= 2;
  const int mb = t & 1, s = t >> 1;  // transform (row pair) and mirror slot
  const bool s0 = s == 0;
  const int c1 = s, c2 = s0 ? TT / 2 : TT - s;
  PassTw<M, E, S::NP - 1> tw1, tw2;  // last-pass twiddles of the thread's two columns
  if constexpr (MIR) {
    tw1.from_table(c1);
    tw2.from_table(c2);
  }
  const int nrb = nrb_of(rows);
  const uint32_t row_bytes = (uint32_t)n_in * sizeof(float);
  // (slice, row block) walks of the consumer and of the producer (one unit ahead),
  // advanced by gridDim.x units without divisions
  const int gz = (int)(gridDim.x / nrb), grb = (int)(gridDim.x - gz * nrb);
  auto advance = [&](int& z, int& rb) {
    z += gz;
    rb += grb;
    if (rb >= nrb) {
      rb -= nrb;
      ++z;
    }
  };
  int pz = (int)(blockIdx.x / nrb), prb = (int)(blockIdx.x - (blockIdx.x / nrb) * nrb);
  auto issue = [&]() {
    const int r0 = prb * RB;
    const int nr = min(RB, rows - r0);
    mbar_expect_tx(full, nr * row_bytes);
    for (int q = 0; q < nr; ++q)
      bulk_g2s(stage + q * n_in, x + pz * x_slice_stride + (long long)(r0 + q) * x_row_stride,
               row_bytes, full);
    advance(pz, prb);
  };
  if (t == 0) {
    mbar_init(full, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (t == 0 && (long long)blockIdx.x < nunits) issue();
  int it = 0;
  int z = (int)(blockIdx.x / nrb), rb = (int)(blockIdx.x - (blockIdx.x / nrb) * nrb);
  for (long long u = blockIdx.x; u < nunits; u += gridDim.x, ++it, advance(z, rb)) {
    const int r0 = rb * RB;
    mbar_wait(full, (uint32_t)(it & 1));
    c32 v[NB][E];
#pragma unroll
    for (int m = 0; m < EL; ++m) {
      const int j = t + TT * m;
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        float a = 0.f, c = 0.f;
        if (j < n_in) {
          if (r0 + 2 * b < rows) a = stage[(2 * b) * n_in + j];
          if (r0 + 2 * b + 1 < rows) c = stage[(2 * b + 1) * n_in + j];
        }
        v[b][m] = mk(a, c);
      }
    }
    if constexpr (MIR && TF_K1_BULKST) {
      if (t == 0) bulk_wait_read<0>();  // the previous unit's output copy has left sm
    }
    __syncthreads();  // the stage is free: refill it with the next unit
    if (t == 0 && u + gridDim.x < nunits) {
      fence_proxy_async_smem();
      issue();
    }
    if constexpr (MIR) {
      fftn_to_last<M, E, 0, ZP, NB>(v, sm, SB, t);
      // last pass in the mirror-pair mapping: thread t = 2s + b takes columns c1 = s,
      // c2 = T - s (s = 0: 0 and T/2) of transform b, so Z(k) and Z(M - k) are both in
      // its registers and the split needs no shared-memory round trip
      {
        c32 w[2][1][E];
#pragma unroll
        for (int m = 0; m < E; ++m) {
          w[0][0][m] = sm[mb * SB + canon_word<M, E>(c1, m)];
          w[1][0][m] = sm[mb * SB + canon_word<M, E>(c2, m)];
        }
        fft_pass<M, E, S::NP - 1, false, false, false, 1>(w[0], &tw1);
        fft_pass<M, E, S::NP - 1, false, false, false, 1>(w[1], &tw2);
        float4* blk = reinterpret_cast<float4*>(T + ((long long)z * nrb + rb) * H * RB);
        float4* dst = blk + mb;
        if constexpr (TF_K1_BULKST) {
          __syncthreads();  // every thread's last-pass loads are done: sm is free
          dst = reinterpret_cast<float4*>(sm) + mb;
        }
        auto split = [](c32 zk, c32 zm) {
          return make_float4(0.5f * (zk.x + zm.x), 0.5f * (zk.y - zm.y), 0.5f * (zk.y + zm.y),
                             0.5f * (zm.x - zk.x));
        };
#pragma unroll
        for (int m = 0; m < E / 2; ++m) {
          const c32 m1 = s0 ? w[0][0][(E - m) % E] : w[1][0][E - 1 - m];
          const c32 m2 = s0 ? w[1][0][E - 1 - m] : w[0][0][E - 1 - m];
          dst[2 * (c1 + TT * m)] = split(w[0][0][m], m1);
          dst[2 * (c2 + TT * m)] = split(w[1][0][m], m2);
        }
        if (s0) dst[2 * (M / 2)] = split(w[0][0][E / 2], w[0][0][E / 2]);
        if constexpr (TF_K1_BULKST) {
          static_assert(!TF_K1_BULKST || H * RB <= NB * SB, "output block fits the exchange");
          fence_proxy_async_smem();
          __syncthreads();
          if (t == 0) {
            bulk_s2g(blk, sm, (uint32_t)(H * RB * sizeof(c32)));
            bulk_commit();
          }
        }
      }
    } else {
      fftn<M, E, false, ZP, false, NB>(v, sm, SB, t);
#pragma unroll
      for (int m = E / 2; m < E; ++m)
#pragma unroll
        for (int b = 0; b < NB; ++b) sm[b * SB + t + TT * m - M / 2] = v[b][m];
      __syncthreads();
      float4* dst = reinterpret_cast<float4*>(T + ((long long)z * nrb + rb) * H * RB);
      auto emit = [&](int k, int m, bool self) {
        float4 o[NB];
#pragma unroll
        for (int b = 0; b < NB; ++b) {
          const c32 zk = v[b][m];
          const c32 zm = self ? zk : sm[b * SB + M / 2 - k];
          const c32 xa = scale(mk(zk.x + zm.x, zk.y - zm.y), 0.5f);
          const c32 xb = scale(mk(zk.y + zm.y, zm.x - zk.x), 0.5f);
          o[b] = make_float4(xa.x, xa.y, xb.x, xb.y);
        }
        st_global_v8(dst + 2 * k, o[0], o[1]);
      };
#pragma unroll
      for (int m = 0; m < E / 2; ++m) {
        const int k = t + TT * m;
        emit(k, m, k == 0);
      }
      if (t == 0) emit(M / 2, E / 2, true);
    }
    // the next unit's pass-0 exchange store must not overtake the mirror reads:
    // its first shared write follows the stage barrier above, which every
    // thread reaches only after finishing this unit
  }
  if constexpr (MIR && TF_K1_BULKST) {
    if (t == 0) bulk_wait<0>();  // the last output copy is complete before the CTA exits
  }
}

// ============================================================ K3: rows, inverse
// T: [nslices][nrb][M/2+1][4]; out: [nslices][rows][o_row_stride]
// out[n] = alpha * y[n] + beta * aux[n] for n < n_out (n_out <= M/2).
// Thread t of group g inverts block rb's two row pairs with complex FFTs of
// Z = Y_a + i Y_b (Hermitian extension Z(j) = conj Y_a(M-j) + i conj Y_b(M-j)
// for j > M/2).  TF_K3_MIRROR (default): thread t = 2s + b loads the 16-byte
// (Ya, Yb) words of columns s and T - s of row pair b -- each other's Hermitian
// mirrors -- and runs the first pass on both before the first exchange.  Otherwise
// it loads the 32 contiguous bytes of its own k = t + T m (m < E/2) and the
// mirrored half comes from partner thread T-t via shared memory.
// AUXBULK: the four aux rows are prefetched into shared memory by 1-D bulk
// copies issued at kernel start (needs 16-byte aligned rows of n_out*4 bytes).
template <int M, int E, int G, bool AUXBULK, int NB>
__global__ void __launch_bounds__(G*(M / E), (M >= 8192 ? 1 : 2))
k_rows_inv(const c32* __restrict__ T, float* __restrict__ out, const float* __restrict__ aux,
           int rows, int n_out, long long o_slice_stride, long long o_row_stride, float alpha,
           float beta, int pf_dist, int obulk) {
  constexpr int TT = M / E;
  constexpr int H = M / 2 + 1;
  constexpr int SB = group_stride(M, NB * G);
  constexpr int NR = 2 * NB;  // rows per group
  static_assert(2 * H <= SB, "pair buffer must fit the exchange buffer");
  extern __shared__ __align__(16) c32 smem[];
  const int g = threadIdx.x / TT;
  const int t = threadIdx.x - g * TT;
  const int z = blockIdx.y;
  const int nrb = nrb_of(rows);
  // NB == 2: a group owns a 4-row block; NB == 1: half a block (row pair b0)
  const int unit = blockIdx.x * G + g;
  const int rb_raw = NB == 2 ? unit : unit >> 1;
  const int b0 = NB == 2 ? 0 : (unit & 1);
  const int rb = min(rb_raw, nrb - 1);  // surplus groups redo the last block
  const bool writer = rb_raw < nrb;
  const int r0 = rb * RB + 2 * b0;
  const float4* src = reinterpret_cast<const float4*>(T + ((long long)z * nrb + rb) * H * RB);
  c32* sm = smem + g * NB * SB;  // transform b: (Ya, Yb)(k) at words b*SB + 2k, +1
  // AUXBULK region after the exchange buffers: [G][NR][M/2] fp32 + one mbarrier
  float* auxs = reinterpret_cast<float*>(smem + G * NB * SB) + g * NR * (M / 2);
  uint64_t* abar = reinterpret_cast<uint64_t*>(reinterpret_cast<float*>(smem + G * NB * SB) +
                                               G * NR * (M / 2));
  const long long zo = z * o_slice_stride;
  if constexpr (AUXBULK) {
    if (threadIdx.x == 0) {
      mbar_init(abar, G);  // one arrival (with or without tx) per group
      fence_mbar_init();
    }
    // with one group the initialising thread is the only one to arrive, and the
    // other threads wait on the barrier only after the FFT's own CTA barriers
    if constexpr (G > 1) __syncthreads();
    if (t == 0 && writer) {
      const int nr = min(NR, rows - r0);
      const uint32_t bytes = (uint32_t)n_out * sizeof(float);
      mbar_expect_tx(abar, nr * bytes);  // one arrival per group
      for (int q = 0; q < nr; ++q)
        bulk_g2s(auxs + q * (M / 2), aux + zo + (long long)(r0 + q) * o_row_stride, bytes, abar);
    } else if (t == 0) {
      mbar_arrive(abar);
    }
  }

  // L2 prefetch for the CTA pf_dist blocks ahead (about one resident wave later):
  // its spectrum block (and aux rows) are in L2 when it starts
  // issued after the CTA barrier by a warp other than the barrier initialiser, so
  // no warp waits on it
  if (pf_dist > 0 && threadIdx.x == (blockDim.x > 32 ? 32 : 0)) {
    const long long lin = (long long)blockIdx.y * gridDim.x + blockIdx.x + pf_dist;
    if (lin < (long long)gridDim.x * gridDim.y) {
      const int zz = (int)(lin / gridDim.x), ux = (int)(lin - (long long)zz * gridDim.x);
      const int nrb_ = nrb_of(rows);
#pragma unroll
      for (int gg = 0; gg < G; ++gg) {
        const int u = ux * G + gg;
        const int rbr = NB == 2 ? u : u >> 1;
        if (rbr >= nrb_ || (NB == 1 && (u & 1))) continue;
        bulk_prefetch_l2(T + ((long long)zz * nrb_ + rbr) * H * RB, (uint32_t)(H * RB * sizeof(c32)));
        if (AUXBULK)
          for (int q = 0; q < RB && rbr * RB + q < rows; ++q)
            bulk_prefetch_l2(aux + zz * o_slice_stride + (long long)(rbr * RB + q) * o_row_stride,
                             (uint32_t)n_out * sizeof(float));
      }
    }
  }
  auto fix = [&](int k, float4& y) {
    if (k == 0 || k == M / 2) { y.y = 0.f; y.w = 0.f; }  // irfft drops Im(DC, Nyquist)
  };
  using S = FftShape<M, E>;
  constexpr bool MIR = TF_K3_MIRROR && NB == 2 && TT % 32 == 0 && S::NP >= 2;
  c32 v[NB][E];
  if constexpr (MIR) {
    // first pass in the mirror-pair mapping (as in k_rows_fwd_pf): thread t = 2s + b
    // loads the 16-byte (Ya, Yb) words of columns c1 = s and c2 = T - s (s = 0: 0 and
    // T/2) of row pair b, which hold each other's Hermitian mirrors, runs pass 0 on
    // both and stores them to the first exchange -- no mirror round trip
    const int mb = t & 1, s = t >> 1;
    const bool s0 = s == 0;
    const int c1 = s, c2 = s0 ? TT / 2 : TT - s;
    const float4* sb = src + mb;
    float4 y1[E / 2], y2[E / 2], yn;
#pragma unroll
    for (int m = 0; m < E / 2; ++m) {
      y1[m] = __ldg(sb + 2 * (c1 + TT * m));
      y2[m] = __ldg(sb + 2 * (c2 + TT * m));
    }
    if (s0) {
      yn = __ldg(sb + 2 * (M / 2));
      fix(0, y1[0]);
      fix(M / 2, yn);
    }
    PassTw<M, E, 1> tw;
    tw.from_table(t);
    c32 w[2][1][E];
#pragma unroll
    for (int m = 0; m < E / 2; ++m) {
      w[0][0][m] = mk(y1[m].x - y1[m].w, y1[m].y + y1[m].z);  // Ya + i Yb
      w[1][0][m] = mk(y2[m].x - y2[m].w, y2[m].y + y2[m].z);
    }
#pragma unroll
    for (int m = E / 2; m < E; ++m) {  // conj(Ya) + i conj(Yb) at M - j
      const float4 a = s0 ? (m == E / 2 ? yn : y1[E - m]) : y2[E - 1 - m];
      const float4 c = s0 ? y2[E - 1 - m] : y1[E - 1 - m];
      w[0][0][m] = mk(a.x + a.w, a.z - a.y);
      w[1][0][m] = mk(c.x + c.w, c.z - c.y);
    }
    fft_pass<M, E, 0, true, false, false, 1>(w[0], (const PassTw<M, E, 0>*)nullptr);
    fft_pass<M, E, 0, true, false, false, 1>(w[1], (const PassTw<M, E, 0>*)nullptr);
    fft_store<M, E, 0, 1>(w[0], sm + mb * SB, SB, c1);
    fft_store<M, E, 0, 1>(w[1], sm + mb * SB, SB, c2);
    __syncthreads();
    load_canonical<M, E, NB>(v, sm, SB, t);
    __syncthreads();
    fft_passes_from<M, E, 1, true, false, true, NB, false>(v, sm, SB, t, TwTable(), &tw);
  } else {
    float4 lo[E / 2][NB];
#pragma unroll
    for (int m = 0; m < E / 2; ++m) {
      if constexpr (NB == 2) ld_global_nc_v8(src + 2 * (t + TT * m), lo[m][0], lo[m][NB - 1]);
      else lo[m][0] = __ldg(src + 2 * (t + TT * m) + b0);
    }
    float4 nyq[NB];
    if (t == 0)
#pragma unroll
      for (int b = 0; b < NB; ++b) nyq[b] = __ldg(src + 2 * (M / 2) + b + b0);
#pragma unroll
    for (int m = 0; m < E / 2; ++m)
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        fix(t + TT * m, lo[m][b]);
        *reinterpret_cast<float4*>(sm + b * SB + 2 * (t + TT * m)) = lo[m][b];
      }
    if (t == 0)
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        fix(M / 2, nyq[b]);
        *reinterpret_cast<float4*>(sm + b * SB + 2 * (M / 2)) = nyq[b];
      }
    __syncthreads();
#pragma unroll
    for (int m = 0; m < E; ++m)
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        if (m < E / 2) {
          const float4 y = lo[m][b];
          v[b][m] = mk(y.x - y.w, y.y + y.z);  // Ya + i Yb
        } else {
          const int j = t + TT * m;
          const float4 y = *reinterpret_cast<const float4*>(sm + b * SB + 2 * (M - j));
          v[b][m] = mk(y.x + y.w, y.z - y.y);  // conj(Ya) + i conj(Yb)
        }
      }
    __syncthreads();
    fftn<M, E, true, false, true, NB>(v, sm, SB, t);
  }
  if constexpr (AUXBULK) mbar_wait(abar, 0);
  if (!writer) return;
  if constexpr (TF_K3_BULKST && G == 1 && NB == 2) {
    if (obulk) {  // 16-byte aligned output rows: stage them, one bulk copy per row
      static_assert(NR * (M / 2) * sizeof(float) <= NB * SB * sizeof(c32), "rows fit");
      float* so = reinterpret_cast<float*>(sm);
      __syncthreads();  // every thread's last exchange reads are done: sm is free
#pragma unroll
      for (int q = 0; q < NR; ++q) {
        const float* a = aux ? aux + zo + (long long)(r0 + q) * o_row_stride : nullptr;
#pragma unroll
        for (int m = 0; m < E / 2; ++m) {
          const int n = t + TT * m;
          if (n < n_out) {
            float y = alpha * ((q & 1) ? v[q >> 1][m].y : v[q >> 1][m].x);
            if constexpr (AUXBULK) y = fmaf(beta, auxs[q * (M / 2) + n], y);
            else if (a && r0 + q < rows) y = fmaf(beta, __ldg(a + n), y);
            so[q * (M / 2) + n] = y;
          }
        }
      }
      fence_proxy_async_smem();
      __syncthreads();
      if (t == 0) {
        for (int q = 0; q < NR && r0 + q < rows; ++q)
          bulk_s2g(out + zo + (long long)(r0 + q) * o_row_stride, so + q * (M / 2),
                   (uint32_t)n_out * sizeof(float));
        bulk_commit();
        bulk_wait_read<0>();  // the staged rows have left shared memory
      }
      return;
    }
  }

#pragma unroll
  for (int q = 0; q < NR; ++q) {
    const int r = r0 + q;
    if (r >= rows) break;
    float* o = out + zo + (long long)r * o_row_stride;
    const float* a = aux ? aux + zo + (long long)r * o_row_stride : nullptr;
#pragma unroll
    for (int m = 0; m < E / 2; ++m) {
      const int n = t + TT * m;
      if (n < n_out) {
        float y = alpha * ((q & 1) ? v[q >> 1][m].y : v[q >> 1][m].x);
        if constexpr (AUXBULK) y = fmaf(beta, auxs[q * (M / 2) + n], y);
        else if (a) y = fmaf(beta, __ldg(a + n), y);
        o[n] = y;
      }
    }
  }
}

// element ix of column c of slice z in the row-blocked layout
__device__ __forceinline__ long long tidx(int z, int ix, int c, int nrb, int H) {
  return (((long long)z * nrb + (ix >> 2)) * H + c) * RB + (ix & 3);
}

// ============================================================ K2: column convolution
// Column c of slice z: elements ix < col_len (zero beyond, col_len <= M/2) of
// T; PSF columns PQ[c][kx], Bi[c][kx], kx in [0, M).  Generic variant for small
// M: one column per thread group, slices in sequence, direct gathers.
template <int M, int E, int G, bool FLIP>
__global__ void __launch_bounds__(G*(M / E))
k_cols_conv(c32* __restrict__ T, const c32* __restrict__ PQ, const float* __restrict__ Bi,
            int ncols, int col_len, int nslices) {
  constexpr int TT = M / E;
  constexpr int SB = group_stride(M, G);
  extern __shared__ __align__(16) c32 smem[];
  const int g = threadIdx.x / TT;
  const int t = threadIdx.x - g * TT;
  const int nrb = nrb_of(col_len);
  c32* sm = smem + g * SB;
  const int nsteps = (ncols + G * gridDim.x - 1) / (G * gridDim.x);
  for (int step = 0; step < nsteps; ++step) {
    const int c = (step * gridDim.x + blockIdx.x) * G + g;
    const bool active = c < ncols;
    c32 pq[E];
    float bi[FLIP ? E : 1];
#pragma unroll
    for (int m = 0; m < E; ++m) {
      const int kx = t + TT * m;
      pq[m] = active ? __ldg(PQ + (long long)c * M + kx) : mk(0.f, 0.f);
      if constexpr (FLIP) bi[m] = active ? __ldg(Bi + (long long)c * M + kx) : 0.f;
    }
    for (int z = 0; z < nslices; ++z) {
      c32 v[E];
#pragma unroll
      for (int m = 0; m < E / 2; ++m) {
        const int j = t + TT * m;
        v[m] = (active && j < col_len) ? T[tidx(z, j, c, nrb, M / 2 + 1)] : mk(0.f, 0.f);
      }
      fft<M, E, false, true, false>(v, sm, t);
#pragma unroll
      for (int m = 0; m < E; ++m) {
        if constexpr (FLIP) {
          // (Fr P + Fi Bi, Fi Q + Fr Bi)
          v[m] = pfma(mk(v[m].y, v[m].x), mk(bi[m], bi[m]), pmul(v[m], pq[m]));
        } else {
          v[m] = pmul(v[m], pq[m]);
        }
      }
      // no barrier: the forward transform's last shared-memory read is fenced by
      // the barrier inside fft(), and its last pass is register-only
      fft<M, E, true, false, true>(v, sm, t);
#pragma unroll
      for (int m = 0; m < E / 2; ++m) {
        const int j = t + TT * m;
        if (active && j < col_len) T[tidx(z, j, c, nrb, M / 2 + 1)] = v[m];
      }
    }
  }
}

// twiddles of the column kernel: one table entry per pass + squarings (a 2 KB
// pass-1 table and a 30 KB last-pass table measured slower)
using K2Tw = TwTable;

// K2 for 1024 <= M <= 4096: a persistent, TMA-fed column kernel.  Each CTA walks
// its (column, slice) items, column-major, keeping the column's PSF in registers
// across all slices.  Thread 0 keeps the next S items in flight: TMA 4-D tensor
// copies (box = 32 B x BOXR row blocks) gather the column's pieces from every
// row block into a contiguous shared stage, completing on the stage's `full`
// mbarrier; a stage is refilled only after every thread has arrived on its
// `empty` mbarrier (release/acquire ordering of the generic reads before the
// async-proxy write; a bare __syncthreads is not enough since BAR.SYNC lets the
// issuing warp run ahead).
// * the FFT exchanges alternate between two shared buffers, so each exchange
//   costs one CTA barrier instead of two;
// * results go straight to global memory: 8-byte stores, 4 consecutive lanes
//   complete one 32-byte row-block piece, addresses from a per-thread base plus
//   a constant stride (no per-element index arithmetic);
// * the (column, slice) walk is kept in counters -- no divisions in the loop.
// Shared memory: S input stages + 2 exchange buffers (102 KB at M = 4096, two
// CTAs per SM).
template <int M, int E, int S, bool FLIP>
__global__ void __launch_bounds__(M / E, 2)
k_cols_conv_pp(const __grid_constant__ CUtensorMap tmap, const c32* __restrict__ PQ,
               const float* __restrict__ Bi, int ncols, int nrb, int nslices, int boxr,
               c32* __restrict__ T) {
  constexpr int TT = M / E;
  constexpr int SB = group_stride(M, 1);
  constexpr int CL = M / 2;
  constexpr int H = M / 2 + 1;
  static_assert(FftShape<M, E>::NP % 2 == 1, "ping-pong needs an even exchange count");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  c32* inb = reinterpret_cast<c32*>(smem_raw);   // [S][CL]
  c32* xbuf = inb + S * CL;                       // [2][SB]
  uint64_t* full = reinterpret_cast<uint64_t*>(xbuf + 2 * SB);
  uint64_t* empty = full + S;
  const int t = threadIdx.x;
  if ((int)blockIdx.x >= ncols) return;
  const int my_cols = (ncols - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
  const long long nitems = (long long)my_cols * nslices;
  const int nbox = (nrb + boxr - 1) / boxr;
  const uint32_t box_bytes = (uint32_t)boxr * RB * sizeof(c32);
  const int col_len = nrb * RB;
  // producer walk (thread 0): item -> (column, slice), S items ahead of the consumer
  int p_col = blockIdx.x, p_sl = 0;
  auto issue = [&](int s) {
    mbar_expect_tx(&full[s], nbox * box_bytes);
    for (int q = 0; q < nbox; ++q)
      tma_load_4d(inb + s * CL + q * boxr * RB, &tmap, 0, p_col, q * boxr, p_sl, &full[s]);
    if (++p_sl == nslices) {
      p_sl = 0;
      p_col += gridDim.x;
    }
  };
  if (t == 0) {
    tma_prefetch_desc(&tmap);
#pragma unroll
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], TT);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (t == 0)
    for (int s = 0; s < S && s < nitems; ++s) issue(s);

  const K2Tw twt;
  c32 pq[E];
  float bi[FLIP ? E : 1];
  // consumer walk: per-thread store base of element j = t (+ 256 m) of (col, sl)
  int c_col = blockIdx.x, c_sl = 0;
  const long long m_stride = (long long)(TT / RB) * H * RB;  // j += TT -> 64 row blocks on
  const long long slice_stride = (long long)nrb * H * RB;
  const long long t_off = (long long)(t >> 2) * H * RB + (t & 3);
  for (long long i = 0; i < nitems; ++i) {
    const int s = (int)(i % S);
    const uint32_t parity = (uint32_t)((i / S) & 1);
    if (c_sl == 0) {
#pragma unroll
      for (int m = 0; m < E; ++m) {
        pq[m] = __ldg(PQ + (long long)c_col * M + t + TT * m);
        if constexpr (FLIP) bi[m] = __ldg(Bi + (long long)c_col * M + t + TT * m);
      }
    }
    mbar_wait(&full[s], parity);
    c32 v[1][E];
    const c32* in = inb + s * CL;
#pragma unroll
    for (int m = 0; m < E / 2; ++m) {
      const int j = t + TT * m;
      v[0][m] = j < col_len ? in[j] : mk(0.f, 0.f);
    }
    mbar_arrive(&empty[s]);
    fftn<M, E, false, true, false, 1, K2Tw, true>(v, xbuf, SB, t, twt);
    if (t == 0 && i + S < nitems) {
      mbar_wait(&empty[s], parity);
      issue(s);
    }
#pragma unroll
    for (int m = 0; m < E; ++m) {
      if constexpr (FLIP) {
        v[0][m] = pfma(mk(v[0][m].y, v[0][m].x), mk(bi[m], bi[m]), pmul(v[0][m], pq[m]));
      } else {
        v[0][m] = pmul(v[0][m], pq[m]);
      }
    }
    fftn<M, E, true, false, true, 1, K2Tw, true>(v, xbuf, SB, t, twt);
    c32* dst = T + c_sl * slice_stride + (long long)c_col * RB + t_off;
#pragma unroll
    for (int m = 0; m < E / 2; ++m) {
      if (t + TT * m < col_len) dst[m * m_stride] = v[0][m];
    }
    if (++c_sl == nslices) {
      c_sl = 0;
      c_col += gridDim.x;
    }
  }
}

// K2 for M = 2048 / 4096 on two radix-64-sized passes: E = 64 elements per thread,
// TT = M/64 threads per column transform (one or two warps), G = 4 independent
// groups per CTA, one CTA per SM.  Against k_cols_conv_pp (E = 16, three passes)
// this halves the shared-memory exchanges per (column, slice) item -- one
// exchange per transform instead of two, 2 x 32 KB stored and loaded instead of
// 4 x 32 KB -- which, with the FP32 pipe, bound the column pass (an exchange-only
// variant of k_cols_conv_pp ran 1.23 ms of its 1.99 ms; profiles/r02).
// * The CTA walks columns c = blockIdx.x + k gridDim.x; its four groups split the
//   column's slices (group g: z = g, g+4, ...).  64 complex elements per thread
//   leave no registers for the PSF, so the column's PSF (12 B per frequency) is
//   bulk-copied into shared memory once per column (CTA barrier at each column
//   change; the copy is waited for only at the PSF product).  Reading it through
//   L1 instead doubled the kernel time (the 48 KB column does not stay in L1 next
//   to ~180 KB of shared memory).
// * Each group runs its own pipeline over named barriers of its TT threads.  The
//   next item's 4-D TMA gather lands in the group's exchange buffer as soon as the
//   second exchange has been read (`empty` mbarrier), i.e. during the last pass
//   and the stores, so no separate input stage is needed.
// * The pass-1 twiddles depend only on the thread (k = t): computed once.
// * Exchange padding: word w at w + w/TT (pass-0 radix == TT, so a thread's
//   pass-0 outputs and the canonical reads both hit distinct bank pairs).
template <int M, bool FLIP>
__global__ void __launch_bounds__(4 * (M / 64), 1)
k_cols_conv64(const __grid_constant__ CUtensorMap tmap, const c32* __restrict__ PQ,
              const float* __restrict__ Bi, int ncols, int nrb, int nslices, int boxr,
              c32* __restrict__ T) {
  constexpr int E = 64, TT = M / E, G = 4;
  constexpr int H = M / 2 + 1;
  constexpr int XW = M + M / TT;  // padded exchange words per group
  using S = FftShape<M, E>;
  static_assert(S::NP == 2 && (1 << S::LFIRST) == TT, "two passes, pass-0 radix == TT");
  constexpr int R0 = TT, ST0 = E / R0;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int g = threadIdx.x / TT, t = threadIdx.x - g * TT;
  c32* pq_s = reinterpret_cast<c32*>(smem_raw);                  // [M]
  float* bi_s = reinterpret_cast<float*>(pq_s + M);                // [M]
  c32* xb = reinterpret_cast<c32*>(bi_s + M) + g * XW;             // [G][XW]
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<c32*>(bi_s + M) + G * XW);
  uint64_t* full = bars + 2 * g;
  uint64_t* empty = full + 1;
  uint64_t* psf_full = bars + 2 * G;
  const int bar_id = 1 + g;
  if (threadIdx.x == 0) mbar_init(psf_full, 1);
  if (t == 0) {
    mbar_init(full, 1);
    mbar_init(empty, TT);
  }
  if (threadIdx.x == 0) fence_mbar_init();
  __syncthreads();
  if ((int)blockIdx.x >= ncols) return;
  const bool active = g < nslices;
  const int my_cols = (ncols - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
  const int nz_g = active ? (nslices - g + G - 1) / G : 0;
  const int nitems = my_cols * nz_g;
  const int nbox = (nrb + boxr - 1) / boxr;
  const uint32_t box_bytes = (uint32_t)boxr * RB * sizeof(c32);
  const int col_len = nrb * RB;
  int p_col = blockIdx.x, p_z = g, issued = 0;
  auto issue = [&]() {
    mbar_expect_tx(full, nbox * box_bytes);
    for (int q = 0; q < nbox; ++q)
      tma_load_4d(xb + q * boxr * RB, &tmap, 0, p_col, q * boxr, p_z, full);
    ++issued;
    p_z += G;
    if (p_z >= nslices) {
      p_z = g;
      p_col += gridDim.x;
    }
  };
  if (t == 0 && nitems > 0) {
    tma_prefetch_desc(&tmap);
    issue();
  }
  PassTw<M, E, 1> tw;
  tw.from_table(t);
  const long long m_stride = (long long)(TT / RB) * H * RB;
  const long long slice_stride = (long long)nrb * H * RB;
  const long long t_off = (long long)(t >> 2) * H * RB + (t & 3);
  auto exchange = [&](c32 (&v)[1][E]) {
#pragma unroll
    for (int i = 0; i < ST0; ++i)
#pragma unroll
      for (int r = 0; r < R0; ++r) xb[(t + i * TT) * (R0 + 1) + r] = v[0][i + r * ST0];
    named_bar_sync(bar_id, TT);
#pragma unroll
    for (int m = 0; m < E; ++m) v[0][m] = xb[t + (TT + 1) * m];
  };
  int item = 0;
  for (int k = 0; k < my_cols; ++k) {
    const int c = blockIdx.x + k * gridDim.x;
    __syncthreads();  // every group is done with the previous column's PSF
    if (threadIdx.x == 0) {
      mbar_expect_tx(psf_full, M * (uint32_t)(sizeof(c32) + (FLIP ? sizeof(float) : 0)));
      bulk_g2s(pq_s, PQ + (long long)c * M, M * sizeof(c32), psf_full);
      if constexpr (FLIP) bulk_g2s(bi_s, Bi + (long long)c * M, M * sizeof(float), psf_full);
      if (k + 1 < my_cols) {
        bulk_prefetch_l2(PQ + (long long)(c + gridDim.x) * M, M * sizeof(c32));
        if constexpr (FLIP) bulk_prefetch_l2(Bi + (long long)(c + gridDim.x) * M, M * sizeof(float));
      }
    }
    bool psf_ready = false;
    for (int z = g; active && z < nslices; z += G, ++item) {
      mbar_wait(full, (uint32_t)(item & 1));
      c32 v[1][E];
#pragma unroll
      for (int m = 0; m < E / 2; ++m) {
        const int j = t + TT * m;
        v[0][m] = j < col_len ? xb[j] : mk(0.f, 0.f);
      }
      fft_pass<M, E, 0, false, true, false, 1>(v, (const PassTw<M, E, 0>*)nullptr);
      named_bar_sync(bar_id, TT);  // the input (in xb) has been read by the whole group
      exchange(v);
      fft_pass<M, E, 1, false, false, false, 1>(v, &tw);
      if (!psf_ready) {
        mbar_wait(psf_full, (uint32_t)(k & 1));
        psf_ready = true;
      }
#pragma unroll
      for (int m = 0; m < E; ++m) {
        const c32 pq = pq_s[t + TT * m];
        if constexpr (FLIP) {
          const float bi = bi_s[t + TT * m];
          v[0][m] = pfma(mk(v[0][m].y, v[0][m].x), mk(bi, bi), pmul(v[0][m], pq));
        } else {
          v[0][m] = pmul(v[0][m], pq);
        }
      }
      fft_pass<M, E, 0, true, false, false, 1>(v, (const PassTw<M, E, 0>*)nullptr);
      named_bar_sync(bar_id, TT);  // the first exchange has been read
      exchange(v);
      mbar_arrive(empty);
      if (t == 0 && issued < nitems) {
        mbar_wait(empty, (uint32_t)(item & 1));
        issue();
      }
      fft_pass<M, E, 1, true, false, true, 1>(v, &tw);
      c32* dst = T + z * slice_stride + (long long)c * RB + t_off;
#pragma unroll
      for (int m = 0; m < E / 2; ++m) {
        if (t + TT * m < col_len) dst[m * m_stride] = v[0][m];
      }
    }
  }
}

// forward-only column FFT (PSF spectra): S[z][c][kx] = FFT_ix(column c of T)
template <int M, int E, int G>
__global__ void __launch_bounds__(G*(M / E))
k_cols_fwd(const c32* __restrict__ T, c32* __restrict__ Sout, int ncols, int col_len,
           long long s_slice_stride) {
  constexpr int TT = M / E;
  extern __shared__ __align__(16) c32 smem[];
  const int g = threadIdx.x / TT;
  const int t = threadIdx.x - g * TT;
  const int z = blockIdx.y;
  const int c = blockIdx.x * G + g;
  const bool active = c < ncols;
  const int nrb = nrb_of(col_len);
  c32 v[E];
#pragma unroll
  for (int m = 0; m < E; ++m) {
    const int j = t + TT * m;
    v[m] = (active && j < col_len) ? T[tidx(z, j, c, nrb, M / 2 + 1)] : mk(0.f, 0.f);
  }
  fft<M, E, false>(v, smem + g * group_stride(M, G), t);
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
  if (!(d0 > -n && d1 > -n && (i0 < n || i0 > M - n) && (i1 < n || i1 > M - n))) {
    kmain[id] = 0.f;  // outside the lag support |d| <= n - 1
    kflip[id] = 0.f;
    return;
  }
  // K(-d) = K(d) (D and cos are even, u(-d) = -u(d) exactly): the thread of the
  // representative d0 > 0 or (d0 = 0, d1 >= 0) writes both lags -- half the fp64 work
  if (!(d0 > 0 || (d0 == 0 && d1 >= 0))) return;
  const int jlo = -(nd / 2), jhi = (nd + 1) / 2 - 1;
  const bool even = (nd % 2) == 0;
  double k = 0.0, kn = 0.0;
  for (int a = 0; a < n_angles; ++a) {
    const double u = d0 * cs[2 * a] + d1 * cs[2 * a + 1];
    k += dirichlet(u, nd, jlo, jhi);
    if (even) kn += cospi(u);
  }
  kn *= 0.5;
  const float km = (float)((k - kn) / nd), kf = (float)(-kn / nd);
  const long long mirror = (long long)(d0 == 0 ? 0 : M - d0) * M + (d1 <= 0 ? -d1 : M - d1);
  kmain[id] = km;
  kflip[id] = kf;
  kmain[mirror] = km;
  kflip[mirror] = kf;
}

// The reference's lag kernel K(d) = Re type1(1 at every polar sample) on its odd
// grid of side m (toeplitz.py:102-103, fp64 closed form), stored ifftshifted:
// out[i0][i1] = K(d0, d1) with d = i for i <= (m-1)/2, else i - m.  Its fft2 is
// the reference's PsfKernel.spectrum.
__global__ void k_psf_kernel_grid(double* __restrict__ out, int m, const double* __restrict__ cs,
                                  int n_angles, int nd) {
  const long long id = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (id >= (long long)m * m) return;
  const int i0 = (int)(id / m), i1 = (int)(id - (long long)i0 * m);
  const int h = (m - 1) / 2;
  const int d0 = i0 <= h ? i0 : i0 - m;
  const int d1 = i1 <= h ? i1 : i1 - m;
  const int jlo = -(nd / 2), jhi = (nd + 1) / 2 - 1;
  double k = 0.0;
  for (int a = 0; a < n_angles; ++a) k += dirichlet(d0 * cs[2 * a] + d1 * cs[2 * a + 1], nd, jlo, jhi);
  out[id] = k;
}

int psf_kernel_grid(int m, const double* cs, int n_angles, int nd, double* out, cudaStream_t st) {
  const int bs = 256;
  const long long nb = ((long long)m * m + bs - 1) / bs;
  k_psf_kernel_grid<<<(unsigned)nb, bs, 0, st>>>(out, m, cs, n_angles, nd);
  return check_launch("k_psf_kernel_grid");
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

// 4-D tensor map over the row-blocked half spectrum: dims (fp32 units)
// {8 = 4 rows x re/im, M/2+1 columns, nrb row blocks, nslices}; box {8, 1, boxr, 1}
int encode_tmap(CUtensorMap* map, c32* T, int M, int nrb, long long nslices, int boxr) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    TF_TRY(check_cuda(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q),
                      "cudaGetDriverEntryPoint(cuTensorMapEncodeTiled)"));
    if (!fn || q != cudaDriverEntryPointSuccess) {
      set_error("cuTensorMapEncodeTiled unavailable");
      return TF_ECUDA;
    }
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  const cuuint64_t H = M / 2 + 1;
  const cuuint64_t dims[4] = {8, H, (cuuint64_t)nrb, (cuuint64_t)nslices};
  const cuuint64_t strides[3] = {32, H * 32, H * 32 * (cuuint64_t)nrb};
  const cuuint32_t box[4] = {8, 1, (cuuint32_t)boxr, 1};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  const CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, T, dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
    return TF_ECUDA;
  }
  return TF_OK;
}

// ============================================================ host dispatch
namespace {

constexpr int E_DEFAULT = 16;

template <int M>
constexpr int eper() { return M < E_DEFAULT ? M : E_DEFAULT; }

template <int M, int NB = 2>
constexpr int rows_g() {  // thread groups per CTA in K1/K3 (each group: NB row pairs)
  constexpr int T = M / eper<M>();
  constexpr int g = (NB == 2 ? 256 : 512) / T;
  return g < 1 ? 1 : (g > 16 ? 16 : g);
}
template <int M>
constexpr int cols_g() {  // columns per CTA in the generic K2
  constexpr int T = M / eper<M>();
  constexpr int g = 128 / T;
  return g < 1 ? 1 : g;
}

template <int M, int NB>
int launch_rows_fwd_t(const float* x, c32* T, int rows, int n_in, long long xs, long long xr,
                      long long nslices, cudaStream_t st) {
  constexpr int E = eper<M>(), G = rows_g<M, NB>();
  constexpr int TT = M / E;
  const size_t smem = sizeof(c32) * NB * G * group_stride(M, NB * G);
  const int units = nrb_of(rows) * (2 / NB);
  const int gx = (units + G - 1) / G;
  KernelTimer tm;
  timer_begin(tm, 0, st);
  for (long long z0 = 0; z0 < nslices; z0 += 65535) {
    const int nz = (int)std::min<long long>(65535, nslices - z0);
    c32* Tz = T + z0 * (long long)(M / 2 + 1) * RB * nrb_of(rows);
    auto kern = (2 * n_in <= M) ? k_rows_fwd<M, E, G, true, NB> : k_rows_fwd<M, E, G, false, NB>;
    TF_TRY(prep_kernel(kern, smem));
    kern<<<dim3(gx, nz), G * TT, smem, st>>>(x + z0 * xs, Tz, rows, n_in, xs, xr);
  }
  timer_end(tm);
  return check_launch("k_rows_fwd");
}

template <int M>
int launch_rows_fwd_pf(const float* x, c32* T, int rows, int n_in, long long xs, long long xr,
                       long long nslices, cudaStream_t st) {
  constexpr int E = eper<M>();
  constexpr int TT = M / E;
  const size_t smem = sizeof(c32) * 2 * group_stride(M, 2) + sizeof(float) * RB * n_in + 16;
  auto kern = (2 * n_in <= M) ? k_rows_fwd_pf<M, E, true> : k_rows_fwd_pf<M, E, false>;
  TF_TRY(prep_kernel(kern, smem));
  int per_sm = 0;
  TF_TRY(check_cuda(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, TT, smem),
                    "occupancy"));
  const long long nunits = (long long)nrb_of(rows) * nslices;
  const int grid = (int)std::max<long long>(1, std::min<long long>(nunits,
                                                                  (long long)std::max(1, per_sm) * num_sms()));
  KernelTimer tm;
  timer_begin(tm, 0, st);
  kern<<<grid, TT, smem, st>>>(x, T, rows, n_in, xs, xr, nunits);
  timer_end(tm);
  return check_launch("k_rows_fwd_pf");
}


template <int M>
int launch_rows_fwd(const float* x, c32* T, int rows, int n_in, long long xs, long long xr,
                    long long nslices, cudaStream_t st) {
  const size_t pf_smem = sizeof(c32) * 2 * group_stride(M, 2) + sizeof(float) * RB * n_in + 16;
  // persistent bulk-prefetched variant when rows are 16-byte aligned blocks
  if (M >= 1024 && n_in % 4 == 0 && xr % 4 == 0 && xs % 4 == 0 &&
      reinterpret_cast<uintptr_t>(x) % 16 == 0 && pf_smem <= 200 * 1024)
    return launch_rows_fwd_pf<M>(x, T, rows, n_in, xs, xr, nslices, st);
  return launch_rows_fwd_t<M, 2>(x, T, rows, n_in, xs, xr, nslices, st);
}

// How many blocks ahead a K3 CTA prefetches the spectrum block and aux rows into
// L2: one per SM, about half a resident wave ahead.  Measured on 64 x 2048^2:
// 0.92 -> 0.78 ms (110-200 equal, 592 thrashes).
#ifndef TF_K3_PF_X2
#define TF_K3_PF_X2 2  // K3 L2 prefetch distance in half SM counts
#endif
inline int k3_l2pf() { return num_sms() * TF_K3_PF_X2 / 2; }

template <int M, int NB>
int launch_rows_inv_t(const c32* T, float* out, const float* aux, int rows, int n_out,
                      long long os, long long orow, float alpha, float beta, long long nslices,
                      cudaStream_t st) {
  constexpr int E = eper<M>(), G = rows_g<M, NB>();
  constexpr int TT = M / E;
  if (2 * n_out > M) return fail_arg("k_rows_inv: n_out %d exceeds M/2", n_out);
  // bulk-prefetch aux rows when they are 16-byte aligned blocks
  const bool bulk = aux && (n_out % 4 == 0) && (orow % 4 == 0) && (os % 4 == 0) &&
                    (reinterpret_cast<uintptr_t>(aux) % 16 == 0);
  const int obulk = (n_out % 4 == 0) && (orow % 4 == 0) && (os % 4 == 0) &&
                    (reinterpret_cast<uintptr_t>(out) % 16 == 0);
  const size_t smem = sizeof(c32) * NB * G * group_stride(M, NB * G) +
                      (bulk ? sizeof(float) * G * 2 * NB * (M / 2) + 16 : 0);
  auto kern = bulk ? k_rows_inv<M, E, G, true, NB> : k_rows_inv<M, E, G, false, NB>;
  TF_TRY(prep_kernel(kern, smem));
  const int units = nrb_of(rows) * (2 / NB);
  const int gx = (units + G - 1) / G;
  KernelTimer tm;
  timer_begin(tm, 2, st);
  for (long long z0 = 0; z0 < nslices; z0 += 65535) {
    const int nz = (int)std::min<long long>(65535, nslices - z0);
    kern<<<dim3(gx, nz), G * TT, smem, st>>>(T + z0 * (long long)(M / 2 + 1) * RB * nrb_of(rows),
                                             out + z0 * os, aux ? aux + z0 * os : nullptr, rows,
                                             n_out, os, orow, alpha, beta, k3_l2pf(), obulk);
  }
  timer_end(tm);
  return check_launch("k_rows_inv");
}

template <int M>
int launch_rows_inv(const c32* T, float* out, const float* aux, int rows, int n_out,
                    long long os, long long orow, float alpha, float beta, long long nslices,
                    cudaStream_t st) {
  return launch_rows_inv_t<M, 2>(T, out, aux, rows, n_out, os, orow, alpha, beta, nslices, st);
}

constexpr int CONV_STAGES = 2;

template <int M, bool FLIP, int NS = CONV_STAGES>
int launch_cols_conv_pp_t(c32* T, const c32* PQ, const float* Bi, int col_len,
                          long long nslices, cudaStream_t st) {
  constexpr int E = eper<M>();
  constexpr int TT = M / E;
  const int ncols = M / 2 + 1;
  const int nrb = nrb_of(col_len);
  const int boxr = std::min(nrb, 256);
  CUtensorMap map;
  TF_TRY(encode_tmap(&map, T, M, nrb, nslices, boxr));
  const size_t smem = sizeof(c32) * ((size_t)NS * (M / 2) + 2 * group_stride(M, 1)) +
                      2 * NS * sizeof(uint64_t);
  auto kern = k_cols_conv_pp<M, E, NS, FLIP>;
  TF_TRY(prep_kernel(kern, smem));
  int blocks_per_sm = 0;
  TF_TRY(check_cuda(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, kern, TT, smem),
                    "occupancy"));
  const int grid = std::max(1, std::min(ncols, std::max(1, blocks_per_sm) * num_sms()));
  KernelTimer tm;
  timer_begin(tm, 1, st);
  kern<<<grid, TT, smem, st>>>(map, PQ, Bi, ncols, nrb, (int)nslices, boxr, T);
  timer_end(tm);
  return check_launch("k_cols_conv_pp");
}

template <int M, bool FLIP>
int launch_cols_conv64_t(c32* T, const c32* PQ, const float* Bi, int col_len, long long nslices,
                         cudaStream_t st) {
  constexpr int TT = M / 64, G = 4;
  const int ncols = M / 2 + 1;
  const int nrb = nrb_of(col_len);
  const int boxr = std::min(nrb, 256);
  CUtensorMap map;
  TF_TRY(encode_tmap(&map, T, M, nrb, nslices, boxr));
  const size_t smem = (sizeof(c32) + sizeof(float)) * M + sizeof(c32) * G * (size_t)(M + M / TT) +
                      (2 * G + 1) * sizeof(uint64_t);
  auto kern = k_cols_conv64<M, FLIP>;
  TF_TRY(prep_kernel(kern, smem));
  const int grid = std::max(1, std::min(ncols, num_sms()));
  KernelTimer tm;
  timer_begin(tm, 1, st);
  kern<<<grid, G * TT, smem, st>>>(map, PQ, Bi, ncols, nrb, (int)nslices, boxr, T);
  timer_end(tm);
  return check_launch("k_cols_conv64");
}

template <int M, bool FLIP>
int launch_cols_conv_t(c32* T, const c32* PQ, const float* Bi, int col_len, long long nslices,
                       cudaStream_t st) {
  constexpr int E = eper<M>(), G = cols_g<M>();
  constexpr int TT = M / E;
  const int ncols = M / 2 + 1;
  const size_t smem = sizeof(c32) * G * group_stride(M, G);
  auto kern = k_cols_conv<M, E, G, FLIP>;
  TF_TRY(prep_kernel(kern, smem));
  int blocks_per_sm = 0;
  TF_TRY(check_cuda(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, kern, G * TT, smem),
                    "occupancy"));
  const int grid = std::max(1, std::min((ncols + G - 1) / G, blocks_per_sm * num_sms()));
  KernelTimer tm;
  timer_begin(tm, 1, st);
  kern<<<grid, G * TT, smem, st>>>(T, PQ, Bi, ncols, col_len, (int)nslices);
  timer_end(tm);
  return check_launch("k_cols_conv");
}

template <int M>
int launch_cols_conv(c32* T, const c32* PQ, const float* Bi, int col_len, long long nslices,
                     bool flip, cudaStream_t st) {
  if (2 * col_len > M) return fail_arg("k_cols_conv: column length %d exceeds M/2", col_len);
#ifndef TF_K2_E64
#define TF_K2_E64 1
#endif
  if constexpr (TF_K2_E64 && (M == 2048 || M == 4096)) {
    return flip ? launch_cols_conv64_t<M, true>(T, PQ, Bi, col_len, nslices, st)
                : launch_cols_conv64_t<M, false>(T, PQ, Bi, col_len, nslices, st);
  }
  if constexpr (M >= 1024 && M <= 4096) {
    return flip ? launch_cols_conv_pp_t<M, true>(T, PQ, Bi, col_len, nslices, st)
                : launch_cols_conv_pp_t<M, false>(T, PQ, Bi, col_len, nslices, st);
  }
  return flip ? launch_cols_conv_t<M, true>(T, PQ, Bi, col_len, nslices, st)
              : launch_cols_conv_t<M, false>(T, PQ, Bi, col_len, nslices, st);
}

template <int M>
int launch_cols_fwd(const c32* T, c32* Sout, int col_len, long long nslices, cudaStream_t st) {
  constexpr int E = eper<M>(), G = cols_g<M>();
  constexpr int TT = M / E;
  const int ncols = M / 2 + 1;
  const size_t smem = sizeof(c32) * G * group_stride(M, G);
  auto kern = k_cols_fwd<M, E, G>;
  TF_TRY(prep_kernel(kern, smem));
  kern<<<dim3((ncols + G - 1) / G, (unsigned)nslices), G * TT, smem, st>>>(
      T, Sout, ncols, col_len, (long long)ncols * M);
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
    // ws: lags [2][M][M] f32 | T [2][M/4][M/2+1][4] c32 | spec [2][M/2+1][M] c32
    const long long MM = (long long)M * M;
    const long long H = M / 2 + 1;
    float* lags = reinterpret_cast<float*>(ws);
    c32* T = reinterpret_cast<c32*>(ws + 2 * MM * sizeof(float));
    c32* spec = T + 2 * H * M;
    const bool flip = (nd % 2) == 0;
    TF_TRY(psf_lags_launch(lags, n, M, cs, n_angles, nd, st));
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

// Half spectrum of real images for the forward NUFFT (type2): K1 over the N rows
// (zero padded to M), then the forward column FFT of the M/2+1 half-spectrum
// columns: S[z][ky][kx], ky in [0, M/2], kx in [0, M).
template <int M>
struct SpectrumFn {
  static int run(const float* img, long long nslices, int n, c32* T, c32* S, cudaStream_t st) {
    const long long img_sz = (long long)n * n;
    TF_TRY(launch_rows_fwd<M>(img, T, n, n, img_sz, n, nslices, st));
    return launch_cols_fwd<M>(T, S, n, nslices, st);
  }
};

}  // namespace

int psf_lags_launch(float* lags, int n, int M, const double* cs, int n_angles, int nd,
                    cudaStream_t st) {
  const long long MM = (long long)M * M;
  const int bs = 256;
  k_psf_lags<<<(unsigned)((MM + bs - 1) / bs), bs, 0, st>>>(lags, lags + MM, n, M, cs, n_angles,
                                                             nd);
  return check_launch("k_psf_lags");
}

size_t spectrum_workspace_bytes(int n, int M) {
  return (size_t)(M / 2 + 1) * RB * nrb_of(n) * sizeof(c32);  // row pass output per slice
}

int real_spectrum(const float* img, long long nslices, int n, int M, void* T, void* S,
                  cudaStream_t st) {
  if (2 * n > M) return fail_arg("spectrum side %d < 2N = %d", M, 2 * n);
  return dispatch_m<SpectrumFn>(M, img, nslices, n, reinterpret_cast<c32*>(T),
                                reinterpret_cast<c32*>(S), st);
}

int toeplitz_apply(const float* x, float* out, const float* aux, float alpha, float beta,
                   long long nslices, int n, int M, const void* PQ, const float* Bi, bool flip,
                   void* ws, size_t ws_bytes, cudaStream_t st) {
  if (is_side5(M))
    return toeplitz_apply5(x, out, aux, alpha, beta, nslices, n, M, PQ, Bi, flip, ws, ws_bytes, st);
  const long long per = (long long)(M / 2 + 1) * RB * nrb_of(n) * (long long)sizeof(c32);
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
  if (is_side5(M)) return psf_build5(n, M, cs, n_angles, nd, PQ, Bi, ws, st);
  return dispatch_m<PsfFn>(M, n, cs, n_angles, nd, reinterpret_cast<c32*>(PQ), Bi,
                           reinterpret_cast<char*>(ws), st);
}

int init_twiddles_toeplitz() { return check_cuda(init_twiddles_tu(), "twiddle init (toeplitz)"); }

}  // namespace tf
