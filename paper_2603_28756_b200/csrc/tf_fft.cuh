// Register/shared-memory Stockham FFT engine for power-of-two lengths.
//
// A length-M transform is run by a *group* of T = M/E threads; thread t keeps
// the E elements {t + T*m : m < E} in registers ("canonical layout").  Each
// pass applies radix-R butterflies (R | E, R <= 64) to register-resident data;
// between passes the group exchanges through a padded shared-memory buffer
// (word i lives at i + i/16, which keeps every exchange at the 2-wavefront
// minimum for 8-byte elements).  The first radix may be smaller than E, all
// later ones equal E; then the first pass's input set and the last pass's
// output set of thread t are both its canonical set, which lets the Toeplitz
// column kernel multiply by the PSF and start the inverse transform without a
// shared-memory round trip (toeplitz.cu, k_cols_conv).
//
// Zero-padding is exploited explicitly: ZIN = the upper half of the canonical
// inputs (m >= E/2, i.e. indices >= M/2) is zero, HOUT = only the lower half of
// the outputs is needed; the first/last butterflies are pruned accordingly.
//
// Forward = e^{-2 pi i jk/M} (numpy.fft sign); INV = conjugate, unnormalised.
// Twiddles: fp32 per-length tables e^{-2 pi i j/L} built in fp64 once per device
// (tf_init).  A pass's butterfly needs only its base twiddle w (one table word)
// and the squares w^2, w^4, w^8 (dft_fold below).
//
// Butterflies (dft_fold): a radix-R pass computes X[q] = sum_r u_r w^r W_R^{rq}
// as log2 R levels of radix-2 DIT steps, Z[q] = E + t O, Z[q + n/2] = 2E - Z[q],
// with the external twiddle folded into each step's t = w^{R/n} W_n^q.  On the
// paired-fp32 datapath that is 3 instructions per butterfly (two FFMA2 for
// E + t O, one FFMA2 for 2E - Z) instead of a complex multiply per input plus
// two FADD2 -- about 20 % fewer FP instructions per twiddled radix-16 pass.
#pragma once
#include "tf_complex.cuh"

namespace tf {

constexpr int TW_MAX = 16384;  // largest supported transform length
// Concatenated per-length tables: W_L^j = e^{-2 pi i j/L} at word (L - 2) + j for
// L = 2, 4, ..., TW_MAX, so the twiddles of one pass are contiguous in k.
constexpr int TW_WORDS = 2 * TW_MAX - 2;
// one copy per translation unit (internal linkage, no relocatable device code);
// every TU that runs FFTs fills its copy from ensure_init() via init_twiddles_tu()
static __device__ c32 g_twiddle[TW_WORDS];

__host__ __device__ constexpr int ilog2(int v) { return v <= 1 ? 0 : 1 + ilog2(v >> 1); }
__host__ __device__ constexpr int pad_idx(int i) { return i + (i >> 4); }
// exchange-buffer stride (c32 words) for `groups` concurrent buffers: spaced by
// 16/groups bank pairs so that cross-buffer accesses of 16/groups consecutive
// words by one warp never collide
__host__ __device__ constexpr int group_stride(int M, int groups) {
  return pad_idx(M) + 16 + ((((groups >= 16 ? 0 : 16 / groups) - pad_idx(M)) % 16) + 16) % 16;
}

// e^{-2 pi i k / L}
template <int L>
__device__ __forceinline__ c32 tw_w(int k) {
  return g_twiddle[(L - 2) + k];
}

constexpr float kH = 0.70710678118654752440f;  // 1/sqrt 2

// ---------------------------------------------------- FMA-folded codelet
// cos(2 pi q / 64); W_n^q = (cos64(64q/n), -cos64(64q/n - 16)) for n | 64.  q is a
// constant after unrolling, so the lookup folds to an immediate.  (The 16ths are
// the same fp32 values the radix-16 codelets always used.)
__device__ __forceinline__ float cos64(int q) {
  const float c[64] = {
      1.f, 0.9951847195625305f, 0.9807852506637573f, 0.9569403529167175f,
      0.9238795042037964f, 0.8819212913513184f, 0.8314695954322815f, 0.7730104327201843f,
      0.7071067690849304f, 0.6343932747840881f, 0.5555702447891235f, 0.4713967442512512f,
      0.3826834261417389f, 0.290284663438797f, 0.19509032368659973f, 0.0980171412229538f,
      0.f, -0.0980171412229538f, -0.19509032368659973f, -0.290284663438797f,
      -0.3826834261417389f, -0.4713967442512512f, -0.5555702447891235f, -0.6343932747840881f,
      -0.7071067690849304f, -0.7730104327201843f, -0.8314695954322815f, -0.8819212913513184f,
      -0.9238795042037964f, -0.9569403529167175f, -0.9807852506637573f, -0.9951847195625305f,
      -1.f, -0.9951847195625305f, -0.9807852506637573f, -0.9569403529167175f,
      -0.9238795042037964f, -0.8819212913513184f, -0.8314695954322815f, -0.7730104327201843f,
      -0.7071067690849304f, -0.6343932747840881f, -0.5555702447891235f, -0.4713967442512512f,
      -0.3826834261417389f, -0.290284663438797f, -0.19509032368659973f, -0.0980171412229538f,
      0.f, 0.0980171412229538f, 0.19509032368659973f, 0.290284663438797f,
      0.3826834261417389f, 0.4713967442512512f, 0.5555702447891235f, 0.6343932747840881f,
      0.7071067690849304f, 0.7730104327201843f, 0.8314695954322815f, 0.8819212913513184f,
      0.9238795042037964f, 0.9569403529167175f, 0.9807852506637573f, 0.9951847195625305f,
  };
  return c[q & 63];
}

// e + o t (forward) or e + o conj(t) (INV): two FFMA2
template <bool INV>
__device__ __forceinline__ c32 cfma(c32 e, c32 o, c32 t) {
  const c32 p = pfma(o, mk(t.x, t.x), e);
  return INV ? pfma(mk(o.y, o.x), mk(t.y, -t.y), p) : pfma(mk(o.y, o.x), mk(-t.y, t.y), p);
}
// 2e - z: one FFMA2 (the partner output of a folded radix-2 step)
__device__ __forceinline__ c32 twice_minus(c32 e, c32 z) {
  return pfma(e, mk(2.f, 2.f), mk(-z.x, -z.y));
}

// In-place X[q] = sum_r u_r w^r W_R^{rq} (TW; else w = 1), conjugated for INV,
// output X[q] in u[q].  pw[j] = w^{2^j}.  Radix-2 DIT over r: with Z_{r0,s} the
// (R/s)-point twiddled DFT of u_{r0 + s j},
//   Z_{r0,s}[q] = Z_{r0,2s}[q] + t Z_{r0+s,2s}[q],  Z_{r0,s}[q + n/2] = 2 Z_{r0,2s}[q] - Z_{r0,s}[q],
// t = w^s W_n^q, n = R/s; Z_{r0,s}[q] lives at position r0 + s q.  Steps whose t
// is 1 or -i (no TW) are two FADD2; all others three FFMA2.  ZIN: u[R/2..] == 0
// (not read); HOUT: only X[0..R/2-1] are produced.
// one radix-2 level (n = 2^LV) of dft_fold: a -> b
template <int R, int LV, bool INV, bool ZIN, bool HOUT, bool TW>
__device__ __forceinline__ void fold_level(const c32 (&a)[R], c32 (&b)[R], const c32* pw) {
  constexpr int LR = ilog2(R);
  constexpr int n = 1 << LV, s = R >> LV, h = n >> 1, nq = n >= 4 ? n / 4 : 1;
  constexpr bool last = LV == LR;
  c32 ws = mk(1.f, 0.f);
  c32 tq[nq];  // w^s W_n^{q'}, 0 < q' < n/4
  if constexpr (TW) {
    ws = pw[LR - LV];
#pragma unroll
    for (int qp = 1; qp < nq; ++qp)
      tq[qp] = cmul(ws, mk(cos64(qp * 64 / n), -cos64(qp * 64 / n - 16)));
  }
#pragma unroll
  for (int r0 = 0; r0 < s; ++r0) {
#pragma unroll
    for (int q = 0; q < h; ++q) {
      const int pos0 = r0 + s * q, pos1 = pos0 + R / 2;
      const c32 e = a[r0 + 2 * s * q];
      if constexpr (ZIN && LV == 1) {
        b[pos0] = e;
        b[pos1] = e;
      } else {
        const c32 o = a[r0 + s + 2 * s * q];
        const int qp = q % nq;
        const bool quarter = n >= 4 && q >= nq;
        if (!TW && qp == 0) {
          const c32 to = quarter ? rot_q<INV>(o) : o;
          b[pos0] = cadd(e, to);
          if constexpr (!(HOUT && last)) b[pos1] = csub(e, to);
        } else {
          c32 t = qp == 0 ? ws
                  : TW    ? tq[qp]
                          : mk(cos64(qp * 64 / n), -cos64(qp * 64 / n - 16));
          if (quarter) t = mk(t.y, -t.x);  // -i t
          const c32 z = cfma<INV>(e, o, t);
          b[pos0] = z;
          if constexpr (!(HOUT && last)) b[pos1] = twice_minus(e, z);
        }
      }
    }
  }
}

template <int R, int LV, bool INV, bool ZIN, bool HOUT, bool TW>
__device__ __forceinline__ void fold_levels(c32 (&a)[R], const c32* pw) {
  if constexpr (LV <= ilog2(R)) {
    c32 b[R];
    fold_level<R, LV, INV, ZIN, HOUT, TW>(a, b, pw);
    fold_levels<R, LV + 1, INV, ZIN, HOUT, TW>(b, pw);
#pragma unroll
    for (int r = 0; r < R; ++r) a[r] = b[r];
  }
}

template <int R, bool INV, bool ZIN, bool HOUT, bool TW>
__device__ __forceinline__ void dft_fold(c32 (&u)[R], const c32* pw) {
  fold_levels<R, 1, INV, ZIN, HOUT, TW>(u, pw);
}

// --------------------------------------------------------------- engine

template <int M, int E>
struct FftShape {
  static_assert((M & (M - 1)) == 0 && M >= 2 && M <= TW_MAX, "power-of-two length");
  static_assert(E <= M && (E & (E - 1)) == 0, "E");
  static constexpr int T = M / E;  // threads per transform
  static constexpr int L = ilog2(M);
  static constexpr int LE = ilog2(E);
  static constexpr int NP = (L + LE - 1) / LE;  // passes
  static constexpr int LFIRST = L - (NP - 1) * LE;
  __host__ __device__ static constexpr int lradix(int p) { return p == 0 ? LFIRST : LE; }
  __host__ __device__ static constexpr int ns(int p) {
    return p == 0 ? 1 : (1 << (LFIRST + (p - 1) * LE));
  }
};

// exchange-buffer word of canonical element m of thread t
template <int M, int E>
__device__ __forceinline__ int canon_word(int t, int m) {
  constexpr int T = M / E;
  if constexpr (T % 16 == 0) return pad_idx(t) + m * (T + T / 16);
  else return pad_idx(t + T * m);
}

// Forward twiddle powers of pass P for thread t: p[i][j] = w_i^{2^j},
// w_i = e^{-2 pi i k_i/(NS R)}, k_i = (t + i T) mod NS.
template <int M, int E, int P>
struct PassTw {
  using S = FftShape<M, E>;
  static constexpr int LR = S::lradix(P);
  static constexpr int R = 1 << LR;
  static constexpr int NS = S::ns(P);
  static constexpr int ST = E / R;
  c32 p[ST][LR > 0 ? LR : 1];
  // base twiddle from the table, its powers by squaring (FP work)
  __device__ __forceinline__ void from_table(int t) {
#pragma unroll
    for (int i = 0; i < ST; ++i) {
      const int k = (t + i * S::T) & (NS - 1);
      p[i][0] = tw_w<NS * R>(k);
#pragma unroll
      for (int j = 1; j < LR; ++j) p[i][j] = cmul(p[i][j - 1], p[i][j - 1]);
    }
  }
};

// default twiddle source: table + squaring
struct TwTable {
  template <int M, int E, int P>
  __device__ __forceinline__ void operator()(PassTw<M, E, P>& tw, int t) const {
    tw.from_table(t);
  }
};

template <int M, int E, int P, bool INV, bool ZIN, bool HOUT, int NB>
__device__ __forceinline__ void fft_pass(c32 (&v)[NB][E], const PassTw<M, E, P>* tw) {
  using S = FftShape<M, E>;
  constexpr int R = 1 << S::lradix(P);
  constexpr int ST = E / R;  // butterflies per thread
#pragma unroll
  for (int i = 0; i < ST; ++i) {
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      c32 u[R];
#pragma unroll
      for (int r = 0; r < (ZIN ? R / 2 : R); ++r) u[r] = v[b][i + r * ST];
      if constexpr (P > 0 && R > 1) dft_fold<R, INV, ZIN, HOUT, true>(u, tw->p[i]);
      else dft_fold<R, INV, ZIN, HOUT, false>(u, nullptr);
#pragma unroll
      for (int r = 0; r < (HOUT ? R / 2 : R); ++r) v[b][i + r * ST] = u[r];
    }
  }
}

// write pass-P outputs to the exchange buffer in Stockham order:
// element (i, r) of butterfly b = t + i T goes to word (b/NS) NS R + b%NS + r NS
template <int M, int E, int P, int NB>
__device__ __forceinline__ void fft_store(const c32 (&v)[NB][E], c32* sm, int sbs, int t) {
  using S = FftShape<M, E>;
  constexpr int R = 1 << S::lradix(P);
  constexpr int NS = S::ns(P);
  constexpr int ST = E / R;
#pragma unroll
  for (int i = 0; i < ST; ++i) {
    const int bf = t + i * S::T;
    const int base = pad_idx((bf / NS) * NS * R + (bf & (NS - 1)));
    // base % 16 < NS or NS % 16 == 0, so the padding of base + r NS splits exactly
#pragma unroll
    for (int b = 0; b < NB; ++b)
#pragma unroll
      for (int r = 0; r < R; ++r) sm[b * sbs + base + r * NS + ((r * NS) >> 4)] = v[b][i + r * ST];
  }
}


template <int M, int E, int NB>
__device__ __forceinline__ void load_canonical(c32 (&v)[NB][E], const c32* sm, int sbs, int t) {
#pragma unroll
  for (int m = 0; m < E; ++m)
#pragma unroll
    for (int b = 0; b < NB; ++b) v[b][m] = sm[b * sbs + canon_word<M, E>(t, m)];
}

// Pass P with its twiddles already in `tw` (null for P = 0).  The twiddles of
// pass P+1 are fetched *before* the exchange that precedes it, so their loads
// (and squarings) overlap the shared-memory round trip and the barrier
// instead of stalling the next pass (TF_TW_EARLY = 0 restores in-place fetches).
#ifndef TF_TW_EARLY
#define TF_TW_EARLY 1
#endif
template <int M, int E, int P, bool INV, bool ZIN, bool HOUT, int NB, bool PP, typename TwF>
__device__ __forceinline__ void fft_passes_from(c32 (&v)[NB][E], c32* sm, int sbs, int t,
                                                const TwF& twf,
                                                const PassTw<M, E, P>* tw = nullptr) {
  using S = FftShape<M, E>;
  constexpr bool LAST = P + 1 == S::NP;
  if constexpr (P > 0) {
    if constexpr (TF_TW_EARLY) {
      fft_pass<M, E, P, INV, false, HOUT && LAST, NB>(v, tw);
    } else {
      PassTw<M, E, P> own;
      twf(own, t);
      fft_pass<M, E, P, INV, false, HOUT && LAST, NB>(v, &own);
    }
  } else {
    fft_pass<M, E, P, INV, ZIN, HOUT && LAST, NB>(v, (const PassTw<M, E, P>*)nullptr);
  }
  if constexpr (!LAST) {
    PassTw<M, E, P + 1> next;
    if constexpr (TF_TW_EARLY) twf(next, t);
    // ping-pong: exchange P uses buffer half P % 2, so the next exchange's stores
    // cannot overwrite words still being read and the trailing barrier goes away
    c32* buf = (PP && (P & 1)) ? sm + NB * sbs : sm;
    fft_store<M, E, P, NB>(v, buf, sbs, t);
    __syncthreads();
    load_canonical<M, E, NB>(v, buf, sbs, t);
    if constexpr (!PP) __syncthreads();
    fft_passes_from<M, E, P + 1, INV, ZIN, HOUT, NB, PP>(v, sm, sbs, t, twf, &next);
  }
}

// NB independent transforms per thread (interleaved for ILP, one barrier per
// exchange): on entry v[b][m] = x_b[t + T m]; on exit v[b][m] = X_b[t + T m].
// Transform b exchanges through sm + b*sbs (PP: also sm + (NB+b)*sbs, used on
// odd exchanges; valid back-to-back only when every call makes an even number of
// exchanges, i.e. NP odd).  ZIN: v[b][m] for m >= E/2 is zero (not read).  HOUT:
// only m < E/2 is valid on exit.  Every thread of the CTA must call it
// (contains barriers).  twf fills the forward twiddles of passes >= 1.
template <int M, int E, bool INV, bool ZIN, bool HOUT, int NB, typename TwF = TwTable,
          bool PP = false>
__device__ __forceinline__ void fftn(c32 (&v)[NB][E], c32* sm, int sbs, int t,
                                     const TwF& twf = TwF()) {
  static_assert(!PP || (FftShape<M, E>::NP % 2 == 1), "ping-pong needs an even exchange count");
  fft_passes_from<M, E, 0, INV, ZIN, HOUT, NB, PP>(v, sm, sbs, t, twf);
}

// Forward passes 0 .. NP-2 of fftn (no ping-pong), ending with pass NP-2's outputs
// stored in the exchange buffer and a barrier.  The caller loads the last pass's
// inputs in a thread mapping of its own (any canonical columns t, via canon_word)
// and runs the last pass itself with fft_pass<M, E, NP-1, ...> -- e.g. so that one
// thread holds both halves of a Hermitian mirror pair (k_rows_fwd_pf).
template <int M, int E, int P, bool ZIN, int NB>
__device__ __forceinline__ void fftn_to_last(c32 (&v)[NB][E], c32* sm, int sbs, int t,
                                             const PassTw<M, E, P>* tw = nullptr) {
  using S = FftShape<M, E>;
  static_assert(S::NP >= 2 && P + 1 < S::NP, "needs a last exchange");
  if constexpr (P > 0) fft_pass<M, E, P, false, false, false, NB>(v, tw);
  else fft_pass<M, E, 0, false, ZIN, false, NB>(v, (const PassTw<M, E, 0>*)nullptr);
  if constexpr (P + 2 < S::NP) {
    PassTw<M, E, P + 1> next;
    next.from_table(t);
    fft_store<M, E, P, NB>(v, sm, sbs, t);
    __syncthreads();
    load_canonical<M, E, NB>(v, sm, sbs, t);
    __syncthreads();
    fftn_to_last<M, E, P + 1, ZIN, NB>(v, sm, sbs, t, &next);
  } else {
    fft_store<M, E, P, NB>(v, sm, sbs, t);
    __syncthreads();
  }
}

// single transform
template <int M, int E, bool INV, bool ZIN = false, bool HOUT = false>
__device__ __forceinline__ void fft(c32 (&v)[E], c32* sm, int t) {
  c32 (&vv)[1][E] = *reinterpret_cast<c32(*)[1][E]>(&v);
  fftn<M, E, INV, ZIN, HOUT, 1>(vv, sm, 0, t);
}

template <int M, int E>
__device__ __forceinline__ void store_canonical(const c32 (&v)[E], c32* sm, int t) {
#pragma unroll
  for (int m = 0; m < E; ++m) sm[canon_word<M, E>(t, m)] = v[m];
}

// per-length tables W_L^j at word (L - 2) + j, computed in fp64
static __global__ void k_twiddle_init(c32* tw) {
  const int w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= TW_WORDS) return;
  int L = 2;
  while (w >= 2 * L - 2) L <<= 1;  // table L occupies words [L-2, 2L-2)
  const int j = w - (L - 2);
  double s, c;
  sincospi(-2.0 * (double)j / L, &s, &c);
  tw[w] = mk((float)c, (float)s);
}

// fill this translation unit's tables on the current device (synchronous)
static inline cudaError_t init_twiddles_tu() {
  c32* p = nullptr;
  cudaError_t e = cudaGetSymbolAddress((void**)&p, g_twiddle);
  if (e != cudaSuccess) return e;
  k_twiddle_init<<<(TW_WORDS + 255) / 256, 256>>>(p);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return cudaDeviceSynchronize();
}

}  // namespace tf
