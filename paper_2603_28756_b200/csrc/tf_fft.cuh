// Register/shared-memory Stockham FFT engine for power-of-two lengths.
//
// A length-M transform is run by a *group* of T = M/E threads; thread t keeps
// the E elements {t + T*m : m < E} in registers ("canonical layout").  Each
// pass applies radix-R butterflies (R | E, R <= 16) to register-resident data;
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
// Twiddles: fp32 table of e^{-2 pi i j/TW_MAX} built in fp64 once per device
// (tf_init); powers w^r by a log-depth product tree (error ~log2 R ulp).
#pragma once
#include "tf_complex.cuh"

namespace tf {

constexpr int TW_MAX = 16384;  // largest supported transform length
// Concatenated per-length tables: W_L^j = e^{-2 pi i j/L} at word (L - 2) + j for
// L = 2, 4, ..., TW_MAX, so the twiddles of one pass are contiguous in k.
constexpr int TW_WORDS = 2 * TW_MAX - 2;
// Direct power tables for radix-16 passes (TwDirect): for NS in {2,4,8,16}
// the powers W_{16 NS}^{k r} laid out [r][k] at tws_base(NS); for the M = 4096
// last pass (NS = 256, k = t) the powers W_4096^{t r} laid out [r-1][t].
constexpr int TWS_WORDS = 16 * 31;
__host__ __device__ constexpr int tws_base(int ns) { return 16 * (ns - 1); }
// one copy per translation unit (internal linkage, no relocatable device code);
// every TU that runs FFTs fills its copy from ensure_init() via init_twiddles_tu()
static __device__ c32 g_twiddle[TW_WORDS];
static __device__ c32 g_tw_small[TWS_WORDS];
static __device__ c32 g_tw_t256[15 * 256];

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

// --------------------------------------------------------------- codelets
// In-place DFT of u[0..R-1]; output X[k] in u[k].  ZIN: u[R/2..R-1] == 0 on
// entry (not read).  HOUT: only X[0..R/2-1] are produced.

template <bool INV, bool ZIN = false, bool HOUT = false>
__device__ __forceinline__ void dft4(c32& u0, c32& u1, c32& u2, c32& u3) {
  c32 t0, t1, t2, t3;
  if constexpr (ZIN) {
    t0 = u0; t1 = u0; t2 = u1; t3 = rot_q<INV>(u1);
  } else {
    t0 = cadd(u0, u2); t1 = csub(u0, u2);
    t2 = cadd(u1, u3); t3 = rot_q<INV>(csub(u1, u3));
  }
  u0 = cadd(t0, t2);
  u1 = cadd(t1, t3);
  if constexpr (!HOUT) {
    u2 = csub(t0, t2);
    u3 = csub(t1, t3);
  }
}

constexpr float kH = 0.70710678118654752440f;  // 1/sqrt 2

template <bool INV>
__device__ __forceinline__ c32 w8_1(c32 a) { return rot_e<INV>(a, kH); }  // e^{-+i pi/4}
template <bool INV>
__device__ __forceinline__ c32 w8_3(c32 a) {                           // e^{-+3i pi/4}
  const c32 p = pmul(a, mk(-kH, -kH));
  return INV ? pfma(mk(a.y, a.x), mk(-kH, kH), p) : pfma(mk(a.y, a.x), mk(kH, -kH), p);
}

template <bool INV, bool ZIN = false, bool HOUT = false>
__device__ __forceinline__ void dft8(c32 (&u)[8]) {
  c32 a[4], b[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if constexpr (ZIN) {
      a[k] = u[k]; b[k] = u[k];
    } else {
      a[k] = cadd(u[k], u[k + 4]); b[k] = csub(u[k], u[k + 4]);
    }
  }
  b[1] = w8_1<INV>(b[1]);
  b[2] = rot_q<INV>(b[2]);
  b[3] = w8_3<INV>(b[3]);
  dft4<INV, false, HOUT>(a[0], a[1], a[2], a[3]);
  dft4<INV, false, HOUT>(b[0], b[1], b[2], b[3]);
#pragma unroll
  for (int m = 0; m < (HOUT ? 2 : 4); ++m) {
    u[2 * m] = a[m];
    u[2 * m + 1] = b[m];
  }
}

template <bool INV>
__device__ __forceinline__ c32 w16(c32 a, int e) {  // a * W16^e for e in {1,2,3,4,6,9}
  const float c1 = 0.92387953251128675613f, s1 = 0.38268343236508977173f;
  switch (e) {
    case 1: return INV ? cmul(a, mk(c1, s1)) : cmul(a, mk(c1, -s1));
    case 2: return w8_1<INV>(a);
    case 3: return INV ? cmul(a, mk(s1, c1)) : cmul(a, mk(s1, -c1));
    case 4: return rot_q<INV>(a);
    case 6: return w8_3<INV>(a);
    default: return INV ? cmul(a, mk(-c1, -s1)) : cmul(a, mk(-c1, s1));  // 9
  }
}

template <bool INV, bool ZIN = false, bool HOUT = false>
__device__ __forceinline__ void dft16(c32 (&u)[16]) {
  // 16 = 4 x 4: DFT4 over l of u[k + 4l], twiddle W16^{km}, DFT4 over k -> X[m + 4j]
  c32 y[4][4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    c32 a0 = u[k], a1 = u[k + 4], a2, a3;
    if constexpr (!ZIN) { a2 = u[k + 8]; a3 = u[k + 12]; }
    dft4<INV, ZIN>(a0, a1, a2, a3);
    y[k][0] = a0; y[k][1] = a1; y[k][2] = a2; y[k][3] = a3;
  }
#pragma unroll
  for (int k = 1; k < 4; ++k)
#pragma unroll
    for (int m = 1; m < 4; ++m) y[k][m] = w16<INV>(y[k][m], k * m);
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    c32 a0 = y[0][m], a1 = y[1][m], a2 = y[2][m], a3 = y[3][m];
    dft4<INV, false, HOUT>(a0, a1, a2, a3);
    u[m] = a0; u[m + 4] = a1;
    if constexpr (!HOUT) { u[m + 8] = a2; u[m + 12] = a3; }
  }
}

template <int R, bool INV, bool ZIN, bool HOUT>
__device__ __forceinline__ void dft(c32 (&u)[R]) {
  if constexpr (R == 1) {
  } else if constexpr (R == 2) {
    if constexpr (ZIN) {
      u[1] = u[0];
    } else {
      const c32 s = cadd(u[0], u[1]), d = csub(u[0], u[1]);
      u[0] = s; u[1] = d;
    }
  } else if constexpr (R == 4) {
    dft4<INV, ZIN, HOUT>(u[0], u[1], u[2], u[3]);
  } else if constexpr (R == 8) {
    dft8<INV, ZIN, HOUT>(u);
  } else {
    static_assert(R == 16, "radix");
    dft16<INV, ZIN, HOUT>(u);
  }
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

// Forward twiddles of pass P for thread t: wp[i][r] = w_i^r, w_i = e^{-2 pi i k_i/(NS R)},
// k_i = (t + i T) mod NS, from the per-length table and a log-depth product tree.
template <int M, int E, int P>
struct PassTw {
  using S = FftShape<M, E>;
  static constexpr int R = 1 << S::lradix(P);
  static constexpr int NS = S::ns(P);
  static constexpr int ST = E / R;
  c32 w[ST][R];
  // table entry W^k + log-depth product tree for the other powers (FP work)
  __device__ __forceinline__ void from_table(int t) {
#pragma unroll
    for (int i = 0; i < ST; ++i) {
      const int k = (t + i * S::T) & (NS - 1);
      w[i][1] = tw_w<NS * R>(k);
#pragma unroll
      for (int r = 2; r < R; ++r) w[i][r] = cmul(w[i][r / 2], w[i][r - r / 2]);
    }
  }
  // every power straight from a table where one exists (memory instead of FP
  // work; used by the FMA-bound column kernel): [r][k] tables for NS <= 16 and
  // the per-thread [r][t] table of the M = 4096 last pass
  __device__ __forceinline__ void from_table_direct(int t) {
#pragma unroll
    for (int i = 0; i < ST; ++i) {
      const int k = (t + i * S::T) & (NS - 1);
      if constexpr (R == 16 && NS >= 2 && NS <= 16) {
#pragma unroll
        for (int r = 1; r < R; ++r) w[i][r] = g_tw_small[tws_base(NS) + r * NS + k];
      } else if constexpr (R == 16 && NS == 256 && S::T == 256) {
#pragma unroll
        for (int r = 1; r < R; ++r) w[i][r] = __ldg(g_tw_t256 + (r - 1) * 256 + k);
      } else {
        w[i][1] = tw_w<NS * R>(k);
#pragma unroll
        for (int r = 2; r < R; ++r) w[i][r] = cmul(w[i][r / 2], w[i][r - r / 2]);
      }
    }
  }
};

// default twiddle source: table + product tree
struct TwTable {
  template <int M, int E, int P>
  __device__ __forceinline__ void operator()(PassTw<M, E, P>& tw, int t) const {
    tw.from_table(t);
  }
};

// small [r][k] power tables where NS <= 16 (L1-resident, 2 KB), product tree for
// the per-thread last-pass powers (whose 30 KB table would live in L2)
struct TwMixed {
  template <int M, int E, int P>
  __device__ __forceinline__ void operator()(PassTw<M, E, P>& tw, int t) const {
    using PT = PassTw<M, E, P>;
    if constexpr (PT::R == 16 && PT::NS >= 2 && PT::NS <= 16) tw.from_table_direct(t);
    else tw.from_table(t);
  }
};

// direct power tables (see PassTw::from_table_direct)
struct TwDirect {
  template <int M, int E, int P>
  __device__ __forceinline__ void operator()(PassTw<M, E, P>& tw, int t) const {
    tw.from_table_direct(t);
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
      if constexpr (P > 0 && R > 1) {
#pragma unroll
        for (int r = 1; r < (ZIN ? R / 2 : R); ++r)
          u[r] = INV ? cmulc(u[r], tw->w[i][r]) : cmul(u[r], tw->w[i][r]);
      }
      dft<R, INV, ZIN, HOUT>(u);
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
// (or product-tree FMAs) overlap the shared-memory round trip and the barrier
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

static __global__ void k_twiddle_init_small(c32* small, c32* t256) {
  const int w = blockIdx.x * blockDim.x + threadIdx.x;
  double s, c;
  if (w < TWS_WORDS) {
    int ns = 1;
    while (w >= tws_base(2 * ns)) ns *= 2;  // segment [tws_base(ns), tws_base(2 ns))
    const int e = w - tws_base(ns), r = e / ns, k = e - r * ns;
    const int L = 16 * ns;
    sincospi(-2.0 * (double)((k * r) % L) / L, &s, &c);
    small[w] = mk((float)c, (float)s);
  }
  if (w < 15 * 256) {
    const int r = w / 256 + 1, t = w % 256;
    sincospi(-2.0 * (double)((t * r) % 4096) / 4096.0, &s, &c);
    t256[w] = mk((float)c, (float)s);
  }
}

// fill this translation unit's tables on the current device (synchronous)
static inline cudaError_t init_twiddles_tu() {
  c32 *p = nullptr, *q = nullptr, *u = nullptr;
  cudaError_t e = cudaGetSymbolAddress((void**)&p, g_twiddle);
  if (e == cudaSuccess) e = cudaGetSymbolAddress((void**)&q, g_tw_small);
  if (e == cudaSuccess) e = cudaGetSymbolAddress((void**)&u, g_tw_t256);
  if (e != cudaSuccess) return e;
  k_twiddle_init<<<(TW_WORDS + 255) / 256, 256>>>(p);
  k_twiddle_init_small<<<(15 * 256 + 255) / 256, 256>>>(q, u);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return cudaDeviceSynchronize();
}

}  // namespace tf
