// Register/shared-memory Stockham FFT engine for power-of-two lengths.
//
// A length-M transform is run by a *group* of T = M/E threads; thread t keeps
// the E elements {t + T*m : m < E} in registers ("canonical layout").  Each
// pass applies radix-R butterflies (R | E, R <= 16) to register-resident
// data; between passes the group exchanges through a padded shared-memory
// buffer (index i -> i + i/16 keeps every exchange at the 2-wavefront minimum
// for 8-byte elements).  With the first radix possibly smaller than 16 and all
// later ones equal to E, both the first pass's input set and the last pass's
// output set of thread t are exactly its canonical set, which is what lets the
// Toeplitz column kernel multiply by the PSF and start the inverse transform
// without touching shared memory (see toeplitz.cu, k_cols_conv).
//
// Forward transforms use e^{-2 pi i jk/M} (numpy.fft sign); INV uses the
// conjugate and is unnormalised.  Twiddles come from a fp32 table of
// e^{-2 pi i j/TW_MAX} built once per device in fp64 (tf_init), with powers
// w^r formed by a log-depth product tree (error ~log2(R) ulp).
#pragma once
#include "tf_complex.cuh"

namespace tf {

constexpr int TW_MAX = 16384;  // largest supported transform length
// defined once: the library is a single translation unit (lib.cu)
__device__ c32 g_twiddle[TW_MAX];

__host__ __device__ constexpr int ilog2(int v) { return v <= 1 ? 0 : 1 + ilog2(v >> 1); }
__host__ __device__ constexpr int pad_idx(int i) { return i + (i >> 4); }
// padded exchange-buffer stride per group, chosen == 4 (mod 16) so that
// concurrently used group buffers start on different bank pairs
__host__ __device__ constexpr int group_stride(int M) {
  return pad_idx(M) + ((4 - (pad_idx(M) % 16)) + 16) % 16 + 16;
}

template <bool INV>
__device__ __forceinline__ c32 tw_table(int j) {  // e^{-+2 pi i j / TW_MAX}
  c32 w = g_twiddle[j];
  return INV ? conj(w) : w;
}

// --------------------------------------------------------------- codelets
// In-place DFT of u[0..R-1]; output X[k] in u[k].

template <bool INV>
__device__ __forceinline__ void dft2(c32& a, c32& b) {
  c32 s = cadd(a, b), d = csub(a, b);
  a = s; b = d;
}

template <bool INV>
__device__ __forceinline__ void dft4(c32& u0, c32& u1, c32& u2, c32& u3) {
  c32 t0 = cadd(u0, u2), t1 = csub(u0, u2);
  c32 t2 = cadd(u1, u3), t3 = rot_q<INV>(csub(u1, u3));
  u0 = cadd(t0, t2); u2 = csub(t0, t2);
  u1 = cadd(t1, t3); u3 = csub(t1, t3);
}

// e^{-+ i pi/4} and e^{-+ 3 i pi/4}
template <bool INV>
__device__ __forceinline__ c32 w8_1(c32 a) {
  const float h = 0.70710678118654752440f;
  return INV ? scale(mk(a.x - a.y, a.y + a.x), h) : scale(mk(a.x + a.y, a.y - a.x), h);
}
template <bool INV>
__device__ __forceinline__ c32 w8_3(c32 a) {
  const float h = 0.70710678118654752440f;
  return INV ? scale(mk(-a.x - a.y, a.x - a.y), h) : scale(mk(a.y - a.x, -a.x - a.y), h);
}

template <bool INV>
__device__ __forceinline__ void dft8(c32 (&u)[8]) {
  c32 a[4], b[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    a[k] = cadd(u[k], u[k + 4]);
    b[k] = csub(u[k], u[k + 4]);
  }
  b[1] = w8_1<INV>(b[1]);
  b[2] = rot_q<INV>(b[2]);
  b[3] = w8_3<INV>(b[3]);
  dft4<INV>(a[0], a[1], a[2], a[3]);
  dft4<INV>(b[0], b[1], b[2], b[3]);
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    u[2 * m] = a[m];
    u[2 * m + 1] = b[m];
  }
}

template <bool INV>
__device__ __forceinline__ c32 w16(c32 a, int e) {  // a * W16^e, e in [0,16)
  // cos/sin(2 pi e/16)
  const float c1 = 0.92387953251128675613f, s1 = 0.38268343236508977173f;
  const float h = 0.70710678118654752440f;
  switch (e & 15) {
    case 0: return a;
    case 1: return INV ? cmul(a, mk(c1, s1)) : cmul(a, mk(c1, -s1));
    case 2: return w8_1<INV>(a);
    case 3: return INV ? cmul(a, mk(s1, c1)) : cmul(a, mk(s1, -c1));
    case 4: return rot_q<INV>(a);
    case 6: return w8_3<INV>(a);
    case 9: return INV ? cmul(a, mk(-c1, -s1)) : cmul(a, mk(-c1, s1));
    default: {
      float c = cospif(e / 8.0f), s = sinpif(e / 8.0f);
      return INV ? cmul(a, mk(c, s)) : cmul(a, mk(c, -s));
    }
  }
  (void)h;
}

template <bool INV>
__device__ __forceinline__ void dft16(c32 (&u)[16]) {
  c32 y[4][4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    c32 a0 = u[k], a1 = u[k + 4], a2 = u[k + 8], a3 = u[k + 12];
    dft4<INV>(a0, a1, a2, a3);
    y[k][0] = a0; y[k][1] = a1; y[k][2] = a2; y[k][3] = a3;
  }
#pragma unroll
  for (int k = 1; k < 4; ++k)
#pragma unroll
    for (int m = 1; m < 4; ++m) y[k][m] = w16<INV>(y[k][m], k * m);
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    c32 a0 = y[0][m], a1 = y[1][m], a2 = y[2][m], a3 = y[3][m];
    dft4<INV>(a0, a1, a2, a3);
    u[m] = a0; u[m + 4] = a1; u[m + 8] = a2; u[m + 12] = a3;
  }
}

template <int R, bool INV>
__device__ __forceinline__ void dft(c32 (&u)[R]) {
  if constexpr (R == 1) {
  } else if constexpr (R == 2) {
    dft2<INV>(u[0], u[1]);
  } else if constexpr (R == 4) {
    dft4<INV>(u[0], u[1], u[2], u[3]);
  } else if constexpr (R == 8) {
    dft8<INV>(u);
  } else {
    static_assert(R == 16, "radix");
    dft16<INV>(u);
  }
}

// --------------------------------------------------------------- engine

template <int M, int E>
struct FftShape {
  static_assert((M & (M - 1)) == 0 && M >= 2 && M <= TW_MAX, "power-of-two length");
  static_assert(E <= M && (E & (E - 1)) == 0, "E");
  static constexpr int T = M / E;          // threads per transform
  static constexpr int L = ilog2(M);
  static constexpr int LE = ilog2(E);
  static constexpr int NP = (L + LE - 1) / LE;  // passes
  static constexpr int LFIRST = L - (NP - 1) * LE;
  __host__ __device__ static constexpr int lradix(int p) { return p == 0 ? LFIRST : LE; }
  __host__ __device__ static constexpr int ns(int p) { return p == 0 ? 1 : (1 << (LFIRST + (p - 1) * LE)); }
  static constexpr int SB = group_stride(M);  // smem c32 per group
};

template <int M, int E, int P, bool INV>
__device__ __forceinline__ void fft_pass(c32 (&v)[E], int t) {
  using S = FftShape<M, E>;
  constexpr int R = 1 << S::lradix(P);
  constexpr int NS = S::ns(P);
  constexpr int ST = E / R;  // butterflies per thread
#pragma unroll
  for (int i = 0; i < ST; ++i) {
    c32 u[R];
#pragma unroll
    for (int r = 0; r < R; ++r) u[r] = v[i + r * ST];
    if constexpr (P > 0 && R > 1) {
      const int b = t + i * S::T;
      const int k = b & (NS - 1);
      // w = e^{-2 pi i k / (NS*R)}
      c32 w = tw_table<INV>(k * (TW_MAX / (NS * R)));
      c32 wp[R];
      wp[1] = w;
#pragma unroll
      for (int r = 2; r < R; ++r) wp[r] = cmul(wp[r / 2], wp[r - r / 2]);
#pragma unroll
      for (int r = 1; r < R; ++r) u[r] = cmul(u[r], wp[r]);
    }
    dft<R, INV>(u);
#pragma unroll
    for (int r = 0; r < R; ++r) v[i + r * ST] = u[r];
  }
}

// write pass-P outputs to the exchange buffer in Stockham order
template <int M, int E, int P>
__device__ __forceinline__ void fft_store(const c32 (&v)[E], c32* sm, int t) {
  using S = FftShape<M, E>;
  constexpr int R = 1 << S::lradix(P);
  constexpr int NS = S::ns(P);
  constexpr int ST = E / R;
#pragma unroll
  for (int i = 0; i < ST; ++i) {
    const int b = t + i * S::T;
    const int base = (b / NS) * NS * R + (b & (NS - 1));
#pragma unroll
    for (int r = 0; r < R; ++r) sm[pad_idx(base + r * NS)] = v[i + r * ST];
  }
}

template <int M, int E>
__device__ __forceinline__ void load_canonical(c32 (&v)[E], const c32* sm, int t) {
  using S = FftShape<M, E>;
#pragma unroll
  for (int m = 0; m < E; ++m) v[m] = sm[pad_idx(t + S::T * m)];
}

template <int M, int E, int P, bool INV>
__device__ __forceinline__ void fft_passes_from(c32 (&v)[E], c32* sm, int t) {
  using S = FftShape<M, E>;
  fft_pass<M, E, P, INV>(v, t);
  if constexpr (P + 1 < S::NP) {
    fft_store<M, E, P>(v, sm, t);
    __syncthreads();
    load_canonical<M, E>(v, sm, t);
    __syncthreads();
    fft_passes_from<M, E, P + 1, INV>(v, sm, t);
  }
}

// Full transform: on entry v[m] = x[t + T m]; on exit v[m] = X[t + T m].
// Every thread of the CTA must call it (it contains __syncthreads).
template <int M, int E, bool INV>
__device__ __forceinline__ void fft(c32 (&v)[E], c32* sm, int t) {
  fft_passes_from<M, E, 0, INV>(v, sm, t);
}

}  // namespace tf
