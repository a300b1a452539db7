// Length-M = 5Q transforms (Q a power of two, 256 <= Q <= 1024) on top of the
// power-of-two engine (tf_fft.cuh).  M = 5Q is the FFT side whenever it is the
// smallest admissible one: N = 640, 1280, 2560 (C5) run on M = 1280, 2560, 5120
// instead of 2048, 4096, 8192 (2.56x less FFT work at N = 2560).
//
// A transform is run by T5 = 5Q/16 threads, seen as 5 subgroups of T' = Q/16.
// With n = n1 + Q n2 (n1 < Q, n2 < 5) and k = 5 k1 + k2 (DIF over n2):
//   z_k2[n1]      = W_M^{n1 k2} sum_n2 x[n1 + Q n2] W_5^{n2 k2}      (radix-5 step)
//   X[5 k1 + k2]  = FFT_Q(z_k2)[k1]                                  (5 Q-point FFTs)
// Two register layouts:
//   I ("strided"): thread t < Q/4 holds x[t + (Q/4) m], m < 20 (n1 = t + (Q/4) j,
//                  n2 = m / 4 with m = j + 4 n2); the other Q/16 threads hold nothing;
//   G ("grouped"): thread p = k2 T' + t' holds X[5 (t' + T' m') + k2], m' < 16,
//                  i.e. the canonical layout of subgroup k2's Q-point transform.
// fft5_fwd maps I -> G, fft5_inv (the transposed algorithm, conjugated) G -> I;
// each adds one shared-memory exchange to the Q-point transform's two.
#pragma once
#include "tf_fft.cuh"

namespace tf {

constexpr int Q5_MIN = 256, Q5_MAX = 1024;
// W_{5Q}^j for j < Q at word (Q - Q5_MIN) + j, Q = 256, 512, 1024 (one copy per TU)
constexpr int TW5_WORDS = (2 * Q5_MAX - Q5_MIN);
static __device__ c32 g_tw5[TW5_WORDS];

template <int Q>
struct Fft5Shape {
  static_assert(Q >= Q5_MIN && Q <= Q5_MAX && (Q & (Q - 1)) == 0, "Q");
  static constexpr int M = 5 * Q;
  static constexpr int E = 16;
  static constexpr int TP = Q / E;      // threads per subgroup
  static constexpr int T5 = 5 * TP;     // threads per transform
  static constexpr int TI = Q / 4;      // active threads in layout I
  static constexpr int SBQ = group_stride(Q, 4);  // exchange words per subgroup
  static constexpr int SMEM_WORDS = 5 * SBQ;      // >= M
};

// radix-5 DFT in place (forward e^{-2 pi i/5}; INV conjugate)
template <bool INV>
__device__ __forceinline__ void dft5(c32 (&a)[5]) {
  constexpr float c1 = 0.30901699437494742410f, c2 = -0.80901699437494742410f;
  constexpr float s1 = 0.95105651629515357212f, s2 = 0.58778525229247312917f;
  const c32 t1 = cadd(a[1], a[4]), t2 = cadd(a[2], a[3]);
  const c32 t3 = csub(a[1], a[4]), t4 = csub(a[2], a[3]);
  const c32 x0 = cadd(a[0], cadd(t1, t2));
  const c32 b1 = pfma(t1, mk(c1, c1), pfma(t2, mk(c2, c2), a[0]));
  const c32 b2 = pfma(t1, mk(c2, c2), pfma(t2, mk(c1, c1), a[0]));
  const c32 d1 = pfma(t3, mk(s1, s1), pmul(t4, mk(s2, s2)));
  const c32 d2 = pfma(t3, mk(s2, s2), pmul(t4, mk(-s1, -s1)));
  const c32 r1 = rot_q<INV>(d1), r2 = rot_q<INV>(d2);  // -+ i d
  a[0] = x0;
  a[1] = cadd(b1, r1);
  a[4] = csub(b1, r1);
  a[2] = cadd(b2, r2);
  a[3] = csub(b2, r2);
}

// w^1..w^4 of w = W_M^{n1}
template <int Q>
__device__ __forceinline__ void tw5_powers(int n1, c32 (&w)[5]) {
  w[1] = g_tw5[(Q - Q5_MIN) + n1];
  w[2] = cmul(w[1], w[1]);
  w[3] = cmul(w[2], w[1]);
  w[4] = cmul(w[2], w[2]);
}

// I -> G.  xi: layout I (ZIN: x[n] = 0 for n >= M/2, i.e. m >= 10, not read).
// sm: Fft5Shape<Q>::SMEM_WORDS words; every thread of the transform calls it.
template <int Q, bool ZIN>
__device__ __forceinline__ void fft5_fwd(const c32 (&xi)[20], c32 (&v)[16], c32* sm, int p) {
  using S = Fft5Shape<Q>;
  constexpr int TP = S::TP;
  if (p < S::TI) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      c32 a[5];
#pragma unroll
      for (int n2 = 0; n2 < 5; ++n2) {
        const int m = j + 4 * n2;
        a[n2] = (ZIN && m >= 10) ? mk(0.f, 0.f) : xi[m];
      }
      dft5<false>(a);
      const int n1 = p + S::TI * j;
      c32 w[5];
      tw5_powers<Q>(n1, w);
      const int word = canon_word<Q, 16>(n1 % TP, n1 / TP);
      sm[word] = a[0];
#pragma unroll
      for (int k2 = 1; k2 < 5; ++k2) sm[k2 * S::SBQ + word] = cmul(a[k2], w[k2]);
    }
  }
  __syncthreads();
  const int g = p / TP, t = p - g * TP;
  c32 (&vv)[1][16] = *reinterpret_cast<c32(*)[1][16]>(&v);
  load_canonical<Q, 16, 1>(vv, sm + g * S::SBQ, 0, t);
  __syncthreads();  // the Q-point transform reuses the buffers
  fftn<Q, 16, false, false, false, 1>(vv, sm + g * S::SBQ, 0, t);
}

// G -> I, unnormalised inverse (conjugate twiddles).  HOUT: only xo[m] for m < 10
// (n < M/2) are produced.
template <int Q, bool HOUT>
__device__ __forceinline__ void fft5_inv(c32 (&v)[16], c32 (&xo)[20], c32* sm, int p) {
  using S = Fft5Shape<Q>;
  constexpr int TP = S::TP;
  const int g = p / TP, t = p - g * TP;
  c32 (&vv)[1][16] = *reinterpret_cast<c32(*)[1][16]>(&v);
  fftn<Q, 16, true, false, false, 1>(vv, sm + g * S::SBQ, 0, t);
  // the last pass is register-only and the transform's last exchange is fenced
  store_canonical<Q, 16>(v, sm + g * S::SBQ, t);
  __syncthreads();
  if (p < S::TI) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n1 = p + S::TI * j;
      const int word = canon_word<Q, 16>(n1 % TP, n1 / TP);
      c32 w[5];
      tw5_powers<Q>(n1, w);
      c32 a[5];
      a[0] = sm[word];
#pragma unroll
      for (int k2 = 1; k2 < 5; ++k2) a[k2] = cmulc(sm[k2 * S::SBQ + word], w[k2]);
      dft5<true>(a);
#pragma unroll
      for (int n2 = 0; n2 < 5; ++n2) {
        const int m = j + 4 * n2;
        if (!HOUT || m < 10) xo[m] = a[n2];
      }
    }
  }
  __syncthreads();  // buffers free for the caller
}

// W_{5Q}^j tables in fp64
static __global__ void k_twiddle5_init(c32* tw) {
  const int w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= TW5_WORDS) return;
  int Q = Q5_MIN;
  while (w >= (2 * Q - Q5_MIN)) Q <<= 1;  // segment Q occupies [Q - Q5_MIN, 2Q - Q5_MIN)
  const int j = w - (Q - Q5_MIN);
  double s, c;
  sincospi(-2.0 * (double)j / (5.0 * Q), &s, &c);
  tw[w] = mk((float)c, (float)s);
}

static inline cudaError_t init_twiddles5_tu() {
  c32* p = nullptr;
  cudaError_t e = cudaGetSymbolAddress((void**)&p, g_tw5);
  if (e != cudaSuccess) return e;
  k_twiddle5_init<<<(TW5_WORDS + 255) / 256, 256>>>(p);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return cudaDeviceSynchronize();
}

}  // namespace tf
