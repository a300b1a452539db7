// Complex fp32 arithmetic on Blackwell's paired-fp32 datapath.
//
// sm_100a executes add/mul/fma on a float2 register pair as one FADD2 / FMUL2
// / FFMA2 instruction (__fadd2_rn & co., crt/sm_100_rt.h).  A complex number is
// exactly such a pair, so a complex add is one instruction and a complex
// multiply two (FMUL2 with the broadcast real part, FFMA2 with the swapped
// operand) where the scalar form needs two and four.  ptxas folds the lane
// swaps, broadcasts and single-lane negations used below into operand
// modifiers (`R.F32x2.LO_HI`, `R.F32`, `.NP`; checked with cuobjdump), so the
// helpers cost no moves.  Note x + 0 is NOT folded (IEEE -0), so zero-padded
// inputs are pruned explicitly by the FFT codelets.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace tf {

typedef float2 c32;

__device__ __forceinline__ c32 mk(float x, float y) { return make_float2(x, y); }

__device__ __forceinline__ c32 cadd(c32 a, c32 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ c32 csub(c32 a, c32 b) { return __fadd2_rn(a, mk(-b.x, -b.y)); }
__device__ __forceinline__ c32 pmul(c32 a, c32 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ c32 pfma(c32 a, c32 b, c32 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ c32 scale(c32 a, float s) { return pmul(a, mk(s, s)); }

// a * w
__device__ __forceinline__ c32 cmul(c32 a, c32 w) {
  return pfma(mk(a.y, a.x), mk(-w.y, w.y), pmul(a, mk(w.x, w.x)));
}
// a * conj(w)
__device__ __forceinline__ c32 cmulc(c32 a, c32 w) {
  return pfma(mk(a.y, a.x), mk(w.y, -w.y), pmul(a, mk(w.x, w.x)));
}
__device__ __forceinline__ c32 conj(c32 a) { return mk(a.x, -a.y); }
// a * (-i), a * (+i)
__device__ __forceinline__ c32 mul_mi(c32 a) { return mk(a.y, -a.x); }
__device__ __forceinline__ c32 mul_pi(c32 a) { return mk(-a.y, a.x); }
// multiply by e^{-+ i pi/2} (forward / inverse quarter turn)
template <bool INV>
__device__ __forceinline__ c32 rot_q(c32 a) {
  return INV ? mul_pi(a) : mul_mi(a);
}
// a * h(1 -+ i) : the e^{-+ i pi/4} twiddle scaled by h = 1/sqrt2, two instructions
template <bool INV>
__device__ __forceinline__ c32 rot_e(c32 a, float h) {
  const c32 p = pmul(a, mk(h, h));
  return INV ? pfma(mk(a.y, a.x), mk(-h, h), p) : pfma(mk(a.y, a.x), mk(h, -h), p);
}

}  // namespace tf
