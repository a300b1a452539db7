// Complex fp32 arithmetic on Blackwell's paired-fp32 datapath.
//
// sm_100a executes `add/sub/mul/fma.rn.f32x2` as single FADD2/FMUL2/FFMA2
// instructions on a 64-bit register pair.  A complex number is exactly such a
// pair, so a complex add is one instruction and a complex multiply is two
// (FMUL2 with a broadcast real part + FFMA2 with the swapped operand), where the
// scalar form needs two and four.  ptxas folds the swaps, broadcasts and
// single-lane negations below into operand modifiers (checked with cuobjdump:
// `R.F32x2.LO_HI`, `R.F32`, `.NP`), so none of the helpers costs a move.
#pragma once
#include <cstdint>

namespace tf {

struct __align__(8) c32 {
  float x, y;
};

__device__ __forceinline__ c32 mk(float x, float y) { c32 r; r.x = x; r.y = y; return r; }

__device__ __forceinline__ unsigned long long pk(c32 a) {
  unsigned long long r;
  asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a.x), "f"(a.y));
  return r;
}
__device__ __forceinline__ c32 upk(unsigned long long r) {
  c32 a;
  asm("mov.b64 {%0,%1}, %2;" : "=f"(a.x), "=f"(a.y) : "l"(r));
  return a;
}

__device__ __forceinline__ c32 cadd(c32 a, c32 b) {
  unsigned long long r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk(a)), "l"(pk(b)));
  return upk(r);
}
__device__ __forceinline__ c32 csub(c32 a, c32 b) {
  unsigned long long r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk(a)), "l"(pk(b)));
  return upk(r);
}
// elementwise a*b (both lanes)
__device__ __forceinline__ c32 pmul(c32 a, c32 b) {
  unsigned long long r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk(a)), "l"(pk(b)));
  return upk(r);
}
// elementwise a*b + c
__device__ __forceinline__ c32 pfma(c32 a, c32 b, c32 c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(pk(a)), "l"(pk(b)), "l"(pk(c)));
  return upk(r);
}
__device__ __forceinline__ c32 scale(c32 a, float s) { return pmul(a, mk(s, s)); }

// a * w
__device__ __forceinline__ c32 cmul(c32 a, c32 w) {
  c32 p = pmul(a, mk(w.x, w.x));
  return pfma(mk(a.y, a.x), mk(-w.y, w.y), p);
}
// a * conj(w)
__device__ __forceinline__ c32 cmulc(c32 a, c32 w) {
  c32 p = pmul(a, mk(w.x, w.x));
  return pfma(mk(a.y, a.x), mk(w.y, -w.y), p);
}
__device__ __forceinline__ c32 conj(c32 a) { return mk(a.x, -a.y); }
// a * (-i) and a * (+i)
__device__ __forceinline__ c32 mul_mi(c32 a) { return mk(a.y, -a.x); }
__device__ __forceinline__ c32 mul_pi(c32 a) { return mk(-a.y, a.x); }
// a + s*(-i)*b  with s = +1 (forward, e^{-i pi/2}) handled by the caller via rot()
template <bool INV>
__device__ __forceinline__ c32 rot_q(c32 a) {  // multiply by e^{-+ i pi/2}
  return INV ? mul_pi(a) : mul_mi(a);
}

}  // namespace tf
