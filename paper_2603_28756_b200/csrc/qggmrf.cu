// qGGMRF prior fused with the momentum update (K4) and the objective
// reductions (K5) -- SURVEY.md §8 rows a8-a11, a14, a15.
//
// Reference: tomoforge/qggmrf.py:117-130 (rho, rho'), :142-189 (prior_grad with
// ghost/halo validity), :192-217 (prior_energy over the lexicographically
// positive half stencil, halo_hi pairs counted by the lower slab);
// tomoforge/solver.py:147-169 (the loop: grad at y, f_new = y - grad/L,
// optional clamp, objective, restart, momentum).
//
// Data layout: volumes are [z][ix][iy] fp32 (reference data[ix, iy]); the
// stencil offset (dz, dy, dx) moves (z, ix, iy).  Both kernels stream along z
// (2.5-D): a CTA owns a 32 (iy) x 8 (ix) column tile and marches through the
// slab keeping the last planes of y (K4, 3 planes) or f_new (K5, 2 planes) in
// shared memory with a one-voxel ring.
//
// K4 forms the extrapolated point on the fly, y = f + c (f - f_prev), and
// K y = K f + c (K f - K f_prev) by linearity, so a solver iteration needs a
// single Toeplitz apply (of f_new) instead of the reference's two
// (solver.py:149 and :157).  K5 returns, in fp64, E(f_new), the direct
// fidelity <f_new, K f_new/2 - R*g> and the increment
// <f_new - f, (K f_new + K f)/2 - R*g> used for the restart test.
#include <type_traits>

#include "tf_common.cuh"

namespace tf {

struct PriorConsts {
  float inv_sp;      // 1 / sigma^p
  float inv_psp;     // 1 / (p sigma^p)
  float c0;          // (p - q) log2(T sigma)
  float pq;          // p - q
  float qp;          // q / p
  float p;           // p
  float pm1;         // p - 1
  float w[4];        // stencil weights by number of nonzero offset components (1, 2, 3)
};

constexpr int TX = 32, TY = 8;
constexpr int HX = TX + 2, HY = TY + 2;  // tile with a one-voxel ring
constexpr int HALO_ELEMS = HX * HY;       // 340: thread i loads elements i and i + 256

// MUFU transcendentals (log2 / exp2: one XU instruction each)
__device__ __forceinline__ float lg2a(float x) {
  float r;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float ex2a(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// 1/x for x >= 1 on the FMA pipe: integer seed (rel. error < 12.5 %) and three
// Newton steps (error squares each step: < 4e-8), two lanes at a time.  Keeps
// the XU free for log2/exp2, which bound these kernels.
__device__ __forceinline__ float2 rcp2_ge1(float2 x) {
  float2 y = mk(__int_as_float(0x7EF311C3 - __float_as_int(x.x)),
                __int_as_float(0x7EF311C3 - __float_as_int(x.y)));
  const float2 nx = mk(-x.x, -x.y), one = mk(1.f, 1.f);
#pragma unroll
  for (int i = 0; i < 3; ++i) y = pfma(y, pfma(nx, y, one), y);
  return y;
}

// v = (|d| / (T sigma))^(p-q) for two differences; t = log2|d| (v = 0 at d = 0)
__device__ __forceinline__ float2 qg_v2(float2 d, float2& t, const PriorConsts& pc) {
  t = mk(lg2a(fabsf(d.x)), lg2a(fabsf(d.y)));
  const float2 e = pfma(mk(pc.pq, pc.pq), t, mk(-pc.c0, -pc.c0));
  return mk(ex2a(e.x), ex2a(e.y));
}

// sigma^p rho'(d) = sign(d) |d|^(p-1) (1 + (q/p) v) / (1 + v)^2   (qggmrf.py:124-130)
// XRCP: the reciprocal on the XU (MUFU.RCP) instead of Newton on the FMA pipe;
// kernels that are issue-bound with XU headroom use it for a share of the pairs.
__device__ __forceinline__ float2 rcp2_xu(float2 x) {
  float2 y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y.x) : "f"(x.x));
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y.y) : "f"(x.y));
  return y;
}

template <bool P2, bool XRCP = false>
__device__ __forceinline__ float2 drho2(float2 d, const PriorConsts& pc) {
  float2 t;
  const float2 v = qg_v2(d, t, pc);
  const float2 one = mk(1.f, 1.f);
  const float2 r = XRCP ? rcp2_xu(cadd(v, one)) : rcp2_ge1(cadd(v, one));
  const float2 s = pmul(pfma(mk(pc.qp, pc.qp), v, one), pmul(r, r));
  float2 mag;
  if constexpr (P2) mag = d;
  else mag = mk(copysignf(ex2a(pc.pm1 * t.x), d.x), copysignf(ex2a(pc.pm1 * t.y), d.y));
  return pmul(mag, s);
}

// p sigma^p rho(d) = |d|^p / (1 + v)   (qggmrf.py:117-121)
template <bool P2, bool XRCP = false>
__device__ __forceinline__ float2 rho2(float2 d, const PriorConsts& pc) {
  float2 t;
  const float2 v = qg_v2(d, t, pc);
  const float2 r = XRCP ? rcp2_xu(cadd(v, mk(1.f, 1.f))) : rcp2_ge1(cadd(v, mk(1.f, 1.f)));
  float2 mag;
  if constexpr (P2) mag = pmul(d, d);
  else mag = mk(ex2a(pc.p * t.x), ex2a(pc.p * t.y));
  return pmul(mag, r);
}

template <int NT>
__device__ __forceinline__ double block_sum_d(double v, double* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x < 32) {
    r = threadIdx.x < NT / 32 ? sh[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) r += __shfl_down_sync(0xffffffffu, r, o);
  }
  return r;
}

// Plane pointers of a slab with optional halo planes z = -1 and z = nz.
struct Planes {
  const float* main;  // [nz][n][n]
  const float* lo;    // plane z = -1 or null (invalid: cliques dropped)
  const float* hi;    // plane z = nz or null
  __device__ __forceinline__ const float* at(int z, int nz, long long nn) const {
    if (z < 0) return lo;
    if (z >= nz) return hi;
    return main + z * nn;
  }
};

// The two halo-tile elements a thread stages per plane, resolved once per CTA:
// tile position and in-plane offset, or -1 outside the grid.
struct HaloSlots {
  int sm[2];
  long long off[2];
  __device__ __forceinline__ void init(int h, int w) {
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int e = threadIdx.x + k * TX * TY;
      const int ly = e / HX, lx = e - ly * HX;
      const int gx = blockIdx.y * TY + ly - 1, gy = blockIdx.x * TX + lx - 1;
      sm[k] = e < HALO_ELEMS ? e : -1;
      off[k] = (e < HALO_ELEMS && gx >= 0 && gx < h && gy >= 0 && gy < w) ? (long long)gx * w + gy
                                                                          : -1;
    }
  }
};

// In-plane neighbour masks of voxel (ix, iy): weight * [neighbour inside the slice]
struct InPlaneW {
  float w8[9];  // index (dy+1)*3 + (dx+1): offsets in the same plane (centre unused)
  float wz[9];  // the same (dy, dx) on the planes above/below (weight class + 1)
  __device__ __forceinline__ void init(int ix, int iy, int h, int w, const PriorConsts& pc) {
#pragma unroll
    for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
      for (int dx = -1; dx <= 1; ++dx) {
        const bool ok = ix + dy >= 0 && ix + dy < h && iy + dx >= 0 && iy + dx < w;
        const int k = (dy != 0) + (dx != 0);
        w8[(dy + 1) * 3 + dx + 1] = ok ? pc.w[k] : 0.f;
        wz[(dy + 1) * 3 + dx + 1] = ok ? pc.w[k + 1] : 0.f;
      }
  }
};

// ============================================================ K4
// grad = K y - R*g + lam * grad_prior(y)   (Kf/Kfp/rstar may be null -> 0)
// write_grad == 0: out = y - grad / L  [clamped at 0 if NONNEG]   (the update)
// write_grad == 1: out = grad                                     (prior_grad API)
// partial[block] = sum grad^2 over the block's voxels (fp64)
// The 26 (3-D) or 8 (2-D) differences of a voxel are evaluated two at a time on
// the paired-fp32 datapath; per pair the XU runs only log2 and exp2.
template <bool THREE_D, bool P2, bool NONNEG>
__global__ void __launch_bounds__(TX* TY)
k_prior_update(Planes F, Planes FP, const float* __restrict__ Kf, const float* Kfp,
               const float* __restrict__ rstar, float* f_new,
               double* __restrict__ partial, int nz, int h, int w, float c, float lam,
               float inv_L, int write_grad, PriorConsts pc, const float* __restrict__ c_dev) {
  __shared__ float ys[3][HY][HX];
  __shared__ double red[TX * TY / 32];
  if (c_dev) c = *c_dev;  // momentum decided on the device (tf_solver_decide)
  const int tx = threadIdx.x % TX, ty = threadIdx.x / TX;
  const int iy = blockIdx.x * TX + tx;  // contiguous axis
  const int ix = blockIdx.y * TY + ty;
  const long long nn = (long long)h * w;
  const bool inside = ix < h && iy < w;
  HaloSlots hs;
  hs.init(h, w);
  InPlaneW ipw;
  ipw.init(ix, iy, h, w, pc);
  float* ysf = &ys[0][0][0];

  // Software pipeline: the halo-tile values of the next plane (raw f and
  // f_prev at this thread's two slots) and the per-voxel operands (K f, K f_prev,
  // R*g) of the next plane are loaded into registers one step ahead, so global
  // latency overlaps the current plane's stencil.
  float hf[2], hp[2];
  auto fetch_plane = [&](int zz) {
    const float* pf = F.at(zz, nz, nn);
    const float* pp = FP.at(zz, nz, nn);
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      hf[k] = hp[k] = 0.f;
      if (hs.sm[k] >= 0 && pf && hs.off[k] >= 0) {
        hf[k] = __ldg(pf + hs.off[k]);
        hp[k] = __ldg(pp + hs.off[k]);
      }
    }
  };
  // y = f + c (f - f_prev) into ring slot s (0 outside the grid / invalid plane)
  auto commit_plane = [&](int s) {
#pragma unroll
    for (int k = 0; k < 2; ++k)
      if (hs.sm[k] >= 0) ysf[s * HALO_ELEMS + hs.sm[k]] = fmaf(c, hf[k] - hp[k], hf[k]);
  };
  float nkf = 0.f, nkp = 0.f, nrs = 0.f;
  auto fetch_ops = [&](int zz) {
    if (!inside || zz >= nz) return;
    const long long o = zz * nn + (long long)ix * w + iy;
    if (Kf) {
      nkf = __ldg(Kf + o);
      nkp = Kfp[o];  // plain load: Kfp may alias f_new (solver ring)
    }
    if (rstar) nrs = __ldg(rstar + o);
  };

  const float glam = lam * pc.inv_sp;
  double gsq = 0.0;
  if (THREE_D) {
    fetch_plane(-1);
    commit_plane(2);
    fetch_plane(0);
    commit_plane(0);
    fetch_plane(1);
  } else {
    fetch_plane(0);
  }
  fetch_ops(0);
  for (int z = 0; z < nz; ++z) {
    const int s0 = THREE_D ? z % 3 : 0, sp = (z + 1) % 3, sm = (z + 2) % 3;  // z, z+1, z-1
    if (THREE_D) {
      commit_plane(sp);      // plane z+1, loaded during the previous step
      fetch_plane(z + 2);    // in flight during this step
    } else {
      commit_plane(0);       // 8-neighbour stencil: slices are independent
      if (z + 1 < nz) fetch_plane(z + 1);
    }
    const float kfv = nkf, kpv = nkp, rsv = nrs;
    fetch_ops(z + 1);
    __syncthreads();
    if (inside) {
      const float yv = ys[s0][ty + 1][tx + 1];
      float2 acc = mk(0.f, 0.f);
      // in-plane: 8 neighbours as 4 pairs
      float nb[8], wv[8];
      {
        int q = 0;
#pragma unroll
        for (int j = 0; j < 9; ++j) {
          if (j == 4) continue;
          nb[q] = ys[s0][ty + j / 3][tx + j % 3];
          wv[q] = ipw.w8[j];
          ++q;
        }
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 g = drho2<P2>(mk(yv - nb[2 * i], yv - nb[2 * i + 1]), pc);
        acc = pfma(mk(wv[2 * i], wv[2 * i + 1]), g, acc);
      }
      if (THREE_D) {
        // planes z-1 and z+1: same (dy, dx) paired across the two planes
        const bool lo_ok = z > 0 || FP.lo != nullptr;
        const bool hi_ok = z + 1 < nz || FP.hi != nullptr;
        if (lo_ok && hi_ok) {  // interior plane (uniform branch): both planes valid
#pragma unroll
          for (int j = 0; j < 9; ++j) {
            const float a = ys[sm][ty + j / 3][tx + j % 3];
            const float b = ys[sp][ty + j / 3][tx + j % 3];
            acc = pfma(mk(ipw.wz[j], ipw.wz[j]), drho2<P2>(mk(yv - a, yv - b), pc), acc);
          }
        } else {
          const float lo_w = lo_ok ? 1.f : 0.f, hi_w = hi_ok ? 1.f : 0.f;
#pragma unroll
          for (int j = 0; j < 9; ++j) {
            const float a = ys[sm][ty + j / 3][tx + j % 3];
            const float b = ys[sp][ty + j / 3][tx + j % 3];
            const float2 g = drho2<P2>(mk(yv - a, yv - b), pc);
            acc = pfma(mk(ipw.wz[j] * lo_w, ipw.wz[j] * hi_w), g, acc);
          }
        }
      }
      const long long o = z * nn + (long long)ix * w + iy;
      const float ky = fmaf(c, kfv - kpv, kfv);
      const float grad = fmaf(glam, acc.x + acc.y, ky - rsv);
      if (write_grad) {
        f_new[o] = grad;
      } else {
        float fn = fmaf(-grad, inv_L, yv);
        if (NONNEG) fn = fmaxf(fn, 0.f);
        f_new[o] = fn;
      }
      gsq = fma((double)grad, (double)grad, gsq);
    }
    __syncthreads();
  }
  const double r = block_sum_d<TX * TY>(gsq, red);
  if (threadIdx.x == 0) partial[blockIdx.y * gridDim.x + blockIdx.x] = r;
}

// every TF_XRCP_K4-th (K5: TF_XRCP_K5-th) clique pair of the tiled kernels takes its
// reciprocal on the XU, balancing XU against issue.  The gradient part of K45 uses
// the same choice (its update must equal K4's bit for bit), and K45's XU also
// carries the energy's transcendentals: 6 is best for K45 (measured on 64 x 2048^2:
// K45 5.36 ms at 3, 5.32 at 6, 5.35 with none; K4 alone 3.15 / 3.17 / 3.20)
#ifndef TF_K45_MB3
#define TF_K45_MB3 1  // allow the 3-CTA K45 when the wave count favours it
#endif
#ifndef TF_XRCP_K4
#define TF_XRCP_K4 6
#endif
#ifndef TF_XRCP_K5
#define TF_XRCP_K5 0
#endif

// ============================================================ K4, symmetric pairs (3-D)
// rho' is odd, so the 26-neighbour gradient needs each clique once:
//   grad_prior(p) = sum_k w_k(p, p+o_k) G_k(p) - sum_k w_k(p-o_k, p) G_k(p - o_k),
//   G_k(q) = rho'(y_q - y_{q+o_k}),
// over the 13 offsets o_k of the half stencil (4 in the plane, 9 towards z+1);
// w is the clique weight times [both voxels in the slice].
//
// A CTA owns a 32 x (8 RY) column tile (RY voxels per thread, rows ty + 8 r).
// Per plane step a thread evaluates the 13 G of each of its voxels (forward
// terms, summed in registers) and 1-2 of the "strip" G on the tile's
// one-voxel ring that are backward terms of tile voxels; all go to shared
// memory unweighted, and after a barrier each voxel adds its 13 weighted
// backward terms.  The z+1 cliques of plane z are the backward terms of plane
// z+1, so they are kept one step (double buffer); with a slab halo below, a
// pre-step at z = -1 produces the cliques between the halo plane and plane 0.
// Half the log2/exp2 work of k_prior_update, for ~30 more shared-memory
// accesses per voxel.  Tiles whose ring lies inside the slice (all but the
// outermost) take weights straight from the constant bank; edge tiles derive
// them from four neighbour bits.
template <int RY>
struct SymTile {
  static constexpr int W = TX, H = TY * RY;       // tile
  static constexpr int RW = W + 2, RH = H + 2;    // with the ring
  static constexpr int CELLS = RW * RH;
  static constexpr int NT = TX * TY;
  static constexpr int SLOTS = (CELLS + NT - 1) / NT;  // ring cells staged per thread
  // (dy, dx): (0,1) (1,-1) (1,0) (1,1) in the plane, then (-1..1, -1..1) towards z+1
  __host__ __device__ static constexpr int dy(int k) { return k == 0 ? 0 : k < 4 ? 1 : (k - 4) / 3 - 1; }
  __host__ __device__ static constexpr int dx(int k) { return k == 0 ? 1 : k < 4 ? k - 2 : (k - 4) % 3 - 1; }
  // weight class: number of nonzero components of (dz, dy, dx)
  __host__ __device__ static constexpr int cls(int k) { return (k >= 4) + (dy(k) != 0) + (dx(k) != 0); }
  // ring-cell offset of the partner voxel within a plane
  __host__ __device__ static constexpr int off(int k) { return dy(k) * RW + dx(k); }
  // ring cells of the box "tile - o_k" that are outside the tile
  __host__ __device__ static constexpr int strip(int k) {
    return W * H - (H - (dy(k) != 0)) * (W - (dx(k) != 0));
  }
  __host__ __device__ static constexpr int strips() {
    int n = 0;
    for (int k = 0; k < 13; ++k) n += strip(k);
    return n;
  }
  static constexpr int GSLOTS = 4 + 2 * 9;  // in-plane G, then two buffers of z+1 G
  static_assert(strips() <= 2 * NT, "at most two strip cliques per thread");

  // strip clique i: packed (qa | qb << 11 | k << 22), qa / qb its ring cells; -1 if none
  __device__ static int strip_item(int i) {
    if (i >= strips()) return -1;
    int k = 0;
#pragma unroll
    for (int kk = 0; kk < 13; ++kk)
      if (k == kk && i >= strip(kk)) {
        i -= strip(kk);
        ++k;
      }
    int ddy = 0, ddx = 0;
#pragma unroll
    for (int kk = 0; kk < 13; ++kk)
      if (kk == k) {
        ddy = dy(kk);
        ddx = dx(kk);
      }
    int r, cc;
    const int nrow = ddy != 0 ? W : 0;  // the ring row first (dy = +-1), then a ring column
    if (i < nrow) {
      r = ddy == 1 ? -1 : H;
      cc = i - ddx;
    } else {
      r = (ddy == -1 ? 1 : 0) + (i - nrow);
      cc = ddx == 1 ? -1 : W;
    }
    const int qa = (r + 1) * RW + cc + 1;
    return qa | (qa + ddy * RW + ddx) << 11 | k << 22;
  }
};

// FUSED (K45): additionally the K5 sums of the CURRENT iterate F -- its energy
// over the half stencil (+ pairs into F.hi), <F, Kf/2 - R*g> and the increment
// <F - FP, (Kf + Kfp)/2 - R*g> -- from the same tiles and operands, while the
// update part computes the NEXT iterate at y = F + c (F - FP) with the momentum
// c of the no-restart branch.  F's planes are staged in fsf; partial[4 b + j] =
// {E(F), fid, dfid, sum grad^2}.
template <int RY, bool P2, bool NONNEG, bool EDGE, bool FUSED = false>
__device__ __forceinline__ void prior_sym_tile(const Planes& F, const Planes& FP,
                                               const float* __restrict__ Kf,
                                               const float* Kfp,  // may alias f_new
                                               const float* __restrict__ rstar,
                                               float* f_new, double* partial, int nz,
                                               int h, int w, float c, float lam, float inv_L,
                                               int write_grad, const PriorConsts& pc, float* ysf,
                                               float* gsf, double* red, float* fsf = nullptr,
                                               bool energy = false) {
  using S = SymTile<RY>;
  // per-voxel operands: Kf, Kfp, R*g (+ FP when fused)
  constexpr int NOP = FUSED ? 4 : 3;
  using Ops = float[NOP][RY];
  constexpr int CELLS = S::CELLS, NT = S::NT;
  const int tx = threadIdx.x % TX, ty = threadIdx.x / TX;
  const int gx0 = blockIdx.y * S::H, gy0 = blockIdx.x * S::W;
  const int iy = gy0 + tx;
  const long long nn = (long long)h * w;
  const int me0 = (ty + 1) * S::RW + tx + 1;  // own ring cell of row r: me0 + r TY RW
  bool inside[RY];
  int vo[RY];     // own in-plane offsets
  int nbits[RY];  // EDGE: neighbour bits (x-, x+, y-, y+, inside)
#pragma unroll
  for (int r = 0; r < RY; ++r) {
    const int ix = gx0 + ty + TY * r;
    inside[r] = !EDGE || (ix < h && iy < w);
    vo[r] = ix * w + iy;
    nbits[r] = (ix > 0) | (ix + 1 < h) << 1 | (iy > 0) << 2 | (iy + 1 < w) << 3 | inside[r] << 4;
  }
  // ring cells this thread stages (cell threadIdx + m NT) and their in-plane offsets
  int coff[S::SLOTS];
#pragma unroll
  for (int m = 0; m < S::SLOTS; ++m) {
    const int e = threadIdx.x + m * NT;
    const int ly = e / S::RW, lx = e - ly * S::RW;
    const int gx = gx0 + ly - 1, gy = gy0 + lx - 1;
    coff[m] = (e < CELLS && gx >= 0 && gx < h && gy >= 0 && gy < w) ? gx * w + gy : -1;
  }
  constexpr bool LAST_PARTIAL = CELLS % NT != 0;
  const bool last_ok = !LAST_PARTIAL || threadIdx.x + (S::SLOTS - 1) * NT < CELLS;
  // weight of the clique between voxel r and voxel r + s*o_k (s = +1 forward, -1 backward)
  auto wgt = [&](int r, int k, int s) -> float {
    const float wc = pc.w[S::cls(k)];
    if constexpr (!EDGE) {
      return wc;
    } else {
      const int ddy = s * S::dy(k), ddx = s * S::dx(k);
      const int need = 16 | (ddy < 0 ? 1 : ddy > 0 ? 2 : 0) | (ddx < 0 ? 4 : ddx > 0 ? 8 : 0);
      return (nbits[r] & need) == need ? wc : 0.f;
    }
  };
  const int it0 = S::strip_item(threadIdx.x), it1 = S::strip_item(threadIdx.x + NT);

  float hf[S::SLOTS], hp[S::SLOTS];
  auto fetch_plane = [&](int zz) {
    const float* pf = F.at(zz, nz, nn);
    const float* pp = FP.at(zz, nz, nn);
    const bool ok = pf != nullptr;
#pragma unroll
    for (int m = 0; m < S::SLOTS; ++m) {
      const bool v = ok && coff[m] >= 0;
      hf[m] = v ? __ldg(pf + coff[m]) : 0.f;
      hp[m] = v ? __ldg(pp + coff[m]) : 0.f;
    }
  };
  auto fetch_ops = [&](int zz, Ops& o) {
    if (zz >= nz) return;
    const long long base = zz * nn;
#pragma unroll
    for (int r = 0; r < RY; ++r) {
      if (Kf) {
        o[0][r] = inside[r] ? __ldg(Kf + base + vo[r]) : 0.f;
        o[1][r] = inside[r] ? Kfp[base + vo[r]] : 0.f;  // may alias f_new
      }
      if (rstar) o[2][r] = inside[r] ? __ldg(rstar + base + vo[r]) : 0.f;
      if constexpr (FUSED) o[NOP - 1][r] = inside[r] ? __ldg(FP.main + base + vo[r]) : 0.f;
    }
  };

  const float glam = lam * pc.inv_sp;
  const bool has_lo = FP.lo != nullptr;
  double gsq = 0.0, e_acc = 0.0, fid = 0.0, dfid = 0.0;
  Ops opA, opB;
#pragma unroll
  for (int j = 0; j < NOP; ++j)
#pragma unroll
    for (int r = 0; r < RY; ++r) opA[j][r] = opB[j][r] = 0.f;

  // One plane step; S0 = z & 1 is a compile-time constant, so every shared-memory
  // offset below is an immediate.  `cur` holds this plane's operands, `nxt`
  // receives the next plane's.
  auto step = [&](auto s0c, int z, Ops& cur, Ops& nxt) {
    constexpr int S0 = decltype(s0c)::value, S1 = S0 ^ 1;
    float* yw = ysf + S1 * CELLS + threadIdx.x;  // plane z+1 lands in slot S1
#pragma unroll
    for (int m = 0; m < S::SLOTS; ++m)
      if (m + 1 < S::SLOTS || last_ok) yw[m * NT] = fmaf(c, hf[m] - hp[m], hf[m]);
    if constexpr (FUSED) {
      float* fw = fsf + S1 * CELLS + threadIdx.x;
#pragma unroll
      for (int m = 0; m < S::SLOTS; ++m)
        if (m + 1 < S::SLOTS || last_ok) fw[m * NT] = hf[m];
    }
    fetch_plane(z + 2);
    fetch_ops(z + 1, nxt);
    __syncthreads();
    // ---- phase A: own cliques (forward terms) and strip cliques -> shared memory
    const float* ya = ysf + S0 * CELLS;
    const float* yb = ysf + S1 * CELLS;
    float* gin = gsf;                          // in-plane G of plane z
    float* gcur = gsf + (4 + 9 * S0) * CELLS;  // z+1 G of plane z
    float yv[RY], f_in[RY], f_x[RY];
#pragma unroll
    for (int r = 0; r < RY; ++r) {
      yv[r] = ya[me0 + r * TY * S::RW];
      f_in[r] = f_x[r] = 0.f;
    }
    auto strip_d = [&](int item) {
      const int qa = item & 2047, qb = (item >> 11) & 2047;
      return ya[qa] - ((item >> 22) >= 4 ? yb : ya)[qb];
    };
    auto strip_dst = [&](int item) {
      const int qa = item & 2047, k = item >> 22;
      return k * CELLS + qa + (k >= 4 ? 9 * CELLS * S0 : 0);
    };
    constexpr int NOWN = 13 * RY;
    constexpr int NEVAL = (NOWN + 3) & ~1;  // + up to two strip cliques, even
    float2 yy2 = mk(0.f, 0.f), nb2 = mk(0.f, 0.f);
#pragma unroll
    for (int e = 0; e < NEVAL; ++e) {
      float yself, ynb;
      if (e < NOWN) {
        const int r = e / 13, k = e % 13;
        yself = yv[r];
        ynb = (k < 4 ? ya : yb)[me0 + r * TY * S::RW + S::off(k)];
      } else {
        const int item = e == NOWN ? it0 : e == NOWN + 1 ? it1 : -1;
        if (item >= 0) {
          const int qa = item & 2047, qb = (item >> 11) & 2047;
          yself = ya[qa];
          ynb = ((item >> 22) >= 4 ? yb : ya)[qb];
        } else {
          yself = ynb = 0.f;
        }
      }
      if (e & 1) {
        yy2.y = yself;
        nb2.y = ynb;
        const bool xr = TF_XRCP_K4 > 0 && (e / 2) % TF_XRCP_K4 == TF_XRCP_K4 - 1;
        const float2 g = xr ? drho2<P2, true>(csub(yy2, nb2), pc) : drho2<P2>(csub(yy2, nb2), pc);
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          const int ee = e - 1 + h2;
          const float gv = h2 ? g.y : g.x;
          if (ee < NOWN) {
            const int r = ee / 13, k = ee % 13;
            const int cell = me0 + r * TY * S::RW;
            if (k < 4) {
              gin[k * CELLS + cell] = gv;
              f_in[r] = fmaf(wgt(r, k, 1), gv, f_in[r]);
            } else {
              gcur[(k - 4) * CELLS + cell] = gv;
              f_x[r] = fmaf(wgt(r, k, 1), gv, f_x[r]);
            }
          } else {
            const int item = ee == NOWN ? it0 : ee == NOWN + 1 ? it1 : -1;
            if (item >= 0) gsf[strip_dst(item)] = gv;
          }
        }
      } else {
        yy2.x = yself;
        nb2.x = ynb;
      }
    }
    (void)strip_d;
    // ---- fused: energy of F's plane z over the half stencil (K5's sums)
    float xf[RY];
    (void)xf;
    if constexpr (FUSED) {
      const float* fa = fsf + S0 * CELLS;
      const float* fb = fsf + S1 * CELLS;
      const float up = (z + 1 < nz || F.hi != nullptr) ? 1.f : 0.f;
      float eacc[RY];
#pragma unroll
      for (int r = 0; r < RY; ++r) {
        xf[r] = fa[me0 + r * TY * S::RW];
        eacc[r] = 0.f;
      }
      if (energy && z >= 0) {
        constexpr int NE = 13 * RY, NEV = (NE + 1) & ~1;
        float2 x2 = mk(0.f, 0.f), n2 = mk(0.f, 0.f);
#pragma unroll
        for (int e = 0; e < NEV; ++e) {
          float xs = 0.f, xn = 0.f;
          if (e < NE) {
            const int r = e / 13, k = e % 13;
            xs = xf[r];
            xn = (k < 4 ? fa : fb)[me0 + r * TY * S::RW + S::off(k)];
          }
          if (e & 1) {
            x2.y = xs;
            n2.y = xn;
            const float2 g = rho2<P2>(csub(x2, n2), pc);
#pragma unroll
            for (int h2 = 0; h2 < 2; ++h2) {
              const int ee = e - 1 + h2;
              if (ee < NE) {
                const int r = ee / 13, k = ee % 13;
                eacc[r] = fmaf(k < 4 ? wgt(r, k, 1) : wgt(r, k, 1) * up, h2 ? g.y : g.x, eacc[r]);
              }
            }
          } else {
            x2.x = xs;
            n2.x = xn;
          }
        }
#pragma unroll
        for (int r = 0; r < RY; ++r)
          if (inside[r]) e_acc += (double)(eacc[r] * pc.inv_psp);
      }
    }
    __syncthreads();
    // ---- phase B: backward terms, gradient, update
    if (z >= 0) {
      const bool lo_ok = z > 0 || has_lo;
      const bool hi_ok = z + 1 < nz || FP.hi != nullptr;
      const float* gprev = gsf + (4 + 9 * S1) * CELLS;  // z+1 G of plane z-1
      float* outz = f_new + z * nn;
#pragma unroll
      for (int r = 0; r < RY; ++r) {
        const int cell = me0 + r * TY * S::RW;
        float b_in = 0.f, b_x = 0.f;
#pragma unroll
        for (int k = 0; k < 4; ++k) b_in = fmaf(wgt(r, k, -1), gin[k * CELLS + cell - S::off(k)], b_in);
        if (lo_ok) {
#pragma unroll
          for (int k = 4; k < 13; ++k)
            b_x = fmaf(wgt(r, k, -1), gprev[(k - 4) * CELLS + cell - S::off(k)], b_x);
        }
        const float prior = (f_in[r] - b_in) + ((hi_ok ? f_x[r] : 0.f) - b_x);
        const float ky = fmaf(c, cur[0][r] - cur[1][r], cur[0][r]);
        const float grad = fmaf(glam, prior, ky - cur[2][r]);
        if constexpr (FUSED) {
          if (inside[r]) {  // K5's fidelity sums of F (fp32 products, fp64 running sums)
            const float fnv = xf[r], kfn = cur[0][r], kf = cur[1][r], rs = cur[2][r];
            fid += (double)(fnv * fmaf(0.5f, kfn, -rs));
            dfid += (double)((fnv - cur[NOP - 1][r]) * (fmaf(0.5f, kfn + kf, 0.f) - rs));
          }
        }
        if (inside[r]) {
          if (write_grad) {
            outz[vo[r]] = grad;
          } else {
            float fn = fmaf(-grad, inv_L, yv[r]);
            if (NONNEG) fn = fmaxf(fn, 0.f);
            outz[vo[r]] = fn;
          }
          gsq = fma((double)grad, (double)grad, gsq);
        }
      }
    }
  };
  using I0 = std::integral_constant<int, 0>;
  using I1 = std::integral_constant<int, 1>;
  // prologue: plane z0 into its slot, plane z0+1 in registers
  const int z0 = has_lo ? -1 : 0;
  fetch_plane(z0);
  {
    float* yw = ysf + (z0 & 1) * CELLS + threadIdx.x;
#pragma unroll
    for (int m = 0; m < S::SLOTS; ++m)
      if (m + 1 < S::SLOTS || last_ok) yw[m * NT] = fmaf(c, hf[m] - hp[m], hf[m]);
    if constexpr (FUSED) {
      float* fw = fsf + (z0 & 1) * CELLS + threadIdx.x;
#pragma unroll
      for (int m = 0; m < S::SLOTS; ++m)
        if (m + 1 < S::SLOTS || last_ok) fw[m * NT] = hf[m];
    }
  }
  fetch_plane(z0 + 1);
  if (has_lo) step(I1{}, -1, opB, opA);  // cliques halo -> plane 0; fetches plane 0's operands
  else fetch_ops(0, opA);
  for (int z = 0; z < nz; z += 2) {
    step(I0{}, z, opA, opB);
    if (z + 1 < nz) step(I1{}, z + 1, opB, opA);
  }
  const int b = blockIdx.y * gridDim.x + blockIdx.x;
  if constexpr (FUSED) {
    const double r0 = block_sum_d<NT>(e_acc, red);
    const double r1 = block_sum_d<NT>(fid, red);
    const double r2 = block_sum_d<NT>(dfid, red);
    const double r3 = block_sum_d<NT>(gsq, red);
    if (threadIdx.x == 0) {
      partial[4 * b] = r0;
      partial[4 * b + 1] = r1;
      partial[4 * b + 2] = r2;
      partial[4 * b + 3] = r3;
    }
  } else {
    const double r = block_sum_d<NT>(gsq, red);
    if (threadIdx.x == 0) partial[b] = r;
  }
}

#ifndef TF_K4_RY
#define TF_K4_RY 2
#endif
#ifndef TF_K4_MINB
#define TF_K4_MINB 3
#endif
constexpr int K4_RY = TF_K4_RY;

template <bool P2, bool NONNEG>
__global__ void __launch_bounds__(TX* TY, TF_K4_MINB)
k_prior_update_sym(Planes F, Planes FP, const float* __restrict__ Kf, const float* Kfp,
                   const float* __restrict__ rstar, float* f_new,
                   double* __restrict__ partial, int nz, int h, int w, float c, float lam,
                   float inv_L, int write_grad, PriorConsts pc, const float* __restrict__ c_dev,
                   const double* __restrict__ only_if) {
  using S = SymTile<K4_RY>;
  extern __shared__ float sym_smem[];
  if (only_if && *only_if == 0.0) return;  // conditional re-run (after a restart only)
  if (c_dev) c = *c_dev;  // momentum decided on the device (tf_solver_decide)
  __shared__ double red[TX * TY / 32];
  float* ys = sym_smem;                // [2][CELLS]
  float* gs = sym_smem + 2 * S::CELLS;  // [GSLOTS][CELLS]
  const bool interior = blockIdx.y * S::H >= 1 && (blockIdx.y + 1) * S::H + 1 <= h &&
                        blockIdx.x * S::W >= 1 && (blockIdx.x + 1) * S::W + 1 <= w;
  if (interior)
    prior_sym_tile<K4_RY, P2, NONNEG, false>(F, FP, Kf, Kfp, rstar, f_new, partial, nz, h, w, c,
                                             lam, inv_L, write_grad, pc, ys, gs, red);
  else
    prior_sym_tile<K4_RY, P2, NONNEG, true>(F, FP, Kf, Kfp, rstar, f_new, partial, nz, h, w, c,
                                            lam, inv_L, write_grad, pc, ys, gs, red);
}

// K45: K5 of iteration k fused with K4 of iteration k+1 (one pass over the slab
// instead of two; same transcendental work).  The momentum of the no-restart
// branch is computed here from the device state with tf_solver_decide's exact
// fp64 arithmetic, so when iteration k does not restart the result is the one
// the unfused K5 -> decide -> K4 sequence gives; after a restart the solver
// re-runs K4 with c = 0 (k_prior_update_sym with `only_if` = the restart flag).
// MB: resident CTAs per SM the registers are budgeted for.  MB = 3 (80 registers,
// small spills) is ~2 % faster per SM than MB = 2 (128 registers) but each CTA --
// which walks every plane of its tile column -- runs ~1.47x longer, so it only pays
// when the tile count fills enough waves (k45_minblocks(); profiles/r02).
template <bool P2, bool NONNEG, int MB>
__global__ void __launch_bounds__(TX* TY, MB)
k_prior_energy_update(Planes F, Planes FP, const float* __restrict__ Kf, const float* Kfp,
                      const float* __restrict__ rstar, float* f_new, double* __restrict__ partial,
                      int nz, int h, int w, float lam, float inv_L, int energy, PriorConsts pc,
                      const double* __restrict__ state) {
  using S = SymTile<K4_RY>;
  extern __shared__ float sym_smem[];
  __shared__ double red[TX * TY / 32];
  const double t = state[3];
  const double t_next = __dadd_rn(1.0, sqrt(__dadd_rn(1.0, __dmul_rn(__dmul_rn(4.0, t), t)))) / 2.0;
  const float c = (float)((t - 1.0) / t_next);
  float* ys = sym_smem;                                   // [2][CELLS]
  float* gs = sym_smem + 2 * S::CELLS;                    // [GSLOTS][CELLS]
  float* fs = sym_smem + (2 + S::GSLOTS) * S::CELLS;      // [2][CELLS]
  const bool interior = blockIdx.y * S::H >= 1 && (blockIdx.y + 1) * S::H + 1 <= h &&
                        blockIdx.x * S::W >= 1 && (blockIdx.x + 1) * S::W + 1 <= w;
  if (interior)
    prior_sym_tile<K4_RY, P2, NONNEG, false, true>(F, FP, Kf, Kfp, rstar, f_new, partial, nz, h, w,
                                                   c, lam, inv_L, 0, pc, ys, gs, red, fs,
                                                   energy != 0);
  else
    prior_sym_tile<K4_RY, P2, NONNEG, true, true>(F, FP, Kf, Kfp, rstar, f_new, partial, nz, h, w,
                                                  c, lam, inv_L, 0, pc, ys, gs, red, fs,
                                                  energy != 0);
}

static size_t sym_smem_bytes(bool fused = false) {
  using S = SymTile<K4_RY>;
  return sizeof(float) * (2 + S::GSLOTS + (fused ? 2 : 0)) * S::CELLS;
}
static dim3 sym_grid(int h, int w) {
  using S = SymTile<K4_RY>;
  return dim3((w + S::W - 1) / S::W, (h + S::H - 1) / S::H);
}

// ============================================================ K5
// partial[block*3 + {0,1,2}] = { E(f_new) (half stencil + halo_hi pairs),
//   <f_new, K f_new / 2 - R*g>,  <f_new - f, (K f_new + K f)/2 - R*g> (0 if f null) }
template <bool THREE_D, bool P2>
__global__ void __launch_bounds__(TX* TY)
k_energy_fid(Planes FN, const float* __restrict__ f, const float* __restrict__ Kfn,
             const float* __restrict__ Kf, const float* __restrict__ rstar,
             double* __restrict__ partial, int nz, int h, int w, int with_prior, PriorConsts pc) {
  __shared__ float xs[2][HY][HX];
  __shared__ double red[TX * TY / 32];
  const int tx = threadIdx.x % TX, ty = threadIdx.x / TX;
  const int iy = blockIdx.x * TX + tx;
  const int ix = blockIdx.y * TY + ty;
  const long long nn = (long long)h * w;
  const bool inside = ix < h && iy < w;
  HaloSlots hs;
  hs.init(h, w);
  InPlaneW ipw;
  ipw.init(ix, iy, h, w, pc);
  float* xsf = &xs[0][0][0];
  // software pipeline as in K4: next plane's halo values and per-voxel operands
  // are fetched into registers one step ahead
  float hv[2];
  auto fetch_plane = [&](int zz) {
    const float* pf = FN.at(zz, nz, nn);
#pragma unroll
    for (int k = 0; k < 2; ++k)
      hv[k] = (hs.sm[k] >= 0 && pf && hs.off[k] >= 0) ? __ldg(pf + hs.off[k]) : 0.f;
  };
  auto commit_plane = [&](int s) {
#pragma unroll
    for (int k = 0; k < 2; ++k)
      if (hs.sm[k] >= 0) xsf[s * HALO_ELEMS + hs.sm[k]] = hv[k];
  };
  float n_fn = 0.f, n_kfn = 0.f, n_rs = 0.f, n_f = 0.f, n_kf = 0.f;
  auto fetch_ops = [&](int zz) {
    if (!inside || zz >= nz) return;
    const long long o = zz * nn + (long long)ix * w + iy;
    if (!with_prior) n_fn = __ldg(FN.main + o);  // with the prior it is the tile centre
    if (Kfn) n_kfn = __ldg(Kfn + o);
    if (rstar) n_rs = __ldg(rstar + o);
    if (f && Kfn) {
      n_f = __ldg(f + o);
      n_kf = __ldg(Kf + o);
    }
  };
  double e_acc = 0.0, fid = 0.0, dfid = 0.0;
  if (with_prior) {
    if (THREE_D) {
      fetch_plane(0);
      commit_plane(0);
      fetch_plane(1);
    } else {
      fetch_plane(0);
    }
  }
  fetch_ops(0);
  for (int z = 0; z < nz; ++z) {
    const int s0 = THREE_D ? (z & 1) : 0, s1 = (z + 1) & 1;
    const bool up = THREE_D && (z + 1 < nz || FN.hi != nullptr);
    if (with_prior) {
      if (THREE_D) {
        commit_plane(s1);  // plane z+1 (zeros past an absent halo; unused then)
        fetch_plane(z + 2);
      } else {
        commit_plane(0);
        if (z + 1 < nz) fetch_plane(z + 1);
      }
    }
    float fnv = n_fn;
    const float kfn = n_kfn, rs = n_rs, fv = n_f, kf = n_kf;
    fetch_ops(z + 1);
    __syncthreads();
    if (inside) {
      if (with_prior) fnv = xs[s0][ty + 1][tx + 1];
      // fp32 products (one rounding, like the fp32 operands), fp64 running sums
      if (Kfn) fid += (double)(fnv * fmaf(0.5f, kfn, -rs));
      if (f && Kfn) dfid += (double)((fnv - fv) * (fmaf(0.5f, kfn + kf, 0.f) - rs));
      if (with_prior) {
        const float xv = fnv;
        // half stencil in the plane: (0,0,1), (0,1,-1), (0,1,0), (0,1,1) as two pairs
        float2 acc = mk(0.f, 0.f);
        {
          const float2 g0 = rho2<P2>(mk(xv - xs[s0][ty + 1][tx + 2], xv - xs[s0][ty + 2][tx]), pc);
          acc = pfma(mk(ipw.w8[5], ipw.w8[6]), g0, acc);
          const float2 g1 =
              rho2<P2>(mk(xv - xs[s0][ty + 2][tx + 1], xv - xs[s0][ty + 2][tx + 2]), pc);
          acc = pfma(mk(ipw.w8[7], ipw.w8[8]), g1, acc);
        }
        if (up) {  // dz = 1: all nine (dy, dx): four pairs and one single (paired with a dummy)
#pragma unroll
          for (int i = 0; i < 5; ++i) {
            const int j0 = 2 * i, j1 = 2 * i + 1 < 9 ? 2 * i + 1 : 8;
            const float2 g = rho2<P2>(mk(xv - xs[s1][ty + j0 / 3][tx + j0 % 3],
                                         xv - xs[s1][ty + j1 / 3][tx + j1 % 3]), pc);
            acc = pfma(mk(ipw.wz[j0], 2 * i + 1 < 9 ? ipw.wz[j1] : 0.f), g, acc);
          }
        }
        e_acc += (double)((acc.x + acc.y) * pc.inv_psp);
      }
    }
    __syncthreads();
  }
  const int b = blockIdx.y * gridDim.x + blockIdx.x;
  const double r0 = block_sum_d<TX * TY>(e_acc, red);
  const double r1 = block_sum_d<TX * TY>(fid, red);
  const double r2 = block_sum_d<TX * TY>(dfid, red);
  if (threadIdx.x == 0) {
    partial[3 * b] = r0;
    partial[3 * b + 1] = r1;
    partial[3 * b + 2] = r2;
  }
}

// out[j] = sum_b partial[b*nv + j]  (one block, fixed order: deterministic)
__global__ void __launch_bounds__(1024)
k_sum_partials(const double* __restrict__ partial, int nblocks, int nv, double* __restrict__ out) {
  __shared__ double red[32];
  for (int j = 0; j < nv; ++j) {
    double s = 0.0;
    for (int b = threadIdx.x; b < nblocks; b += blockDim.x) s += partial[(long long)b * nv + j];
    const double r = block_sum_d<1024>(s, red);
    if (threadIdx.x == 0) out[j] = r;
  }
}

// out_j = sum_b partial[b*nv + j] for the non-null out_j (j < 4); skipped entirely
// when only_if points at 0.0 (the conditional K4 after a restart decision)
__global__ void __launch_bounds__(1024)
k_sum_partials_to(const double* __restrict__ partial, int nblocks, int nv, double* o0,
                  double* o1, double* o2, double* o3, const double* __restrict__ only_if) {
  if (only_if && *only_if == 0.0) return;
  __shared__ double red[32];
  double* outs[4] = {o0, o1, o2, o3};
  for (int j = 0; j < nv; ++j) {
    double s = 0.0;
    for (int b = threadIdx.x; b < nblocks; b += blockDim.x) s += partial[(long long)b * nv + j];
    const double r = block_sum_d<1024>(s, red);
    if (threadIdx.x == 0 && outs[j]) *outs[j] = r;
  }
}

// ============================================================ K5, tiled (3-D, with the prior)
// Same sums as k_energy_fid on the SymTile geometry of K4: a 32 x (8 RY) tile,
// RY voxels per thread, the 13 half-stencil cliques of each voxel evaluated
// two at a time (13 RY is even for RY = 2, so no lane idles), plane steps
// unrolled by two so the ring slots are compile-time shared-memory offsets.
template <int RY, bool P2, bool EDGE>
__device__ __forceinline__ void energy_tile(const Planes& FN, const float* __restrict__ f,
                                            const float* __restrict__ Kfn,
                                            const float* __restrict__ Kf,
                                            const float* __restrict__ rstar,
                                            double* __restrict__ partial, int nz, int h, int w,
                                            const PriorConsts& pc, float* xsf, double* red) {
  using S = SymTile<RY>;
  constexpr int CELLS = S::CELLS, NT = S::NT;
  const int tx = threadIdx.x % TX, ty = threadIdx.x / TX;
  const int gx0 = blockIdx.y * S::H, gy0 = blockIdx.x * S::W;
  const int iy = gy0 + tx;
  const long long nn = (long long)h * w;
  const int me0 = (ty + 1) * S::RW + tx + 1;
  bool inside[RY];
  int vo[RY], nbits[RY];
#pragma unroll
  for (int r = 0; r < RY; ++r) {
    const int ix = gx0 + ty + TY * r;
    inside[r] = !EDGE || (ix < h && iy < w);
    vo[r] = ix * w + iy;
    nbits[r] = (ix > 0) | (ix + 1 < h) << 1 | (iy > 0) << 2 | (iy + 1 < w) << 3 | inside[r] << 4;
  }
  int coff[S::SLOTS];
#pragma unroll
  for (int m = 0; m < S::SLOTS; ++m) {
    const int e = threadIdx.x + m * NT;
    const int ly = e / S::RW, lx = e - ly * S::RW;
    const int gx = gx0 + ly - 1, gy = gy0 + lx - 1;
    coff[m] = (e < CELLS && gx >= 0 && gx < h && gy >= 0 && gy < w) ? gx * w + gy : -1;
  }
  const bool last_ok = CELLS % NT == 0 || threadIdx.x + (S::SLOTS - 1) * NT < CELLS;
  auto wgt = [&](int r, int k) -> float {  // clique (p, p + o_k)
    const float wc = pc.w[S::cls(k)];
    if constexpr (!EDGE) {
      return wc;
    } else {
      const int ddy = S::dy(k), ddx = S::dx(k);
      const int need = 16 | (ddy < 0 ? 1 : ddy > 0 ? 2 : 0) | (ddx < 0 ? 4 : ddx > 0 ? 8 : 0);
      return (nbits[r] & need) == need ? wc : 0.f;
    }
  };
  float hv[S::SLOTS];
  auto fetch_plane = [&](int zz) {
    const float* pf = FN.at(zz, nz, nn);
    const bool ok = pf != nullptr && zz <= nz;
#pragma unroll
    for (int m = 0; m < S::SLOTS; ++m) hv[m] = ok && coff[m] >= 0 ? __ldg(pf + coff[m]) : 0.f;
  };
  auto fetch_ops = [&](int zz, float (&o)[4][RY]) {
    if (zz >= nz) return;
    const long long base = zz * nn;
#pragma unroll
    for (int r = 0; r < RY; ++r) {
      const bool in = inside[r];
      o[0][r] = Kfn && in ? __ldg(Kfn + base + vo[r]) : 0.f;
      o[1][r] = rstar && in ? __ldg(rstar + base + vo[r]) : 0.f;
      o[2][r] = f && Kfn && in ? __ldg(f + base + vo[r]) : 0.f;
      o[3][r] = f && Kfn && in ? __ldg(Kf + base + vo[r]) : 0.f;
    }
  };
  auto commit = [&](int slot) {
    float* xw = xsf + slot * CELLS + threadIdx.x;
#pragma unroll
    for (int m = 0; m < S::SLOTS; ++m)
      if (m + 1 < S::SLOTS || last_ok) xw[m * NT] = hv[m];
  };
  double e_acc = 0.0, fid = 0.0, dfid = 0.0;
  float opA[4][RY], opB[4][RY];
#pragma unroll
  for (int r = 0; r < RY; ++r)
#pragma unroll
    for (int j = 0; j < 4; ++j) opA[j][r] = opB[j][r] = 0.f;

  auto step = [&](auto s0c, int z, float (&cur)[4][RY], float (&nxt)[4][RY]) {
    constexpr int S0 = decltype(s0c)::value, S1 = S0 ^ 1;
    commit(S1);  // plane z+1 (zeros past an absent halo)
    fetch_plane(z + 2);
    fetch_ops(z + 1, nxt);
    __syncthreads();
    const float* xa = xsf + S0 * CELLS;
    const float* xb = xsf + S1 * CELLS;
    const float up = (z + 1 < nz || FN.hi != nullptr) ? 1.f : 0.f;
    float xv[RY], acc[RY];
#pragma unroll
    for (int r = 0; r < RY; ++r) {
      xv[r] = xa[me0 + r * TY * S::RW];
      acc[r] = 0.f;
    }
    constexpr int NOWN = 13 * RY, NEVAL = (NOWN + 1) & ~1;
    float2 x2 = mk(0.f, 0.f), n2 = mk(0.f, 0.f);
#pragma unroll
    for (int e = 0; e < NEVAL; ++e) {
      float xs = 0.f, xn = 0.f;
      if (e < NOWN) {
        const int r = e / 13, k = e % 13;
        xs = xv[r];
        xn = (k < 4 ? xa : xb)[me0 + r * TY * S::RW + S::off(k)];
      }
      if (e & 1) {
        x2.y = xs;
        n2.y = xn;
        const bool xr = TF_XRCP_K5 > 0 && (e / 2) % TF_XRCP_K5 == TF_XRCP_K5 - 1;
        const float2 g = xr ? rho2<P2, true>(csub(x2, n2), pc) : rho2<P2>(csub(x2, n2), pc);
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          const int ee = e - 1 + h2;
          if (ee < NOWN) {
            const int r = ee / 13, k = ee % 13;
            acc[r] = fmaf(k < 4 ? wgt(r, k) : wgt(r, k) * up, h2 ? g.y : g.x, acc[r]);
          }
        }
      } else {
        x2.x = xs;
        n2.x = xn;
      }
    }
#pragma unroll
    for (int r = 0; r < RY; ++r) {
      if (!inside[r]) continue;
      const float fnv = xv[r], kfn = cur[0][r], rs = cur[1][r], fv = cur[2][r], kf = cur[3][r];
      // fp32 products (one rounding, like the fp32 operands), fp64 running sums
      if (Kfn) fid += (double)(fnv * fmaf(0.5f, kfn, -rs));
      if (f && Kfn) dfid += (double)((fnv - fv) * (fmaf(0.5f, kfn + kf, 0.f) - rs));
      e_acc += (double)(acc[r] * pc.inv_psp);
    }
    __syncthreads();  // slot S0 is overwritten by the next step's commit
  };
  using I0 = std::integral_constant<int, 0>;
  using I1 = std::integral_constant<int, 1>;
  fetch_plane(0);
  commit(0);
  fetch_plane(1);
  fetch_ops(0, opA);
  for (int z = 0; z < nz; z += 2) {
    step(I0{}, z, opA, opB);
    if (z + 1 < nz) step(I1{}, z + 1, opB, opA);
  }
  const int b = blockIdx.y * gridDim.x + blockIdx.x;
  const double r0 = block_sum_d<NT>(e_acc, red);
  const double r1 = block_sum_d<NT>(fid, red);
  const double r2 = block_sum_d<NT>(dfid, red);
  if (threadIdx.x == 0) {
    partial[3 * b] = r0;
    partial[3 * b + 1] = r1;
    partial[3 * b + 2] = r2;
  }
}

template <bool P2>
__global__ void __launch_bounds__(TX* TY, TF_K4_MINB)
k_energy_fid_t(Planes FN, const float* __restrict__ f, const float* __restrict__ Kfn,
               const float* __restrict__ Kf, const float* __restrict__ rstar,
               double* __restrict__ partial, int nz, int h, int w, PriorConsts pc) {
  using S = SymTile<K4_RY>;
  __shared__ float xs[2 * S::CELLS];
  __shared__ double red[TX * TY / 32];
  const bool interior = blockIdx.y * S::H >= 1 && (blockIdx.y + 1) * S::H + 1 <= h &&
                        blockIdx.x * S::W >= 1 && (blockIdx.x + 1) * S::W + 1 <= w;
  if (interior)
    energy_tile<K4_RY, P2, false>(FN, f, Kfn, Kf, rstar, partial, nz, h, w, pc, xs, red);
  else
    energy_tile<K4_RY, P2, true>(FN, f, Kfn, Kf, rstar, partial, nz, h, w, pc, xs, red);
}

// ============================================================ solver decision (device)
// One iteration's restart / momentum / stop decision (solver.py:147-180), the
// same fp64 arithmetic as the host loop, so the iteration loop never waits on
// the host.  vals = {E(f_new), sum grad^2, fidelity increment};
// state = {obj, fid, prior, t, c}; rec = {obj_new, fid_new, prior_new,
// sum grad^2, restarted, converged, finite, dobj}.
__global__ void k_solver_decide(const double* __restrict__ vals, double* __restrict__ state,
                                float* __restrict__ c_out, double* __restrict__ rec, double lam,
                                int with_prior, int restart, double tol) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const double e_new = with_prior ? vals[0] : 0.0, gsq = vals[1], dfid = vals[2];
  const double obj = state[0], fid = state[1], prior = state[2], t = state[3];
  // explicit roundings (no FMA contraction): the host's Python float arithmetic
  const double dobj = __dadd_rn(dfid, __dmul_rn(lam, __dadd_rn(e_new, -prior)));
  const double obj_new = __dadd_rn(obj, dobj);
  const bool restarted = restart && dobj > 0.0;
  const double t_next =
      restarted ? 1.0 : __dadd_rn(1.0, sqrt(__dadd_rn(1.0, __dmul_rn(__dmul_rn(4.0, t), t)))) / 2.0;
  const double c_next = restarted ? 0.0 : (t - 1.0) / t_next;
  const bool converged = !restarted && fabs(dobj) <= tol * fabs(obj);
  rec[0] = obj_new;
  rec[1] = __dadd_rn(fid, dfid);
  rec[2] = e_new;
  rec[3] = gsq;
  rec[4] = restarted ? 1.0 : 0.0;
  rec[5] = converged ? 1.0 : 0.0;
  rec[6] = isfinite(obj_new) ? 1.0 : 0.0;
  rec[7] = dobj;
  state[0] = obj_new;
  state[1] = __dadd_rn(fid, dfid);
  state[2] = e_new;
  state[3] = t_next;
  state[4] = c_next;
  *c_out = (float)c_next;
}

int solver_decide(const double* vals, double* state, float* c_out, double* rec, double lam,
                  int with_prior, int restart, double tol, cudaStream_t st) {
  k_solver_decide<<<1, 32, 0, st>>>(vals, state, c_out, rec, lam, with_prior, restart, tol);
  return check_launch("k_solver_decide");
}

// ============================================================ host side
static PriorConsts make_consts(double sigma, double p, double q, double T, const double* w3) {
  PriorConsts pc;
  const double sp = pow(sigma, p);
  pc.inv_sp = (float)(1.0 / sp);
  pc.inv_psp = (float)(1.0 / (p * sp));
  pc.c0 = (float)((p - q) * log2(T * sigma));
  pc.pq = (float)(p - q);
  pc.qp = (float)(q / p);
  pc.p = (float)p;
  pc.pm1 = (float)(p - 1.0);
  pc.w[0] = 0.f;
  pc.w[1] = (float)w3[0];
  pc.w[2] = (float)w3[1];
  pc.w[3] = (float)w3[2];
  return pc;
}

static dim3 tile_grid(int h, int w) { return dim3((w + TX - 1) / TX, (h + TY - 1) / TY); }

long long prior_partials(int h, int w) {
  const dim3 g = tile_grid(h, w);
  return (long long)g.x * g.y;
}

int prior_update(const float* f, const float* f_lo, const float* f_hi, const float* fp,
                 const float* fp_lo, const float* fp_hi, const float* Kf, const float* Kfp,
                 const float* rstar, float* f_new, int nz, int h, int w_, float c, float lam, float inv_L,
                 int nonneg, int write_grad, int three_d, double sigma, double p, double q,
                 double T, const double* w, double* partial, double* out_gsq, const float* c_dev,
                 cudaStream_t st, const double* only_if) {
  if (only_if && !three_d) return fail_arg("conditional update is 3-D only");
  const PriorConsts pc = make_consts(sigma, p, q, T, w);
  const dim3 grid = tile_grid(h, w_);
  const Planes F{f, f_lo, f_hi}, FP{fp, fp_lo, fp_hi};
  const bool p2 = p == 2.0;
#define TF_K4(TD, P2V, NN)                                                                    \
  k_prior_update<TD, P2V, NN><<<grid, TX * TY, 0, st>>>(F, FP, Kf, Kfp, rstar, f_new, partial, \
                                                         nz, h, w_, c, lam, inv_L, write_grad, pc, c_dev)
  const dim3 sgrid = sym_grid(h, w_);
  const size_t ssmem = sym_smem_bytes();
#define TF_K4S(P2V, NN)                                                                      \
  do {                                                                                       \
    TF_TRY(prep_kernel(k_prior_update_sym<P2V, NN>, ssmem));                                 \
    k_prior_update_sym<P2V, NN><<<sgrid, TX * TY, ssmem, st>>>(                              \
        F, FP, Kf, Kfp, rstar, f_new, partial, nz, h, w_, c, lam, inv_L, write_grad, pc, c_dev, \
        only_if);                                                                            \
  } while (0)
  // 3-D: the symmetric-clique tile kernel; 2-D (single slices): the direct stencil
  if (three_d) {
    if (p2) { if (nonneg) TF_K4S(true, true); else TF_K4S(true, false); }
    else { if (nonneg) TF_K4S(false, true); else TF_K4S(false, false); }
  } else {
    if (p2) { if (nonneg) TF_K4(false, true, true); else TF_K4(false, true, false); }
    else { if (nonneg) TF_K4(false, false, true); else TF_K4(false, false, false); }
  }
#undef TF_K4
#undef TF_K4S
  TF_TRY(check_launch("k_prior_update"));
  const int nparts = three_d ? (int)(sgrid.x * sgrid.y) : (int)(grid.x * grid.y);
  k_sum_partials_to<<<1, 1024, 0, st>>>(partial, nparts, 1, out_gsq, nullptr, nullptr, nullptr,
                                        only_if);
  return check_launch("k_sum_partials");
}

int prior_energy_update(const float* f, const float* f_lo, const float* f_hi, const float* fp,
                        const float* fp_lo, const float* fp_hi, const float* Kf, const float* Kfp,
                        const float* rstar, float* f_new, int nz, int h, int w_, const double* state,
                        float lam, float inv_L, int nonneg, int with_prior, double sigma, double p,
                        double q, double T, const double* w, double* partial, double* out_e,
                        double* out_fid, double* out_dfid, double* out_gsq, cudaStream_t st) {
  const PriorConsts pc = make_consts(sigma, p, q, T, w);
  const Planes F{f, f_lo, f_hi}, FP{fp, fp_lo, fp_hi};
  const dim3 sgrid = sym_grid(h, w_);
  const size_t smem = sym_smem_bytes(true);
  // waves of tile columns at 2 vs 3 CTAs per SM (a 3-CTA wave is ~1.47x longer)
  const long long tiles = (long long)sgrid.x * sgrid.y, sms = num_sms();
  const bool mb3 = TF_K45_MB3 && 147 * ((tiles + 3 * sms - 1) / (3 * sms)) <
                                      100 * ((tiles + 2 * sms - 1) / (2 * sms));
#define TF_K45(P2V, NN)                                                                        \
  do {                                                                                         \
    auto kern = mb3 ? k_prior_energy_update<P2V, NN, 3> : k_prior_energy_update<P2V, NN, 2>;   \
    TF_TRY(prep_kernel(kern, smem));                                                           \
    kern<<<sgrid, TX * TY, smem, st>>>(F, FP, Kf, Kfp, rstar, f_new, partial, nz, h, w_, lam,  \
                                       inv_L, with_prior, pc, state);                          \
  } while (0)
  if (p == 2.0) { if (nonneg) TF_K45(true, true); else TF_K45(true, false); }
  else { if (nonneg) TF_K45(false, true); else TF_K45(false, false); }
#undef TF_K45
  TF_TRY(check_launch("k_prior_energy_update"));
  k_sum_partials_to<<<1, 1024, 0, st>>>(partial, (int)(sgrid.x * sgrid.y), 4, out_e, out_fid,
                                        out_dfid, out_gsq, nullptr);
  return check_launch("k_sum_partials");
}

int energy_fid(const float* fn, const float* fn_hi, const float* f, const float* Kfn,
               const float* Kf, const float* rstar, int nz, int h, int w_, int with_prior,
               int three_d, double sigma, double p, double q, double T, const double* w,
               double* partial, double* out3, cudaStream_t st) {
  const PriorConsts pc = make_consts(sigma, p, q, T, w);
  const dim3 grid = tile_grid(h, w_);
  const Planes FN{fn, nullptr, fn_hi};
  const bool p2 = p == 2.0;
  if (three_d && with_prior) {  // 3-D energy on K4's tile geometry
    const dim3 sg = sym_grid(h, w_);
    if (p2) k_energy_fid_t<true><<<sg, TX * TY, 0, st>>>(FN, f, Kfn, Kf, rstar, partial, nz, h, w_, pc);
    else k_energy_fid_t<false><<<sg, TX * TY, 0, st>>>(FN, f, Kfn, Kf, rstar, partial, nz, h, w_, pc);
    TF_TRY(check_launch("k_energy_fid_t"));
    k_sum_partials<<<1, 1024, 0, st>>>(partial, (int)(sg.x * sg.y), 3, out3);
    return check_launch("k_sum_partials");
  }
  if (three_d) {
    if (p2) k_energy_fid<true, true><<<grid, TX * TY, 0, st>>>(FN, f, Kfn, Kf, rstar, partial, nz, h, w_, with_prior, pc);
    else k_energy_fid<true, false><<<grid, TX * TY, 0, st>>>(FN, f, Kfn, Kf, rstar, partial, nz, h, w_, with_prior, pc);
  } else {
    if (p2) k_energy_fid<false, true><<<grid, TX * TY, 0, st>>>(FN, f, Kfn, Kf, rstar, partial, nz, h, w_, with_prior, pc);
    else k_energy_fid<false, false><<<grid, TX * TY, 0, st>>>(FN, f, Kfn, Kf, rstar, partial, nz, h, w_, with_prior, pc);
  }
  TF_TRY(check_launch("k_energy_fid"));
  k_sum_partials<<<1, 1024, 0, st>>>(partial, (int)(grid.x * grid.y), 3, out3);
  return check_launch("k_sum_partials");
}

}  // namespace tf
