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
#include "tf_common.cuh"

namespace tf {

struct PriorConsts {
  float inv_sp;      // 1 / sigma^p
  float inv_psp;     // 1 / (p sigma^p)
  float log2_ts;     // log2(T sigma)
  float pq;          // p - q
  float qp;          // q / p
  float p;           // p
  float w[4];        // stencil weights by number of nonzero offset components (1, 2, 3)
};

constexpr int TX = 32, TY = 8;

// v = (|d| / (T sigma))^(p-q), via the SFU (lg2/ex2); v = 0 at d = 0
__device__ __forceinline__ float qg_v(float ad, const PriorConsts& pc) {
  return exp2f(pc.pq * (__log2f(ad) - pc.log2_ts));
}

// rho'(d) = sign(d) |d|^(p-1) / sigma^p * (1 + (q/p) v) / (1 + v)^2  (qggmrf.py:124-130)
template <bool P2>
__device__ __forceinline__ float rho_prime(float d, const PriorConsts& pc) {
  const float ad = fabsf(d);
  const float v = qg_v(ad, pc);
  const float onev = 1.f + v;
  const float shape = __fdividef(fmaf(pc.qp, v, 1.f), onev * onev);
  float mag;
  if constexpr (P2) mag = d;  // sign(d) |d|
  else mag = copysignf(exp2f((pc.p - 1.f) * __log2f(ad)), d);
  return mag * pc.inv_sp * shape;
}

// rho(d) = |d|^p / (p sigma^p) / (1 + v)  (qggmrf.py:117-121)
template <bool P2>
__device__ __forceinline__ float rho(float d, const PriorConsts& pc) {
  const float ad = fabsf(d);
  const float v = qg_v(ad, pc);
  float mag;
  if constexpr (P2) mag = d * d;
  else mag = exp2f(pc.p * __log2f(ad));
  return __fdividef(mag * pc.inv_psp, 1.f + v);
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

// ============================================================ K4
// grad = K y - R*g + lam * grad_prior(y)   (Kf/Kfp/rstar may be null -> 0)
// write_grad == 0: out = y - grad / L  [clamped at 0 if NONNEG]   (the update)
// write_grad == 1: out = grad                                     (prior_grad API)
// partial[block] = sum grad^2 over the block's voxels (fp64)
template <bool THREE_D, bool P2, bool NONNEG>
__global__ void __launch_bounds__(TX* TY)
k_prior_update(Planes F, Planes FP, const float* __restrict__ Kf, const float* __restrict__ Kfp,
               const float* __restrict__ rstar, float* __restrict__ f_new,
               double* __restrict__ partial, int nz, int h, int w, float c, float lam,
               float inv_L, int write_grad, PriorConsts pc) {
  __shared__ float ys[3][TY + 2][TX + 2];
  __shared__ double red[TX * TY / 32];
  const int tx = threadIdx.x % TX, ty = threadIdx.x / TX;
  const int iy = blockIdx.x * TX + tx;  // contiguous axis
  const int ix = blockIdx.y * TY + ty;
  const long long nn = (long long)h * w;
  const bool inside = ix < h && iy < w;

  // y on plane zz into ring slot s (0 outside the grid or on an invalid plane)
  auto load_plane = [&](int zz, int s) {
    const float* pf = F.at(zz, nz, nn);
    const float* pp = FP.at(zz, nz, nn);
    for (int e = threadIdx.x; e < (TY + 2) * (TX + 2); e += TX * TY) {
      const int ly = e / (TX + 2), lx = e - ly * (TX + 2);
      const int gx = blockIdx.y * TY + ly - 1, gy = blockIdx.x * TX + lx - 1;
      float val = 0.f;
      if (pf && gx >= 0 && gx < h && gy >= 0 && gy < w) {
        const long long o = (long long)gx * w + gy;
        const float a = __ldg(pf + o);
        const float b = __ldg(pp + o);
        val = fmaf(c, a - b, a);
      }
      ys[s][ly][lx] = val;
    }
  };

  // in-plane validity of the 8 neighbours (dy, dx) of this voxel
  const bool okm_x = ix > 0, okp_x = ix + 1 < h, okm_y = iy > 0, okp_y = iy + 1 < w;
  double gsq = 0.0;
  if (THREE_D) {
    load_plane(-1, 2);
    load_plane(0, 0);
  }
  for (int z = 0; z < nz; ++z) {
    const int s0 = THREE_D ? z % 3 : 0, sp = (z + 1) % 3, sm = (z + 2) % 3;  // z, z+1, z-1
    if (THREE_D) load_plane(z + 1, sp);
    else load_plane(z, 0);  // 8-neighbour stencil: slices are independent
    __syncthreads();
    if (inside) {
      const float yv = ys[s0][ty + 1][tx + 1];
      float acc = 0.f;
      // in-plane neighbours (dz = 0)
#pragma unroll
      for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
        for (int dx = -1; dx <= 1; ++dx) {
          if (dy == 0 && dx == 0) continue;
          const bool ok = (dy < 0 ? okm_x : dy > 0 ? okp_x : true) &&
                          (dx < 0 ? okm_y : dx > 0 ? okp_y : true);
          const int k = (dy != 0) + (dx != 0);
          const float wgt = THREE_D ? pc.w[k] : pc.w[k];
          if (ok) acc = fmaf(wgt, rho_prime<P2>(yv - ys[s0][ty + 1 + dy][tx + 1 + dx], pc), acc);
        }
      if (THREE_D) {
        const bool okz[2] = {z > 0 || FP.lo != nullptr, z + 1 < nz || FP.hi != nullptr};
#pragma unroll
        for (int side = 0; side < 2; ++side) {
          if (!okz[side]) continue;
          const int sl = side ? sp : sm;
#pragma unroll
          for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
            for (int dx = -1; dx <= 1; ++dx) {
              const bool ok = (dy < 0 ? okm_x : dy > 0 ? okp_x : true) &&
                              (dx < 0 ? okm_y : dx > 0 ? okp_y : true);
              const int k = 1 + (dy != 0) + (dx != 0);
              if (ok)
                acc = fmaf(pc.w[k], rho_prime<P2>(yv - ys[sl][ty + 1 + dy][tx + 1 + dx], pc), acc);
            }
        }
      }
      const long long o = z * nn + (long long)ix * w + iy;
      float ky = 0.f;
      if (Kf) {
        const float kfv = __ldg(Kf + o), kpv = __ldg(Kfp + o);
        ky = fmaf(c, kfv - kpv, kfv);
      }
      const float grad = fmaf(lam, acc, ky - (rstar ? __ldg(rstar + o) : 0.f));
      if (write_grad) {
        f_new[o] = grad;
      } else {
        float fn = fmaf(-grad, inv_L, yv);
        if (NONNEG) fn = fmaxf(fn, 0.f);
        f_new[o] = fn;
      }
      gsq += (double)grad * (double)grad;
    }
    __syncthreads();
  }
  const double r = block_sum_d<TX * TY>(gsq, red);
  if (threadIdx.x == 0) partial[blockIdx.y * gridDim.x + blockIdx.x] = r;
}

// ============================================================ K5
// partial[block*3 + {0,1,2}] = { E(f_new) (half stencil + halo_hi pairs),
//   <f_new, K f_new / 2 - R*g>,  <f_new - f, (K f_new + K f)/2 - R*g> (0 if f null) }
template <bool THREE_D, bool P2>
__global__ void __launch_bounds__(TX* TY)
k_energy_fid(Planes FN, const float* __restrict__ f, const float* __restrict__ Kfn,
             const float* __restrict__ Kf, const float* __restrict__ rstar,
             double* __restrict__ partial, int nz, int h, int w, int with_prior, PriorConsts pc) {
  __shared__ float xs[2][TY + 2][TX + 2];
  __shared__ double red[TX * TY / 32];
  const int tx = threadIdx.x % TX, ty = threadIdx.x / TX;
  const int iy = blockIdx.x * TX + tx;
  const int ix = blockIdx.y * TY + ty;
  const long long nn = (long long)h * w;
  const bool inside = ix < h && iy < w;
  auto load_plane = [&](int zz, int s) {
    const float* pf = FN.at(zz, nz, nn);
    for (int e = threadIdx.x; e < (TY + 2) * (TX + 2); e += TX * TY) {
      const int ly = e / (TX + 2), lx = e - ly * (TX + 2);
      const int gx = blockIdx.y * TY + ly - 1, gy = blockIdx.x * TX + lx - 1;
      float val = 0.f;
      if (pf && gx >= 0 && gx < h && gy >= 0 && gy < w) val = __ldg(pf + (long long)gx * w + gy);
      xs[s][ly][lx] = val;
    }
  };
  const bool okp_x = ix + 1 < h, okm_y = iy > 0, okp_y = iy + 1 < w, okm_x = ix > 0;
  double e_acc = 0.0, fid = 0.0, dfid = 0.0;
  if (with_prior && THREE_D) load_plane(0, 0);
  for (int z = 0; z < nz; ++z) {
    const int s0 = THREE_D ? (z & 1) : 0, s1 = (z + 1) & 1;
    const bool up = THREE_D && (z + 1 < nz || FN.hi != nullptr);
    if (with_prior && up) load_plane(z + 1, s1);
    if (with_prior && !THREE_D) load_plane(z, 0);
    __syncthreads();
    if (inside) {
      const long long o = z * nn + (long long)ix * w + iy;
      const float fnv = __ldg(FN.main + o);
      const float kfn = Kfn ? __ldg(Kfn + o) : 0.f, rs = rstar ? __ldg(rstar + o) : 0.f;
      if (Kfn) fid += (double)fnv * (double)fmaf(0.5f, kfn, -rs);
      if (f && Kfn) {
        const float fv = __ldg(f + o), kf = __ldg(Kf + o);
        dfid += (double)(fnv - fv) * (double)(fmaf(0.5f, kfn + kf, 0.f) - rs);
      }
      if (with_prior) {
        const float xv = xs[s0][ty + 1][tx + 1];
        float acc = 0.f;
        // dz = 0: (0, 0, 1), (0, 1, -1), (0, 1, 0), (0, 1, 1)
        if (okp_y) acc = fmaf(pc.w[1], rho<P2>(xv - xs[s0][ty + 1][tx + 2], pc), acc);
        if (okp_x) {
          if (okm_y) acc = fmaf(pc.w[2], rho<P2>(xv - xs[s0][ty + 2][tx], pc), acc);
          acc = fmaf(pc.w[1], rho<P2>(xv - xs[s0][ty + 2][tx + 1], pc), acc);
          if (okp_y) acc = fmaf(pc.w[2], rho<P2>(xv - xs[s0][ty + 2][tx + 2], pc), acc);
        }
        if (up) {  // dz = 1: all nine (dy, dx)
#pragma unroll
          for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
            for (int dx = -1; dx <= 1; ++dx) {
              const bool ok = (dy < 0 ? okm_x : dy > 0 ? okp_x : true) &&
                              (dx < 0 ? okm_y : dx > 0 ? okp_y : true);
              const int k = 1 + (dy != 0) + (dx != 0);
              if (ok) acc = fmaf(pc.w[k], rho<P2>(xv - xs[s1][ty + 1 + dy][tx + 1 + dx], pc), acc);
            }
        }
        e_acc += (double)acc;
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

// ============================================================ host side
static PriorConsts make_consts(double sigma, double p, double q, double T, const double* w3) {
  PriorConsts pc;
  const double sp = pow(sigma, p);
  pc.inv_sp = (float)(1.0 / sp);
  pc.inv_psp = (float)(1.0 / (p * sp));
  pc.log2_ts = (float)log2(T * sigma);
  pc.pq = (float)(p - q);
  pc.qp = (float)(q / p);
  pc.p = (float)p;
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
                 double T, const double* w, double* partial, double* out_gsq, cudaStream_t st) {
  const PriorConsts pc = make_consts(sigma, p, q, T, w);
  const dim3 grid = tile_grid(h, w_);
  const Planes F{f, f_lo, f_hi}, FP{fp, fp_lo, fp_hi};
  const bool p2 = p == 2.0;
#define TF_K4(TD, P2V, NN)                                                                    \
  k_prior_update<TD, P2V, NN><<<grid, TX * TY, 0, st>>>(F, FP, Kf, Kfp, rstar, f_new, partial, \
                                                         nz, h, w_, c, lam, inv_L, write_grad, pc)
  if (three_d) {
    if (p2) { if (nonneg) TF_K4(true, true, true); else TF_K4(true, true, false); }
    else { if (nonneg) TF_K4(true, false, true); else TF_K4(true, false, false); }
  } else {
    if (p2) { if (nonneg) TF_K4(false, true, true); else TF_K4(false, true, false); }
    else { if (nonneg) TF_K4(false, false, true); else TF_K4(false, false, false); }
  }
#undef TF_K4
  TF_TRY(check_launch("k_prior_update"));
  k_sum_partials<<<1, 1024, 0, st>>>(partial, (int)(grid.x * grid.y), 1, out_gsq);
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
