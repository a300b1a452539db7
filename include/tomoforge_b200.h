/*
 * tomoforge_b200.h -- C-ABI of libtomoforge_b200.so, the B200 (sm_100a)
 * implementation of the Fourier-domain MBIR iterative core.
 *
 * Conventions (all entry points):
 *   - array arguments are DEVICE pointers owned by the caller; fp32 unless
 *     stated; volumes are row-major [slice][x][y] (reference layout data[ix, iy],
 *     tomoforge/geometry.py:1-13);
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream);
 *   - return 0 on success, -1 bad argument/shape, -2 CUDA error, -3 unsupported;
 *     tf_last_error() describes the last failure on the calling thread;
 *   - no global state except the per-device twiddle table built by tf_init();
 *     calls on distinct buffers/streams are re-entrant.
 *
 * The reference interface each entry point replaces is cited (paths relative to
 * the reference package pkg/src/tomoforge/).
 */
#ifndef TOMOFORGE_B200_H
#define TOMOFORGE_B200_H

#ifdef __cplusplus
extern "C" {
#endif

const char* tf_last_error(void);
int tf_version(void);

/* Build the per-device twiddle table on the current device (idempotent). */
int tf_init(void);

/* FFT side M used for an N x N source grid: the smallest M >= 2N-1 among the
 * powers of two and 5 * 2^k (k = 8, 9, 10: a radix-5 step, e.g. N = 2560 -> 5120).
 * Replaces padded_side_for (toeplitz.py:53-60), which picks the smallest ODD
 * 7-smooth side; the even grid is exact for the re-embedded lag kernels
 * (DESIGN.md §3).  Returns M, or -1 for unsupported N (> 4096). */
int tf_fft_side(int n);

/* Bytes of workspace tf_toeplitz_apply needs to process `nslices` slices in one
 * pass (it chunks over slices when given less, down to one slice). */
long long tf_toeplitz_workspace_bytes(int n, int M, long long nslices);
long long tf_psf_workspace_bytes(int M);

/* PSF spectra of the normal operator for an N x N grid.
 * Replaces compute_psf / build_psf (toeplitz.py:85-131).
 *   d_cossin : [n_angles][2] fp64 (cos theta, sin theta)
 *   nd       : detector bins (radial samples per angle); even nd enables the
 *              Nyquist flip term (toeplitz.py:106-114)
 *   d_PQ     : out [M/2+1][M] float2  ((A+Re B)/M^2, (A-Re B)/M^2)
 *   d_Bi     : out [M/2+1][M] float   Im B / M^2 (zeros for odd nd)
 *   d_ws     : tf_psf_workspace_bytes(M) bytes of scratch */
int tf_psf_build(int n, int M, int n_angles, const double* d_cossin, int nd, void* d_PQ,
                 float* d_Bi, void* d_ws, long long ws_bytes, void* stream);

/* The reference's lag kernel on its odd padded grid of side m (padded_side_for,
 * toeplitz.py:53-60): d_out [m][m] fp64 = K(d) = sum_theta sum_j cos(w_j d.e_theta)
 * (the adjoint NUFFT of unit weights, toeplitz.py:102), ifftshifted (lag d at
 * d mod m).  fft2(d_out) is PsfKernel.spectrum (toeplitz.py:63-82). */
int tf_psf_kernel(int m, int n_angles, const double* d_cossin, int nd, double* d_out,
                  void* stream);

/* out = alpha * (K x) + beta * aux over a stack of nslices N x N slices.
 * Replaces _apply_batch (toeplitz.py:134-149); with alpha=1, beta=-1, aux=R*g
 * it is fidelity_grad (toeplitz.py:233-241).  aux may be NULL.  x != out. */
int tf_toeplitz_apply(const float* d_x, float* d_out, const float* d_aux, float alpha,
                      float beta, long long nslices, int n, int M, const void* d_PQ,
                      const float* d_Bi, int has_flip, void* d_ws, long long ws_bytes,
                      void* stream);

/* Deterministic fp64 sums: d_out[0] = sum x*a, d_out[1] = sum x*b (b may be
 * NULL -> 0).  Replaces the np.sum(arr * kf), np.sum(arr * rstar) terms of
 * fidelity_loss / objective (toeplitz.py:226-230, solver.py:95-101).
 * d_ws: tf_reduce_workspace_bytes() bytes. */
long long tf_reduce_workspace_bytes(void);
int tf_dot2(const float* d_x, const float* d_a, const float* d_b, long long n, double* d_out,
            double* d_ws, void* stream);

/* ---- qGGMRF prior + momentum update (K4) and objective reductions (K5) ----
 * Volumes [nz][h][w] (w contiguous); *_lo / *_hi are optional halo planes (z = -1, z = nz) of a
 * slab (NULL: cliques across that face are dropped, qggmrf.py:142-160).
 * weights3 (HOST pointer): stencil weights for offsets with 1, 2, 3 nonzero
 * components (3-D: face, edge, corner; 2-D: face, diagonal, unused), as
 * _build_stencil (qggmrf.py:86-97).  d_ws: tf_prior_workspace_bytes(n). */
long long tf_prior_workspace_bytes(int h, int w);

/* y = f + c (f - f_prev), K y = K f + c (K f - K f_prev),
 * grad = K y - R*g + lam * sum_s b_s rho'(y_v - y_{v+s})  (prior_grad, qggmrf.py:172-189);
 * write_grad = 0: out = y - grad * inv_L (clamped at 0 if nonneg) -- solver.py:149-156;
 * write_grad = 1: out = grad.  d_Kf/d_Kfp/d_rstar may be NULL (treated as 0).
 * d_out may alias d_Kfp (each voxel's K f_prev is read before its output is
 * written; the solver keeps 4 volumes + R*g this way); no other aliasing.
 * *d_gsq = sum grad^2 (fp64). */
int tf_prior_update(const float* d_f, const float* d_f_lo, const float* d_f_hi, const float* d_fp,
                    const float* d_fp_lo, const float* d_fp_hi, const float* d_Kf,
                    const float* d_Kfp, const float* d_rstar, float* d_out, int nz, int h, int w,
                    float c, float lam, float inv_L, int nonneg, int write_grad, int three_d,
                    double sigma, double p, double q, double T, const double* weights3,
                    double* d_ws, double* d_gsq, void* stream);

/* tf_prior_update with the momentum coefficient read on the device: c = *d_c when
 * d_c is not NULL (written by tf_solver_decide), so the host does not have to wait
 * for the previous iteration's restart decision before launching the next. */
int tf_prior_update_dc(const float* d_f, const float* d_f_lo, const float* d_f_hi,
                       const float* d_fp, const float* d_fp_lo, const float* d_fp_hi,
                       const float* d_Kf, const float* d_Kfp, const float* d_rstar, float* d_out,
                       int nz, int h, int w, float c, const float* d_c, float lam, float inv_L,
                       int nonneg, int write_grad, int three_d, double sigma, double p, double q,
                       double T, const double* weights3, double* d_ws, double* d_gsq,
                       void* stream);

/* tf_prior_update_dc (write_grad = 0, 3-D) run only when *d_only_if != 0 (the
 * restart flag of tf_solver_decide's record), with c = *d_c: the solver re-runs
 * the update after a restart; otherwise the launch (and the *d_gsq write) is a
 * no-op.  The momentum argument is taken from d_c only. */
int tf_prior_update_if(const float* d_f, const float* d_f_lo, const float* d_f_hi,
                       const float* d_fp, const float* d_fp_lo, const float* d_fp_hi,
                       const float* d_Kf, const float* d_Kfp, const float* d_rstar, float* d_out,
                       int nz, int h, int w, const float* d_c, float lam, float inv_L, int nonneg,
                       double sigma, double p, double q, double T, const double* weights3,
                       double* d_ws, double* d_gsq, const double* d_only_if, void* stream);

/* K45: one pass over a 3-D slab that computes tf_energy_fid's sums for the
 * current iterate f (= d_f, previous iterate d_fp, K f = d_Kf, K f_prev = d_Kfp)
 *   *d_energy = E(f) (half stencil + pairs into d_f_hi; 0 if !with_prior),
 *   *d_fid = <f, K f / 2 - R*g>,  *d_dfid = <f - f_prev, (K f + K f_prev)/2 - R*g>
 * together with tf_prior_update_dc's update for the NEXT iterate,
 *   d_out = y - (K y - R*g + lam grad_prior(y)) inv_L,  y = f + c (f - f_prev),
 * with c the no-restart momentum (t - 1) / t', t' = (1 + sqrt(1 + 4 t^2)) / 2,
 * t = d_state[3], in tf_solver_decide's fp64 arithmetic; *d_gsq = sum grad^2.
 * (solver.py:147-180 / qggmrf.py:172-217.)  If the decision for f restarts, the
 * caller re-runs the update with tf_prior_update_if.  d_out may alias d_Kfp;
 * output pointers may be NULL (not written). */
int tf_prior_energy_update(const float* d_f, const float* d_f_lo, const float* d_f_hi,
                           const float* d_fp, const float* d_fp_lo, const float* d_fp_hi,
                           const float* d_Kf, const float* d_Kfp, const float* d_rstar,
                           float* d_out, int nz, int h, int w, const double* d_state, float lam,
                           float inv_L, int nonneg, int with_prior, double sigma, double p,
                           double q, double T, const double* weights3, double* d_ws,
                           double* d_energy, double* d_fid, double* d_dfid, double* d_gsq,
                           void* stream);

/* The restart / momentum / stop decision of one iteration, on the device
 * (tomoforge/solver.py:147-180: restart when the objective increases, momentum
 * t' = (1 + sqrt(1 + 4 t^2)) / 2, stop when |dobj| <= tol |obj| without a restart).
 * d_vals = {E(f_new), sum grad^2, fidelity increment} (fp64);
 * d_state = {obj, fid, prior, t, c} (fp64, updated in place); *d_c = next c (fp32);
 * d_rec = {obj_new, fid_new, prior_new, sum grad^2, restarted, converged, finite, dobj}. */
int tf_solver_decide(const double* d_vals, double* d_state, float* d_c, double* d_rec, double lam,
                     int with_prior, int restart, double tol, void* stream);

/* d_out3 (fp64) = { E(f_new) over the half stencil plus pairs into d_fn_hi
 *   (prior_energy, qggmrf.py:192-217; 0 if !with_prior),
 *   <f_new, K f_new / 2 - R*g>  (fidelity minus g'g/2, toeplitz.py:226-230),
 *   <f_new - f, (K f_new + K f)/2 - R*g>  (fidelity increment; 0 if d_f NULL) }. */
int tf_energy_fid(const float* d_fn, const float* d_fn_hi, const float* d_f, const float* d_Kfn,
                  const float* d_Kf, const float* d_rstar, int nz, int h, int w, int with_prior,
                  int three_d, double sigma, double p, double q, double T, const double* weights3,
                  double* d_ws, double* d_out3, void* stream);

/* ---- NUFFT back-projection / FBP (K7, K8) --------------------------------
 * Replaces radon._back_project_rows (radon.py:124-128), ramp_filter_apply
 * (radon.py:137-142), fbp (radon.py:145-160) and nufft.type1 (nufft.py:203-223).
 *
 * tf_detector_rows: one DFT of length nd (<= 8192, any factorisation) per row of
 *   d_rows [nrows][nd] fp32.  mode 0: d_out = complex64 [nrows][nd] polar
 *   samples in signed-frequency order, sample jj of row i multiplied by
 *   d_sphase[(i % n_angles) * nd + jj] (complex64), by |w_j| if ramp, and by
 *   scale.  mode 1: d_out = fp32 [nrows][nd] ramp-filtered rows (x |w|, inverse
 *   DFT, real part) times scale; d_sphase unused. */
int tf_detector_rows(const float* d_rows, long long nrows, int nd, int n_angles,
                     const void* d_sphase, int mode, int ramp, float scale, void* d_out,
                     void* stream);

/* Bytes of workspace tf_nufft_type1 needs per pass of `nslices` slices on an
 * os x os grid (it chunks over slices when given less, down to one). */
long long tf_nufft_workspace_bytes(int os, long long nslices);

/* Type-1 NUFFT of nslices sample vectors (d_samples complex64, slice stride
 * sample_stride) onto the N x N grid, by Kaiser-Bessel gridding of width
 * `width` on an os x os grid (os a power of two, 32 <= os <= 8192, os >= 2N):
 *   d_tile_ptr / d_tile_idx : int32 CSR of the samples whose window touches
 *                             each 4-row band of each 32 x 32 grid tile (entry
 *                             (tb * (os/32) + ta) * 8 + band; (os/32)^2 * 8 + 1
 *                             pointers), samples ascending
 *   d_tile_order: int32 [(os/32)^2] order in which the tiles are launched (a
 *             permutation; NULL = natural order); heaviest tiles first keeps
 *             the dense centre tiles off the end of the launch
 *   d_ab     : int32 [S][2] first window index (x, y), in [0, os)
 *   d_wts    : fp32 [S][2*width] Kaiser-Bessel weights (x taps, then y taps)
 *   d_prephase: complex64 [os] = e^{-2 pi i a (N/2) / os}
 *   d_deapod : fp32 [N] deapodisation
 * d_out = scale * deapod[ix] deapod[iy] * (inverse grid FFT)[ix][iy]:
 * fp32 real part, or complex64 when out_complex.  Deterministic. */
int tf_nufft_type1(const void* d_samples, long long sample_stride, long long nslices, int n,
                   int os, int width, const int* d_tile_ptr, const int* d_tile_idx,
                   const int* d_tile_order, const void* d_ab, const float* d_wts, const void* d_prephase,
                   const float* d_deapod, float scale, int out_complex, void* d_out, void* d_ws,
                   long long ws_bytes, void* stream);

/* Plan tables of tf_nufft_type1 on the device: for every sample m (d_kxy:
 * [S][2] fp64 radial-frequency coordinates) and axis, the first window index
 * a0 = ceil(k os / (2 pi) - width/2) mod os (d_ab: int32 [S][2]) and the width
 * Kaiser-Bessel weights I0(beta sqrt(1 - (2x/width)^2)) (d_wts: fp32 [S][2*width]),
 * evaluated in fp64 (replaces NufftPlan._windows, nufft.py:158-164). */
int tf_nufft_plan_weights(const double* d_kxy, long long n_samples, int os, int width,
                          double beta, void* d_ab, float* d_wts, void* stream);

/* ---- forward projector --------------------------------
 * Type-2 NUFFT (nufft.type2, nufft.py:184-200) of nslices real N x N images:
 * deapodise, half spectrum of the offset-0 embedding on the os x os grid, then
 * per sample the width x width window gathered with the Kaiser-Bessel weights
 * and the conjugate pre-phase; d_out[z][m] (complex64) = that sum times
 * d_factor[m] (complex64, NULL = 1).  Tables as for tf_nufft_type1. */
long long tf_nufft_type2_workspace_bytes(int n, int os, long long nslices);
int tf_nufft_type2(const float* d_image, long long nslices, int n, int os, int width,
                   const void* d_ab, const float* d_wts, const void* d_prephase,
                   const float* d_deapod, const void* d_factor, long long n_samples, void* d_out,
                   void* d_ws, long long ws_bytes, void* stream);

/* Brute-force type-2 sum in fp64 (the oracle nufft.direct_dft, nufft.py:230-249):
 * d_out[m] (complex128) = sum_{ix,iy} d_image[ix][iy] exp(-i (kx x + ky y)) with
 * x = ix - (n-1)/2, (kx, ky) = d_kxy[m] (fp64 [S][2]); d_image fp64 [n][n]. */
int tf_direct_dft(const double* d_image, int n, const double* d_kxy, long long n_samples,
                  void* d_out, void* stream);

/* Real parts of the inverse DFTs of nrows complex rows given in signed-frequency
 * order (the ifftshift + ifft of radon.forward_project, radon.py:91-96), times
 * scale: d_out fp32 [nrows][nd]. */
int tf_detector_rows_inv(const void* d_samples, long long nrows, int nd, float scale,
                         float* d_out, void* stream);

/* ---- Lanczos-3 resampling (K9) ----------------------------------------------
 * One axis of the separable upsampler of multires.upsample (multires.py:145-195):
 *   d_out[o][t][i] = sum_{k < taps} d_weights[t][k] * d_in[o][d_start[t] + k][i]
 * for o < outer, t < n_tgt, i < inner (d_in is [outer][n_src][inner] fp32).
 * d_start (int32 [n_tgt]) / d_weights (fp32 [n_tgt][taps], taps <= 8) are the
 * band of the reference's edge-clamped, row-normalised interpolation matrix. */
int tf_resample_axis(const float* d_in, float* d_out, long long outer, int n_src, int n_tgt,
                     long long inner, const int* d_start, const float* d_weights, int taps,
                     void* stream);

/* All three axes of multires.upsample (multires.py:167-195) in one pass (K9f):
 *   d_out[tz][i][j] = sum_{a,b,c} wz[t][a] wx[i][b] wy[j][c]
 *                      d_src[sz[t]+a][sx[i]+b][sy[j]+c],   t = t_begin + tz,
 * for tz < nzt, i < ht, j < wt; d_src is [zs][hs][ws] fp32.  Each band (start
 * int32 [n_tgt], weights fp32 [n_tgt][k], k <= 8) is the reference matrix's
 * edge-clamped, row-normalised band (as tf_resample_axis).  Upsampling only
 * (hs <= ht, ws <= wt); a slab of the target is [t_begin, t_begin + nzt).
 * win_rows / win_cols bound the coarse window of every 32 x 128 target tile
 * (<= 40 / 136): the span of the tile's band starts plus the taps. */
int tf_upsample3(const float* d_src, int zs, int hs, int ws, float* d_out, int t_begin, int nzt,
                 int ht, int wt, const int* d_sz, const float* d_wz, int kz, const int* d_sx,
                 const float* d_wx, int kx, const int* d_sy, const float* d_wy, int ky,
                 int win_rows, int win_cols, void* stream);

/* Per-kernel CUDA-event timing used by bench.py for the roofline numbers.
 * Enable (clears totals), run, then collect: ms_out[slot] = total ms and
 * n_out[slot] = launches per slot (0 k_rows_fwd, 1 k_cols_conv, 2 k_rows_inv). */
int tf_timing_enable(int on);
int tf_timing_collect(double* ms_out, long long* n_out, int nslots);

/* Peer-memory halo exchange (z-slab runtime; replaces the NCCL send/recv of
 * runtime.exchange_halos, reference runtime.py:323-342).  After a stream-ordered
 * peer copy of a boundary plane into a neighbour's inbox (IPC-mapped device
 * memory), tf_halo_signal publishes `value` in the inbox slot's flag word
 * (uint64, system-scope fence first); tf_halo_wait makes the stream wait until
 * both flags (NULL = no neighbour) are >= value.  Single-thread kernels. */
int tf_halo_signal(void* d_flag, unsigned long long value, void* stream);
int tf_halo_wait(const void* d_flag_lo, const void* d_flag_hi, unsigned long long value,
                 void* stream);

#ifdef __cplusplus
}
#endif
#endif /* TOMOFORGE_B200_H */
