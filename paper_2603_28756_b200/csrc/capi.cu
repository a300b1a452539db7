// extern "C" boundary of libtomoforge_b200.so (declared in include/tomoforge_b200.h).
//
// Every entry point takes device pointers owned by the caller, a cudaStream_t
// (as void*), and returns 0 on success, -1 for a bad argument/shape, -2 for a
// CUDA error, -3 for an unsupported configuration; tf_last_error() returns a
// thread-local description of the last failure.  The library holds no state
// except the per-device twiddle table built by tf_init().
#include <cstdarg>
#include <mutex>
#include <string>
#include <vector>

#include "tf_common.cuh"

namespace tf {

static thread_local std::string g_err;

void set_error(const std::string& msg) { g_err = msg; }

int fail_arg(const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  set_error(buf);
  return TF_EARG;
}

int check_cuda(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return TF_OK;
  set_error(std::string(what) + ": " + cudaGetErrorString(e));
  return TF_ECUDA;
}

int check_launch(const char* what) { return check_cuda(cudaGetLastError(), what); }

// ---- per-kernel timing (slots: 0 rows_fwd, 1 cols_conv, 2 rows_inv, ...)
constexpr int TIMER_SLOTS = 16;
static std::mutex g_timer_mu;
static bool g_timing = false;
struct PendingTiming { cudaEvent_t a, b; int slot; };
static std::vector<PendingTiming> g_pending;
static double g_time_ms[TIMER_SLOTS];
static long long g_time_n[TIMER_SLOTS];

void timer_begin(KernelTimer& t, int slot, cudaStream_t st) {
  if (!g_timing) return;
  t.slot = slot;
  t.st = st;
  cudaEventCreate(&t.a);
  cudaEventCreate(&t.b);
  cudaEventRecord(t.a, st);
}

void timer_end(KernelTimer& t) {
  if (t.slot < 0) return;
  cudaEventRecord(t.b, t.st);
  std::lock_guard<std::mutex> lk(g_timer_mu);
  g_pending.push_back({t.a, t.b, t.slot});
}

static std::mutex g_init_mu;
static std::vector<int> g_inited;  // per device ordinal
static std::vector<int> g_sms;

int init_twiddles_toeplitz();
int init_twiddles_nufft();
int init_twiddles_toeplitz5();

int ensure_init() {
  int dev = 0;
  TF_TRY(check_cuda(cudaGetDevice(&dev), "cudaGetDevice"));
  std::lock_guard<std::mutex> lk(g_init_mu);
  if ((int)g_inited.size() <= dev) {
    g_inited.resize(dev + 1, 0);
    g_sms.resize(dev + 1, 0);
  }
  if (!g_inited[dev]) {
    TF_TRY(init_twiddles_toeplitz());
    TF_TRY(init_twiddles_nufft());
    TF_TRY(init_twiddles_toeplitz5());
    int sms = 0;
    TF_TRY(check_cuda(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev),
                      "cudaDeviceGetAttribute"));
    g_sms[dev] = sms;
    g_inited[dev] = 1;
  }
  return TF_OK;
}

int num_sms() {
  int dev = 0;
  cudaGetDevice(&dev);
  return (dev < (int)g_sms.size() && g_sms[dev] > 0) ? g_sms[dev] : 148;
}

// defined in the component translation units
int toeplitz_apply(const float* x, float* out, const float* aux, float alpha, float beta,
                   long long nslices, int n, int M, const void* PQ, const float* Bi, bool flip,
                   void* ws, size_t ws_bytes, cudaStream_t st);
size_t psf_workspace_bytes(int M);
int psf_build(int n, int M, const double* cs, int n_angles, int nd, void* PQ, float* Bi,
              void* ws, size_t ws_bytes, cudaStream_t st);
int psf_kernel_grid(int m, const double* cs, int n_angles, int nd, double* out, cudaStream_t st);
int reduce_blocks();
long long prior_partials(int h, int w);
int prior_update(const float* f, const float* f_lo, const float* f_hi, const float* fp,
                 const float* fp_lo, const float* fp_hi, const float* Kf, const float* Kfp,
                 const float* rstar, float* f_new, int nz, int h, int w_, float c, float lam,
                 float inv_L, int nonneg, int write_grad, int three_d, double sigma, double p,
                 double q, double T, const double* w, double* partial, double* out_gsq,
                 const float* c_dev, cudaStream_t st, const double* only_if);
int prior_energy_update(const float* f, const float* f_lo, const float* f_hi, const float* fp,
                        const float* fp_lo, const float* fp_hi, const float* Kf, const float* Kfp,
                        const float* rstar, float* f_new, int nz, int h, int w_, const double* state,
                        float lam, float inv_L, int nonneg, int with_prior, double sigma, double p,
                        double q, double T, const double* w, double* partial, double* out_e,
                        double* out_fid, double* out_dfid, double* out_gsq, cudaStream_t st);
int solver_decide(const double* vals, double* state, float* c_out, double* rec, double lam,
                  int with_prior, int restart, double tol, cudaStream_t st);
int energy_fid(const float* fn, const float* fn_hi, const float* f, const float* Kfn,
               const float* Kf, const float* rstar, int nz, int h, int w_, int with_prior,
               int three_d, double sigma, double p, double q, double T, const double* w,
               double* partial, double* out3, cudaStream_t st);
int dot2(const float* x, const float* a, const float* b, long long n, double* out, double* ws,
         cudaStream_t st);
size_t nufft_workspace_bytes(int os, long long nslices);
int direct_dft(const double* img, int n, const double* kxy, long long S, void* out,
               cudaStream_t st);
size_t type2_workspace_bytes(int n, int os, long long nslices);
int nufft_type2(const float* img, long long nslices, int n, int os, int w, const void* ab,
                const float* wts, const void* preph, const float* deapod, const void* factor,
                long long n_samples, void* out, void* ws, size_t ws_bytes, cudaStream_t st);
int detector_rows_inv(const void* c, long long nrows, int nd, float gain, float* out,
                      cudaStream_t st);
int nufft_plan_weights(const double* kxy, long long S, int os, int w, double beta, void* ab,
                       float* wts, cudaStream_t st);
int upsample3(const float* src, int zs, int hs, int ws, float* out, int t_begin, int nzt, int ht,
              int wt, const int* sz, const float* wz, int kz, const int* sx, const float* wx, int kx,
              const int* sy, const float* wy, int ky, int nrm, int ncm, cudaStream_t st);
int resample_axis(const float* in, float* out, long long outer, int n_src, int n_tgt,
                  long long inner, const int* s0, const float* w, int K, cudaStream_t st);
int detector_rows(const float* rows, long long nrows, int nd, int n_angles, const void* sph,
                  int mode, int ramp, float scale, void* out, cudaStream_t st);
int nufft_type1(const void* samples, long long s_stride, long long nslices, int n, int os, int w,
                const int* tile_ptr, const int* tile_idx, const int* tile_order, const void* ab,
                const float* wts,
                const void* preph, const float* deapod, float scale, int cplx, void* out,
                void* ws, size_t ws_bytes, cudaStream_t st);

int halo_signal(unsigned long long* flag, unsigned long long value, cudaStream_t st);
int halo_wait(const unsigned long long* flag_lo, const unsigned long long* flag_hi,
              unsigned long long value, cudaStream_t st);

}  // namespace tf

using namespace tf;

extern "C" {

const char* tf_last_error(void) { return g_err.c_str(); }

int tf_version(void) { return 1; }

int tf_init(void) { return ensure_init(); }

int tf_fft_side(int n) {
  if (n < 1) return fail_arg("source side must be positive");
  int M = 8;
  while (M < 2 * n - 1) M <<= 1;
  if (M > 8192) return fail_arg("source side %d exceeds the supported maximum 4096", n);
  // a 5 * 2^k side (radix-5 step, toeplitz5.cu) when it is smaller
  for (int q = 256; q <= 1024; q <<= 1)
    if (5 * q >= 2 * n - 1 && 5 * q < M) return 5 * q;
  return M;
}

long long tf_toeplitz_workspace_bytes(int n, int M, long long nslices) {
  // row-blocked half spectra: [nslices][ceil(n/4)][M/2+1][4] complex64
  return (long long)(M / 2 + 1) * 4 * ((n + 3) / 4) * (long long)sizeof(c32) * nslices;
}

long long tf_psf_workspace_bytes(int M) { return (long long)psf_workspace_bytes(M); }

int tf_psf_build(int n, int M, int n_angles, const double* d_cossin, int nd, void* d_PQ,
                 float* d_Bi, void* d_ws, long long ws_bytes, void* stream) {
  TF_TRY(ensure_init());
  if (n < 1 || M < 2 * n - 1 || !(is_pow2(M) || is_side5(M)))
    return fail_arg("bad psf sides n=%d M=%d", n, M);
  if (n_angles < 1 || nd < 1) return fail_arg("bad sampling (angles=%d, nd=%d)", n_angles, nd);
  if (!d_cossin || !d_PQ || !d_Bi || !d_ws) return fail_arg("null pointer");
  return psf_build(n, M, d_cossin, n_angles, nd, d_PQ, d_Bi, d_ws, (size_t)ws_bytes,
                   (cudaStream_t)stream);
}

int tf_psf_kernel(int m, int n_angles, const double* d_cossin, int nd, double* d_out,
                  void* stream) {
  TF_TRY(ensure_init());
  if (m < 1 || m % 2 == 0 || m > 32768) return fail_arg("kernel grid side must be odd, got %d", m);
  if (n_angles < 1 || nd < 1) return fail_arg("bad sampling (angles=%d, nd=%d)", n_angles, nd);
  if (!d_cossin || !d_out) return fail_arg("null pointer");
  return psf_kernel_grid(m, d_cossin, n_angles, nd, d_out, (cudaStream_t)stream);
}

int tf_toeplitz_apply(const float* d_x, float* d_out, const float* d_aux, float alpha,
                      float beta, long long nslices, int n, int M, const void* d_PQ,
                      const float* d_Bi, int has_flip, void* d_ws, long long ws_bytes,
                      void* stream) {
  TF_TRY(ensure_init());
  if (n < 1 || M < 2 * n - 1 || !(is_pow2(M) || is_side5(M)))
    return fail_arg("bad sides n=%d M=%d", n, M);
  if (nslices < 0) return fail_arg("negative slice count");
  if (nslices == 0) return TF_OK;
  if (!d_x || !d_out || !d_PQ || (has_flip && !d_Bi) || !d_ws)
    return fail_arg("null pointer");
  if (d_x == d_out) return fail_arg("in-place apply is not supported");
  return toeplitz_apply(d_x, d_out, d_aux, alpha, beta, nslices, n, M, d_PQ, d_Bi, has_flip != 0,
                        d_ws, (size_t)ws_bytes, (cudaStream_t)stream);
}

long long tf_reduce_workspace_bytes(void) {
  if (ensure_init() != TF_OK) return -1;
  return (long long)reduce_blocks() * 4 * (long long)sizeof(double);
}

int tf_dot2(const float* d_x, const float* d_a, const float* d_b, long long n, double* d_out,
            double* d_ws, void* stream) {
  TF_TRY(ensure_init());
  if (n < 0 || !d_x || !d_a || !d_out || !d_ws) return fail_arg("bad tf_dot2 arguments");
  return dot2(d_x, d_a, d_b, n, d_out, d_ws, (cudaStream_t)stream);
}

long long tf_prior_workspace_bytes(int h, int w) {
  if (h < 1 || w < 1) return fail_arg("bad slice shape");
  return prior_partials(h, w) * 3 * (long long)sizeof(double);
}

static int check_prior(int h, int w, int nz, double sigma, double p, double q, double T) {
  if (h < 1 || w < 1 || nz < 1) return fail_arg("bad volume shape (%d x %d x %d)", nz, h, w);
  if (!(1.0 <= q && q < p && p <= 2.0)) return fail_arg("require 1 <= q < p <= 2");
  if (!(sigma > 0) || !(T > 0)) return fail_arg("sigma and T must be positive");
  return TF_OK;
}

int tf_prior_update_dc(const float* d_f, const float* d_f_lo, const float* d_f_hi,
                       const float* d_fp, const float* d_fp_lo, const float* d_fp_hi,
                       const float* d_Kf, const float* d_Kfp, const float* d_rstar, float* d_out,
                       int nz, int h, int w, float c, const float* d_c, float lam, float inv_L,
                       int nonneg, int write_grad, int three_d, double sigma, double p, double q,
                       double T, const double* weights3, double* d_ws, double* d_gsq,
                       void* stream);

int tf_prior_update(const float* d_f, const float* d_f_lo, const float* d_f_hi, const float* d_fp,
                    const float* d_fp_lo, const float* d_fp_hi, const float* d_Kf,
                    const float* d_Kfp, const float* d_rstar, float* d_out, int nz, int h, int w,
                    float c, float lam, float inv_L, int nonneg, int write_grad, int three_d,
                    double sigma, double p, double q, double T, const double* weights3,
                    double* d_ws, double* d_gsq, void* stream) {
  return tf_prior_update_dc(d_f, d_f_lo, d_f_hi, d_fp, d_fp_lo, d_fp_hi, d_Kf, d_Kfp, d_rstar,
                            d_out, nz, h, w, c, nullptr, lam, inv_L, nonneg, write_grad, three_d,
                            sigma, p, q, T, weights3, d_ws, d_gsq, stream);
}

int tf_prior_update_dc(const float* d_f, const float* d_f_lo, const float* d_f_hi,
                       const float* d_fp, const float* d_fp_lo, const float* d_fp_hi,
                       const float* d_Kf, const float* d_Kfp, const float* d_rstar, float* d_out,
                       int nz, int h, int w, float c, const float* d_c, float lam, float inv_L,
                       int nonneg, int write_grad, int three_d, double sigma, double p, double q,
                       double T, const double* weights3, double* d_ws, double* d_gsq,
                       void* stream) {
  TF_TRY(ensure_init());
  TF_TRY(check_prior(h, w, nz, sigma, p, q, T));
  if (!d_f || !d_fp || !d_out || !d_ws || !d_gsq || !weights3) return fail_arg("null pointer");
  if ((d_Kf == nullptr) != (d_Kfp == nullptr)) return fail_arg("Kf and Kfp must both be given");
  if ((d_f_lo == nullptr) != (d_fp_lo == nullptr) || (d_f_hi == nullptr) != (d_fp_hi == nullptr))
    return fail_arg("halo planes of f and f_prev must both be given");
  return prior_update(d_f, d_f_lo, d_f_hi, d_fp, d_fp_lo, d_fp_hi, d_Kf, d_Kfp, d_rstar, d_out, nz,
                      h, w, c, lam, inv_L, nonneg, write_grad, three_d, sigma, p, q, T, weights3, d_ws,
                      d_gsq, d_c, (cudaStream_t)stream, nullptr);
}

int tf_prior_update_if(const float* d_f, const float* d_f_lo, const float* d_f_hi,
                       const float* d_fp, const float* d_fp_lo, const float* d_fp_hi,
                       const float* d_Kf, const float* d_Kfp, const float* d_rstar, float* d_out,
                       int nz, int h, int w, const float* d_c, float lam, float inv_L, int nonneg,
                       double sigma, double p, double q, double T, const double* weights3,
                       double* d_ws, double* d_gsq, const double* d_only_if, void* stream) {
  TF_TRY(ensure_init());
  TF_TRY(check_prior(h, w, nz, sigma, p, q, T));
  if (!d_f || !d_fp || !d_out || !d_ws || !d_gsq || !weights3 || !d_c || !d_only_if)
    return fail_arg("null pointer");
  if ((d_Kf == nullptr) != (d_Kfp == nullptr)) return fail_arg("Kf and Kfp must both be given");
  if ((d_f_lo == nullptr) != (d_fp_lo == nullptr) || (d_f_hi == nullptr) != (d_fp_hi == nullptr))
    return fail_arg("halo planes of f and f_prev must both be given");
  return prior_update(d_f, d_f_lo, d_f_hi, d_fp, d_fp_lo, d_fp_hi, d_Kf, d_Kfp, d_rstar, d_out, nz,
                      h, w, 0.f, lam, inv_L, nonneg, 0, 1, sigma, p, q, T, weights3, d_ws, d_gsq, d_c,
                      (cudaStream_t)stream, d_only_if);
}

int tf_prior_energy_update(const float* d_f, const float* d_f_lo, const float* d_f_hi,
                           const float* d_fp, const float* d_fp_lo, const float* d_fp_hi,
                           const float* d_Kf, const float* d_Kfp, const float* d_rstar,
                           float* d_out, int nz, int h, int w, const double* d_state, float lam,
                           float inv_L, int nonneg, int with_prior, double sigma, double p,
                           double q, double T, const double* weights3, double* d_ws,
                           double* d_energy, double* d_fid, double* d_dfid, double* d_gsq,
                           void* stream) {
  TF_TRY(ensure_init());
  TF_TRY(check_prior(h, w, nz, sigma, p, q, T));
  if (!d_f || !d_fp || !d_Kf || !d_Kfp || !d_rstar || !d_out || !d_ws || !weights3 || !d_state)
    return fail_arg("null pointer");
  if ((d_f_lo == nullptr) != (d_fp_lo == nullptr) || (d_f_hi == nullptr) != (d_fp_hi == nullptr))
    return fail_arg("halo planes of f and f_prev must both be given");
  if (d_out == d_f || d_out == d_fp || d_out == d_Kf || d_out == d_rstar)
    return fail_arg("output may alias only d_Kfp");
  return prior_energy_update(d_f, d_f_lo, d_f_hi, d_fp, d_fp_lo, d_fp_hi, d_Kf, d_Kfp, d_rstar,
                             d_out, nz, h, w, d_state, lam, inv_L, nonneg, with_prior, sigma, p, q,
                             T, weights3, d_ws, d_energy, d_fid, d_dfid, d_gsq,
                             (cudaStream_t)stream);
}

int tf_solver_decide(const double* d_vals, double* d_state, float* d_c, double* d_rec, double lam,
                     int with_prior, int restart, double tol, void* stream) {
  TF_TRY(ensure_init());
  if (!d_vals || !d_state || !d_c || !d_rec) return fail_arg("null pointer");
  if (!(tol > 0)) return fail_arg("tol must be positive");
  return solver_decide(d_vals, d_state, d_c, d_rec, lam, with_prior, restart, tol,
                       (cudaStream_t)stream);
}

int tf_energy_fid(const float* d_fn, const float* d_fn_hi, const float* d_f, const float* d_Kfn,
                  const float* d_Kf, const float* d_rstar, int nz, int h, int w, int with_prior,
                  int three_d, double sigma, double p, double q, double T, const double* weights3,
                  double* d_ws, double* d_out3, void* stream) {
  TF_TRY(ensure_init());
  TF_TRY(check_prior(h, w, nz, sigma, p, q, T));
  if (!d_fn || !d_ws || !d_out3 || !weights3) return fail_arg("null pointer");
  if (d_f && (!d_Kf || !d_Kfn)) return fail_arg("increment needs Kf and Kf_new");
  return energy_fid(d_fn, d_fn_hi, d_f, d_Kfn, d_Kf, d_rstar, nz, h, w, with_prior, three_d, sigma, p,
                    q, T, weights3, d_ws, d_out3, (cudaStream_t)stream);
}

long long tf_nufft_workspace_bytes(int os, long long nslices) {
  if (os < 1 || nslices < 0) return fail_arg("bad NUFFT workspace query");
  return (long long)nufft_workspace_bytes(os, nslices);
}

int tf_detector_rows(const float* d_rows, long long nrows, int nd, int n_angles,
                     const void* d_sphase, int mode, int ramp, float scale, void* d_out,
                     void* stream) {
  TF_TRY(ensure_init());
  if (nrows < 0 || !d_rows || !d_out) return fail_arg("bad tf_detector_rows arguments");
  if (mode != 0 && mode != 1) return fail_arg("mode must be 0 (samples) or 1 (ramp rows)");
  if (nrows == 0) return TF_OK;
  return detector_rows(d_rows, nrows, nd, n_angles, d_sphase, mode, ramp, scale, d_out,
                       (cudaStream_t)stream);
}

int tf_nufft_type1(const void* d_samples, long long sample_stride, long long nslices, int n,
                   int os, int width, const int* d_tile_ptr, const int* d_tile_idx,
                   const int* d_tile_order, const void* d_ab, const float* d_wts, const void* d_prephase,
                   const float* d_deapod, float scale, int out_complex, void* d_out, void* d_ws,
                   long long ws_bytes, void* stream) {
  TF_TRY(ensure_init());
  if (nslices < 0 || n < 1) return fail_arg("bad NUFFT shape");
  if (nslices == 0) return TF_OK;
  if (!d_samples || !d_tile_ptr || !d_tile_idx || !d_ab || !d_wts || !d_prephase || !d_deapod ||
      !d_out || !d_ws)
    return fail_arg("null pointer");
  return nufft_type1(d_samples, sample_stride, nslices, n, os, width, d_tile_ptr, d_tile_idx,
                     d_tile_order, d_ab,
                     d_wts, d_prephase, d_deapod, scale, out_complex, d_out, d_ws,
                     (size_t)ws_bytes, (cudaStream_t)stream);
}

int tf_nufft_plan_weights(const double* d_kxy, long long n_samples, int os, int width,
                          double beta, void* d_ab, float* d_wts, void* stream) {
  TF_TRY(ensure_init());
  if (n_samples < 0 || os < 2 || width < 2 || width > 16) return fail_arg("bad plan arguments");
  if (n_samples > 0 && (!d_kxy || !d_ab || !d_wts)) return fail_arg("null pointer");
  return nufft_plan_weights(d_kxy, n_samples, os, width, beta, d_ab, d_wts, (cudaStream_t)stream);
}

long long tf_nufft_type2_workspace_bytes(int n, int os, long long nslices) {
  if (n < 1 || os < 2 || nslices < 0) return fail_arg("bad type2 workspace query");
  return (long long)type2_workspace_bytes(n, os, nslices);
}

int tf_nufft_type2(const float* d_image, long long nslices, int n, int os, int width,
                   const void* d_ab, const float* d_wts, const void* d_prephase,
                   const float* d_deapod, const void* d_factor, long long n_samples, void* d_out,
                   void* d_ws, long long ws_bytes, void* stream) {
  TF_TRY(ensure_init());
  if (nslices < 0 || n < 1 || n_samples < 0) return fail_arg("bad type2 shape");
  if (nslices == 0 || n_samples == 0) return TF_OK;
  if (!d_image || !d_ab || !d_wts || !d_prephase || !d_deapod || !d_out || !d_ws)
    return fail_arg("null pointer");
  return nufft_type2(d_image, nslices, n, os, width, d_ab, d_wts, d_prephase, d_deapod, d_factor,
                     n_samples, d_out, d_ws, (size_t)ws_bytes, (cudaStream_t)stream);
}

int tf_detector_rows_inv(const void* d_samples, long long nrows, int nd, float scale,
                         float* d_out, void* stream) {
  TF_TRY(ensure_init());
  if (nrows < 0 || (nrows > 0 && (!d_samples || !d_out))) return fail_arg("bad arguments");
  return detector_rows_inv(d_samples, nrows, nd, scale, d_out, (cudaStream_t)stream);
}

int tf_direct_dft(const double* d_image, int n, const double* d_kxy, long long n_samples,
                  void* d_out, void* stream) {
  TF_TRY(ensure_init());
  if (n < 1 || n_samples < 0) return fail_arg("bad direct DFT shape");
  if (n_samples > 0 && (!d_image || !d_kxy || !d_out)) return fail_arg("null pointer");
  return direct_dft(d_image, n, d_kxy, n_samples, d_out, (cudaStream_t)stream);
}

int tf_upsample3(const float* d_src, int zs, int hs, int ws, float* d_out, int t_begin, int nzt,
                 int ht, int wt, const int* d_sz, const float* d_wz, int kz, const int* d_sx,
                 const float* d_wx, int kx, const int* d_sy, const float* d_wy, int ky,
                 int win_rows, int win_cols, void* stream) {
  TF_TRY(ensure_init());
  if (zs < 1 || hs < 1 || ws < 1 || ht < 1 || wt < 1 || nzt < 0 || t_begin < 0)
    return fail_arg("bad upsample shapes");
  if (!d_src || !d_out || !d_sz || !d_wz || !d_sx || !d_wx || !d_sy || !d_wy)
    return fail_arg("null pointer");
  if (d_src == d_out) return fail_arg("in-place resampling is not supported");
  return upsample3(d_src, zs, hs, ws, d_out, t_begin, nzt, ht, wt, d_sz, d_wz, kz, d_sx, d_wx, kx,
                   d_sy, d_wy, ky, win_rows, win_cols, (cudaStream_t)stream);
}

int tf_resample_axis(const float* d_in, float* d_out, long long outer, int n_src, int n_tgt,
                     long long inner, const int* d_start, const float* d_weights, int taps,
                     void* stream) {
  TF_TRY(ensure_init());
  if (outer < 0 || n_src < 1 || n_tgt < 1 || inner < 1 || taps < 1)
    return fail_arg("bad resampling shape");
  if (!d_in || !d_out || !d_start || !d_weights) return fail_arg("null pointer");
  if (d_in == d_out) return fail_arg("in-place resampling is not supported");
  return resample_axis(d_in, d_out, outer, n_src, n_tgt, inner, d_start, d_weights, taps,
                       (cudaStream_t)stream);
}

int tf_timing_enable(int on) {
  std::lock_guard<std::mutex> lk(g_timer_mu);
  g_timing = on != 0;
  for (int i = 0; i < TIMER_SLOTS; ++i) { g_time_ms[i] = 0.0; g_time_n[i] = 0; }
  return TF_OK;
}

// Synchronise the recorded events and return per-slot (total ms, launch count).
int tf_timing_collect(double* ms_out, long long* n_out, int nslots) {
  std::lock_guard<std::mutex> lk(g_timer_mu);
  for (auto& p : g_pending) {
    float ms = 0.f;
    TF_TRY(check_cuda(cudaEventSynchronize(p.b), "cudaEventSynchronize"));
    TF_TRY(check_cuda(cudaEventElapsedTime(&ms, p.a, p.b), "cudaEventElapsedTime"));
    g_time_ms[p.slot] += ms;
    g_time_n[p.slot] += 1;
    cudaEventDestroy(p.a);
    cudaEventDestroy(p.b);
  }
  g_pending.clear();
  for (int i = 0; i < nslots && i < TIMER_SLOTS; ++i) {
    ms_out[i] = g_time_ms[i];
    n_out[i] = g_time_n[i];
  }
  return TF_OK;
}


int tf_halo_signal(void* d_flag, unsigned long long value, void* stream) {
  TF_TRY(ensure_init());
  if (!d_flag) return fail_arg("null flag");
  return halo_signal(reinterpret_cast<unsigned long long*>(d_flag), value, (cudaStream_t)stream);
}

int tf_halo_wait(const void* d_flag_lo, const void* d_flag_hi, unsigned long long value,
                 void* stream) {
  TF_TRY(ensure_init());
  return halo_wait(reinterpret_cast<const unsigned long long*>(d_flag_lo),
                   reinterpret_cast<const unsigned long long*>(d_flag_hi), value,
                   (cudaStream_t)stream);
}

}  // extern "C"
