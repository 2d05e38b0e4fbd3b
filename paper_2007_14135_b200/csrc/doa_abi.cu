// C ABI of libdoa (include/doa.h): argument validation, plan/workspace management, error
// reporting, and the composition of the kernels into doa_run / doa_run_host.
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "doa_internal.cuh"

namespace {

thread_local std::string g_err;
thread_local int g_launches = 0;

doa_status_t fail(doa_status_t st, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
doa_status_t fail(doa_status_t st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}

doa_status_t cuda_fail(cudaError_t e, const char* where) {
  return fail(e == cudaErrorMemoryAllocation ? DOA_ERR_OUT_OF_MEMORY : DOA_ERR_CUDA, "%s: %s (%s)", where,
              cudaGetErrorName(e), cudaGetErrorString(e));
}

bool aligned(const void* p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

#define DOA_CHECK_PLAN(p)                                                                          \
  do {                                                                                             \
    if (!(p)) return fail(DOA_ERR_INVALID_ARG, "%s: plan is NULL", __func__);                      \
    if (doa::current_device() != (p)->device)                                                      \
      return fail(DOA_ERR_INVALID_ARG, "%s: plan was created on device %d, current device is %d", \
                  __func__, (p)->device, doa::current_device());                                   \
  } while (0)
#define DOA_CHECK_PTR(ptr, al)                                                                         \
  do {                                                                                                 \
    if (!(ptr)) return fail(DOA_ERR_INVALID_ARG, "%s: %s is NULL", __func__, #ptr);                    \
    if (!aligned((ptr), (al))) return fail(DOA_ERR_INVALID_ARG, "%s: %s is not %d-byte aligned", __func__, #ptr, (int)(al)); \
  } while (0)
#define DOA_CHECK_B(p, B)                                                                                  \
  do {                                                                                                     \
    if ((B) < 0 || (B) > (p)->max_batch)                                                                   \
      return fail(DOA_ERR_INVALID_ARG, "%s: B=%lld outside [0, max_batch=%lld]", __func__, (long long)(B), \
                  (long long)(p)->max_batch);                                                              \
  } while (0)
#define DOA_TRY(expr, where)                       \
  do {                                             \
    cudaError_t e_ = (expr);                       \
    if (e_ != cudaSuccess) return cuda_fail(e_, where); \
  } while (0)

// R / lambda / V scratch for doa_run, allocated on first use.
cudaError_t ensure_run_scratch(doa_plan_s* p) {
  if (p->R) return cudaSuccess;
  const size_t B = (size_t)p->max_batch, M = (size_t)p->M;
  cudaError_t e = cudaMalloc((void**)&p->R, B * M * M * 2 * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc((void**)&p->lam, B * M * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc((void**)&p->V, B * M * M * 2 * sizeof(double));
  if (e == cudaSuccess && M <= 16) e = cudaMalloc(&p->cov_ws, doa::cov_workspace_bytes());
  if (e == cudaSuccess && p->cov_ws) e = cudaMemset(p->cov_ws, 0, doa::cov_workspace_bytes());   // tickets
  if (e != cudaSuccess) {
    cudaFree(p->R); cudaFree(p->lam); cudaFree(p->V); cudaFree(p->cov_ws);
    p->R = nullptr; p->lam = nullptr; p->V = nullptr; p->cov_ws = nullptr;
  }
  return e;
}

// S3-S6 for either plan geometry: ULA -> Toeplitz coefficients + fused DMMA scan/peak test;
// general array -> array coefficients + DMMA scan into the plan's f buffer + 2-D peak search.
cudaError_t spectrum_stage(const doa_plan_s* p, const double* lam, const double* V, int64_t B, float* P,
                           int32_t* info, cudaStream_t s) {
  if (p->geom == 1) return doa::launch_array_spectrum(p, lam, V, B, P, info, s);
  if (p->engine != DOA_ENGINE_TOEPLITZ_FP64) {
    cudaError_t e = doa::launch_vec32(p, lam, V, B, info, s);
    if (e != cudaSuccess) return e;
    return doa::launch_scan_direct_form(p, B, P, s);
  }
  cudaError_t e = doa::launch_coef(p, lam, V, B, info, s);
  if (e != cudaSuccess) return e;
  return doa::launch_scan(p, B, P, s);
}

// S4-S6 for the ULA plans among plans[0..nplans): consecutive direct-compatible plans share one scan
// launch (up to kMaxCoefPlans); the coefficients must be in place and the counters zeroed.
// P (nullable) is used only when nplans == 1.
cudaError_t scan_stage(doa_plan_s* const* plans, int nplans, int64_t B, float* P, cudaStream_t st) {
  cudaError_t e = cudaSuccess;
  for (int a = 0; a < nplans && e == cudaSuccess;) {
    if (plans[a]->geom == 1) { ++a; continue; }
    if (plans[a]->engine != DOA_ENGINE_TOEPLITZ_FP64) {
      e = doa::launch_scan_direct_form(plans[a], B, nplans == 1 ? P : nullptr, st);
      ++a;
      continue;
    }
    const doa_plan_s* grp[doa::kMaxCoefPlans] = {};
    int n = 0;
    while (a < nplans && n < doa::kMaxCoefPlans && plans[a]->geom == 0 && plans[a]->engine == DOA_ENGINE_TOEPLITZ_FP64 &&
           (n == 0 || doa::direct_compatible(plans[a], grp[0])))
      grp[n++] = plans[a++];
    e = doa::launch_scan_plans(grp, n, B, nplans == 1 ? P : nullptr, st);
  }
  return e;
}

// S1-S7 for nplans plans sharing M and D on device buffers (doa_run_multi, doa_run, and doa_run_host
// per chunk): the covariance once (plans[0]'s scratch); for M <= 16 and up to kMaxCoefPlans ULA
// plans the frame kernel (eigendecomposition + every plan's coefficients in one launch, V never
// leaves the SM), otherwise the eigendecomposition once and per plan S3; then the scans (one launch
// per group of grid-sharing plans) and the peak selection.  Plan a's outputs live at
// idx + a*ldo*D, val + a*ldo*D, npk + a*ldo, info + a*ldo.
cudaError_t run_plans(doa_plan_s* const* plans, int nplans, const float* X, int64_t B, int64_t N, int32_t* idx,
                      float* val, int32_t* npk, int32_t* info, int64_t ldo, cudaStream_t st,
                      cudaEvent_t x_consumed = nullptr, float* P = nullptr) {
  doa_plan_s* p = plans[0];
  const int M = p->M, D = p->D;
  cudaError_t e = doa::launch_covariance(X, B, N, M, p->R, st, p->cov_ws);
  if (e == cudaSuccess && x_consumed) e = cudaEventRecord(x_consumed, st);   // X no longer needed
  bool fused = M <= 16 && nplans <= doa::kMaxCoefPlans;
  for (int a = 0; a < nplans; ++a) fused &= plans[a]->geom == 0 && plans[a]->engine == DOA_ENGINE_TOEPLITZ_FP64;
  if (fused) {
    doa::CoefPlans cp = {};
    cp.nplans = nplans;
    for (int a = 0; a < nplans; ++a) {
      cp.alg[a] = plans[a]->alg; cp.coef[a] = plans[a]->coef; cp.cnt[a] = plans[a]->cnt;
      cp.info[a] = info + (size_t)a * ldo;
    }
    if (e == cudaSuccess) e = doa::launch_eig16_coef(p->R, B, M, D, nullptr, nullptr, cp, st);
  } else {
    if (e == cudaSuccess) e = doa::launch_eig(p->R, B, M, p->lam, p->V, info, st);
    for (int a = 1; a < nplans && e == cudaSuccess; ++a)        // every plan starts from the eig flags
      e = cudaMemcpyAsync(info + (size_t)a * ldo, info, (size_t)B * sizeof(int32_t), cudaMemcpyDeviceToDevice, st);
    const doa_plan_s* ula[64];
    int32_t* ula_info[64];
    int nu = 0;
    for (int a = 0; a < nplans && e == cudaSuccess; ++a) {
      doa_plan_s* q = plans[a];
      if (q->geom == 1) e = doa::launch_array_spectrum(q, p->lam, p->V, B, nplans == 1 ? P : nullptr, info + (size_t)a * ldo, st);
      else if (q->engine != DOA_ENGINE_TOEPLITZ_FP64) e = doa::launch_vec32(q, p->lam, p->V, B, info + (size_t)a * ldo, st);
      else if (nu < 64) { ula[nu] = q; ula_info[nu++] = info + (size_t)a * ldo; }
      else e = doa::launch_coef(q, p->lam, p->V, B, info + (size_t)a * ldo, st);
    }
    if (e == cudaSuccess && nu) e = doa::launch_coef_multi(ula, nu, p->lam, p->V, B, ula_info, st);
  }
  if (e == cudaSuccess) e = scan_stage(plans, nplans, B, P, st);
  for (int a0 = 0; a0 < nplans && e == cudaSuccess; a0 += 4) {     // S7: one launch per 4 plans
    doa::SelectPlans sp = {};
    sp.nplans = nplans - a0 < 4 ? nplans - a0 : 4;
    for (int k = 0; k < sp.nplans; ++k) {
      doa_plan_s* q = plans[a0 + k];
      const size_t a = (size_t)(a0 + k);
      sp.cnt[k] = q->cnt; sp.cidx[k] = q->cand_idx; sp.cf[k] = q->cand_f; sp.cap[k] = q->cap;
      sp.idx[k] = idx + a * ldo * D; sp.val[k] = val + a * ldo * D; sp.npk[k] = npk + a * ldo;
      sp.info[k] = info + a * ldo;
      q->last_B = B;
      q->coef_B = q->geom == 0 ? B : 0;
    }
    e = doa::launch_select_multi(sp, D, B, st);
  }
  return e;
}

doa_status_t check_plan_set(const char* fn, const doa_plan_t* plans, int32_t nplans, int64_t B) {
  if (!plans || nplans < 1) return fail(DOA_ERR_INVALID_ARG, "%s: need nplans >= 1 plans", fn);
  const int dev = doa::current_device();
  for (int k = 0; k < nplans; ++k) {
    if (!plans[k]) return fail(DOA_ERR_INVALID_ARG, "%s: plans[%d] is NULL", fn, k);
    if (plans[k]->device != dev)
      return fail(DOA_ERR_INVALID_ARG, "%s: plans[%d] was created on device %d, current device is %d", fn, k,
                  plans[k]->device, dev);
    if (plans[k]->M != plans[0]->M || plans[k]->D != plans[0]->D)
      return fail(DOA_ERR_INVALID_ARG, "%s: plans must share M and D", fn);
    if (B < 0 || B > plans[k]->max_batch)
      return fail(DOA_ERR_INVALID_ARG, "%s: B=%lld outside [0, max_batch=%lld] of plans[%d]", fn, (long long)B,
                  (long long)plans[k]->max_batch, k);
    for (int j = 0; j < k; ++j)
      if (plans[j] == plans[k]) return fail(DOA_ERR_INVALID_ARG, "%s: plans[%d] repeats plans[%d]", fn, k, j);
  }
  return DOA_OK;
}

}  // namespace

namespace doa {
void count_launch() { ++g_launches; }
}  // namespace doa

extern "C" {

int32_t doa_version(void) { return 1; }

doa_status_t doa_generate(int32_t M, double d_over_lambda, int32_t D, const double* theta_deg,
                          int32_t theta_per_frame, double snr_db, uint64_t seed, int64_t frame0, int64_t B,
                          int64_t N, float* X, doa_stream_t stream) {
  g_launches = 0;
  if (M < 1 || M > doa::kMaxM) return fail(DOA_ERR_INVALID_ARG, "doa_generate: M=%d outside [1, %d]", M, doa::kMaxM);
  if (D < 1 || D > 63) return fail(DOA_ERR_INVALID_ARG, "doa_generate: D=%d outside [1, 63]", D);
  if (N < 1 || N > ((int64_t)1 << 24)) return fail(DOA_ERR_INVALID_ARG, "doa_generate: N=%lld outside [1, 2^24]", (long long)N);
  if (B >= ((int64_t)1 << 31)) return fail(DOA_ERR_INVALID_ARG, "doa_generate: B=%lld >= 2^31", (long long)B);
  if (B < 0 || frame0 < 0) return fail(DOA_ERR_INVALID_ARG, "doa_generate: negative B or frame0");
  if (!(d_over_lambda > 0.0) || !std::isfinite(d_over_lambda) || !std::isfinite(snr_db))
    return fail(DOA_ERR_INVALID_ARG, "doa_generate: d/lambda must be positive and snr_db finite");
  if (B == 0) return DOA_OK;
  DOA_CHECK_PTR(theta_deg, 8);
  DOA_CHECK_PTR(X, 8);
  DOA_TRY(doa::launch_generate(M, d_over_lambda, D, theta_deg, theta_per_frame ? 1 : 0, snr_db, seed, frame0, B, N, X,
                               reinterpret_cast<cudaStream_t>(stream)),
          "doa_generate");
  return DOA_OK;
}
int32_t doa_last_launch_count(void) { return g_launches; }
const char* doa_last_error(void) { return g_err.c_str(); }

const char* doa_status_string(doa_status_t s) {
  switch (s) {
    case DOA_OK: return "DOA_OK";
    case DOA_ERR_INVALID_ARG: return "DOA_ERR_INVALID_ARG";
    case DOA_ERR_UNSUPPORTED: return "DOA_ERR_UNSUPPORTED";
    case DOA_ERR_OUT_OF_MEMORY: return "DOA_ERR_OUT_OF_MEMORY";
    case DOA_ERR_CUDA: return "DOA_ERR_CUDA";
  }
  return "DOA_ERR_UNKNOWN";
}

doa_status_t doa_plan_create(doa_plan_t* plan, int32_t M, double d_over_lambda, int32_t D, double theta0_deg,
                             double dtheta_deg, int64_t L, int32_t alg, int64_t max_batch) {
  g_launches = 0;
  if (!plan) return fail(DOA_ERR_INVALID_ARG, "doa_plan_create: plan out-pointer is NULL");
  *plan = nullptr;
  if (M < 2) return fail(DOA_ERR_INVALID_ARG, "doa_plan_create: M=%d < 2", M);
  if (M > doa::kMaxM) return fail(DOA_ERR_UNSUPPORTED, "doa_plan_create: M=%d > %d", M, doa::kMaxM);
  if (D < 1 || D >= M) return fail(DOA_ERR_INVALID_ARG, "doa_plan_create: D=%d outside [1, M-1]", D);
  if (!(d_over_lambda > 0.0) || !std::isfinite(d_over_lambda))
    return fail(DOA_ERR_INVALID_ARG, "doa_plan_create: d/lambda=%g must be positive and finite", d_over_lambda);
  if (L < 3 || L >= (int64_t)1 << 31) return fail(DOA_ERR_INVALID_ARG, "doa_plan_create: L=%lld outside [3, 2^31)", (long long)L);
  if (!(dtheta_deg > 0.0) || !std::isfinite(dtheta_deg))
    return fail(DOA_ERR_INVALID_ARG, "doa_plan_create: dtheta=%g must be positive", dtheta_deg);
  if (!(theta0_deg >= -90.0)) return fail(DOA_ERR_INVALID_ARG, "doa_plan_create: theta0=%g < -90", theta0_deg);
  if (!(theta0_deg + (double)(L - 1) * dtheta_deg <= 90.0 + 1e-9))
    return fail(DOA_ERR_INVALID_ARG, "doa_plan_create: grid end %g > 90", theta0_deg + (double)(L - 1) * dtheta_deg);
  if (alg < DOA_ALG_PHD || alg > DOA_ALG_MN) return fail(DOA_ERR_INVALID_ARG, "doa_plan_create: alg=%d", alg);
  if (max_batch < 1) return fail(DOA_ERR_INVALID_ARG, "doa_plan_create: max_batch=%lld < 1", (long long)max_batch);

  doa_plan_s* p = new doa_plan_s();
  std::memset(p, 0, sizeof *p);
  p->device = doa::current_device();
  p->M = M; p->D = D; p->alg = alg; p->dl = d_over_lambda; p->theta0 = theta0_deg; p->dtheta = dtheta_deg;
  p->L = L; p->max_batch = max_batch;
  // Q26: a grid whose last point (Q8 arithmetic) is exactly -theta0 is built from both ends and the
  // scan evaluates mirrored angle pairs together.  DOA_SCAN_MIRROR=0 (A/B and tests only) keeps
  // the symmetric grid but scans every angle separately.
  {
    volatile double end = (double)(L - 1) * dtheta_deg;   // rounded multiply, then rounded add (no FMA)
    end = end + theta0_deg;
    p->sym = (end == -theta0_deg) ? 1 : 0;
    const char* ev = std::getenv("DOA_SCAN_MIRROR");
    p->mirror = p->sym && !(ev && ev[0] == '0');
  }
  // interior minima of a degree-(M-1) trig polynomial over ceil(2 d/lambda) periods, x2 margin, >= 32
  int cap = 2 * ((M - 1) * (int)std::ceil(2.0 * d_over_lambda) + 1);
  cap = (cap + 31) & ~31;
  p->cap = cap;
  const size_t B = (size_t)max_batch;
  cudaError_t e = cudaSuccess;
  auto al = [&](void** ptr, size_t bytes) { if (e == cudaSuccess) e = cudaMalloc(ptr, bytes); };
  al((void**)&p->cnt, B * sizeof(int32_t));
  al((void**)&p->cand_idx, B * cap * sizeof(int32_t));
  al((void**)&p->cand_f, B * cap * sizeof(double));
  al((void**)&p->coef, doa::coef_words(max_batch, M) * sizeof(double));
  // the DMMA scan reads whole 8-frame groups: rows of frames past B in the last group must hold
  // defined values (their results are discarded)
  if (e == cudaSuccess) e = cudaMemset(p->coef, 0, doa::coef_words(max_batch, M) * sizeof(double));
  if (e != cudaSuccess) {
    doa_plan_destroy(p);
    return cuda_fail(e, "doa_plan_create: workspace allocation");
  }
  *plan = p;
  return DOA_OK;
}

doa_status_t doa_plan_create_array(doa_plan_t* plan, int32_t M, const double* positions, int32_t D, double az0_deg,
                                   double daz_deg, int64_t naz, double el0_deg, double del_deg, int64_t nel,
                                   int32_t az_wrap, int32_t alg, int64_t max_batch) {
  g_launches = 0;
  if (!plan) return fail(DOA_ERR_INVALID_ARG, "doa_plan_create_array: plan out-pointer is NULL");
  *plan = nullptr;
  if (M < 2) return fail(DOA_ERR_INVALID_ARG, "doa_plan_create_array: M=%d < 2", M);
  if (M > 16) return fail(DOA_ERR_UNSUPPORTED, "doa_plan_create_array: M=%d > 16", M);
  if (D < 1 || D >= M) return fail(DOA_ERR_INVALID_ARG, "doa_plan_create_array: D=%d outside [1, M-1]", D);
  if (!positions) return fail(DOA_ERR_INVALID_ARG, "doa_plan_create_array: positions is NULL");
  for (int i = 0; i < 3 * M; ++i)
    if (!std::isfinite(positions[i])) return fail(DOA_ERR_INVALID_ARG, "doa_plan_create_array: non-finite position");
  if (naz < 1 || nel < 1) return fail(DOA_ERR_INVALID_ARG, "doa_plan_create_array: naz, nel must be >= 1");
  const int64_t L = naz * nel;
  if (L < 3 || L >= (int64_t)1 << 31) return fail(DOA_ERR_INVALID_ARG, "doa_plan_create_array: L=%lld outside [3, 2^31)", (long long)L);
  if (!std::isfinite(az0_deg) || !std::isfinite(el0_deg) || !std::isfinite(daz_deg) || !std::isfinite(del_deg) ||
      (naz > 1 && !(daz_deg > 0.0)) || (nel > 1 && !(del_deg > 0.0)))
    return fail(DOA_ERR_INVALID_ARG, "doa_plan_create_array: grid steps must be positive and finite");
  if (alg < DOA_ALG_PHD || alg > DOA_ALG_MN) return fail(DOA_ERR_INVALID_ARG, "doa_plan_create_array: alg=%d", alg);
  if (max_batch < 1) return fail(DOA_ERR_INVALID_ARG, "doa_plan_create_array: max_batch < 1");

  doa_plan_s* p = new doa_plan_s();
  std::memset(p, 0, sizeof *p);
  p->device = doa::current_device();
  p->M = M; p->D = D; p->alg = alg; p->geom = 1;
  p->az0 = az0_deg; p->daz = daz_deg; p->naz = naz; p->el0 = el0_deg; p->del = del_deg; p->nel = nel;
  p->wrap = az_wrap ? 1 : 0;
  p->L = L; p->max_batch = max_batch;
  p->cap = 128;
  const int npair = M * (M - 1) / 2;
  std::vector<double> dp((size_t)3 * (npair > 0 ? npair : 1));
  for (int a = 0, k = 0; a < M; ++a)
    for (int b = a + 1; b < M; ++b, ++k)
      for (int c = 0; c < 3; ++c) dp[3 * k + c] = positions[3 * b + c] - positions[3 * a + c];   // r_q - r_p
  const size_t B = (size_t)max_batch;
  const size_t kw = (size_t)((max_batch + 7) / 8) * doa::array_ksteps(M) * 32;
  cudaError_t e = cudaSuccess;
  auto al = [&](void** ptr, size_t bytes) { if (e == cudaSuccess) e = cudaMalloc(ptr, bytes); };
  al((void**)&p->cnt, B * sizeof(int32_t));
  al((void**)&p->cand_idx, B * p->cap * sizeof(int32_t));
  al((void**)&p->cand_f, B * p->cap * sizeof(double));
  al((void**)&p->coef, kw * sizeof(double));
  if (e == cudaSuccess) e = cudaMemset(p->coef, 0, kw * sizeof(double));   // partial last 8-frame group
  al((void**)&p->dpos, dp.size() * sizeof(double));
  al((void**)&p->fbuf, B * (size_t)L * sizeof(double));
  if (e == cudaSuccess) e = cudaMemcpy(p->dpos, dp.data(), dp.size() * sizeof(double), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    doa_plan_destroy(p);
    return cuda_fail(e, "doa_plan_create_array: workspace allocation");
  }
  *plan = p;
  return DOA_OK;
}

doa_status_t doa_plan_destroy(doa_plan_t p) {
  if (!p) return DOA_OK;
  const int cur = doa::current_device();
  const int dev = p->device;
  if (cur != dev) cudaSetDevice(dev);                   // free on the plan's device
  cudaDeviceSynchronize();
  cudaFree(p->dpos); cudaFree(p->fbuf); cudaFree(p->x32);
  cudaFree(p->cnt); cudaFree(p->cand_idx); cudaFree(p->cand_f); cudaFree(p->coef);
  cudaFree(p->R); cudaFree(p->lam); cudaFree(p->V); cudaFree(p->cov_ws);
  cudaFree(p->dX[0]); cudaFree(p->dX[1]); cudaFree(p->d_out);
  if (p->copy_stream) cudaStreamDestroy(p->copy_stream);
  for (int k = 0; k < 2; ++k) {
    if (p->ev_copied[k]) cudaEventDestroy(p->ev_copied[k]);
    if (p->ev_used[k]) cudaEventDestroy(p->ev_used[k]);
  }
  delete p;
  if (cur != dev) cudaSetDevice(cur);
  return DOA_OK;
}

int32_t doa_plan_capacity(doa_plan_t p) { return p ? p->cap : 0; }

doa_status_t doa_plan_info(doa_plan_t p, doa_plan_info_t* out) {
  if (!p) return fail(DOA_ERR_INVALID_ARG, "doa_plan_info: plan is NULL");
  if (!out) return fail(DOA_ERR_INVALID_ARG, "doa_plan_info: out is NULL");
  out->M = p->M; out->D = p->D; out->alg = p->alg; out->geom = p->geom; out->device = p->device;
  out->capacity = p->cap; out->L = p->L; out->max_batch = p->max_batch;
  out->engine = p->engine; out->reserved = 0;
  return DOA_OK;
}

doa_status_t doa_plan_set_engine(doa_plan_t p, int32_t engine) {
  g_launches = 0;
  DOA_CHECK_PLAN(p);
  if (engine != DOA_ENGINE_TOEPLITZ_FP64 && engine != DOA_ENGINE_DIRECT_FP32 && engine != DOA_ENGINE_DIRECT_TF32X3)
    return fail(DOA_ERR_INVALID_ARG, "doa_plan_set_engine: unknown engine %d", engine);
  if (p->geom != 0) return fail(DOA_ERR_UNSUPPORTED, "doa_plan_set_engine: general-array plans have one engine");
  if (engine != DOA_ENGINE_TOEPLITZ_FP64) {
    if (p->M > 16) return fail(DOA_ERR_UNSUPPORTED, "doa_plan_set_engine: the direct-form engines support M <= 16 (M=%d)", p->M);
    if (!p->x32)
      DOA_TRY(cudaMalloc((void**)&p->x32, (size_t)p->max_batch * (p->M - p->D) * p->M * 2 * sizeof(float)),
              "doa_plan_set_engine: vectors");
  }
  p->engine = engine;
  p->coef_B = 0;                                        // coefficients of the other engine are stale
  p->last_B = 0;
  return DOA_OK;
}

doa_status_t doa_covariance(doa_plan_t p, const float* X, int64_t B, int64_t N, double* R, doa_stream_t s) {
  g_launches = 0;
  DOA_CHECK_PLAN(p);
  DOA_CHECK_B(p, B);
  if (N < 1) return fail(DOA_ERR_INVALID_ARG, "doa_covariance: N=%lld < 1", (long long)N);
  if (B == 0) return DOA_OK;
  DOA_CHECK_PTR(X, 8);
  DOA_CHECK_PTR(R, 16);
  DOA_TRY(doa::launch_covariance(X, B, N, p->M, R, (cudaStream_t)s), "doa_covariance");
  return DOA_OK;
}

doa_status_t doa_eig(doa_plan_t p, const double* R, int64_t B, double* lambda, double* V, int32_t* info,
                     doa_stream_t s) {
  g_launches = 0;
  DOA_CHECK_PLAN(p);
  DOA_CHECK_B(p, B);
  if (B == 0) return DOA_OK;
  DOA_CHECK_PTR(R, 16);
  DOA_CHECK_PTR(lambda, 8);
  DOA_CHECK_PTR(V, 16);
  DOA_CHECK_PTR(info, 4);
  DOA_TRY(doa::launch_eig(R, B, p->M, lambda, V, info, (cudaStream_t)s), "doa_eig");
  return DOA_OK;
}

doa_status_t doa_spectrum(doa_plan_t p, const double* lambda, const double* V, int64_t B, float* P, int32_t* info,
                          doa_stream_t s) {
  g_launches = 0;
  DOA_CHECK_PLAN(p);
  DOA_CHECK_B(p, B);
  if (B == 0) { p->last_B = 0; return DOA_OK; }
  DOA_CHECK_PTR(lambda, 8);
  DOA_CHECK_PTR(V, 16);
  DOA_CHECK_PTR(info, 4);
  if (P && !aligned(P, 4)) return fail(DOA_ERR_INVALID_ARG, "doa_spectrum: P is not 4-byte aligned");
  DOA_TRY(spectrum_stage(p, lambda, V, B, P, info, (cudaStream_t)s), "doa_spectrum");
  p->last_B = B;
  p->coef_B = p->geom == 0 ? B : 0;
  return DOA_OK;
}

doa_status_t doa_peaks(doa_plan_t p, int64_t B, int32_t* idx, float* val, int32_t* npk, int32_t* info,
                       doa_stream_t s) {
  g_launches = 0;
  DOA_CHECK_PLAN(p);
  DOA_CHECK_B(p, B);
  if (B != p->last_B)
    return fail(DOA_ERR_INVALID_ARG, "doa_peaks: B=%lld differs from the preceding doa_spectrum (B=%lld)",
                (long long)B, (long long)p->last_B);
  if (B == 0) return DOA_OK;
  DOA_CHECK_PTR(idx, 4);
  DOA_CHECK_PTR(val, 4);
  DOA_CHECK_PTR(npk, 4);
  DOA_CHECK_PTR(info, 4);
  DOA_TRY(doa::launch_select(p, B, idx, val, npk, info, (cudaStream_t)s), "doa_peaks");
  return DOA_OK;
}

doa_status_t doa_run(doa_plan_t p, const float* X, int64_t B, int64_t N, int32_t* idx, float* val, int32_t* npk,
                     float* P, int32_t* info, doa_stream_t s) {
  g_launches = 0;
  DOA_CHECK_PLAN(p);
  DOA_CHECK_B(p, B);
  if (N < 1) return fail(DOA_ERR_INVALID_ARG, "doa_run: N=%lld < 1", (long long)N);
  if (B == 0) return DOA_OK;
  DOA_CHECK_PTR(X, 8);
  DOA_CHECK_PTR(idx, 4);
  DOA_CHECK_PTR(val, 4);
  DOA_CHECK_PTR(npk, 4);
  DOA_CHECK_PTR(info, 4);
  if (P && !aligned(P, 4)) return fail(DOA_ERR_INVALID_ARG, "doa_run: P is not 4-byte aligned");
  DOA_TRY(ensure_run_scratch(p), "doa_run: scratch allocation");
  DOA_TRY(run_plans(&p, 1, X, B, N, idx, val, npk, info, B, (cudaStream_t)s, nullptr, P), "doa_run");
  return DOA_OK;
}

doa_status_t doa_run_multi(const doa_plan_t* plans, int32_t nplans, const float* X, int64_t B, int64_t N,
                           int32_t* idx, float* val, int32_t* npk, int32_t* info, doa_stream_t s) {
  g_launches = 0;
  const doa_status_t st = check_plan_set("doa_run_multi", plans, nplans, B);
  if (st != DOA_OK) return st;
  if (N < 1) return fail(DOA_ERR_INVALID_ARG, "doa_run_multi: N=%lld < 1", (long long)N);
  if (B == 0) return DOA_OK;
  DOA_CHECK_PTR(X, 8);
  DOA_CHECK_PTR(idx, 4);
  DOA_CHECK_PTR(val, 4);
  DOA_CHECK_PTR(npk, 4);
  DOA_CHECK_PTR(info, 4);
  DOA_TRY(ensure_run_scratch(plans[0]), "doa_run_multi: scratch allocation");
  DOA_TRY(run_plans(plans, nplans, X, B, N, idx, val, npk, info, B, (cudaStream_t)s), "doa_run_multi");
  return DOA_OK;
}

doa_status_t doa_scan_multi(const doa_plan_t* plans, int32_t nplans, int64_t B, doa_stream_t s) {
  g_launches = 0;
  const doa_status_t st = check_plan_set("doa_scan_multi", plans, nplans, B);
  if (st != DOA_OK) return st;
  if (nplans > doa::kMaxCoefPlans)
    return fail(DOA_ERR_INVALID_ARG, "doa_scan_multi: nplans=%d > %d", nplans, doa::kMaxCoefPlans);
  for (int a = 0; a < nplans; ++a) {
    if (plans[a]->geom != 0) return fail(DOA_ERR_UNSUPPORTED, "doa_scan_multi: plans[%d] is a general-array plan", a);
    if (a > 0 && !doa::direct_compatible(plans[a], plans[0]))
      return fail(DOA_ERR_INVALID_ARG, "doa_scan_multi: plans[%d] does not share the grid of plans[0]", a);
    if (plans[a]->engine != plans[0]->engine)
      return fail(DOA_ERR_INVALID_ARG, "doa_scan_multi: plans[%d] uses another scan engine than plans[0]", a);
    if (B > plans[a]->coef_B)
      return fail(DOA_ERR_INVALID_ARG, "doa_scan_multi: plans[%d] holds coefficients for %lld frames, B=%lld", a,
                  (long long)plans[a]->coef_B, (long long)B);
  }
  if (B == 0) return DOA_OK;
  cudaStream_t st2 = (cudaStream_t)s;
  const doa_plan_s* grp[doa::kMaxCoefPlans] = {};
  for (int a = 0; a < nplans; ++a) {
    grp[a] = plans[a];
    DOA_TRY(cudaMemsetAsync(plans[a]->cnt, 0, (size_t)B * sizeof(int32_t), st2), "doa_scan_multi: counters");
  }
  if (plans[0]->engine != DOA_ENGINE_TOEPLITZ_FP64) {
    for (int a = 0; a < nplans; ++a) DOA_TRY(doa::launch_scan_direct_form(plans[a], B, nullptr, st2), "doa_scan_multi");
  } else {
    DOA_TRY(doa::launch_scan_plans(grp, nplans, B, nullptr, st2), "doa_scan_multi");
  }
  for (int a = 0; a < nplans; ++a) plans[a]->last_B = B;
  return DOA_OK;
}

doa_status_t doa_run_host(const doa_plan_t* plans, int32_t nplans, const float* X_host, int64_t B, int64_t N,
                          int32_t* idx_host, float* val_host, int32_t* npk_host, int32_t* info_host,
                          doa_stream_t s) {
  {
    const doa_status_t st0 = check_plan_set("doa_run_host", plans, nplans, B);
    if (st0 != DOA_OK) return st0;
  }
  doa_plan_s* p = plans[0];
  if (N < 1) return fail(DOA_ERR_INVALID_ARG, "doa_run_host: N=%lld < 1", (long long)N);
  if (B == 0) return DOA_OK;
  if (!X_host || !idx_host || !val_host || !npk_host || !info_host)
    return fail(DOA_ERR_INVALID_ARG, "doa_run_host: NULL host pointer");
  cudaStream_t st = (cudaStream_t)s;
  const int M = p->M, D = p->D;
  // chunk of frames per H2D copy: ~128 MiB, at most B
  const size_t frame_bytes = (size_t)N * M * 2 * sizeof(float);
  int64_t chunk = (int64_t)((128u << 20) / frame_bytes);
  if (chunk < 1) chunk = 1;
  if (chunk > B) chunk = B;
  const size_t need = (size_t)chunk * frame_bytes;
  DOA_TRY(ensure_run_scratch(p), "doa_run_host: scratch allocation");
  if (p->dX_bytes < need) {
    cudaFree(p->dX[0]); cudaFree(p->dX[1]);
    p->dX[0] = p->dX[1] = nullptr;
    p->dX_bytes = 0;
    DOA_TRY(cudaMalloc((void**)&p->dX[0], need), "doa_run_host: staging");
    DOA_TRY(cudaMalloc((void**)&p->dX[1], need), "doa_run_host: staging");
    p->dX_bytes = need;
  }
  const size_t out_words = (size_t)nplans * p->max_batch * (2 * D + 2);
  if (p->d_out_words < out_words) {
    cudaFree(p->d_out);
    p->d_out = nullptr;
    p->d_out_words = 0;
    DOA_TRY(cudaMalloc((void**)&p->d_out, out_words * sizeof(int32_t)), "doa_run_host: outputs");
    p->d_out_words = out_words;
  }
  if (!p->copy_stream) {
    DOA_TRY(cudaStreamCreateWithFlags(&p->copy_stream, cudaStreamNonBlocking), "doa_run_host: stream");
    for (int k = 0; k < 2; ++k) {
      DOA_TRY(cudaEventCreateWithFlags(&p->ev_copied[k], cudaEventDisableTiming), "doa_run_host: event");
      DOA_TRY(cudaEventCreateWithFlags(&p->ev_used[k], cudaEventDisableTiming), "doa_run_host: event");
    }
    // buffers start "free"
    for (int k = 0; k < 2; ++k) DOA_TRY(cudaEventRecord(p->ev_used[k], st), "doa_run_host: record");
  }
  int32_t* d_idx = p->d_out;                                              // [nplans][B][D]
  float* d_val = reinterpret_cast<float*>(d_idx + (size_t)nplans * B * D);  // [nplans][B][D]
  int32_t* d_npk = reinterpret_cast<int32_t*>(d_val + (size_t)nplans * B * D);  // [nplans][B]
  int32_t* d_info = d_npk + (size_t)nplans * B;                           // [nplans][B]
  int launches = 0;
  int k = 0;
  for (int64_t b0 = 0; b0 < B; b0 += chunk, k ^= 1) {
    const int64_t nb = (b0 + chunk <= B) ? chunk : B - b0;
    // the copy into buffer k may start once the compute that last read it has finished
    DOA_TRY(cudaStreamWaitEvent(p->copy_stream, p->ev_used[k], 0), "doa_run_host: wait");
    DOA_TRY(cudaMemcpyAsync(p->dX[k], X_host + (size_t)b0 * N * M * 2, (size_t)nb * frame_bytes,
                            cudaMemcpyHostToDevice, p->copy_stream), "doa_run_host: H2D");
    DOA_TRY(cudaEventRecord(p->ev_copied[k], p->copy_stream), "doa_run_host: record");
    DOA_TRY(cudaStreamWaitEvent(st, p->ev_copied[k], 0), "doa_run_host: wait");
    g_launches = 0;
    DOA_TRY(run_plans(plans, nplans, p->dX[k], nb, N, d_idx + (size_t)b0 * D, d_val + (size_t)b0 * D, d_npk + b0,
                      d_info + b0, B, st, p->ev_used[k]), "doa_run_host/run");
    launches += g_launches;
  }
  for (int a = 0; a < nplans; ++a) plans[a]->last_B = plans[a]->coef_B = 0;
  const size_t nBD = (size_t)nplans * B * D, nB = (size_t)nplans * B;
  DOA_TRY(cudaMemcpyAsync(idx_host, d_idx, nBD * sizeof(int32_t), cudaMemcpyDeviceToHost, st), "D2H");
  DOA_TRY(cudaMemcpyAsync(val_host, d_val, nBD * sizeof(float), cudaMemcpyDeviceToHost, st), "D2H");
  DOA_TRY(cudaMemcpyAsync(npk_host, d_npk, nB * sizeof(int32_t), cudaMemcpyDeviceToHost, st), "D2H");
  DOA_TRY(cudaMemcpyAsync(info_host, d_info, nB * sizeof(int32_t), cudaMemcpyDeviceToHost, st), "D2H");
  DOA_TRY(cudaStreamSynchronize(st), "doa_run_host: sync");
  g_launches = launches;
  return DOA_OK;
}

}  // extern "C"
