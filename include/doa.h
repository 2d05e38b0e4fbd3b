/*
 * doa.h — C ABI of the B200-native noise-subspace DOA hot path (libdoa.so).
 *
 * Method: Eray & Temizel, arXiv 2007.14135, "Performance Analysis of Noise Subspace-based
 * Narrowband DOA Estimation Algorithms on CPU and GPU".  Citations "P:n" are lines of the
 * paper text; "Qn" are the readings of silent/ambiguous points listed in
 * DESIGN.md §2.
 *
 * Problem statement: an M-element uniform linear array with
 * spacing d (ratio d/lambda), D known narrowband sources, N snapshots X per frame and a scan
 * grid theta_i = theta0 + i*dtheta (degrees from broadside, i in [0, L)).  Per frame return the
 * pseudo-spectrum P(theta_i) = 1 / (a(theta_i)^H C a(theta_i)) of one of PHD / MUSIC / EV / MN
 * and its D strongest local maxima (the DOA estimates), with the steering vector
 * a_m(theta) = exp(-j*2*pi*(d/lambda)*m*sin(theta)), m = 0..M-1 (Q6).
 *
 * Conventions shared by every call
 *  - Every data pointer is a DEVICE pointer owned by the caller (e.g. a torch CUDA tensor),
 *    except in doa_run_host, whose X/outputs are HOST pointers.  Complex numbers are
 *    interleaved (re, im): complex64 = 2 x float (8-byte aligned), complex128 = 2 x double
 *    (16-byte aligned).  All arrays are dense row-major.
 *  - Calls are asynchronous: they validate their arguments on the host, enqueue kernels on
 *    `stream` and return.  Only doa_plan_create / doa_plan_destroy / doa_run_host synchronise.
 *  - Invalid arguments return DOA_ERR_INVALID_ARG (or DOA_ERR_UNSUPPORTED) synchronously and
 *    enqueue nothing.  A CUDA launch / allocation failure returns DOA_ERR_CUDA /
 *    DOA_ERR_OUT_OF_MEMORY; doa_last_error() gives the detail (thread-local).
 *  - B == 0 is valid and enqueues nothing.
 *  - Per-frame numerical conditions never fail a call; they set bits of the caller's
 *    info[b] (DOA_INFO_*): doa_eig overwrites info[b]; doa_spectrum and doa_peaks OR into it.
 *  - A plan belongs to the CUDA device that was current when it was created; every call on it
 *    must be made with that device current, else DOA_ERR_INVALID_ARG (nothing enqueued).
 *  - A plan owns only its workspace (candidate lists and, for doa_run, R / lambda / V /
 *    coefficient scratch for max_batch frames).  One plan must not be used from two streams
 *    at once; doa_peaks consumes the candidates written by the preceding doa_spectrum on the
 *    same plan, in stream order.
 *  - Arithmetic: fp32 inputs, fp64 everywhere inside; P and peak values are
 *    reported in fp32, saturating at FLT_MAX (Q12).
 */
#ifndef DOA_H_
#define DOA_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct doa_plan_s* doa_plan_t;
typedef struct CUstream_st* doa_stream_t;   /* == cudaStream_t; NULL = legacy default stream */

/* Table 3: the four noise-subspace estimators. */
typedef enum {
  DOA_ALG_PHD = 0,    /* C = e_min e_min^H                         (Table 3) */
  DOA_ALG_MUSIC = 1,  /* C = E_n E_n^H          */
  DOA_ALG_EV = 2,     /* C = sum_k (1/lambda_k) e_k e_k^H  (Q1)          */
  DOA_ALG_MN = 3      /* C = w w^H, w = P_n e1 / (e1^H P_n e1)     (Q5)      */
} doa_alg_t;

typedef enum {
  DOA_OK = 0,
  DOA_ERR_INVALID_ARG = 1,
  DOA_ERR_UNSUPPORTED = 2,
  DOA_ERR_OUT_OF_MEMORY = 3,
  DOA_ERR_CUDA = 4
} doa_status_t;

enum {
  DOA_INFO_NOCONV = 1,          /* Jacobi hit 30 sweeps; outputs are the last iterate (Q15)     */
  DOA_INFO_DEGENERATE = 2,      /* EV noise eigenvalue <= 100 eps lambda_max (clamped), or MN
                                   e1^H P_n e1 <= 100 eps (w = P_n e1 unnormalised)             */
  DOA_INFO_CAND_OVERFLOW = 4,   /* more local maxima than the plan's candidate capacity; the
                                   peaks are chosen from the first `capacity` found             */
  DOA_INFO_UNDERDETERMINED = 8  /* fewer than D local maxima (npk < D; padding -1 / 0)          */
};

/* Create a plan.  M in [2, 64] (M > 64: DOA_ERR_UNSUPPORTED); 1 <= D < M; d_over_lambda > 0;
 * grid theta_i = theta0_deg + i*dtheta_deg (multiply then add, round-to-nearest; Q8) for i in
 * [0, L), 3 <= L < 2^31, dtheta_deg > 0, theta0_deg >= -90, theta0_deg + (L-1)*dtheta_deg <=
 * 90 (+1e-9); alg a doa_alg_t; max_batch >= 1 frames per call.  Allocates the workspace
 * (synchronous).  On failure *plan is set to NULL. */
doa_status_t doa_plan_create(doa_plan_t* plan, int32_t M, double d_over_lambda, int32_t D,
                             double theta0_deg, double dtheta_deg, int64_t L, int32_t alg,
                             int64_t max_batch);

/* General array geometry on an azimuth x elevation grid (the paper's own UCA
 * workload).  positions: HOST double [M][3], element coordinates in
 * wavelengths; steering is Eq. 2, a_k = exp{ j 2 pi (x_k sin(az) sin(el) + y_k cos(az)
 * sin(el) + z_k cos(el)) } with el measured from +z (el = 90 deg is the xy plane; the paper's
 * naming).  Grid az_i = az0 + i*daz (i < naz), el_j = el0 + j*del (j < nel), flattened
 * azimuth-major p = i*nel + j; L = naz*nel in [3, 2^31).  az_wrap != 0: azimuth neighbours wrap
 * (a full 360-degree azimuth range).  M in [2, 16] (M > 16: DOA_ERR_UNSUPPORTED); 1 <= D < M.
 * doa_covariance / doa_eig are as for ULA plans; doa_spectrum computes f on the grid (P, when
 * given, is float [B][naz][nel]) and the 2-D local maxima of P (8-neighbourhood; a neighbour
 * earlier in raster order must be strictly larger in f, a later one larger or equal; neighbours
 * outside the grid are ignored — DESIGN.md G2); doa_peaks returns raster indices p.  Allocates an
 * fp64 spectrum buffer of max_batch * L doubles. */
doa_status_t doa_plan_create_array(doa_plan_t* plan, int32_t M, const double* positions, int32_t D,
                                   double az0_deg, double daz_deg, int64_t naz, double el0_deg,
                                   double del_deg, int64_t nel, int32_t az_wrap, int32_t alg,
                                   int64_t max_batch);

/* Free the plan and its workspace (synchronises the device).  NULL is a no-op. */
doa_status_t doa_plan_destroy(doa_plan_t plan);

/* Number of candidate slots per frame the plan reserves (>= 2*((M-1)*ceil(2 d/lambda)+1)). */
int32_t doa_plan_capacity(doa_plan_t plan);

/* The plan's parameters, for callers that validate their buffers against it (the Python binding
 * does): M, D, alg, geom (0 = ULA, 1 = general array), the CUDA device ordinal the plan (and its
 * workspace) belongs to, candidate capacity, L (grid points) and max_batch.  Host-only, no
 * synchronisation.  NULL plan or out -> DOA_ERR_INVALID_ARG. */
typedef struct {
  int32_t M, D, alg, geom, device, capacity;
  int64_t L, max_batch;
  int32_t engine, reserved;       /* DOA_ENGINE_* (doa_plan_set_engine) */
} doa_plan_info_t;
doa_status_t doa_plan_info(doa_plan_t plan, doa_plan_info_t* out);

/* Scan engines of a ULA plan.  Step-5 (Table 2) evaluates
 * f = a^H C a with C the Step-4 noise-subspace form (Table 3):
 *   DOA_ENGINE_TOEPLITZ_FP64 (default, the product): C reduced to its Toeplitz sums c_k, f as an
 *     fp64 contraction with a per-angle table on the FP64 tensor pipe (DMMA) — DESIGN.md §5, §7;
 *   DOA_ENGINE_DIRECT_FP32: the paper's own direct form f = sum_j |x_j^H a|^2 over the weighted
 *     noise vectors x_j = sqrt(w_j) e_j (MN: the normalised w; PHD: e_min), one thread per angle
 *     as in §4.3, every product and sum on the FP32 pipe (vectors and steering formed in
 *     fp64 and rounded to fp32; north_star's "FP32-pipe sincos+FMA" alternative);
 *   DOA_ENGINE_DIRECT_TF32X3: the same direct form as a GEMM on the 5th-generation tensor cores
 *     (tcgen05.mma kind::tf32 with TMEM accumulators; every fp32 operand split into tf32 head and
 *     tail, three products: ~fp32 accuracy).  Both direct-form engines are A/B
 *     engine for evidence: several times slower than the Toeplitz contraction at c4, and its fp32
 *     rounding can move peak indices and exceed 1e-3 dB near deep nulls
 *     (tests/test_gpu_fp32_engine.py).
 * doa_spectrum / doa_run / doa_run_multi / doa_run_host / doa_scan_multi of the plan then use the
 * engine (doa_run_multi keeps the eigendecomposition shared; the frame kernel is used only when
 * every plan is Toeplitz).  The fp32 engine allocates max_batch*(M-D)*M complex64 (synchronous).
 * Errors: NULL plan or unknown engine -> DOA_ERR_INVALID_ARG; general-array plans, or
 * a direct-form engine with M > 16 -> DOA_ERR_UNSUPPORTED; allocation failure ->
 * DOA_ERR_OUT_OF_MEMORY.  Must not be called while work on the plan is in flight. */
enum { DOA_ENGINE_TOEPLITZ_FP64 = 0, DOA_ENGINE_DIRECT_FP32 = 1, DOA_ENGINE_DIRECT_TF32X3 = 2 };
doa_status_t doa_plan_set_engine(doa_plan_t plan, int32_t engine);

/* S1 — sample covariance, Eq. 3 / Table 2 Step-1:
 *   R[b] = (1/N) sum_n x_b[n] x_b[n]^H   (1/N, Q20).
 * X: complex64 [B][N][M] (snapshot-major: x_m[n] of frame b at X[(b*N+n)*M+m]).
 * R: complex128 [B][M][M], full Hermitian, real diagonal.  fp32 products are exact in fp64;
 * sums are accumulated in fp64 in a fixed order (deterministic).  N >= 1, 1 <= B <= max_batch. */
doa_status_t doa_covariance(doa_plan_t plan, const float* X, int64_t B, int64_t N, double* R,
                            doa_stream_t stream);

/* S2 — Hermitian eigendecomposition of R (Table 2 Step-2 `jsvd`; Q3), one warp per matrix,
 * parallel (round-robin) cyclic Jacobi in fp64.  Only the upper triangle of R[b] is read.
 * Stop when off(A) <= 10 eps ||R||_F (off computed directly), at most 30 sweeps (Q15).
 * lambda: double [B][M] ascending (stable, Q2).  V: complex128 [B][M][M], column j (V[b][i][j],
 * i = 0..M-1) is the unit eigenvector of lambda[b][j].  info[b] is OVERWRITTEN (NOCONV or 0). */
doa_status_t doa_eig(doa_plan_t plan, const double* R, int64_t B, double* lambda, double* V,
                     int32_t* info, doa_stream_t stream);

/* S3-S6 — noise subspace (Table 3 Step-3), Step-4 form C reduced to its Toeplitz diagonal sums
 * c_k = sum_p C[p][p+k], pseudo-spectrum scan over the plan's grid
 * (Table 2 Step-5) f_i = a_i^H C a_i = c_0 + 2 sum_k Re(c_k e^{-j pi k u_i}),
 * u_i = 2 (d/lambda) sin(theta_i), floored at 1e-300 (Q12), and local-maximum candidate
 * detection (Step-6 findPeaks; Q9/Q10) into the plan's candidate lists.
 * lambda/V as produced by doa_eig.  P: NULL, or float [B][L] receiving 1/f_i (fp32, saturating).
 * info[b] |= DEGENERATE where applicable.  Batches of B > 16 frames run the scan as an FP64
 * tensor-core (DMMA) contraction; B <= 16 runs the direct scan (steering generated once per angle
 * in registers, csrc/scan_direct.cu), which rounds differently (both within the parity bars). */
doa_status_t doa_spectrum(doa_plan_t plan, const double* lambda, const double* V, int64_t B,
                          float* P, int32_t* info, doa_stream_t stream);

/* S7 — PeakSelection (Table 2 Step-6; Q11): per frame order the plan's candidates by
 * (f ascending, index ascending) and keep min(D, count).  idx: int32 [B][D] grid indices (-1
 * padding), val: float [B][D] = 1/f (0 padding), npk: int32 [B].  info[b] |= CAND_OVERFLOW,
 * UNDERDETERMINED.  B must equal the preceding doa_spectrum's B. */
doa_status_t doa_peaks(doa_plan_t plan, int64_t B, int32_t* idx, float* val, int32_t* npk,
                       int32_t* info, doa_stream_t stream);

/* S1-S7 fused: X (device, as doa_covariance) -> idx/val/npk/info (device, as doa_peaks),
 * P nullable (as doa_spectrum).  info[b] is overwritten.  Uses plan scratch for R, lambda, V
 * (max_batch frames), allocated by the first doa_run / doa_run_host on the plan (that first call
 * synchronises the device once). */
doa_status_t doa_run(doa_plan_t plan, const float* X, int64_t B, int64_t N, int32_t* idx,
                     float* val, int32_t* npk, float* P, int32_t* info, doa_stream_t stream);

/* S1-S7 for several plans on one batch, device buffers: nplans >= 1 distinct plans that share M
 * and D (typically PHD, MUSIC, EV and MN on one grid).  X as doa_covariance; the covariance and
 * the eigendecomposition run once (in plans[0]'s scratch), then every plan's S3-S7; outputs per
 * plan a: idx int32 [nplans][B][D], val float [nplans][B][D], npk int32 [nplans][B], info int32
 * [nplans][B] (overwritten), all device pointers.  For small batches (B <= 16) plans that share
 * the grid (M, d/lambda, theta0, dtheta, L) are evaluated by ONE direct scan launch that generates
 * the steering once per angle for all of them (csrc/scan_direct.cu) — the non-tensor-core path
 * for single frames; larger batches use the FP64 tensor-core (DMMA) contraction per plan.  The
 * two paths round differently (both within the parity bars), so a frame's P can differ in the
 * last bits between a batch of <= 16 and a larger one.  Per-plan candidate lists are left for
 * doa_peaks as after doa_spectrum.  Errors as doa_run; the plans must be distinct, created on the
 * current device, with max_batch >= B. */
doa_status_t doa_run_multi(const doa_plan_t* plans, int32_t nplans, const float* X, int64_t B,
                           int64_t N, int32_t* idx, float* val, int32_t* npk, int32_t* info,
                           doa_stream_t stream);

/* S4-S6 again, for 1..4 ULA plans that share M, d/lambda and the grid (typically the four
 * estimators), from the Toeplitz coefficients each plan holds from its most recent doa_spectrum,
 * doa_run or doa_run_multi call (covering at least B frames): the pseudo-spectrum scan and the
 * local-maximum candidates (Table 2 Step-5/6) exactly as those calls run them (B <= 16:
 * one direct-scan launch for all the plans; otherwise one FP64 tensor-core scan launch per plan).
 * The plans' candidate lists are reset and rebuilt, so doa_peaks on each plan afterwards returns
 * what the producing call returned.  Used to re-scan and to time the scan stage on its own
 * (bench.py's roofline).  Errors: general-array
 * plans -> DOA_ERR_UNSUPPORTED; plans that differ in the grid, nplans > 4, or B above the frames
 * the plans hold coefficients for -> DOA_ERR_INVALID_ARG (nothing enqueued). */
doa_status_t doa_scan_multi(const doa_plan_t* plans, int32_t nplans, int64_t B, doa_stream_t stream);

/* End-to-end variant of doa_run with HOST buffers, for nplans >= 1 plans that share M and D
 * (typically the four estimators): X_host complex64 [B][N][M] is copied host->device in chunks
 * on a second stream into device staging owned by plans[0], overlapping each chunk's copy with
 * the compute of the previous chunk; per chunk S1-S2 run once and S3-S7 once per plan; the
 * peak lists come back to the host outputs idx_host int32 [nplans][B][D], val_host float
 * [nplans][B][D], npk_host int32 [nplans][B], info_host int32 [nplans][B].  Synchronises
 * `stream` before returning.  X_host should be pinned (page-locked) for asynchronous copies;
 * pageable memory is accepted and copied synchronously by the driver.  The staging buffers are
 * allocated on first use (and grown if a later call needs more). */
doa_status_t doa_run_host(const doa_plan_t* plans, int32_t nplans, const float* X_host, int64_t B,
                          int64_t N, int32_t* idx_host, float* val_host, int32_t* npk_host,
                          int32_t* info_host, doa_stream_t stream);

/* On-device synthetic snapshots of the signal model Eq. 1:
 * X = A(theta) S + W for the ULA a_m(theta) = exp(-j*pi*m*u), u = 2*(d/lambda)*sin(theta) (Q6), with
 * D uncorrelated unit-power CN(0,1) sources and CN(0, sigma^2) noise, sigma^2 = 10^(-snr_db/10)
 * (Q13, Q14).  Randomness is counter-based (Philox4x32-10, key = seed): sample k of snapshot n of
 * frame f (k < D: source k, else the noise of element k - D) comes from counter (k/2, n, f_lo,
 * f_hi) and Box-Muller in fp64, so every frame is reproducible on its own and independent of B,
 * frame0 and the launch configuration (synth/philox.py is the same generator in numpy).
 *  theta_deg  DEVICE double, [D] (theta_per_frame = 0: same DOAs for every frame) or [B][D]
 *             (theta_per_frame = 1), degrees from broadside.
 *  frame0     global index of the first frame (frames frame0 .. frame0+B-1 are generated).
 *  X          DEVICE complex64 [B][N][M] (output, overwritten).
 * Errors: M < 1, M > 64, D < 1, D > 63, N < 1, N > 2^24, B >= 2^31, d_over_lambda <= 0, non-finite snr_db, NULL or
 * misaligned pointers -> DOA_ERR_INVALID_ARG (nothing enqueued).  Asynchronous on `stream`.
 * Test-input machinery, not part of the estimator: the hot path never calls it. */
doa_status_t doa_generate(int32_t M, double d_over_lambda, int32_t D, const double* theta_deg,
                          int32_t theta_per_frame, double snr_db, uint64_t seed, int64_t frame0,
                          int64_t B, int64_t N, float* X, doa_stream_t stream);

/* Kernel launches the most recent call on this thread enqueued (for launch accounting). */
int32_t doa_last_launch_count(void);

const char* doa_status_string(doa_status_t status);
const char* doa_last_error(void);
int32_t doa_version(void);

#ifdef __cplusplus
}
#endif

#endif /* DOA_H_ */
