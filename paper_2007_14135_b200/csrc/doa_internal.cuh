// Internal declarations shared by the libdoa translation units (not part of the ABI).
#pragma once

#include <cuda_runtime.h>
#include <cfloat>
#include <cstdint>

#include "../../include/doa.h"

namespace doa {

constexpr int kMaxM = 64;
constexpr int kMaxSweeps = 30;          // Q15
constexpr double kFloor = 1e-300;       // Q12

// Coefficient vector per frame, K = 4*S entries in two k-step-aligned halves, S = SE + SO k-steps of
// 4 with SE = ceil(M/4) (even part) and SO = ceil((M-1)/4) (odd part); SE = (S+1)/2 for every M:
//   coef[0]             = c_0                 (real; trace of C)
//   coef[k]             = 2 Re c_k, k = 1..M-1 (multiplies cos(k psi))        j <  4 SE: even part
//   coef[4 SE + k - 1]  = 2 Im c_k, k = 1..M-1 (multiplies sin(k psi))        j >= 4 SE: odd part
//   every other j       = 0                    (padding)
// so that f(psi) = E(psi) + O(psi), E = sum_{j<4SE} coef[j] T_j(psi) even in psi and
// O = sum_{j>=4SE} coef[j] T_j(psi) odd in psi, with T = (1, cos psi..cos (M-1)psi, 0.., sin psi..
// sin (M-1)psi, 0..) and psi = pi u, u = 2 (d/lambda) sin(theta).  c_k = sum_p C[p][p+k] (DESIGN.md
// §5).  On a symmetric grid (Q26) the mirrored angle has psi -> -psi, so f = E - O there: one
// contraction serves both angles of a mirrored pair.
// Stored in the DMMA A-fragment order of 8-frame groups: element (b, j) lives at
//   ((b/8)*S + j/4)*32 + (b%8)*4 + j%4
// so one coalesced 8-byte load per k-step gives every lane its m8n8k4 A operand.
__host__ __device__ constexpr int ksteps_even(int M) { return (M + 3) / 4; }
__host__ __device__ constexpr int ksteps(int M) { return (M + 3) / 4 + (M + 2) / 4; }
__host__ __device__ constexpr int coef_cos(int k) { return k; }                          // k = 0..M-1
__host__ __device__ constexpr int coef_sin(int M, int k) { return 4 * ksteps_even(M) + k - 1; }   // k = 1..M-1
__host__ __device__ inline size_t coef_index(int64_t b, int j, int S) {
  return ((size_t)(b >> 3) * S + (j >> 2)) * 32 + (size_t)(b & 7) * 4 + (j & 3);
}
inline size_t coef_words(int64_t max_batch, int M) { return (size_t)((max_batch + 7) / 8) * ksteps(M) * 32; }

// Q12: P = 1/f reported in fp32, saturating at FLT_MAX.
__device__ __forceinline__ float to_p32(double f) {
  const double p = 1.0 / f;
  return p > (double)FLT_MAX ? FLT_MAX : (float)p;
}
// Floor and peak tests run on the IEEE bit patterns: for positive doubles they order like the
// values (integer compares keep the FP64 pipe free).
constexpr long long kInfBits = 0x7FF0000000000000LL;        // bits of +inf
constexpr long long kFloorBits = 0x01A56E1FC2F8F359LL;      // bits of 1e-300 (kFloor, Q12)
// max(f, 1e-300) with NaN, +-0 and negative values -> 1e-300 (the oracle's floor), on the bits
__device__ __forceinline__ long long floor_bits(long long x) {
  x = x > kInfBits ? kFloorBits : x;
  return x > kFloorBits ? x : kFloorBits;
}

// Grid angle (Q8, Q26): theta_i = theta0 + i dtheta (rounded multiply, then rounded add); on a
// symmetric grid the upper half i >= ceil(L/2) is built from the other end, -theta_{L-1-i}.
// u = 2 (d/lambda) sin(theta) with sinpi, odd in theta, so mirrored angles give u exactly negated.
__device__ __forceinline__ double grid_u(int64_t i, double theta0, double dtheta, double dl, int L, bool sym) {
  double th;
  if (sym && i >= (L + 1) / 2) th = -__dadd_rn(__dmul_rn((double)(L - 1 - i), dtheta), theta0);
  else th = __dadd_rn(__dmul_rn((double)i, dtheta), theta0);
  return 2.0 * dl * sinpi(th / 180.0);
}

// Peak test for the warp-window scans (scan_direct.cu, scan_fp32.cu): a warp owns 64 consecutive tile
// positions, lane l positions 2l and 2l+1 (0 and 63 are halo).  Peak test on one lane's pair of consecutive positions (v0 at window position 2 lane, v1 at
// 2 lane + 1; floored bits) and candidate append.  REV: tile index i holds grid index L-1-i.
template <bool REV>
__device__ __forceinline__ void window_peaks(long long v0, long long v1, int lane, int base, int ilo, int ihi, int L,
                                             int cap, int32_t* cnt, int32_t* cidx, double* cf) {
  const long long vl = __shfl_up_sync(0xffffffffu, v1, 1);          // left of position 2 lane
  const long long vr = __shfl_down_sync(0xffffffffu, v0, 1);        // right of position 2 lane + 1
  // forward (Q10): f_i < f_{i-1} and f_i <= f_{i+1}; REV (grid index decreasing with i):
  // f_i < f_{i+1} and f_i <= f_{i-1}
  const bool h0 = REV ? (v0 < v1 && v0 <= vl) : (v0 < vl && v0 <= v1);
  const bool h1 = REV ? (v1 < vr && v1 <= v0) : (v1 < v0 && v1 <= vr);
  const int i0 = base + 2 * lane, i1 = i0 + 1;
  const bool d0 = h0 && lane > 0 && i0 >= ilo && i0 <= ihi;            // position 0 is halo
  const bool d1 = h1 && lane < 31 && i1 >= ilo && i1 <= ihi;           // position 63 is halo
  if (d0) {
    const int slot = atomicAdd(cnt, 1);
    if (slot < cap) { cidx[slot] = REV ? L - 1 - i0 : i0; cf[slot] = __longlong_as_double(v0); }
  }
  if (d1) {
    const int slot = atomicAdd(cnt, 1);
    if (slot < cap) { cidx[slot] = REV ? L - 1 - i1 : i1; cf[slot] = __longlong_as_double(v1); }
  }
}

template <bool REV>
__device__ __forceinline__ void window_P(long long v0, long long v1, int lane, int base, int whi, int L, float* P) {
  const int i0 = base + 2 * lane, i1 = i0 + 1;
  if (lane > 0 && i0 >= 0 && i0 <= whi) P[REV ? L - 1 - i0 : i0] = to_p32(__longlong_as_double(v0));
  if (lane < 31 && i1 >= 0 && i1 <= whi) P[REV ? L - 1 - i1 : i1] = to_p32(__longlong_as_double(v1));
}

}  // namespace doa

struct doa_plan_s {
  int32_t M, D, alg, cap;
  int32_t device;                 // CUDA device the plan's workspace lives on; calls must run there
  int32_t geom;                   // 0: ULA (Toeplitz scan); 1: general array on an az x el grid
  double dl, theta0, dtheta;
  int64_t L, max_batch;
  int32_t sym;                    // Q26: theta0 + (L-1) dtheta == -theta0 (grid built from both ends)
  int32_t mirror;                 // scan evaluates mirrored angle pairs with one contraction (sym only)
  // general-array plans (geom == 1): grid az_i = az0 + i daz (i < naz), el_j = el0 + j del (j < nel),
  // flattened azimuth-major; element-pair position differences r_q - r_p (p < q) in wavelengths
  double az0, daz, el0, del;
  int64_t naz, nel;
  int32_t wrap;
  double* dpos;                   // [M(M-1)/2][3] device
  double* fbuf;                   // [max_batch][L] floored f of the last doa_spectrum (device)
  int32_t engine;                 // DOA_ENGINE_*: S3-S6 as the fp64 Toeplitz DMMA contraction or the fp32 direct form
  float* x32;                     // [max_batch][M-D][M] complex64 weighted noise vectors (fp32 engine, lazily)
  int64_t last_B;                 // B of the last doa_spectrum (consumed by doa_peaks)
  int64_t coef_B;                 // frames whose S3 coefficients the plan holds (doa_scan_multi)
  // workspace (device)
  int32_t* cnt;                   // [max_batch]           candidate counters
  int32_t* cand_idx;              // [max_batch][cap]
  double* cand_f;                 // [max_batch][cap]
  double* coef;                   // [max_batch][2M]
  double* R;                      // [max_batch][M][M][2]  doa_run scratch
  double* lam;                    // [max_batch][M]
  double* V;                      // [max_batch][M][M][2]
  void* cov_ws;                   // small-batch multi-CTA covariance workspace (cov_workspace_bytes)
  // doa_run_host staging (lazily sized on first use)
  float* dX[2];
  size_t dX_bytes;
  int32_t* d_out;                 // idx/val/npk/info for nplans x max_batch frames
  size_t d_out_words;
  cudaStream_t copy_stream;
  cudaEvent_t ev_copied[2], ev_used[2];
};

namespace doa {

// Launchers (enqueue only; return cudaGetLastError() of the launch).  Each increments the
// thread-local launch counter.
// ws: nullable workspace of cov_workspace_bytes() (zero-initialised once) for the small-batch
// multi-CTA covariance (B <= kDirectMaxB, N > 256, M <= 16); without it the per-frame kernels run
cudaError_t launch_covariance(const float* X, int64_t B, int64_t N, int M, double* R, cudaStream_t s,
                              void* ws = nullptr);
size_t cov_workspace_bytes();
cudaError_t launch_eig(const double* R, int64_t B, int M, double* lam, double* V, int32_t* info, cudaStream_t s);
cudaError_t launch_coef(const doa_plan_s* p, const double* lam, const double* V, int64_t B, int32_t* info,
                        cudaStream_t s);
// S3 for several plans sharing M, D from one set of eigenpairs (one launch for M <= 16)
constexpr int kMaxCoefPlans = 4;
struct CoefPlans {
  int alg[kMaxCoefPlans];
  double* coef[kMaxCoefPlans];
  int32_t* cnt[kMaxCoefPlans];
  int32_t* info[kMaxCoefPlans];
  int nplans;
};
// The frame kernel for M <= 16 (csrc/eig16.cu): S2 + S3 for up to kMaxCoefPlans ULA plans in one
// launch; lam / V nullable (not written); each plan's info[b] is overwritten (NOCONV | DEGENERATE).
cudaError_t launch_eig16_coef(const double* R, int64_t B, int M, int D, double* lam, double* V, const CoefPlans& cp,
                              cudaStream_t s);
cudaError_t launch_coef_multi(const doa_plan_s* const* plans, int nplans, const double* lam, const double* V,
                              int64_t B, int32_t* const* info, cudaStream_t s);
cudaError_t launch_scan(const doa_plan_s* p, int64_t B, float* P, cudaStream_t s);
// S4-S6 for 1..kMaxCoefPlans direct_compatible ULA plans (coefficients in place, counters zeroed):
// one direct-scan launch for all of them (B <= kDirectMaxB) or one DMMA launch per plan; P
// (nplans == 1 only) nullable
cudaError_t launch_scan_plans(const doa_plan_s* const* plans, int nplans, int64_t B, float* P, cudaStream_t s);
cudaError_t launch_select(const doa_plan_s* p, int64_t B, int32_t* idx, float* val, int32_t* npk, int32_t* info,
                          cudaStream_t s);
// S7 for up to kMaxCoefPlans plans sharing D in one launch
struct SelectPlans {
  const int32_t* cnt[4];
  const int32_t* cidx[4];
  const double* cf[4];
  int cap[4];
  int32_t* idx[4];
  float* val[4];
  int32_t* npk[4];
  int32_t* info[4];
  int nplans;
};
cudaError_t launch_select_multi(const SelectPlans& sp, int D, int64_t B, cudaStream_t s);
// Direct (non-tensor-core) scan for small batches (csrc/scan_direct.cu): one launch evaluates up to
// kMaxDirectPlans ULA plans that share M, d/lambda and the grid (e.g. the four estimators of a
// frame), steering generated once per angle.  `p` supplies the shared parameters; the plans'
// coefficients must be in place (launch_coef) and their candidate counters zeroed.
constexpr int kMaxDirectPlans = 4;
constexpr int64_t kDirectMaxB = 16;      // batches up to this size take the direct scan
struct DirectScanArgs {
  const double* coef[kMaxDirectPlans];
  int32_t* cnt[kMaxDirectPlans];
  int32_t* cidx[kMaxDirectPlans];
  double* cf[kMaxDirectPlans];
  float* P[kMaxDirectPlans];
  int nplans;
};
cudaError_t launch_scan_direct(const DirectScanArgs& args, const doa_plan_s* p, int64_t B, cudaStream_t s);
// NEXT-2, the fp32 direct-form engine (csrc/scan_fp32.cu): S3 as weighted complex64 vectors into
// p->x32 (counters zeroed, DEGENERATE ORed into info), and the FP32-pipe scan + candidates
cudaError_t launch_vec32(const doa_plan_s* p, const double* lam, const double* V, int64_t B, int32_t* info,
                         cudaStream_t s);
cudaError_t launch_scan_f32(const doa_plan_s* p, int64_t B, float* P, cudaStream_t s);
// the same direct form on the 5th-generation tensor cores: tcgen05.mma kind::tf32, 3xTF32 split,
// accumulators in TMEM (csrc/scan_tc.cu)
cudaError_t launch_scan_tc(const doa_plan_s* p, int64_t B, float* P, cudaStream_t s);
// S4-S6 of a direct-form engine plan (DOA_ENGINE_DIRECT_FP32 or DOA_ENGINE_DIRECT_TF32X3)
inline cudaError_t launch_scan_direct_form(const doa_plan_s* p, int64_t B, float* P, cudaStream_t s) {
  return p->engine == DOA_ENGINE_DIRECT_TF32X3 ? launch_scan_tc(p, B, P, s) : launch_scan_f32(p, B, P, s);
}
// plans that may share one direct scan launch (same M, d/lambda, grid; ULA)
bool direct_compatible(const doa_plan_s* a, const doa_plan_s* b);
// general-array plans (csrc/array.cu): coefficients, scan into fbuf, 2-D candidates (+ optional P)
cudaError_t launch_array_spectrum(const doa_plan_s* p, const double* lam, const double* V, int64_t B, float* P,
                                  int32_t* info, cudaStream_t s);
__host__ __device__ constexpr int array_terms(int M) { return 1 + M * (M - 1); }   // c_0 + (Re, Im) per pair
__host__ __device__ constexpr int array_ksteps(int M) { return (array_terms(M) + 3) / 4; }

// NEXT-3: on-device Eq. 1 snapshots (csrc/generate.cu)
cudaError_t launch_generate(int M, double dl, int D, const double* theta, int per_frame, double snr_db, uint64_t seed,
                            int64_t frame0, int64_t B, int64_t N, float* X, cudaStream_t s);

void count_launch();

// Per-device launch configuration (csrc/runtime.cu): SM count of the current device, and the
// occupancy of `func` at (threads, smem) on the current device — setting its dynamic-smem
// attribute there first when smem > 48 KB.  Cached per (kernel, device); thread-safe.
int current_device();
int sm_count();
int kernel_occupancy(const void* func, int threads, size_t smem);
template <typename F>
inline int kernel_occupancy(F* func, int threads, size_t smem) {
  return kernel_occupancy(reinterpret_cast<const void*>(func), threads, smem);
}

}  // namespace doa
