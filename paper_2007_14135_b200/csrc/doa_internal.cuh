// Internal declarations shared by the libdoa translation units (not part of the ABI).
#pragma once

#include <cuda_runtime.h>
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
  int64_t last_B;                 // B of the last doa_spectrum (consumed by doa_peaks)
  // workspace (device)
  int32_t* cnt;                   // [max_batch]           candidate counters
  int32_t* cand_idx;              // [max_batch][cap]
  double* cand_f;                 // [max_batch][cap]
  double* coef;                   // [max_batch][2M]
  double* R;                      // [max_batch][M][M][2]  doa_run scratch
  double* lam;                    // [max_batch][M]
  double* V;                      // [max_batch][M][M][2]
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
cudaError_t launch_covariance(const float* X, int64_t B, int64_t N, int M, double* R, cudaStream_t s);
cudaError_t launch_eig(const double* R, int64_t B, int M, double* lam, double* V, int32_t* info, cudaStream_t s);
cudaError_t launch_coef(const doa_plan_s* p, const double* lam, const double* V, int64_t B, int32_t* info,
                        cudaStream_t s);
cudaError_t launch_scan(const doa_plan_s* p, int64_t B, float* P, cudaStream_t s);
cudaError_t launch_select(const doa_plan_s* p, int64_t B, int32_t* idx, float* val, int32_t* npk, int32_t* info,
                          cudaStream_t s);
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
