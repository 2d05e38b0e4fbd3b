// S3 (noise subspace -> Toeplitz coefficients), S4+S5+S6 (steering generation, pseudo-spectrum
// scan, local-maximum candidates) and S7 (top-D selection).
//
// Toeplitz identity: for a ULA, a_m = z^m with z = e^{-j psi}, psi = pi u,
// u = 2 (d/lambda) sin(theta), so for any Hermitian C
//     a^H C a = sum_{p,q} C_pq z^{q-p} = c_0 + 2 Re sum_{k>=1} c_k z^k,   c_k = sum_p C[p][p+k].
// Each (frame, angle) then costs 2(M-1) fp64 FMAs against a per-angle table
// T(psi) = (1, cos k psi, sin k psi) shared by every frame — the scan is the real contraction
// F[b][i] = sum_j coef[b][j] T[j][i] with K = 2M (Table 2 Step-5).
#include <cfloat>

#include "doa_internal.cuh"

namespace doa {
namespace {

__device__ __forceinline__ float to_p32(double f) {
  const double p = 1.0 / f;
  return p > (double)FLT_MAX ? FLT_MAX : (float)p;      // Q12: fp32 P saturates at FLT_MAX
}

// ---------------------------------------------------------------------------------------------
// S3: one warp per frame.  Table 3 Step-3 noise-subspace objects as weighted vectors
// {(w_j, u_j)}, C = sum_j w_j u_j u_j^H, and c_k = sum_j w_j sum_p u_j[p] conj(u_j[p+k]).
//   PHD: u = e_0 (smallest eigenvalue), w = 1.     MUSIC: u_j = e_j, j < K = M-D, w = 1.
//   EV : u_j = e_j, w_j = 1/lambda_j (Q1), clamped at 100 eps lambda_max (DEGENERATE).
//   MN : u = P_n e1 / (e1^H P_n e1), P_n e1 = sum_j e_j conj(e_j[0]) (Q5); p0 <= 100 eps: DEGENERATE.
// Also zeroes the frame's candidate counter for the scan that follows.
__global__ void __launch_bounds__(128) coef_kernel(const double* __restrict__ lam, const double2* __restrict__ V,
                                                  int64_t B, int M, int D, int alg, double* __restrict__ coef,
                                                  int32_t* __restrict__ cnt, int32_t* __restrict__ info) {
  __shared__ double2 mn_w[4][kMaxM];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t b = (int64_t)blockIdx.x * 4 + warp;
  if (b >= B) return;
  const double2* Vb = V + (size_t)b * M * M;
  const double* lb = lam + (size_t)b * M;
  const int K = M - D;
  int flag = 0;
  int nv = 1;
  if (alg == DOA_ALG_MUSIC || alg == DOA_ALG_EV) nv = K;
  double lfloor = 0.0;
  if (alg == DOA_ALG_EV) {
    lfloor = 100.0 * DBL_EPSILON * fmax(lb[M - 1], 0.0);
    for (int j = 0; j < K; ++j) if (lb[j] <= lfloor) flag |= DOA_INFO_DEGENERATE;
  }
  if (alg == DOA_ALG_MN) {
    double p0 = 0.0;
    for (int j = 0; j < K; ++j) { const double2 v = Vb[j]; p0 += v.x * v.x + v.y * v.y; }
    const bool degen = !(p0 > 100.0 * DBL_EPSILON);
    if (degen) flag |= DOA_INFO_DEGENERATE;
    const double lp = degen ? 1.0 : 1.0 / p0;
    for (int i = lane; i < M; i += 32) {
      double pr = 0.0, pi = 0.0;
      for (int j = 0; j < K; ++j) {
        const double2 e = Vb[(size_t)i * M + j], e0 = Vb[j];
        // e_j[i] * conj(e_j[0])
        pr += e.x * e0.x + e.y * e0.y;
        pi += e.y * e0.x - e.x * e0.y;
      }
      mn_w[warp][i] = degen ? make_double2(pr, pi) : make_double2(pr * lp, pi * lp);
    }
    __syncwarp();
  }
  double* cb = coef + (size_t)b * nj(M);
  for (int k = lane; k < M; k += 32) {
    double cr = 0.0, ci = 0.0;
    for (int j = 0; j < nv; ++j) {
      double w = 1.0;
      if (alg == DOA_ALG_EV) w = lb[j] <= lfloor ? (lfloor > 0.0 ? 1.0 / lfloor : 1.0) : 1.0 / lb[j];
      double sr = 0.0, si = 0.0;
      for (int p = 0; p + k < M; ++p) {
        double2 x, y;
        if (alg == DOA_ALG_MN) { x = mn_w[warp][p]; y = mn_w[warp][p + k]; }
        else { x = Vb[(size_t)p * M + j]; y = Vb[(size_t)(p + k) * M + j]; }
        // u[p] conj(u[p+k])
        sr += x.x * y.x + x.y * y.y;
        si += x.y * y.x - x.x * y.y;
      }
      cr += w * sr;
      ci += w * si;
    }
    if (k == 0) { cb[0] = cr; cb[2 * M - 1] = 0.0; }
    else { cb[k] = 2.0 * cr; cb[M - 1 + k] = 2.0 * ci; }
  }
  if (lane == 0) {
    cnt[b] = 0;
    if (info) info[b] |= flag;
  }
}

// ---------------------------------------------------------------------------------------------
// S4-S6 (first version, DFMA): each lane owns one angle of a 32-angle warp block whose end lanes
// are halo (lanes 1..30 decide; warp stride 30).  The lane's table T (2M doubles) is generated
// once in registers with fp64 sincospi, then the CTA's frame range is streamed: per frame a
// warp-uniform coefficient load, 2M-1 DFMAs, a neighbour exchange by shuffles and the peak test
// f_i < f_{i-1} && f_i <= f_{i+1} on interior indices (Q9/Q10).
constexpr int kScanWarps = 4;
constexpr int kScanStride = 30;

template <int M>
__global__ void __launch_bounds__(kScanWarps * 32) scan_kernel(const double* __restrict__ coef, int64_t B,
                                                              int64_t frames_per_cta, double dl, double theta0,
                                                              double dtheta, int64_t L, int cap,
                                                              int32_t* __restrict__ cnt, int32_t* __restrict__ cidx,
                                                              double* __restrict__ cf, float* __restrict__ P) {
  constexpr int NJ = nj(M);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t wblk = (int64_t)blockIdx.x * kScanWarps + warp;
  const int64_t i = wblk * kScanStride - 1 + lane;
  const bool valid = (i >= 0 && i < L);
  double T[NJ];
  T[0] = 1.0;
  if (valid) {
    const double th = __dadd_rn(__dmul_rn((double)i, dtheta), theta0);   // Q8: multiply then add
    const double u = 2.0 * dl * sinpi(th / 180.0);
#pragma unroll
    for (int k = 1; k < M; ++k) {
      double s, c;
      sincospi((double)k * u, &s, &c);
      T[k] = c;
      T[M - 1 + k] = s;
    }
  } else {
#pragma unroll
    for (int k = 1; k < M; ++k) { T[k] = 0.0; T[M - 1 + k] = 0.0; }
  }
  const bool own = lane >= 1 && lane <= kScanStride && valid;
  const bool decide = own && i >= 1 && i <= L - 2;
  const int64_t b0 = (int64_t)blockIdx.y * frames_per_cta;
  const int64_t b1 = min(B, b0 + frames_per_cta);
  for (int64_t b = b0; b < b1; ++b) {
    const double* cb = coef + (size_t)b * NJ;
    double acc = __ldg(cb);
#pragma unroll
    for (int j = 1; j < NJ - 1; ++j) acc = fma(__ldg(cb + j), T[j], acc);
    const double f = acc > kFloor ? acc : kFloor;
    const double fl = __shfl_up_sync(0xffffffffu, f, 1);
    const double fr = __shfl_down_sync(0xffffffffu, f, 1);
    if (decide && f < fl && f <= fr) {
      const int slot = atomicAdd(cnt + b, 1);
      if (slot < cap) {
        cidx[(size_t)b * cap + slot] = (int32_t)i;
        cf[(size_t)b * cap + slot] = f;
      }
    }
    if (P && own) P[(size_t)b * L + i] = to_p32(f);
  }
}

// Same algorithm for any M <= 64 with the table in shared memory (runtime M; used for M > 32,
// where a register-resident table would spill).
__global__ void __launch_bounds__(kScanWarps * 32) scan_kernel_smem(const double* __restrict__ coef, int64_t B, int M,
                                                                   int64_t frames_per_cta, double dl, double theta0,
                                                                   double dtheta, int64_t L, int cap,
                                                                   int32_t* __restrict__ cnt,
                                                                   int32_t* __restrict__ cidx, double* __restrict__ cf,
                                                                   float* __restrict__ P) {
  extern __shared__ double tsm[];
  const int NJ = nj(M);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* T = tsm + (size_t)warp * NJ * 32;          // T[j][lane]
  const int64_t wblk = (int64_t)blockIdx.x * kScanWarps + warp;
  const int64_t i = wblk * kScanStride - 1 + lane;
  const bool valid = (i >= 0 && i < L);
  T[lane] = 1.0;
  T[(NJ - 1) * 32 + lane] = 0.0;
  double u = 0.0;
  if (valid) {
    const double th = __dadd_rn(__dmul_rn((double)i, dtheta), theta0);
    u = 2.0 * dl * sinpi(th / 180.0);
  }
  for (int k = 1; k < M; ++k) {
    double sn = 0.0, c = 0.0;
    if (valid) sincospi((double)k * u, &sn, &c);
    T[k * 32 + lane] = c;
    T[(M - 1 + k) * 32 + lane] = sn;
  }
  __syncwarp();
  const bool own = lane >= 1 && lane <= kScanStride && valid;
  const bool decide = own && i >= 1 && i <= L - 2;
  const int64_t b0 = (int64_t)blockIdx.y * frames_per_cta;
  const int64_t b1 = min(B, b0 + frames_per_cta);
  for (int64_t b = b0; b < b1; ++b) {
    const double* cb = coef + (size_t)b * NJ;
    double acc = __ldg(cb);
    for (int j = 1; j < NJ - 1; ++j) acc = fma(__ldg(cb + j), T[j * 32 + lane], acc);
    const double f = acc > kFloor ? acc : kFloor;
    const double fl = __shfl_up_sync(0xffffffffu, f, 1);
    const double fr = __shfl_down_sync(0xffffffffu, f, 1);
    if (decide && f < fl && f <= fr) {
      const int slot = atomicAdd(cnt + b, 1);
      if (slot < cap) {
        cidx[(size_t)b * cap + slot] = (int32_t)i;
        cf[(size_t)b * cap + slot] = f;
      }
    }
    if (P && own) P[(size_t)b * L + i] = to_p32(f);
  }
}

int64_t scan_frames_per_cta(int64_t gx, int64_t B) {
  // frame chunk: enough CTAs for ~8 waves on 148 SMs, at least 16 frames per CTA
  int64_t fpc = (gx * B) / (148 * 16 * 8);
  fpc = fpc < 16 ? 16 : fpc;
  if (fpc > B) fpc = B;
  return fpc;
}

template <int M>
cudaError_t launch_scan_t(const doa_plan_s* p, int64_t B, float* P, cudaStream_t s) {
  const int64_t nwb = (p->L + kScanStride - 1) / kScanStride;
  const int64_t gx = (nwb + kScanWarps - 1) / kScanWarps;
  const int64_t fpc = scan_frames_per_cta(gx, B);
  const int64_t gy = (B + fpc - 1) / fpc;
  count_launch();
  scan_kernel<M><<<dim3((unsigned)gx, (unsigned)gy), kScanWarps * 32, 0, s>>>(
      p->coef, B, fpc, p->dl, p->theta0, p->dtheta, p->L, p->cap, p->cnt, p->cand_idx, p->cand_f, P);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// S7: one warp per frame.  Rank every stored candidate by (f ascending, index ascending) and
// scatter the first D (PeakSelection; Q11).
__global__ void __launch_bounds__(128) select_kernel(int64_t B, int D, int cap, const int32_t* __restrict__ cnt,
                                                    const int32_t* __restrict__ cidx, const double* __restrict__ cf,
                                                    int32_t* __restrict__ idx, float* __restrict__ val,
                                                    int32_t* __restrict__ npk, int32_t* __restrict__ info) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t b = (int64_t)blockIdx.x * 4 + warp;
  if (b >= B) return;
  const int nraw = cnt[b];
  const int n = nraw < cap ? nraw : cap;
  const int32_t* ci = cidx + (size_t)b * cap;
  const double* cfv = cf + (size_t)b * cap;
  for (int c = lane; c < n; c += 32) {
    const double fc = cfv[c];
    const int ic = ci[c];
    int rk = 0;
    for (int j = 0; j < n; ++j) {
      const double fj = cfv[j];
      rk += (fj < fc) || (fj == fc && ci[j] < ic);
    }
    if (rk < D) {
      idx[(size_t)b * D + rk] = ic;
      val[(size_t)b * D + rk] = to_p32(fc);
    }
  }
  for (int k = n + lane; k < D; k += 32) {
    idx[(size_t)b * D + k] = -1;
    val[(size_t)b * D + k] = 0.0f;
  }
  if (lane == 0) {
    npk[b] = n < D ? n : D;
    int fl = 0;
    if (nraw > cap) fl |= DOA_INFO_CAND_OVERFLOW;
    if (n < D) fl |= DOA_INFO_UNDERDETERMINED;
    info[b] |= fl;
  }
}

}  // namespace

cudaError_t launch_coef(const doa_plan_s* p, const double* lam, const double* V, int64_t B, int32_t* info,
                        cudaStream_t s) {
  count_launch();
  coef_kernel<<<(unsigned)((B + 3) / 4), 128, 0, s>>>(lam, reinterpret_cast<const double2*>(V), B, p->M, p->D,
                                                       p->alg, p->coef, p->cnt, info);
  return cudaGetLastError();
}

cudaError_t launch_scan(const doa_plan_s* p, int64_t B, float* P, cudaStream_t s) {
  switch (p->M) {
#define DOA_SCAN_CASE(m) case m: return launch_scan_t<m>(p, B, P, s);
    DOA_SCAN_CASE(2) DOA_SCAN_CASE(3) DOA_SCAN_CASE(4) DOA_SCAN_CASE(5) DOA_SCAN_CASE(6) DOA_SCAN_CASE(7)
    DOA_SCAN_CASE(8) DOA_SCAN_CASE(9) DOA_SCAN_CASE(10) DOA_SCAN_CASE(11) DOA_SCAN_CASE(12) DOA_SCAN_CASE(13)
    DOA_SCAN_CASE(14) DOA_SCAN_CASE(15) DOA_SCAN_CASE(16) DOA_SCAN_CASE(17) DOA_SCAN_CASE(18) DOA_SCAN_CASE(19)
    DOA_SCAN_CASE(20) DOA_SCAN_CASE(21) DOA_SCAN_CASE(22) DOA_SCAN_CASE(23) DOA_SCAN_CASE(24)
    DOA_SCAN_CASE(25) DOA_SCAN_CASE(26) DOA_SCAN_CASE(27) DOA_SCAN_CASE(28) DOA_SCAN_CASE(29)
    DOA_SCAN_CASE(30) DOA_SCAN_CASE(31) DOA_SCAN_CASE(32)
#undef DOA_SCAN_CASE
    default: {
      const int64_t nwb = (p->L + kScanStride - 1) / kScanStride;
      const int64_t gx = (nwb + kScanWarps - 1) / kScanWarps;
      const int64_t fpc = scan_frames_per_cta(gx, B);
      const int64_t gy = (B + fpc - 1) / fpc;
      const size_t smem = (size_t)kScanWarps * nj(p->M) * 32 * sizeof(double);
      static bool attr = false;
      if (!attr) {
        cudaFuncSetAttribute(scan_kernel_smem, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(kScanWarps * nj(kMaxM) * 32 * sizeof(double)));
        attr = true;
      }
      count_launch();
      scan_kernel_smem<<<dim3((unsigned)gx, (unsigned)gy), kScanWarps * 32, smem, s>>>(
          p->coef, B, p->M, fpc, p->dl, p->theta0, p->dtheta, p->L, p->cap, p->cnt, p->cand_idx, p->cand_f, P);
      return cudaGetLastError();
    }
  }
}

cudaError_t launch_select(const doa_plan_s* p, int64_t B, int32_t* idx, float* val, int32_t* npk, int32_t* info,
                          cudaStream_t s) {
  count_launch();
  select_kernel<<<(unsigned)((B + 3) / 4), 128, 0, s>>>(B, p->D, p->cap, p->cnt, p->cand_idx, p->cand_f, idx, val,
                                                         npk, info);
  return cudaGetLastError();
}

}  // namespace doa
