// S3 (noise subspace -> Toeplitz coefficients), S4+S5+S6 (steering generation, pseudo-spectrum
// scan, local-maximum candidates) and S7 (top-D selection).
//
// Toeplitz identity: for a ULA, a_m = z^m with z = e^{-j psi}, psi = pi u,
// u = 2 (d/lambda) sin(theta), so for any Hermitian C
//     a^H C a = sum_{p,q} C_pq z^{q-p} = c_0 + 2 Re sum_{k>=1} c_k z^k,   c_k = sum_p C[p][p+k].
// Each (frame, angle) then costs 2(M-1) fp64 FMAs against a per-angle table
// T(psi) = (1, cos k psi, sin k psi) shared by every frame — the scan is the real contraction
// F[b][i] = sum_j coef[b][j] T[j][i] (Table 2 Step-5), K = 4S (even and odd halves, see
// doa_internal.cuh), run on the FP64 tensor pipe (DMMA, mma.sync m8n8k4 f64) with the table
// staged once per CTA in shared memory.  On symmetric grids (Q26) one contraction
// yields a mirrored pair of angles (f = E + O and E - O).
#include <cfloat>

#include "doa_internal.cuh"

namespace doa {
namespace {


// T_j(psi) in the split layout of doa_internal.cuh: j = 0 -> 1; 1..M-1 -> cos(j psi);
// JE..JE+M-2 -> sin((j-JE+1) psi) with JE = 4 ceil(M/4); else 0.
// psi = pi u; cospi/sinpi of the exact multiple j*u (one rounding) — no recurrence.  Both are
// exactly even / odd in u, so T(-u) is T(u) with the odd half negated bit for bit.
__device__ __forceinline__ double table_entry(int j, int M, double u) {
  const int JE = 4 * ksteps_even(M);
  if (j == 0) return 1.0;
  if (j < M) return cospi((double)j * u);
  if (j >= JE && j < JE + M - 1) return sinpi((double)(j - JE + 1) * u);
  return 0.0;
}

// Named barriers over the CTA's 256 threads (id 0 is __syncthreads): bar_sync waits until the
// 128 threads of the other warp group have arrived; bar_arrive signals without waiting.
__device__ __forceinline__ void bar_sync(int id) {
  if (id == 1) asm volatile("bar.sync 1, 256;\n" ::: "memory");
  else asm volatile("bar.sync 2, 256;\n" ::: "memory");
}
__device__ __forceinline__ void bar_arrive(int id) {
  if (id == 1) asm volatile("bar.arrive 1, 256;\n" ::: "memory");
  else asm volatile("bar.arrive 2, 256;\n" ::: "memory");
}

__device__ __forceinline__ void dmma_884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}
// D = A B + C with a separate accumulator input C
__device__ __forceinline__ void dmma_884c(double& d0, double& d1, double a, double b, double c0, double c1) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};\n"
               : "=d"(d0), "=d"(d1)
               : "d"(a), "d"(b), "d"(c0), "d"(c1));
}

// ---------------------------------------------------------------------------------------------
// S3 (Table 3 Step-3/4): noise-subspace objects as weighted vectors {(w_j, u_j)},
// C = sum_j w_j u_j u_j^H, reduced to the Toeplitz sums c_k = sum_p C[p][p+k]:
//   PHD: u = e_0 (smallest eigenvalue), w = 1.     MUSIC: u_j = e_j, j < K = M-D, w = 1.
//   EV : u_j = e_j, w_j = 1/lambda_j (Q1), clamped at 100 eps lambda_max (DEGENERATE, G1).
//   MN : u = P_n e1 / (e1^H P_n e1), P_n e1 = sum_j e_j conj(e_j[0]) (Q5); p0 <= 100 eps: DEGENERATE.
// The coefficients go to the scan's A-fragment layout (coef_index); the frame's candidate counter
// is zeroed for the scan that follows.
//
constexpr int kCoefWaves = 2;     // coef_mma_kernel CTAs = resident slots x waves (persistent warps)

// S3 for M <= 16 on the FP64 tensor pipe.  C = X U^H with U = the noise vectors (columns of V)
// and X = (w_j u_j) (weights only for EV; MN: the single vector w of Table 3 Step-3), i.e.
//   C_re = X_re U_re^T + X_im U_im^T,   C_im = X_im U_re^T - X_re U_im^T   (16 x 16, inner dim j),
// as DMMA m8n8k4 products over the upper 8x8 tiles (0,0), (0,1), (1,1) — at most 48 DMMAs per
// frame — with the operand fragments read once from shared memory (U staged as re/im planes
// [j][p], row stride 20 doubles: conflict-free staging stores and fragment loads).  The tiles go back through shared memory and lanes k < M add the
// diagonal c_k = sum_p C[p][p+k] in ascending p.  Fixed orders throughout: deterministic.  Replaces
// a lag-per-lane loop (round-1 coef_kernel) whose shared-memory traffic (~1000 wavefronts per frame)
// bound it; this one moves ~150.
constexpr int kCoefMmaWarps = 8;
constexpr int kCoefMmaLd = 20;                         // plane row stride (doubles), = 4 mod 16: conflict-free fragments
constexpr int kCoefMmaPlane = 16 * kCoefMmaLd;         // doubles per plane

// One frame's S3 by one warp.  Ure/Uim: the warp's planes holding the frame's eigenvectors
// u_j[p] at j * ld + p (ascending j, zero outside j < K, p < M, up to 16 x 16); they are
// overwritten (MN: vector 0 <- w; then the C tiles).  lb: the frame's ascending eigenvalues.
__device__ __forceinline__ void coef_frame_mma(int lane, double* Ure, double* Uim, const double* lb, int M, int D,
                                               int alg, double* __restrict__ coef, int64_t b,
                                               int32_t* __restrict__ cnt, int32_t* __restrict__ info) {
  constexpr int ld = kCoefMmaLd;
  const int S = ksteps(M);
  const int K = M - D;
  int flag = 0;
  int nv = (alg == DOA_ALG_MUSIC || alg == DOA_ALG_EV) ? K : 1;
  // EV weights w_j = 1/lambda_j (Q1), clamped at 100 eps lambda_max (DEGENERATE)
  double wj[4] = {1.0, 1.0, 1.0, 1.0};                 // weight of row j = 4J + lane%4 of X
  if (alg == DOA_ALG_EV) {
    // lane j < K loads lambda_j once; weights and the DEGENERATE test are lane-parallel
    const double lmax = lb[M - 1];
    const double lfloor = 100.0 * DBL_EPSILON * fmax(lmax, 0.0);
    const double lj = lane < K ? lb[lane] : 1.0;
    const bool deg = lane < K && lj <= lfloor;
    if (__any_sync(0xffffffffu, deg)) flag |= DOA_INFO_DEGENERATE;
    const double w = lane < K ? (deg ? (lfloor > 0.0 ? 1.0 / lfloor : 1.0) : 1.0 / lj) : 0.0;
#pragma unroll
    for (int J = 0; J < 4; ++J) wj[J] = __shfl_sync(0xffffffffu, w, 4 * J + (lane & 3));
  } else if (alg == DOA_ALG_MN) {
    // w = P_n e1 / (e1^H P_n e1): P_n e1 = sum_j e_j conj(e_j[0]), e1^H P_n e1 = sum_j |e_j[0]|^2
    double p0 = lane < K ? Ure[lane * ld] * Ure[lane * ld] + Uim[lane * ld] * Uim[lane * ld] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) p0 += __shfl_xor_sync(0xffffffffu, p0, o);   // fixed tree order
    const bool degen = !(p0 > 100.0 * DBL_EPSILON);
    if (degen) flag |= DOA_INFO_DEGENERATE;
    const double lp = degen ? 1.0 : 1.0 / p0;
    double pr = 0.0, pi = 0.0;
    if (lane < M)
      for (int j = 0; j < K; ++j) {
        const double er = Ure[j * ld + lane], ei = Uim[j * ld + lane], e0r = Ure[j * ld], e0i = Uim[j * ld];
        pr += er * e0r + ei * e0i;                     // e_j[i] * conj(e_j[0])
        pi += ei * e0r - er * e0i;
      }
    __syncwarp();
    if (lane < 16) {
      Ure[lane] = degen ? pr : pr * lp;                // vector 0 <- w (zero beyond M)
      Uim[lane] = degen ? pi : pi * lp;
    }
    __syncwarp();
  }
  const int nJ = (nv + 3) >> 2;                        // k-steps over j
  const int r4 = lane & 3, c8 = lane >> 2;
  // fragments: A[p][j] = x_j[p] (row p = 8P + c8, col j = 4J + r4); B[j][q] = u_j[q] (q = 8Q + c8)
  double ar[2][4], ai[2][4], br[2][4], bi[2][4];
#pragma unroll
  for (int J = 0; J < 4; ++J)
#pragma unroll
    for (int P = 0; P < 2; ++P) {
      const int o = (4 * J + r4) * ld + 8 * P + c8;
      const bool ok = 4 * J + r4 < nv;                   // rows j >= nv (e.g. MN beyond w) are zero
      const double ur = ok ? Ure[o] : 0.0, ui = ok ? Uim[o] : 0.0;
      br[P][J] = ur;
      bi[P][J] = ui;
      ar[P][J] = wj[J] * ur;
      ai[P][J] = wj[J] * ui;
    }
  // upper tiles (P, Q) = (0,0), (0,1), (1,1); C_re, C_im accumulators
  double cr[3][2], ci[3][2];
#pragma unroll
  for (int t = 0; t < 3; ++t) { cr[t][0] = cr[t][1] = ci[t][0] = ci[t][1] = 0.0; }
#pragma unroll
  for (int J = 0; J < 4; ++J) {
    if (J >= nJ) break;
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      const int P = t == 2 ? 1 : 0, Q = t == 0 ? 0 : 1;
      dmma_884(cr[t][0], cr[t][1], ar[P][J], br[Q][J]);
      dmma_884(cr[t][0], cr[t][1], ai[P][J], bi[Q][J]);
      dmma_884(ci[t][0], ci[t][1], ai[P][J], br[Q][J]);
      dmma_884(ci[t][0], ci[t][1], -ar[P][J], bi[Q][J]);
    }
  }
  __syncwarp();                                        // every lane has its fragments: reuse the planes
  double* Cre = Ure;                                   // C[p][q] at p * ld + q
  double* Cim = Uim;
#pragma unroll
  for (int t = 0; t < 3; ++t) {
    const int P = t == 2 ? 1 : 0, Q = t == 0 ? 0 : 1;
    const int o = (8 * P + c8) * ld + 8 * Q + 2 * r4;
    Cre[o] = cr[t][0]; Cre[o + 1] = cr[t][1];
    Cim[o] = ci[t][0]; Cim[o + 1] = ci[t][1];
  }
  __syncwarp();
  if (lane < M) {
    const int k = lane;
    double dr[16], di[16];                             // all loads first, then the adds in ascending p
#pragma unroll
    for (int pp = 0; pp < 16; ++pp) {
      const bool ok = pp + k < M;
      dr[pp] = ok ? Cre[pp * ld + pp + k] : 0.0;
      di[pp] = ok ? Cim[pp * ld + pp + k] : 0.0;
    }
    double sr = 0.0, si = 0.0;
#pragma unroll
    for (int pp = 0; pp < 16; ++pp) { sr += dr[pp]; si += di[pp]; }
    if (k == 0) coef[coef_index(b, 0, S)] = sr;
    else {
      coef[coef_index(b, coef_cos(k), S)] = 2.0 * sr;
      coef[coef_index(b, coef_sin(M, k), S)] = 2.0 * si;
    }
  }
  const int JE = 4 * ksteps_even(M);
  for (int j = lane; j < 4 * S; j += 32)                                                // K padding
    if ((j >= M && j < JE) || j >= JE + M - 1) coef[coef_index(b, j, S)] = 0.0;
  if (lane == 0) {
    cnt[b] = 0;
    if (info && flag) info[b] |= flag;           // no read-modify-write round trip when clean
  }
  __syncwarp();                                        // C planes are read above before the next stores
}

// S3 for up to kMaxCoefPlans plans sharing M and D from the same eigenpairs (e.g. the four
// estimators): each frame's eigenvectors are read from HBM once, then every plan's coefficients
// are produced from them in turn by the warp (coef_frame_mma).  Persistent warps: frame b, then
// b + stride, ...; the next frame's V loads are issued before the current frame is processed.
__global__ void __launch_bounds__(kCoefMmaWarps * 32) coef_mma_kernel(const double* __restrict__ lam,
                                                                      const double2* __restrict__ V, int64_t B,
                                                                      int M, int D, CoefPlans cp) {
  constexpr int ld = kCoefMmaLd;
  extern __shared__ double cmsm[];                     // per warp: Ure, Uim planes; later C_re, C_im
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* Ure = cmsm + (size_t)warp * 2 * kCoefMmaPlane;
  double* Uim = Ure + kCoefMmaPlane;
  const int K = M - D;
  bool only_phd = true;
  for (int a = 0; a < cp.nplans; ++a) only_phd &= cp.alg[a] == DOA_ALG_PHD;
  const int nload = only_phd ? 1 : K;                  // eigenvector columns needed
  const int64_t stride = (int64_t)gridDim.x * kCoefMmaWarps;
  int64_t b = (int64_t)blockIdx.x * kCoefMmaWarps + warp;
  double2 tv[8];                                       // the whole 16 x 16 (j, p) slot grid, zero outside
  auto load_v = [&](int64_t bb) {
    const double2* Vb = V + (size_t)bb * M * M;
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const int e = lane + 32 * r, pp = e & 15, j = e >> 4;
      tv[r] = (bb < B && pp < M && j < nload) ? __ldg(Vb + pp * M + j) : make_double2(0.0, 0.0);
    }
  };
  load_v(b);
  for (; b < B; b += stride) {
    const double2 cur[8] = {tv[0], tv[1], tv[2], tv[3], tv[4], tv[5], tv[6], tv[7]};
    load_v(b + stride);
    for (int a = 0; a < cp.nplans; ++a) {
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const int e = lane + 32 * r, pp = e & 15, j = e >> 4;
        Ure[j * ld + pp] = cur[r].x;
        Uim[j * ld + pp] = cur[r].y;
      }
      __syncwarp();
      coef_frame_mma(lane, Ure, Uim, lam + (size_t)b * M, M, D, cp.alg[a], cp.coef[a], b, cp.cnt[a], cp.info[a]);
    }
  }
}

// S3 for 16 < M <= 64: the same DMMA formulation with one CTA (8 warps) per frame.  MP = 32 / 64
// padded rows, TP = MP/8 tile rows; the TP(TP+1)/2 upper 8x8 tiles of C = X U^H are dealt
// round-robin to the warps; per k-step J over the noise vectors every warp loads the fragments of
// its tiles' row / column blocks from the shared re/im planes and issues 4 DMMAs per tile.  The
// tiles then overwrite the planes and threads k < M add the diagonals in ascending p.
constexpr int kCoefBigWarps = 8;
template <int MP>
struct CoefBig {
  static constexpr int TP = MP / 8;
  static constexpr int NT = TP * (TP + 1) / 2;           // upper tiles
  static constexpr int TPW = (NT + kCoefBigWarps - 1) / kCoefBigWarps;   // tiles per warp (max)
  static constexpr int LD = MP + 4;                      // plane row stride (doubles), = 4 mod 16
  static constexpr int PLANE = MP * LD;                  // rows j < MP (K < M <= MP)
  static constexpr size_t SMEM = (size_t)2 * PLANE * sizeof(double) + MP * sizeof(double);
};

template <int MP>
__global__ void __launch_bounds__(kCoefBigWarps * 32) coef_big_kernel(const double* __restrict__ lam,
                                                                      const double2* __restrict__ V, int64_t B,
                                                                      int M, int D, int alg,
                                                                      double* __restrict__ coef,
                                                                      int32_t* __restrict__ cnt,
                                                                      int32_t* __restrict__ info) {
  using C = CoefBig<MP>;
  constexpr int ld = C::LD, TP = C::TP, NT = C::NT, TPW = C::TPW, T = kCoefBigWarps * 32;
  extern __shared__ double cbsm[];
  double* Ure = cbsm;                                    // [j][p]
  double* Uim = Ure + C::PLANE;
  double* wsh = Uim + C::PLANE;                          // [MP] EV weights
  __shared__ int flag_s;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t b = blockIdx.x;
  const double2* Vb = V + (size_t)b * M * M;
  const double* lb = lam + (size_t)b * M;
  const int S = ksteps(M);
  const int K = M - D;
  const int nload = (alg == DOA_ALG_PHD) ? 1 : K;
  if (tid == 0) flag_s = 0;
  // stage the noise vectors: V[p][j] -> planes [j][p] (coalesced global reads along j)
  for (int e = tid; e < MP * MP; e += T) {
    const int pp = e / MP, j = e - (e / MP) * MP;
    const double2 v = (pp < M && j < nload) ? __ldg(Vb + pp * M + j) : make_double2(0.0, 0.0);
    Ure[j * ld + pp] = v.x;
    Uim[j * ld + pp] = v.y;
  }
  if (alg == DOA_ALG_EV && tid < MP) {
    const double lfloor = 100.0 * DBL_EPSILON * fmax(lb[M - 1], 0.0);
    double w = 0.0;
    if (tid < K) {
      w = lb[tid] <= lfloor ? (lfloor > 0.0 ? 1.0 / lfloor : 1.0) : 1.0 / lb[tid];
      if (lb[tid] <= lfloor) atomicOr(&flag_s, DOA_INFO_DEGENERATE);
    }
    wsh[tid] = w;
  }
  __syncthreads();
  int nv = (alg == DOA_ALG_MUSIC || alg == DOA_ALG_EV) ? K : 1;
  if (alg == DOA_ALG_MN) {
    // e1^H P_n e1 = sum_j |e_j[0]|^2 over all K noise vectors (K up to 63): lane-strided partial
    // sums in ascending j, then a fixed xor tree (deterministic)
    double p0 = 0.0;
    for (int j = lane; j < K; j += 32) p0 += Ure[j * ld] * Ure[j * ld] + Uim[j * ld] * Uim[j * ld];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) p0 += __shfl_xor_sync(0xffffffffu, p0, o);   // fixed tree order
    const bool degen = !(p0 > 100.0 * DBL_EPSILON);
    const double lp = degen ? 1.0 : 1.0 / p0;
    double pr = 0.0, pi = 0.0;
    if (tid < M)
      for (int j = 0; j < K; ++j) {
        const double er = Ure[j * ld + tid], ei = Uim[j * ld + tid], e0r = Ure[j * ld], e0i = Uim[j * ld];
        pr += er * e0r + ei * e0i;                       // e_j[i] * conj(e_j[0])
        pi += ei * e0r - er * e0i;
      }
    __syncthreads();
    if (tid < MP) {
      Ure[tid] = degen ? pr : pr * lp;                   // vector 0 <- w (zero beyond M)
      Uim[tid] = degen ? pi : pi * lp;
    }
    if (tid == 0 && degen) flag_s |= DOA_INFO_DEGENERATE;
    __syncthreads();
  }
  const int nJ = (nv + 3) >> 2;
  const int r4 = lane & 3, c8 = lane >> 2;
  const bool ev = alg == DOA_ALG_EV;
  int tP[TPW], tQ[TPW];
#pragma unroll
  for (int u = 0; u < TPW; ++u) {
    int t = warp + u * kCoefBigWarps, P = 0;
    if (t >= NT) t = -1;
    int rem = t < 0 ? 0 : t;
    while (rem >= TP - P) { rem -= TP - P; ++P; }      // row-major upper tiles: row P has TP - P tiles
    tP[u] = t < 0 ? -1 : P;
    tQ[u] = P + rem;
  }
  double cr[TPW][2], ci[TPW][2];
#pragma unroll
  for (int u = 0; u < TPW; ++u) { cr[u][0] = cr[u][1] = ci[u][0] = ci[u][1] = 0.0; }
  for (int J = 0; J < nJ; ++J) {
    const int j = 4 * J + r4;
    const bool ok = j < nv;
    const double w = ev ? (ok ? wsh[j] : 0.0) : 1.0;
#pragma unroll
    for (int u = 0; u < TPW; ++u) {
      if (tP[u] < 0) continue;                           // warp-uniform
      const int oa = j * ld + 8 * tP[u] + c8, ob = j * ld + 8 * tQ[u] + c8;
      const double ur = ok ? Ure[ob] : 0.0, ui = ok ? Uim[ob] : 0.0;
      const double xr = ok ? w * Ure[oa] : 0.0, xi = ok ? w * Uim[oa] : 0.0;
      dmma_884(cr[u][0], cr[u][1], xr, ur);
      dmma_884(cr[u][0], cr[u][1], xi, ui);
      dmma_884(ci[u][0], ci[u][1], xi, ur);
      dmma_884(ci[u][0], ci[u][1], -xr, ui);
    }
  }
  __syncthreads();                                       // all fragments read: the planes become C
  double* Cre = Ure;                                     // C[p][q] at p * ld + q
  double* Cim = Uim;
#pragma unroll
  for (int u = 0; u < TPW; ++u) {
    if (tP[u] < 0) continue;
    const int o = (8 * tP[u] + c8) * ld + 8 * tQ[u] + 2 * r4;
    Cre[o] = cr[u][0]; Cre[o + 1] = cr[u][1];
    Cim[o] = ci[u][0]; Cim[o + 1] = ci[u][1];
  }
  __syncthreads();
  if (tid < M) {
    const int k = tid;
    double sr = 0.0, si = 0.0;
    for (int pp = 0; pp + k < M; ++pp) { sr += Cre[pp * ld + pp + k]; si += Cim[pp * ld + pp + k]; }
    if (k == 0) coef[coef_index(b, 0, S)] = sr;
    else {
      coef[coef_index(b, coef_cos(k), S)] = 2.0 * sr;
      coef[coef_index(b, coef_sin(M, k), S)] = 2.0 * si;
    }
  }
  const int JE = 4 * ksteps_even(M);
  for (int j = tid; j < 4 * S; j += T)                                                  // K padding
    if ((j >= M && j < JE) || j >= JE + M - 1) coef[coef_index(b, j, S)] = 0.0;
  if (tid == 0) {
    cnt[b] = 0;
    if (info && flag_s) info[b] |= flag_s;
  }
}

// ---------------------------------------------------------------------------------------------
// S4-S6: the scan on the FP64 tensor pipe (mma.sync m8n8k4 f64).
//
// Work tile = (angle column x, frame chunk y).  An angle column is NB consecutive angle blocks of
// W = 8*NA grid angles (positions 0 and W-1 of a block are halo; blocks advance by W-2 so every
// interior angle is decided by exactly one lane).  The steering table of a column is generated
// once into shared memory in DMMA B-fragment order
//     Ts[k][s][t][lane] = T_{4s + lane%4}(angle base_k + 8t + lane/4)
// (fp64 sincospi, no recurrence) so every B-fragment load is one conflict-free 8-byte LDS.
// The CTA's 8 warps stream disjoint 8-frame groups of the chunk (warp w: g0+w, g0+w+8, ...):
// one coalesced A-fragment load per k-step (issued before the group's turn barrier, reused for
// all blocks),
// S x NA DMMAs per block (8 independent accumulator chains), then the fused epilogue:
//   D fragment: lane holds frame lane/4, block positions 16(lane%4) + 0..15.
//   floor (Q12) + peak test (Q9/Q10) in the INTEGER domain — for positive doubles the IEEE bits
//   order like the values, so the FP64 pipe stays with the DMMAs; 17 compares per 16 angles in
//   registers, two shuffles for the run ends; atomic append to the frame's candidate list (the
//   value picked by a select tree on the run index); optional fp32 P.
// MIRROR (symmetric grids, Q26): the blocks cover only the lower half i <= H = ceil(L/2) (one
// angle past the middle as the last neighbour); the odd k-steps accumulate O, the even ones E on
// top of it (O is the first E DMMA's C operand), and the tile yields f_i = E + O straight from the
// tensor pipe and f_{L-1-i} = E - O = f_i - 2 O by one DFMA (psi_{L-1-i} = -psi_i exactly):
// half the DMMAs and half the steering table per grid angle.  In the mirrored half the grid index
// runs backwards through the tile, so the peak test's strict/non-strict sides swap.
// Grid: blockIdx.x = angle column, blockIdx.y = frame chunk (~4 waves of resident CTAs).
// (A persistent tile loop, a software-pipelined and a warp-specialised producer/consumer variant
// were measured and were slower on c4; see profiles/README.md.)
constexpr int kCtaWarps = 8;
constexpr int kScanNA = 8;        // 8-angle tiles per block (a lane owns 2*NA consecutive angles)
#ifndef DOA_SCAN_MINB
#define DOA_SCAN_MINB 2
#endif
constexpr int kScanMinBlocks = DOA_SCAN_MINB; // __launch_bounds__ min blocks per SM
#ifndef DOA_SCAN_WAVES
#define DOA_SCAN_WAVES 4
#endif

// Shape by k-steps S (M <= 64 -> S <= 32): 8 tiles of 8 angles per block; S <= 8 (M <= 16) keeps
// the A fragments of a group in registers with a one-group prefetch and uses two blocks per column
// (one in the mirrored variant, whose two accumulator sets double the registers); larger S streams
// the A fragment of each k-step from L1/L2 and uses one block (table: S x 8 x 32 doubles = up to
// 64 KB of smem).
template <int S, bool MIRROR>
struct ScanShape {
  static constexpr int NA = kScanNA;                     // 8-angle tiles per block
  static constexpr int W = 8 * NA;                           // angles per block (incl. 2 halo)
  static constexpr bool STREAM_A = S > 8;
  static constexpr int NB = STREAM_A ? 1 : (MIRROR ? 1 : 2);   // blocks per column
  static constexpr int SE = MIRROR ? (S + 1) / 2 : S;        // k-steps of the even part E
};

// Angle position inside a block of column n of 8-angle tile t: the D fragment gives lane (r, q)
// columns n = 2q + e of every tile, so with this permutation of the table's columns lane q holds
// the 16 CONSECUTIVE angles 16q + (2t + e) of its frame — the peak test runs in registers and only
// the two run ends cross lanes.
template <int NA>
__host__ __device__ constexpr int tile_pos(int t, int n) { return 2 * NA * (n >> 1) + 2 * t + (n & 1); }

// Floor (Q12), neighbour exchange, peak test (Q9/Q10), candidate append and optional fp32 P for
// one accumulator set; v[j] (j = 2t + e) is the lane's angle at block position 16q + j.
// REV: the set holds grid index L-1-i at tile index i (mirrored half).
// Decided tile indices: interior positions 1..W-2 with i in [ilo, ihi]; P written for i in [0, whi].
// Deferred candidate store: the lane's first candidate of an epilogue takes its slot with an atomic
// whose result is consumed only at the lane's next epilogue (or the kernel's end), so the global
// atomic's round trip overlaps the warp's next DMMA phase instead of stalling the epilogue (and with
// it the other warp group's turn).  Further candidates of the same epilogue are stored at once.
struct PendingCand {
  int slot, b, idx;
  long long f;
};
__device__ __forceinline__ void flush_cand(PendingCand& pc, int cap, int32_t* __restrict__ cidx,
                                           double* __restrict__ cf) {
  if (pc.slot >= 0 && pc.slot < cap) {
    cidx[(size_t)pc.b * cap + pc.slot] = pc.idx;
    cf[(size_t)pc.b * cap + pc.slot] = __longlong_as_double(pc.f);
  }
  pc.slot = -1;
}

template <int NA, bool WRITE_P, bool REV>
__device__ __forceinline__ void scan_epilogue(long long (&v)[2 * NA], int lane, int base, int ilo, int ihi, int whi,
                                              int L, int b, bool frame_ok, int cap, int32_t* __restrict__ cnt,
                                              int32_t* __restrict__ cidx, double* __restrict__ cf,
                                              float* __restrict__ P, PendingCand& pc) {
  constexpr int W = 8 * NA, R = 2 * NA;
  const int q = lane & 3;
  // Fast path: if every value of the warp's tile is a positive double above the floor and not NaN
  // (checked on the high words, conservatively), the raw bits already are the floored values;
  // otherwise the whole tile takes the explicit floor, which maps negative values, +-0 and NaNs to
  // 1e-300 like the oracle's max(f, 1e-300) (Q12).  For positive doubles the IEEE bits order like
  // the values, so the whole test runs in the integer domain and the FP64 pipe stays with the DMMAs.
  int hmin = 0x7FFFFFFF, hmax = (int)0x80000000;
#pragma unroll
  for (int j = 0; j < R; ++j) {
    const int hi = (int)(v[j] >> 32);
    hmin = min(hmin, hi);
    hmax = max(hmax, hi);
  }
  if (__any_sync(0xffffffffu, hmin <= (int)(kFloorBits >> 32) || hmax >= (int)(kInfBits >> 32))) {
#pragma unroll
    for (int j = 0; j < R; ++j) {
      long long x = v[j];
      x = x > kInfBits ? kFloorBits : x;
      v[j] = x > kFloorBits ? x : kFloorBits;
    }
  }
  // run ends: left of v[0] is lane q-1's v[R-1], right of v[R-1] is lane q+1's v[0]; positions 0
  // and W-1 of the block are halo and never decided, so q = 0 / q = 3 take any value.
  const long long vl = __shfl_sync(0xffffffffu, v[R - 1], q > 0 ? lane - 1 : lane);
  const long long vr = __shfl_sync(0xffffffffu, v[0], q < 3 ? lane + 1 : lane);
  // Forward (Q10: f_i < f_{i-1} and f_i <= f_{i+1}): with d_j = v_j < v_{j-1}, j is a minimum iff
  // d_j && !d_{j+1}.  REV (grid index decreasing along the run): g_j = v_{j-1} < v_j, j is a
  // minimum iff g_{j+1} && !g_j.
  unsigned m = 0;
#pragma unroll
  for (int j = 0; j <= R; ++j) {
    const long long cur = j < R ? v[j] : vr;
    const long long prv = j > 0 ? v[j - 1] : vl;
    m |= (unsigned)(REV ? (prv < cur) : (cur < prv)) << j;
  }
  unsigned hit = REV ? ((m >> 1) & ~m) : (m & ~(m >> 1));
  hit &= (1u << R) - 1;
  if (!frame_ok) hit = 0;
  while (hit) {                                            // local maxima of P (rare)
    const int j = __ffs(hit) - 1;
    hit &= hit - 1;
    const int pos = R * q + j, i = base + pos;
    if (pos < 1 || pos > W - 2 || i < ilo || i > ihi) continue;   // halo / grid ends (Q9)
    long long f;                                           // v[j]: select tree on the bits of j
    {
      long long t[R / 2];
#pragma unroll
      for (int k = 0; k < R / 2; ++k) t[k] = (j & 1) ? v[2 * k + 1] : v[2 * k];
#pragma unroll
      for (int w = R / 4, bit = 2; w >= 1; w /= 2, bit *= 2)
#pragma unroll
        for (int k = 0; k < w; ++k) t[k] = (j & bit) ? t[2 * k + 1] : t[2 * k];
      f = t[0];
    }
    if (pc.slot < 0) {                                     // deferred: stored at the next flush
      pc.slot = atomicAdd(cnt + b, 1);
      pc.b = b;
      pc.idx = REV ? L - 1 - i : i;
      pc.f = f;
      continue;
    }
    const int slot = atomicAdd(cnt + b, 1);
    if (slot < cap) {
      cidx[(size_t)b * cap + slot] = REV ? L - 1 - i : i;
      cf[(size_t)b * cap + slot] = __longlong_as_double(f);
    }
  }
  if (WRITE_P && frame_ok) {
    float* Pb = P + (size_t)b * L;
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const int pos = R * q + j, i = base + pos;
      if (pos >= 1 && pos <= W - 2 && i >= 0 && i <= whi) Pb[REV ? L - 1 - i : i] = to_p32(__longlong_as_double(v[j]));
    }
  }
}

template <int S, bool WRITE_P, bool MIRROR>
__global__ void __launch_bounds__(kCtaWarps * 32, kScanMinBlocks) scan_cta_kernel(const double* __restrict__ coef, int64_t B, int M,
                                                                   int64_t per, double dl, double theta0, double dtheta, int L,
                                                                   bool sym, int cap, int32_t* __restrict__ cnt,
                                                                   int32_t* __restrict__ cidx,
                                                                   double* __restrict__ cf, float* __restrict__ P) {
  using Shape = ScanShape<S, MIRROR>;
  constexpr int NA = Shape::NA, W = Shape::W, NB = Shape::NB, SE = Shape::SE;
  constexpr bool STREAM_A = Shape::STREAM_A;
  constexpr int SA = STREAM_A ? 1 : S;                           // register-held A fragments
  extern __shared__ double Ts[];                                 // [NB][S][NA][32]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r = lane >> 2;
  const int H = (L + 1) / 2;                                     // lower half [0, H) (MIRROR)
  const int Lt = MIRROR ? H + 1 : L;                             // table-valid tile indices [0, Lt)
  const int64_t ngroups = (B + 7) / 8;
  const int64_t y = blockIdx.y;
  const int blk0 = (int)blockIdx.x * NB;
  for (int e = threadIdx.x; e < NB * S * NA * 32; e += kCtaWarps * 32) {
    const int ln = e & 31, t = (e >> 5) % NA, s = (e / (32 * NA)) % S, k = e / (32 * NA * S);
    const int i = (blk0 + k) * (W - 2) - 1 + tile_pos<NA>(t, ln >> 2);
    const int j = 4 * s + (ln & 3);
    double v = (j == 0) ? 1.0 : 0.0;
    if (i >= 0 && i < Lt) v = table_entry(j, M, grid_u(i, theta0, dtheta, dl, L, sym));
    Ts[e] = v;
  }
  __syncthreads();
  const int64_t g0 = y * per;
  const int64_t g1 = (g0 + per < ngroups) ? g0 + per : ngroups;
  // Ping-pong: warps 0-3 and 4-7 take turns on the DMMA pipe — a warp group issues
  // its block's DMMAs, hands the pipe to the other group (named barriers 1/2) and runs its
  // epilogue while the other group's DMMAs execute, so the pipe never idles on an epilogue phase
  // that all warps would otherwise reach together.  Trip counts are CTA-uniform (warps past the
  // chunk's last group still take their turns, without work).
  const int wg = warp >> 2;
  const int64_t nit = (g1 - g0 + kCtaWarps - 1) / kCtaWarps;
  PendingCand pcand;
  pcand.slot = -1; pcand.b = 0; pcand.idx = 0; pcand.f = 0;
  if (wg == 1) bar_arrive(1);
  for (int64_t it = 0; it < nit; ++it) {
    const int64_t g = g0 + warp + it * kCtaWarps;
    const bool gv = g < g1;                                      // warp-uniform
    const double* cgc = coef + ((size_t)g * S) * 32 + lane;   // this group's A fragments
    double a[SA];
    if (!STREAM_A && gv) {
      // this group's operands, loaded before the turn barrier: the L2 round trip overlaps the wait
      // (a one-group-ahead prefetch held 16 more registers and was 2.5% slower)
#pragma unroll
      for (int s = 0; s < SA; ++s) a[s] = __ldg(cgc + s * 32);
    }
    const int b = (int)(g * 8) + r;
    const bool frame_ok = gv && b < B;
#pragma unroll 1
    for (int k = 0; k < NB; ++k) {
      const int base = (blk0 + k) * (W - 2) - 1;
      if (base + 1 >= (MIRROR ? H : L)) break;                 // CTA-uniform
      const double* Tk = Ts + (size_t)k * S * NA * 32 + lane;
      double acc[NA][2], aco[MIRROR ? NA : 1][2];
#pragma unroll
      for (int t = 0; t < NA; ++t) { acc[t][0] = 0.0; acc[t][1] = 0.0; }
      if (MIRROR) {
#pragma unroll
        for (int t = 0; t < (MIRROR ? NA : 1); ++t) { aco[t][0] = 0.0; aco[t][1] = 0.0; }
      }
      bar_sync(1 + wg);                         // my group's turn on the pipe
      if (gv) {
        if (!MIRROR) {
#pragma unroll
          for (int s = 0; s < S; ++s) {
            const double av = STREAM_A ? __ldg(cgc + s * 32) : a[STREAM_A ? 0 : s];
#pragma unroll
            for (int t = 0; t < NA; ++t) dmma_884(acc[t][0], acc[t][1], av, Tk[(s * NA + t) * 32]);
          }
        } else {
          // O chains first, then the E chains accumulate onto O: acc = E + O = f_i directly, and
          // f_{L-1-i} = E - O = acc - 2 O takes one DFMA per element (two separate chains combined
          // with two DADDs per element were 6% slower: the DADDs share the FP64 datapath)
#pragma unroll
          for (int s = 0; SE + s < S; ++s) {
            const double ao = STREAM_A ? __ldg(cgc + (SE + s) * 32) : a[STREAM_A ? 0 : SE + s];
#pragma unroll
            for (int t = 0; t < NA; ++t) dmma_884(aco[MIRROR ? t : 0][0], aco[MIRROR ? t : 0][1], ao, Tk[((SE + s) * NA + t) * 32]);
          }
#pragma unroll
          for (int s = 0; s < SE; ++s) {
            const double ae = STREAM_A ? __ldg(cgc + s * 32) : a[STREAM_A ? 0 : s];
#pragma unroll
            for (int t = 0; t < NA; ++t) {
              if (s == 0) dmma_884c(acc[t][0], acc[t][1], ae, Tk[t * 32], aco[MIRROR ? t : 0][0], aco[MIRROR ? t : 0][1]);
              else dmma_884(acc[t][0], acc[t][1], ae, Tk[(s * NA + t) * 32]);
            }
          }
        }
      }
      bar_arrive(2 - wg);                       // hand the pipe to the other group
      if (!gv) continue;
      flush_cand(pcand, cap, cidx, cf);                // the previous epilogue's deferred candidate
      if (!MIRROR) {
        long long fi[2 * NA];
#pragma unroll
        for (int t = 0; t < NA; ++t) {
          fi[2 * t] = __double_as_longlong(acc[t][0]);
          fi[2 * t + 1] = __double_as_longlong(acc[t][1]);
        }
        scan_epilogue<NA, WRITE_P, false>(fi, lane, base, 1, L - 2, L - 1, L, b, frame_ok, cap, cnt, cidx, cf, P, pcand);
      } else {
        long long fl[2 * NA], fh[2 * NA];
#pragma unroll
        for (int t = 0; t < NA; ++t)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const double ev = acc[t][e], od = aco[MIRROR ? t : 0][e];
            fl[2 * t + e] = __double_as_longlong(ev);                    // f_i       = (O + E)
            fh[2 * t + e] = __double_as_longlong(fma(-2.0, od, ev));     // f_{L-1-i} = f_i - 2 O
          }
        scan_epilogue<NA, WRITE_P, false>(fl, lane, base, 1, H - 1, H - 1, L, b, frame_ok, cap, cnt, cidx, cf, P, pcand);
        scan_epilogue<NA, WRITE_P, true>(fh, lane, base, 1, L - 1 - H, L - 1 - H, L, b, frame_ok, cap, cnt, cidx, cf, P, pcand);
      }
    }
  }
  flush_cand(pcand, cap, cidx, cf);
  if (wg == 0) bar_sync(1);                       // consume the other group's last hand-off
}

template <int S, bool MIRROR>
cudaError_t launch_scan_cta(const doa_plan_s* p, int64_t B, float* P, cudaStream_t s) {
  using Shape = ScanShape<S, MIRROR>;
  constexpr int NA = Shape::NA, W = Shape::W, NB = Shape::NB;
  const size_t smem = (size_t)NB * S * NA * 32 * sizeof(double);
  const int occ = kernel_occupancy(scan_cta_kernel<S, false, MIRROR>, kCtaWarps * 32, smem);
  if (P) kernel_occupancy(scan_cta_kernel<S, true, MIRROR>, kCtaWarps * 32, smem);   // sets its smem attribute
  const int64_t span = MIRROR ? (p->L + 1) / 2 : p->L;          // tile indices the blocks own
  const int64_t nwb = (span + (W - 2) - 1) / (W - 2);            // angle blocks owning [0, span)
  const int64_t gx = (nwb + NB - 1) / NB;                        // angle columns
  const int64_t ngroups = (B + 7) / 8;
  const int64_t slots = (int64_t)sm_count() * occ;
  // frame chunks.  Large batches: ~4 waves of resident CTAs with >= 64 groups (8 per warp) per CTA.
  // Small batches (fewer than 4 waves' worth of 256-group CTAs): k whole waves (gx * gy <= k *
  // slots) of CTAs with >= 256 groups each, so the per-CTA steering table stays amortised (B = 8192
  // at c4: one wave of 512-group CTAs, 0.202 -> 0.183 ms per launch; profiles/scan_ab_r02x.txt).
  const int64_t kw = (gx * ngroups) / (slots * 256);
  int64_t per, gy;
  if (kw >= DOA_SCAN_WAVES) {
    per = (gx * ngroups) / (DOA_SCAN_WAVES * slots);
    if (per < 64) per = 64;
    if (per > ngroups) per = ngroups;
    gy = (ngroups + per - 1) / per;
  } else {
    gy = ((kw < 1 ? 1 : kw) * slots) / gx;
    if (gy < 1) gy = 1;
    if (gy > ngroups) gy = ngroups;
    per = (ngroups + gy - 1) / gy;
  }
  const dim3 grid((unsigned)gx, (unsigned)gy);
  const bool sym = p->sym != 0;
  count_launch();
  if (P)
    scan_cta_kernel<S, true, MIRROR><<<grid, kCtaWarps * 32, smem, s>>>(
        p->coef, B, p->M, per, p->dl, p->theta0, p->dtheta, (int)p->L, sym, p->cap, p->cnt, p->cand_idx, p->cand_f, P);
  else
    scan_cta_kernel<S, false, MIRROR><<<grid, kCtaWarps * 32, smem, s>>>(
        p->coef, B, p->M, per, p->dl, p->theta0, p->dtheta, (int)p->L, sym, p->cap, p->cnt, p->cand_idx, p->cand_f, P);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// S7: one warp per (plan, frame).  Rank every stored candidate by (f ascending, index ascending)
// and scatter the first D (PeakSelection; Q11).  One launch serves up to kMaxCoefPlans
// plans (blockIdx.y = plan).
__global__ void __launch_bounds__(128) select_kernel(int64_t B, int D, SelectPlans sp) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t b = (int64_t)blockIdx.x * 4 + warp;
  const int a = blockIdx.y;
  if (b >= B) return;
  const int cap = sp.cap[a];
  const int nraw = sp.cnt[a][b];
  const int n = nraw < cap ? nraw : cap;
  const int32_t* ci = sp.cidx[a] + (size_t)b * cap;
  const double* cfv = sp.cf[a] + (size_t)b * cap;
  int32_t* idx = sp.idx[a];
  float* val = sp.val[a];
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
    sp.npk[a][b] = n < D ? n : D;
    int fl = 0;
    if (nraw > cap) fl |= DOA_INFO_CAND_OVERFLOW;
    if (n < D) fl |= DOA_INFO_UNDERDETERMINED;
    if (fl) sp.info[a][b] |= fl;
  }
}

}  // namespace

cudaError_t launch_coef_multi(const doa_plan_s* const* plans, int nplans, const double* lam, const double* V,
                              int64_t B, int32_t* const* info, cudaStream_t s) {
  const int M = plans[0]->M;
  if (M <= 16) {
    CoefPlans cp = {};
    for (int a0 = 0; a0 < nplans; a0 += kMaxCoefPlans) {
      cp.nplans = nplans - a0 < kMaxCoefPlans ? nplans - a0 : kMaxCoefPlans;
      for (int a = 0; a < cp.nplans; ++a) {
        const doa_plan_s* q = plans[a0 + a];
        cp.alg[a] = q->alg; cp.coef[a] = q->coef; cp.cnt[a] = q->cnt; cp.info[a] = info[a0 + a];
      }
      const size_t smem = (size_t)kCoefMmaWarps * 2 * kCoefMmaPlane * sizeof(double);
      const int occ = kernel_occupancy(coef_mma_kernel, kCoefMmaWarps * 32, smem);
      int64_t nb = (B + kCoefMmaWarps - 1) / kCoefMmaWarps;
      const int64_t slots = (int64_t)sm_count() * occ * kCoefWaves;
      if (nb > slots) nb = slots;
      count_launch();
      coef_mma_kernel<<<(unsigned)nb, kCoefMmaWarps * 32, smem, s>>>(lam, reinterpret_cast<const double2*>(V), B, M,
                                                                     plans[0]->D, cp);
      const cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
  for (int a = 0; a < nplans; ++a) {
    const doa_plan_s* p = plans[a];
    auto go = [&](auto kern, size_t smem) {
      kernel_occupancy(kern, kCoefBigWarps * 32, smem);               // sets the smem attribute
      count_launch();
      kern<<<(unsigned)B, kCoefBigWarps * 32, smem, s>>>(lam, reinterpret_cast<const double2*>(V), B, M, p->D, p->alg,
                                                         p->coef, p->cnt, info[a]);
    };
    if (M <= 32) go(coef_big_kernel<32>, CoefBig<32>::SMEM);
    else go(coef_big_kernel<64>, CoefBig<64>::SMEM);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_coef(const doa_plan_s* p, const double* lam, const double* V, int64_t B, int32_t* info,
                        cudaStream_t s) {
  return launch_coef_multi(&p, 1, lam, V, B, &info, s);
}

bool direct_compatible(const doa_plan_s* a, const doa_plan_s* b) {
  return a->geom == 0 && b->geom == 0 && a->M == b->M && a->dl == b->dl && a->theta0 == b->theta0 &&
         a->dtheta == b->dtheta && a->L == b->L && a->mirror == b->mirror && a->cap == b->cap && a->engine == b->engine;
}

// S4-S6 for up to kMaxCoefPlans direct-compatible ULA plans whose coefficients are in place (and
// counters zeroed): small batches take ONE direct-scan launch for all the plans (the steering is
// generated once per angle), larger ones one DMMA scan launch per plan.  (A single DMMA launch
// whose frame groups ran over all the plans — the steering table of a CTA serving every plan — was
// measured no faster on c4 and its per-group plan selection cost the kernel 7%; see
// profiles/README.md.)  P (single plan only) nullable.
cudaError_t launch_scan_plans(const doa_plan_s* const* plans, int nplans, int64_t B, float* P, cudaStream_t s) {
  const doa_plan_s* p = plans[0];
  if (B <= kDirectMaxB) {                                 // small batch: direct scan (scan_direct.cu)
    DirectScanArgs a = {};
    a.nplans = nplans;
    for (int k = 0; k < nplans; ++k) {
      a.coef[k] = plans[k]->coef; a.cnt[k] = plans[k]->cnt; a.cidx[k] = plans[k]->cand_idx;
      a.cf[k] = plans[k]->cand_f; a.P[k] = nplans == 1 ? P : nullptr;
    }
    return launch_scan_direct(a, p, B, s);
  }
  if (nplans > 1) {
    for (int k = 0; k < nplans; ++k) {
      const cudaError_t e = launch_scan_plans(plans + k, 1, B, nullptr, s);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
  switch (ksteps(p->M)) {
#define DOA_SCAN_CASE(k) \
  case k: return p->mirror ? launch_scan_cta<k, true>(p, B, P, s) : launch_scan_cta<k, false>(p, B, P, s);
    DOA_SCAN_CASE(1) DOA_SCAN_CASE(2) DOA_SCAN_CASE(3) DOA_SCAN_CASE(4) DOA_SCAN_CASE(5) DOA_SCAN_CASE(6)
    DOA_SCAN_CASE(7) DOA_SCAN_CASE(8) DOA_SCAN_CASE(9) DOA_SCAN_CASE(10) DOA_SCAN_CASE(11) DOA_SCAN_CASE(12)
    DOA_SCAN_CASE(13) DOA_SCAN_CASE(14) DOA_SCAN_CASE(15) DOA_SCAN_CASE(16) DOA_SCAN_CASE(17) DOA_SCAN_CASE(18)
    DOA_SCAN_CASE(19) DOA_SCAN_CASE(20) DOA_SCAN_CASE(21) DOA_SCAN_CASE(22) DOA_SCAN_CASE(23) DOA_SCAN_CASE(24)
    DOA_SCAN_CASE(25) DOA_SCAN_CASE(26) DOA_SCAN_CASE(27) DOA_SCAN_CASE(28) DOA_SCAN_CASE(29) DOA_SCAN_CASE(30)
    DOA_SCAN_CASE(31) DOA_SCAN_CASE(32)
#undef DOA_SCAN_CASE
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_scan(const doa_plan_s* p, int64_t B, float* P, cudaStream_t s) {
  return launch_scan_plans(&p, 1, B, P, s);
}

cudaError_t launch_select_multi(const SelectPlans& sp, int D, int64_t B, cudaStream_t s) {
  if (B <= 0 || sp.nplans <= 0) return cudaSuccess;
  count_launch();
  select_kernel<<<dim3((unsigned)((B + 3) / 4), (unsigned)sp.nplans), 128, 0, s>>>(B, D, sp);
  return cudaGetLastError();
}

cudaError_t launch_select(const doa_plan_s* p, int64_t B, int32_t* idx, float* val, int32_t* npk, int32_t* info,
                          cudaStream_t s) {
  SelectPlans sp = {};
  sp.nplans = 1;
  sp.cnt[0] = p->cnt; sp.cidx[0] = p->cand_idx; sp.cf[0] = p->cand_f; sp.cap[0] = p->cap;
  sp.idx[0] = idx; sp.val[0] = val; sp.npk[0] = npk; sp.info[0] = info;
  return launch_select_multi(sp, p->D, B, s);
}

}  // namespace doa
