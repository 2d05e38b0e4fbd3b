// S2 — batched Hermitian eigendecomposition (Table 2 Step-2 `jsvd`; read as the
// eigendecomposition of the Hermitian PSD covariance, Q3), one warp per matrix.
//
// Parallel cyclic Jacobi with the round-robin ("circle") ordering: n/2 disjoint rotations per
// round, n-1 rounds per sweep (n = M rounded up to even; an odd M gets a decoupled zero dummy
// index that no rotation ever touches).  All rotations of a round are computed from the same
// iterate and applied together: A <- J^H A J, V <- V J with J = prod_k J_k (disjoint blocks).
// Each J_k is Golub & Van Loan's sym.schur2 after the phase rotation diag(1, e^{-j phi}) that
// makes a_pq real (the same rotation family as the oracle's cyclic-by-rows sweep, but a different
// ordering — the two implementations share no code).
// A and V live in shared memory (padded rows); fp64 throughout; the stop rule is
// off(A) = sqrt(sum_{i!=j} |a_ij|^2) <= 10 eps ||R||_F evaluated directly at the start of every
// sweep, capped at 30 sweeps (Q15).  Eigenvalues are sorted ascending, ties by index (Q2).
#include <cfloat>
#include <cstdlib>

#include "doa_internal.cuh"

namespace doa {
namespace {

struct Rot {
  double c, s, er, ei;   // J = diag(1, e) [[c, s], [-s, c]],  e = er + j ei = e^{-j phi}
  int p, q;
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int MAXM, int WARPS>
__global__ void __launch_bounds__(WARPS * 32) eig_kernel(const double2* __restrict__ R, int64_t B, int M,
                                                 double* __restrict__ lam_out, double2* __restrict__ V_out,
                                                 int32_t* __restrict__ info) {
  constexpr int LD = MAXM + 1;
  extern __shared__ double2 smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t b = (int64_t)blockIdx.x * WARPS + warp;
  if (b >= B) return;
  double2* A = smem + (size_t)warp * (2 * MAXM * LD);
  double2* V = A + MAXM * LD;
  __shared__ Rot rot[WARPS][MAXM / 2];
  __shared__ int rank_s[WARPS][MAXM];
  const int n = (M + 1) & ~1;
  const int h = n / 2;
  const double2* Rb = R + (size_t)b * M * M;

  double nrm = 0.0;
  for (int e = lane; e < n * n; e += 32) {
    const int i = e / n, j = e - (e / n) * n;
    double2 v = make_double2(0.0, 0.0);
    if (i < M && j < M) {
      if (i <= j) v = Rb[(size_t)i * M + j];
      else { const double2 t = Rb[(size_t)j * M + i]; v = make_double2(t.x, -t.y); }
      if (i == j) v.y = 0.0;
    }
    A[i * LD + j] = v;
    V[i * LD + j] = make_double2(i == j ? 1.0 : 0.0, 0.0);
    nrm += v.x * v.x + v.y * v.y;
  }
  nrm = sqrt(warp_sum(nrm));
  const double tol = 10.0 * DBL_EPSILON * nrm;
  __syncwarp();

  int sweep = 0;
  int flag = 0;
  for (;; ++sweep) {
    double off = 0.0;
    for (int e = lane; e < n * n; e += 32) {
      const int i = e / n, j = e - (e / n) * n;
      if (i != j) { const double2 v = A[i * LD + j]; off += v.x * v.x + v.y * v.y; }
    }
    off = sqrt(warp_sum(off));
    if (off <= tol) break;
    if (sweep == kMaxSweeps) { flag |= DOA_INFO_NOCONV; break; }
    for (int r = 0; r < n - 1; ++r) {
      // phase 1: rotation parameters of the round's n/2 disjoint pairs
      if (lane < h) {
        int p, q;
        if (lane == 0) { p = r; q = n - 1; }
        else { p = (r + lane) % (n - 1); q = (r - lane + (n - 1)) % (n - 1); }
        if (p > q) { const int t = p; p = q; q = t; }
        const double2 apq = A[p * LD + q];
        const double rr = sqrt(apq.x * apq.x + apq.y * apq.y);
        Rot ro;
        ro.p = p; ro.q = q;
        if (rr == 0.0) { ro.c = 1.0; ro.s = 0.0; ro.er = 1.0; ro.ei = 0.0; }
        else {
          const double app = A[p * LD + p].x, aqq = A[q * LD + q].x;
          ro.er = apq.x / rr; ro.ei = -apq.y / rr;                      // conj(a_pq)/|a_pq|
          const double tau = (aqq - app) / (2.0 * rr);
          const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
          ro.c = 1.0 / sqrt(1.0 + t * t);
          ro.s = t * ro.c;
        }
        rot[warp][lane] = ro;
      }
      __syncwarp();
      // phase 2: A <- A J (columns p, q of every row)
      for (int e = lane; e < n * h; e += 32) {
        const int i = e / h, k = e - (e / h) * h;
        const Rot ro = rot[warp][k];
        const double2 x = A[i * LD + ro.p], y = A[i * LD + ro.q];
        // e*y
        const double eyr = ro.er * y.x - ro.ei * y.y, eyi = ro.er * y.y + ro.ei * y.x;
        A[i * LD + ro.p] = make_double2(ro.c * x.x - ro.s * eyr, ro.c * x.y - ro.s * eyi);
        A[i * LD + ro.q] = make_double2(ro.s * x.x + ro.c * eyr, ro.s * x.y + ro.c * eyi);
      }
      __syncwarp();
      // phase 3: A <- J^H A (rows p, q of every column) and V <- V J
      for (int e = lane; e < n * h; e += 32) {
        const int j = e / h, k = e - (e / h) * h;
        const Rot ro = rot[warp][k];
        const double2 x = A[ro.p * LD + j], y = A[ro.q * LD + j];
        // conj(e)*y
        const double eyr = ro.er * y.x + ro.ei * y.y, eyi = ro.er * y.y - ro.ei * y.x;
        A[ro.p * LD + j] = make_double2(ro.c * x.x - ro.s * eyr, ro.c * x.y - ro.s * eyi);
        A[ro.q * LD + j] = make_double2(ro.s * x.x + ro.c * eyr, ro.s * x.y + ro.c * eyi);
        const double2 vx = V[j * LD + ro.p], vy = V[j * LD + ro.q];
        const double vyr = ro.er * vy.x - ro.ei * vy.y, vyi = ro.er * vy.y + ro.ei * vy.x;
        V[j * LD + ro.p] = make_double2(ro.c * vx.x - ro.s * vyr, ro.c * vx.y - ro.s * vyi);
        V[j * LD + ro.q] = make_double2(ro.s * vx.x + ro.c * vyr, ro.s * vx.y + ro.c * vyi);
      }
      __syncwarp();
      // phase 4: exact zeros on the rotated pairs, real diagonal
      if (lane < h) {
        const Rot ro = rot[warp][lane];
        if (ro.s != 0.0 || ro.er != 1.0 || ro.ei != 0.0) {
          A[ro.p * LD + ro.q] = make_double2(0.0, 0.0);
          A[ro.q * LD + ro.p] = make_double2(0.0, 0.0);
        }
        A[ro.p * LD + ro.p].y = 0.0;
        A[ro.q * LD + ro.q].y = 0.0;
      }
      __syncwarp();
    }
  }

  // ascending stable sort of the diagonal (ties by index), permute V's columns
  for (int i = lane; i < M; i += 32) {
    const double li = A[i * LD + i].x;
    int rk = 0;
    for (int j = 0; j < M; ++j) {
      const double lj = A[j * LD + j].x;
      rk += (lj < li) || (lj == li && j < i);
    }
    rank_s[warp][i] = rk;
    lam_out[(size_t)b * M + rk] = li;
  }
  __syncwarp();
  double2* Vb = V_out + (size_t)b * M * M;
  for (int e = lane; e < M * M; e += 32) {
    const int i = e / M, j = e - (e / M) * M;
    Vb[(size_t)i * M + rank_s[warp][j]] = V[i * LD + j];
  }
  if (lane == 0) info[b] = flag;
}

template <int MAXM, int WARPS>
cudaError_t launch_eig_t(const double* R, int64_t B, int M, double* lam, double* V, int32_t* info, cudaStream_t s) {
  constexpr int LD = MAXM + 1;
  const size_t smem = (size_t)WARPS * 2 * MAXM * LD * sizeof(double2);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(eig_kernel<MAXM, WARPS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  count_launch();
  eig_kernel<MAXM, WARPS><<<(unsigned)((B + WARPS - 1) / WARPS), WARPS * 32, smem, s>>>(reinterpret_cast<const double2*>(R), B, M, lam,
                                                             reinterpret_cast<double2*>(V), info);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_eig16(const double* R, int64_t B, int M, double* lam, double* V, int32_t* info, cudaStream_t s);

cudaError_t launch_eig(const double* R, int64_t B, int M, double* lam, double* V, int32_t* info, cudaStream_t s) {
  static const bool legacy = getenv("DOA_EIG_SMEM") != nullptr;   // A/B switch for tuning only
  if (M <= 16 && !legacy) return launch_eig16(R, B, M, lam, V, info, s);
  if (M <= 16) return launch_eig_t<16, 4>(R, B, M, lam, V, info, s);
  if (M <= 32) return launch_eig_t<32, 2>(R, B, M, lam, V, info, s);
  return launch_eig_t<64, 1>(R, B, M, lam, V, info, s);
}

}  // namespace doa
