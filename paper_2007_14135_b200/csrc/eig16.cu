// S2 for M <= 16: batched Hermitian Jacobi eigendecomposition, one warp per matrix, with the
// eigenvector matrix resident in registers.  (Table 2 Step-2 `jsvd`; Q3.)
//
// Ordering: parallel cyclic Jacobi, circle-method round robin on n = 16 indices (M < 16 is padded
// with decoupled zero indices that no rotation ever touches).  The 8 disjoint pairs of a round
// always sit in fixed SLOTS (0,1), (2,3), ..., (14,15); after each round the slot contents move by
// the fixed "caterpillar" permutation pi (slot 0 fixed, the other 15 slots rotate along one circle),
// so every pair of indices meets exactly once per 15-round sweep.  sigma[slot] = logical index.
//
//   A (Hermitian, logical indexing, upper triangle only) lives in shared memory.  Per round:
//     phase 1  lanes 0..7   : rotation of slot-pair k from (a_xx, a_yy, a_xy), x = sigma[2k],
//                             y = sigma[2k+1]; the 2x2 diagonal block gets its closed form
//                             (a_xx - t|a_xy|, a_yy + t|a_xy|, 0) (Golub & Van Loan sym.schur2).
//     phase 2  lanes 0..27  : one off-diagonal 2x2 block (slot pairs r < s): B <- J_r^H B J_s.
//              all 32 lanes : V <- V J on registers.
//   V lives in registers: lane (row i = lane % 16, half h = lane / 16) holds V[i][slots 8h..8h+7];
//     its 4 slot pairs are local, and pi moves only two slots across halves per round (one
//     complex shuffle).
// Rotations: J = diag(1, e) [[c, s], [-s, c]], e = conj(a_xy)/|a_xy|, tau = (a_yy - a_xx)/(2|a_xy|),
// t = sign(tau)/(|tau| + sqrt(1 + tau^2)), c = 1/sqrt(1 + t^2), s = t c; skipped when a_xy == 0.
// Stop rule at the start of every sweep: off(A) = sqrt(sum_{i != j} |a_ij|^2) <= 10 eps ||R||_F,
// at most 30 sweeps (Q15).  Eigenvalues ascending, ties by logical index (Q2).
#include <cfloat>

#include "doa_internal.cuh"

namespace doa {
namespace {

constexpr int kN = 16;            // padded order
constexpr int kLd = 17;           // smem row stride (double2)
constexpr int kEigWarps = 4;

struct Prm {
  double c, s, er, ei;
};

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// canonical Hermitian access: element (i, j) of the logical matrix, stored at [min][max]
__device__ __forceinline__ double2 aget(const double2* A, int i, int j) {
  if (i <= j) return A[i * kLd + j];
  const double2 v = A[j * kLd + i];
  return make_double2(v.x, -v.y);
}
__device__ __forceinline__ void aset(double2* A, int i, int j, double2 v) {
  if (i <= j) A[i * kLd + j] = v;
  else A[j * kLd + i] = make_double2(v.x, -v.y);
}

// caterpillar: next slot of slot s
__device__ __forceinline__ int cat_next(int s) {
  if (s == 0) return 0;
  if (s == 1) return 2;
  if (s == 14) return 15;
  return (s & 1) ? s - 2 : s + 2;
}

__global__ void __launch_bounds__(kEigWarps * 32) eig16_kernel(const double2* __restrict__ R, int64_t B, int M,
                                                             double* __restrict__ lam_out,
                                                             double2* __restrict__ V_out,
                                                             int32_t* __restrict__ info) {
  __shared__ double2 As[kEigWarps][kN * kLd];
  __shared__ Prm prm[kEigWarps][kN / 2];
  __shared__ int sig[kEigWarps][2][kN];
  __shared__ int rank_s[kEigWarps][kN];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t b = (int64_t)blockIdx.x * kEigWarps + warp;
  if (b >= B) return;
  double2* A = As[warp];
  const double2* Rb = R + (size_t)b * M * M;

  // load the upper triangle (zero-padded to 16) and ||R||_F
  double nrm = 0.0;
  for (int e = lane; e < kN * kN; e += 32) {
    const int i = e >> 4, j = e & 15;
    if (i > j) continue;
    double2 v = make_double2(0.0, 0.0);
    if (j < M) v = Rb[(size_t)i * M + j];
    if (i == j) v.y = 0.0;
    A[i * kLd + j] = v;
    nrm += (i == j ? 1.0 : 2.0) * (v.x * v.x + v.y * v.y);
  }
  if (lane < kN) sig[warp][0][lane] = lane;
  nrm = sqrt(wsum(nrm));
  const double tol = 10.0 * DBL_EPSILON * nrm;

  // V registers: row vi, slots 8h..8h+7 (initially slot == logical index, V = I)
  const int vi = lane & 15, h = lane >> 4;
  double2 v[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) v[k] = make_double2(vi == 8 * h + k ? 1.0 : 0.0, 0.0);

  // this lane's off-diagonal slot-pair block (rb < sb), lanes 0..27
  int rb = 0, sb = 0;
  {
    int l = lane < 28 ? lane : 0;
    for (int r = 0; r < 8; ++r) {
      const int cntr = 7 - r;
      if (l < cntr) { rb = r; sb = r + 1 + l; break; }
      l -= cntr;
    }
  }
  __syncwarp();

  int flag = 0;
  int cur = 0;
  for (int sweep = 0;; ++sweep) {
    double off = 0.0;
    for (int e = lane; e < kN * kN; e += 32) {
      const int i = e >> 4, j = e & 15;
      if (i < j) { const double2 a = A[i * kLd + j]; off += a.x * a.x + a.y * a.y; }
    }
    off = sqrt(2.0 * wsum(off));
    if (off <= tol) break;
    if (sweep == kMaxSweeps) { flag |= DOA_INFO_NOCONV; break; }
    for (int rnd = 0; rnd < kN - 1; ++rnd) {
      const int* sc = sig[warp][cur];
      // ---- phase 1: rotation parameters + closed-form diagonal blocks
      if (lane < 8) {
        const int x = sc[2 * lane], y = sc[2 * lane + 1];
        const double2 axy = aget(A, x, y);
        const double r2 = axy.x * axy.x + axy.y * axy.y;
        Prm p;
        if (r2 == 0.0) {
          p.c = 1.0; p.s = 0.0; p.er = 1.0; p.ei = 0.0;
        } else {
          const double axx = A[x * kLd + x].x, ayy = A[y * kLd + y].x;
          const double rr = sqrt(r2);
          p.er = axy.x / rr;
          p.ei = -axy.y / rr;
          const double tau = (ayy - axx) / (2.0 * rr);
          const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
          p.c = 1.0 / sqrt(1.0 + t * t);
          p.s = t * p.c;
          A[x * kLd + x].x = axx - t * rr;
          A[y * kLd + y].x = ayy + t * rr;
          aset(A, x, y, make_double2(0.0, 0.0));
        }
        prm[warp][lane] = p;
      }
      __syncwarp();
      // ---- phase 2a: off-diagonal block (rb, sb): B <- J_r^H B J_s
      if (lane < 28) {
        const Prm pr = prm[warp][rb], ps = prm[warp][sb];
        const int xr = sc[2 * rb], yr = sc[2 * rb + 1], xs = sc[2 * sb], ys = sc[2 * sb + 1];
        double2 b00 = aget(A, xr, xs), b01 = aget(A, xr, ys), b10 = aget(A, yr, xs), b11 = aget(A, yr, ys);
        // columns: c0' = c b0 - s (e b1), c1' = s b0 + c (e b1), with e = e_s
        {
          double2 t0 = make_double2(ps.er * b01.x - ps.ei * b01.y, ps.er * b01.y + ps.ei * b01.x);
          double2 t1 = make_double2(ps.er * b11.x - ps.ei * b11.y, ps.er * b11.y + ps.ei * b11.x);
          const double2 n00 = make_double2(ps.c * b00.x - ps.s * t0.x, ps.c * b00.y - ps.s * t0.y);
          const double2 n01 = make_double2(ps.s * b00.x + ps.c * t0.x, ps.s * b00.y + ps.c * t0.y);
          const double2 n10 = make_double2(ps.c * b10.x - ps.s * t1.x, ps.c * b10.y - ps.s * t1.y);
          const double2 n11 = make_double2(ps.s * b10.x + ps.c * t1.x, ps.s * b10.y + ps.c * t1.y);
          b00 = n00; b01 = n01; b10 = n10; b11 = n11;
        }
        // rows: r0' = c r0 - s (conj(e) r1), r1' = s r0 + c (conj(e) r1), with e = e_r
        {
          const double2 t0 = make_double2(pr.er * b10.x + pr.ei * b10.y, pr.er * b10.y - pr.ei * b10.x);
          const double2 t1 = make_double2(pr.er * b11.x + pr.ei * b11.y, pr.er * b11.y - pr.ei * b11.x);
          aset(A, xr, xs, make_double2(pr.c * b00.x - pr.s * t0.x, pr.c * b00.y - pr.s * t0.y));
          aset(A, xr, ys, make_double2(pr.c * b01.x - pr.s * t1.x, pr.c * b01.y - pr.s * t1.y));
          aset(A, yr, xs, make_double2(pr.s * b00.x + pr.c * t0.x, pr.s * b00.y + pr.c * t0.y));
          aset(A, yr, ys, make_double2(pr.s * b01.x + pr.c * t1.x, pr.s * b01.y + pr.c * t1.y));
        }
      }
      // ---- phase 2b: V <- V J for this lane's four slot pairs (registers)
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const Prm p = prm[warp][4 * h + kk];
        const double2 vx = v[2 * kk], vy = v[2 * kk + 1];
        const double2 t = make_double2(p.er * vy.x - p.ei * vy.y, p.er * vy.y + p.ei * vy.x);
        v[2 * kk] = make_double2(p.c * vx.x - p.s * t.x, p.c * vx.y - p.s * t.y);
        v[2 * kk + 1] = make_double2(p.s * vx.x + p.c * t.x, p.s * vx.y + p.c * t.y);
      }
      // ---- caterpillar: slots move s -> pi(s) (sigma in smem, V in registers)
      if (lane < kN) sig[warp][cur ^ 1][cat_next(lane)] = sc[lane];
      {
        const double2 send = h ? v[1] : v[6];
        const double2 recv = make_double2(__shfl_xor_sync(0xffffffffu, send.x, 16),
                                          __shfl_xor_sync(0xffffffffu, send.y, 16));
        const double2 o0 = v[0], o1 = v[1], o2 = v[2], o3 = v[3], o4 = v[4], o5 = v[5], o6 = v[6], o7 = v[7];
        v[0] = h ? recv : o0;
        v[1] = o3;
        v[2] = h ? o0 : o1;
        v[3] = o5;
        v[4] = o2;
        v[5] = o7;
        v[6] = o4;
        v[7] = h ? o6 : recv;
      }
      cur ^= 1;
      __syncwarp();
    }
  }

  // ascending stable sort of the logical diagonal, then scatter V's columns (slot -> logical)
  const int* sc = sig[warp][cur];
  if (lane < M) {
    const double li = A[lane * kLd + lane].x;
    int rk = 0;
    for (int j = 0; j < M; ++j) {
      const double lj = A[j * kLd + j].x;
      rk += (lj < li) || (lj == li && j < lane);
    }
    rank_s[warp][lane] = rk;
    lam_out[(size_t)b * M + rk] = li;
  }
  __syncwarp();
  if (vi < M) {
    double2* Vrow = V_out + (size_t)b * M * M + (size_t)vi * M;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int j = sc[8 * h + k];
      if (j < M) Vrow[rank_s[warp][j]] = v[k];
    }
  }
  if (lane == 0) info[b] = flag;
}

}  // namespace

cudaError_t launch_eig16(const double* R, int64_t B, int M, double* lam, double* V, int32_t* info, cudaStream_t s) {
  count_launch();
  eig16_kernel<<<(unsigned)((B + kEigWarps - 1) / kEigWarps), kEigWarps * 32, 0, s>>>(
      reinterpret_cast<const double2*>(R), B, M, lam, reinterpret_cast<double2*>(V), info);
  return cudaGetLastError();
}

}  // namespace doa
