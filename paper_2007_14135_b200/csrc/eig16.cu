// S2 for M <= 16: batched Hermitian Jacobi eigendecomposition (Table 2 Step-2 `jsvd`, PAPER.md
// P:80; read as the Hermitian eigendecomposition, Q3).  Two kernels with bitwise identical results:
//   eig16h_kernel  (B >= 2048, throughput): two matrices per warp, one per 16-lane half;
//   eig16s_kernel  (B <  2048, latency):    one matrix per CTA of two warps, software-pipelined.
//
// Ordering: parallel cyclic Jacobi with the circle-method round robin on n = 16 indices (n = 8
// for M <= 8; M < n is padded with decoupled zero indices that no rotation ever touches).  The
// n/2 disjoint pairs of a round always sit in fixed SLOTS (0,1), (2,3), ...; after each round every
// index moves to the next slot of the "caterpillar" permutation pi (slot 0 fixed, the other slots
// along one (n-1)-cycle), so every pair of indices meets exactly once per sweep and, because
// pi^(n-1) = id, slots coincide with the original indices again at every sweep boundary.
//
//   A (Hermitian, physical slot order, upper triangle only) lives in shared memory,
//   double-buffered: each round reads buffer `cur` and writes every upper element of buffer `nxt`
//   at its PERMUTED position (pi(i), pi(j)) (conjugated when the permutation swaps the triangle),
//   so the permutation costs only static per-lane store addresses.  The smem layout
//   (i, j) -> i*17 + (j ^ (i/2)) and the lane -> block orders minimise bank conflicts (offline
//   search with the quarter-warp model of 16-byte accesses).
//   Per round: rotation of every slot pair from (a_xx, a_yy, a_xy) and the closed-form 2x2
//   diagonal block (a_xx - t|a_xy|, a_yy + t|a_xy|, 0); every off-diagonal 2x2 block (slot pairs
//   r < s): B <- J_r^H B J_s; V <- V J in registers (the slot permutation is register renaming
//   plus one complex shuffle per row).
// Rotation: J = diag(1, e) [[c, s], [-s, c]], e = conj(a_xy)/|a_xy|, with the short-chain
// parameters of Golub & Van Loan sym.schur2 after the phase step (see phase 1 below).
// Stop rule at the start of every sweep: off(A) = sqrt(sum_{i != j} |a_ij|^2) <= 10 eps ||R||_F,
// computed directly, at most 30 sweeps (Q15).  Eigenvalues ascending, ties by index (Q2).
#include <cfloat>

#include "doa_internal.cuh"

namespace doa {
namespace {

constexpr int kLd = 17;           // smem row stride (double2)
#ifndef DOA_EIG_HALF_MIN_B
#define DOA_EIG_HALF_MIN_B 2048  // below this batch size eig16s_kernel (latency) runs
#endif

// eig16s: warp-0 lane -> off-diagonal slot-pair block (index into the row-major list of r < s
// pairs), from the quarter-warp bank-conflict search of round 1 (layout i*17 + (j ^ (i/2)))
__device__ constexpr int kBlockOrder[28] = {14, 11, 10, 16, 13, 8, 25, 15, 4, 6, 19, 12, 21, 26,
                                             1, 17, 18, 7, 23, 24, 22, 20, 9, 27, 3, 2, 0, 5};


// Branch-free reciprocal (square root) for positive normal arguments: MUFU seed (rsqrt/rcp
// .approx.ftz.f64) + one third-order correction, within 1 ulp (tools/rsqrt_check.cu,
// tests/test_gpu_rsqrt.py).  The library versions add special-case branches that cost a third of
// the rotation-parameter instructions.  The rotation code feeds them unguarded values (a zero
// pivot gives inf/NaN intermediates) and selects the identity rotation at the end, keeping selects
// off the latency chain.  With e = 1 - x y0^2 (the seed's relative error is below 2^-20, measured
// 9.2e-7, so (5/16) e^3 < 2^-61) y = y0 (1 + e/2 + 3e^2/8): four dependent FP64 operations instead
// of the six of two Newton steps on the rotation-parameter chain; rcp likewise y0 (1 + e + e^2).
__device__ __forceinline__ double rsqrt_pos(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double e = fma(-(x * y), y, 1.0);
  return fma(y * e, fma(e, 0.375, 0.5), y);
}
__device__ __forceinline__ double rcp_pos(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double e = fma(-x, y, 1.0);
  return fma(y, fma(e, e, e), y);
}

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {   // conj(a) * b
  return make_double2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}

// ---------------------------------------------------------------------------------------------
// S3 in the eigensolver's epilogue (the "frame kernel"): Table 3's Step-3/4
// for up to kMaxCoefPlans estimators straight from the converged eigenpairs, reduced to
// the Toeplitz sums c_k = sum_p C[p][p+k] of DESIGN.md §5, so V never leaves the SM.  With
// g_{k,j} = sum_{p < M-k} V[p][j] conj(V[p+k][j]) (column j = eigenvector of the j-th smallest
// eigenvalue, Q2):
//   PHD   c_k = g_{k,0}                                   (C = e_min e_min^H, Q4)
//   MUSIC c_k = sum_{j<K} g_{k,j}                          (C = E_n E_n^H, K = M - D)
//   EV    c_k = sum_{j<K} w_j g_{k,j}, w_j = 1/lambda_j    (Q1; clamped at 100 eps lambda_max, G1)
//   MN    c_k = sum_{p < M-k} w_p conj(w_{p+k}),  w = P_n e1 / (e1^H P_n e1),
//         (P_n e1)_p = sum_{j<K} V[p][j] conj(V[0][j])     (Q5; e1^H P_n e1 <= 100 eps: unnormalised, G1)
// Executed by a 16-lane group (hl = lane within it); every sum runs in a fixed ascending order, so
// eig16h and eig16s (same eigenpairs, same routine) give bitwise identical coefficients.
// Shared memory (the eigensolver's own buffers, so the fused kernel needs no extra smem and keeps
// its occupancy):
//   Vs  [N][N+1]: columns j < N eigenvectors in rank order, Vs[p (N+1) + j] = V[p][j] (written by
//       the caller); column N: scratch for MN's w
//   Gs  [N][N+1] scratch g_{k,j} in columns j < N; may alias Vs (every read of Vs's columns j < N
//       precedes the first write of Gs)
//   LE  [N]: .x = ascending eigenvalues lambda_r (written by the caller), .y = EV weights
// Outputs per plan a: coefficients in the scan's A-fragment layout (coef_index), cnt[b] = 0 and
// info[b] = eigflag | DEGENERATE (overwritten).  `live`: this group holds a real frame b < B.
template <int N>
__device__ __forceinline__ void frame_coef(int hl, unsigned gmask, double2* Vs, double2* Gs, double2* LE, int M,
                                           int D, const CoefPlans& cp, int64_t b, bool live, int eigflag) {
  constexpr int LDV = N + 1;
  auto lam = [&](int r) { return LE[r].x; };
  const int K = M - D;
  bool need_ev = false, need_mn = false;
#pragma unroll
  for (int a = 0; a < kMaxCoefPlans; ++a)
    if (a < cp.nplans) { need_ev |= cp.alg[a] == DOA_ALG_EV; need_mn |= cp.alg[a] == DOA_ALG_MN; }
  // (a) lane j: column j into registers (zero beyond M)
  const int j = hl;
  double2 col[N];
#pragma unroll
  for (int p = 0; p < N; ++p) col[p] = (j < M && p < M) ? Vs[p * LDV + j] : make_double2(0.0, 0.0);
  int flag_ev = 0, flag_mn = 0;
  if (need_ev) {                                        // EV weights, lane-parallel (G1 clamp)
    const double lfloor = 100.0 * DBL_EPSILON * fmax(lam(M - 1), 0.0);
    const double lj = hl < K ? lam(hl) : 1.0;
    const bool deg = hl < K && lj <= lfloor;
    if (__ballot_sync(0xffffffffu, deg) & gmask) flag_ev = DOA_INFO_DEGENERATE;
    if (hl < N) LE[hl].y = hl < K ? (deg ? (lfloor > 0.0 ? 1.0 / lfloor : 1.0) : 1.0 / lj) : 0.0;
  }
  if (need_mn) {                                        // w_p on lane p, p0 on every lane (same order)
    const int p = hl;
    double wr = 0.0, wi = 0.0, p0 = 0.0;
#pragma unroll
    for (int j = 0; j < N; ++j) {
      if (j < K) {
        const double2 v0 = Vs[j], vp = p < M ? Vs[p * LDV + j] : make_double2(0.0, 0.0);
        wr = fma(vp.x, v0.x, wr);                       // V[p][j] conj(V[0][j])
        wr = fma(vp.y, v0.y, wr);
        wi = fma(vp.y, v0.x, wi);
        wi = fma(-vp.x, v0.y, wi);
        p0 = fma(v0.x, v0.x, p0);
        p0 = fma(v0.y, v0.y, p0);
      }
    }
    const bool degen = !(p0 > 100.0 * DBL_EPSILON);
    if (degen) flag_mn = DOA_INFO_DEGENERATE;
    const double lp = degen ? 1.0 : 1.0 / p0;
    if (p < N) Vs[p * LDV + N] = degen ? make_double2(wr, wi) : make_double2(wr * lp, wi * lp);   // zero for p >= M
  }
  __syncwarp();                                         // every read of Vs's columns j < N is done
  // g_{k,j} for every lag k from the column in registers (Gs may overwrite Vs from here on)
#pragma unroll
  for (int k = 0; k < N; ++k) {
    double gr = 0.0, gi = 0.0;
#pragma unroll
    for (int p = 0; p + k < N; ++p) {                   // V[p][j] conj(V[p+k][j]), ascending p
      gr = fma(col[p].x, col[p + k].x, gr);
      gr = fma(col[p].y, col[p + k].y, gr);
      gi = fma(col[p].y, col[p + k].x, gi);
      gi = fma(-col[p].x, col[p + k].y, gi);
    }
    if (j < N) Gs[k * LDV + j] = make_double2(gr, gi);
  }
  __syncwarp();
  // (b) lane k: combine over j (ascending) and write every plan's coefficients
  const int k = hl;
  double2 phd = make_double2(0.0, 0.0), mus = phd, ev = phd, mn = phd;
  if (k < M) {
    phd = Gs[k * LDV];
#pragma unroll
    for (int j = 0; j < N; ++j) {
      if (j < K) {
        const double2 g = Gs[k * LDV + j];
        mus.x += g.x;
        mus.y += g.y;
        if (need_ev) {
          const double w = LE[j].y;
          ev.x = fma(w, g.x, ev.x);
          ev.y = fma(w, g.y, ev.y);
        }
      }
    }
    if (need_mn) {
#pragma unroll
      for (int p = 0; p < N; ++p) {
        if (p + k < M) {                                // w_p conj(w_{p+k}), ascending p
          const double2 x = Vs[p * LDV + N], y = Vs[(p + k) * LDV + N];
          mn.x = fma(x.x, y.x, mn.x);
          mn.x = fma(x.y, y.y, mn.x);
          mn.y = fma(x.y, y.x, mn.y);
          mn.y = fma(-x.x, y.y, mn.y);
        }
      }
    }
  }
  const int S = ksteps(M), JE = 4 * ksteps_even(M);
#pragma unroll
  for (int a = 0; a < kMaxCoefPlans; ++a) {
    if (a >= cp.nplans || !live) continue;
    const int alg = cp.alg[a];
    double* coef = cp.coef[a];
    const double2 c = alg == DOA_ALG_PHD ? phd : (alg == DOA_ALG_MUSIC ? mus : (alg == DOA_ALG_EV ? ev : mn));
    if (k < M) {
      if (k == 0) coef[coef_index(b, 0, S)] = c.x;
      else {
        coef[coef_index(b, coef_cos(k), S)] = 2.0 * c.x;
        coef[coef_index(b, coef_sin(M, k), S)] = 2.0 * c.y;
      }
    }
    for (int jj = hl; jj < 4 * S; jj += 16)                                          // K padding
      if ((jj >= M && jj < JE) || jj >= JE + M - 1) coef[coef_index(b, jj, S)] = 0.0;
    if (hl == 0) {
      cp.cnt[a][b] = 0;
      cp.info[a][b] = eigflag | (alg == DOA_ALG_EV ? flag_ev : 0) | (alg == DOA_ALG_MN ? flag_mn : 0);
    }
  }
}

// eig16h (batches): two matrices per warp, one per 16-lane half.  Phase 1 of both matrices runs
// in the same instructions (lanes 0-7 and 16-23); each lane of a half owns one full row of V (16
// complex) and two of the 28 off-diagonal blocks.  A converged matrix keeps running with identity
// rotations (c = 1, s = 0, e = 1: exact copies), so its outputs equal eig16s's whatever its
// partner needs.
constexpr int kHWarps = 2;
#ifndef DOA_EIGH_MINB
#define DOA_EIGH_MINB 6
#endif
__device__ __forceinline__ double flipb(double x, int bit) {      // conjugate when bit set
  return __longlong_as_double(__double_as_longlong(x) ^ ((long long)bit << 63));
}
__device__ __forceinline__ double hsum(double v) {               // sum over a 16-lane half
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
// N = 16 or 8 (M <= 8 uses the 8-index round robin: 7 rounds of 4 rotations per sweep).
template <int N> struct HLd { static constexpr int LD = N == 16 ? kLd : 9; };
template <int N>
__device__ __forceinline__ int aidxT(int i, int j) { return i * HLd<N>::LD + (j ^ (i >> 1)); }
__host__ __device__ constexpr int cat_next_c(int s, int n) {
  return s == 0 ? 0 : (s == 1 ? 2 : (s == n - 2 ? n - 1 : ((s & 1) ? s - 2 : s + 2)));
}
template <int N>
__device__ __forceinline__ int cat_nextT(int s) { return cat_next_c(s, N); }

// eig16h_kernel<16> shared-memory layout and lane -> block assignment (tools/eig_layout_color.py):
// off-diagonal element (i < j) of the slot-ordered matrix at slot kOff16[i][j] (16-byte units), the
// real diagonal as 16 doubles from slot kDiag16.  Every element is read by exactly one
// (instruction, quarter-warp) group per round and written by exactly one; the slots' bank groups
// (slot mod 8) are an 8-edge-colouring of the bipartite (load group x store group) multigraph, so
// every block load, permuted store and phase-1 access is bank-conflict-free.  Lane hl rotates block
// kLaneBlk16[0][hl] in pass 1 and, for hl < 12, kLaneBlk16[1][hl] in pass 2, which shares its row
// pair with the pass-1 block (so pass 2 loads one pair's rotation parameters).  Block index =
// row-major position among the 28 slot-pair blocks r < s.
__device__ constexpr unsigned char kOff16[16][16] = {
    {255, 0, 3, 8, 11, 1, 9, 4, 17, 2, 10, 18, 26, 19, 27, 35},
    {255, 255, 16, 12, 25, 24, 33, 34, 43, 41, 42, 51, 50, 58, 59, 49},
    {255, 255, 255, 67, 32, 57, 40, 20, 28, 7, 36, 5, 15, 75, 13, 48},
    {255, 255, 255, 255, 83, 6, 56, 14, 22, 21, 30, 23, 29, 64, 31, 44},
    {255, 255, 255, 255, 255, 65, 38, 46, 54, 62, 37, 45, 39, 47, 72, 80},
    {255, 255, 255, 255, 255, 255, 52, 73, 60, 91, 55, 63, 53, 61, 81, 88},
    {255, 255, 255, 255, 255, 255, 255, 69, 68, 71, 76, 99, 79, 89, 77, 96},
    {255, 255, 255, 255, 255, 255, 255, 255, 66, 74, 82, 104, 70, 78, 97, 90},
    {255, 255, 255, 255, 255, 255, 255, 255, 255, 84, 98, 85, 112, 105, 86, 106},
    {255, 255, 255, 255, 255, 255, 255, 255, 255, 255, 120, 93, 101, 113, 109, 107},
    {255, 255, 255, 255, 255, 255, 255, 255, 255, 255, 255, 114, 117, 94, 121, 92},
    {255, 255, 255, 255, 255, 255, 255, 255, 255, 255, 255, 255, 87, 100, 102, 115},
    {255, 255, 255, 255, 255, 255, 255, 255, 255, 255, 255, 255, 255, 110, 129, 108},
    {255, 255, 255, 255, 255, 255, 255, 255, 255, 255, 255, 255, 255, 255, 116, 95},
    {255, 255, 255, 255, 255, 255, 255, 255, 255, 255, 255, 255, 255, 255, 255, 103},
    {255, 255, 255, 255, 255, 255, 255, 255, 255, 255, 255, 255, 255, 255, 255, 255},
};
__device__ constexpr signed char kLaneBlk16[2][16] = {
    {0, 2, 4, 7, 9, 11, 13, 15, 18, 20, 22, 25, 6, 17, 24, 27},
    {1, 3, 5, 8, 10, 12, 14, 16, 19, 21, 23, 26, -1, -1, -1, -1}};
constexpr int kDiag16 = 136;

// Element addressing of one matrix buffer: N = 16 the coloured layout above, N = 8 the XOR layout.
template <int N>
__device__ __forceinline__ int offslot(int i, int j) {            // i < j
  if constexpr (N == 16) return kOff16[i][j];
  else return aidxT<N>(i, j);
}
template <int N>
__device__ __forceinline__ double* diagp(double2* A, int i) {
  if constexpr (N == 16) return reinterpret_cast<double*>(A + kDiag16) + i;
  else return &A[aidxT<N>(i, i)].x;
}
template <int N>
__device__ __forceinline__ int blk_of(int hl, int u) {             // lane's block in pass u, -1: none
  constexpr int NP = N / 2, NBLK = NP * (NP - 1) / 2;
  if constexpr (N == 16) return kLaneBlk16[u][hl];
  else return (u == 0 && hl < NBLK) ? hl : -1;
}

// FUSE: the frame kernel — S3 for the plans in `cp` runs in the epilogue (frame_coef); lam_out /
// V_out / info may then be NULL (not written).
template <int N, bool FUSE>
__global__ void __launch_bounds__(kHWarps * 32, DOA_EIGH_MINB) eig16h_kernel(const double2* __restrict__ R,
                                                                             int64_t B, int M,
                                                                             double* __restrict__ lam_out,
                                                                             double2* __restrict__ V_out,
                                                                             int32_t* __restrict__ info,
                                                                             int D, CoefPlans cp) {
  // A double buffer per half: the packed layout (off-diagonal slots < 130, diagonal doubles from
  // slot kDiag16) for N = 16, the XOR layout for N = 8.  The frame epilogue uses the two buffers of
  // a half as one [N][N+1] scratch (V rank-ordered, then the lag sums over it).
  constexpr int BUF = N == 16 ? kDiag16 + 8 : N * HLd<N>::LD;
  __shared__ double2 As[kHWarps][2][2][BUF];                       // [warp][half][buffer]
  // rotation parameters (c, s) at [0, N/2) and (Re e, Im e) at [N/2, N) per slot pair, 16-byte
  // entries: the pairs of a half sit in distinct bank groups, so every lane -> pair pattern is
  // conflict-free; after the sweeps, the frame epilogue's eigenvalues / EV weights
  __shared__ double2 prm[kHWarps][2][N];
  __shared__ int rank_s[kHWarps][2][N];
  static_assert(2 * BUF >= N * (N + 1), "frame epilogue scratch");
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int hm = lane >> 4, hl = lane & 15;
  const int64_t b = ((int64_t)blockIdx.x * kHWarps + warp) * 2 + hm;
  const bool valid = b < B;
  double2* const Pc = prm[warp][hm];
  double2* const Pe = prm[warp][hm] + N / 2;

  // ||R||_F and off(A) are summed in the same order as eig16s's (lane partials over the element
  // strides of 32, i.e. this half-lane's even and odd strides of 16, added, then the tree), so both
  // kernels take identical stop decisions and a frame's results do not depend on B.
  double nrm_e = 0.0, nrm_o = 0.0;
  {
    const double2* Rb = R + (size_t)(valid ? b : 0) * M * M;
    double2* A0 = As[warp][hm][0];
    for (int e = hl; e < N * N; e += 16) {
      const int i = e / N, j = e % N;
      if (i > j) continue;
      double2 v = make_double2(0.0, 0.0);
      if (valid && j < M) v = Rb[(size_t)i * M + j];
      if (i == j) {
        v.y = 0.0;
        *diagp<N>(A0, i) = v.x;
      } else {
        A0[offslot<N>(i, j)] = v;
      }
      const double t = (i == j ? 1.0 : 2.0) * (v.x * v.x + v.y * v.y);
      if ((e / 16) & 1) nrm_o += t; else nrm_e += t;
    }
  }
  const double tol = 10.0 * DBL_EPSILON * sqrt(hsum(nrm_e + nrm_o));

  double2 v[N];                                           // row hl of this half's V
#pragma unroll
  for (int k = 0; k < N; ++k) v[k] = make_double2(k == hl ? 1.0 : 0.0, 0.0);

  // the lane's off-diagonal blocks: pass 0 and (N = 16, hl < 12) pass 1, which shares the row pair
  constexpr int NP = N / 2;
  const int blk[2] = {blk_of<N>(hl, 0), blk_of<N>(hl, 1)};
  const bool has1 = blk[0] >= 0, has2 = blk[1] >= 0;
  int rb[2], sb[2], rd[2][4], wr[2][4], sgm[2];
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    int l = blk[u] < 0 ? 0 : blk[u];
    int r0 = 0, s0 = 1;
    for (int r = 0; r < NP; ++r) {
      const int cntr = NP - 1 - r;
      if (l < cntr) { r0 = r; s0 = r + 1 + l; break; }
      l -= cntr;
    }
    rb[u] = r0; sb[u] = s0;
    const int i0 = 2 * r0, i1 = i0 + 1, j0 = 2 * s0, j1 = j0 + 1;
    rd[u][0] = offslot<N>(i0, j0); rd[u][1] = offslot<N>(i0, j1);
    rd[u][2] = offslot<N>(i1, j0); rd[u][3] = offslot<N>(i1, j1);
    const int pr[2] = {cat_nextT<N>(i0), cat_nextT<N>(i1)}, pc[2] = {cat_nextT<N>(j0), cat_nextT<N>(j1)};
    int m = 0;
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int x = pr[a], y = pc[c];
        wr[u][2 * a + c] = x < y ? offslot<N>(x, y) : offslot<N>(y, x);
        m |= (x < y ? 0 : 1) << (2 * a + c);
      }
    sgm[u] = m;
  }
  const int kx = 2 * (hl % NP), ky = kx + 1, px = cat_nextT<N>(kx), py = cat_nextT<N>(ky);
  const int rxy = offslot<N>(kx, ky);
  const int wxy = px < py ? offslot<N>(px, py) : offslot<N>(py, px);
  __syncwarp();

  // One off-diagonal block: B <- J_r^H B J_s (same operations, same order as eig16s)
  auto rotate_block = [&](const double2* A, double2* An, int u, double2 rcs, double2 ree, double2 scs, double2 see) {
    const double2 b00 = A[rd[u][0]], b01 = A[rd[u][1]], b10 = A[rd[u][2]], b11 = A[rd[u][3]];
    const double pc = rcs.x, ps = rcs.y, qc = scs.x, qs = scs.y;
    const double2 t0 = cmul(see, b01), t1 = cmul(see, b11);
    const double2 n00 = make_double2(qc * b00.x - qs * t0.x, qc * b00.y - qs * t0.y);
    const double2 n01 = make_double2(qs * b00.x + qc * t0.x, qs * b00.y + qc * t0.y);
    const double2 n10 = make_double2(qc * b10.x - qs * t1.x, qc * b10.y - qs * t1.y);
    const double2 n11 = make_double2(qs * b10.x + qc * t1.x, qs * b10.y + qc * t1.y);
    const double2 u0 = cmulc(ree, n10), u1 = cmulc(ree, n11);
    const int m = sgm[u];
    An[wr[u][0]] = make_double2(pc * n00.x - ps * u0.x, flipb(pc * n00.y - ps * u0.y, m & 1));
    An[wr[u][1]] = make_double2(pc * n01.x - ps * u1.x, flipb(pc * n01.y - ps * u1.y, (m >> 1) & 1));
    An[wr[u][2]] = make_double2(ps * n00.x + pc * u0.x, flipb(ps * n00.y + pc * u0.y, (m >> 2) & 1));
    An[wr[u][3]] = make_double2(ps * n01.x + pc * u1.x, flipb(ps * n01.y + pc * u1.y, (m >> 3) & 1));
  };

  int flag = 0;
  int cur = 0;
  bool act = valid;
  for (int sweep = 0;; ++sweep) {
    {
      const double2* A = As[warp][hm][cur];
      double off_e = 0.0, off_o = 0.0;
#pragma unroll
      for (int it = 0; it < N * N / 16; ++it) {
        const int e = hl + 16 * it, i = e / N, j = e % N;
        if (i < j) {
          const double2 a = A[offslot<N>(i, j)];
          if (it & 1) off_o += a.x * a.x + a.y * a.y; else off_e += a.x * a.x + a.y * a.y;
        }
      }
      const double off = sqrt(2.0 * hsum(off_e + off_o));
      if (act && off <= tol) act = false;
      else if (act && sweep == kMaxSweeps) { flag |= DOA_INFO_NOCONV; act = false; }
    }
    if (!__any_sync(0xffffffffu, act)) break;
#pragma unroll 1
    for (int rnd = 0; rnd < N - 1; ++rnd) {
      double2* A = As[warp][hm][cur];
      double2* An = As[warp][hm][cur ^ 1];
      if (hl < NP) {                                     // phase 1: rotation of slot pair hl
        const double2 axy = A[rxy];
        const double axx = *diagp<N>(A, kx), ayy = *diagp<N>(A, ky);
        const double r2 = axy.x * axy.x + axy.y * axy.y;
        const bool rot = act && r2 > 1e-300;             // frozen matrices: identity rotations
        const double ir = rsqrt_pos(r2);
        const double rr = r2 * ir;
        const double d = 0.5 * (ayy - axx);
        const double h2 = fma(d, d, r2);
        const double irh = rsqrt_pos(h2);
        const double hh = h2 * irh;
        const double q = fabs(d) + hh;
        const double uu = 0.5 * q * irh;                 // c^2
        const double iu = rsqrt_pos(uu);                 // 2 hh q = 4 h2 uu: s = r / sqrt(2 hh q) = r irh iu / 2
        const double sabs = (0.5 * rr * irh) * iu;
        const double trabs = r2 * rcp_pos(q);
        const double tr = rot ? (d < 0.0 ? -trabs : trabs) : 0.0;
        Pc[hl] = make_double2(rot ? uu * iu : 1.0, rot ? (d < 0.0 ? -sabs : sabs) : 0.0);
        Pe[hl] = make_double2(rot ? axy.x * ir : 1.0, rot ? -axy.y * ir : 0.0);
        *diagp<N>(An, px) = axx - tr;
        *diagp<N>(An, py) = ayy + tr;
        An[wxy] = act ? make_double2(0.0, 0.0) : axy;    // frozen: keep the element as it is
      }
      __syncwarp();
      double2 rcs = make_double2(1.0, 0.0), ree = rcs;
      if (has1) {
        rcs = Pc[rb[0]]; ree = Pe[rb[0]];
        rotate_block(A, An, 0, rcs, ree, Pc[sb[0]], Pe[sb[0]]);
      }
      if (has2) rotate_block(A, An, 1, rcs, ree, Pc[sb[1]], Pe[sb[1]]);   // same row pair as pass 0
      // V <- V J on the lane's row, then the slot permutation (register renaming + moves)
      double2 t[N];
#pragma unroll
      for (int k = 0; k < NP; ++k) {
        const double2 cs = Pc[k], ee = Pe[k];
        const double2 vx = v[2 * k], vy = v[2 * k + 1];
        const double2 ey = cmul(ee, vy);
        t[cat_next_c(2 * k, N)] = make_double2(cs.x * vx.x - cs.y * ey.x, cs.x * vx.y - cs.y * ey.y);
        t[cat_next_c(2 * k + 1, N)] = make_double2(cs.y * vx.x + cs.x * ey.x, cs.y * vx.y + cs.x * ey.y);
      }
#pragma unroll
      for (int k = 0; k < N; ++k) v[k] = t[k];
      cur ^= 1;
      __syncwarp();
    }
  }

  double2* A = As[warp][hm][cur];
  if (hl < M) {
    const double li = *diagp<N>(A, hl);
    int rk = 0;
    for (int j = 0; j < M; ++j) {
      const double lj = *diagp<N>(A, j);
      rk += (lj < li) || (lj == li && j < hl);
    }
    rank_s[warp][hm][hl] = rk;
    if (valid && lam_out) lam_out[(size_t)b * M + rk] = li;
    if (FUSE) prm[warp][hm][rk].x = li;               // the rotation parameters are no longer needed
  }
  __syncwarp();
  if (valid && hl < M && V_out) {
    double2* Vrow = V_out + (size_t)b * M * M + (size_t)hl * M;
#pragma unroll
    for (int k = 0; k < N; ++k)
      if (k < M) Vrow[rank_s[warp][hm][k]] = v[k];
  }
  if (valid && hl == 0 && info) info[b] = flag;
  if (FUSE) {
    // rank-ordered V over both buffers (every lane has read A's diagonal before the __syncwarp
    // above), then S3 with the lag sums overwriting it in place
    double2* Vs = &As[warp][hm][0][0];
    if (hl < M) {
#pragma unroll
      for (int k = 0; k < N; ++k)
        if (k < M) Vs[hl * (N + 1) + rank_s[warp][hm][k]] = v[k];
    }
    __syncwarp();
    frame_coef<N>(hl, hm ? 0xffff0000u : 0x0000ffffu, Vs, Vs, prm[warp][hm], M, D, cp, b, valid, flag);
  }
}


// Small-batch variant (latency): one matrix per CTA of three warps, software-pipelined like a
// systolic array.  Warp 0 owns the 28 off-diagonal blocks (one per lane); warp 2 is the "pilot":
// lane k recomputes (same operations) the rotated element of the block that becomes next-round pair
// k's off-diagonal element and derives the NEXT round's rotation from it and the post-rotation
// diagonal; warp 1 applies the current round's rotations to V (lane l: row l/2, slot half l%2, 8
// complex in registers) at the same time.  One CTA barrier per round, so a round's critical path is
// one block update plus one rotation-parameter chain, and each warp's instruction stream is short
// (with the pilot inside warp 0 its stream was the serial sum of both; 74 us per matrix at M = 16).  Same rotation formulas, operation order, stop-rule sums (lanes 0-15
// of warp 0 reproduce eig16h's partial sums and tree) and slot permutation as eig16h_kernel, so
// both kernels give bitwise identical eigenpairs (tests/test_gpu_parity.py::
// test_eig_kernels_bitwise_equal) and a frame's result does not depend on B.
struct RotP {
  double c, s, er, ei, tr;
};
__device__ __forceinline__ RotP rot_params_s(double axx, double ayy, double2 axy) {
  const double r2 = axy.x * axy.x + axy.y * axy.y;
  const bool rot = r2 > 1e-300;                              // a_xy ~ 0: identity rotation
  const double ir = rsqrt_pos(r2);
  const double rr = r2 * ir;
  const double d = 0.5 * (ayy - axx);
  const double h2 = fma(d, d, r2);
  const double irh = rsqrt_pos(h2);
  const double hh = h2 * irh;
  const double q = fabs(d) + hh;
  const double uu = 0.5 * q * irh;                       // c^2 (same operations as eig16h)
  const double iu = rsqrt_pos(uu);
  const double sabs = (0.5 * rr * irh) * iu;
  const double trabs = r2 * rcp_pos(q);
  RotP p;
  p.tr = rot ? (d < 0.0 ? -trabs : trabs) : 0.0;
  p.c = rot ? uu * iu : 1.0;
  p.s = rot ? (d < 0.0 ? -sabs : sabs) : 0.0;
  p.er = rot ? axy.x * ir : 1.0;
  p.ei = rot ? -axy.y * ir : 0.0;
  return p;
}
__host__ __device__ constexpr int cat_prev_c(int t, int n) {
  return t == 0 ? 0 : (t == 2 ? 1 : (t == n - 1 ? n - 2 : ((t & 1) ? t + 2 : t - 2)));
}
// V registers of a slot half g: old local slot feeding new local slot l (-1: from the other half)
__host__ __device__ constexpr int vsrc_c(int n, int g, int l) {
  return cat_prev_c((n / 2) * g + l, n) / (n / 2) == g ? cat_prev_c((n / 2) * g + l, n) - (n / 2) * g : -1;
}
__device__ __forceinline__ double2 sel2(bool p, double2 a, double2 b) {
  return make_double2(p ? a.x : b.x, p ? a.y : b.y);
}

constexpr int kSThreads = 96;      // eig16s: warp 0 blocks, warp 1 V, warp 2 pilot
#ifdef DOA_EIG_TRACE
__device__ long long g_eig_trace[8 * 512];      // tools/eig16s_trace.cu: clock64 per round and warp
#define EIG_TRACE(slot) do { if (blockIdx.x == 0 && lane == 0 && rg < 512) g_eig_trace[8 * rg + (slot)] = clock64(); } while (0)
#else
#define EIG_TRACE(slot) do { } while (0)
#endif
template <int N, bool FUSE>
__global__ void __launch_bounds__(kSThreads) eig16s_kernel(const double2* __restrict__ R, int64_t B, int M,
                                                    double* __restrict__ lam_out, double2* __restrict__ V_out,
                                                    int32_t* __restrict__ info, int D, CoefPlans cp) {
  constexpr int NP = N / 2, NBLK = NP * (NP - 1) / 2, SPL = N / 2, RPW = 32 / (N / 4) / 2;
  // V: lane l of warp 1 holds row l / (N/8 * ...) -- N = 16: row l/2, slot half l%2; N = 8: row
  // l/2 for l < 16 (lanes 16-31 idle), slot half l%2
  __shared__ double2 As[2][N * HLd<N>::LD];
  __shared__ double2 Pcs[2][NP], Pee[2][NP];
  __shared__ double Dp[2][N];
  __shared__ int rank_s[N];
  __shared__ int go_s;
  (void)RPW;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t b = blockIdx.x;
  const double2* Rb = R + (size_t)b * M * M;

  // ---- load; ||R||_F in eig16h's order (lanes 0-15 of warp 0)
  double nrm_e = 0.0, nrm_o = 0.0;
  for (int e = tid; e < N * N; e += kSThreads) {
    const int i = e / N, j = e % N;
    if (i > j) continue;
    double2 v = make_double2(0.0, 0.0);
    if (j < M) v = Rb[(size_t)i * M + j];
    if (i == j) {
      v.y = 0.0;
      Dp[1][cat_prev_c(i, N)] = v.x;                  // dpost_{-1}[pinv(i)] = d[i]
    } else {
      As[0][aidxT<N>(i, j)] = v;
    }
  }
  __syncthreads();
  if (warp == 0 && lane < 16) {                        // from the staged copy: loads in flight together
#pragma unroll
    for (int it = 0; it < N * N / 16; ++it) {
      const int e = lane + 16 * it, i = e / N, j = e % N;
      if (i > j) continue;
      const double2 v = i == j ? make_double2(Dp[1][cat_prev_c(i, N)], 0.0) : As[0][aidxT<N>(i, j)];
      const double t = (i == j ? 1.0 : 2.0) * (v.x * v.x + v.y * v.y);
      if (it & 1) nrm_o += t; else nrm_e += t;
    }
  }
  double tol = 0.0;
  if (warp == 0) tol = 10.0 * DBL_EPSILON * sqrt(hsum(nrm_e + nrm_o));

  // ---- per-lane geometry (warp 0: block lane < NBLK; warp 1: V; warp 2 lane k < NP: the pilot of
  // next-round pair k, i.e. the block one of whose rotated elements becomes that pair's a_xy)
  const bool hasb = warp == 0 && lane < NBLK;
  auto decode = [&](int t, int& r0, int& s0) {
    r0 = 0; s0 = 1;
    for (int r = 0; r < NP; ++r) {
      const int cntr = NP - 1 - r;
      if (t < cntr) { r0 = r; s0 = r + 1 + t; break; }
      t -= cntr;
    }
  };
  int rb = 0, sb = 1;
  if (warp == 2) {
    for (int t = 0; t < NBLK; ++t) {
      int r0, s0;
      decode(t, r0, s0);
      for (int e = 0; e < 4; ++e) {
        const int x = cat_next_c(2 * r0 + (e >> 1), N), y = cat_next_c(2 * s0 + (e & 1), N);
        if ((x >> 1) == (y >> 1) && (x >> 1) == lane) { rb = r0; sb = s0; }
      }
    }
  } else {
    decode(hasb ? (N == 16 ? kBlockOrder[lane] : lane) : 0, rb, sb);
  }
  int rdo[4], wro[4], cjm = 0;
  {
    const int ii[2] = {2 * rb, 2 * rb + 1}, jj[2] = {2 * sb, 2 * sb + 1};
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        rdo[2 * a + c] = aidxT<N>(ii[a], jj[c]);
        const int x = cat_next_c(ii[a], N), y = cat_next_c(jj[c], N);
        wro[2 * a + c] = x < y ? aidxT<N>(x, y) : aidxT<N>(y, x);
        cjm |= (x < y ? 0 : 1) << (2 * a + c);
      }
  }
  bool pil = false;
  int pe = 0, pk = 0, pxo = 0, pyo = 1, pcj = 0;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int i = 2 * rb + (e >> 1), j = 2 * sb + (e & 1);
    const int x = cat_next_c(i, N), y = cat_next_c(j, N);
    if (warp == 2 && lane < NP && (x >> 1) == (y >> 1)) {
      pil = true; pe = e; pk = x >> 1;
      pxo = (x & 1) ? j : i;
      pyo = (x & 1) ? i : j;
      pcj = (x & 1) ? 1 : 0;
    }
  }
  const int zk = lane & (NP - 1);
  const int zx = cat_next_c(2 * zk, N), zy = cat_next_c(2 * zk + 1, N);
  const int zpos = zx < zy ? aidxT<N>(zx, zy) : aidxT<N>(zy, zx);
  const int zsrc = aidxT<N>(2 * zk, 2 * zk + 1);
  const int g = lane & 1, vrow = lane >> 1;            // warp 1: V row, slot half
  double2 v[SPL];
#pragma unroll
  for (int l = 0; l < SPL; ++l) v[l] = make_double2(vrow == SPL * g + l ? 1.0 : 0.0, 0.0);

  // ---- first round's rotations
  if (warp == 0 && lane < NP) {
    const double axx = Dp[1][cat_prev_c(2 * zk, N)], ayy = Dp[1][cat_prev_c(2 * zk + 1, N)];
    const RotP p = rot_params_s(axx, ayy, As[0][zsrc]);
    Pcs[0][zk] = make_double2(p.c, p.s);
    Pee[0][zk] = make_double2(p.er, p.ei);
    Dp[0][2 * zk] = axx - p.tr;
    Dp[0][2 * zk + 1] = ayy + p.tr;
  }
  __syncthreads();

  int flag = 0;
  int pb = 0;
  for (int sweep = 0;; ++sweep) {
    if (warp == 0) {                                   // stop rule, eig16h's summation order
      const double2* A = As[pb];
      double off_e = 0.0, off_o = 0.0;
      if (lane < 16) {
#pragma unroll
        for (int it = 0; it < N * N / 16; ++it) {
          const int e = lane + 16 * it, i = e / N, j = e % N;
          if (i < j) {
            const double2 a = A[aidxT<N>(i, j)];
            if (it & 1) off_o += a.x * a.x + a.y * a.y; else off_e += a.x * a.x + a.y * a.y;
          }
        }
      }
      const double off = sqrt(2.0 * hsum(off_e + off_o));
      if (lane == 0) {
        int go = 1;
        if (off <= tol) go = 0;
        else if (sweep == kMaxSweeps) { flag |= DOA_INFO_NOCONV; go = 0; }
        go_s = go;
      }
    }
    __syncthreads();
    if (!go_s) break;
#pragma unroll 1
    for (int rnd = 0; rnd < N - 1; ++rnd) {
#ifdef DOA_EIG_TRACE
      const int rg = sweep * (N - 1) + rnd;
#endif
      if (warp == 2) EIG_TRACE(0);
      if (warp == 0 || warp == 2) {
        // warp 0 rotates the blocks; warp 2 (pilot) recomputes, with the same operations, the one
        // rotated element that becomes its next-round pair's a_xy and derives that rotation, so the
        // rotation-parameter chain runs beside the block updates instead of after them
        const double2* A = As[pb];
        double2* An = As[pb ^ 1];
        const double2 rcs = Pcs[pb][rb], ree = Pee[pb][rb], scs = Pcs[pb][sb], see = Pee[pb][sb];
        const double2 b00 = A[rdo[0]], b01 = A[rdo[1]], b10 = A[rdo[2]], b11 = A[rdo[3]];
        const double pc = rcs.x, ps = rcs.y, qc = scs.x, qs = scs.y;
        const double2 t0 = cmul(see, b01), t1 = cmul(see, b11);
        const double2 n00 = make_double2(qc * b00.x - qs * t0.x, qc * b00.y - qs * t0.y);
        const double2 n01 = make_double2(qs * b00.x + qc * t0.x, qs * b00.y + qc * t0.y);
        const double2 n10 = make_double2(qc * b10.x - qs * t1.x, qc * b10.y - qs * t1.y);
        const double2 n11 = make_double2(qs * b10.x + qc * t1.x, qs * b10.y + qc * t1.y);
        const double2 u0 = cmulc(ree, n10), u1 = cmulc(ree, n11);
        const double2 o0 = make_double2(pc * n00.x - ps * u0.x, pc * n00.y - ps * u0.y);
        const double2 o1 = make_double2(pc * n01.x - ps * u1.x, pc * n01.y - ps * u1.y);
        const double2 o2 = make_double2(ps * n00.x + pc * u0.x, ps * n00.y + pc * u0.y);
        const double2 o3 = make_double2(ps * n01.x + pc * u1.x, ps * n01.y + pc * u1.y);
        if (hasb) {
          An[wro[0]] = make_double2(o0.x, flipb(o0.y, cjm & 1));
          An[wro[1]] = make_double2(o1.x, flipb(o1.y, (cjm >> 1) & 1));
          An[wro[2]] = make_double2(o2.x, flipb(o2.y, (cjm >> 2) & 1));
          An[wro[3]] = make_double2(o3.x, flipb(o3.y, (cjm >> 3) & 1));
        }
        if (warp == 0 && lane < NP) An[zpos] = make_double2(0.0, 0.0);   // the zeroed pair elements
        if (warp == 0) EIG_TRACE(2);
        if (pil) {                                                  // next round's rotation
          const double2 pv = sel2(pe >= 2, sel2(pe & 1, o3, o2), sel2(pe & 1, o1, o0));
          const double axx = Dp[pb][pxo], ayy = Dp[pb][pyo];
          const RotP p = rot_params_s(axx, ayy, make_double2(pv.x, flipb(pv.y, pcj)));
          EIG_TRACE(1);
          Pcs[pb ^ 1][pk] = make_double2(p.c, p.s);
          Pee[pb ^ 1][pk] = make_double2(p.er, p.ei);
          Dp[pb ^ 1][2 * pk] = axx - p.tr;
          Dp[pb ^ 1][2 * pk + 1] = ayy + p.tr;
        }
      } else if (warp == 1 && (N == 16 || lane < 16)) {
        // V <- V J on row vrow, slot half g; then the slot permutation (one complex crosses)
        double2 nv[SPL];
#pragma unroll
        for (int kk = 0; kk < SPL / 2; ++kk) {
          const double2 cs = Pcs[pb][(SPL / 2) * g + kk], ee = Pee[pb][(SPL / 2) * g + kk];
          const double2 vx = v[2 * kk], vy = v[2 * kk + 1];
          const double2 ey = cmul(ee, vy);
          nv[2 * kk] = make_double2(cs.x * vx.x - cs.y * ey.x, cs.x * vx.y - cs.y * ey.y);
          nv[2 * kk + 1] = make_double2(cs.y * vx.x + cs.x * ey.x, cs.y * vx.y + cs.x * ey.y);
        }
        const double2 send = sel2(g == 0, nv[SPL - 2], nv[1]);
        const unsigned msk = N == 16 ? 0xffffffffu : 0x0000ffffu;
        const double2 recv = make_double2(__shfl_xor_sync(msk, send.x, 1), __shfl_xor_sync(msk, send.y, 1));
#pragma unroll
        for (int l = 0; l < SPL; ++l) {
          const int s0 = vsrc_c(N, 0, l), s1 = vsrc_c(N, 1, l);
          const double2 a0 = s0 < 0 ? recv : nv[s0 < 0 ? 0 : s0];
          const double2 a1 = s1 < 0 ? recv : nv[s1 < 0 ? 0 : s1];
          v[l] = s0 == s1 ? a0 : sel2(g == 0, a0, a1);
        }
        EIG_TRACE(3);
      }
      pb ^= 1;
      __syncthreads();
    }
  }

  if (warp == 0 && lane < M) {                         // lambda_s = dpost_{t-1}[pinv(s)]
    const double li = Dp[pb ^ 1][cat_prev_c(lane, N)];
    int rk = 0;
    for (int j = 0; j < M; ++j) {
      const double lj = Dp[pb ^ 1][cat_prev_c(j, N)];
      rk += (lj < li) || (lj == li && j < lane);
    }
    rank_s[lane] = rk;
    if (lam_out) lam_out[(size_t)b * M + rk] = li;
    if (FUSE) (&Pcs[0][0])[rk].x = li;                  // the rotation parameters are no longer needed
  }
  __syncthreads();
  if (warp == 1 && vrow < M) {
    if (V_out) {
      double2* Vrow = V_out + (size_t)b * M * M + (size_t)vrow * M;
#pragma unroll
      for (int l = 0; l < SPL; ++l)
        if (SPL * g + l < M) Vrow[rank_s[SPL * g + l]] = v[l];
    }
    if (FUSE) {                                         // rank-ordered V for frame_coef
#pragma unroll
      for (int l = 0; l < SPL; ++l)
        if (SPL * g + l < M) As[0][vrow * (N + 1) + rank_s[SPL * g + l]] = v[l];
    }
  }
  if (tid == 0 && info) info[b] = flag;
  if (FUSE) {
    // warp 0 runs S3 on both 16-lane halves (the same frame; only half 0 writes), exactly as one
    // half of eig16h does, so the coefficients are bitwise the same for any B
    if (warp == 0) flag = __shfl_sync(0xffffffffu, flag, 0);
    __syncthreads();
    if (warp == 0)
      frame_coef<N>(lane & 15, lane < 16 ? 0x0000ffffu : 0xffff0000u, As[0], As[1], &Pcs[0][0], M, D, cp, b,
                    lane < 16, flag);
  }
}

}  // namespace

namespace {
// Kernel choice for M <= 16: small batches (latency-bound) take the CTA-per-matrix pipelined
// kernel; it performs the same operations in the same order as eig16h, so the results are bitwise
// the same (tests/test_gpu_parity.py::test_eig_kernels_bitwise_equal).
template <bool FUSE>
cudaError_t launch16(const double* R, int64_t B, int M, double* lam, double* V, int32_t* info, int D,
                     const CoefPlans& cp, cudaStream_t s) {
  count_launch();
  const double2* R2 = reinterpret_cast<const double2*>(R);
  double2* V2 = reinterpret_cast<double2*>(V);
  if (B < DOA_EIG_HALF_MIN_B) {
    if (M <= 8) eig16s_kernel<8, FUSE><<<(unsigned)B, kSThreads, 0, s>>>(R2, B, M, lam, V2, info, D, cp);
    else eig16s_kernel<16, FUSE><<<(unsigned)B, kSThreads, 0, s>>>(R2, B, M, lam, V2, info, D, cp);
    return cudaGetLastError();
  }
  const unsigned g = (unsigned)((B + 2 * kHWarps - 1) / (2 * kHWarps));
  if (M <= 8) eig16h_kernel<8, FUSE><<<g, kHWarps * 32, 0, s>>>(R2, B, M, lam, V2, info, D, cp);
  else eig16h_kernel<16, FUSE><<<g, kHWarps * 32, 0, s>>>(R2, B, M, lam, V2, info, D, cp);
  return cudaGetLastError();
}
}  // namespace

cudaError_t launch_eig16(const double* R, int64_t B, int M, double* lam, double* V, int32_t* info, cudaStream_t s) {
  const CoefPlans none = {};
  return launch16<false>(R, B, M, lam, V, info, 0, none, s);
}

// The frame kernel: S2 + S3 in one launch (M <= 16, up to kMaxCoefPlans ULA plans sharing M, D).
// lam / V may be NULL (not written); every plan's info[b] is overwritten.
cudaError_t launch_eig16_coef(const double* R, int64_t B, int M, int D, double* lam, double* V, const CoefPlans& cp,
                              cudaStream_t s) {
  return launch16<true>(R, B, M, lam, V, nullptr, D, cp, s);
}

}  // namespace doa
