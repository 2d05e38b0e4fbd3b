// S2 for M <= 16: batched Hermitian Jacobi eigendecomposition — eig16_kernel (one warp per
// matrix, described below) and eig16h_kernel (the default: the same rounds with two matrices per
// warp, one per 16-lane half; see its comment further down).
// (Table 2 Step-2 `jsvd`; read as the Hermitian eigendecomposition, Q3.)
//
// Ordering: parallel cyclic Jacobi with the circle-method round robin on n = 16 indices (M < 16
// is padded with decoupled zero indices that no rotation ever touches).  The 8 disjoint pairs of a
// round always sit in fixed SLOTS (0,1), (2,3), ..., (14,15); after each round every index moves
// to the next slot of the "caterpillar" permutation pi (slot 0 fixed, slots 1..15 rotate along
// one 15-cycle), so every pair of indices meets exactly once per 15-round sweep and, because
// pi^15 = id, slots coincide with the original indices again at every sweep boundary.
//
//   A (Hermitian, physical slot order, upper triangle only) lives in shared memory,
//   double-buffered: each round reads buffer `cur` and writes every upper element of buffer `nxt`
//   at its PERMUTED position (pi(i), pi(j)) (conjugated when the permutation swaps the triangle),
//   so the permutation costs only static per-lane store addresses.  The smem layout
//   (i, j) -> i*17 + (j ^ (i/2)) and the lane -> block order below minimise bank conflicts of the
//   block reads / permuted writes and the phase-1 accesses (offline search with the quarter-warp
//   model of 16-byte accesses: 47 wavefronts per round for these 14 instructions vs 57 for the
//   previous i*19 layout, ideal 40).
//     phase 1  lanes 0..7   : rotation of slot pair k from (a_xx, a_yy, a_xy) and the closed-form
//                             2x2 diagonal block (a_xx - t|a_xy|, a_yy + t|a_xy|, 0)
//                             (Golub & Van Loan sym.schur2 after the phase rotation).
//     phase 2  lanes 0..27  : one off-diagonal 2x2 block (slot pairs r < s): B <- J_r^H B J_s.
//              all 32 lanes : V <- V J in registers.
//   V lives in registers: lane (row i = lane % 16, half h = lane / 16) holds V[i][slots 8h..8h+7];
//   its four slot pairs are local and pi moves only two slots across the halves per round (one
//   complex shuffle); the rest of pi is register renaming.
// Rotation: J = diag(1, e) [[c, s], [-s, c]], e = conj(a_xy)/|a_xy|, tau = (a_yy - a_xx)/(2|a_xy|),
// t = sign(tau)/(|tau| + sqrt(1 + tau^2)), c = 1/sqrt(1 + t^2), s = t c; identity when a_xy == 0.
// Stop rule at the start of every sweep: off(A) = sqrt(sum_{i != j} |a_ij|^2) <= 10 eps ||R||_F,
// at most 30 sweeps (Q15).  Eigenvalues ascending, ties by index (Q2).
#include <cfloat>

#include "doa_internal.cuh"

namespace doa {
namespace {

constexpr int kN = 16;            // padded order
constexpr int kLd = 17;           // smem row stride (double2)
constexpr int kEigWarps = 4;
#ifndef DOA_EIG_HALF_MIN_B
#define DOA_EIG_HALF_MIN_B 2048  // below this batch size M > 8 uses eig16_kernel
#endif
#ifndef DOA_EIG_MINB
#define DOA_EIG_MINB 5
#endif

__device__ __forceinline__ int aidx(int i, int j) { return i * kLd + (j ^ (i >> 1)); }

// lane -> off-diagonal slot-pair block (index into the row-major list of r < s pairs)
__device__ constexpr int kBlockOrder[28] = {14, 11, 10, 16, 13, 8, 25, 15, 4, 6, 19, 12, 21, 26,
                                             1, 17, 18, 7, 23, 24, 22, 20, 9, 27, 3, 2, 0, 5};

// Rotation parameters of one slot pair.  Padded to 48 bytes so the eight pairs'
// 16-byte halves fall in distinct shared-memory banks: phase 2b's loads (pairs k and k+4 in one
// instruction) and phase 2a's (pairs rb, sb over 28 lanes) are single wavefronts.
struct __align__(16) Prm {
  double c, s, er, ei;
  double pad0, pad1;
};

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// caterpillar: next slot of slot s
__device__ __forceinline__ int cat_next(int s) {
  if (s == 0) return 0;
  if (s == 1) return 2;
  if (s == 14) return 15;
  return (s & 1) ? s - 2 : s + 2;
}

// Branch-free reciprocal (square root) for positive normal arguments: MUFU seed (rsqrt/rcp
// .approx.ftz.f64) + two Newton steps, ~1 ulp.  The library versions add special-case branches
// that cost a third of the rotation-parameter instructions.
__device__ __forceinline__ double rsqrt_pos(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double hx = 0.5 * x;
  y = y * fma(-hx * y, y, 1.5);
  y = y * fma(-hx * y, y, 1.5);
  return y;
}
__device__ __forceinline__ double rcp_pos(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  y = y * fma(-x, y, 2.0);
  y = y * fma(-x, y, 2.0);
  return y;
}

// x with its sign bit XORed (conjugation of a stored imaginary part): integer pipe, not FP64
__device__ __forceinline__ double flip(double x, long long sgn) {
  return __longlong_as_double(__double_as_longlong(x) ^ sgn);
}

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {   // conj(a) * b
  return make_double2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}

__global__ void __launch_bounds__(kEigWarps * 32, DOA_EIG_MINB) eig16_kernel(const double2* __restrict__ R,
                                                                             int64_t B, int M,
                                                                             double* __restrict__ lam_out,
                                                                             double2* __restrict__ V_out,
                                                                             int32_t* __restrict__ info) {
  __shared__ double2 As[kEigWarps][2][kN * kLd];
  __shared__ Prm prm[kEigWarps][kN / 2];
  __shared__ int rank_s[kEigWarps][kN];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t b = (int64_t)blockIdx.x * kEigWarps + warp;
  if (b >= B) return;
  const double2* Rb = R + (size_t)b * M * M;

  // load the upper triangle (zero-padded to 16) and ||R||_F
  double nrm = 0.0;
  {
    double2* A0 = As[warp][0];
    for (int e = lane; e < kN * kN; e += 32) {
      const int i = e >> 4, j = e & 15;
      if (i > j) continue;
      double2 v = make_double2(0.0, 0.0);
      if (j < M) v = Rb[(size_t)i * M + j];
      if (i == j) v.y = 0.0;
      A0[aidx(i, j)] = v;
      nrm += (i == j ? 1.0 : 2.0) * (v.x * v.x + v.y * v.y);
    }
  }
  nrm = sqrt(wsum(nrm));
  const double tol = 10.0 * DBL_EPSILON * nrm;

  // V registers: row vi, slots 8h..8h+7 (V = I)
  const int vi = lane & 15, h = lane >> 4;
  double2 v[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) v[k] = make_double2(vi == 8 * h + k ? 1.0 : 0.0, 0.0);

  // static per-lane geometry.  Off-diagonal block (rb < sb) for lanes 0..27.
  int rb = 0, sb = 1;
  {
    int l = lane < 28 ? kBlockOrder[lane] : 0;
    for (int r = 0; r < 8; ++r) {
      const int cntr = 7 - r;
      if (l < cntr) { rb = r; sb = r + 1 + l; break; }
      l -= cntr;
    }
  }
  const int i0 = 2 * rb, i1 = 2 * rb + 1, j0 = 2 * sb, j1 = 2 * sb + 1;
  const int rd00 = aidx(i0, j0), rd01 = aidx(i0, j1), rd10 = aidx(i1, j0), rd11 = aidx(i1, j1);
  int wr[4];
  long long sg[4];                      // sign bit to XOR into Im: set when the permutation swapped the triangle
  {
    const int pr[2] = {cat_next(i0), cat_next(i1)}, pc[2] = {cat_next(j0), cat_next(j1)};
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int x = pr[a], y = pc[c];
        wr[2 * a + c] = x < y ? aidx(x, y) : aidx(y, x);
        sg[2 * a + c] = x < y ? 0LL : (long long)0x8000000000000000ULL;
      }
  }
  // phase-1 geometry (lanes 0..7): pair k = lane
  const int kx = 2 * (lane & 7), ky = kx + 1, px = cat_next(kx), py = cat_next(ky);
  const int rxy = aidx(kx, ky), rxx = aidx(kx, kx), ryy = aidx(ky, ky);
  const int wxx = aidx(px, px), wyy = aidx(py, py), wxy = px < py ? aidx(px, py) : aidx(py, px);
  __syncwarp();

  int flag = 0;
  int cur = 0;
  int nsw = 0;
  for (int sweep = 0;; ++sweep) {
    nsw = sweep;
    {
      const double2* A = As[warp][cur];
      double off = 0.0;
      for (int e = lane; e < kN * kN; e += 32) {
        const int i = e >> 4, j = e & 15;
        if (i < j) { const double2 a = A[aidx(i, j)]; off += a.x * a.x + a.y * a.y; }
      }
      off = sqrt(2.0 * wsum(off));
      if (off <= tol) break;
      if (sweep == kMaxSweeps) { flag |= DOA_INFO_NOCONV; break; }
    }
#pragma unroll 1
    for (int rnd = 0; rnd < kN - 1; ++rnd) {
      const double2* A = As[warp][cur];
      double2* An = As[warp][cur ^ 1];
      // ---- phase 1: rotation of slot pair k = lane & 7 + closed-form diagonal block.  Computed
      // branch-free by all lanes (lanes 8..31 on a dummy pair); only lanes 0..7 store.
      // Reciprocal square roots (MUFU seed + Newton, ~1 ulp) replace IEEE div/sqrt.
      {
        // only lanes 0..7 read (shared-memory wavefronts scale with the active lanes); the
        // others run the same instructions on a harmless dummy pair and store nothing
        double2 axy = make_double2(1.0, 0.0);
        double axx = 0.0, ayy = 0.0;
        if (lane < 8) {
          axy = A[rxy];
          axx = A[rxx].x;
          ayy = A[ryy].x;
        }
        const double r2 = axy.x * axy.x + axy.y * axy.y;
        const bool rot = r2 > 1e-300;                         // a_xy ~ 0: identity rotation
        // Short-chain parameters (same rotation as GvL sym.schur2): with d = (a_yy - a_xx)/2,
        // r = |a_xy|, h = sqrt(d^2 + r^2), q = |d| + h:  t = sign(d) r / q,  c = sqrt(q / 2h),
        // s = sign(d) r / sqrt(2 h q)  (c^2 + s^2 = 1 exactly in exact arithmetic), t r = sign(d) r^2 / q.
        // c's critical path is two MUFU+Newton reciprocal square roots instead of four chained
        // reciprocal (square) roots; s, e and t r run on parallel branches.
        const double ir = rsqrt_pos(rot ? r2 : 1.0);          // 1/|a_xy|
        const double rr = r2 * ir;                            // |a_xy|
        const double d = 0.5 * (ayy - axx);
        const double h2 = fma(d, d, r2);
        const double irh = rsqrt_pos(rot ? h2 : 1.0);          // 1/h
        const double h = h2 * irh;
        const double q = fabs(d) + h;
        const double u = 0.5 * q * irh;                       // c^2, in [1/2, 1]
        const double sabs = rr * rsqrt_pos(2.0 * h * q);
        const double trabs = r2 * rcp_pos(rot ? q : 1.0);
        const double tr = rot ? (d < 0.0 ? -trabs : trabs) : 0.0;   // t |a_xy|
        Prm p;
        p.c = rot ? u * rsqrt_pos(u) : 1.0;
        p.s = rot ? (d < 0.0 ? -sabs : sabs) : 0.0;
        p.er = rot ? axy.x * ir : 1.0;
        p.ei = rot ? -axy.y * ir : 0.0;
        if (lane < 8) {
          prm[warp][lane] = p;
          An[wxx] = make_double2(axx - tr, 0.0);
          An[wyy] = make_double2(ayy + tr, 0.0);
          An[wxy] = make_double2(0.0, 0.0);
        }
      }
      __syncwarp();
      // ---- phase 2a: off-diagonal block (rb, sb): B <- J_r^H B J_s, stored permuted
      if (lane < 28) {
        const Prm pr = prm[warp][rb], ps = prm[warp][sb];
        const double2 b00 = A[rd00], b01 = A[rd01], b10 = A[rd10], b11 = A[rd11];
        const double2 es = make_double2(ps.er, ps.ei), er = make_double2(pr.er, pr.ei);
        // columns (J_s): c0' = c b0 - s (e b1), c1' = s b0 + c (e b1)
        const double2 t0 = cmul(es, b01), t1 = cmul(es, b11);
        const double2 n00 = make_double2(ps.c * b00.x - ps.s * t0.x, ps.c * b00.y - ps.s * t0.y);
        const double2 n01 = make_double2(ps.s * b00.x + ps.c * t0.x, ps.s * b00.y + ps.c * t0.y);
        const double2 n10 = make_double2(ps.c * b10.x - ps.s * t1.x, ps.c * b10.y - ps.s * t1.y);
        const double2 n11 = make_double2(ps.s * b10.x + ps.c * t1.x, ps.s * b10.y + ps.c * t1.y);
        // rows (J_r^H): r0' = c r0 - s (conj(e) r1), r1' = s r0 + c (conj(e) r1)
        const double2 u0 = cmulc(er, n10), u1 = cmulc(er, n11);
        An[wr[0]] = make_double2(pr.c * n00.x - pr.s * u0.x, flip(pr.c * n00.y - pr.s * u0.y, sg[0]));
        An[wr[1]] = make_double2(pr.c * n01.x - pr.s * u1.x, flip(pr.c * n01.y - pr.s * u1.y, sg[1]));
        An[wr[2]] = make_double2(pr.s * n00.x + pr.c * u0.x, flip(pr.s * n00.y + pr.c * u0.y, sg[2]));
        An[wr[3]] = make_double2(pr.s * n01.x + pr.c * u1.x, flip(pr.s * n01.y + pr.c * u1.y, sg[3]));
      }
      // ---- phase 2b: V <- V J on this lane's four slot pairs (registers)
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const Prm p = prm[warp][4 * h + kk];
        const double2 vx = v[2 * kk], vy = v[2 * kk + 1];
        const double2 t = cmul(make_double2(p.er, p.ei), vy);
        v[2 * kk] = make_double2(p.c * vx.x - p.s * t.x, p.c * vx.y - p.s * t.y);
        v[2 * kk + 1] = make_double2(p.s * vx.x + p.c * t.x, p.s * vx.y + p.c * t.y);
      }
      // ---- caterpillar on V's column slots: s -> pi(s)
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

  // after whole sweeps slot == index (pi^15 = id): ascending stable sort of the diagonal
  const double2* A = As[warp][cur];
  if (lane < M) {
    const double li = A[aidx(lane, lane)].x;
    int rk = 0;
    for (int j = 0; j < M; ++j) {
      const double lj = A[aidx(j, j)].x;
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
      const int j = 8 * h + k;
      if (j < M) Vrow[rank_s[warp][j]] = v[k];
    }
  }
#ifdef DOA_EIG_COUNT
  flag |= nsw << 8;                                      // diagnostic builds only: sweeps in bits 8+
#endif
  if (lane == 0) info[b] = flag;
}

// Half-warp variant: two matrices per warp, one per 16-lane half.  Phase 1 of both
// matrices runs in the same instructions (lanes 0-7 and 16-23), so the redundant rotation lanes
// drop from 24 to 16 per matrix; each lane of a half owns one full row of V (16 complex) and two
// of the 28 off-diagonal blocks.  A converged matrix keeps running with identity rotations
// (c = 1, s = 0, e = 1: exact copies), so its outputs equal the one-matrix kernel's whatever
// its partner needs.
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
// half-lane -> block (row-major r < s index): pass 1 lanes 0-15 take entries 0-15, pass 2 lanes
// 0-11 entries 16-27; from the quarter-warp bank-conflict search (48 wavefronts per round for
// the block loads / permuted stores + phase 1, against 70 in natural order; ideal 38)
__device__ constexpr int kHalfOrder[28] = {11, 8, 13, 5, 10, 4, 2, 25, 22, 0, 15, 23, 19, 20,
                                           21, 18, 12, 7, 14, 27, 26, 9, 17, 16, 1, 3, 6, 24};

// N = 16 or 8 (M <= 8 uses the 8-index round robin: 7 rounds of 4 rotations per sweep).
template <int N> struct HLd { static constexpr int LD = N == 16 ? kLd : 9; };
template <int N>
__device__ __forceinline__ int aidxT(int i, int j) { return i * HLd<N>::LD + (j ^ (i >> 1)); }
__host__ __device__ constexpr int cat_next_c(int s, int n) {
  return s == 0 ? 0 : (s == 1 ? 2 : (s == n - 2 ? n - 1 : ((s & 1) ? s - 2 : s + 2)));
}
template <int N>
__device__ __forceinline__ int cat_nextT(int s) { return cat_next_c(s, N); }

template <int N>
__global__ void __launch_bounds__(kHWarps * 32, DOA_EIGH_MINB) eig16h_kernel(const double2* __restrict__ R,
                                                                             int64_t B, int M,
                                                                             double* __restrict__ lam_out,
                                                                             double2* __restrict__ V_out,
                                                                             int32_t* __restrict__ info) {
  __shared__ double2 As[kHWarps][2][2][N * HLd<N>::LD];          // [warp][half][buffer]
  __shared__ Prm prm[kHWarps][2][N / 2];
  __shared__ int rank_s[kHWarps][2][N];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int hm = lane >> 4, hl = lane & 15;
  const int64_t b = ((int64_t)blockIdx.x * kHWarps + warp) * 2 + hm;
  const bool valid = b < B;
  Prm* pm = prm[warp][hm];

  // ||R||_F and off(A) are summed in the same order as eig16_kernel's (lane partials over the
  // element strides of 32, i.e. this half-lane's even and odd strides of 16, added, then the tree),
  // so both kernels take identical stop decisions and a frame's results do not depend on B.
  double nrm_e = 0.0, nrm_o = 0.0;
  {
    const double2* Rb = R + (size_t)(valid ? b : 0) * M * M;
    for (int e = hl; e < N * N; e += 16) {
      const int i = e / N, j = e % N;
      if (i > j) continue;
      double2 v = make_double2(0.0, 0.0);
      if (valid && j < M) v = Rb[(size_t)i * M + j];
      if (i == j) v.y = 0.0;
      As[warp][hm][0][aidxT<N>(i, j)] = v;
      const double t = (i == j ? 1.0 : 2.0) * (v.x * v.x + v.y * v.y);
      if ((e / 16) & 1) nrm_o += t; else nrm_e += t;
    }
  }
  const double tol = 10.0 * DBL_EPSILON * sqrt(hsum(nrm_e + nrm_o));

  double2 v[N];                                           // row hl of this half's V
#pragma unroll
  for (int k = 0; k < N; ++k) v[k] = make_double2(k == hl ? 1.0 : 0.0, 0.0);

  // off-diagonal blocks per lane: t = hl (+ 16) < NBLK, row-major (r < s) order
  constexpr int NP = N / 2, NBLK = NP * (NP - 1) / 2, BPL = (NBLK + 15) / 16;
  int rb2[BPL], sb2[BPL], rd[BPL][4], wr[BPL][4], sgm[BPL];
#pragma unroll
  for (int u = 0; u < BPL; ++u) {
    int l = hl + 16 * u;
    l = l < NBLK ? (N == 16 ? kHalfOrder[l] : l) : 0;
    int rb = 0, sb = 1;
    for (int r = 0; r < NP; ++r) {
      const int cntr = NP - 1 - r;
      if (l < cntr) { rb = r; sb = r + 1 + l; break; }
      l -= cntr;
    }
    rb2[u] = rb; sb2[u] = sb;
    const int i0 = 2 * rb, i1 = i0 + 1, j0 = 2 * sb, j1 = j0 + 1;
    rd[u][0] = aidxT<N>(i0, j0); rd[u][1] = aidxT<N>(i0, j1); rd[u][2] = aidxT<N>(i1, j0); rd[u][3] = aidxT<N>(i1, j1);
    const int pr[2] = {cat_nextT<N>(i0), cat_nextT<N>(i1)}, pc[2] = {cat_nextT<N>(j0), cat_nextT<N>(j1)};
    int m = 0;
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int x = pr[a], y = pc[c];
        wr[u][2 * a + c] = x < y ? aidxT<N>(x, y) : aidxT<N>(y, x);
        m |= (x < y ? 0 : 1) << (2 * a + c);
      }
    sgm[u] = m;
  }
  const bool has2 = hl + 16 < NBLK;
  const int kx = 2 * (hl % NP), ky = kx + 1, px = cat_nextT<N>(kx), py = cat_nextT<N>(ky);
  const int rxy = aidxT<N>(kx, ky), rxx = aidxT<N>(kx, kx), ryy = aidxT<N>(ky, ky);
  const int wxx = aidxT<N>(px, px), wyy = aidxT<N>(py, py), wxy = px < py ? aidxT<N>(px, py) : aidxT<N>(py, px);
  __syncwarp();

  int flag = 0;
  int cur = 0;
  bool act = valid;
  for (int sweep = 0;; ++sweep) {
    {
      const double2* A = As[warp][hm][cur];
      double off_e = 0.0, off_o = 0.0;
      for (int e = hl; e < N * N; e += 16) {
        const int i = e / N, j = e % N;
        if (i < j) {
          const double2 a = A[aidxT<N>(i, j)];
          if ((e / 16) & 1) off_o += a.x * a.x + a.y * a.y; else off_e += a.x * a.x + a.y * a.y;
        }
      }
      const double off = sqrt(2.0 * hsum(off_e + off_o));
      if (act && off <= tol) act = false;
      else if (act && sweep == kMaxSweeps) { flag |= DOA_INFO_NOCONV; act = false; }
    }
    if (!__any_sync(0xffffffffu, act)) break;
#pragma unroll 1
    for (int rnd = 0; rnd < N - 1; ++rnd) {
      const double2* A = As[warp][hm][cur];
      double2* An = As[warp][hm][cur ^ 1];
      {
        double2 axy = make_double2(1.0, 0.0);
        double axx = 0.0, ayy = 0.0;
        if (hl < NP) {
          axy = A[rxy];
          axx = A[rxx].x;
          ayy = A[ryy].x;
        }
        const double r2 = axy.x * axy.x + axy.y * axy.y;
        const bool rot = act && r2 > 1e-300;               // frozen matrices: identity rotations
        const double ir = rsqrt_pos(rot ? r2 : 1.0);
        const double rr = r2 * ir;
        const double d = 0.5 * (ayy - axx);
        const double h2 = fma(d, d, r2);
        const double irh = rsqrt_pos(rot ? h2 : 1.0);
        const double hh = h2 * irh;
        const double q = fabs(d) + hh;
        const double uu = 0.5 * q * irh;
        const double sabs = rr * rsqrt_pos(2.0 * hh * q);
        const double trabs = r2 * rcp_pos(rot ? q : 1.0);
        const double tr = rot ? (d < 0.0 ? -trabs : trabs) : 0.0;
        Prm p;
        p.c = rot ? uu * rsqrt_pos(uu) : 1.0;
        p.s = rot ? (d < 0.0 ? -sabs : sabs) : 0.0;
        p.er = rot ? axy.x * ir : 1.0;
        p.ei = rot ? -axy.y * ir : 0.0;
        if (hl < NP) {
          pm[hl] = p;
          An[wxx] = make_double2(axx - tr, 0.0);
          An[wyy] = make_double2(ayy + tr, 0.0);
          An[wxy] = act ? make_double2(0.0, 0.0) : A[rxy];   // frozen: keep the element as it is
        }
      }
      __syncwarp();
#pragma unroll
      for (int u = 0; u < BPL; ++u) {
        if (u == 1 && !has2) break;
        const Prm pr = pm[rb2[u]], ps = pm[sb2[u]];
        const double2 b00 = A[rd[u][0]], b01 = A[rd[u][1]], b10 = A[rd[u][2]], b11 = A[rd[u][3]];
        const double2 es = make_double2(ps.er, ps.ei), er = make_double2(pr.er, pr.ei);
        const double2 t0 = cmul(es, b01), t1 = cmul(es, b11);
        const double2 n00 = make_double2(ps.c * b00.x - ps.s * t0.x, ps.c * b00.y - ps.s * t0.y);
        const double2 n01 = make_double2(ps.s * b00.x + ps.c * t0.x, ps.s * b00.y + ps.c * t0.y);
        const double2 n10 = make_double2(ps.c * b10.x - ps.s * t1.x, ps.c * b10.y - ps.s * t1.y);
        const double2 n11 = make_double2(ps.s * b10.x + ps.c * t1.x, ps.s * b10.y + ps.c * t1.y);
        const double2 u0 = cmulc(er, n10), u1 = cmulc(er, n11);
        const int m = sgm[u];
        An[wr[u][0]] = make_double2(pr.c * n00.x - pr.s * u0.x, flipb(pr.c * n00.y - pr.s * u0.y, m & 1));
        An[wr[u][1]] = make_double2(pr.c * n01.x - pr.s * u1.x, flipb(pr.c * n01.y - pr.s * u1.y, (m >> 1) & 1));
        An[wr[u][2]] = make_double2(pr.s * n00.x + pr.c * u0.x, flipb(pr.s * n00.y + pr.c * u0.y, (m >> 2) & 1));
        An[wr[u][3]] = make_double2(pr.s * n01.x + pr.c * u1.x, flipb(pr.s * n01.y + pr.c * u1.y, (m >> 3) & 1));
      }
      // V <- V J on the lane's row, then the slot permutation (register renaming + moves)
      double2 t[N];
#pragma unroll
      for (int k = 0; k < NP; ++k) {
        const Prm p = pm[k];
        const double2 vx = v[2 * k], vy = v[2 * k + 1];
        const double2 ey = cmul(make_double2(p.er, p.ei), vy);
        t[cat_next_c(2 * k, N)] = make_double2(p.c * vx.x - p.s * ey.x, p.c * vx.y - p.s * ey.y);
        t[cat_next_c(2 * k + 1, N)] = make_double2(p.s * vx.x + p.c * ey.x, p.s * vx.y + p.c * ey.y);
      }
#pragma unroll
      for (int k = 0; k < N; ++k) v[k] = t[k];
      cur ^= 1;
      __syncwarp();
    }
  }

  const double2* A = As[warp][hm][cur];
  if (hl < M) {
    const double li = A[aidxT<N>(hl, hl)].x;
    int rk = 0;
    for (int j = 0; j < M; ++j) {
      const double lj = A[aidxT<N>(j, j)].x;
      rk += (lj < li) || (lj == li && j < hl);
    }
    rank_s[warp][hm][hl] = rk;
    if (valid) lam_out[(size_t)b * M + rk] = li;
  }
  __syncwarp();
  if (valid && hl < M) {
    double2* Vrow = V_out + (size_t)b * M * M + (size_t)hl * M;
#pragma unroll
    for (int k = 0; k < N; ++k)
      if (k < M) Vrow[rank_s[warp][hm][k]] = v[k];
  }
  if (valid && hl == 0) info[b] = flag;
}

}  // namespace

cudaError_t launch_eig16(const double* R, int64_t B, int M, double* lam, double* V, int32_t* info, cudaStream_t s) {
  count_launch();
  // small batches of M > 8 (latency-bound single frames) take the one-warp-per-matrix kernel,
  // whose single-matrix round is shorter; it performs the same operations in the same order, so
  // the results are bitwise the same (tests/test_gpu_parity.py::test_eig_kernels_bitwise_equal)
  if (M <= 8 || B >= DOA_EIG_HALF_MIN_B) {
    const unsigned g = (unsigned)((B + 2 * kHWarps - 1) / (2 * kHWarps));
    if (M <= 8)
      eig16h_kernel<8><<<g, kHWarps * 32, 0, s>>>(reinterpret_cast<const double2*>(R), B, M, lam,
                                                   reinterpret_cast<double2*>(V), info);
    else
      eig16h_kernel<16><<<g, kHWarps * 32, 0, s>>>(reinterpret_cast<const double2*>(R), B, M, lam,
                                                    reinterpret_cast<double2*>(V), info);
    return cudaGetLastError();
  }
  eig16_kernel<<<(unsigned)((B + kEigWarps - 1) / kEigWarps), kEigWarps * 32, 0, s>>>(
      reinterpret_cast<const double2*>(R), B, M, lam, reinterpret_cast<double2*>(V), info);
  return cudaGetLastError();
}

}  // namespace doa
