// S2 for 16 < M <= 64: batched Hermitian Jacobi eigendecomposition, one CTA per matrix
// (N = 32: 128 threads, N = 64: 512 threads).  (Table 2 Step-2 `jsvd`; Q3.)
//
// Same algorithm as eig16_kernel (csrc/eig16.cu), scaled to N = 32 / 64 padded indices:
//   * circle-method round robin in fixed slots (N/2 disjoint pairs per round) with the
//     "caterpillar" permutation pi (slot 0 fixed, slots 1..N-1 on one (N-1)-cycle), folded into
//     the smem store addresses; pi^(N-1) = id, so slots equal indices again after every sweep;
//   * A = upper triangle in shared memory, double-buffered, swizzled layout aidxN (conflict search);
//   * phase 1 (threads < N/2): rotation parameters of the N/2 pairs + closed-form diagonal blocks;
//     phase 2: thread t < (N/2)(N/2-1)/2 updates off-diagonal 2x2 block t (B <- J_r^H B J_s);
//     every thread updates its 8 V entries in registers (V <- V J);
//   * V in registers: thread (row i = t / (N/8), group h = t % (N/8)) holds V[i][8h .. 8h+7];
//     pi moves one complex value to each neighbouring group per round (adjacent lanes: shuffles).
// Rotation and stop rule as eig16 (GvL sym.schur2 after the phase rotation; off(A) computed
// directly <= 10 eps ||R||_F before each sweep, at most 30 sweeps, Q15); eigenvalues ascending.
#include <cfloat>

#include "doa_internal.cuh"

namespace doa {
namespace {


struct PrmN {
  double c, s, er, ei;
};

// MUFU seed + one third-order correction (as csrc/eig16.cu; accuracy in tools/rsqrt_check.cu)
__device__ __forceinline__ double rsqrt_p(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double e = fma(-(x * y), y, 1.0);
  return fma(y * e, fma(e, 0.375, 0.5), y);
}
__device__ __forceinline__ double rcp_p(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double e = fma(-x, y, 1.0);
  return fma(y, fma(e, e, e), y);
}
__device__ __forceinline__ double2 cmulN(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cmulcN(double2 a, double2 b) {   // conj(a) * b
  return make_double2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
__device__ __forceinline__ int cat_nextN(int s, int N) {
  if (s == 0) return 0;
  if (s == 1) return 2;
  if (s == N - 2) return N - 1;
  return (s & 1) ? s - 2 : s + 2;
}

template <int N>
struct EigN {
  static constexpr int LD = N + 2;
  static constexpr int Q = N / 8;                 // V groups of 8 slots per row
  static constexpr int T = N * Q;                 // threads
  static constexpr int NP = N / 2;                // pairs per round
  static constexpr int NBLK = NP * (NP - 1) / 2;  // off-diagonal 2x2 blocks
};

// Shared memory serves a 16-byte-per-lane load in quarter-warps of 8 lanes, which must hit distinct
// 16-byte bank quads (slot % 8).  Phase 2b's quarter-warps read pairs 4h + kk, h = 0..7, and phase
// 2a's read about 8 consecutive pairs sb; the swizzle slot = p ^ ((p >> 3) & 3) keeps both
// conflict-free (2a: at most 2-way when the 8 pairs straddle a multiple of 8).
template <int N>
__device__ __forceinline__ int prm_slot(int p) { return p ^ ((p >> 3) & 3); }
template <int N>
__device__ __forceinline__ PrmN load_prm(const double2* cs, const double2* ee, int p) {
  const double2 a = cs[prm_slot<N>(p)], e = ee[prm_slot<N>(p)];
  PrmN r;
  r.c = a.x; r.s = a.y; r.er = e.x; r.ei = e.y;
  return r;
}

// A layout: row stride N + 2, columns XOR-swizzled within aligned groups of 8 by (j/2) ^ 2(i/2);
// chosen by an offline search over the 2a block loads and permuted stores (quarter-warps of 8
// lanes, 16-byte entries): 667 wavefronts per round at N = 64 against 993 for i*(N+3) + (j ^ i/2)
// and an ideal of 496.
template <int N>
__device__ __forceinline__ int aidxN(int i, int j) {
  return i * EigN<N>::LD + (j ^ ((((j >> 1) & 7) ^ ((i >> 1) * 2)) & 7));
}

template <int N>
__device__ __forceinline__ double block_sum(double v, double* red) {
  constexpr int T = EigN<N>::T;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < T / 32; ++w) s += red[w];                   // fixed order
  return s;
}

template <int N>
__global__ void __launch_bounds__(EigN<N>::T, 1) eigN_kernel(const double2* __restrict__ R, int64_t B, int M,
                                                             double* __restrict__ lam_out,
                                                             double2* __restrict__ V_out,
                                                             int32_t* __restrict__ info) {
  using E = EigN<N>;
  constexpr int LD = E::LD, Q = E::Q, NP = E::NP, NBLK = E::NBLK;
  extern __shared__ double2 As[];                                   // [2][N * LD]
  // rotation parameters as two arrays of 16-byte entries (c, s) and (er, ei), pair p at prm_slot(p)
  __shared__ double2 prm_cs[NP], prm_ee[NP];
  __shared__ double red[32];
  __shared__ int rank_s[N];
  const int tid = threadIdx.x;
  const int64_t b = blockIdx.x;
  const double2* Rb = R + (size_t)b * M * M;
  double2* A0 = As;

  double nrm = 0.0;
  for (int e = tid; e < N * N; e += E::T) {
    const int i = e / N, j = e - (e / N) * N;
    if (i > j) continue;
    double2 v = make_double2(0.0, 0.0);
    if (j < M) v = Rb[(size_t)i * M + j];
    if (i == j) v.y = 0.0;
    A0[aidxN<N>(i, j)] = v;
    nrm += (i == j ? 1.0 : 2.0) * (v.x * v.x + v.y * v.y);
  }
  nrm = sqrt(block_sum<N>(nrm, red));
  const double tol = 10.0 * DBL_EPSILON * nrm;

  const int vi = tid / Q, h = tid % Q;
  double2 v[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) v[k] = make_double2(vi == 8 * h + k ? 1.0 : 0.0, 0.0);

  // static geometry: off-diagonal block t = (rb < sb), read offsets and permuted write offsets
  const bool has_blk = tid < NBLK;
  int rb = 0, sb = 1;
  {
    int l = has_blk ? tid : 0;
    for (int r = 0; r < NP; ++r) {
      const int cntr = NP - 1 - r;
      if (l < cntr) { rb = r; sb = r + 1 + l; break; }
      l -= cntr;
    }
  }
  const int i0 = 2 * rb, i1 = i0 + 1, j0 = 2 * sb, j1 = j0 + 1;
  const int rd00 = aidxN<N>(i0, j0), rd01 = aidxN<N>(i0, j1), rd10 = aidxN<N>(i1, j0), rd11 = aidxN<N>(i1, j1);
  int wr[4];
  double sg[4];
  {
    const int pr[2] = {cat_nextN(i0, N), cat_nextN(i1, N)}, pc[2] = {cat_nextN(j0, N), cat_nextN(j1, N)};
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int x = pr[a], y = pc[c];
        wr[2 * a + c] = x < y ? aidxN<N>(x, y) : aidxN<N>(y, x);
        sg[2 * a + c] = x < y ? 1.0 : -1.0;
      }
  }
  const int kp = tid < NP ? tid : 0;
  const int kx = 2 * kp, ky = kx + 1, px = cat_nextN(kx, N), py = cat_nextN(ky, N);
  const int rxy = aidxN<N>(kx, ky), rxx = aidxN<N>(kx, kx), ryy = aidxN<N>(ky, ky);
  const int wxx = aidxN<N>(px, px), wyy = aidxN<N>(py, py), wxy = px < py ? aidxN<N>(px, py) : aidxN<N>(py, px);
  __syncthreads();

  int flag = 0;
  int cur = 0;
  for (int sweep = 0;; ++sweep) {
    double off = 0.0;
    {
      const double2* A = As + cur * N * LD;
      for (int e = tid; e < N * N; e += E::T) {
        const int i = e / N, j = e - (e / N) * N;
        if (i < j) { const double2 a = A[aidxN<N>(i, j)]; off += a.x * a.x + a.y * a.y; }
      }
    }
    off = sqrt(2.0 * block_sum<N>(off, red));
    if (off <= tol) break;
    if (sweep == kMaxSweeps) { flag |= DOA_INFO_NOCONV; break; }
    for (int rnd = 0; rnd < N - 1; ++rnd) {
      const double2* A = As + cur * N * LD;
      double2* An = As + (cur ^ 1) * N * LD;
      // ---- phase 1: rotations of the N/2 slot pairs + closed-form diagonal blocks
      if (tid < NP) {
        const double2 axy = A[rxy];
        const double axx = A[rxx].x, ayy = A[ryy].x;
        const double r2 = axy.x * axy.x + axy.y * axy.y;
        const bool rot = r2 > 1e-300;                         // a_xy ~ 0: identity rotation
        // Short-chain parameters (same rotation as GvL sym.schur2): with d = (a_yy - a_xx)/2,
        // r = |a_xy|, h = sqrt(d^2 + r^2), q = |d| + h:  t = sign(d) r / q,  c = sqrt(q / 2h),
        // s = sign(d) r / sqrt(2 h q)  (c^2 + s^2 = 1 exactly in exact arithmetic), t r = sign(d) r^2 / q.
        // c's critical path is two MUFU+correction reciprocal square roots instead of four chained
        // reciprocal (square) roots; s, e and t r run on parallel branches.  The MUFU inputs are not
        // guarded (a zero pivot gives inf/NaN intermediates): the identity is selected at the end,
        // keeping selects off the chain.
        const double ir = rsqrt_p(r2);          // 1/|a_xy|
        const double rr = r2 * ir;                            // |a_xy|
        const double d = 0.5 * (ayy - axx);
        const double h2 = fma(d, d, r2);
        const double irh = rsqrt_p(h2);          // 1/h
        const double h = h2 * irh;
        const double q = fabs(d) + h;
        const double u = 0.5 * q * irh;                       // c^2, in [1/2, 1]
        const double iu = rsqrt_p(u);                         // 2 h q = 4 h2 c^2: s = r irh iu / 2
        const double sabs = (0.5 * rr * irh) * iu;
        const double trabs = r2 * rcp_p(q);
        const double tr = rot ? (d < 0.0 ? -trabs : trabs) : 0.0;   // t |a_xy|
        PrmN p;
        p.c = rot ? u * iu : 1.0;
        p.s = rot ? (d < 0.0 ? -sabs : sabs) : 0.0;
        p.er = rot ? axy.x * ir : 1.0;
        p.ei = rot ? -axy.y * ir : 0.0;
        prm_cs[prm_slot<N>(tid)] = make_double2(p.c, p.s);
        prm_ee[prm_slot<N>(tid)] = make_double2(p.er, p.ei);
        An[wxx] = make_double2(axx - tr, 0.0);
        An[wyy] = make_double2(ayy + tr, 0.0);
        An[wxy] = make_double2(0.0, 0.0);
      }
      __syncthreads();
      // ---- phase 2a: off-diagonal block (rb, sb)
      if (has_blk) {
        const PrmN pr = load_prm<N>(prm_cs, prm_ee, rb), ps = load_prm<N>(prm_cs, prm_ee, sb);
        const double2 b00 = A[rd00], b01 = A[rd01], b10 = A[rd10], b11 = A[rd11];
        const double2 es = make_double2(ps.er, ps.ei), er = make_double2(pr.er, pr.ei);
        const double2 t0 = cmulN(es, b01), t1 = cmulN(es, b11);
        const double2 n00 = make_double2(ps.c * b00.x - ps.s * t0.x, ps.c * b00.y - ps.s * t0.y);
        const double2 n01 = make_double2(ps.s * b00.x + ps.c * t0.x, ps.s * b00.y + ps.c * t0.y);
        const double2 n10 = make_double2(ps.c * b10.x - ps.s * t1.x, ps.c * b10.y - ps.s * t1.y);
        const double2 n11 = make_double2(ps.s * b10.x + ps.c * t1.x, ps.s * b10.y + ps.c * t1.y);
        const double2 u0 = cmulcN(er, n10), u1 = cmulcN(er, n11);
        An[wr[0]] = make_double2(pr.c * n00.x - pr.s * u0.x, sg[0] * (pr.c * n00.y - pr.s * u0.y));
        An[wr[1]] = make_double2(pr.c * n01.x - pr.s * u1.x, sg[1] * (pr.c * n01.y - pr.s * u1.y));
        An[wr[2]] = make_double2(pr.s * n00.x + pr.c * u0.x, sg[2] * (pr.s * n00.y + pr.c * u0.y));
        An[wr[3]] = make_double2(pr.s * n01.x + pr.c * u1.x, sg[3] * (pr.s * n01.y + pr.c * u1.y));
      }
      // ---- phase 2b: V <- V J on this thread's four slot pairs
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const PrmN p = load_prm<N>(prm_cs, prm_ee, 4 * h + kk);
        const double2 vx = v[2 * kk], vy = v[2 * kk + 1];
        const double2 t = cmulN(make_double2(p.er, p.ei), vy);
        v[2 * kk] = make_double2(p.c * vx.x - p.s * t.x, p.c * vx.y - p.s * t.y);
        v[2 * kk + 1] = make_double2(p.s * vx.x + p.c * t.x, p.s * vx.y + p.c * t.y);
      }
      // ---- caterpillar on V's slots (groups of 8; neighbouring groups are adjacent lanes)
      {
        const double2 s_next = v[6], s_prev = v[1];
        const double2 r_prev = make_double2(__shfl_up_sync(0xffffffffu, s_next.x, 1),
                                            __shfl_up_sync(0xffffffffu, s_next.y, 1));
        const double2 r_next = make_double2(__shfl_down_sync(0xffffffffu, s_prev.x, 1),
                                            __shfl_down_sync(0xffffffffu, s_prev.y, 1));
        const double2 o0 = v[0], o1 = v[1], o2 = v[2], o3 = v[3], o4 = v[4], o5 = v[5], o6 = v[6], o7 = v[7];
        const bool first = h == 0, last = h == Q - 1;
        v[0] = first ? o0 : r_prev;
        v[1] = o3;
        v[2] = first ? o1 : o0;
        v[3] = o5;
        v[4] = o2;
        v[5] = o7;
        v[6] = o4;
        v[7] = last ? o6 : r_next;
      }
      cur ^= 1;
      __syncthreads();
    }
  }

  const double2* A = As + cur * N * LD;
  if (tid < M) {
    const double li = A[aidxN<N>(tid, tid)].x;
    int rk = 0;
    for (int j = 0; j < M; ++j) {
      const double lj = A[aidxN<N>(j, j)].x;
      rk += (lj < li) || (lj == li && j < tid);
    }
    rank_s[tid] = rk;
    lam_out[(size_t)b * M + rk] = li;
  }
  __syncthreads();
  if (vi < M) {
    double2* Vrow = V_out + (size_t)b * M * M + (size_t)vi * M;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int j = 8 * h + k;
      if (j < M) Vrow[rank_s[j]] = v[k];
    }
  }
  if (tid == 0) info[b] = flag;
}

template <int N>
cudaError_t launch_eigN_t(const double* R, int64_t B, int M, double* lam, double* V, int32_t* info, cudaStream_t s) {
  const size_t smem = (size_t)2 * N * EigN<N>::LD * sizeof(double2);
  kernel_occupancy(eigN_kernel<N>, EigN<N>::T, smem);               // sets the smem attribute on this device
  count_launch();
  eigN_kernel<N><<<(unsigned)B, EigN<N>::T, smem, s>>>(reinterpret_cast<const double2*>(R), B, M, lam,
                                                       reinterpret_cast<double2*>(V), info);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_eigN(const double* R, int64_t B, int M, double* lam, double* V, int32_t* info, cudaStream_t s) {
  if (M <= 32) return launch_eigN_t<32>(R, B, M, lam, V, info, s);
  return launch_eigN_t<64>(R, B, M, lam, V, info, s);
}

}  // namespace doa
