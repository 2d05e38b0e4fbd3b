// ORACLE — test infrastructure only.  Plain, slow, obviously-correct fp64 CPU reference for
// the DOA hot path of Eray & Temizel, arXiv 2007.14135 ("Performance Analysis of Noise
// Subspace-based Narrowband DOA Estimation Algorithms on CPU and GPU").
//
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may
// load this library.  The product path (paper_2007_14135_b200/) never links, imports or calls
// it, and it shares no code, header, table or constant generator with the CUDA library.
//
// Every routine follows one step of the paper's Table 2 (§3.2) / Table 3
// in the paper's order, written as its plain definition in IEEE double precision.
// Readings of silent / garbled points are the SURVEY.md §8(c) Q-numbers, listed in DESIGN.md §2.
// Build: g++ -O2 -std=c++17 -ffp-contract=off -fPIC -shared (no fast-math, no intrinsics).
//
// Layouts (all row-major, complex numbers interleaved as (re, im)):
//   X  [N][M]  complex64   one frame of snapshots, snapshot-major (x_m[n] at X[n*M+m])
//   R  [M][M]  complex128  sample covariance
//   V  [M][M]  complex128  eigenvectors, column j = eigenvector of lambda[j] (ascending)
//   C  [M][M]  complex128  Table-3 Step-4 matrix
//   f  [L]     double      floored quadratic form f_c(theta_i) = max(a^H C a, 1e-300); P = 1/f_c
//
// Parity status of each function is recorded in DESIGN.md §4 (all functions here are pinned
// by tests/test_oracle_*.py; none is "parity unpinned").
#include <algorithm>
#include <cfloat>
#include <cmath>
#include <complex>
#include <cstdint>
#include <thread>
#include <vector>

namespace {

typedef std::complex<double> cd;

const int ALG_PHD = 0, ALG_MUSIC = 1, ALG_EV = 2, ALG_MN = 3;
const int INFO_NOCONV = 1, INFO_DEGENERATE = 2, INFO_UNDERDETERMINED = 8;
const int MAX_SWEEPS = 30;
const double F_FLOOR = 1e-300;

// Table 2 Step-1 / Eq. 3: R = (1/N) sum_n x[n] x[n]^H, i.e.
// R_ij = (sum_n x_i[n] * conj(x_j[n])) / N, sequential n loop (1/N).
void covariance(const float* X, int64_t N, int M, std::vector<cd>& R) {
  R.assign((size_t)M * M, cd(0.0, 0.0));
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < M; ++j) {
      double sr = 0.0, si = 0.0;
      for (int64_t n = 0; n < N; ++n) {
        const double ar = X[2 * (n * M + i)], ai = X[2 * (n * M + i) + 1];
        const double br = X[2 * (n * M + j)], bi = X[2 * (n * M + j) + 1];
        // x_i * conj(x_j) = (ar + j ai)(br - j bi)
        sr += ar * br + ai * bi;
        si += ai * br - ar * bi;
      }
      R[(size_t)i * M + j] = cd(sr / (double)N, si / (double)N);
    }
}

double frob(const std::vector<cd>& A) {
  double s = 0.0;
  for (const cd& a : A) s += std::norm(a);
  return std::sqrt(s);
}

double offdiag(const std::vector<cd>& A, int M) {
  double s = 0.0;  // computed directly, not by subtraction
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < M; ++j)
      if (i != j) s += std::norm(A[(size_t)i * M + j]);
  return std::sqrt(s);
}

// Table 2 Step-2 (Eigen JacobiSVD).  For the Hermitian PSD R the SVD is the
// eigendecomposition.  Textbook cyclic-by-rows complex Jacobi: Golub & Van Loan
// sym.schur2 on the 2x2 block after a phase rotation that makes a_pq real.
// Stop when off(A) <= 10*eps*||R||_F, at most 30 sweeps.  lambda ascending,
// stable.  Returns the number of sweeps performed.
int eig(const std::vector<cd>& R, int M, std::vector<double>& lam, std::vector<cd>& V, int* info) {
  std::vector<cd> A = R;
  std::vector<cd> W((size_t)M * M, cd(0.0, 0.0));
  for (int i = 0; i < M; ++i) W[(size_t)i * M + i] = cd(1.0, 0.0);
  for (int i = 0; i < M; ++i) A[(size_t)i * M + i] = cd(A[(size_t)i * M + i].real(), 0.0);
  const double tol = 10.0 * DBL_EPSILON * frob(R);
  int sweep = 0;
  for (;; ++sweep) {
    if (offdiag(A, M) <= tol) break;
    if (sweep == MAX_SWEEPS) { *info |= INFO_NOCONV; break; }
    for (int p = 0; p < M - 1; ++p)
      for (int q = p + 1; q < M; ++q) {
        const cd apq = A[(size_t)p * M + q];
        const double r = std::abs(apq);
        if (r == 0.0) continue;
        const double app = A[(size_t)p * M + p].real(), aqq = A[(size_t)q * M + q].real();
        const cd e = std::conj(apq) / r;                       // e^{-j phi}, phi = arg a_pq
        const double tau = (aqq - app) / (2.0 * r);
        const double t = (tau >= 0.0 ? 1.0 : -1.0) / (std::fabs(tau) + std::sqrt(1.0 + tau * tau));
        const double c = 1.0 / std::sqrt(1.0 + t * t);
        const double s = t * c;
        // J = diag(1, e) [[c, s], [-s, c]]:  J_pp = c, J_pq = s, J_qp = -s e, J_qq = c e.
        const cd Jpp(c, 0.0), Jpq(s, 0.0), Jqp = -s * e, Jqq = c * e;
        for (int i = 0; i < M; ++i) {                           // A <- A J (columns p, q)
          const cd aip = A[(size_t)i * M + p], aiq = A[(size_t)i * M + q];
          A[(size_t)i * M + p] = aip * Jpp + aiq * Jqp;
          A[(size_t)i * M + q] = aip * Jpq + aiq * Jqq;
        }
        for (int j = 0; j < M; ++j) {                           // A <- J^H A (rows p, q)
          const cd apj = A[(size_t)p * M + j], aqj = A[(size_t)q * M + j];
          A[(size_t)p * M + j] = std::conj(Jpp) * apj + std::conj(Jqp) * aqj;
          A[(size_t)q * M + j] = std::conj(Jpq) * apj + std::conj(Jqq) * aqj;
        }
        for (int i = 0; i < M; ++i) {                           // V <- V J
          const cd vip = W[(size_t)i * M + p], viq = W[(size_t)i * M + q];
          W[(size_t)i * M + p] = vip * Jpp + viq * Jqp;
          W[(size_t)i * M + q] = vip * Jpq + viq * Jqq;
        }
        A[(size_t)p * M + q] = cd(0.0, 0.0);
        A[(size_t)q * M + p] = cd(0.0, 0.0);
        A[(size_t)p * M + p] = cd(A[(size_t)p * M + p].real(), 0.0);
        A[(size_t)q * M + q] = cd(A[(size_t)q * M + q].real(), 0.0);
      }
  }
  std::vector<int> order(M);
  for (int i = 0; i < M; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
    return A[(size_t)a * M + a].real() < A[(size_t)b * M + b].real();
  });
  lam.resize(M);
  V.assign((size_t)M * M, cd(0.0, 0.0));
  for (int j = 0; j < M; ++j) {
    lam[j] = A[(size_t)order[j] * M + order[j]].real();
    for (int i = 0; i < M; ++i) V[(size_t)i * M + j] = W[(size_t)i * M + order[j]];
  }
  return sweep;
}

// Table 3 Step-3, in the readings of SURVEY Q1/Q2/Q4/Q5.  Produces the noise-subspace
// objects as a weighted set of vectors {(w_k, u_k)} such that the Step-4 matrix is
// C = sum_k w_k u_k u_k^H:
//   PHD   : e_min = column 0                                   C = e_min e_min^H
//   MUSIC : E_n = columns 0..K-1, K = M - D                     C = E_n E_n^H
//   EV    : same E_n, weights 1/lambda_k  (north_star; Q1)      C = sum_k (1/lambda_k) e_k e_k^H
//   MN    : P_n = E_n E_n^H, lambda' = (e1^H P_n e1)^-1, valph = lambda' P_n e1   C = valph valph^H
// Degenerate guards: an EV noise eigenvalue <= 100 eps lambda_max is clamped to
// that floor (weight 1 if the floor is 0); MN with e1^H P_n e1 <= 100 eps keeps valph = P_n e1.
struct Subspace {
  std::vector<double> w;             // weights
  std::vector<std::vector<cd>> u;    // vectors
};

Subspace noise_subspace(int alg, int M, int D, const std::vector<double>& lam, const std::vector<cd>& V, int* info) {
  Subspace S;
  const int K = M - D;
  auto col = [&](int k) {
    std::vector<cd> v(M);
    for (int i = 0; i < M; ++i) v[i] = V[(size_t)i * M + k];
    return v;
  };
  if (alg == ALG_PHD) {
    S.w.push_back(1.0);
    S.u.push_back(col(0));
  } else if (alg == ALG_MUSIC) {
    for (int k = 0; k < K; ++k) { S.w.push_back(1.0); S.u.push_back(col(k)); }
  } else if (alg == ALG_EV) {
    const double lmax = std::max(lam[M - 1], 0.0);
    const double floor_ = 100.0 * DBL_EPSILON * lmax;
    for (int k = 0; k < K; ++k) {
      double wk;
      if (lam[k] <= floor_) { *info |= INFO_DEGENERATE; wk = floor_ > 0.0 ? 1.0 / floor_ : 1.0; }
      else wk = 1.0 / lam[k];
      S.w.push_back(wk);
      S.u.push_back(col(k));
    }
  } else {  // MN
    std::vector<cd> p(M, cd(0.0, 0.0));             // P_n e1 = sum_k e_k conj(e_k[0])
    for (int k = 0; k < K; ++k)
      for (int i = 0; i < M; ++i) p[i] += V[(size_t)i * M + k] * std::conj(V[(size_t)0 * M + k]);
    double p0 = 0.0;                                 // e1^H P_n e1 = sum_k |e_k[0]|^2
    for (int k = 0; k < K; ++k) p0 += std::norm(V[(size_t)0 * M + k]);
    if (p0 <= 100.0 * DBL_EPSILON) { *info |= INFO_DEGENERATE; }
    else { const double lp = 1.0 / p0; for (int i = 0; i < M; ++i) p[i] *= lp; }
    S.w.push_back(1.0);
    S.u.push_back(p);
  }
  return S;
}

// Grid angle theta_i (Q26): theta0 + i*dtheta (rounded multiply, then
// rounded add, no FMA).  When the grid is symmetric about 0 — its last point computed that way is
// exactly -theta0, as for every -a:d:a grid of the paper ("-90:0.01:90") — the upper half
// is built from the other end, theta_i = -theta_{L-1-i} for i >= H = ceil(L/2), so the computed
// grid is exactly symmetric like the mathematical one (MATLAB's colon also builds a:d:b from
// both ends).
bool grid_symmetric(double theta0, double dtheta, int64_t L) {
  return L >= 2 && theta0 + (double)(L - 1) * dtheta == -theta0;
}
double grid_theta(double theta0, double dtheta, int64_t L, bool sym, int64_t i) {
  if (sym && i >= (L + 1) / 2) return -(theta0 + (double)(L - 1 - i) * dtheta);
  return theta0 + (double)i * dtheta;
}

// Table 2 Step-5 on the ULA grid: theta_i as grid_theta,
// u_i = 2 (d/lambda) sin(theta_i * pi/180), a_m = exp(-j pi m u_i) formed per element (no
// recurrence).  invP = a^H C a evaluated as the sum of squares sum_k w_k |u_k^H a|^2 (identical
// to a^H (sum_k w_k u_k u_k^H) a), floored at 1e-300 (Q12).
void spectrum(const Subspace& S, int M, double dl, double theta0, double dtheta, int64_t L, int64_t i0, int64_t i1,
              double* f) {
  const double pi = 3.14159265358979323846;
  const bool sym = grid_symmetric(theta0, dtheta, L);
  std::vector<cd> a(M);
  for (int64_t i = i0; i < i1; ++i) {
    const double th = grid_theta(theta0, dtheta, L, sym, i);
    const double u = 2.0 * dl * std::sin(th * pi / 180.0);
    for (int m = 0; m < M; ++m) {
      const double ph = pi * (double)m * u;
      a[m] = cd(std::cos(ph), -std::sin(ph));
    }
    double acc = 0.0;
    for (size_t k = 0; k < S.u.size(); ++k) {
      cd ip(0.0, 0.0);
      for (int m = 0; m < M; ++m) ip += std::conj(S.u[k][m]) * a[m];
      acc += S.w[k] * std::norm(ip);
    }
    f[i] = acc > F_FLOOR ? acc : F_FLOOR;
  }
}

// Table 2 Step-6: findPeaks on f (local minima of f = local maxima of P; interior only,
// strict on the left, non-strict on the right: SURVEY Q9/Q10), then PeakSelection: order by
// (f ascending, index ascending) and keep min(D, count) (Q11).  Returns the candidate count.
int64_t peaks(const double* f, int64_t L, int D, int32_t* idx, double* fval, int32_t* npk) {
  std::vector<std::pair<double, int64_t>> cand;
  for (int64_t i = 1; i + 1 < L; ++i)
    if (f[i] < f[i - 1] && f[i] <= f[i + 1]) cand.push_back({f[i], i});
  std::sort(cand.begin(), cand.end());
  const int n = (int)std::min<int64_t>(D, (int64_t)cand.size());
  for (int k = 0; k < D; ++k) {
    idx[k] = k < n ? (int32_t)cand[k].second : -1;
    fval[k] = k < n ? cand[k].first : 0.0;
  }
  *npk = n;
  return (int64_t)cand.size();
}

// general array geometry on an azimuth x elevation grid (the paper's own
// UCA workload).  Steering is Eq. 2 written out per element, with
// positions in wavelengths: a_k = exp{ j 2 pi (x_k sin(az) sin(el) + y_k cos(az) sin(el) +
// z_k cos(el)) }; grid az_i = az0 + i*daz, el_j = el0 + j*del (multiply then add), flattened
// azimuth-major p = i*nel + j.  invP = sum_k w_k |u_k^H a|^2, floored (Q12).
void spectrum_array(const Subspace& S, int M, const double* pos, double az0, double daz, int64_t nel,
                    double el0, double del, int64_t p0, int64_t p1, double* f) {
  const double pi = 3.14159265358979323846;
  std::vector<cd> a(M);
  for (int64_t p = p0; p < p1; ++p) {
    const int64_t ia = p / nel, ie = p % nel;
    const double az = (az0 + (double)ia * daz) * pi / 180.0;
    const double el = (el0 + (double)ie * del) * pi / 180.0;
    for (int m = 0; m < M; ++m) {
      const double ph = 2.0 * pi * (pos[3 * m] * std::sin(az) * std::sin(el) +
                                    pos[3 * m + 1] * std::cos(az) * std::sin(el) + pos[3 * m + 2] * std::cos(el));
      a[m] = cd(std::cos(ph), std::sin(ph));
    }
    double acc = 0.0;
    for (size_t k = 0; k < S.u.size(); ++k) {
      cd ip(0.0, 0.0);
      for (int m = 0; m < M; ++m) ip += std::conj(S.u[k][m]) * a[m];
      acc += S.w[k] * std::norm(ip);
    }
    f[p] = acc > F_FLOOR ? acc : F_FLOOR;
  }
}

// 2-D findPeaks (reading DESIGN.md G2): p is a local minimum of f (maximum of P) iff for each of
// its 8 neighbours n: f_p < f_n when n precedes p in raster order, f_p <= f_n when it follows
// (a plateau collapses to its first raster point).  Azimuth wraps when `wrap`; neighbours beyond
// the elevation range (or the azimuth range without wrap) do not exist.  Then PeakSelection as
// in 1-D: order by (f ascending, raster index ascending), keep min(D, count).
int64_t peaks2d(const double* f, int64_t naz, int64_t nel, int wrap, int D, int32_t* idx, double* fval,
                int32_t* npk) {
  std::vector<std::pair<double, int64_t>> cand;
  for (int64_t ia = 0; ia < naz; ++ia)
    for (int64_t ie = 0; ie < nel; ++ie) {
      const int64_t p = ia * nel + ie;
      bool peak = true;
      for (int da = -1; da <= 1 && peak; ++da)
        for (int de = -1; de <= 1 && peak; ++de) {
          if (da == 0 && de == 0) continue;
          int64_t ja = ia + da;
          const int64_t je = ie + de;
          if (je < 0 || je >= nel) continue;
          if (ja < 0 || ja >= naz) {
            if (!wrap) continue;
            ja = (ja + naz) % naz;
          }
          const int64_t n = ja * nel + je;
          if (n == p) continue;
          if (n < p ? !(f[p] < f[n]) : !(f[p] <= f[n])) peak = false;
        }
      if (peak) cand.push_back({f[p], p});
    }
  std::sort(cand.begin(), cand.end());
  const int n = (int)std::min<int64_t>(D, (int64_t)cand.size());
  for (int k = 0; k < D; ++k) {
    idx[k] = k < n ? (int32_t)cand[k].second : -1;
    fval[k] = k < n ? cand[k].first : 0.0;
  }
  *npk = n;
  return (int64_t)cand.size();
}

// P = 1/f_c reported in fp32, saturating at FLT_MAX.
float to_p32(double f) {
  const double p = 1.0 / f;
  return p > (double)FLT_MAX ? FLT_MAX : (float)p;
}

void pack(const std::vector<cd>& A, double* out) {
  for (size_t i = 0; i < A.size(); ++i) { out[2 * i] = A[i].real(); out[2 * i + 1] = A[i].imag(); }
}
std::vector<cd> unpack(const double* in, size_t n) {
  std::vector<cd> A(n);
  for (size_t i = 0; i < n; ++i) A[i] = cd(in[2 * i], in[2 * i + 1]);
  return A;
}

}  // namespace

extern "C" {

int oracle_version(void) { return 1; }

void oracle_covariance(const float* X, int64_t N, int M, double* R) {
  std::vector<cd> Rv;
  covariance(X, N, M, Rv);
  pack(Rv, R);
}

// Returns sweeps performed; info gets NOCONV.
int oracle_eig(const double* R, int M, double* lam, double* V, int* info) {
  std::vector<double> l;
  std::vector<cd> Vv;
  int inf = 0;
  const int sw = eig(unpack(R, (size_t)M * M), M, l, Vv, &inf);
  for (int i = 0; i < M; ++i) lam[i] = l[i];
  pack(Vv, V);
  *info = inf;
  return sw;
}

// Table 3 Step-4 matrix C = sum_k w_k u_k u_k^H (explicitly formed; used by pins and by the
// tie-certification bound of the tests).
void oracle_projector(int alg, int M, int D, const double* lam, const double* V, double* C, int* info) {
  std::vector<double> l(lam, lam + M);
  int inf = 0;
  Subspace S = noise_subspace(alg, M, D, l, unpack(V, (size_t)M * M), &inf);
  std::vector<cd> Cm((size_t)M * M, cd(0.0, 0.0));
  for (size_t k = 0; k < S.u.size(); ++k)
    for (int p = 0; p < M; ++p)
      for (int q = 0; q < M; ++q) Cm[(size_t)p * M + q] += S.w[k] * S.u[k][p] * std::conj(S.u[k][q]);
  pack(Cm, C);
  *info = inf;
}

// f_c over the whole grid; angle range split over `nthreads` std::threads (contiguous chunks).
void oracle_spectrum(int alg, int M, int D, double dl, const double* lam, const double* V, double theta0,
                     double dtheta, int64_t L, double* f, int nthreads, int* info) {
  std::vector<double> l(lam, lam + M);
  int inf = 0;
  Subspace S = noise_subspace(alg, M, D, l, unpack(V, (size_t)M * M), &inf);
  if (nthreads <= 1) {
    spectrum(S, M, dl, theta0, dtheta, L, 0, L, f);
  } else {
    std::vector<std::thread> th;
    for (int t = 0; t < nthreads; ++t) {
      const int64_t a = L * t / nthreads, b = L * (t + 1) / nthreads;
      th.emplace_back([&, a, b] { spectrum(S, M, dl, theta0, dtheta, L, a, b, f); });
    }
    for (auto& x : th) x.join();
  }
  *info = inf;
}

int64_t oracle_peaks(const double* f, int64_t L, int D, int32_t* idx, double* fval, int32_t* npk) {
  return peaks(f, L, D, idx, fval, npk);
}

// Whole hot path for a batch of frames X[B][N][M] with one algorithm; frames spread over
// `nthreads` std::threads.  Outputs per frame: idx[D] (-1 pad), val[D] = (float)(1/f) (0 pad),
// npk, info (NOCONV | DEGENERATE | UNDERDETERMINED), sweeps.  P (nullable) gets (float)(1/f_c).
void oracle_run_batch(int alg, int M, int D, double dl, double theta0, double dtheta, int64_t L,
                      const float* X, int64_t B, int64_t N, int32_t* idx, float* val, int32_t* npk,
                      int32_t* info, int32_t* sweeps, float* P, int nthreads) {
  auto work = [&](int64_t b0, int64_t b1) {
    std::vector<double> f((size_t)L);
    std::vector<cd> R, V;
    std::vector<double> lam;
    std::vector<double> fv(D);
    for (int64_t b = b0; b < b1; ++b) {
      int inf = 0;
      covariance(X + (size_t)b * N * M * 2, N, M, R);
      const int sw = eig(R, M, lam, V, &inf);
      Subspace S = noise_subspace(alg, M, D, lam, V, &inf);
      spectrum(S, M, dl, theta0, dtheta, L, 0, L, f.data());
      peaks(f.data(), L, D, idx + b * D, fv.data(), npk + b);
      for (int k = 0; k < D; ++k) val[b * D + k] = k < npk[b] ? to_p32(fv[k]) : 0.0f;
      if (npk[b] < D) inf |= INFO_UNDERDETERMINED;
      info[b] = inf;
      if (sweeps) sweeps[b] = sw;
      if (P)
        for (int64_t i = 0; i < L; ++i) P[(size_t)b * L + i] = to_p32(f[i]);
    }
  };
  if (nthreads <= 1 || B == 1) {
    work(0, B);
  } else {
    std::vector<std::thread> th;
    for (int t = 0; t < nthreads; ++t) {
      const int64_t a = B * t / nthreads, c = B * (t + 1) / nthreads;
      if (a < c) th.emplace_back(work, a, c);
    }
    for (auto& x : th) x.join();
  }
}

// NEXT-1: spectrum of a general array on the az x el grid (f_c[naz*nel], azimuth-major).
void oracle_spectrum_array(int alg, int M, int D, const double* pos, const double* lam, const double* V,
                           double az0, double daz, int64_t naz, double el0, double del, int64_t nel, double* f,
                           int nthreads, int* info) {
  std::vector<double> l(lam, lam + M);
  int inf = 0;
  Subspace S = noise_subspace(alg, M, D, l, unpack(V, (size_t)M * M), &inf);
  const int64_t L = naz * nel;
  if (nthreads <= 1) {
    spectrum_array(S, M, pos, az0, daz, nel, el0, del, 0, L, f);
  } else {
    std::vector<std::thread> th;
    for (int t = 0; t < nthreads; ++t) {
      const int64_t a = L * t / nthreads, b = L * (t + 1) / nthreads;
      th.emplace_back([&, a, b] { spectrum_array(S, M, pos, az0, daz, nel, el0, del, a, b, f); });
    }
    for (auto& x : th) x.join();
  }
  *info = inf;
}

int64_t oracle_peaks2d(const double* f, int64_t naz, int64_t nel, int wrap, int D, int32_t* idx, double* fval,
                       int32_t* npk) {
  return peaks2d(f, naz, nel, wrap, D, idx, fval, npk);
}

// NEXT-1 whole path for a batch of frames of a general array.
void oracle_run_array_batch(int alg, int M, int D, const double* pos, double az0, double daz, int64_t naz,
                            double el0, double del, int64_t nel, int wrap, const float* X, int64_t B, int64_t N,
                            int32_t* idx, float* val, int32_t* npk, int32_t* info, float* P, int nthreads) {
  const int64_t L = naz * nel;
  auto work = [&](int64_t b0, int64_t b1) {
    std::vector<double> f((size_t)L), fv(D);
    std::vector<cd> R, V;
    std::vector<double> lam;
    for (int64_t b = b0; b < b1; ++b) {
      int inf = 0;
      covariance(X + (size_t)b * N * M * 2, N, M, R);
      eig(R, M, lam, V, &inf);
      Subspace S = noise_subspace(alg, M, D, lam, V, &inf);
      spectrum_array(S, M, pos, az0, daz, nel, el0, del, 0, L, f.data());
      peaks2d(f.data(), naz, nel, wrap, D, idx + b * D, fv.data(), npk + b);
      for (int k = 0; k < D; ++k) val[b * D + k] = k < npk[b] ? to_p32(fv[k]) : 0.0f;
      if (npk[b] < D) inf |= INFO_UNDERDETERMINED;
      info[b] = inf;
      if (P)
        for (int64_t i = 0; i < L; ++i) P[(size_t)b * L + i] = to_p32(f[i]);
    }
  };
  if (nthreads <= 1 || B == 1) {
    work(0, B);
  } else {
    std::vector<std::thread> th;
    for (int t = 0; t < nthreads; ++t) {
      const int64_t a = B * t / nthreads, c = B * (t + 1) / nthreads;
      if (a < c) th.emplace_back(work, a, c);
    }
    for (auto& x : th) x.join();
  }
}

}  // extern "C"
