// general array geometry on an azimuth x elevation grid — the paper's own
// workload (8-element UCA; scan ranges 360 x {1, 30, 60, 90}).
//
// Steering is Eq. 2 with positions in wavelengths.  Without the ULA's Toeplitz structure
// the quadratic form still reduces to a real contraction: with z_pq = conj(a_p) a_q =
// exp(j 2 pi (r_q - r_p) . u(az, el)),
//     f = a^H C a = sum_p C_pp + 2 sum_{p<q} ( Re C_pq cos(phi_pq) - Im C_pq sin(phi_pq) ),
// K = 1 + M(M-1) terms per (frame, angle) against a per-angle table shared by all frames, so the
// scan runs on the same FP64 DMMA machinery as the ULA path (table in shared memory in B-fragment
// order, coefficients in the A-fragment layout).  The 2-D peak search (8-neighbourhood, azimuth
// wrap, raster tie rule — DESIGN.md G2) runs on the floored f written to the plan's buffer.
#include <cfloat>

#include "doa_internal.cuh"

namespace doa {
namespace {

constexpr double kFloorA = 1e-300;          // Q12

__device__ __forceinline__ float to_p32a(double f) {
  const double p = 1.0 / f;
  return p > (double)FLT_MAX ? FLT_MAX : (float)p;
}

__device__ __forceinline__ void dmma_a(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void pair_of(int idx, int M, int& p, int& q) {
  p = 0;
  while (idx >= M - 1 - p) { idx -= M - 1 - p; ++p; }
  q = p + 1 + idx;
}

// S3 for general arrays: one warp per frame; same noise-subspace objects as the ULA path
// (Table 3, Q1/Q5, G1), then c_0 = trace C and (2 Re C_pq, -2 Im C_pq) for p < q,
// C_pq = sum_j w_j u_j[p] conj(u_j[q]), written in the DMMA A-fragment layout.
__global__ void __launch_bounds__(128) coef_array_kernel(const double* __restrict__ lam,
                                                        const double2* __restrict__ V, int64_t B, int M, int D,
                                                        int alg, double* __restrict__ coef,
                                                        int32_t* __restrict__ cnt, int32_t* __restrict__ info) {
  __shared__ double2 Us[4][16 * 17];
  __shared__ double ws[4][16];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t b = (int64_t)blockIdx.x * 4 + warp;
  if (b >= B) return;
  const int ld = 17;
  double2* U = Us[warp];
  const int S = array_ksteps(M), K = array_terms(M);
  const double2* Vb = V + (size_t)b * M * M;
  const double* lb = lam + (size_t)b * M;
  const int Kn = M - D;
  int flag = 0;
  const int nload = (alg == DOA_ALG_PHD) ? 1 : Kn;
  for (int e = lane; e < M * M; e += 32) {
    const int p = e / M, j = e - (e / M) * M;
    if (j < nload) U[j * ld + p] = Vb[e];
  }
  int nv = (alg == DOA_ALG_MUSIC || alg == DOA_ALG_EV) ? Kn : 1;
  if (lane < 16) ws[warp][lane] = 1.0;
  if (alg == DOA_ALG_EV) {
    const double lfloor = 100.0 * DBL_EPSILON * fmax(lb[M - 1], 0.0);
    for (int j = 0; j < Kn; ++j) if (lb[j] <= lfloor) flag |= DOA_INFO_DEGENERATE;
    if (lane < Kn) ws[warp][lane] = lb[lane] <= lfloor ? (lfloor > 0.0 ? 1.0 / lfloor : 1.0) : 1.0 / lb[lane];
  }
  __syncwarp();
  if (alg == DOA_ALG_MN) {
    double p0 = 0.0;
    for (int j = 0; j < Kn; ++j) { const double2 v = U[j * ld]; p0 += v.x * v.x + v.y * v.y; }
    const bool degen = !(p0 > 100.0 * DBL_EPSILON);
    if (degen) flag |= DOA_INFO_DEGENERATE;
    const double lp = degen ? 1.0 : 1.0 / p0;
    double2 wv = make_double2(0.0, 0.0);
    if (lane < M) {
      double pr = 0.0, pi = 0.0;
      for (int j = 0; j < Kn; ++j) {
        const double2 e = U[j * ld + lane], e0 = U[j * ld];
        pr += e.x * e0.x + e.y * e0.y;
        pi += e.y * e0.x - e.x * e0.y;
      }
      wv = degen ? make_double2(pr, pi) : make_double2(pr * lp, pi * lp);
    }
    __syncwarp();
    if (lane < M) U[lane] = wv;
    __syncwarp();
  }
  const int npair = M * (M - 1) / 2;
  for (int it = lane; it <= npair; it += 32) {
    if (it == 0) {                                   // c_0 = trace C = sum_j w_j ||u_j||^2
      double c0 = 0.0;
      for (int j = 0; j < nv; ++j) {
        double s = 0.0;
        for (int p = 0; p < M; ++p) { const double2 x = U[j * ld + p]; s += x.x * x.x + x.y * x.y; }
        c0 += ws[warp][j] * s;
      }
      coef[coef_index(b, 0, S)] = c0;
    } else {
      int p, q;
      pair_of(it - 1, M, p, q);
      double cr = 0.0, ci = 0.0;
      for (int j = 0; j < nv; ++j) {
        const double2 x = U[j * ld + p], y = U[j * ld + q];        // u[p] conj(u[q])
        cr += ws[warp][j] * (x.x * y.x + x.y * y.y);
        ci += ws[warp][j] * (x.y * y.x - x.x * y.y);
      }
      coef[coef_index(b, 2 * it - 1, S)] = 2.0 * cr;
      coef[coef_index(b, 2 * it, S)] = -2.0 * ci;
    }
  }
  for (int j = K + lane; j < 4 * S; j += 32) coef[coef_index(b, j, S)] = 0.0;
  if (lane == 0) {
    cnt[b] = 0;
    if (info) info[b] |= flag;
  }
}

template <int M>
struct ArrShape {
  static constexpr int K = 1 + M * (M - 1);
  static constexpr int S = (K + 3) / 4;
  static constexpr int NA = (64 / S) < 1 ? 1 : ((64 / S) > 8 ? 8 : (64 / S));
  static constexpr int W = 8 * NA;             // angles per block (no halo: f is stored)
  static constexpr int NB = 2;
};
constexpr int kArrWarps = 8;
template <int M>
__global__ void __launch_bounds__(kArrWarps * 32) scan_array_kernel(const double* __restrict__ coef, int64_t B,
                                                                   int64_t per, const double* __restrict__ dpos,
                                                                   double az0, double daz, double el0, double del,
                                                                   int64_t nel, int64_t L, double* __restrict__ fbuf) {
  using Sh = ArrShape<M>;
  constexpr int K = Sh::K, S = Sh::S, NA = Sh::NA, W = Sh::W, NB = Sh::NB;
  extern __shared__ double Ta[];                                   // [NB][S][NA][32]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int q = lane & 3, r = lane >> 2;
  const int64_t col0 = (int64_t)blockIdx.x * NB * W;
  // the column's direction sines / cosines once per angle (Eq. 2), then one cospi / sinpi per entry
  __shared__ double dir[NB * W][4];                                // sin az, cos az, sin el, cos el
  for (int a = threadIdx.x; a < NB * W; a += kArrWarps * 32) {
    const int64_t pt = col0 + a;
    if (pt < L) {
      const int64_t ia = pt / nel, ie = pt - (pt / nel) * nel;
      const double az = __dadd_rn(__dmul_rn((double)ia, daz), az0);
      const double el = __dadd_rn(__dmul_rn((double)ie, del), el0);
      sincospi(az / 180.0, &dir[a][0], &dir[a][1]);
      sincospi(el / 180.0, &dir[a][2], &dir[a][3]);
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < NB * S * NA * 32; e += kArrWarps * 32) {
    const int ln = e & 31, t = (e >> 5) % NA, s = (e / (32 * NA)) % S, k = e / (32 * NA * S);
    const int a = k * W + 8 * t + (ln >> 2);
    const int64_t pt = col0 + a;
    const int j = 4 * s + (ln & 3);
    double v = j == 0 ? 1.0 : 0.0;
    if (pt < L && j > 0 && j < K) {   // z_pq = exp(j pi arg): (cos, sin) at j = (odd, even), Eq. 2
      const double saz = dir[a][0], caz = dir[a][1], sel = dir[a][2], cel = dir[a][3];
      const int pr = (j - 1) >> 1;
      const double arg = 2.0 * (dpos[3 * pr] * saz * sel + dpos[3 * pr + 1] * caz * sel + dpos[3 * pr + 2] * cel);
      v = (j & 1) ? cospi(arg) : sinpi(arg);
    }
    Ta[e] = v;
  }
  __syncthreads();
  const int64_t ngroups = (B + 7) / 8;
  const int64_t g0 = (int64_t)blockIdx.y * per;
  const int64_t g1 = (g0 + per < ngroups) ? g0 + per : ngroups;
  for (int64_t g = g0 + warp; g < g1; g += kArrWarps) {
    const double* cg = coef + ((size_t)g * S) * 32 + lane;
    const int64_t b = g * 8 + r;
    // M <= 8 (S <= 16): the group's A fragments in registers, loaded once for both blocks (e1 360x90
    // x 4096: 1.014 -> 0.982 ms per plan); larger M streams them from L1 per k-step (registers)
    constexpr bool AREG = S <= 16;
    double areg[AREG ? S : 1];
    if (AREG) {
#pragma unroll
      for (int s = 0; s < (AREG ? S : 1); ++s) areg[s] = __ldg(cg + s * 32);
    }
#pragma unroll 1
    for (int k = 0; k < NB; ++k) {
      const int64_t base = col0 + (int64_t)k * W;
      if (base >= L) break;
      const double* Tk = Ta + (size_t)k * S * NA * 32 + lane;
      double acc[NA][2];
#pragma unroll
      for (int t = 0; t < NA; ++t) { acc[t][0] = 0.0; acc[t][1] = 0.0; }
      if constexpr (AREG) {
#pragma unroll
        for (int s = 0; s < S; ++s) {
#pragma unroll
          for (int t = 0; t < NA; ++t) dmma_a(acc[t][0], acc[t][1], areg[s], Tk[(s * NA + t) * 32]);
        }
      } else {
#pragma unroll 4
        for (int s = 0; s < S; ++s) {
          const double a = __ldg(cg + s * 32);
#pragma unroll
          for (int t = 0; t < NA; ++t) dmma_a(acc[t][0], acc[t][1], a, Tk[(s * NA + t) * 32]);
        }
      }
      if (b < B) {
#pragma unroll
        for (int t = 0; t < NA; ++t)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int64_t pt = base + 8 * t + 2 * q + e;
            const double f = acc[t][e];
            if (pt < L) fbuf[(size_t)b * L + pt] = f > kFloorA ? f : kFloorA;   // NaN -> floor (Q12)
          }
      }
    }
  }
}

// 2-D findPeaks (G2) on the floored f: thread per (frame, grid point).
__global__ void peaks2d_kernel(const double* __restrict__ fbuf, int64_t B, int64_t naz, int64_t nel, int wrap,
                               int cap, int32_t* __restrict__ cnt, int32_t* __restrict__ cidx,
                               double* __restrict__ cf, float* __restrict__ P) {
  const int64_t L = naz * nel;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < B * L; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = e / L, p = e - (e / L) * L;
    const double* fb = fbuf + (size_t)b * L;
    const double fp = fb[p];
    if (P) P[e] = to_p32a(fp);
    const int64_t ia = p / nel, ie = p - (p / nel) * nel;
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
        const double fn = fb[n];
        if (n < p ? !(fp < fn) : !(fp <= fn)) peak = false;
      }
    if (peak) {
      const int slot = atomicAdd(cnt + b, 1);
      if (slot < cap) {
        cidx[(size_t)b * cap + slot] = (int32_t)p;
        cf[(size_t)b * cap + slot] = fp;
      }
    }
  }
}

// The same 2-D findPeaks on tiles: a CTA takes TA consecutive azimuth rows of one frame (all nel
// elevations) plus the two neighbouring rows (wrapped when the azimuth wraps), stages them in shared
// memory once — (TA+2) x (nel+2) values, a sentinel column on each side and sentinel halo rows
// where no neighbour exists (no wrap at the grid edge, or naz == 1, whose wrapped rows are the
// point's own row) — and tests every core point against its 8 neighbours there without branches.
// Raster order decides strictness: a neighbour that precedes the point must be strictly larger
// (fp < n), one that follows may be equal (fp <= n).  The row above precedes the point unless it is
// the wrapped last row; the row below follows it unless it is the wrapped first row; within a row
// the left neighbour precedes, the right one follows.  f is floored, so never NaN; the sentinel is
// a NaN and the tests are the unordered ones (!(fp >= n), !(fp > n)), so a missing neighbour never
// blocks a peak — the rule of peaks2d_kernel.  Same candidates (their list order may differ;
// doa_peaks sorts).  Staging: one warp per tile row (the row's source is warp-uniform), 8-byte
// asynchronous copies (LDGSTS) so a thread's loads are all in flight at once; rows shorter than a
// warp use a flat element walk.  Used when (TA+2) * (nel+2) fits the tile (nel <= kPk2MaxNel).
constexpr int kPk2Vals = 2048;       // core values per tile (TA = kPk2Vals / nel rows)
constexpr int kPk2MaxNel = 2048;
constexpr int kPkRows = 11;           // core rows per sliding-window work item
__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(src) : "memory");
}
__global__ void __launch_bounds__(256) peaks2d_tile_kernel(const double* __restrict__ fbuf, int64_t naz, int64_t nel,
                                                           int TA, int wrap, int cap, int32_t* __restrict__ cnt,
                                                           int32_t* __restrict__ cidx, double* __restrict__ cf,
                                                           float* __restrict__ P) {
  extern __shared__ double ft[];                       // [TA + 2][nel + 2]: rows ia0-1 .. ia0+TA
  const int64_t L = naz * nel;
  const int64_t b = blockIdx.y;
  const int nazI = (int)naz, nelI = (int)nel, W = nelI + 2;
  const int ia0 = (int)blockIdx.x * TA;
  const int nr = ia0 + TA <= nazI ? TA : nazI - ia0;   // core rows of this tile
  const double* fb = fbuf + (size_t)b * L;
  const double kSent = __longlong_as_double(0x7FF8000000000000LL);   // quiet NaN
  auto src_row = [&](int r) {                          // source row of tile row r (-1: sentinel row)
    const int ja = ia0 - 1 + r;
    if (ja >= 0 && ja < nazI) return ja;
    if (!wrap || nazI == 1) return -1;
    return ja < 0 ? nazI - 1 : 0;
  };
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  if (nelI >= 32) {
    for (int r = warp; r < nr + 2; r += nwarps) {
      const int ja = src_row(r);
      double* dst = ft + r * W;
      if (lane == 0) { dst[0] = kSent; dst[nelI + 1] = kSent; }
      if (ja < 0) {
        for (int c = lane; c < nelI; c += 32) dst[1 + c] = kSent;
      } else {
        const double* src = fb + (size_t)ja * nelI;
        for (int c = lane; c < nelI; c += 32) cp_async8(dst + 1 + c, src + c);
      }
    }
  } else {
    const int nvals = (nr + 2) * W;
    const int sr = (int)(blockDim.x / W), se = (int)(blockDim.x - sr * W);
    int r = (int)(threadIdx.x / W), c = (int)(threadIdx.x - r * W);
    for (int e = threadIdx.x; e < nvals; e += blockDim.x, r += sr, c += se) {
      if (c >= W) { c -= W; ++r; }
      const int ja = src_row(r);
      if (ja < 0 || c == 0 || c > nelI) ft[e] = kSent;
      else cp_async8(ft + e, fb + (size_t)ja * nelI + (c - 1));
    }
  }
  asm volatile("cp.async.wait_all;\n" ::: "memory");
  __syncthreads();
  // Tests: work item = (chunk of kPkRows core rows, elevation column); a thread slides a 3 x 3
  // window down its column, so each point costs 3 shared loads instead of 9 (the tile is bound by
  // shared-memory bandwidth), and consecutive lanes take consecutive columns (conflict-free).
  const int nchunks = (nr + kPkRows - 1) / kPkRows;
  const int items = nchunks * nelI;
  const int sc = (int)(blockDim.x / nelI), se = (int)(blockDim.x - sc * nelI);
  int ch = (int)(threadIdx.x / nelI), ie = (int)(threadIdx.x - ch * nelI);
  for (int it = threadIdx.x; it < items; it += blockDim.x, ch += sc, ie += se) {
    if (ie >= nelI) { ie -= nelI; ++ch; }
    const int r0 = ch * kPkRows;                         // first core row of the chunk
    const double* col = ft + r0 * W + ie;                // tile row r0 = the row above core row r0
    double a0 = col[0], a1 = col[1], a2 = col[2];
    double b0 = col[W], b1 = col[W + 1], b2 = col[W + 2];
#pragma unroll
    for (int k = 0; k < kPkRows; ++k) {
      if (r0 + k >= nr) break;
      const double* cr = col + (k + 2) * W;
      const double c0 = cr[0], c1 = cr[1], c2 = cr[2];
      const int ia = ia0 + r0 + k;
      const double fp = b1;
      // unordered tests (ltu: fp < n, leu: fp <= n; both true for the NaN sentinel)
      bool peak;
      if (ia != 0 && ia != nazI - 1) {                   // interior row: above precedes, below follows
        unsigned pk;
        asm("{\n\t.reg .pred p;\n\t"
            "setp.ltu.f64 p, %1, %2;\n\t"
            "setp.ltu.and.f64 p, %1, %3, p;\n\t"
            "setp.ltu.and.f64 p, %1, %4, p;\n\t"
            "setp.ltu.and.f64 p, %1, %5, p;\n\t"
            "setp.leu.and.f64 p, %1, %6, p;\n\t"
            "setp.leu.and.f64 p, %1, %7, p;\n\t"
            "setp.leu.and.f64 p, %1, %8, p;\n\t"
            "setp.leu.and.f64 p, %1, %9, p;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(pk)
            : "d"(fp), "d"(a0), "d"(a1), "d"(a2), "d"(b0), "d"(b2), "d"(c0), "d"(c1), "d"(c2));
        peak = pk != 0;
      } else {                                           // first / last row: wrapped neighbours' order
        const bool upf = ia == 0, dnf = ia != nazI - 1;  // row above follows p / row below follows p
        const bool pu = upf ? (!(fp > a0) & !(fp > a1) & !(fp > a2)) : (!(fp >= a0) & !(fp >= a1) & !(fp >= a2));
        const bool pd = dnf ? (!(fp > c0) & !(fp > c1) & !(fp > c2)) : (!(fp >= c0) & !(fp >= c1) & !(fp >= c2));
        peak = pu & pd & !(fp >= b0) & !(fp > b2);
      }
      const int64_t pidx = (int64_t)ia * nel + ie;
      if (P) P[(size_t)b * L + pidx] = to_p32a(fp);
      if (peak) {
        const int slot = atomicAdd(cnt + b, 1);
        if (slot < cap) {
          cidx[(size_t)b * cap + slot] = (int32_t)pidx;
          cf[(size_t)b * cap + slot] = fp;
        }
      }
      a0 = b0; a1 = b1; a2 = b2;
      b0 = c0; b1 = c1; b2 = c2;
    }
  }
}

template <int M>
cudaError_t launch_scan_array_t(const doa_plan_s* p, int64_t B, cudaStream_t s) {
  using Sh = ArrShape<M>;
  const size_t smem = (size_t)Sh::NB * Sh::S * Sh::NA * 32 * sizeof(double);
  kernel_occupancy(scan_array_kernel<M>, kArrWarps * 32, smem);     // sets the smem attribute on this device
  const int64_t cols = (p->L + Sh::NB * Sh::W - 1) / (Sh::NB * Sh::W);
  const int64_t ngroups = (B + 7) / 8;
  int64_t per = (cols * ngroups) / ((int64_t)sm_count() * 8);
  if (per < 8) per = 8;
  if (per > ngroups) per = ngroups;
  const int64_t gy = (ngroups + per - 1) / per;
  count_launch();
  scan_array_kernel<M><<<dim3((unsigned)cols, (unsigned)gy), kArrWarps * 32, smem, s>>>(
      p->coef, B, per, p->dpos, p->az0, p->daz, p->el0, p->del, p->nel, p->L, p->fbuf);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_array_spectrum(const doa_plan_s* p, const double* lam, const double* V, int64_t B, float* P,
                                  int32_t* info, cudaStream_t s) {
  count_launch();
  coef_array_kernel<<<(unsigned)((B + 3) / 4), 128, 0, s>>>(lam, reinterpret_cast<const double2*>(V), B, p->M,
                                                             p->D, p->alg, p->coef, p->cnt, info);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  switch (p->M) {
#define DOA_ARR_CASE(m) case m: e = launch_scan_array_t<m>(p, B, s); break;
    DOA_ARR_CASE(2) DOA_ARR_CASE(3) DOA_ARR_CASE(4) DOA_ARR_CASE(5) DOA_ARR_CASE(6) DOA_ARR_CASE(7)
    DOA_ARR_CASE(8) DOA_ARR_CASE(9) DOA_ARR_CASE(10) DOA_ARR_CASE(11) DOA_ARR_CASE(12) DOA_ARR_CASE(13)
    DOA_ARR_CASE(14) DOA_ARR_CASE(15) DOA_ARR_CASE(16)
#undef DOA_ARR_CASE
    default: return cudaErrorInvalidValue;
  }
  if (e != cudaSuccess) return e;
  count_launch();
  if (p->nel <= kPk2MaxNel && B < 65536) {
    const int TA = (int)(kPk2Vals / p->nel < 1 ? 1 : kPk2Vals / p->nel);
    const size_t smem = (size_t)(TA + 2) * (p->nel + 2) * sizeof(double);
    kernel_occupancy(peaks2d_tile_kernel, 256, smem);                  // sets the smem attribute (> 48 KB)
    const dim3 grid((unsigned)((p->naz + TA - 1) / TA), (unsigned)B);
    peaks2d_tile_kernel<<<grid, 256, smem, s>>>(p->fbuf, p->naz, p->nel, TA, p->wrap, p->cap, p->cnt, p->cand_idx,
                                                p->cand_f, P);
    return cudaGetLastError();
  }
  const int64_t tot = B * p->L;
  int blocks = (int)((tot + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  peaks2d_kernel<<<blocks, 256, 0, s>>>(p->fbuf, B, p->naz, p->nel, p->wrap, p->cap, p->cnt, p->cand_idx,
                                        p->cand_f, P);
  return cudaGetLastError();
}

}  // namespace doa
