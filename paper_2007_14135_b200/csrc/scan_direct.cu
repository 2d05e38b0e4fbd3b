// S4-S6 for small batches: the direct (non-tensor-core) scan — north_star's "otherwise" branch of
// "the grid scan as an E_n^H A(theta) contraction on tensor cores only when batch x grid makes it
// genuinely dense".  With a handful of frames the DMMA contraction of spectrum.cu has at most one
// real row in its 8-row A fragments and spends most of its time building a per-CTA steering table
// (2(M-1) sincospi per angle); here the steering is generated once per angle in registers and
// shared by every (plan, frame) combination of the launch — e.g. all four estimators of a frame.
//
// Per angle (Table 2 Step-5; Toeplitz form of DESIGN.md §5, fp64 on the FP64 pipe):
//   f = c_0 + sum_{k=1}^{M-1} (2 Re c_k) cos(k psi) + (2 Im c_k) sin(k psi),  psi = pi u,
// with e^{j k psi} from e^{j psi} = (cospi(u), sinpi(u)) by the recurrence w_k = w_{k-1} w_1,
// refreshed with the exact sincospi(k u) at every k = 0 mod 8 (error <= ~8 ulp of the steering;
// the Q18 tie bound allows 10 M ulp of sum |c_k|).  On symmetric grids (Q26) a lane's angle pair
// (i, L-1-i) shares the steering (u_{L-1-i} = -u_i exactly): f_i = E + O, f_{L-1-i} = E - O.
//
// Layout: a warp owns a window of 64 consecutive tile positions, two per lane (lane l: positions
// 2l, 2l+1), windows advance by 62 so that every interior angle is decided exactly once; the peak
// test (Q9/Q10 on floored f, integer domain as in the DMMA epilogue) needs one shuffle per side.
// Candidates go to each plan's lists exactly as in the DMMA scan, so doa_peaks is shared.
#include "doa_internal.cuh"

namespace doa {
namespace {

constexpr int kDirWarps = 4;
constexpr int kDirCombos = 4;         // (plan, frame) combinations per CTA (grid y = chunks of them)
constexpr int kDirWin = 64;           // tile positions per warp window (62 decided)

__device__ __forceinline__ double2 cmul_d(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 wexact(int k, double u) {    // e^{j k pi u}, exact multiple k u
  double s, c;
  sincospi((double)k * u, &s, &c);
  return make_double2(c, s);
}

template <bool MIRROR>
__global__ void __launch_bounds__(kDirWarps * 32) scan_direct_kernel(DirectScanArgs a, int64_t B, int M, double dl,
                                                                     double theta0, double dtheta, int L, bool sym,
                                                                     int cap) {
  extern __shared__ double2 dcs[];    // [kDirCombos][M]: (c_0, 0) at k = 0, (2 Re c_k, 2 Im c_k) at k >= 1
  const int S = ksteps(M);
  const int64_t ncomb = (int64_t)a.nplans * B;
  const int64_t cbase = (int64_t)blockIdx.y * kDirCombos;
  const int nc = (int)(ncomb - cbase < kDirCombos ? ncomb - cbase : kDirCombos);
  for (int e = threadIdx.x; e < kDirCombos * M; e += blockDim.x) {
    const int c = e / M, k = e - (e / M) * M;
    double2 v = make_double2(0.0, 0.0);
    if (c < nc) {
      const int64_t comb = cbase + c;
      const int p = (int)(comb / B);
      const int64_t b = comb - (int64_t)p * B;
      const double* cf = a.coef[p];
      v = k == 0 ? make_double2(cf[coef_index(b, 0, S)], 0.0)
                 : make_double2(cf[coef_index(b, coef_cos(k), S)], cf[coef_index(b, coef_sin(M, k), S)]);
    }
    dcs[e] = v;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int H = (L + 1) / 2;
  const int Lt = MIRROR ? H + 1 : L;                  // computed tile positions [0, Lt)
  const int span = MIRROR ? H : L;                    // positions owned by the windows
  const int nwin = (span + (kDirWin - 2) - 1) / (kDirWin - 2);
  for (int w = blockIdx.x * kDirWarps + warp; w < nwin; w += gridDim.x * kDirWarps) {
    const int base = w * (kDirWin - 2) - 1;
    double u[2];
    double2 w1[2], wk[2];
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      int i = base + 2 * lane + s;
      i = i < 0 ? 0 : (i >= Lt ? Lt - 1 : i);
      u[s] = grid_u(i, theta0, dtheta, dl, L, sym);
      w1[s] = wexact(1, u[s]);
      wk[s] = w1[s];
    }
    double E[kDirCombos][2], O[kDirCombos][2];
#pragma unroll
    for (int c = 0; c < kDirCombos; ++c) {
      const double c0 = dcs[c * M].x;
      E[c][0] = E[c][1] = c0;
      O[c][0] = O[c][1] = 0.0;
    }
    for (int k = 1; k < M; ++k) {
      if (k > 1) {
#pragma unroll
        for (int s = 0; s < 2; ++s) wk[s] = (k & 7) == 0 ? wexact(k, u[s]) : cmul_d(wk[s], w1[s]);
      }
#pragma unroll
      for (int c = 0; c < kDirCombos; ++c) {
        const double2 cc = dcs[c * M + k];
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          E[c][s] = fma(cc.x, wk[s].x, E[c][s]);
          O[c][s] = fma(cc.y, wk[s].y, O[c][s]);
        }
      }
    }
#pragma unroll
    for (int c = 0; c < kDirCombos; ++c) {
      if (c >= nc) break;                              // CTA-uniform
      const int64_t comb = cbase + c;
      const int p = (int)(comb / B);
      const int64_t b = comb - (int64_t)p * B;
      int32_t* cnt = a.cnt[p] + b;
      int32_t* cidx = a.cidx[p] + (size_t)b * cap;
      double* cfv = a.cf[p] + (size_t)b * cap;
      float* P = a.P[p] ? a.P[p] + (size_t)b * L : nullptr;
      const long long lo0 = floor_bits(__double_as_longlong(E[c][0] + O[c][0]));
      const long long lo1 = floor_bits(__double_as_longlong(E[c][1] + O[c][1]));
      if (!MIRROR) {
        window_peaks<false>(lo0, lo1, lane, base, 1, L - 2, L, cap, cnt, cidx, cfv);
        if (P) window_P<false>(lo0, lo1, lane, base, L - 1, L, P);
      } else {
        const long long hi0 = floor_bits(__double_as_longlong(E[c][0] - O[c][0]));
        const long long hi1 = floor_bits(__double_as_longlong(E[c][1] - O[c][1]));
        window_peaks<false>(lo0, lo1, lane, base, 1, H - 1, L, cap, cnt, cidx, cfv);
        window_peaks<true>(hi0, hi1, lane, base, 1, L - 1 - H, L, cap, cnt, cidx, cfv);
        if (P) {
          window_P<false>(lo0, lo1, lane, base, H - 1, L, P);
          window_P<true>(hi0, hi1, lane, base, L - 1 - H, L, P);
        }
      }
    }
  }
}

}  // namespace

cudaError_t launch_scan_direct(const DirectScanArgs& args, const doa_plan_s* p, int64_t B, cudaStream_t s) {
  if (B <= 0 || args.nplans <= 0) return cudaSuccess;
  const int64_t ncomb = (int64_t)args.nplans * B;
  const int64_t chunks = (ncomb + kDirCombos - 1) / kDirCombos;
  const int64_t span = p->mirror ? (p->L + 1) / 2 : p->L;
  const int64_t nwin = (span + (kDirWin - 2) - 1) / (kDirWin - 2);
  int64_t gx = (nwin + kDirWarps - 1) / kDirWarps;
  const int64_t cap_x = (int64_t)sm_count() * 8;     // grid-stride beyond ~8 CTAs per SM
  if (gx > cap_x) gx = cap_x;
  const size_t smem = (size_t)kDirCombos * p->M * sizeof(double2);
  const dim3 grid((unsigned)gx, (unsigned)chunks);
  count_launch();
  if (p->mirror)
    scan_direct_kernel<true><<<grid, kDirWarps * 32, smem, s>>>(args, B, p->M, p->dl, p->theta0, p->dtheta,
                                                                (int)p->L, p->sym != 0, p->cap);
  else
    scan_direct_kernel<false><<<grid, kDirWarps * 32, smem, s>>>(args, B, p->M, p->dl, p->theta0, p->dtheta,
                                                                 (int)p->L, p->sym != 0, p->cap);
  return cudaGetLastError();
}

}  // namespace doa
