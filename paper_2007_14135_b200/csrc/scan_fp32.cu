// the FP32-pipe direct-form scan, selected per plan with
// doa_plan_set_engine(plan, DOA_ENGINE_DIRECT_FP32): north_star's "otherwise FP32-pipe sincos+FMA"
// engine behind the same ABI as the product's fp64 Toeplitz contraction (DMMA), so the two can be
// A/B'd on identical inputs (tests/test_gpu_fp32_engine.py, profiles/ncu_scan_f32_*).
//
// Step-5 (Table 2) in the paper's own per-angle form, one angle per thread as in §4.3
// (P:132), with the noise-subspace products of Table 3 kept as vectors:
//     f(theta) = sum_j | x_j^H a(theta) |^2,   x_j = sqrt(w_j) u_j,
//   PHD: x_0 = e_min;  MUSIC: x_j = e_j (j < K = M - D);  EV: x_j = e_j / sqrt(lambda_j) (Q1, G1 clamp);
//   MN: x_0 = P_n e1 / (e1^H P_n e1) (Q5, G1),
// i.e. a^H C a for C = sum_j x_j x_j^H.  The vectors are formed in fp64 from the eigenpairs and
// rounded once to complex64; the steering a_m = exp(-j pi m u) (Q6) is evaluated with fp64 sincospi
// and rounded to fp32; every product and sum of the scan runs on the FP32 pipe (4 M K FFMA per
// (frame, angle) against the Toeplitz form's 2(M-1) DMMA flops).  f is then floored (Q12) and
// peak-tested (Q9/Q10) in fp64 exactly like the other scans, so doa_peaks is shared.  M <= 16.
#include <cfloat>

#include "doa_internal.cuh"

namespace doa {
namespace {

constexpr int kF32Warps = 4;
constexpr int kF32Vecs = 192;      // frames x vectors staged per CTA (24 KB at M = 16): 16 frames of
                                   // MUSIC/EV (K = 12), 192 of PHD/MN, so the steering setup amortises
constexpr int kF32Win = 64;        // tile positions per warp window (62 decided)

// S3 for the fp32 engine: one warp per frame writes the nv weighted vectors x_j (complex64,
// [B][K][M], K = M - D slots per frame, nv = K for MUSIC/EV, 1 for PHD/MN), zeroes the candidate
// counter and ORs DEGENERATE into info.
__global__ void __launch_bounds__(128) vec32_kernel(const double* __restrict__ lam, const double2* __restrict__ V,
                                                    int64_t B, int M, int D, int alg, float2* __restrict__ X,
                                                    int32_t* __restrict__ cnt, int32_t* __restrict__ info) {
  const int lane = threadIdx.x & 31;
  const int64_t b = (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
  if (b >= B) return;
  const int K = M - D;
  const double* lb = lam + (size_t)b * M;
  const double2* Vb = V + (size_t)b * M * M;
  float2* Xb = X + (size_t)b * K * M;
  int flag = 0;
  if (alg == DOA_ALG_MN) {
    // w = P_n e1 / (e1^H P_n e1): lane p sums V[p][j] conj(V[0][j]) over j < K in ascending j
    double p0 = 0.0, wr = 0.0, wi = 0.0;
    for (int j = 0; j < K; ++j) {
      const double2 v0 = Vb[j];
      p0 = fma(v0.x, v0.x, fma(v0.y, v0.y, p0));
      if (lane < M) {
        const double2 vp = Vb[(size_t)lane * M + j];
        wr = fma(vp.x, v0.x, fma(vp.y, v0.y, wr));
        wi = fma(vp.y, v0.x, fma(-vp.x, v0.y, wi));
      }
    }
    const bool degen = !(p0 > 100.0 * DBL_EPSILON);
    if (degen) flag = DOA_INFO_DEGENERATE;
    const double lp = degen ? 1.0 : 1.0 / p0;
    if (lane < M) Xb[lane] = make_float2((float)(wr * lp), (float)(wi * lp));
  } else {
    const int nv = alg == DOA_ALG_PHD ? 1 : K;
    const double lfloor = 100.0 * DBL_EPSILON * fmax(lb[M - 1], 0.0);
    for (int e = lane; e < nv * M; e += 32) {
      const int j = e / M, m = e - (e / M) * M;
      double sw = 1.0;
      if (alg == DOA_ALG_EV) {
        const double lj = lb[j];
        sw = lj <= lfloor ? (lfloor > 0.0 ? rsqrt(lfloor) : 1.0) : rsqrt(lj);
      }
      const double2 v = Vb[(size_t)m * M + j];
      Xb[(size_t)j * M + m] = make_float2((float)(sw * v.x), (float)(sw * v.y));
    }
    if (alg == DOA_ALG_EV) {
      bool deg = false;
      for (int j = lane; j < K; j += 32) deg |= lb[j] <= lfloor;
      if (__any_sync(0xffffffffu, deg)) flag = DOA_INFO_DEGENERATE;
    }
  }
  if (lane == 0) {
    cnt[b] = 0;
    if (info && flag) info[b] |= flag;
  }
}

// The scan.  Grid x: groups of warp windows (grid-stride), y: chunks of kF32Frames frames whose
// vectors are staged in shared memory (every lane reads the same x_jm: broadcast).  Each lane keeps
// the fp32 steering of its two angles in registers and loops over the chunk's frames.
template <int MT>
__global__ void __launch_bounds__(kF32Warps * 32, 3) scan_f32_kernel(const float2* __restrict__ X, int64_t B, int K,
                                                                  int nv, int M, double dl, double theta0,
                                                                  double dtheta, int L, bool sym, int cap,
                                                                  int32_t* __restrict__ cnt,
                                                                  int32_t* __restrict__ cidx, double* __restrict__ cf,
                                                                  float* __restrict__ P, int fpc) {
  extern __shared__ float4 xs4[];                          // [f][j][MT/2] pairs of complex64
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t b0 = (int64_t)blockIdx.y * fpc;
  const int nb = (int)(B - b0 < fpc ? B - b0 : fpc);
  float2* xs = reinterpret_cast<float2*>(xs4);
  for (int e = threadIdx.x; e < nb * nv * MT; e += kF32Warps * 32) {
    const int f = e / (nv * MT), r = e - f * (nv * MT), j = r / MT, m = r - (r / MT) * MT;
    xs[e] = m < M ? X[((size_t)(b0 + f) * K + j) * M + m] : make_float2(0.f, 0.f);
  }
  __syncthreads();
  const int nwin = (L + (kF32Win - 2) - 1) / (kF32Win - 2);
  for (int w = blockIdx.x * kF32Warps + warp; w < nwin; w += gridDim.x * kF32Warps) {
    const int base = w * (kF32Win - 2) - 1;
    float2 a0[MT], a1[MT];                                  // a_m = exp(-j pi m u) = (cos, -sin)
    {
      int i0 = base + 2 * lane, i1 = i0 + 1;
      i0 = i0 < 0 ? 0 : (i0 >= L ? L - 1 : i0);
      i1 = i1 < 0 ? 0 : (i1 >= L ? L - 1 : i1);
      const double u0 = grid_u(i0, theta0, dtheta, dl, L, sym), u1 = grid_u(i1, theta0, dtheta, dl, L, sym);
#pragma unroll
      for (int m = 0; m < MT; ++m) {
        double s, c;
        sincospi((double)m * u0, &s, &c);
        a0[m] = make_float2((float)c, (float)-s);
        sincospi((double)m * u1, &s, &c);
        a1[m] = make_float2((float)c, (float)-s);
      }
    }
    for (int f = 0; f < nb; ++f) {
      const float4* xf = xs4 + (size_t)f * nv * (MT / 2);
      float acc0 = 0.f, acc1 = 0.f;
      for (int j = 0; j < nv; ++j) {
        float pr0 = 0.f, pi0 = 0.f, pr1 = 0.f, pi1 = 0.f;
#pragma unroll
        for (int h = 0; h < MT / 2; ++h) {                   // conj(x_m) a_m for m = 2h, 2h+1
          const float4 x = xf[j * (MT / 2) + h];
          const float2 p0 = a0[2 * h], q0 = a0[2 * h + 1], p1 = a1[2 * h], q1 = a1[2 * h + 1];
          pr0 = fmaf(x.x, p0.x, fmaf(x.y, p0.y, pr0));
          pi0 = fmaf(x.x, p0.y, fmaf(-x.y, p0.x, pi0));
          pr1 = fmaf(x.x, p1.x, fmaf(x.y, p1.y, pr1));
          pi1 = fmaf(x.x, p1.y, fmaf(-x.y, p1.x, pi1));
          pr0 = fmaf(x.z, q0.x, fmaf(x.w, q0.y, pr0));
          pi0 = fmaf(x.z, q0.y, fmaf(-x.w, q0.x, pi0));
          pr1 = fmaf(x.z, q1.x, fmaf(x.w, q1.y, pr1));
          pi1 = fmaf(x.z, q1.y, fmaf(-x.w, q1.x, pi1));
        }
        acc0 = fmaf(pr0, pr0, fmaf(pi0, pi0, acc0));
        acc1 = fmaf(pr1, pr1, fmaf(pi1, pi1, acc1));
      }
      const int64_t b = b0 + f;
      const long long v0 = floor_bits(__double_as_longlong((double)acc0));
      const long long v1 = floor_bits(__double_as_longlong((double)acc1));
      window_peaks<false>(v0, v1, lane, base, 1, L - 2, L, cap, cnt + b, cidx + (size_t)b * cap, cf + (size_t)b * cap);
      if (P) window_P<false>(v0, v1, lane, base, L - 1, L, P + (size_t)b * L);
    }
  }
}

}  // namespace

cudaError_t launch_vec32(const doa_plan_s* p, const double* lam, const double* V, int64_t B, int32_t* info,
                         cudaStream_t s) {
  if (B <= 0) return cudaSuccess;
  count_launch();
  vec32_kernel<<<(unsigned)((B + 3) / 4), 128, 0, s>>>(lam, reinterpret_cast<const double2*>(V), B, p->M, p->D, p->alg,
                                                       reinterpret_cast<float2*>(p->x32), p->cnt, info);
  return cudaGetLastError();
}

cudaError_t launch_scan_f32(const doa_plan_s* p, int64_t B, float* P, cudaStream_t s) {
  if (B <= 0) return cudaSuccess;
  const int K = p->M - p->D;
  const int nv = (p->alg == DOA_ALG_MUSIC || p->alg == DOA_ALG_EV) ? K : 1;
  const int MT = p->M <= 8 ? 8 : 16;
  const int fpc = kF32Vecs / nv > 0 ? kF32Vecs / nv : 1;
  const size_t smem = (size_t)fpc * nv * MT * sizeof(float2);
  const int64_t nwin = (p->L + (kF32Win - 2) - 1) / (kF32Win - 2);
  const int64_t gx = (nwin + kF32Warps - 1) / kF32Warps;
  const dim3 grid((unsigned)gx, (unsigned)((B + fpc - 1) / fpc));
  const float2* X = reinterpret_cast<const float2*>(p->x32);
  count_launch();
  if (MT == 8)
    scan_f32_kernel<8><<<grid, kF32Warps * 32, smem, s>>>(X, B, K, nv, p->M, p->dl, p->theta0, p->dtheta, (int)p->L,
                                                          p->sym != 0, p->cap, p->cnt, p->cand_idx, p->cand_f, P, fpc);
  else
    scan_f32_kernel<16><<<grid, kF32Warps * 32, smem, s>>>(X, B, K, nv, p->M, p->dl, p->theta0, p->dtheta, (int)p->L,
                                                           p->sym != 0, p->cap, p->cnt, p->cand_idx, p->cand_f, P, fpc);
  return cudaGetLastError();
}

}  // namespace doa
