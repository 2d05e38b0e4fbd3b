// NEXT-3: on-device synthetic snapshots of the signal model Eq. 1,
// X = A(theta) S + W for a ULA, so a streaming workload needs no host->device transfer of X.
//
// Counter-based randomness (Philox4x32-10, Salmon et al. SC'11): one call per (frame, snapshot
// n, pair index c) with counter (c, n, frame_lo, frame_hi) and key (seed_lo, seed_hi) gives four
// 32-bit words = two Box-Muller pairs = two CN(0,1) samples: sample k of a snapshot (k < D: source
// k, else noise of element k - D) uses call c = k/2, words (2(k%2), 2(k%2)+1).  Box-Muller in
// fp64: u = (word + 0.5) 2^-32, r = sqrt(-2 ln u1), z = r (cos 2 pi u2 + j sin 2 pi u2), CN(0,1) =
// z / sqrt(2).  Sources unit power, noise sigma^2 = 10^(-SNR/10) (Q13, Q14); steering
// a_m = exp(-j pi m u), u = 2 (d/lambda) sin theta (Q6); X formed in fp64, rounded once to
// complex64, stored X[b][n][m].  synth/philox.py implements the same generator in numpy; the
// GPU test compares the two element by element.  Input generation only — none of the estimator's
// arithmetic is here.
#include <cmath>

#include "doa_internal.cuh"

namespace doa {
namespace {

struct Philox4 {
  uint32_t x[4];
};

__device__ __forceinline__ Philox4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0,
                                                 uint32_t k1) {
  constexpr uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(M0, c0), lo0 = M0 * c0;
    const uint32_t hi1 = __umulhi(M1, c2), lo1 = M1 * c2;
    const uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    k0 += W0; k1 += W1;
  }
  Philox4 o;
  o.x[0] = c0; o.x[1] = c1; o.x[2] = c2; o.x[3] = c3;
  return o;
}

__device__ __forceinline__ double2 cnormal(uint32_t a, uint32_t b) {
  const double u1 = ((double)a + 0.5) * 0x1p-32, u2 = ((double)b + 0.5) * 0x1p-32;
  const double r = sqrt(-2.0 * log(u1)) * 0.70710678118654752440;   // / sqrt(2): E|z|^2 = 1
  double sn, cs;
  sincospi(2.0 * u2, &sn, &cs);
  return make_double2(r * cs, r * sn);
}

constexpr int kMaxGenD = 63;
constexpr int kGenThreads = 256;

// CTA = (frame, chunk of 256 snapshots), thread = snapshot.  The frame's steering matrix
// a[m][d] = exp(-j pi m u_d) is formed once per CTA in shared memory; each thread draws its D
// source samples (registers for D <= DT), then per element m its noise sample and the mix.
template <int DT>
__global__ void __launch_bounds__(kGenThreads) generate_kernel(int M, double dl, int D, const double* __restrict__ theta,
                                                               int per_frame, double sigma, uint32_t k0, uint32_t k1,
                                                               int64_t frame0, int64_t N, float2* __restrict__ X) {
  extern __shared__ double2 steer[];                    // [M][D]
  const int64_t b = blockIdx.x;                         // frames on x (up to 2^31 - 1)
  const int64_t n = (int64_t)blockIdx.y * kGenThreads + threadIdx.x;
  const double* th = theta + (per_frame ? b * D : 0);
  for (int e = threadIdx.x; e < M * D; e += kGenThreads) {
    const int m = e / D, d = e - (e / D) * D;
    const double u = 2.0 * dl * sinpi(th[d] / 180.0);
    double sn, cs;
    sincospi((double)m * u, &sn, &cs);                  // a_m = cos(pi m u) - j sin(pi m u)
    steer[e] = make_double2(cs, -sn);
  }
  __syncthreads();
  if (n >= N) return;
  const uint64_t f = (uint64_t)(frame0 + b);
  const uint32_t c2 = (uint32_t)f, c3 = (uint32_t)(f >> 32), c1 = (uint32_t)n;
  constexpr int DS = DT > 0 ? DT : kMaxGenD;
  double2 s[DS];
#pragma unroll
  for (int d = 0; d < DS; ++d) {
    if (d >= D) break;
    const Philox4 w = philox4x32_10((uint32_t)(d >> 1), c1, c2, c3, k0, k1);
    s[d] = (d & 1) ? cnormal(w.x[2], w.x[3]) : cnormal(w.x[0], w.x[1]);
  }
  float2* xo = X + ((size_t)b * N + n) * M;
  for (int m = 0; m < M; ++m) {
    const int k = D + m;
    const Philox4 w = philox4x32_10((uint32_t)(k >> 1), c1, c2, c3, k0, k1);
    const double2 z = (k & 1) ? cnormal(w.x[2], w.x[3]) : cnormal(w.x[0], w.x[1]);
    double xr = sigma * z.x, xi = sigma * z.y;
    const double2* am = steer + m * D;
#pragma unroll
    for (int d = 0; d < DS; ++d) {
      if (d >= D) break;
      const double2 a = am[d];
      xr += a.x * s[d].x - a.y * s[d].y;
      xi += a.x * s[d].y + a.y * s[d].x;
    }
    xo[m] = make_float2((float)xr, (float)xi);
  }
}

}  // namespace

cudaError_t launch_generate(int M, double dl, int D, const double* theta, int per_frame, double snr_db,
                            uint64_t seed, int64_t frame0, int64_t B, int64_t N, float* X, cudaStream_t s) {
  count_launch();
  const double sigma = std::sqrt(std::pow(10.0, -snr_db / 10.0));
  const dim3 grid((unsigned)B, (unsigned)((N + kGenThreads - 1) / kGenThreads));
  const size_t smem = (size_t)M * D * sizeof(double2);
  auto go = [&](auto kern) {
    kernel_occupancy(kern, kGenThreads, smem);          // sets the smem attribute on this device
    kern<<<grid, kGenThreads, smem, s>>>(M, dl, D, theta, per_frame, sigma, (uint32_t)seed, (uint32_t)(seed >> 32),
                                        frame0, N, reinterpret_cast<float2*>(X));
  };
  if (D <= 4) go(generate_kernel<4>);
  else if (D <= 8) go(generate_kernel<8>);
  else go(generate_kernel<0>);
  return cudaGetLastError();
}

}  // namespace doa
