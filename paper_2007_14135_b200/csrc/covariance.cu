// S1 — sample covariance R = (1/N) X X^H  (Eq. 3; Table 2 Step-1).
//
// One CTA per frame.  Snapshots are streamed through shared memory in chunks and converted
// fp32 -> fp64 once on the way in (conversions run at 1/4 of the DFMA rate on B200, so each
// element is converted once per frame, not once per use).  Each thread owns a 2x2 register
// block (bi <= bj) of the upper block-triangle and a snapshot slice; fp32 products are exact in
// fp64, sums are fp64 in a fixed order (slice-strided, then a fixed-order slice reduction), so
// the result is deterministic.  The lower triangle is written as the exact conjugate mirror.
#include "doa_internal.cuh"

namespace doa {
namespace {

constexpr int kCovThreads = 256;
constexpr int kChunkDoubles2 = 2048;   // snapshots*M complex doubles staged per chunk (32 KiB)

__global__ void __launch_bounds__(kCovThreads) covariance_kernel(const float2* __restrict__ X, int64_t N, int M,
                                                                 double2* __restrict__ R) {
  extern __shared__ double2 sm[];
  const int Mp = (M + 1) & ~1;                     // padded to even
  const int nb = Mp / 2;                           // 2-blocks per side
  const int nblk = nb * (nb + 1) / 2;              // upper block triangle
  const int nslice = max(1, kCovThreads / nblk);
  const int chunk = max(1, kChunkDoubles2 / Mp);   // snapshots per chunk
  double2* xs = sm;                                // [chunk][Mp]
  double2* red = sm + (size_t)chunk * Mp;          // [nslice][nblk][4]
  const int64_t b = blockIdx.x;
  const float2* Xb = X + (size_t)b * N * M;
  const int tid = threadIdx.x;

  // this thread's (block, slice) assignments: blk = tid % nblk ... strided over nblk*nslice
  double acc[4][4][2];                              // up to 4 blocks per thread (M=64: 528 blocks/256 thr)
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int e = 0; e < 4; ++e) acc[q][e][0] = acc[q][e][1] = 0.0;

  for (int64_t n0 = 0; n0 < N; n0 += chunk) {
    const int cn = (int)((N - n0) < chunk ? (N - n0) : chunk);
    __syncthreads();
    for (int e = tid; e < cn * Mp; e += kCovThreads) {
      const int n = e / Mp, m = e - n * Mp;
      double2 v = make_double2(0.0, 0.0);
      if (m < M) {
        const float2 x = Xb[(size_t)(n0 + n) * M + m];
        v = make_double2((double)x.x, (double)x.y);
      }
      xs[e] = v;
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int w = tid + q * kCovThreads;
      if (w < nblk * nslice) {
      const int blk = w % nblk, sl = w / nblk;
      // decode blk -> (bi, bj), bi <= bj, row-major over the upper block triangle
      int bi = 0, rem = blk;
      while (rem >= nb - bi) { rem -= nb - bi; ++bi; }
      const int bj = bi + rem;
      for (int n = sl; n < cn; n += nslice) {
        const double2* xr = xs + (size_t)n * Mp;
        const double2 a0 = xr[2 * bi], a1 = xr[2 * bi + 1];
        const double2 c0 = xr[2 * bj], c1 = xr[2 * bj + 1];
        // x_i conj(x_j) = (ar br + ai bi) + j (ai br - ar bi)
        acc[q][0][0] = fma(a0.x, c0.x, fma(a0.y, c0.y, acc[q][0][0]));
        acc[q][0][1] = fma(a0.y, c0.x, fma(-a0.x, c0.y, acc[q][0][1]));
        acc[q][1][0] = fma(a0.x, c1.x, fma(a0.y, c1.y, acc[q][1][0]));
        acc[q][1][1] = fma(a0.y, c1.x, fma(-a0.x, c1.y, acc[q][1][1]));
        acc[q][2][0] = fma(a1.x, c0.x, fma(a1.y, c0.y, acc[q][2][0]));
        acc[q][2][1] = fma(a1.y, c0.x, fma(-a1.x, c0.y, acc[q][2][1]));
        acc[q][3][0] = fma(a1.x, c1.x, fma(a1.y, c1.y, acc[q][3][0]));
        acc[q][3][1] = fma(a1.y, c1.x, fma(-a1.x, c1.y, acc[q][3][1]));
      }
      }
    }
  }
  // fixed-order reduction over slices
  __syncthreads();
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int w = tid + q * kCovThreads;
    if (w >= nblk * nslice) continue;
    const int blk = w % nblk, sl = w / nblk;
#pragma unroll
    for (int e = 0; e < 4; ++e) red[((size_t)sl * nblk + blk) * 4 + e] = make_double2(acc[q][e][0], acc[q][e][1]);
  }
  __syncthreads();
  const double invN = (double)N;
  double2* Rb = R + (size_t)b * M * M;
  for (int w = tid; w < nblk * 4; w += kCovThreads) {
    const int blk = w >> 2, e = w & 3;
    double sr = 0.0, si = 0.0;
    for (int sl = 0; sl < nslice; ++sl) {
      const double2 v = red[((size_t)sl * nblk + blk) * 4 + e];
      sr += v.x;
      si += v.y;
    }
    int bi = 0, rem = blk;
    while (rem >= nb - bi) { rem -= nb - bi; ++bi; }
    const int bj = bi + rem;
    const int i = 2 * bi + (e >> 1), j = 2 * bj + (e & 1);
    if (i >= M || j >= M || i > j) continue;       // lower entries of diagonal blocks come from the mirror
    double2 v = make_double2(sr / invN, si / invN);
    if (i == j) v.y = 0.0;
    Rb[(size_t)i * M + j] = v;
    if (i != j) Rb[(size_t)j * M + i] = make_double2(v.x, -v.y);
  }
}

}  // namespace

cudaError_t launch_cov16(const float* X, int64_t B, int64_t N, int M, double* R, cudaStream_t s);

cudaError_t launch_covariance(const float* X, int64_t B, int64_t N, int M, double* R, cudaStream_t s) {
  if (M <= 16) return launch_cov16(X, B, N, M, R, s);
  const int Mp = (M + 1) & ~1;
  const int nb = Mp / 2, nblk = nb * (nb + 1) / 2;
  const int nslice = nblk >= kCovThreads ? 1 : kCovThreads / nblk;
  const int chunk = kChunkDoubles2 / Mp;
  const size_t smem = ((size_t)chunk * Mp + (size_t)nslice * nblk * 4) * sizeof(double2);
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(covariance_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr_set = true;
  }
  count_launch();
  covariance_kernel<<<(unsigned)B, kCovThreads, smem, s>>>(reinterpret_cast<const float2*>(X), N, M,
                                                             reinterpret_cast<double2*>(R));
  return cudaGetLastError();
}

}  // namespace doa
