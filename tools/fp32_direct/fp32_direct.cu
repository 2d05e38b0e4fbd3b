// comparison kernel only (NOT the product path): the north-star-named
// fp32 direct form of the scan, f(theta) = sum_k w_k |e_k^H a(theta)|^2 with a_m = exp(-j pi u m)
// generated with fp32 sincospi, evaluated on the FP32 pipe.  Used by tools/fp32_direct_eval.py to
// evidence (ncu time + parity against the fp64 oracle) why the product scan is the fp64 Toeplitz
// contraction on the DMMA pipe.
//
// Layout: U[b][k][m] complex64 = w_k^(1/2) e_k (weights folded in), k < K; one thread per angle,
// a CTA covers 128 angles and loops over a chunk of frames; the frame's vectors are staged in smem.
#include <cuda_runtime.h>
#include <cstdint>

namespace {

template <int M>
__global__ void __launch_bounds__(128) direct_kernel(const float2* __restrict__ U, int64_t B, int K, int64_t fpc,
                                                     float theta0, float dtheta, double theta0_d, double dtheta_d,
                                                     float dl, int64_t L, int exact_u, float* __restrict__ F) {
  extern __shared__ float2 us[];                    // [K][M]
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = i < L;
  // steering in fp32: u = 2 (d/lambda) sin(theta); exact_u = 1 rounds the fp64 u to fp32 (best case)
  float u;
  if (exact_u) {
    const double th = __dadd_rn(__dmul_rn((double)i, dtheta_d), theta0_d);
    u = (float)(2.0 * (double)dl * sinpi(th / 180.0));
  } else {
    const float th = theta0 + (float)i * dtheta;
    u = 2.0f * dl * sinpif(th / 180.0f);
  }
  float ar[M], ai[M];
#pragma unroll
  for (int m = 0; m < M; ++m) {
    float s, c;
    sincospif(u * (float)m, &s, &c);
    ar[m] = c;
    ai[m] = -s;
  }
  const int64_t b0 = (int64_t)blockIdx.y * fpc, b1 = (b0 + fpc < B) ? b0 + fpc : B;
  for (int64_t b = b0; b < b1; ++b) {
    __syncthreads();
    for (int e = threadIdx.x; e < K * M; e += blockDim.x) us[e] = U[(size_t)b * K * M + e];
    __syncthreads();
    float acc = 0.f;
    for (int k = 0; k < K; ++k) {
      float pr = 0.f, pi = 0.f;
#pragma unroll
      for (int m = 0; m < M; ++m) {          // conj(e_m) a_m
        const float2 e = us[k * M + m];
        pr = fmaf(e.x, ar[m], fmaf(e.y, ai[m], pr));
        pi = fmaf(e.x, ai[m], fmaf(-e.y, ar[m], pi));
      }
      acc = fmaf(pr, pr, fmaf(pi, pi, acc));
    }
    if (valid) F[(size_t)b * L + i] = acc;
  }
}

}  // namespace

extern "C" int fp32_direct_scan(const void* U, int64_t B, int K, int M, double theta0, double dtheta, double dl,
                                int64_t L, int exact_u, float* F, void* stream) {
  const int64_t gx = (L + 127) / 128;
  int64_t fpc = (gx * B) / (148 * 16);
  if (fpc < 1) fpc = 1;
  if (fpc > B) fpc = B;
  const int64_t gy = (B + fpc - 1) / fpc;
  const size_t smem = (size_t)K * M * sizeof(float2);
  cudaStream_t s = (cudaStream_t)stream;
  const float2* u = reinterpret_cast<const float2*>(U);
  switch (M) {
    case 8: direct_kernel<8><<<dim3((unsigned)gx, (unsigned)gy), 128, smem, s>>>(u, B, K, fpc, (float)theta0, (float)dtheta, theta0, dtheta, (float)dl, L, exact_u, F); break;
    case 16: direct_kernel<16><<<dim3((unsigned)gx, (unsigned)gy), 128, smem, s>>>(u, B, K, fpc, (float)theta0, (float)dtheta, theta0, dtheta, (float)dl, L, exact_u, F); break;
    default: return 1;
  }
  return (int)cudaGetLastError();
}
