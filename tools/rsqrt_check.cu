// Accuracy of the eigensolvers' rsqrt / rcp: MUFU seeds and the one-step third-order corrections
// (csrc/eig16.cu) against correctly rounded references, over log-uniform positive arguments.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/rsqrt_check tools/rsqrt_check.cu
#include <cstdio>
#include <cmath>
__global__ void k(double* out, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  unsigned long long h = 0x9E3779B97F4A7C15ULL * (i + 1);
  h ^= h >> 29; h *= 0xBF58476D1CE4E5B9ULL; h ^= h >> 32;
  const double u = (double)(h >> 11) * 0x1.0p-53;          // [0, 1)
  const double x = exp2(-300.0 + 600.0 * u);
  double y0, r0;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y0) : "d"(x));
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r0) : "d"(x));
  const double e = fma(-(x * y0), y0, 1.0);
  const double y = fma(y0 * e, fma(e, 0.375, 0.5), y0);
  const double er = fma(-x, r0, 1.0);
  const double r = fma(r0, fma(er, er, er), r0);
  const double yref = 1.0 / sqrt(x), rref = 1.0 / x;
  out[4 * i + 0] = fabs(y0 / yref - 1.0);
  out[4 * i + 1] = fabs(y / yref - 1.0);
  out[4 * i + 2] = fabs(r0 / rref - 1.0);
  out[4 * i + 3] = fabs(r / rref - 1.0);
}
int main() {
  const int n = 1 << 22;
  double* d; cudaMalloc(&d, 4ull * n * sizeof(double));
  k<<<n / 256, 256>>>(d, n);
  double* h = new double[4ull * n];
  cudaMemcpy(h, d, 4ull * n * sizeof(double), cudaMemcpyDeviceToHost);
  double m[4] = {0, 0, 0, 0};
  for (long i = 0; i < n; ++i) for (int j = 0; j < 4; ++j) m[j] = fmax(m[j], h[4 * i + j]);
  printf("{\"samples\": %d, \"rsqrt_seed_max_rel\": %.3e, \"rsqrt_max_rel\": %.3e, \"rcp_seed_max_rel\": %.3e, \"rcp_max_rel\": %.3e, \"ulp\": %.3e}\n",
         n, m[0], m[1], m[2], m[3], 0x1.0p-53);
  return 0;
}
