// Single-warp dependent-chain latencies on B200 (cycles per op): DFMA, DMUL, DADD, MUFU.RSQ64H
// (+ the two Newton steps used by the eigensolver), FFMA, LDS round trip, bar.sync of 64 threads.
#include <cstdio>
__device__ __forceinline__ double rsq_approx(double x) { double y; asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x)); return y; }
__global__ void lat(double* out, long long* cyc, double seed) {
  __shared__ double sm[64];
  double a = seed, b = 1.0000001, c = 1e-9;
  float fa = (float)seed;
  long long t0, t1;
  const int n = 1024;
  sm[threadIdx.x] = seed;
  __syncthreads();
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) a = fma(a, b, c);
  t1 = clock64(); if (threadIdx.x == 0) cyc[0] = (t1 - t0);
  // DMUL chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) a = a * b;
  t1 = clock64(); if (threadIdx.x == 0) cyc[1] = (t1 - t0);
  // DADD chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) a = a + c;
  t1 = clock64(); if (threadIdx.x == 0) cyc[2] = (t1 - t0);
  // MUFU.RSQ64H chain
  double r = a;
  t0 = clock64();
  for (int i = 0; i < n; ++i) r = rsq_approx(r + 1.0);
  t1 = clock64(); if (threadIdx.x == 0) cyc[3] = (t1 - t0);
  // FFMA chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) fa = fmaf(fa, 1.0000001f, 1e-9f);
  t1 = clock64(); if (threadIdx.x == 0) cyc[4] = (t1 - t0);
  // LDS dependent chain (pointer chase through smem index)
  int idx = threadIdx.x & 63;
  volatile int* si = reinterpret_cast<volatile int*>(sm);
  if (threadIdx.x < 64) si[threadIdx.x] = (threadIdx.x + 1) & 63;
  __syncthreads();
  t0 = clock64();
  for (int i = 0; i < n; ++i) idx = si[idx];
  t1 = clock64(); if (threadIdx.x == 0) cyc[5] = (t1 - t0);
  // bar.sync (CTA of 64)
  t0 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  t1 = clock64(); if (threadIdx.x == 0) cyc[6] = (t1 - t0);
  // __syncwarp
  t0 = clock64();
  for (int i = 0; i < n; ++i) __syncwarp();
  t1 = clock64(); if (threadIdx.x == 0) cyc[7] = (t1 - t0);
  out[threadIdx.x] = a + r + fa + idx;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 64 * 8); cudaMalloc(&c, 16 * 8);
  lat<<<1, 64>>>(o, c, 1.5); cudaDeviceSynchronize();
  lat<<<1, 64>>>(o, c, 1.5); long long h[16]; cudaMemcpy(h, c, 16 * 8, cudaMemcpyDeviceToHost);
  const char* nm[] = {"DFMA", "DMUL", "DADD", "MUFU.RSQ64H(+DADD)", "FFMA", "LDS chase", "bar.sync 64", "syncwarp"};
  for (int i = 0; i < 8; ++i) printf("{\"op\": \"%s\", \"cycles_per_op\": %.2f}\n", nm[i], h[i] / 1024.0);
  return 0;
}
