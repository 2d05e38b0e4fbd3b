// Dependent-chain latencies on this GPU (one warp): DFMA, DMUL, DADD, MUFU rsqrt/rcp f64 approx,
// the rsqrt_pos idiom (MUFU + 2 Newton), LDS.64, SHFL, a 64-thread named barrier and __syncthreads.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/lat tools/lat_fp64.cu && /tmp/lat
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double rsqrt_pos(double x) {
  double y;
  asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double hx = 0.5 * x;
  y = y * fma(-hx * y, y, 1.5);
  y = y * fma(-hx * y, y, 1.5);
  return y;
}

template <int OP>
__global__ void k(double* out, long long* cyc, int iters) {
  __shared__ double sm[64];
  __shared__ int si[64];
  sm[threadIdx.x] = 1.0 + threadIdx.x * 1e-9;
  si[threadIdx.x] = threadIdx.x;
  __syncthreads();
  double x = 1.0 + threadIdx.x * 1e-12, y = 0.999999, z = 1e-7;
  int idx = threadIdx.x;
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (OP == 0) x = fma(x, y, z);
    if (OP == 1) x = x * y;
    if (OP == 2) x = x + z;
    if (OP == 3) { double r; asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); x = r; }
    if (OP == 4) x = rsqrt_pos(x);
    if (OP == 5) idx = si[idx & 63];
    if (OP == 6) x = __shfl_xor_sync(0xffffffffu, x, 1);
    if (OP == 7) { asm volatile("bar.sync 1, 64;"); x = x + z; }
    if (OP == 8) { __syncthreads(); x = x + z; }
    if (OP == 9) { double r; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); x = r; }
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; }
  out[threadIdx.x] = x + idx;
}

int main() {
  double* d; long long* c;
  cudaMalloc(&d, 64 * 8); cudaMalloc(&c, 8);
  const char* names[] = {"DFMA", "DMUL", "DADD", "MUFU.RSQ64H", "rsqrt_pos (MUFU+2 Newton)", "LDS.32 dep",
                         "SHFL f64", "bar.sync 64 thr (2 warps) + DADD", "__syncthreads (2 warps) + DADD", "MUFU.RCP64H"};
  const int iters = 4096;
  auto run = [&](auto kern, int i) {
    kern<<<1, 64>>>(d, c, iters); cudaDeviceSynchronize();
    kern<<<1, 64>>>(d, c, iters); cudaDeviceSynchronize();
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("{\"op\": \"%s\", \"cycles_per_iter\": %.2f}\n", names[i], (double)h / iters);
  };
  run(k<0>, 0); run(k<1>, 1); run(k<2>, 2); run(k<3>, 3); run(k<4>, 4); run(k<5>, 5); run(k<6>, 6);
  run(k<7>, 7); run(k<8>, 8); run(k<9>, 9);
  return 0;
}
