// DMMA m8n8k4 f64 issue/latency probe: NCH independent accumulator chains per warp, W warps per
// SM sub-partition.  Reports clocks per DMMA per SMSP (16 = full DMMA rate).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int NCH>
__global__ void lat_k(double* out, int iters, long long* clk) {
  double a = 1e-3 * threadIdx.x, b = 1.0 - 1e-4 * threadIdx.x;
  double c[NCH][2];
#pragma unroll
  for (int k = 0; k < NCH; ++k) c[k][0] = c[k][1] = 0.0;
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < NCH; ++k) dmma(c[k][0], c[k][1], a, b);
  }
  const long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int k = 0; k < NCH; ++k) s += c[k][0] + c[k][1];
  if (s == 1234.5) out[0] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) clk[0] = t1 - t0;
}

int main() {
  double* d;
  long long* clk;
  cudaMalloc(&d, 64);
  cudaMalloc(&clk, 8);
  const int iters = 4096;
  auto run = [&](const char* nm, int nch, int warps_per_smsp, auto launch) {
    launch(148, 32 * 4 * warps_per_smsp);
    cudaDeviceSynchronize();
    launch(148, 32 * 4 * warps_per_smsp);
    long long c;
    cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
    const double per = (double)c / (iters * (double)nch * warps_per_smsp);
    printf("{\"chains\":%d,\"warps_per_smsp\":%d,\"clk_per_dmma_per_smsp\":%.2f,\"clk_per_iter_per_warp\":%.1f}\n",
           nch, warps_per_smsp, per, (double)c / iters);
  };
  for (int w : {1, 2, 4}) {
    run("1", 1, w, [&](int g, int t) { lat_k<1><<<g, t>>>(d, iters, clk); });
    run("2", 2, w, [&](int g, int t) { lat_k<2><<<g, t>>>(d, iters, clk); });
    run("4", 4, w, [&](int g, int t) { lat_k<4><<<g, t>>>(d, iters, clk); });
    run("8", 8, w, [&](int g, int t) { lat_k<8><<<g, t>>>(d, iters, clk); });
    run("16", 16, w, [&](int g, int t) { lat_k<16><<<g, t>>>(d, iters, clk); });
  }
  return 0;
}
