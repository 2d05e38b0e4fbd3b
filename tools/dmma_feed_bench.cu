// Microbenchmark: how fast can DMMA m8n8k4 run when its B operand streams from shared memory
// (the scan kernel's inner loop) — vs register-resident operands, and with one B fragment
// feeding two frame groups.  Prints TFLOP/s (fp64) per variant.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

// variant 0: B from smem per DMMA (scan layout), one group per iteration
// variant 1: B from smem, reused for two groups (2 accumulator sets)
// variant 2: B from registers (no LDS)
template <int VAR>
__global__ void __launch_bounds__(256) feed_k(double* out, int iters) {
  __shared__ double Ts[8 * 8 * 32];
  for (int e = threadIdx.x; e < 8 * 8 * 32; e += 256) Ts[e] = 1e-3 * e;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  double a[8], a2[8], breg[8];
#pragma unroll
  for (int s = 0; s < 8; ++s) { a[s] = 1e-2 * (s + lane); a2[s] = a[s] * 0.5; breg[s] = Ts[s * 32 + lane]; }
  double acc[8][2], acc2[8][2];
#pragma unroll
  for (int t = 0; t < 8; ++t) { acc[t][0] = acc[t][1] = acc2[t][0] = acc2[t][1] = 0.0; }
  const double* T = Ts + lane;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int s = 0; s < 8; ++s)
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        if (VAR == 2) {
          dmma(acc[t][0], acc[t][1], a[s], breg[(s + t) & 7]);
        } else {
          const double b = T[(s * 8 + t) * 32];
          dmma(acc[t][0], acc[t][1], a[s], b);
          if (VAR == 1) dmma(acc2[t][0], acc2[t][1], a2[s], b);
        }
      }
  }
  double sm = 0;
#pragma unroll
  for (int t = 0; t < 8; ++t) sm += acc[t][0] + acc[t][1] + acc2[t][0] + acc2[t][1];
  if (sm == 1234.5) out[0] = sm;
}

int main() {
  double* d;
  cudaMalloc(&d, 64);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 2000;
  auto run = [&](const char* name, auto launch, double dmma_per_iter_per_warp, int blocks) {
    launch();
    cudaDeviceSynchronize();
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    const double flop = dmma_per_iter_per_warp * 512.0 * iters * blocks * 8;
    printf("{\"variant\":\"%s\",\"ms\":%.3f,\"TFLOPs\":%.2f}\n", name, best, flop / best / 1e9);
  };
  for (int bps : {2, 3}) {
    const int blocks = 148 * bps;
    printf("# %d CTAs/SM\n", bps);
    run("B from smem, 1 group", [&] { feed_k<0><<<blocks, 256>>>(d, iters); }, 64, blocks);
    run("B from smem, 2 groups", [&] { feed_k<1><<<blocks, 256>>>(d, iters); }, 128, blocks);
    run("B in registers", [&] { feed_k<2><<<blocks, 256>>>(d, iters); }, 64, blocks);
  }
  return 0;
}
