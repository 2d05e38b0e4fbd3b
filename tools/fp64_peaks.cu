// Microbenchmark: FP64 pipe peaks on the B200 (DFMA, DMMA m8n8k4, F2F.F64.F32, SHFL, MUFU.RSQ64H).
// Used to derive the "alu" roofline denominator for the FP64-bound DOA path.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s at %d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)

template<int CH>
__global__ void dfma_k(double* out, int iters, double a, double b) {
  double acc[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) acc[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c];
  if (s == 12345.678) out[0] = s;
}

__global__ void ffma_k(float* out, int iters, float a, float b) {
  float acc[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) acc[c] = threadIdx.x * 1e-3f + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[c] = fmaf(acc[c], a, b);
  }
  float s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += acc[c];
  if (s == 12345.678f) out[0] = s;
}

__global__ void dmma_k(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[4][2];
#pragma unroll
  for (int k = 0; k < 4; ++k) { c[k][0] = 0; c[k][1] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) s += c[k][0] + c[k][1];
  if (s == 12345.678) out[0] = s;
}

// DMMA and DFMA interleaved: do the tensor-DMMA subpipe and the FP64 FMA pipe add up?
template<int ND, int NF>
__global__ void mix_k(double* out, int iters, double x, double y) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[4][2];
  double f[NF];
#pragma unroll
  for (int k = 0; k < 4; ++k) { c[k][0] = 0; c[k][1] = 0; }
#pragma unroll
  for (int k = 0; k < NF; ++k) f[k] = k + threadIdx.x;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < ND; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[k & 3][0]), "+d"(c[k & 3][1]) : "d"(a), "d"(b));
#pragma unroll
    for (int k = 0; k < NF; ++k) f[k] = fma(f[k], x, y);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) s += c[k][0] + c[k][1];
#pragma unroll
  for (int k = 0; k < NF; ++k) s += f[k];
  if (s == 12345.678) out[0] = s;
}

__global__ void cvt_k(double* out, int iters, const float* in) {
  float x[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) x[c] = in[(threadIdx.x + c) & 255];
  double s[8] = {0,0,0,0,0,0,0,0};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 8; ++c) { s[c] = (double)x[c]; x[c] = __int_as_float(__float_as_int(x[c]) ^ (int)(s[c] != 0.5)); }
  }
  double t = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) t += s[c];
  if (t == 12345.678) out[0] = t;
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("{\"gpu\":\"%s\",\"sms\":%d,\"clock_khz_attr\":%d}\n", p.name, p.multiProcessorCount, clk);
  double* d; float* f; CK(cudaMalloc(&d, 64)); CK(cudaMalloc(&f, 4096)); CK(cudaMemset(f, 0, 4096));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int blocks = p.multiProcessorCount * 8, threads = 256;
  int iters = 20000;
  auto run = [&](const char* name, auto launch, double flops_per_iter_per_thread) {
    launch(); CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); launch(); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    double tot = flops_per_iter_per_thread * iters * (double)blocks * threads;
    printf("{\"kernel\":\"%s\",\"ms\":%.4f,\"Gops_per_s\":%.1f}\n", name, best, tot / best / 1e6);
    return 0;
  };
  run("dfma_ch8 (flops=2/fma)", [&]{ dfma_k<8><<<blocks, threads>>>(d, iters, 0.999, 1e-3); }, 16.0);
  run("dfma_ch4", [&]{ dfma_k<4><<<blocks, threads>>>(d, iters, 0.999, 1e-3); }, 8.0);
  run("dfma_ch2", [&]{ dfma_k<2><<<blocks, threads>>>(d, iters, 0.999, 1e-3); }, 4.0);
  run("ffma_ch8", [&]{ ffma_k<<<blocks, threads>>>(f, iters, 0.999f, 1e-3f); }, 16.0);
  // DMMA m8n8k4: 8*8*4 FMA per warp per instr = 256 FMA = 512 flop per warp -> 16 flop per thread per mma
  run("dmma_m8n8k4 x4 (flop)", [&]{ dmma_k<<<blocks, threads>>>(d, iters); }, 4 * 16.0);
  // flops per thread per iter: DMMA 16 flop/thread each, DFMA 2 flop each
  run("mix 4 DMMA + 16 DFMA", [&]{ mix_k<4, 16><<<blocks, threads>>>(d, iters, 0.999, 1e-3); }, 4 * 16.0 + 16 * 2.0);
  run("mix 4 DMMA + 32 DFMA", [&]{ mix_k<4, 32><<<blocks, threads>>>(d, iters, 0.999, 1e-3); }, 4 * 16.0 + 32 * 2.0);
  run("mix 4 DMMA + 8 DFMA", [&]{ mix_k<4, 8><<<blocks, threads>>>(d, iters, 0.999, 1e-3); }, 4 * 16.0 + 8 * 2.0);
  run("cvt_f32_f64 x8 (ops)", [&]{ cvt_k<<<blocks, threads>>>(d, iters, f); }, 8.0);
  return 0;
}
