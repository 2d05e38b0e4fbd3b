/*
 * doa_demo.c — the C ABI (include/doa.h) used from plain C, no Python: generate a batch of
 * synthetic ULA frames on the device (doa_generate, Eq. 1), estimate the DOAs with the fused
 * doa_run for one estimator, and print the estimates next to the true angles plus the device
 * time of the run.
 *
 *   cc -O2 -I include -I /usr/local/cuda/include examples/doa_demo.c \
 *      -L paper_2007_14135_b200 -ldoa -L /usr/local/cuda/lib64 -lcudart -o examples/doa_demo
 *   LD_LIBRARY_PATH=paper_2007_14135_b200 examples/doa_demo [alg M D B N dtheta]
 */
#include <cuda_runtime_api.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "doa.h"

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess) { fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_)); return 1; } \
  } while (0)
#define DK(x)                                                                              \
  do {                                                                                     \
    doa_status_t s_ = (x);                                                                 \
    if (s_ != DOA_OK) { fprintf(stderr, "%s: %s (%s)\n", #x, doa_status_string(s_), doa_last_error()); return 1; } \
  } while (0)

int main(int argc, char** argv) {
  const char* algs[] = {"phd", "music", "ev", "mn"};
  int alg = 1, M = 16, D = 4;
  long long B = 4096, N = 256;
  double dtheta = 0.01;
  if (argc > 1) for (int a = 0; a < 4; ++a) if (!strcmp(argv[1], algs[a])) alg = a;
  if (argc > 2) M = atoi(argv[2]);
  if (argc > 3) D = atoi(argv[3]);
  if (argc > 4) B = atoll(argv[4]);
  if (argc > 5) N = atoll(argv[5]);
  if (argc > 6) dtheta = atof(argv[6]);
  const long long L = llround(180.0 / dtheta) + 1;

  /* true DOAs: D angles spread over [-60, 60] deg, shifted per frame, the same for all snapshots */
  double* th = (double*)malloc(sizeof(double) * B * D);
  for (long long b = 0; b < B; ++b)
    for (int d = 0; d < D; ++d) th[b * D + d] = -60.0 + 120.0 * (d + 0.5) / D + 7.3 * sin(0.37 * b + d);
  double* th_d;
  float* X;
  int32_t *idx_d, *npk_d, *info_d;
  float* val_d;
  CK(cudaMalloc((void**)&th_d, sizeof(double) * B * D));
  CK(cudaMalloc((void**)&X, sizeof(float) * 2 * B * N * M));
  CK(cudaMalloc((void**)&idx_d, sizeof(int32_t) * B * D));
  CK(cudaMalloc((void**)&val_d, sizeof(float) * B * D));
  CK(cudaMalloc((void**)&npk_d, sizeof(int32_t) * B));
  CK(cudaMalloc((void**)&info_d, sizeof(int32_t) * B));
  CK(cudaMemcpy(th_d, th, sizeof(double) * B * D, cudaMemcpyHostToDevice));

  DK(doa_generate(M, 0.5, D, th_d, 1, 15.0, 2026ULL, 0, B, N, X, NULL));
  doa_plan_t plan;
  DK(doa_plan_create(&plan, M, 0.5, D, -90.0, dtheta, L, (doa_alg_t)alg, B));
  DK(doa_run(plan, X, B, N, idx_d, val_d, npk_d, NULL, info_d, NULL));   /* warm-up */
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0, NULL));
  DK(doa_run(plan, X, B, N, idx_d, val_d, npk_d, NULL, info_d, NULL));
  CK(cudaEventRecord(e1, NULL));
  CK(cudaEventSynchronize(e1));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, e0, e1));

  int32_t* idx = (int32_t*)malloc(sizeof(int32_t) * B * D);
  int32_t* npk = (int32_t*)malloc(sizeof(int32_t) * B);
  CK(cudaMemcpy(idx, idx_d, sizeof(int32_t) * B * D, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(npk, npk_d, sizeof(int32_t) * B, cudaMemcpyDeviceToHost));

  /* match each true angle to the nearest estimate; report the worst error over the batch */
  double worst = 0.0;
  long long missing = 0;
  for (long long b = 0; b < B; ++b)
    for (int d = 0; d < D; ++d) {
      double best = 1e9;
      for (int k = 0; k < npk[b]; ++k) {
        const double e = fabs(-90.0 + idx[b * D + k] * dtheta - th[b * D + d]);
        if (e < best) best = e;
      }
      if (best > 1e8) ++missing; else if (best > worst) worst = best;
    }
  printf("alg=%s M=%d D=%d B=%lld N=%lld L=%lld\n", algs[alg], M, D, B, N, L);
  for (long long b = 0; b < 3 && b < B; ++b) {
    printf("frame %lld  true:", b);
    for (int d = 0; d < D; ++d) printf(" %8.3f", th[b * D + d]);
    printf("   estimated:");
    for (int k = 0; k < npk[b]; ++k) printf(" %8.3f", -90.0 + idx[b * D + k] * dtheta);
    printf("\n");
  }
  printf("doa_run: %.3f ms for %lld frames (%.3e frames/s); worst |error| %.4f deg, missing %lld\n", ms, B,
         B / (ms * 1e-3), worst, missing);
  DK(doa_plan_destroy(plan));
  cudaFree(th_d); cudaFree(X); cudaFree(idx_d); cudaFree(val_d); cudaFree(npk_d); cudaFree(info_d);
  free(th); free(idx); free(npk);
  return 0;
}
