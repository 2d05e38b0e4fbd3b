// Per-round timeline of eig16s_kernel<16> on one matrix (clock64 stamps, DOA_EIG_TRACE build of
// csrc/eig16.cu): round start (pilot warp), rotation parameters ready (pilot), block stores issued
// (warp 0), V update done (warp 1).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -o /tmp/tr tools/eig16s_trace.cu
#define DOA_EIG_TRACE
#include "../paper_2007_14135_b200/csrc/eig16.cu"
#include <cstdio>
#include <cmath>
namespace doa { void count_launch() {} }
int main() {
  const int M = 16;
  double2 h[M * M];
  // a random Hermitian matrix: A = X X^H / n from an LCG
  unsigned st = 12345;
  auto rnd = [&]() { st = st * 1664525u + 1013904223u; return (double)(st >> 8) / 16777216.0 - 0.5; };
  double xr[M][64], xi[M][64];
  for (int m = 0; m < M; ++m) for (int n = 0; n < 64; ++n) { xr[m][n] = rnd(); xi[m][n] = rnd(); }
  for (int i = 0; i < M; ++i) for (int j = 0; j < M; ++j) {
    double re = 0, im = 0;
    for (int n = 0; n < 64; ++n) { re += xr[i][n] * xr[j][n] + xi[i][n] * xi[j][n]; im += xi[i][n] * xr[j][n] - xr[i][n] * xi[j][n]; }
    h[i * M + j] = make_double2(re / 64, im / 64);
  }
  double2 *R, *V; double* lam; int* info;
  cudaMalloc(&R, sizeof h); cudaMalloc(&V, sizeof h); cudaMalloc(&lam, M * 8); cudaMalloc(&info, 4);
  cudaMemcpy(R, h, sizeof h, cudaMemcpyHostToDevice);
  doa::CoefPlans cp = {};
  for (int rep = 0; rep < 3; ++rep) {
    doa::eig16s_kernel<16, false><<<1, doa::kSThreads>>>(R, 1, M, lam, V, info, 0, cp);
    cudaDeviceSynchronize();
  }
  long long tr[8 * 512];
  cudaMemcpyFromSymbol(tr, doa::g_eig_trace, sizeof tr);
  int nr = 0;
  while (nr < 512 && tr[8 * nr] != 0 && (nr == 0 || tr[8 * nr] > tr[8 * (nr - 1)])) ++nr;
  printf("rounds %d, total %lld cycles\n", nr, tr[8 * (nr - 1)] - tr[0]);
  double sp = 0, sb = 0, sv = 0, sr = 0, so = 0;
  for (int r = 0; r + 1 < nr; ++r) {
    const long long t0 = tr[8 * r];
    sp += tr[8 * r + 1] - t0; sb += tr[8 * r + 2] - t0; sv += tr[8 * r + 3] - t0; sr += tr[8 * (r + 1)] - t0;
    so += tr[8 * r + 4] - t0;
    if (r < 5 || r % 15 == 0) printf("r%3d: (loads %5lld  pilot element %5lld: DOA_EIG_TRACE slots 5/4, add when needed)  params %5lld  blocks %5lld  V %5lld  next round %5lld\n", r,
                                     tr[8 * r + 5] - t0, tr[8 * r + 4] - t0, tr[8 * r + 1] - t0, tr[8 * r + 2] - t0, tr[8 * r + 3] - t0,
                                     tr[8 * (r + 1)] - t0);
  }
  const int n = nr - 1;
  printf("mean: pilot element %.0f  params %.0f  blocks %.0f  V %.0f  round %.0f cycles\n", so / n, sp / n, sb / n, sv / n, sr / n);
  return 0;
}
