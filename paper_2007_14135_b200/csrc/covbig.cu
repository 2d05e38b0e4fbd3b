// S1 for 16 < M <= 64 on the FP64 tensor pipe: R = (1/N) X X^H (Eq. 3).
//
// One CTA per frame; warps own upper 8x8 tiles of R and accumulate R_re += Xr_I Xr_J^T +
// Xi_I Xi_J^T and R_im += Xi_I Xr_J^T - Xr_I Xi_J^T with mma.sync m8n8k4 f64 (4 DMMAs and 2
// accumulators per tile).  Snapshot chunks are staged through shared memory (coalesced complex64
// loads, converted once, Re/Im planes with a padded stride so the fragment loads are
// conflict-free), double-buffered with a register software pipeline.  fp32 products are exact in
// fp64; the DMMA order is fixed (deterministic).  The tiles are written to R mirrored (exact
// conjugate symmetry, real diagonal).
#include "doa_internal.cuh"

namespace doa {
namespace {

constexpr int kChunk = 32;                     // snapshots per staged chunk (8 k-steps)

__device__ __forceinline__ void dmma_b(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// Tiles of R itself (the round-1 Gram-staging variant was retired).  A warp owns TPW upper 8x8 tiles (I <= J) of the
// M x M covariance and, per k-step, accumulates R_re += Xr_I Xr_J^T + Xi_I Xi_J^T and
// R_im += Xi_I Xr_J^T - Xr_I Xi_J^T directly (4 DMMAs, 2 accumulators per tile), so no Gram
// matrix is staged in shared memory: the CTA needs only the two snapshot stages (69.6 KB at
// MP = 64), two CTAs fit per SM, and the tiles are written to R (mirrored, exact conjugate
// symmetry, real diagonal) straight from the accumulators.
template <int MP>
struct CovBig2 {
  static constexpr int TP = MP / 8;
  static constexpr int NT = TP * (TP + 1) / 2;             // upper tiles of R
  static constexpr int TPW = MP == 64 ? 4 : 2;             // tiles per warp
  static constexpr int WARPS = NT / TPW;                   // 9 (MP = 64) or 5 (MP = 32)
  static constexpr int T = WARPS * 32;
  static constexpr int XS = MP + 4;
  static constexpr size_t STAGE = (size_t)2 * kChunk * XS;
  static constexpr size_t SMEM = 2 * STAGE * 8;
};

template <int MP>
__global__ void __launch_bounds__(CovBig2<MP>::T) covbig2_kernel(const float2* __restrict__ X, int64_t N, int M,
                                                                 double2* __restrict__ R) {
  using C = CovBig2<MP>;
  constexpr int XS = C::XS, TP = C::TP, TPW = C::TPW, T = C::T;
  extern __shared__ double sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int r = lane >> 2, q = lane & 3;
  const int64_t b = blockIdx.x;
  const float2* Xb = X + (size_t)b * N * M;
  // this warp's tiles: row-major upper tiles, TPW consecutive ones
  int tI[TPW], tJ[TPW];
#pragma unroll
  for (int u = 0; u < TPW; ++u) {
    int t = warp * TPW + u, I = 0;
    while (t >= TP - I) { t -= TP - I; ++I; }
    tI[u] = I;
    tJ[u] = I + t;
  }
  double cre[TPW][2], cim[TPW][2];
#pragma unroll
  for (int u = 0; u < TPW; ++u) { cre[u][0] = cre[u][1] = cim[u][0] = cim[u][1] = 0.0; }

  const int64_t nchunks = (N + kChunk - 1) / kChunk;
  constexpr int PER = (kChunk * MP + T - 1) / T;
  float2 pre[PER];
  auto load = [&](int64_t c) {
    const int64_t n0 = c * kChunk;
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int e = tid + u * T, n = e / MP, m = e - (e / MP) * MP;
      pre[u] = (e < kChunk * MP && m < M && n0 + n < N) ? __ldg(Xb + (size_t)(n0 + n) * M + m) : make_float2(0.f, 0.f);
    }
  };
  auto store = [&](int buf) {
    double* Xr = sm + buf * C::STAGE;
    double* Xi = Xr + kChunk * XS;
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int e = tid + u * T, n = e / MP, m = e - (e / MP) * MP;
      if (e < kChunk * MP) {
        Xr[n * XS + m] = (double)pre[u].x;
        Xi[n * XS + m] = (double)pre[u].y;
      }
    }
  };
  load(0);
  store(0);
  __syncthreads();
  for (int64_t c = 0; c < nchunks; ++c) {
    const int buf = (int)(c & 1);
    if (c + 1 < nchunks) load(c + 1);
    const double* Xr = sm + buf * C::STAGE;
    const double* Xi = Xr + kChunk * XS;
#pragma unroll 2
    for (int ks = 0; ks < kChunk / 4; ++ks) {
      const int n = 4 * ks + q;                            // fragment element Y[8I + r][n]
#pragma unroll
      for (int u = 0; u < TPW; ++u) {
        const double ar = Xr[n * XS + 8 * tI[u] + r], ai = Xi[n * XS + 8 * tI[u] + r];
        const double br = Xr[n * XS + 8 * tJ[u] + r], bi = Xi[n * XS + 8 * tJ[u] + r];
        dmma_b(cre[u][0], cre[u][1], ar, br);
        dmma_b(cre[u][0], cre[u][1], ai, bi);
        dmma_b(cim[u][0], cim[u][1], ai, br);
        dmma_b(cim[u][0], cim[u][1], -ar, bi);
      }
    }
    if (c + 1 < nchunks) store(buf ^ 1);
    __syncthreads();
  }
  const double dn = (double)N;
  double2* Rb = R + (size_t)b * M * M;
#pragma unroll
  for (int u = 0; u < TPW; ++u)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int i = 8 * tI[u] + r, j = 8 * tJ[u] + 2 * q + e;
      if (i < M && j < M && i <= j) {
        const double2 v = make_double2(cre[u][e] / dn, i == j ? 0.0 : cim[u][e] / dn);
        Rb[(size_t)i * M + j] = v;
        if (i != j) Rb[(size_t)j * M + i] = make_double2(v.x, -v.y);
      }
    }
}

}  // namespace

template <int MP>
cudaError_t launch_covbig2_t(const float* X, int64_t B, int64_t N, int M, double* R, cudaStream_t s) {
  const size_t smem = CovBig2<MP>::SMEM;
  kernel_occupancy(covbig2_kernel<MP>, CovBig2<MP>::T, smem);        // sets the smem attribute on this device
  count_launch();
  covbig2_kernel<MP><<<(unsigned)B, CovBig2<MP>::T, smem, s>>>(reinterpret_cast<const float2*>(X), N, M,
                                                               reinterpret_cast<double2*>(R));
  return cudaGetLastError();
}

cudaError_t launch_covbig(const float* X, int64_t B, int64_t N, int M, double* R, cudaStream_t s) {
  if (M <= 32) return launch_covbig2_t<32>(X, B, N, M, R, s);
  return launch_covbig2_t<64>(X, B, N, M, R, s);
}

}  // namespace doa
