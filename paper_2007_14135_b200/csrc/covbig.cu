// S1 for 16 < M <= 64 on the FP64 tensor pipe: R = (1/N) X X^H (Eq. 3).
//
// One CTA per frame.  With Y = [Re X^T; Im X^T] (2 MP x N, MP = 32 or 64 padded rows) the real
// Gram G = Y Y^T has RB = 2 MP / 8 row blocks; warp w (RB/2 warps) owns the upper tiles of row
// blocks w and RB-1-w — (RB - w) + (w + 1) = RB + 1 tiles, a perfectly balanced triangle — and
// accumulates them with mma.sync m8n8k4 f64: per k-step it loads the RB column fragments once
// and its two row fragments, then issues RB + 1 DMMAs.  Snapshot chunks are staged through
// shared memory (coalesced complex64 loads, converted once, Re/Im planes with a padded stride so
// the fragment loads are conflict-free), double-buffered.  At the end the tiles go to a shared
// Gram matrix and are combined into the Hermitian R = (G_rr + G_ii) + j (G_ir - G_ri), / N
// (exact conjugate mirror, real diagonal).  fp32 products are exact in fp64; the DMMA order is
// fixed (deterministic).
#include "doa_internal.cuh"

namespace doa {
namespace {

constexpr int kChunk = 32;                     // snapshots per staged chunk (8 k-steps)
#ifndef DOA_COVBIG2
#define DOA_COVBIG2 1                          // tiles of R per warp, no staged Gram (covbig2_kernel)
#endif

__device__ __forceinline__ void dmma_b(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <int MP>
struct CovBig {
  static constexpr int RB = 2 * MP / 8;                  // 8-row blocks of Y
  static constexpr int WARPS = RB / 2;
  static constexpr int XS = MP + 4;                      // plane row stride (doubles), = 4 mod 16: the
                                                         // fragment loads (rows n = 4ks + q, cols r) hit 16 distinct bank pairs per half-warp
  static constexpr int GS = 2 * MP + 1;                  // Gram row stride (doubles)
  static constexpr size_t STAGE = (size_t)2 * kChunk * XS;               // doubles per stage (Re + Im)
  static constexpr size_t SMEM = (2 * STAGE > (size_t)(2 * MP) * GS ? 2 * STAGE : (size_t)(2 * MP) * GS) * 8;
};

template <int MP>
__global__ void __launch_bounds__(CovBig<MP>::WARPS * 32, 1) covbig_kernel(const float2* __restrict__ X, int64_t N,
                                                                           int M, double2* __restrict__ R) {
  using C = CovBig<MP>;
  constexpr int RB = C::RB, WARPS = C::WARPS, XS = C::XS, GS = C::GS, T = WARPS * 32;
  extern __shared__ double sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int r = lane >> 2, q = lane & 3;
  const int64_t b = blockIdx.x;
  const float2* Xb = X + (size_t)b * N * M;
  const int I1 = warp, I2 = RB - 1 - warp;               // this warp's row blocks
  // plane row of row block I: block I < RB/2 is Re of elements 8I..8I+7, else Im of 8(I-RB/2)..
  const int off1 = (I1 < RB / 2 ? 0 : kChunk * XS) + 8 * (I1 % (RB / 2)) + r;
  const int off2 = (I2 < RB / 2 ? 0 : kChunk * XS) + 8 * (I2 % (RB / 2)) + r;

  double acc1[RB][2], acc2[RB][2];
#pragma unroll
  for (int J = 0; J < RB; ++J) { acc1[J][0] = acc1[J][1] = 0.0; acc2[J][0] = acc2[J][1] = 0.0; }

  const int64_t nchunks = (N + kChunk - 1) / kChunk;
  // Software pipeline over snapshot chunks: the next chunk's global loads are issued into
  // registers before this chunk's DMMAs and stored (converted) into the other buffer after them,
  // so their latency overlaps the math instead of stalling the same warps.
  constexpr int PER = kChunk * MP / T;                   // elements per thread per chunk
  float2 pre[PER];
  auto load = [&](int64_t c) {
    const int64_t n0 = c * kChunk;
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int e = tid + u * T, n = e / MP, m = e - (e / MP) * MP;
      pre[u] = (m < M && n0 + n < N) ? __ldg(Xb + (size_t)(n0 + n) * M + m) : make_float2(0.f, 0.f);
    }
  };
  auto store = [&](int buf) {
    double* Xr = sm + buf * C::STAGE;
    double* Xi = Xr + kChunk * XS;
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int e = tid + u * T, n = e / MP, m = e - (e / MP) * MP;
      Xr[n * XS + m] = (double)pre[u].x;
      Xi[n * XS + m] = (double)pre[u].y;
    }
  };
  load(0);
  store(0);
  __syncthreads();
  for (int64_t c = 0; c < nchunks; ++c) {
    const int buf = (int)(c & 1);
    if (c + 1 < nchunks) load(c + 1);
    const double* Xs = sm + buf * C::STAGE;
#pragma unroll 2
    for (int ks = 0; ks < kChunk / 4; ++ks) {
      const int n = 4 * ks + q;                          // fragment element Y[8I + r][n]
      double fr[RB];
#pragma unroll
      for (int J = 0; J < RB; ++J)
        fr[J] = Xs[(J < RB / 2 ? 0 : kChunk * XS) + n * XS + 8 * (J % (RB / 2)) + r];
      const double a1 = Xs[n * XS + off1], a2 = Xs[n * XS + off2];
#pragma unroll
      for (int J = 0; J < RB; ++J) {
        if (J >= I1) dmma_b(acc1[J][0], acc1[J][1], a1, fr[J]);
        if (J >= I2 && I2 != I1) dmma_b(acc2[J][0], acc2[J][1], a2, fr[J]);
      }
    }
    if (c + 1 < nchunks) store(buf ^ 1);                 // other buffer: freed by the last sync
    __syncthreads();
  }
  // tiles -> shared Gram matrix (reuses the staging space), mirrored
  double* G = sm;
#pragma unroll
  for (int J = 0; J < RB; ++J)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int j = 8 * J + 2 * q + e;
      if (J >= I1) {
        const int i = 8 * I1 + r;
        G[i * GS + j] = acc1[J][e];
        G[j * GS + i] = acc1[J][e];
      }
      if (J >= I2 && I2 != I1) {
        const int i = 8 * I2 + r;
        G[i * GS + j] = acc2[J][e];
        G[j * GS + i] = acc2[J][e];
      }
    }
  __syncthreads();
  const double dn = (double)N;
  double2* Rb = R + (size_t)b * M * M;
  for (int e = tid; e < M * M; e += T) {
    const int i = e / M, j = e - (e / M) * M;
    if (i > j) continue;
    const double re = G[i * GS + j] + G[(MP + i) * GS + MP + j];
    const double im = G[(MP + i) * GS + j] - G[i * GS + MP + j];
    const double2 v = make_double2(re / dn, i == j ? 0.0 : im / dn);
    Rb[(size_t)i * M + j] = v;
    if (i != j) Rb[(size_t)j * M + i] = make_double2(v.x, -v.y);
  }
}

// Version 2 (DOA_COVBIG2): tiles of R itself.  A warp owns TPW upper 8x8 tiles (I <= J) of the
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

template <int MP>
cudaError_t launch_covbig_t(const float* X, int64_t B, int64_t N, int M, double* R, cudaStream_t s) {
  const size_t smem = CovBig<MP>::SMEM;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(covbig_kernel<MP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  count_launch();
  covbig_kernel<MP><<<(unsigned)B, CovBig<MP>::WARPS * 32, smem, s>>>(reinterpret_cast<const float2*>(X), N, M,
                                                                      reinterpret_cast<double2*>(R));
  return cudaGetLastError();
}

}  // namespace

template <int MP>
cudaError_t launch_covbig2_t(const float* X, int64_t B, int64_t N, int M, double* R, cudaStream_t s) {
  const size_t smem = CovBig2<MP>::SMEM;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(covbig2_kernel<MP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  count_launch();
  covbig2_kernel<MP><<<(unsigned)B, CovBig2<MP>::T, smem, s>>>(reinterpret_cast<const float2*>(X), N, M,
                                                               reinterpret_cast<double2*>(R));
  return cudaGetLastError();
}

cudaError_t launch_covbig(const float* X, int64_t B, int64_t N, int M, double* R, cudaStream_t s) {
  if (DOA_COVBIG2) {
    if (M <= 32) return launch_covbig2_t<32>(X, B, N, M, R, s);
    return launch_covbig2_t<64>(X, B, N, M, R, s);
  }
  if (M <= 32) return launch_covbig_t<32>(X, B, N, M, R, s);
  return launch_covbig_t<64>(X, B, N, M, R, s);
}

}  // namespace doa
