// S1 for M <= 16 on the FP64 tensor pipe: R = (1/N) X X^H (Eq. 3; Table 2 Step-1).
//
// With Y = [Re X^T; Im X^T] (2*16 x N, rows padded to 16 per half), the real Gram matrix
// G = Y Y^T gives R = (G_rr + G_ii) + j (G_ir - G_ri) blockwise.  One warp per frame computes the
// ten 8x8 tiles of the upper block triangle of G with mma.sync m8n8k4 f64: for k-step n0 every
// lane loads the two complex64 samples x_{n0+q}[r] and x_{n0+q}[8+r] (r = lane/4, q = lane%4),
// converts them once, and the same four doubles serve as both the A fragment (row block I) and the
// B fragment (column block J) of every tile (I, J).  fp32 products are exact in fp64; sums are
// fp64 in the DMMA's fixed order (deterministic).  The tiles are then mirrored through shared
// memory and combined into the full Hermitian R (exact conjugate mirror, real diagonal).
#include "doa_internal.cuh"

namespace doa {
namespace {

constexpr int kCovWarps = 4;
constexpr int kGld = 33;          // smem row stride of the 32x32 Gram matrix (doubles)

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// tile list (I <= J) over the 4 row blocks {Re 0-7, Re 8-15, Im 0-7, Im 8-15}
__device__ constexpr int kTI[10] = {0, 0, 1, 2, 2, 3, 0, 0, 1, 1};
__device__ constexpr int kTJ[10] = {0, 1, 1, 2, 3, 3, 2, 3, 2, 3};

// The ten upper Gram tiles over snapshots [n_begin, n_end) (n_begin a multiple of 4), one warp.
__device__ __forceinline__ void gram_tiles(const float2* __restrict__ Xb, int64_t n_begin, int64_t n_end, int M,
                                           int lane, double (&acc)[10][2]) {
  const int r = lane >> 2, q = lane & 3;
  const bool lo_ok = r < M, hi_ok = r + 8 < M;
#pragma unroll
  for (int t = 0; t < 10; ++t) { acc[t][0] = 0.0; acc[t][1] = 0.0; }
  constexpr int U = 8;                       // k-steps in flight per warp
  int64_t n0 = n_begin;
  for (; n0 + 4 * U <= n_end; n0 += 4 * U) {
    float2 x0[U], x1[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const float2* row = Xb + (size_t)(n0 + 4 * u + q) * M;
      x0[u] = lo_ok ? __ldg(row + r) : make_float2(0.f, 0.f);
      x1[u] = hi_ok ? __ldg(row + r + 8) : make_float2(0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const double y[4] = {(double)x0[u].x, (double)x1[u].x, (double)x0[u].y, (double)x1[u].y};
#pragma unroll
      for (int t = 0; t < 10; ++t) dmma(acc[t][0], acc[t][1], y[kTI[t]], y[kTJ[t]]);
    }
  }
  for (; n0 < n_end; n0 += 4) {              // ragged tail
    const int64_t n = n0 + q;
    float2 a0 = make_float2(0.f, 0.f), a1 = make_float2(0.f, 0.f);
    if (n < n_end) {
      const float2* row = Xb + (size_t)n * M;
      if (lo_ok) a0 = __ldg(row + r);
      if (hi_ok) a1 = __ldg(row + r + 8);
    }
    const double y[4] = {(double)a0.x, (double)a1.x, (double)a0.y, (double)a1.y};
#pragma unroll
    for (int t = 0; t < 10; ++t) dmma(acc[t][0], acc[t][1], y[kTI[t]], y[kTJ[t]]);
  }
}

// Gram tiles -> mirrored smem Gram G -> Hermitian R (/N, exact conjugate mirror, real diagonal)
__device__ __forceinline__ void gram_to_r(const double (&acc)[10][2], double* G, int lane, int64_t N, int M,
                                          double2* __restrict__ Rb) {
  const int r = lane >> 2, q = lane & 3;
#pragma unroll
  for (int t = 0; t < 10; ++t) {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int i = 8 * kTI[t] + r, j = 8 * kTJ[t] + 2 * q + e;
      G[i * kGld + j] = acc[t][e];
      G[j * kGld + i] = acc[t][e];
    }
  }
  __syncwarp();
  const double dn = (double)N;
  for (int e = lane; e < M * M; e += 32) {
    const int i = e / M, j = e - (e / M) * M;
    if (i > j) continue;
    const double re = G[i * kGld + j] + G[(16 + i) * kGld + 16 + j];
    const double im = G[(16 + i) * kGld + j] - G[i * kGld + 16 + j];
    const double2 v = make_double2(re / dn, i == j ? 0.0 : im / dn);
    Rb[(size_t)i * M + j] = v;
    if (i != j) Rb[(size_t)j * M + i] = make_double2(v.x, -v.y);
  }
}

__global__ void __launch_bounds__(kCovWarps * 32) cov16_kernel(const float2* __restrict__ X, int64_t B, int64_t N,
                                                             int M, double2* __restrict__ R) {
  __shared__ double Gs[kCovWarps][32 * kGld];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t b = (int64_t)blockIdx.x * kCovWarps + warp;
  if (b >= B) return;
  const float2* Xb = X + (size_t)b * N * M;
  double acc[10][2];
  gram_tiles(Xb, 0, N, M, lane, acc);

  gram_to_r(acc, Gs[warp], lane, N, M, R + (size_t)b * M * M);
}


// Split-N variant for long frames (N > 256): a CTA of SW = min(8, ceil(N/128)) warps per frame,
// warp w accumulating the snapshots [w Nw, (w+1) Nw) (Nw a multiple of 4); the partial tiles are
// summed in warp order through shared memory (fixed order: deterministic, and the split depends
// only on N, so a frame's R does not depend on the batch).  Cuts the single-frame latency of
// C2/C3 (N = 1024) roughly by SW.
constexpr int kSplitMax = 8;
__global__ void __launch_bounds__(kSplitMax * 32) cov16_split_kernel(const float2* __restrict__ X, int64_t N, int M,
                                                                    int SW, double2* __restrict__ R) {
  __shared__ double part[kSplitMax][10][64];      // the reduced Gram G reuses it afterwards
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t b = blockIdx.x;
  const float2* Xb = X + (size_t)b * N * M;
  const int64_t Nw = ((N + SW - 1) / SW + 3) / 4 * 4;
  const int64_t n_begin = warp * Nw, n_end = n_begin + Nw < N ? n_begin + Nw : N;
  double acc[10][2];
  gram_tiles(Xb, n_begin < N ? n_begin : N, n_end > n_begin ? n_end : n_begin, M, lane, acc);
#pragma unroll
  for (int t = 0; t < 10; ++t) {
    part[warp][t][2 * lane] = acc[t][0];
    part[warp][t][2 * lane + 1] = acc[t][1];
  }
  __syncthreads();
  if (warp != 0) return;
#pragma unroll
  for (int t = 0; t < 10; ++t) {
    double s0 = part[0][t][2 * lane], s1 = part[0][t][2 * lane + 1];
    for (int w = 1; w < SW; ++w) { s0 += part[w][t][2 * lane]; s1 += part[w][t][2 * lane + 1]; }
    acc[t][0] = s0;
    acc[t][1] = s1;
  }
  __syncwarp();
  gram_to_r(acc, &part[0][0][0], lane, N, M, R + (size_t)b * M * M);
}

// Small batches of long frames (B <= kDirectMaxB, N > 256; the single-frame configs C2/C3): the
// frame's snapshots are spread over SC <= 16 CTAs of 8 warps (32 snapshots per warp up to N = 4096)
// so that a single frame uses SC SMs instead of one.  Warp w of CTA c accumulates the snapshot range
// [(8c + w) Nw, (8c + w + 1) Nw); each CTA sums its warps' tiles in warp order and writes one partial
// Gram to the workspace; the CTA that takes the last ticket of the frame sums the SC partials in CTA
// order (fixed order: deterministic; the split depends only on N) and writes R.  The ticket is reset
// for the next call.  Rounds differently from the batched kernels (a different summation order).
constexpr int kMultiCtas = 16;
// snapshots per warp: 32 (one 8-k-step batch of loads in flight, gram_tiles' main loop) while
// 16 CTAs of 8 warps suffice, else the next multiple of 32
__host__ __device__ inline int64_t cov_multi_chunk(int64_t N) {
  const int64_t per = (N + kMultiCtas * kSplitMax - 1) / (kMultiCtas * kSplitMax);
  return per <= 32 ? 32 : (per + 31) / 32 * 32;
}
__global__ void __launch_bounds__(kSplitMax * 32) cov16_multi_kernel(const float2* __restrict__ X, int64_t N, int M,
                                                                    int SC, double* __restrict__ part,
                                                                    unsigned* __restrict__ ticket,
                                                                    double2* __restrict__ R) {
  __shared__ double red[kSplitMax][10][64];
  __shared__ unsigned last_s;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = blockIdx.x;
  const int64_t b = blockIdx.y;
  const float2* Xb = X + (size_t)b * N * M;
  const int64_t Nw = cov_multi_chunk(N);
  int64_t lo = ((int64_t)c * kSplitMax + warp) * Nw, hi = lo + Nw;
  lo = lo < N ? lo : N;                                   // warps past the end get an empty range
  hi = hi < N ? hi : N;
  double acc[10][2];
  gram_tiles(Xb, lo, hi, M, lane, acc);
#pragma unroll
  for (int t = 0; t < 10; ++t) {
    red[warp][t][2 * lane] = acc[t][0];
    red[warp][t][2 * lane + 1] = acc[t][1];
  }
  __syncthreads();
  double* pb = part + ((size_t)b * kMultiCtas + c) * 640;
  for (int e = threadIdx.x; e < 640; e += kSplitMax * 32) {
    const int t = e / 64, k = e - (e / 64) * 64;
    double sum = red[0][t][k];
    for (int w = 1; w < kSplitMax; ++w) sum += red[w][t][k];
    pb[e] = sum;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last_s = atomicAdd(ticket + b, 1u) == (unsigned)(SC - 1);
  __syncthreads();
  if (!last_s) return;
  __threadfence();
  const double* p0 = part + (size_t)b * kMultiCtas * 640;
  double* tot = &red[1][0][0];                           // 640 sums, then red[0] is gram_to_r's G
  for (int e = threadIdx.x; e < 640; e += kSplitMax * 32) {
    double v[kMultiCtas];
#pragma unroll
    for (int cc = 0; cc < kMultiCtas; ++cc) v[cc] = cc < SC ? __ldcg(p0 + (size_t)cc * 640 + e) : 0.0;
    double sum = v[0];
#pragma unroll
    for (int cc = 1; cc < kMultiCtas; ++cc)
      if (cc < SC) sum += v[cc];                          // CTA order
    tot[e] = sum;
  }
  __syncthreads();
  if (warp != 0) return;
#pragma unroll
  for (int t = 0; t < 10; ++t) {
    acc[t][0] = tot[t * 64 + 2 * lane];
    acc[t][1] = tot[t * 64 + 2 * lane + 1];
  }
  if (lane == 0) ticket[b] = 0u;                          // ready for the next call
  __syncwarp();                                           // tot (red[1..]) is read before G overwrites it
  gram_to_r(acc, &red[0][0][0], lane, N, M, R + (size_t)b * M * M);
}

}  // namespace

size_t cov_workspace_bytes() {
  return (size_t)kDirectMaxB * kMultiCtas * 640 * sizeof(double) + (size_t)kDirectMaxB * sizeof(unsigned);
}

cudaError_t launch_cov16(const float* X, int64_t B, int64_t N, int M, double* R, cudaStream_t s, void* ws) {
  count_launch();
  if (ws && B <= kDirectMaxB && N > 256) {
    const int64_t per_cta = cov_multi_chunk(N) * kSplitMax;
    const int SC = (int)((N + per_cta - 1) / per_cta);
    double* part = static_cast<double*>(ws);
    unsigned* ticket = reinterpret_cast<unsigned*>(part + (size_t)kDirectMaxB * kMultiCtas * 640);
    cov16_multi_kernel<<<dim3((unsigned)SC, (unsigned)B), kSplitMax * 32, 0, s>>>(
        reinterpret_cast<const float2*>(X), N, M, SC, part, ticket, reinterpret_cast<double2*>(R));
    return cudaGetLastError();
  }
  if (N > 256) {
    const int SW = (int)((N + 127) / 128 < kSplitMax ? (N + 127) / 128 : kSplitMax);
    cov16_split_kernel<<<(unsigned)B, SW * 32, 0, s>>>(reinterpret_cast<const float2*>(X), N, M, SW,
                                                       reinterpret_cast<double2*>(R));
    return cudaGetLastError();
  }
  cov16_kernel<<<(unsigned)((B + kCovWarps - 1) / kCovWarps), kCovWarps * 32, 0, s>>>(
      reinterpret_cast<const float2*>(X), B, N, M, reinterpret_cast<double2*>(R));
  return cudaGetLastError();
}

}  // namespace doa
