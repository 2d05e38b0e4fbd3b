// SURVEY §8(f) NEXT-2, tensor-core variant: the paper's direct form f = sum_j |x_j^H a(theta)|^2 (Table
// 2 Step-5; the noise-subspace vectors of Table 3, as in csrc/scan_fp32.cu) as a GEMM on
// the 5th-generation tensor cores — tcgen05.mma kind::tf32 with the accumulator in TMEM, each fp32
// operand split into a tf32 head and tail (3xTF32: A_hi B_hi + A_hi B_lo + A_lo B_hi, ~fp32 accuracy).
// Selected with doa_plan_set_engine(plan, DOA_ENGINE_DIRECT_TF32X3).  An A/B engine for evidence, like
// the FP32-pipe one: tcgen05 has no fp64 kinds, so the product path stays on the FP64 tensor pipe.
//
// GEMM per CTA and angle tile (real-ified complex product, K = 32 = [Re; Im] of M <= 16 elements):
//   A (M_mma = 128 rows = angles)           row i:  [cos(pi m u_i) | -sin(pi m u_i)],  m < 16
//   B (N_mma = 256 rows = 8 frames x 16 vector slots x {re, im})
//        (f, j, re): [Re x_j | Im x_j],  (f, j, im): [-Im x_j | Re x_j]      (slots j >= nv: zero)
//   D[i][(f, j, c)] = Re / Im of x_j^H a(theta_i);   f(theta_i, frame f) = sum_{j, c} D^2
// A CTA keeps its 8 frames' B operand in shared memory and sweeps every angle tile, generating A on
// the fly; thread i of the 4 epilogue warps owns TMEM lane i (one angle) and sums its row's 32
// columns per frame — no cross-lane reduction.  Warp w covers 32 consecutive angles, 30 of them
// decided (windows advance by 30), so the peak test needs only in-warp shuffles.
// Operands in shared memory use the canonical K-major no-swizzle UMMA layout: 8-row x 16-byte core
// matrices, K chunks of 16 bytes at LBO = 128 B, 8-row groups at SBO = 1 KB.
#include <cfloat>
#include <cstdint>

#include "doa_internal.cuh"

namespace doa {
namespace {

constexpr int kTcRows = 128;              // angle rows per tile (UMMA M)
constexpr int kTcCols = 256;              // (frame, slot, re/im) columns (UMMA N)
constexpr int kTcFrames = 8;              // frames per CTA
constexpr int kTcWin = 30;                // decided angles per warp window
constexpr int kTcThreads = 128;
constexpr uint32_t kTcTmemCols = 256;

// canonical K-major no-swizzle layout: element (row, k) of a K = 32 fp32 operand
__device__ __forceinline__ uint32_t kmaj_off(int row, int k) {
  return (uint32_t)((row >> 3) * 1024 + (k >> 2) * 128 + (row & 7) * 16 + (k & 3) * 4);
}

__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);            // start address
  d |= (uint64_t)(128 >> 4) << 16;                   // leading byte offset: next 16-byte K chunk
  d |= (uint64_t)(1024 >> 4) << 32;                  // stride byte offset: next 8-row group
  d |= (uint64_t)1 << 46;                            // descriptor version (sm_100)
  return d;                                          // base offset 0, layout SWIZZLE_NONE (0)
}

// instruction descriptor: kind::tf32, D fp32, A/B tf32, both K-major, N = 256, M = 128
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(kTcCols >> 3) << 17) |
                            ((uint32_t)(kTcRows >> 4) << 24);

__device__ __forceinline__ uint32_t to_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n\t}\n"
      :
      : "r"(tmem_d), "l"(a), "l"(b), "r"(kIdesc), "r"(accumulate), "r"(0), "r"(0), "r"(0), "r"(0));
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ bool mbar_try_wait(uint32_t mbar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}\n"
      : "=r"(ok)
      : "r"(mbar), "r"(parity)
      : "memory");
  return ok != 0;
}

__global__ void __launch_bounds__(kTcThreads, 2) scan_tc_kernel(const float2* __restrict__ X, int64_t B, int K, int nv,
                                                                int M, double dl, double theta0, double dtheta, int L,
                                                                bool sym, int cap, int32_t* __restrict__ cnt,
                                                                int32_t* __restrict__ cidx, double* __restrict__ cf,
                                                                float* __restrict__ P) {
  extern __shared__ __align__(1024) uint8_t tc_smem[];
  // [A_hi 16 KB][A_lo 16 KB][B_hi 32 KB][B_lo 32 KB]
  uint8_t* a_hi = tc_smem;
  uint8_t* a_lo = tc_smem + 16384;
  uint8_t* b_hi = tc_smem + 32768;
  uint8_t* b_lo = tc_smem + 65536;
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base_s;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t b0 = (int64_t)blockIdx.x * kTcFrames;
  const int nb = (int)(B - b0 < kTcFrames ? B - b0 : kTcFrames);
  const uint32_t mbar_a = (uint32_t)__cvta_generic_to_shared(&mbar);

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n"
                 :: "r"((uint32_t)__cvta_generic_to_shared(&tmem_base_s)), "r"(kTcTmemCols) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" :: "r"(mbar_a) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  // B operand: this CTA's frames, split into tf32 head / tail (zero for missing frames and slots)
  for (int e = tid; e < kTcCols * 32; e += kTcThreads) {
    const int row = e >> 5, k = e & 31;
    const int f = row >> 5, j = (row >> 1) & 15, c = row & 1, m = k & 15, part = k >> 4;
    float v = 0.f;
    if (f < nb && j < nv && m < M) {
      const float2 x = X[((size_t)(b0 + f) * K + j) * M + m];
      v = c == 0 ? (part == 0 ? x.x : x.y) : (part == 0 ? -x.y : x.x);
    }
    const uint32_t h = to_tf32(v);
    const uint32_t l = to_tf32(v - __uint_as_float(h));
    *reinterpret_cast<uint32_t*>(b_hi + kmaj_off(row, k)) = h;
    *reinterpret_cast<uint32_t*>(b_lo + kmaj_off(row, k)) = l;
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = tmem_base_s;
  const uint32_t sa_hi = (uint32_t)__cvta_generic_to_shared(a_hi), sa_lo = (uint32_t)__cvta_generic_to_shared(a_lo);
  const uint32_t sb_hi = (uint32_t)__cvta_generic_to_shared(b_hi), sb_lo = (uint32_t)__cvta_generic_to_shared(b_lo);

  const int nwin = (L + kTcWin - 1) / kTcWin;            // windows of 30 decided angles
  const int ntile = (nwin + 3) / 4;                      // 4 windows (warps) per tile
  for (int t = 0; t < ntile; ++t) {
    // A operand: row = tid, angle of window 4t + warp at position lane (positions 0, 31 are halo)
    const int w = 4 * t + warp;
    const int base = w * kTcWin - 1;
    int ia = base + lane;
    ia = ia < 0 ? 0 : (ia >= L ? L - 1 : ia);
    {
      const double u = grid_u(ia, theta0, dtheta, dl, L, sym);
      float row[32];                                    // [cos(pi m u) | -sin(pi m u)], m < 16
#pragma unroll
      for (int m = 0; m < 16; ++m) {
        float sn = 0.f, cs = 0.f;
        if (m < M) {
          double r = (double)m * u;                     // exact-multiple argument, reduced mod 2 in fp64
          r -= 2.0 * rint(0.5 * r);
          sincospif((float)r, &sn, &cs);
        }
        row[m] = cs;
        row[16 + m] = -sn;
      }
      // one 16-byte store per K chunk: the 8 lanes of a quarter-warp write 8 rows of one core
      // matrix (128 contiguous bytes) - conflict-free
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        uint32_t h[4], l[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          h[q] = to_tf32(row[4 * c + q]);
          l[q] = to_tf32(row[4 * c + q] - __uint_as_float(h[q]));
        }
        *reinterpret_cast<uint4*>(a_hi + kmaj_off(tid, 4 * c)) = make_uint4(h[0], h[1], h[2], h[3]);
        *reinterpret_cast<uint4*>(a_lo + kmaj_off(tid, 4 * c)) = make_uint4(l[0], l[1], l[2], l[3]);
      }
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");   // generic smem writes -> tensor core
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {                   // K = 32 as 4 steps of 8 (32 bytes)
        const uint32_t ko = kk * 256;
        mma_tf32(tmem, smem_desc(sa_hi + ko), smem_desc(sb_hi + ko), kk > 0);
        mma_tf32(tmem, smem_desc(sa_hi + ko), smem_desc(sb_lo + ko), 1);
        mma_tf32(tmem, smem_desc(sa_lo + ko), smem_desc(sb_hi + ko), 1);
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
                   :: "r"(mbar_a) : "memory");
    }
    while (!mbar_try_wait(mbar_a, (uint32_t)(t & 1))) {
    }
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    // epilogue: lane = angle row; columns 32 f .. 32 f + 31 = frame f's (slot, re/im) values
    const uint32_t trow = tmem + ((uint32_t)(32 * warp) << 16);
    for (int f = 0; f < nb; ++f) {
      float v[32];
      tmem_ld32(trow + 32 * f, v);
      float acc = 0.f;
#pragma unroll
      for (int q = 0; q < 32; ++q) acc = fmaf(v[q], v[q], acc);
      const long long vb = floor_bits(__double_as_longlong((double)acc));
      const long long vl = __shfl_up_sync(0xffffffffu, vb, 1), vr = __shfl_down_sync(0xffffffffu, vb, 1);
      const int i = base + lane;
      const bool inside = lane > 0 && lane < 31 && i >= 0 && i < L;
      const int64_t b = b0 + f;
      if (P && inside) P[(size_t)b * L + i] = to_p32(__longlong_as_double(vb));
      if (inside && i >= 1 && i <= L - 2 && vb < vl && vb <= vr) {       // Q9 / Q10
        const int slot = atomicAdd(cnt + b, 1);
        if (slot < cap) {
          cidx[(size_t)b * cap + slot] = i;
          cf[(size_t)b * cap + slot] = __longlong_as_double(vb);
        }
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();                                     // TMEM and A may be overwritten now
  }
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" :: "r"(tmem), "r"(kTcTmemCols) : "memory");
}

}  // namespace

cudaError_t launch_scan_tc(const doa_plan_s* p, int64_t B, float* P, cudaStream_t s) {
  if (B <= 0) return cudaSuccess;
  const int K = p->M - p->D;
  const int nv = (p->alg == DOA_ALG_MUSIC || p->alg == DOA_ALG_EV) ? K : 1;
  const size_t smem = 98304;
  kernel_occupancy(scan_tc_kernel, kTcThreads, smem);            // sets the > 48 KB smem attribute
  count_launch();
  scan_tc_kernel<<<(unsigned)((B + kTcFrames - 1) / kTcFrames), kTcThreads, smem, s>>>(
      reinterpret_cast<const float2*>(p->x32), B, K, nv, p->M, p->dl, p->theta0, p->dtheta, (int)p->L, p->sym != 0,
      p->cap, p->cnt, p->cand_idx, p->cand_f, P);
  return cudaGetLastError();
}

}  // namespace doa
