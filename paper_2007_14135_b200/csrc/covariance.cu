// S1 dispatch — sample covariance R = (1/N) X X^H (Eq. 3; Table 2 Step-1):
//   M <= 16        cov16_kernel (csrc/cov16.cu): one warp per frame, operands straight from HBM;
//                  N > 256: cov16_split_kernel (a CTA per frame), or — small batches with a
//                  workspace — cov16_multi_kernel (the frame spread over up to 16 CTAs)
//   16 < M <= 64   covbig2_kernel<32|64> (csrc/covbig.cu): one CTA per frame, smem-staged chunks
// All form the real Gram matrix of [Re X^T; Im X^T] on the FP64 tensor pipe (mma.sync m8n8k4).
#include "doa_internal.cuh"

namespace doa {

cudaError_t launch_cov16(const float* X, int64_t B, int64_t N, int M, double* R, cudaStream_t s, void* ws);
cudaError_t launch_covbig(const float* X, int64_t B, int64_t N, int M, double* R, cudaStream_t s);

cudaError_t launch_covariance(const float* X, int64_t B, int64_t N, int M, double* R, cudaStream_t s, void* ws) {
  if (M <= 16) return launch_cov16(X, B, N, M, R, s, ws);
  return launch_covbig(X, B, N, M, R, s);
}

}  // namespace doa
