// S2 dispatch — batched Hermitian eigendecomposition (Table 2 Step-2 `jsvd`; Q3):
//   M <= 16        eig16h_kernel (csrc/eig16.cu): two matrices per warp, one per 16-lane half
//                  (eig16_kernel, one warp per matrix, with DOA_EIG_HALF=0)
//   16 < M <= 64   eigN_kernel<32|64> (csrc/eign.cu): one CTA per matrix
// Both are the parallel (circle-method round robin) cyclic Jacobi with a fixed-slot caterpillar
// permutation; see the kernel files.
#include "doa_internal.cuh"

namespace doa {

cudaError_t launch_eig16(const double* R, int64_t B, int M, double* lam, double* V, int32_t* info, cudaStream_t s);
cudaError_t launch_eigN(const double* R, int64_t B, int M, double* lam, double* V, int32_t* info, cudaStream_t s);

cudaError_t launch_eig(const double* R, int64_t B, int M, double* lam, double* V, int32_t* info, cudaStream_t s) {
  if (M <= 16) return launch_eig16(R, B, M, lam, V, info, s);
  return launch_eigN(R, B, M, lam, V, info, s);
}

}  // namespace doa
