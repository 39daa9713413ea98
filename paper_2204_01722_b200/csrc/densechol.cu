// Dense Cholesky + inverse factor (see densechol.hpp).
#include "densechol.hpp"

#include <cmath>

#include "common.hpp"

namespace hxg {

namespace {

constexpr int kBaseThreads = 512;
constexpr int kBaseWarps = kBaseThreads / 32;

void cublas_ok(cublasStatus_t st, const char* what) {
  if (st != CUBLAS_STATUS_SUCCESS) throw Error(HXG_ERR_CUDA, std::string("cuBLAS ") + what + " failed");
}

// One CTA factors and inverts an n x n block (n <= kDenseBase) held in shared
// memory, column-major with an odd stride (64-bit accesses along a row of
// lanes stay bank-conflict free):
//   1. right-looking Cholesky, column k: pivot, scale the column, rank-1
//      update of the trailing lower triangle (one warp per column, lanes down
//      the rows), L written back over A;
//   2. in-place inversion of L (the unblocked lower, non-unit trti2 order:
//      j = n-1 .. 0, column j below the diagonal = -(1 / L_jj) T x with T the
//      already inverted trailing block; one warp per row, lanes over the
//      columns, fixed-order butterfly), L^-1 written to W with zeros above.
__global__ void __launch_bounds__(kBaseThreads) chol_inv_base_kernel(double* A, int lda, double* W,
                                                                     int ldw, int n, int* info) {
  extern __shared__ double sm[];
  const int LD = n | 1;
  double* xs = sm + (size_t)n * LD;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int c = warp; c < n; c += kBaseWarps)
    for (int r = c + lane; r < n; r += 32) sm[c * LD + r] = A[r + (size_t)c * lda];
  __syncthreads();
  for (int k = 0; k < n; ++k) {
    const double d = sm[k * LD + k];
    if (!(d > 0.0)) {  // uniform: every thread read the same pivot
      if (tid == 0) atomicCAS(info, 0, k + 1);
      return;
    }
    const double r = sqrt(d), ri = 1.0 / r;
    __syncthreads();  // the pivot is read before it is overwritten
    if (tid == 0) sm[k * LD + k] = r;
    for (int i = k + 1 + tid; i < n; i += kBaseThreads) sm[k * LD + i] *= ri;
    __syncthreads();
    for (int j = k + 1 + warp; j < n; j += kBaseWarps) {
      const double ljk = sm[k * LD + j];
      for (int i = j + lane; i < n; i += 32) sm[j * LD + i] -= sm[k * LD + i] * ljk;
    }
    __syncthreads();
  }
  for (int c = warp; c < n; c += kBaseWarps)
    for (int r = c + lane; r < n; r += 32) A[r + (size_t)c * lda] = sm[c * LD + r];
  for (int j = n - 1; j >= 0; --j) {
    const int m = n - j - 1;
    const double inv = 1.0 / sm[j * LD + j];
    for (int i = tid; i < m; i += kBaseThreads) xs[i] = sm[j * LD + j + 1 + i];
    __syncthreads();
    for (int i = warp; i < m; i += kBaseWarps) {
      double acc = 0.0;
      for (int k = lane; k <= i; k += 32) acc += sm[(j + 1 + k) * LD + j + 1 + i] * xs[k];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) sm[j * LD + j + 1 + i] = -inv * acc;
    }
    if (tid == 0) sm[j * LD + j] = inv;
    __syncthreads();
  }
  for (int c = warp; c < n; c += kBaseWarps)
    for (int r = lane; r < n; r += 32) W[r + (size_t)c * ldw] = r >= c ? sm[c * LD + r] : 0.0;
}

size_t base_smem(int n) { return sizeof(double) * ((size_t)n * (n | 1) + n); }

}  // namespace

size_t dense_chol_inv_scratch(int n) {
  if (n <= kDenseBase) return 1;
  const size_t n1 = (size_t)((n / 2 + 31) / 32) * 32, n2 = (size_t)n - n1;
  return n1 * n2;  // the top split is the largest n2 x n1 product
}

void dense_chol_inv_base(cudaStream_t s, double* A, int lda, double* W, int ldw, int n, int* info) {
  if (n <= 0) return;
  if (n > kDenseBase) throw Error(HXG_ERR_INVALID_ARGUMENT, "dense_chol_inv_base: block too large");
  static bool attr = false;
  if (!attr) {
    HXG_CUDA(cudaFuncSetAttribute(chol_inv_base_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)base_smem(kDenseBase)));
    attr = true;
  }
  chol_inv_base_kernel<<<1, kBaseThreads, base_smem(n), s>>>(A, lda, W, ldw, n, info);
  HXG_CUDA(cudaGetLastError());
}

void dense_chol_inv(cublasHandle_t h, cudaStream_t s, double* A, int lda, double* W, int ldw, int n,
                    int* info, double* scratch) {
  if (n <= kDenseBase) {
    dense_chol_inv_base(s, A, lda, W, ldw, n, info);
    return;
  }
  const double one = 1.0, minus_one = -1.0, zero = 0.0;
  const int n1 = ((n / 2 + 31) / 32) * 32, n2 = n - n1;
  double *A21 = A + n1, *A22 = A + n1 + (size_t)n1 * lda;
  double *W21 = W + n1, *W22 = W + n1 + (size_t)n1 * ldw;
  dense_chol_inv(h, s, A, lda, W, ldw, n1, info, scratch);
  double* T = scratch;  // n2 x n1
  cublas_ok(cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_T, n2, n1, n1, &one, A21, lda, W, ldw, &zero, T, n2),
            "gemm (L21)");
  HXG_CUDA(cudaMemcpy2DAsync(A21, sizeof(double) * lda, T, sizeof(double) * n2, sizeof(double) * n2, n1,
                             cudaMemcpyDeviceToDevice, s));
  cublas_ok(cublasDsyrk(h, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, n2, n1, &minus_one, A21, lda, &one, A22, lda),
            "syrk");
  dense_chol_inv(h, s, A22, lda, W22, ldw, n2, info, scratch);
  cublas_ok(cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, n2, n1, n1, &one, A21, lda, W, ldw, &zero, T, n2),
            "gemm (L21 W11)");
  cublas_ok(cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, n2, n1, n2, &minus_one, W22, ldw, T, n2, &zero, W21, ldw),
            "gemm (W21)");
}

}  // namespace hxg
