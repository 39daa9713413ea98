// Dense Cholesky with the inverse factor, on device, for the coarse solvers
// (the pivot blocks of the nested-dissection fronts, the dense coarse mode
// and the h-multigrid bottom).  The reference factors its coarse matrix with
// Eigen's SimplicialLLT (coarse_solver.hpp:18-30); this is the dense kernel
// underneath the device multifrontal replacement.
//
//   dense_chol_inv:  A (lower, leading dimension lda) is overwritten by L
//   (A = L L^T, the strict upper part untouched) and W (n x n, ldw) receives
//   L^-1 with a zero strict upper part.  Recursive blocked form,
//     [A11 .; A21 A22]:  (L11, W11) = rec(A11);  L21 = A21 W11^T;
//     S = A22 - L21 L21^T;  (L22, W22) = rec(S);  W21 = -W22 (L21 W11),
//   with the level-3 products on cuBLAS DGEMM / DSYRK (FP64 tensor cores)
//   and the diagonal blocks of <= kDenseBase rows factored and inverted by one
//   hand-written CTA in shared memory (chol_inv_base_kernel).
#pragma once

#include <cublas_v2.h>
#include <cuda_runtime.h>

#include <cstddef>

namespace hxg {

#ifndef HXG_DENSE_BASE
#define HXG_DENSE_BASE 128
#endif
constexpr int kDenseBase = HXG_DENSE_BASE;

// Scratch (doubles) dense_chol_inv needs for an n x n block.
size_t dense_chol_inv_scratch(int n);

// info (device int): set to the 1-based index of the first non-positive pivot
// of the failing diagonal block if it is still 0 (the potrf convention).
// The cuBLAS handle must be bound to stream s.
void dense_chol_inv(cublasHandle_t h, cudaStream_t s, double* A, int lda, double* W, int ldw,
                    int n, int* info, double* scratch);

// One small eager factorisation through every code path (kernel attributes,
// lazily loaded library kernels), so later calls can be graph-captured.
void dense_chol_inv_warmup(cublasHandle_t h, cudaStream_t s);

// The shared-memory kernel alone (n <= kDenseBase).
void dense_chol_inv_base(cudaStream_t s, double* A, int lda, double* W, int ldw, int n, int* info);

}  // namespace hxg
