// Dense Cholesky + inverse factor (see densechol.hpp).
#include "densechol.hpp"

#include <cmath>

#include "common.hpp"

namespace hxg {

namespace {

// 32 x 32 threads, each owning one 4 x 4 tile of the (<= 128)^2 block.
constexpr int kTile = 4;
constexpr int kTiles = 32;
constexpr int kBaseThreads = kTiles * kTiles;
static_assert(kDenseBase <= kTile * kTiles, "dense base block larger than the thread tile grid");

void cublas_ok(cublasStatus_t st, const char* what) {
  if (st != CUBLAS_STATUS_SUCCESS) throw Error(HXG_ERR_CUDA, std::string("cuBLAS ") + what + " failed");
}

// One CTA factors and inverts an n x n block (n <= kDenseBase).  Thread
// (ti, tj) keeps the 4 x 4 tile (rows 4 ti.., columns 4 tj..) of the lower
// triangle in registers; every step is one barrier:
//   1. right-looking Cholesky, step k: the owners of column k publish it
//      (a double-buffered shared vector), every trailing entry i >= j > k
//      takes a_ij -= a_ik a_jk / a_kk, and the column owners finalise
//      l_kk = sqrt(a_kk), l_ik = a_ik / l_kk;
//   2. L is staged in shared memory (written back over A) and the registers
//      restart from B = I: forward elimination L W = I, step k: the owners of
//      row k finalise W_kj = B_kj / L_kk (j <= k) and publish the row, every
//      entry below takes B_ij -= L_ik W_kj;
//   3. W (zero strict upper part) staged through shared memory to global.
// A failed pivot (a_kk <= 0, the potrf convention) sets *info = k + 1.
__global__ void __launch_bounds__(kBaseThreads, 1) chol_inv_base_kernel(double* A, int lda, double* W,
                                                                        int ldw, int n, int* info) {
  extern __shared__ double sm[];
  const int LD = n | 1;
  double* vec = sm + (size_t)n * LD;  // two 128-entry buffers
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ti = tid / kTiles, tj = tid % kTiles;
  const int r0 = kTile * ti, c0 = kTile * tj;
  const bool active = ti >= tj && c0 < n;
  // coalesced load of the lower triangle, then each thread takes its tile
  for (int c = warp; c < n; c += kBaseThreads / 32)
    for (int r = c + lane; r < n; r += 32) sm[c * LD + r] = A[r + (size_t)c * lda];
  __syncthreads();
  double e[kTile][kTile];
#pragma unroll
  for (int a = 0; a < kTile; ++a)
#pragma unroll
    for (int b = 0; b < kTile; ++b) {
      const int i = r0 + a, j = c0 + b;
      e[a][b] = active && i < n && i >= j ? sm[j * LD + i] : 0.0;
    }
  for (int k = 0; k < n; ++k) {
    double* cb = vec + (k & 1) * 128;
    const int tk = k / kTile, kc = k % kTile;
    if (active && tj == tk) {
#pragma unroll
      for (int a = 0; a < kTile; ++a)
#pragma unroll
        for (int b = 0; b < kTile; ++b)
          if (b == kc && r0 + a >= k && r0 + a < n) cb[r0 + a] = e[a][b];
    }
    __syncthreads();
    const double d = cb[k];
    if (!(d > 0.0)) {  // uniform: every thread read the same pivot
      if (tid == 0) atomicCAS(info, 0, k + 1);
      return;
    }
    if (active && ti >= tk) {
      const double rd = 1.0 / d;
      double li[kTile], lj[kTile];
#pragma unroll
      for (int a = 0; a < kTile; ++a) li[a] = r0 + a > k && r0 + a < n ? cb[r0 + a] * rd : 0.0;
#pragma unroll
      for (int b = 0; b < kTile; ++b) lj[b] = c0 + b > k && c0 + b < n ? cb[c0 + b] : 0.0;
#pragma unroll
      for (int a = 0; a < kTile; ++a)
#pragma unroll
        for (int b = 0; b < kTile; ++b)
          if (c0 + b > k && r0 + a >= c0 + b) e[a][b] -= li[a] * lj[b];
      if (tj == tk) {
        const double r = sqrt(d);
#pragma unroll
        for (int a = 0; a < kTile; ++a)
#pragma unroll
          for (int b = 0; b < kTile; ++b)
            if (b == kc && r0 + a >= k && r0 + a < n) e[a][b] = r0 + a == k ? r : cb[r0 + a] / r;
      }
    }
  }
  // L -> shared memory (kept for the inversion) and back over A
  __syncthreads();
  if (active) {
#pragma unroll
    for (int a = 0; a < kTile; ++a)
#pragma unroll
      for (int b = 0; b < kTile; ++b) {
        const int i = r0 + a, j = c0 + b;
        if (i < n && i >= j) sm[j * LD + i] = e[a][b];
      }
  }
  __syncthreads();
  for (int c = warp; c < n; c += kBaseThreads / 32)
    for (int r = c + lane; r < n; r += 32) A[r + (size_t)c * lda] = sm[c * LD + r];
#pragma unroll
  for (int a = 0; a < kTile; ++a)
#pragma unroll
    for (int b = 0; b < kTile; ++b) e[a][b] = r0 + a == c0 + b ? 1.0 : 0.0;
  for (int k = 0; k < n; ++k) {
    double* rb = vec + (k & 1) * 128;
    const int tk = k / kTile, kc = k % kTile;
    if (active && ti == tk) {
      const double lkk = sm[k * LD + k];
#pragma unroll
      for (int a = 0; a < kTile; ++a)
#pragma unroll
        for (int b = 0; b < kTile; ++b)
          if (a == kc && c0 + b <= k) {
            const double w = e[a][b] / lkk;
            e[a][b] = w;
            rb[c0 + b] = w;
          }
    }
    __syncthreads();
    if (active && ti >= tk) {
      double lik[kTile], wk[kTile];
#pragma unroll
      for (int a = 0; a < kTile; ++a) lik[a] = r0 + a > k && r0 + a < n ? sm[k * LD + r0 + a] : 0.0;
#pragma unroll
      for (int b = 0; b < kTile; ++b) wk[b] = c0 + b <= k ? rb[c0 + b] : 0.0;
#pragma unroll
      for (int a = 0; a < kTile; ++a)
#pragma unroll
        for (int b = 0; b < kTile; ++b)
          if (r0 + a > k && c0 + b <= k) e[a][b] -= lik[a] * wk[b];
    }
  }
  __syncthreads();  // L no longer read: stage W in its place
  if (active) {
#pragma unroll
    for (int a = 0; a < kTile; ++a)
#pragma unroll
      for (int b = 0; b < kTile; ++b) {
        const int i = r0 + a, j = c0 + b;
        if (i < n && i >= j) sm[j * LD + i] = e[a][b];
      }
  }
  __syncthreads();
  for (int c = warp; c < n; c += kBaseThreads / 32)
    for (int r = lane; r < n; r += 32) W[r + (size_t)c * ldw] = r >= c ? sm[c * LD + r] : 0.0;
}

size_t base_smem(int n) { return sizeof(double) * ((size_t)n * (n | 1) + 256); }

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
