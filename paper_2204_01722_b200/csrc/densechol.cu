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

// One CTA factors and inverts an n x n block (n <= kDenseBase), blocked by
// 4 x 4 tiles.  Thread (ti, tj) keeps tile (ti, tj) of the lower triangle in
// registers; the block is padded to 4 T rows with the identity (T = ceil(n/4)),
// which factors to itself and leaves the leading n x n part unchanged.
//   1. right-looking blocked Cholesky, tile step K: the diagonal tile's owner
//      factors it in registers (publishing L_KK, 1 / diag and a failed pivot);
//      the panel tiles below solve X L_KK^T = A_iK and publish X; every
//      trailing tile takes A_ij -= X_i X_j^T (64 FMAs);
//   2. L is staged in shared memory (and written back over A); the registers
//      restart from B = I for the forward elimination L W = I, tile step K:
//      the row-K tiles finalise W_Kj = L_KK^-1 B_Kj and publish them (double
//      buffered), every tile below takes B_ij -= L_iK W_Kj;
//   3. W (zero strict upper part) staged through shared memory to global.
// A failed pivot (a_kk <= 0, the potrf convention) sets *info = k + 1.
__global__ void __launch_bounds__(kBaseThreads, 1) chol_inv_base_kernel(double* A, int lda, double* W,
                                                                        int ldw, int n, int* info) {
  extern __shared__ double sm[];
  const int LD = n | 1;
  constexpr int kMax = kTile * kTiles;
  double* pan = sm + (size_t)n * LD;  // panel X: [kMax][4]
  double* rowb = pan + kMax * kTile;  // W row tiles, two buffers [2][4][kMax]
  double* dia = rowb + 2 * kTile * kMax;  // L_KK (16) + its reciprocal diagonal (4)
  double* rinv = dia + 20;                // 1 / L_kk (kMax)
  __shared__ int fail;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ti = tid / kTiles, tj = tid % kTiles;
  const int T = (n + kTile - 1) / kTile;
  const bool active = ti >= tj && ti < T;
  if (tid == 0) fail = 0;
  for (int c = warp; c < n; c += kBaseThreads / 32)
    for (int r = c + lane; r < n; r += 32) sm[c * LD + r] = A[r + (size_t)c * lda];
  __syncthreads();
  double e[kTile][kTile];
#pragma unroll
  for (int a = 0; a < kTile; ++a)
#pragma unroll
    for (int b = 0; b < kTile; ++b) {
      const int i = kTile * ti + a, j = kTile * tj + b;
      e[a][b] = !active || i < j ? 0.0 : (i < n ? sm[j * LD + i] : (i == j ? 1.0 : 0.0));
    }
  for (int K = 0; K < T; ++K) {
    if (ti == K && tj == K) {  // factor the diagonal tile
#pragma unroll
      for (int c = 0; c < kTile; ++c) {
        const double d = e[c][c];
        if (!(d > 0.0) && fail == 0) fail = kTile * K + c + 1;
        const double r = sqrt(d), ir = 1.0 / r;
        e[c][c] = r;
        dia[16 + c] = ir;
#pragma unroll
        for (int a = c + 1; a < kTile; ++a) e[a][c] *= ir;
#pragma unroll
        for (int b = c + 1; b < kTile; ++b)
#pragma unroll
          for (int a = b; a < kTile; ++a) e[a][b] -= e[a][c] * e[b][c];
      }
#pragma unroll
      for (int a = 0; a < kTile; ++a)
#pragma unroll
        for (int b = 0; b < kTile; ++b) dia[a * kTile + b] = e[a][b];
    }
    __syncthreads();
    if (fail) {  // uniform
      if (tid == 0) atomicCAS(info, 0, fail);
      return;
    }
    if (active && tj == K && ti > K) {  // X = A_iK L_KK^-T, row by row
#pragma unroll
      for (int a = 0; a < kTile; ++a) {
#pragma unroll
        for (int b = 0; b < kTile; ++b) {
          double x = e[a][b];
#pragma unroll
          for (int c = 0; c < b; ++c) x -= e[a][c] * dia[b * kTile + c];
          e[a][b] = x * dia[16 + b];
        }
#pragma unroll
        for (int b = 0; b < kTile; ++b) pan[(kTile * ti + a) * kTile + b] = e[a][b];
      }
    }
    __syncthreads();
    if (active && tj > K) {  // trailing update A_ij -= X_i X_j^T, one rank-1 term per c
#pragma unroll
      for (int c = 0; c < kTile; ++c) {
        double xi[kTile], xj[kTile];
#pragma unroll
        for (int a = 0; a < kTile; ++a) {
          xi[a] = pan[(kTile * ti + a) * kTile + c];
          xj[a] = pan[(kTile * tj + a) * kTile + c];
        }
#pragma unroll
        for (int a = 0; a < kTile; ++a)
#pragma unroll
          for (int b = 0; b < kTile; ++b) e[a][b] -= xi[a] * xj[b];
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
        const int i = kTile * ti + a, j = kTile * tj + b;
        if (i < n && i >= j) sm[j * LD + i] = e[a][b];
      }
  }
  __syncthreads();
  for (int c = warp; c < n; c += kBaseThreads / 32)
    for (int r = c + lane; r < n; r += 32) A[r + (size_t)c * lda] = sm[c * LD + r];
  for (int k = tid; k < kMax; k += kBaseThreads) rinv[k] = k < n ? 1.0 / sm[k * LD + k] : 1.0;
  // L entry (i, j), identity padding beyond n
  auto Lat = [&](int i, int j) { return i < n && j < n ? sm[j * LD + i] : (i == j ? 1.0 : 0.0); };
#pragma unroll
  for (int a = 0; a < kTile; ++a)
#pragma unroll
    for (int b = 0; b < kTile; ++b) e[a][b] = active && kTile * ti + a == kTile * tj + b ? 1.0 : 0.0;
  __syncthreads();
  for (int K = 0; K < T; ++K) {
    double* rb = rowb + (K & 1) * kTile * kMax;
    if (active && ti == K) {  // W_Kj = L_KK^-1 B_Kj, column by column
#pragma unroll
      for (int b = 0; b < kTile; ++b) {
#pragma unroll
        for (int a = 0; a < kTile; ++a) {
          double w = e[a][b];
#pragma unroll
          for (int c = 0; c < a; ++c) w -= Lat(kTile * K + a, kTile * K + c) * e[c][b];
          e[a][b] = w * rinv[kTile * K + a];
        }
      }
#pragma unroll
      for (int a = 0; a < kTile; ++a)
#pragma unroll
        for (int b = 0; b < kTile; ++b) rb[a * kMax + kTile * tj + b] = e[a][b];
    }
    __syncthreads();
    if (active && ti > K && tj <= K) {  // B_ij -= L_iK W_Kj, one rank-1 term per c
#pragma unroll
      for (int c = 0; c < kTile; ++c) {
        double l[kTile], w[kTile];
#pragma unroll
        for (int a = 0; a < kTile; ++a) {
          l[a] = Lat(kTile * ti + a, kTile * K + c);
          w[a] = rb[c * kMax + kTile * tj + a];
        }
#pragma unroll
        for (int a = 0; a < kTile; ++a)
#pragma unroll
          for (int b = 0; b < kTile; ++b) e[a][b] -= l[a] * w[b];
      }
    }
  }
  __syncthreads();  // L no longer read: stage W in its place
  if (active) {
#pragma unroll
    for (int a = 0; a < kTile; ++a)
#pragma unroll
      for (int b = 0; b < kTile; ++b) {
        const int i = kTile * ti + a, j = kTile * tj + b;
        if (i < n && j < n && i >= j) sm[j * LD + i] = e[a][b];
      }
  }
  __syncthreads();
  for (int c = warp; c < n; c += kBaseThreads / 32)
    for (int r = lane; r < n; r += 32) W[r + (size_t)c * ldw] = r >= c ? sm[c * LD + r] : 0.0;
}

size_t base_smem(int n) {
  constexpr int kMax = kTile * kTiles;
  return sizeof(double) * ((size_t)n * (n | 1) + kMax * kTile + 2 * kTile * kMax + 20 + kMax);
}

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

namespace {
__global__ void spd_fill_kernel(double* a, int n) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n * n; e += gridDim.x * blockDim.x) {
    const int r = e % n, c = e / n;
    a[e] = r == c ? (double)n : 1.0 / (1.0 + r + c);
  }
}
}  // namespace

void dense_chol_inv_warmup(cublasHandle_t h, cudaStream_t s) {
  constexpr int n = 2 * kDenseBase + 64;  // two recursion levels
  double *a = nullptr, *w = nullptr, *t = nullptr;
  int* info = nullptr;
  HXG_CUDA(cudaMalloc(&a, sizeof(double) * n * n));
  HXG_CUDA(cudaMalloc(&w, sizeof(double) * n * n));
  HXG_CUDA(cudaMalloc(&t, sizeof(double) * dense_chol_inv_scratch(n)));
  HXG_CUDA(cudaMalloc(&info, sizeof(int)));
  spd_fill_kernel<<<64, 256, 0, s>>>(a, n);
  HXG_CUDA(cudaMemsetAsync(w, 0, sizeof(double) * n * n, s));
  HXG_CUDA(cudaMemsetAsync(info, 0, sizeof(int), s));
  dense_chol_inv(h, s, a, n, w, n, n, info, t);
  HXG_CUDA(cudaStreamSynchronize(s));
  cudaFree(a);
  cudaFree(w);
  cudaFree(t);
  cudaFree(info);
}

}  // namespace hxg
