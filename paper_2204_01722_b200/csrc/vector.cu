#include "vector.hpp"

#include "common.hpp"

namespace hxg {

namespace {

constexpr int kDotBlocks = 592;  // 4 x 148 SMs, fixed for determinism
constexpr int kDotThreads = 256;

__device__ __forceinline__ double block_sum(double v, double* sh) {
  // Fixed-order tree: warp shuffles then one warp over the warp sums.
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) sh[w] = v;
  __syncthreads();
  double r = 0.0;
  if (w == 0) {
    r = lane < (int)(blockDim.x >> 5) ? sh[lane] : 0.0;
    for (int o = 16; o > 0; o >>= 1) r += __shfl_down_sync(0xffffffffu, r, o);
  }
  return r;
}

__global__ void dot_stage1(const double* __restrict__ x, const double* __restrict__ y, long long n,
                           double* partial) {
  __shared__ double sh[32];
  // Contiguous chunk per block; grid-stride inside the chunk.
  long long chunk = (n + gridDim.x - 1) / gridDim.x;
  long long beg = blockIdx.x * chunk, end = beg + chunk < n ? beg + chunk : n;
  double s = 0.0;
  for (long long i = beg + threadIdx.x; i < end; i += blockDim.x) s += x[i] * y[i];
  double r = block_sum(s, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = r;
}

// Same partition and tree with the entries outside `mask` (0) skipped: the
// owned-entry dots of the partitioned solver.
__global__ void dot_stage1_masked(const double* __restrict__ x, const double* __restrict__ y,
                                  const uint8_t* __restrict__ mask, long long n, double* partial) {
  __shared__ double sh[32];
  long long chunk = (n + gridDim.x - 1) / gridDim.x;
  long long beg = blockIdx.x * chunk, end = beg + chunk < n ? beg + chunk : n;
  double s = 0.0;
  for (long long i = beg + threadIdx.x; i < end; i += blockDim.x)
    if (mask[i]) s += x[i] * y[i];
  double r = block_sum(s, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = r;
}

__global__ void dot_stage2(const double* partial, int m, double* out) {
  __shared__ double sh[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < m; i += blockDim.x) s += partial[i];
  double r = block_sum(s, sh);
  if (threadIdx.x == 0) *out = r;
}

inline int grid(long long n) {
  long long g = (n + 255) / 256;
  if (g > 148 * 32) g = 148 * 32;
  return g < 1 ? 1 : (int)g;
}

#define GRID_STRIDE(i, n) \
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < (n); i += (long long)gridDim.x * blockDim.x)

__global__ void k_sub_from(double* y, const double* b, long long n) { GRID_STRIDE(i, n) y[i] = b[i] - y[i]; }
__global__ void k_mask_zero(double* y, const uint8_t* m, long long n) {
  GRID_STRIDE(i, n) if (m[i]) y[i] = 0.0;
}
__global__ void k_mask_copy(double* y, const double* s, const uint8_t* m, long long n) {
  GRID_STRIDE(i, n) if (m[i]) y[i] = s[i];
}
__global__ void k_mask_fill(double* y, double v, const uint8_t* m, long long n) {
  GRID_STRIDE(i, n) if (m[i]) y[i] = v;
}
__global__ void k_add(double* y, const double* x, long long n) { GRID_STRIDE(i, n) y[i] += x[i]; }
__global__ void k_mul(double* y, const double* a, const double* x, long long n) {
  GRID_STRIDE(i, n) y[i] = a[i] * x[i];
}
__global__ void k_recip(double* y, const double* d, long long n, int* zero) {
  GRID_STRIDE(i, n) {
    if (d[i] == 0.0) *zero = 1;
    y[i] = 1.0 / d[i];
  }
}
__global__ void k_cg_xr(double* x, double* r, const double* p, const double* ap, double alpha,
                        long long n) {
  GRID_STRIDE(i, n) {
    x[i] += alpha * p[i];
    r[i] -= alpha * ap[i];
  }
}
__global__ void k_cg_p(double* p, const double* z, double beta, long long n) {
  GRID_STRIDE(i, n) p[i] = z[i] + beta * p[i];
}
// the same updates with the coefficient num / den read from device scalars
__global__ void k_cg_xr_dev(double* x, double* r, const double* p, const double* ap,
                            const double* num, const double* den, long long n) {
  const double alpha = *num / *den;
  GRID_STRIDE(i, n) {
    x[i] += alpha * p[i];
    r[i] -= alpha * ap[i];
  }
}
__global__ void k_cg_p_dev(double* p, const double* z, const double* num, const double* den,
                           long long n) {
  const double beta = *num / *den;
  GRID_STRIDE(i, n) p[i] = z[i] + beta * p[i];
}
__global__ void k_cheb_first(double* x, double* r, double* d, const double* b, const double* inv,
                             double theta, long long n) {
  GRID_STRIDE(i, n) {
    double ri = b[i] - r[i];
    r[i] = ri;
    double di = inv[i] * ri / theta;
    d[i] = di;
    x[i] += di;
  }
}
__global__ void k_cheb_first_zero(double* x, double* d, const double* b, const double* inv,
                                  double theta, long long n) {
  GRID_STRIDE(i, n) {
    double di = inv[i] * b[i] / theta;
    d[i] = di;
    x[i] = 0.0 + di;
  }
}
__global__ void k_cheb_step(double* x, double* r, double* d, const double* b, const double* inv,
                            double c1, double c2, long long n) {
  GRID_STRIDE(i, n) {
    double ri = b[i] - r[i];
    r[i] = ri;
    double di = c1 * d[i] + c2 * inv[i] * ri;
    d[i] = di;
    x[i] += di;
  }
}

__global__ void k_waxpy(double* w, const double* x, double a, const double* y, long long n) {
  GRID_STRIDE(i, n) { w[i] = x[i] + a * y[i]; }
}
__global__ void k_neg(double* y, const double* x, long long n) {
  GRID_STRIDE(i, n) { y[i] = -x[i]; }
}

}  // namespace

DotWorkspace::DotWorkspace() {
  HXG_CUDA(cudaMalloc(&partial, sizeof(double) * (kDotBlocks + 8)));
  HXG_CUDA(cudaMallocHost(&host, sizeof(double) * 8));
}

DotWorkspace::~DotWorkspace() {
  if (partial) cudaFree(partial);
  if (host) cudaFreeHost(host);
}

void dot_async(const double* x, const double* y, long long n, DotWorkspace& ws, int slot,
               cudaStream_t s) {
  dot_stage1<<<kDotBlocks, kDotThreads, 0, s>>>(x, y, n, ws.partial);
  dot_stage2<<<1, kDotThreads, 0, s>>>(ws.partial, kDotBlocks, ws.partial + kDotBlocks + slot);
  HXG_CUDA(cudaMemcpyAsync(ws.host + slot, ws.partial + kDotBlocks + slot, sizeof(double),
                           cudaMemcpyDeviceToHost, s));
}

double* dot_masked_device(const double* x, const double* y, const uint8_t* mask, long long n,
                          DotWorkspace& ws, int slot, cudaStream_t s) {
  if (mask)
    dot_stage1_masked<<<kDotBlocks, kDotThreads, 0, s>>>(x, y, mask, n, ws.partial);
  else
    dot_stage1<<<kDotBlocks, kDotThreads, 0, s>>>(x, y, n, ws.partial);
  dot_stage2<<<1, kDotThreads, 0, s>>>(ws.partial, kDotBlocks, ws.partial + kDotBlocks + slot);
  return ws.partial + kDotBlocks + slot;
}

void dot_to(const double* x, const double* y, long long n, DotWorkspace& ws, double* out,
            cudaStream_t s) {
  dot_stage1<<<kDotBlocks, kDotThreads, 0, s>>>(x, y, n, ws.partial);
  dot_stage2<<<1, kDotThreads, 0, s>>>(ws.partial, kDotBlocks, out);
}
void cg_update_xr_dev(double* x, double* r, const double* p, const double* ap, const double* num,
                      const double* den, long long n, cudaStream_t s) {
  k_cg_xr_dev<<<grid(n), 256, 0, s>>>(x, r, p, ap, num, den, n);
}
void cg_update_p_dev(double* p, const double* z, const double* num, const double* den, long long n,
                     cudaStream_t s) {
  k_cg_p_dev<<<grid(n), 256, 0, s>>>(p, z, num, den, n);
}

double dot(const double* x, const double* y, long long n, DotWorkspace& ws, cudaStream_t s) {
  dot_async(x, y, n, ws, 0, s);
  HXG_CUDA(cudaStreamSynchronize(s));
  return ws.host[0];
}

void vcopy(double* y, const double* x, long long n, cudaStream_t s) {
  HXG_CUDA(cudaMemcpyAsync(y, x, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
}
void vzero(double* y, long long n, cudaStream_t s) {
  HXG_CUDA(cudaMemsetAsync(y, 0, sizeof(double) * n, s));
}
void vsub_from(double* y, const double* b, long long n, cudaStream_t s) {
  k_sub_from<<<grid(n), 256, 0, s>>>(y, b, n);
}
void vmask_zero(double* y, const uint8_t* m, long long n, cudaStream_t s) {
  if (m) k_mask_zero<<<grid(n), 256, 0, s>>>(y, m, n);
}
void vmask_copy(double* y, const double* src, const uint8_t* m, long long n, cudaStream_t s) {
  if (m) k_mask_copy<<<grid(n), 256, 0, s>>>(y, src, m, n);
}
void vmask_fill(double* y, double v, const uint8_t* m, long long n, cudaStream_t s) {
  if (m) k_mask_fill<<<grid(n), 256, 0, s>>>(y, v, m, n);
}
void vadd(double* y, const double* x, long long n, cudaStream_t s) {
  k_add<<<grid(n), 256, 0, s>>>(y, x, n);
}
void vwaxpy(double* w, const double* x, double a, const double* y, long long n, cudaStream_t s) {
  k_waxpy<<<grid(n), 256, 0, s>>>(w, x, a, y, n);
}
void vneg(double* y, const double* x, long long n, cudaStream_t s) {
  k_neg<<<grid(n), 256, 0, s>>>(y, x, n);
}
void vscale_mul(double* y, const double* a, const double* x, long long n, cudaStream_t s) {
  k_mul<<<grid(n), 256, 0, s>>>(y, a, x, n);
}
bool vreciprocal(double* y, const double* d, long long n, cudaStream_t s) {
  int* flag;
  HXG_CUDA(cudaMalloc(&flag, sizeof(int)));
  HXG_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), s));
  k_recip<<<grid(n), 256, 0, s>>>(y, d, n, flag);
  int h = 0;
  HXG_CUDA(cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, s));
  HXG_CUDA(cudaStreamSynchronize(s));
  cudaFree(flag);
  return h == 0;
}
void cg_update_xr(double* x, double* r, const double* p, const double* ap, double alpha,
                  long long n, cudaStream_t s) {
  k_cg_xr<<<grid(n), 256, 0, s>>>(x, r, p, ap, alpha, n);
}
void cg_update_p(double* p, const double* z, double beta, long long n, cudaStream_t s) {
  k_cg_p<<<grid(n), 256, 0, s>>>(p, z, beta, n);
}
void cheb_first(double* x, double* r, double* d, const double* b, const double* inv_diag,
                double theta, long long n, cudaStream_t s) {
  k_cheb_first<<<grid(n), 256, 0, s>>>(x, r, d, b, inv_diag, theta, n);
}
void cheb_first_zero(double* x, double* d, const double* b, const double* inv_diag, double theta,
                     long long n, cudaStream_t s) {
  k_cheb_first_zero<<<grid(n), 256, 0, s>>>(x, d, b, inv_diag, theta, n);
}
void cheb_step(double* x, double* r, double* d, const double* b, const double* inv_diag, double c1,
               double c2, long long n, cudaStream_t s) {
  k_cheb_step<<<grid(n), 256, 0, s>>>(x, r, d, b, inv_diag, c1, c2, n);
}

}  // namespace hxg
