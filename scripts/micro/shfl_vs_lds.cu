// Microbenchmark: throughput of 64-bit shared loads vs 64-bit warp shuffles.
#include <cstdio>
template <int MODE>
__global__ void k(double* out, int iters) {
  __shared__ double s[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) s[i] = i * 0.5;
  __syncthreads();
  int lane = threadIdx.x & 31;
  double a0 = lane, a1 = lane + 1, a2 = lane + 2, a3 = lane + 3;
  double acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
  for (int it = 0; it < iters; ++it) {
    if (MODE == 0 || MODE == 2) {
      int b = (threadIdx.x + it * 64) & 2047;
      acc0 += s[b]; acc1 += s[(b + 32) & 2047]; acc2 += s[(b + 512) & 2047]; acc3 += s[(b + 544) & 2047];
    }
    if (MODE == 1 || MODE == 2) {
      int src = (lane + it) & 31;
      acc0 += __shfl_sync(0xffffffffu, a0, src); acc1 += __shfl_sync(0xffffffffu, a1, src ^ 1);
      acc2 += __shfl_sync(0xffffffffu, a2, src ^ 2); acc3 += __shfl_sync(0xffffffffu, a3, src ^ 3);
      a0 += 1.0; a1 += 1.0; a2 += 1.0; a3 += 1.0;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc0 + acc1 + acc2 + acc3;
}
int main() {
  double* d; cudaMalloc(&d, 1 << 24);
  for (int r = 0; r < 2; ++r) { k<0><<<148*4, 256>>>(d, 2000); k<1><<<148*4, 256>>>(d, 2000); k<2><<<148*4, 256>>>(d, 2000); }
  cudaDeviceSynchronize(); printf("ok\n");
}
