// Microbenchmark: shared-memory wavefronts per LDS.64 for broadcast patterns.
#include <cstdio>
template <int MODE>
__global__ void k(double* out, int iters) {
  __shared__ double s[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = i * 0.5;
  __syncthreads();
  int lane = threadIdx.x & 31;
  int idx;
  if (MODE == 0) idx = 0;                    // all lanes same address
  else if (MODE == 1) idx = (lane / 3) * 1;  // 11 distinct consecutive doubles (3-lane groups)
  else if (MODE == 2) idx = lane;            // 32 distinct consecutive doubles
  else idx = (lane % 16);                    // 16 distinct (2 lanes each)
  double acc = 0.0;
  for (int it = 0; it < iters; ++it) {
    acc += s[(idx + it * 37) & 1023];
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
  double* d; cudaMalloc(&d, 1 << 22);
  k<0><<<148, 256>>>(d, 1000); k<1><<<148, 256>>>(d, 1000); k<2><<<148, 256>>>(d, 1000); k<3><<<148, 256>>>(d, 1000);
  cudaDeviceSynchronize(); printf("ok\n");
}
