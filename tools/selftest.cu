// Bring-up probe: trivial kernel + D2H, built like the library.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(float* p, int n) { int i = blockIdx.x * blockDim.x + threadIdx.x; if (i < n) p[i] = 2.f * i; }
__global__ void kd(const float* __restrict__ s, double* __restrict__ d, long long n, long long q) {
  for (long long i = blockIdx.x; i < n; i += gridDim.x) for (long long c = threadIdx.x; c < q; c += blockDim.x) d[i * q + c] = s[i * q + c];
}
int main() {
  float* p; double* d; cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaMalloc(&p, 1024 * 4); cudaMalloc(&d, 1024 * 8);
  k<<<4, 256, 0, s>>>(p, 1024);
  float h[4]; cudaError_t e = cudaMemcpyAsync(h, p, 16, cudaMemcpyDeviceToHost, s); cudaStreamSynchronize(s);
  printf("trivial: %s %f %f\n", cudaGetErrorString(e), h[1], h[3]);
  kd<<<4, 256, 0, s>>>(p, d, 4, 256);
  double hd[4]; e = cudaMemcpyAsync(hd, d, 32, cudaMemcpyDeviceToHost, s); cudaStreamSynchronize(s);
  printf("f2d: %s %f %f\n", cudaGetErrorString(e), hd[1], hd[3]);
  return 0;
}
