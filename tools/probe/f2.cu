#include <cstdio>
#include <cuda_runtime.h>
struct Taps { float t[64]; };
__device__ __forceinline__ void ffma2(float2& d, float2 a, float2 b) {
  unsigned long long dd = *reinterpret_cast<unsigned long long*>(&d);
  unsigned long long aa = *reinterpret_cast<unsigned long long*>(&a);
  unsigned long long bb = *reinterpret_cast<unsigned long long*>(&b);
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(dd) : "l"(aa), "l"(bb));
  d = *reinterpret_cast<float2*>(&dd);
}
// mode 0: scalar FFMA with tap in UR; mode 1: FFMA2 with tap pair from param
template <int MODE>
__global__ void __launch_bounds__(256,2) k(const __grid_constant__ Taps taps, const float* in, float* out, int iters, int ntap) {
  float win[48];
  for (int i = 0; i < 48; ++i) win[i] = in[threadIdx.x + i];
  float acc[16]; float2 acc2[16];
  for (int c = 0; c < 16; ++c) { acc[c] = 0; acc2[c] = make_float2(0,0); }
  for (int it = 0; it < iters; ++it) {
    const float* w = taps.t + (it & 1) * 32;
    if (MODE == 0) {
#pragma unroll
      for (int kx = 0; kx < 32; ++kx) { float t = w[kx];
#pragma unroll
        for (int c = 0; c < 16; ++c) acc[c] = fmaf(t, win[c + kx], acc[c]); }
    } else {
#pragma unroll
      for (int kp = 0; kp < 16; ++kp) {
        float2 t = *reinterpret_cast<const float2*>(w + 2*kp);
#pragma unroll
        for (int c = 0; c < 16; c += 2) ffma2(acc2[c], t, *reinterpret_cast<float2*>(&win[c + 2*kp]));
        float2 t2 = *reinterpret_cast<const float2*>(w + 2*kp + 32);
#pragma unroll
        for (int c = 1; c < 16; c += 2) ffma2(acc2[c], t2, *reinterpret_cast<float2*>(&win[c + 2*kp + 1]));
      }
    }
    win[0] += 1.0f; win[47] -= 0.5f;
  }
  float s = 0; for (int c = 0; c < 16; ++c) s += acc[c] + acc2[c].x + acc2[c].y;
  out[blockIdx.x * 256 + threadIdx.x] = s;
}
int main() {
  Taps t; for (int i = 0; i < 64; ++i) t.t[i] = 0.001f * i;
  float *in, *out; cudaMalloc(&in, 4096*4); cudaMemset(in, 0, 4096*4); cudaMalloc(&out, 148*8*256*4);
  int iters = 4000; cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int m = 0; m < 2; ++m) for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    if (m == 0) k<0><<<148*2, 256>>>(t, in, out, iters, 32); else k<1><<<148*2, 256>>>(t, in, out, iters, 32);
    cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 148*2*256 * (double)iters * 32 * 16;
    printf("mode %d: %.3f ms  %.2f TFLOP/s\n", m, ms, flops / ms / 1e9);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
