// Probe: register-blocked correlation loop with window LDS from shared memory.
// MODE 0: scalar FFMA, 1 window per row (current kernel); 1: FFMA2 broadcast taps;
// 2: FFMA2 with one window shared by both rows (half the LDS); 3: FFMA2 no LDS (windows in regs)
#include <cstdio>
#include <cuda_runtime.h>
struct Taps { float t[31 * 32]; };
template <int MODE>
__global__ void __launch_bounds__(256, 2) k(const __grid_constant__ Taps taps, const float* in, float* out, int reps) {
  extern __shared__ float sm[];
  const int P = 100;
  for (int i = threadIdx.x; i < 158 * P; i += 256) sm[i] = in[i % 4096];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const float* base = sm + lane * P + (warp & 3) * 16;
  float acc[2][16]; float2 A[2][8], B[2][7]; float b0[2], b15[2];
  for (int j = 0; j < 2; ++j) { for (int c = 0; c < 16; ++c) acc[j][c] = 0; for (int c = 0; c < 8; ++c) A[j][c] = make_float2(0,0); for (int c = 0; c < 7; ++c) B[j][c] = make_float2(0,0); b0[j] = b15[j] = 0; }
  float keep[48];
  for (int q = 0; q < 48; ++q) keep[q] = base[q];
  for (int r = 0; r < reps; ++r) {
    for (int ky = 0; ky < 31; ++ky) {
      const float* w = taps.t + ky * 32;
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        float win[48];
        if (MODE == 3 || (MODE == 2 && j == 1)) {
#pragma unroll
          for (int q = 0; q < 48; ++q) win[q] = keep[q];
        } else {
          const float* rp = base + (ky + 32 * j) * P;
#pragma unroll
          for (int q = 0; q < 12; ++q) { float4 v = *reinterpret_cast<const float4*>(rp + 4 * q); win[4*q]=v.x; win[4*q+1]=v.y; win[4*q+2]=v.z; win[4*q+3]=v.w; }
          if (MODE == 2) {
#pragma unroll
            for (int q = 0; q < 48; ++q) keep[q] = win[q];
          }
        }
#pragma unroll
        for (int kx = 0; kx < 31; ++kx) {
          const float t = w[kx];
          if (MODE == 0) {
#pragma unroll
            for (int c = 0; c < 16; ++c) acc[j][c] = fmaf(t, win[2 + c + kx], acc[j][c]);
          } else if (kx % 2 == 0) {
#pragma unroll
            for (int c = 0; c < 8; ++c) A[j][c] = __ffma2_rn(make_float2(t, t), make_float2(win[2 + 2*c + kx], win[3 + 2*c + kx]), A[j][c]);
          } else {
            b0[j] = fmaf(t, win[2 + kx], b0[j]);
#pragma unroll
            for (int c = 0; c < 7; ++c) B[j][c] = __ffma2_rn(make_float2(t, t), make_float2(win[3 + 2*c + kx], win[4 + 2*c + kx]), B[j][c]);
            b15[j] = fmaf(t, win[17 + kx], b15[j]);
          }
        }
      }
    }
  }
  float s = 0;
  for (int j = 0; j < 2; ++j) { s += b0[j] + b15[j]; for (int c = 0; c < 16; ++c) s += acc[j][c]; for (int c = 0; c < 8; ++c) s += A[j][c].x + A[j][c].y; for (int c = 0; c < 7; ++c) s += B[j][c].x + B[j][c].y; }
  out[blockIdx.x * 256 + threadIdx.x] = s;
}
template <int M> void run(const Taps& t, const float* in, float* out) {
  const int smem = 158 * 100 * 4;
  cudaFuncSetAttribute(k<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int nb; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k<M>, 256, smem);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int reps = 40;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    k<M><<<148 * 2, 256, smem>>>(t, in, out, reps);
    cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 148 * 2 * 256 * (double)reps * 31 * 2 * 31 * 16;
    if (rep == 2) printf("mode %d (%d CTA/SM): %.3f ms  %.2f TFLOP/s\n", M, nb, ms, flops / ms / 1e9);
  }
}
int main() {
  Taps t; for (int i = 0; i < 31 * 32; ++i) t.t[i] = 0.001f * (i % 37);
  float *in, *out; cudaMalloc(&in, 4096*4); cudaMemset(in, 0, 4096*4); cudaMalloc(&out, 148*8*256*4);
  run<0>(t, in, out); run<1>(t, in, out); run<2>(t, in, out); run<3>(t, in, out);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
