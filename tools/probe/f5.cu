// Probe: the config-5 tap loop (RY = 1, KX = 33, 16 outputs per lane, window LDS from a
// staged shared tile) with the taps (a) in the kernel parameter bank (uniform datapath,
// FFMA R, R, UR -- the current kernel) or (b) in shared memory (LDS.128 broadcast per 4
// taps, FFMA R, R, R) -- the latter lets one launch carry any number of z-slices.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int KX = 33, KXP = 36, KY = 33, P = 100, ROWS = 96;
struct Taps { float t[KY * 34]; };
template <int MODE>
__global__ void __launch_bounds__(256, 2) k(const __grid_constant__ Taps taps, const float* in, float* out,
                                           int reps) {
  extern __shared__ __align__(16) float sm[];
  float* tile = sm;
  float* ts = sm + (ROWS * P + 3) / 4 * 4;  // taps [KY][KXP], 16-byte aligned
  for (int i = threadIdx.x; i < ROWS * P; i += 256) tile[i] = in[i & 4095];
  for (int i = threadIdx.x; i < KY * KXP; i += 256) ts[i] = 0.001f * (i % 37);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const float* base = tile + lane * P + (warp & 3) * 16;
  float acc[16];
  for (int c = 0; c < 16; ++c) acc[c] = 0.f;
  for (int r = 0; r < reps; ++r) {
#pragma unroll 1
    for (int ky = 0; ky < KY; ++ky) {
      const float* rp = base + ky * P;
      float win[48];
#pragma unroll
      for (int q = 0; q < 12; ++q) {
        const float4 v = *reinterpret_cast<const float4*>(rp + 4 * q);
        win[4 * q] = v.x; win[4 * q + 1] = v.y; win[4 * q + 2] = v.z; win[4 * q + 3] = v.w;
      }
      if (MODE == 2) {
        // window-element-outer order: consecutive FFMAs share the window register (operand
        // reuse cache), each accumulator still sums its taps in increasing kx order
        const float* w = taps.t + ky * 34;
#pragma unroll
        for (int j = 0; j < 16 + KX - 1; ++j) {
#pragma unroll
          for (int c = 0; c < 16; ++c) {
            const int kx = j - c;
            if (kx >= 0 && kx < KX) acc[c] = fmaf(w[kx], win[j], acc[c]);
          }
        }
      } else if (MODE == 0) {
        const float* w = taps.t + ky * 34;
#pragma unroll
        for (int kx = 0; kx < KX; ++kx) {
          const float t = w[kx];
#pragma unroll
          for (int c = 0; c < 16; ++c) acc[c] = fmaf(t, win[c + kx], acc[c]);
        }
      } else {
        const float* w = ts + ky * KXP;
        float tv[KXP];
#pragma unroll
        for (int q = 0; q < KXP / 4; ++q) {
          const float4 v = *reinterpret_cast<const float4*>(w + 4 * q);
          tv[4 * q] = v.x; tv[4 * q + 1] = v.y; tv[4 * q + 2] = v.z; tv[4 * q + 3] = v.w;
        }
#pragma unroll
        for (int kx = 0; kx < KX; ++kx) {
#pragma unroll
          for (int c = 0; c < 16; ++c) acc[c] = fmaf(tv[kx], win[c + kx], acc[c]);
        }
      }
    }
  }
  float s = 0;
  for (int c = 0; c < 16; ++c) s += acc[c];
  out[blockIdx.x * 256 + threadIdx.x] = s;
}
template <int M> void run(const Taps& t, const float* in, float* out) {
  const int smem = (ROWS * P + 8) * 4 + KY * KXP * 4 + 32;
  cudaFuncSetAttribute(k<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int nb; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k<M>, 256, smem);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int reps = 60;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0);
    k<M><<<148 * 2, 256, smem>>>(t, in, out, reps);
    cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 148 * 2 * 256 * (double)reps * KY * KX * 16;
    if (rep == 3) printf("mode %d (%d CTA/SM): %.3f ms  %.2f TFLOP/s\n", M, nb, ms, flops / ms / 1e9);
  }
}
int main() {
  Taps t; for (int i = 0; i < KY * 34; ++i) t.t[i] = 0.001f * (i % 37);
  float *in, *out; cudaMalloc(&in, 4096*4); cudaMemset(in, 0, 4096*4); cudaMalloc(&out, 148*8*256*4);
  run<0>(t, in, out); run<1>(t, in, out); run<2>(t, in, out); run<0>(t, in, out); run<2>(t, in, out);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
