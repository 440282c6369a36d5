// Probe: scalar tap loop (FFMA R, R, UR), CX columns x RY rows x RZ output planes per lane: the
// RZ planes share each window load (tap rows of RZ different z-slices against one input row).
#include <cstdio>
#include <cuda_runtime.h>
struct Taps { float t[7680]; };

template <int KX, int CX, int RY, int RZ, int MINB>
__global__ void __launch_bounds__(256, MINB) k(const __grid_constant__ Taps taps, const float* in, float* out,
                                              int reps, int KY, int zoff2) {
  extern __shared__ __align__(16) float sm[];
  constexpr int KXP = (KX + 1) & ~1, NQ = (CX + KX - 1 + 3) / 4;
  constexpr int NSTRIP = 64 / CX;       // strips per 64-column tile... warps: NSTRIP x (8 / NSTRIP) row blocks
  constexpr int P = 100;
  const int rows = 32 * RY * (8 / NSTRIP) + KY - 1;
  for (int i = threadIdx.x; i < rows * P; i += 256) sm[i] = in[i & 4095];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const float* base = sm + (lane + (warp / NSTRIP) * 32 * RY) * P + (warp % NSTRIP) * CX;
  float acc[RZ][RY][CX];
  for (int z = 0; z < RZ; ++z)
  for (int j = 0; j < RY; ++j)
    for (int c = 0; c < CX; ++c) acc[z][j][c] = 0;
  for (int r = 0; r < reps; ++r) {
#pragma unroll 1
    for (int ky = 0; ky < KY; ++ky) {
      const float* w = taps.t + ky * KXP;
      const int zoff = 2 * zoff2;  // even: the second slice's tap pairs stay 64-bit loads
#pragma unroll
      for (int j = 0; j < RY; ++j) {
        const float* rp = base + (ky + 32 * j) * P;
        float win[NQ * 4];
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          const float4 v = *reinterpret_cast<const float4*>(rp + 4 * q);
          win[4 * q] = v.x; win[4 * q + 1] = v.y; win[4 * q + 2] = v.z; win[4 * q + 3] = v.w;
        }
#pragma unroll
        for (int z = 0; z < RZ; ++z) {
#pragma unroll
          for (int kx = 0; kx < KX; ++kx) {
            const float t = w[z * zoff + kx];
#pragma unroll
            for (int c = 0; c < CX; ++c) acc[z][j][c] = fmaf(t, win[c + kx], acc[z][j][c]);
          }
        }
      }
    }
  }
  float s = 0;
  for (int z = 0; z < RZ; ++z)
  for (int j = 0; j < RY; ++j)
    for (int c = 0; c < CX; ++c) s += acc[z][j][c];
  out[blockIdx.x * 256 + threadIdx.x] = s;
}

template <int KX, int CX, int RY, int RZ, int MINB>
void run(const Taps& t, const float* in, float* out, int KY) {
  const int smem = (32 * RY * (8 / (64 / CX)) + KY - 1) * 100 * 4;
  auto* f = k<KX, CX, RY, RZ, MINB>;
  cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  int nb;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, f, 256, smem);
  if (nb > MINB) nb = MINB;
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, f);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int reps = 4000 / KY;
  float best = 1e30f;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0);
    f<<<148 * nb, 256, smem>>>(t, in, out, reps, KY, KY * ((KX + 1) / 2));
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep > 0 && ms < best) best = ms;
  }
  const double flops = 2.0 * 148 * nb * 256 * (double)reps * KY * RY * RZ * KX * CX;
  printf("KX %d CX %d RY %d RZ %d: %d CTA/SM, %d regs, smem %d  %.3f ms  %.2f TFLOP/s  (%s)\n", KX, CX, RY,
         RZ, nb, fa.numRegs, smem, best, flops / best / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  static Taps t;
  for (int i = 0; i < 7680; ++i) t.t[i] = 0.001f * (i % 37);
  float *in, *out;
  cudaMalloc(&in, 4096 * 4);
  cudaMemset(in, 0, 4096 * 4);
  cudaMalloc(&out, 148 * 8 * 256 * 4);
  run<7, 16, 2, 1, 2>(t, in, out, 7);
  run<7, 32, 1, 1, 2>(t, in, out, 7);
  run<7, 32, 1, 1, 3>(t, in, out, 7);
  run<9, 16, 2, 1, 2>(t, in, out, 9);
  run<9, 32, 1, 1, 2>(t, in, out, 9);
  run<9, 32, 1, 1, 3>(t, in, out, 9);
  run<11, 16, 2, 1, 2>(t, in, out, 11);
  run<11, 32, 1, 1, 2>(t, in, out, 11);
  run<11, 32, 1, 1, 3>(t, in, out, 11);
  run<13, 16, 2, 1, 2>(t, in, out, 13);
  run<13, 32, 1, 1, 2>(t, in, out, 13);
  run<13, 32, 1, 1, 3>(t, in, out, 13);
  run<15, 16, 2, 1, 2>(t, in, out, 15);
  run<15, 32, 1, 1, 2>(t, in, out, 15);
  run<15, 32, 1, 1, 3>(t, in, out, 15);
  run<17, 16, 2, 1, 2>(t, in, out, 17);
  run<17, 32, 1, 1, 2>(t, in, out, 17);
  run<17, 32, 1, 1, 3>(t, in, out, 17);
  run<21, 16, 2, 1, 2>(t, in, out, 21);
  run<21, 32, 1, 1, 2>(t, in, out, 21);
  run<21, 32, 1, 1, 3>(t, in, out, 21);
  run<25, 16, 2, 1, 2>(t, in, out, 25);
  run<25, 32, 1, 1, 2>(t, in, out, 25);
  run<25, 32, 1, 1, 3>(t, in, out, 25);
  run<31, 16, 2, 1, 2>(t, in, out, 31);
  run<31, 32, 1, 1, 2>(t, in, out, 31);
  run<31, 32, 1, 1, 3>(t, in, out, 31);
  run<33, 16, 2, 1, 2>(t, in, out, 33);
  run<33, 32, 1, 1, 2>(t, in, out, 33);
  run<33, 32, 1, 1, 3>(t, in, out, 33);
  return 0;
}
