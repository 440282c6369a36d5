// Probe: scalar tap loop (FFMA R, R, UR) with different per-lane blockings -- CX columns x RY
// rows per lane -- and with the window LDS removed (NOLDS: upper bound without the loads).
#include <cstdio>
#include <cuda_runtime.h>
struct Taps { float t[7680]; };

template <int KX, int CX, int RY, bool NOLDS, int MINB>
__global__ void __launch_bounds__(256, MINB) k(const __grid_constant__ Taps taps, const float* in, float* out,
                                              int reps, int KY) {
  extern __shared__ __align__(16) float sm[];
  constexpr int KXP = (KX + 1) & ~1, NQ = (CX + KX - 1 + 3) / 4;
  constexpr int NSTRIP = 64 / CX;       // strips per 64-column tile... warps: NSTRIP x (8 / NSTRIP) row blocks
  constexpr int P = 100;
  const int rows = 32 * RY * (8 / NSTRIP) + KY - 1;
  for (int i = threadIdx.x; i < rows * P; i += 256) sm[i] = in[i & 4095];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const float* base = sm + (lane + (warp / NSTRIP) * 32 * RY) * P + (warp % NSTRIP) * CX;
  float acc[RY][CX];
  for (int j = 0; j < RY; ++j)
    for (int c = 0; c < CX; ++c) acc[j][c] = 0;
  float keep[NQ * 4];
  for (int q = 0; q < NQ * 4; ++q) keep[q] = base[q];
  for (int r = 0; r < reps; ++r) {
#pragma unroll 1
    for (int ky = 0; ky < KY; ++ky) {
      const float* w = taps.t + ky * KXP;
#pragma unroll
      for (int j = 0; j < RY; ++j) {
        const float* rp = base + (ky + 32 * j) * P;
        float win[NQ * 4];
        if (NOLDS) {
#pragma unroll
          for (int q = 0; q < NQ * 4; ++q) win[q] = keep[q];
        } else {
#pragma unroll
          for (int q = 0; q < NQ; ++q) {
            const float4 v = *reinterpret_cast<const float4*>(rp + 4 * q);
            win[4 * q] = v.x; win[4 * q + 1] = v.y; win[4 * q + 2] = v.z; win[4 * q + 3] = v.w;
          }
        }
#pragma unroll
        for (int kx = 0; kx < KX; ++kx) {
          const float t = w[kx];
#pragma unroll
          for (int c = 0; c < CX; ++c) acc[j][c] = fmaf(t, win[c + kx], acc[j][c]);
        }
      }
    }
  }
  float s = 0;
  for (int j = 0; j < RY; ++j)
    for (int c = 0; c < CX; ++c) s += acc[j][c];
  out[blockIdx.x * 256 + threadIdx.x] = s;
}

template <int KX, int CX, int RY, bool NOLDS, int MINB>
void run(const Taps& t, const float* in, float* out, int KY) {
  const int smem = (32 * RY * (8 / (64 / CX)) + KY - 1) * 100 * 4;
  auto* f = k<KX, CX, RY, NOLDS, MINB>;
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
  const int reps = 40;
  float best = 1e30f;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0);
    f<<<148 * nb, 256, smem>>>(t, in, out, reps, KY);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep > 0 && ms < best) best = ms;
  }
  const double flops = 2.0 * 148 * nb * 256 * (double)reps * KY * RY * KX * CX;
  printf("KX %d CX %d RY %d nolds %d: %d CTA/SM, %d regs, smem %d  %.3f ms  %.2f TFLOP/s  (%s)\n", KX, CX, RY,
         (int)NOLDS, nb, fa.numRegs, smem, best, flops / best / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  static Taps t;
  for (int i = 0; i < 7680; ++i) t.t[i] = 0.001f * (i % 37);
  float *in, *out;
  cudaMalloc(&in, 4096 * 4);
  cudaMemset(in, 0, 4096 * 4);
  cudaMalloc(&out, 148 * 8 * 256 * 4);
  run<33, 16, 1, false, 2>(t, in, out, 33);
  run<33, 16, 1, false, 5>(t, in, out, 33);
  run<33, 16, 1, true, 2>(t, in, out, 33);
  run<33, 16, 2, false, 2>(t, in, out, 33);
  run<33, 16, 2, false, 3>(t, in, out, 33);
  run<33, 16, 2, true, 2>(t, in, out, 33);
  run<33, 16, 4, false, 1>(t, in, out, 33);
  run<33, 32, 1, false, 2>(t, in, out, 33);
  run<33, 32, 1, false, 1>(t, in, out, 33);
  run<33, 32, 1, true, 2>(t, in, out, 33);
  run<33, 32, 2, false, 1>(t, in, out, 33);
  run<31, 16, 2, false, 3>(t, in, out, 31);
  run<31, 32, 1, false, 2>(t, in, out, 31);
  run<9, 16, 2, false, 2>(t, in, out, 9);
  run<9, 32, 2, false, 2>(t, in, out, 9);
  run<9, 32, 1, false, 2>(t, in, out, 9);
  return 0;
}
