// Probe: tap-loop variants for the large-PSF kernels, c2-shaped (KX = KY = 31, two rows per
// lane, 3 CTAs / SM) and c5-shaped (KX = KY = 33, one row per lane, 2 CTAs / SM).
//   mode 0  scalar FFMA R, R, UR                                   (shipped for KX > 21)
//   mode 1  packed FFMA2, broadcast tap, two accumulator sets + 2 scalar FFMA per odd tap
//   mode 2  packed FFMA2, tap PAIRS (t[2m], t[2m+1]) as the 64-bit uniform operand against an
//           aligned window pair: even columns use the tap row as stored, odd columns a copy
//           shifted by one tap; out[c] = acc[c].x + acc[c].y.  No scalar FFMA at all.
//   mode 3  mode 2 with the lane's two rows ADJACENT (2l, 2l+1): one window load per input
//           row feeds row 2l with tap row ky and row 2l+1 with tap row ky-1 (half the LDS).
#include <cstdio>
#include <cuda_runtime.h>
struct Taps { float t[7680]; };

template <int KX, int RY, int MODE, int MINB>
__global__ void __launch_bounds__(256, MINB) k(const __grid_constant__ Taps taps, const float* in, float* out,
                                              int reps, int KY) {
  extern __shared__ __align__(16) float sm[];
  constexpr int P = 100, KXP = (KX + 1) & ~1, NP = KXP / 2, NQ = (16 + KX - 1 + 3) / 4;
  const int rows = 64 * RY + KY - 1;
  for (int i = threadIdx.x; i < rows * P; i += 256) sm[i] = in[i & 4095];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const float* base = sm + ((MODE == 3 ? 2 * lane : lane) + (warp >> 2) * 32 * RY) * P + (warp & 3) * 16;
  float acc[RY][16];
  float2 A[RY][16];
  float2 B[RY][7];
  float b0[RY], b15[RY];
  for (int j = 0; j < RY; ++j) {
    for (int c = 0; c < 16; ++c) { acc[j][c] = 0; A[j][c] = make_float2(0, 0); }
    for (int c = 0; c < 7; ++c) B[j][c] = make_float2(0, 0);
    b0[j] = b15[j] = 0;
  }
  for (int r = 0; r < reps; ++r) {
#pragma unroll 1
    for (int ky = 0; ky < KY; ++ky) {
      const float* w = taps.t + ky * KXP;           // tap row ky: t[0..KX-1], 0
      const float* ws = taps.t + 3840 + ky * KXP;   // shifted copy: 0, t[0..KX-1]
      if (MODE == 3) {
        const float* wB = taps.t + ((ky + KY - 1) % KY) * KXP;  // tap row of the second output row
        const float* wsB = wB + 3840;
        const float* rp = base + ky * P;
        float win[NQ * 4];
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          const float4 v = *reinterpret_cast<const float4*>(rp + 4 * q);
          win[4 * q] = v.x; win[4 * q + 1] = v.y; win[4 * q + 2] = v.z; win[4 * q + 3] = v.w;
        }
#pragma unroll
        for (int m = 0; m < NP; ++m) {
          const float2 te = make_float2(w[2 * m], w[2 * m + 1]), to = make_float2(ws[2 * m], ws[2 * m + 1]);
          const float2 teB = make_float2(wB[2 * m], wB[2 * m + 1]), toB = make_float2(wsB[2 * m], wsB[2 * m + 1]);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float2 wp = make_float2(win[2 * j + 2 * m], win[2 * j + 2 * m + 1]);
            A[0][2 * j] = __ffma2_rn(te, wp, A[0][2 * j]);
            A[0][2 * j + 1] = __ffma2_rn(to, wp, A[0][2 * j + 1]);
            A[RY - 1][2 * j] = __ffma2_rn(teB, wp, A[RY - 1][2 * j]);
            A[RY - 1][2 * j + 1] = __ffma2_rn(toB, wp, A[RY - 1][2 * j + 1]);
          }
        }
        continue;
      }
#pragma unroll
      for (int j = 0; j < RY; ++j) {
        const float* rp = base + (ky + 32 * j) * P;
        float win[NQ * 4];
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          const float4 v = *reinterpret_cast<const float4*>(rp + 4 * q);
          win[4 * q] = v.x; win[4 * q + 1] = v.y; win[4 * q + 2] = v.z; win[4 * q + 3] = v.w;
        }
        if (MODE == 0) {
#pragma unroll
          for (int kx = 0; kx < KX; ++kx) {
            const float t = w[kx];
#pragma unroll
            for (int c = 0; c < 16; ++c) acc[j][c] = fmaf(t, win[c + kx], acc[j][c]);
          }
        } else if (MODE == 1) {
#pragma unroll
          for (int kx = 0; kx < KX; ++kx) {
            const float t = w[kx];
            if (kx % 2 == 0) {
#pragma unroll
              for (int c = 0; c < 8; ++c)
                A[j][c] = __ffma2_rn(make_float2(t, t), make_float2(win[2 * c + kx], win[1 + 2 * c + kx]), A[j][c]);
            } else {
              b0[j] = fmaf(t, win[kx], b0[j]);
#pragma unroll
              for (int c = 0; c < 7; ++c)
                B[j][c] = __ffma2_rn(make_float2(t, t), make_float2(win[1 + 2 * c + kx], win[2 + 2 * c + kx]), B[j][c]);
              b15[j] = fmaf(t, win[15 + kx], b15[j]);
            }
          }
        } else {
#pragma unroll
          for (int m = 0; m < NP; ++m) {
            const float2 te = make_float2(w[2 * m], w[2 * m + 1]), to = make_float2(ws[2 * m], ws[2 * m + 1]);
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) {
              const float2 wp = make_float2(win[2 * jj + 2 * m], win[2 * jj + 2 * m + 1]);
              A[j][2 * jj] = __ffma2_rn(te, wp, A[j][2 * jj]);
              A[j][2 * jj + 1] = __ffma2_rn(to, wp, A[j][2 * jj + 1]);
            }
          }
        }
      }
    }
  }
  float s = 0;
  for (int j = 0; j < RY; ++j) {
    s += b0[j] + b15[j];
    for (int c = 0; c < 16; ++c) s += acc[j][c] + A[j][c].x + A[j][c].y;
    for (int c = 0; c < 7; ++c) s += B[j][c].x + B[j][c].y;
  }
  out[blockIdx.x * 256 + threadIdx.x] = s;
}

template <int KX, int RY, int M, int MINB>
void run(const Taps& t, const float* in, float* out, int KY) {
  const int smem = (64 * RY + KY - 1) * 100 * 4;
  cudaFuncSetAttribute(k<KX, RY, M, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k<KX, RY, M, MINB>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  int nb;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k<KX, RY, M, MINB>, 256, smem);
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, k<KX, RY, M, MINB>);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int reps = 4000 / KY;
  float best = 1e30f;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0);
    k<KX, RY, M, MINB><<<148 * nb, 256, smem>>>(t, in, out, reps, KY);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep > 0 && ms < best) best = ms;
  }
  const double flops = 2.0 * 148 * nb * 256 * (double)reps * KY * RY * KX * 16;
  printf("KX %d RY %d mode %d: %d CTA/SM, %d regs  %.3f ms  %.2f TFLOP/s  (%s)\n", KX, RY, M, nb, fa.numRegs, best,
         flops / best / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  static Taps t;
  for (int i = 0; i < 7680; ++i) t.t[i] = 0.001f * (i % 37);
  float *in, *out;
  cudaMalloc(&in, 4096 * 4);
  cudaMemset(in, 0, 4096 * 4);
  cudaMalloc(&out, 148 * 8 * 256 * 4);
  run<7, 2, 1, 2>(t, in, out, 7);
  run<9, 2, 1, 2>(t, in, out, 9);
  run<11, 2, 1, 2>(t, in, out, 11);
  run<13, 2, 1, 2>(t, in, out, 13);
  run<15, 2, 1, 2>(t, in, out, 15);
  run<17, 2, 1, 2>(t, in, out, 17);
  run<21, 2, 1, 2>(t, in, out, 21);
  run<25, 2, 1, 2>(t, in, out, 25);
  return 0;
}
