// Measured FP32 FMA peak of the device the plan runs on (the roofline denominator for
// the FFMA-bound convolution passes; MEASURED_PEAKS.json holds only bf16 tensor and copy
// figures).  Every thread runs 16 independent chains of packed `fma.rn.f32x2` (FFMA2, two
// FMAs per instruction) with the correlation loop's operand pattern (tap pair from the
// parameter bank, window pair and accumulator in registers), so neither issue slots nor
// memory bound the FMA pipe; 2 CTAs x 256 threads on every SM, ~2 ms per run.
#include <cuda_runtime.h>

#include <algorithm>

#include "ndc_plan.h"

namespace ndc {
namespace {

struct ProbeTaps {
  float t[64];
};

// The correlation kernel's own operand pattern: a tap pair from the kernel parameter
// bank (uniform datapath), a register window pair and an accumulator pair; 16 chains.
__global__ void __launch_bounds__(256) ffma2_probe(const __grid_constant__ ProbeTaps taps, const float* in,
                                                   float* out, int iters) {
  float2 win[24];  // register pairs (aligned: every FFMA2 operand is one 64-bit register pair)
#pragma unroll
  for (int i = 0; i < 24; ++i) win[i] = make_float2(in[(threadIdx.x + 2 * i) & 1023], in[(threadIdx.x + 2 * i + 1) & 1023]);
  float2 acc[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) acc[c] = make_float2(0.f, 0.f);
  for (int it = 0; it < iters; ++it) {
    const float* w = taps.t + (it & 1) * 32;
#pragma unroll
    for (int kp = 0; kp < 16; ++kp) {
      const float2 t = *reinterpret_cast<const float2*>(w + 2 * kp);
#pragma unroll
      for (int c = 0; c < 16; ++c) acc[c] = __ffma2_rn(t, win[(c + kp) % 24], acc[c]);
    }
    win[0].x += 1.0f;
    win[23].y -= 0.5f;
  }
  float s = 0.0f;
#pragma unroll
  for (int c = 0; c < 16; ++c) s += acc[c].x + acc[c].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

}  // namespace

double probe_fp32_peak(int device) {
  check_cuda(cudaSetDevice(device), "cudaSetDevice");
  cudaDeviceProp prop;
  check_cuda(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
  const int blocks = prop.multiProcessorCount * 2, threads = 256, iters = 4096;
  float *out = nullptr, *in = nullptr;
  cudaStream_t s;
  check_cuda(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "cudaStreamCreate");
  check_cuda(cudaMallocAsync(&out, static_cast<size_t>(blocks) * threads * 4, s), "cudaMallocAsync");
  check_cuda(cudaMallocAsync(&in, 1024 * 4, s), "cudaMallocAsync");
  check_cuda(cudaMemsetAsync(in, 0, 1024 * 4, s), "cudaMemset");
  ProbeTaps taps;
  for (int i = 0; i < 64; ++i) taps.t[i] = 0.001f * static_cast<float>(i);
  cudaEvent_t e0, e1;
  check_cuda(cudaEventCreate(&e0), "cudaEventCreate");
  check_cuda(cudaEventCreate(&e1), "cudaEventCreate");
  double best = 0.0;
  for (int rep = 0; rep < 4; ++rep) {  // the first run also warms the clocks
    check_cuda(cudaEventRecord(e0, s), "cudaEventRecord");
    ffma2_probe<<<blocks, threads, 0, s>>>(taps, in, out, iters);
    check_cuda(cudaGetLastError(), "probe launch");
    check_cuda(cudaEventRecord(e1, s), "cudaEventRecord");
    check_cuda(cudaEventSynchronize(e1), "cudaEventSynchronize");
    float ms = 0.f;
    check_cuda(cudaEventElapsedTime(&ms, e0, e1), "cudaEventElapsedTime");
    const double flops = 2.0 * 2.0 * 16.0 * 16.0 * static_cast<double>(iters) * blocks * threads;
    best = std::max(best, flops / (ms * 1e-3) / 1e12);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFreeAsync(out, s);
  cudaFreeAsync(in, s);
  cudaStreamSynchronize(s);
  cudaStreamDestroy(s);
  return best;
}

}  // namespace ndc
