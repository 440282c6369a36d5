// Measured FP32 FMA peak of the device the plan runs on (the roofline denominator for
// the FFMA-bound convolution passes; MEASURED_PEAKS.json holds only bf16 tensor and copy
// figures).  Every thread runs 16 independent chains of packed `fma.rn.f32x2` (FFMA2, two
// FMAs per instruction, register operands only) so neither issue slots nor memory can
// bound the FMA pipe; 4 CTAs x 256 threads per SM on every SM.
#include <cuda_runtime.h>

#include <algorithm>

#include "ndc_plan.h"

namespace ndc {
namespace {

__global__ void __launch_bounds__(256) ffma2_probe(float* out, int iters, unsigned long long a,
                                                   unsigned long long b) {
  unsigned long long acc[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) acc[c] = static_cast<unsigned long long>(threadIdx.x + c) << 8;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 16; ++c) asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc[c]) : "l"(a), "l"(b));
  }
  float s = 0.0f;
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    const float2 v = *reinterpret_cast<const float2*>(&acc[c]);
    s += v.x + v.y;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

}  // namespace

double probe_fp32_peak(int device) {
  check_cuda(cudaSetDevice(device), "cudaSetDevice");
  cudaDeviceProp prop;
  check_cuda(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
  const int blocks = prop.multiProcessorCount * 4, threads = 256, iters = 1 << 14;
  float* out = nullptr;
  cudaStream_t s;
  check_cuda(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "cudaStreamCreate");
  check_cuda(cudaMallocAsync(&out, static_cast<size_t>(blocks) * threads * 4, s), "cudaMallocAsync");
  cudaEvent_t e0, e1;
  check_cuda(cudaEventCreate(&e0), "cudaEventCreate");
  check_cuda(cudaEventCreate(&e1), "cudaEventCreate");
  // 0.5f x2 and 1.0f x2 as packed pairs: values stay finite, the work is the same
  const unsigned long long a = 0x3f0000003f000000ull, b = 0x3f8000003f800000ull;
  double best = 0.0;
  for (int rep = 0; rep < 4; ++rep) {  // the first run also warms the clocks
    check_cuda(cudaEventRecord(e0, s), "cudaEventRecord");
    ffma2_probe<<<blocks, threads, 0, s>>>(out, iters, a, b);
    check_cuda(cudaGetLastError(), "probe launch");
    check_cuda(cudaEventRecord(e1, s), "cudaEventRecord");
    check_cuda(cudaEventSynchronize(e1), "cudaEventSynchronize");
    float ms = 0.f;
    check_cuda(cudaEventElapsedTime(&ms, e0, e1), "cudaEventElapsedTime");
    const double flops = 2.0 * 2.0 * 16.0 * static_cast<double>(iters) * blocks * threads;
    best = std::max(best, flops / (ms * 1e-3) / 1e12);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFreeAsync(out, s);
  cudaStreamSynchronize(s);
  cudaStreamDestroy(s);
  return best;
}

}  // namespace ndc
