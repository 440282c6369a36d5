// Bring-up probe: canonical 2-D TMA load via libcu++ (CUDA programming guide pattern).
#include <cuda.h>
#include <cuda/barrier>
#include <cstdio>
#include <vector>
using barrier = cuda::barrier<cuda::thread_scope_block>;
namespace cde = cuda::device::experimental;
__global__ void k(const __grid_constant__ CUtensorMap map, float* out, int c0, int c1) {
  __shared__ alignas(128) float sm[32 * 32];
  #pragma nv_diag_suppress static_var_with_dynamic_init
  __shared__ barrier bar;
  if (threadIdx.x == 0) { init(&bar, blockDim.x); cde::fence_proxy_async_shared_cta(); }
  __syncthreads();
  barrier::arrival_token token;
  if (threadIdx.x == 0) {
    cde::cp_async_bulk_tensor_2d_global_to_shared(sm, &map, c0, c1, bar);
    token = cuda::device::barrier_arrive_tx(bar, 1, sizeof(sm));
  } else {
    token = bar.arrive();
  }
  bar.wait(std::move(token));
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) out[i] = sm[i];
}
int main(int argc, char** argv) {
  int W = 128, H = 64;
  std::vector<float> h(W * H); for (int i = 0; i < W * H; ++i) h[i] = i;
  float *d, *o; cudaMalloc(&d, W * H * 4); cudaMalloc(&o, 4096); cudaMemcpy(d, h.data(), W * H * 4, cudaMemcpyHostToDevice);
  void* p = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  typedef CUresult (*F)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  CUtensorMap map; cuuint64_t dims[2] = {(cuuint64_t)W, (cuuint64_t)H}; cuuint64_t str[1] = {(cuuint64_t)W * 4};
  cuuint32_t box[2] = {32, 32}, es[2] = {1, 1};
  CUresult r = ((F)p)(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  int c0 = argc > 1 ? atoi(argv[1]) : 0, c1 = argc > 2 ? atoi(argv[2]) : 0;
  k<<<1, 128>>>(map, o, c0, c1);
  cudaError_t e = cudaDeviceSynchronize();
  float ho[1024]; cudaMemcpy(ho, o, 4096, cudaMemcpyDeviceToHost);
  printf("encode=%d (%d,%d): %s  v[1][1]=%g expect %d\n", (int)r, c0, c1, cudaGetErrorString(e), ho[33], (c1 + 1) * W + c0 + 1);
  int dev; cudaGetDevice(&dev); cudaDeviceProp pr; cudaGetDeviceProperties(&pr, dev); printf("%s cc %d.%d\n", pr.name, pr.major, pr.minor);
  return 0;
}
