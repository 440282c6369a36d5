// Bring-up probe: 3-D TMA tile load (param-space descriptor) with OOB fill.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <int MODE>
__global__ void k(const __grid_constant__ CUtensorMap map, const CUtensorMap* gmap, float* out, int bx, int by, int c0, int c1, int c2) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const CUtensorMap* m = MODE == 0 ? &map : gmap;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)), "r"(bx * by * 4) : "memory");
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
      ::"r"(sa(sm)), "l"((uint64_t)m), "r"(c0), "r"(c1), "r"(c2), "r"(sa(&bar)) : "memory");
  }
  uint32_t done = 0;
  do { asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }" : "=r"(done) : "r"(sa(&bar)), "r"(0) : "memory"); } while (!done);
  for (int i = threadIdx.x; i < bx * by; i += blockDim.x) out[i] = reinterpret_cast<float*>(sm)[i];
}
int main(int argc, char** argv) {
  int ex = argc > 8 ? atoi(argv[8]) : 100, ey = argc > 9 ? atoi(argv[9]) : 50, ez = 2, pitch = 128; int bx = argc > 2 ? atoi(argv[2]) : 68, by = argc > 3 ? atoi(argv[3]) : 64;
  int c0 = argc > 4 ? atoi(argv[4]) : -5, c1 = argc > 5 ? atoi(argv[5]) : -3, c2 = argc > 6 ? atoi(argv[6]) : 1, promo = argc > 7 ? atoi(argv[7]) : 1;
  std::vector<float> h((size_t)pitch * ey * ez);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (float)i;
  float *d, *o; CUtensorMap* gm;
  cudaMalloc(&d, h.size() * 4); cudaMalloc(&o, bx * by * 4); cudaMalloc(&gm, sizeof(CUtensorMap));
  cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  void* p = nullptr; cudaDriverEntryPointQueryResult q;
  cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  printf("entry: %s q=%d p=%p\n", cudaGetErrorString(e), (int)q, p);
  typedef CUresult (*F)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  CUtensorMap map;
  cuuint64_t dims[3] = {(cuuint64_t)ex, (cuuint64_t)ey, (cuuint64_t)ez};
  cuuint64_t str[2] = {(cuuint64_t)pitch * 4, (cuuint64_t)pitch * ey * 4};
  cuuint32_t box[3] = {(cuuint32_t)bx, (cuuint32_t)by, 1}, es[3] = {1, 1, 1};
  CUresult r = ((F)p)(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, promo ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode rc=%d\n", (int)r);
  cudaMemcpy(gm, &map, sizeof(map), cudaMemcpyHostToDevice);
  int mode = argc > 1 ? atoi(argv[1]) : 0;
  size_t smem = bx * by * 4;
  if (mode == 0) { cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); k<0><<<1, 128, smem>>>(map, gm, o, bx, by, c0, c1, c2); }
  else { cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); k<1><<<1, 128, smem>>>(map, gm, o, bx, by, c0, c1, c2); }
  e = cudaDeviceSynchronize();
  std::vector<float> ho(bx * by);
  cudaMemcpy(ho.data(), o, bx * by * 4, cudaMemcpyDeviceToHost);
  // expected at smem (y=3, x=5) = element (z=1, y=0, x=0) = pitch*ey*1
  printf("mode %d box %dx%d at (%d,%d,%d) promo %d: %s  v[1][1]=%g expect %d\n", mode, bx, by, c0, c1, c2, promo, cudaGetErrorString(e), ho[bx + 1], (c0+1>=0&&c1+1>=0)? c2*pitch*ey + (c1+1)*pitch + c0+1 : -1);
  return 0;
}
