// sm_100a device code for the convolution-only deconvolution hot path.
//
// One kernel computes both operators of PAPER.md Properties 1-2:
//   forward  A x  : full convolution  (convolution.hpp:81-123)  = correlation of x with
//                   flip(h) at input offset -2p, input zero outside its extents;
//   adjoint  A^T r: valid correlation  (convolution.hpp:166-174: flip + conv_full + crop_m)
//                   = correlation of r with h at offset 0 -- no flip copy and no
//                   (m+4p)^n temporary.
// Input planes are staged in shared memory by TMA (cp.async.bulk.tensor, out-of-bounds
// zero fill does the padding); the x-taps of one tap row are a compile-time window so
// each thread keeps a 16-output register strip and a (16+KX-1)-float input window; the
// taps themselves live in the kernel's parameter constant bank and are read as uniform
// operands (FFMA R, R, UR).  The epilogue fuses the residual / objective, gradient /
// projection / KKT / fixed-point test, or power-iteration norm, and reduces per CTA in
// f64 (warp shuffle, then 8 warps in fixed order) for a deterministic second pass.
#include <cuda.h>
#include <cuda_runtime.h>

#include "ndc_correlate.cuh"
#include "ndc_internal.h"

namespace ndc {
namespace {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Fixed-order per-image reduction of the CTA partials.
__global__ void finalize_kernel(const double2* partials, long long per_image, int op, double* out0,
                                double* out1, float* scale_out, const int* active) {
  __shared__ double r0[32], r1[32];
  const int b = blockIdx.x;
  if (active != nullptr && active[b] == 0) return;
  const bool pmax = (op == kFinMaxSum);
  double a0 = 0.0, a1 = 0.0;
  const double2* p = partials + static_cast<long long>(b) * per_image;
  for (long long i = threadIdx.x; i < per_image; i += blockDim.x) {
    const double2 v = p[i];
    a0 = pmax ? fmax(a0, v.x) : a0 + v.x;
    a1 += v.y;
  }
  a0 = pmax ? warp_max(a0) : warp_sum(a0);
  a1 = warp_sum(a1);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    r0[warp] = a0;
    r1[warp] = a1;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s0 = r0[0], s1 = r1[0];
    for (int w = 1; w < static_cast<int>(blockDim.x / 32); ++w) {
      s0 = pmax ? fmax(s0, r0[w]) : s0 + r0[w];
      s1 += r1[w];
    }
    switch (op) {
      case kFinHalfSum:
        out0[b] = 0.5 * s0;
        break;
      case kFinNorm: {
        const double l = sqrt(s0);
        out0[b] = l;
        if (scale_out != nullptr) scale_out[b] = static_cast<float>(1.0 / l);
        break;
      }
      default:
        out0[b] = s0;
        if (out1 != nullptr) out1[b] = s1;
        break;
    }
  }
}

// Cross-rank combine of per-rank raw (sum / max) scalars gathered in rank order:
// every rank evaluates the same fixed-order expression, so all ranks take identical
// accept / backtrack / stop decisions.
__global__ void combine_kernel(const double* gathered, int world, int op, double* out0,
                               double* out1, float* scale_out) {
  if (threadIdx.x != 0) return;
  const bool pmax = (op == kFinMaxSum);
  double s0 = gathered[0], s1 = gathered[1];
  for (int r = 1; r < world; ++r) {
    s0 = pmax ? fmax(s0, gathered[2 * r]) : s0 + gathered[2 * r];
    s1 += gathered[2 * r + 1];
  }
  switch (op) {
    case kFinHalfSum:
      out0[0] = 0.5 * s0;
      break;
    case kFinNorm: {
      const double l = sqrt(s0);
      out0[0] = l;
      if (scale_out != nullptr) scale_out[0] = static_cast<float>(1.0 / l);
      break;
    }
    default:
      out0[0] = s0;
      if (out1 != nullptr) out1[0] = s1;
      break;
  }
}

// Row-parallel elementwise kernels over the interior of pitched volumes (pointers at
// the interior origin): grid (blocks_per_image, batch); block j takes rows r = z*ey + y
// strided by gridDim.x, threads stride over x.
__device__ __forceinline__ long long row_off(const Geo& v, int b, long long r) {
  const long long z = r / v.ey, y = r - z * v.ey;
  return static_cast<long long>(b) * v.image + z * v.plane + y * v.pitch;
}

__global__ void pg_trial_kernel(const float* __restrict__ x, const float* __restrict__ g,
                                float* __restrict__ trial, const double* step, const int* active,
                                double2* partials, Geo v) {
  __shared__ double red[32];
  const int b = blockIdx.y;
  if (active != nullptr && active[b] == 0) return;
  const float d = static_cast<float>(step[b]);
  double changed = 0.0;
  for (long long r = blockIdx.x; r < static_cast<long long>(v.ez) * v.ey; r += gridDim.x) {
    const long long base = row_off(v, b, r);
    for (int c = threadIdx.x; c < v.ex; c += blockDim.x) {
      const float xv = x[base + c];
      float t = __fsub_rn(xv, __fmul_rn(g[base + c], d));
      t = t < 0.f ? 0.f : t;
      trial[base + c] = t;
      changed += (t != xv) ? 1.0 : 0.0;
    }
  }
  changed = warp_sum(changed);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = changed;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < static_cast<int>(blockDim.x / 32); ++w) s += red[w];
    partials[static_cast<long long>(b) * gridDim.x + blockIdx.x] = make_double2(0.0, s);
  }
}

__global__ void clamp_count_kernel(const float* __restrict__ src, float* __restrict__ dst,
                                   double2* partials, Geo v) {
  __shared__ double red[32], red2[32];
  const int b = blockIdx.y;
  double neg = 0.0, total = 0.0;
  for (long long r = blockIdx.x; r < static_cast<long long>(v.ez) * v.ey; r += gridDim.x) {
    const long long base = row_off(v, b, r);
    for (int c = threadIdx.x; c < v.ex; c += blockDim.x) {
      const float val = src[base + c];
      const float cv = val < 0.f ? 0.f : val;
      dst[base + c] = cv;
      neg += (val < 0.f) ? 1.0 : 0.0;
      total += static_cast<double>(cv);
    }
  }
  neg = warp_sum(neg);
  total = warp_sum(total);
  if ((threadIdx.x & 31) == 0) {
    red[threadIdx.x >> 5] = total;
    red2[threadIdx.x >> 5] = neg;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0, n = 0.0;
    for (int w = 0; w < static_cast<int>(blockDim.x / 32); ++w) {
      s += red[w];
      n += red2[w];
    }
    partials[static_cast<long long>(b) * gridDim.x + blockIdx.x] = make_double2(s, n);
  }
}

// float64 direct correlation for small problems (the reference-exact power iteration,
// solvers.hpp:127-143): one output per thread, dense [z][y][x] f64 buffers, taps in
// global memory, input zero outside its extents.  out = acc / lam_prev (1 if null);
// with `partials`, per-block sum of out^2 (fixed order).
__global__ void corr_f64_kernel(const double* __restrict__ in, int iz, int iy, int ix,
                                double* __restrict__ out, int oz, int oy, int ox,
                                const double* __restrict__ taps, int KZ, int KY, int KX, int dz,
                                int dy, int dx, const double* lam_prev, double2* partials) {
  __shared__ double red[32];
  const long long n = static_cast<long long>(oz) * oy * ox;
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  double v = 0.0;
  if (i < n) {
    const int x = static_cast<int>(i % ox);
    const int y = static_cast<int>((i / ox) % oy);
    const int z = static_cast<int>(i / (static_cast<long long>(ox) * oy));
    const int z0 = z + dz, y0 = y + dy, x0 = x + dx;
    const int kza = max(0, -z0), kzb = min(KZ, iz - z0);
    const int kya = max(0, -y0), kyb = min(KY, iy - y0);
    const int kxa = max(0, -x0), kxb = min(KX, ix - x0);
    double acc = 0.0;
    for (int kz = kza; kz < kzb; ++kz)
      for (int ky = kya; ky < kyb; ++ky) {
        const double* ip = in + (static_cast<long long>(z0 + kz) * iy + (y0 + ky)) * ix + x0;
        const double* tp = taps + (static_cast<long long>(kz) * KY + ky) * KX;
        for (int kx = kxa; kx < kxb; ++kx) acc = fma(tp[kx], ip[kx], acc);
      }
    v = (lam_prev != nullptr) ? acc * (1.0 / *lam_prev) : acc;
    out[i] = v;
  }
  if (partials != nullptr) {
    double s = warp_sum(v * v);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < static_cast<int>(blockDim.x / 32); ++w) t += red[w];
      partials[blockIdx.x] = make_double2(t, 0.0);
    }
  }
}

__global__ void fill_f64_kernel(double* dst, double value, long long n) {
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    dst[i] = value;
}

__global__ void fill_kernel(float* dst, float value, Geo v) {
  const int b = blockIdx.y;
  for (long long r = blockIdx.x; r < static_cast<long long>(v.ez) * v.ey; r += gridDim.x) {
    const long long base = row_off(v, b, r);
    for (int c = threadIdx.x; c < v.ex; c += blockDim.x) dst[base + c] = value;
  }
}

template <class Src, class Dst, bool kToPitched>
__global__ void repack_kernel(const Src* __restrict__ src, Dst* __restrict__ dst, Geo v) {
  const int b = blockIdx.y;
  const long long rows = static_cast<long long>(v.ez) * v.ey;
  for (long long r = blockIdx.x; r < rows; r += gridDim.x) {
    const long long pr = row_off(v, b, r);
    const long long dr = (static_cast<long long>(b) * rows + r) * v.ex;
    if (kToPitched) {
      for (long long c = threadIdx.x; c < v.ex; c += blockDim.x) dst[pr + c] = static_cast<Dst>(src[dr + c]);
    } else {
      for (long long c = threadIdx.x; c < v.ex; c += blockDim.x) dst[dr + c] = static_cast<Dst>(src[pr + c]);
    }
  }
}

int row_blocks(long long rows) {
  long long nb = rows < 4096 ? rows : 4096;
  return static_cast<int>(nb < 1 ? 1 : nb);
}

}  // namespace

int shared_pitch_for(int kx, int sh) {
  // Row pitch of the staged tile: covers the 4 warps' 16-wide strips plus the KX-1
  // halo, rounded so pitch/4 is odd -> a quarter-warp's LDS.128 at consecutive rows
  // hits 8 disjoint bank quads (conflict-free).
  int need = (kTileX - kRX) + 4 * corr::window_quads(kx, sh);
  int p = (need + 3) / 4 * 4;
  while ((p / 4) % 2 == 0) p += 4;
  return p;
}

size_t correlate_smem_bytes(const CorrGeom& g, bool staging) {
  return static_cast<size_t>(corr::barrier_offset(g.stages, corr::stage_bytes_aligned(g.rows, g.pitch_s), staging)) +
         static_cast<size_t>(kMaxStages) * 8;
}

cudaError_t launch_correlate(int kx, int sh, int ry, const CUtensorMap& map, const CorrGeom& g,
                             const CorrArgs& a, const TapBlock& taps, int batch, int nz_out,
                             cudaStream_t s, cudaStream_t s_edge) {
  if (sh == 0 && ry == 1) return launch_correlate_sh0_ry1(kx, map, g, a, taps, batch, nz_out, s, s_edge);
  if (sh == 0 && ry == 2) return launch_correlate_sh0_ry2(kx, map, g, a, taps, batch, nz_out, s, s_edge);
  if (sh == 2 && ry == 1) return launch_correlate_sh2_ry1(kx, map, g, a, taps, batch, nz_out, s, s_edge);
  if (sh == 2 && ry == 2) return launch_correlate_sh2_ry2(kx, map, g, a, taps, batch, nz_out, s, s_edge);
  return cudaErrorInvalidValue;
}

cudaError_t launch_finalize(const double2* partials, long long per_image, int batch, int op,
                            double* out0, double* out1, float* scale_out, const int* active,
                            cudaStream_t s) {
  finalize_kernel<<<batch, 256, 0, s>>>(partials, per_image, op, out0, out1, scale_out, active);
  return cudaGetLastError();
}

cudaError_t launch_combine(const double* gathered, int world, int op, double* out0, double* out1,
                           float* scale_out, cudaStream_t s) {
  combine_kernel<<<1, 32, 0, s>>>(gathered, world, op, out0, out1, scale_out);
  return cudaGetLastError();
}

cudaError_t launch_pg_trial(const float* x, const float* g, float* trial, const double* step,
                            const int* active, double2* partials, int batch, const Geo& v,
                            int blocks_per_image, cudaStream_t s) {
  dim3 grid(blocks_per_image, batch);
  pg_trial_kernel<<<grid, 256, 0, s>>>(x, g, trial, step, active, partials, v);
  return cudaGetLastError();
}

cudaError_t launch_clamp_count(const float* src, float* dst, double2* partials, int batch,
                               const Geo& v, int blocks_per_image, cudaStream_t s) {
  dim3 grid(blocks_per_image, batch);
  clamp_count_kernel<<<grid, 256, 0, s>>>(src, dst, partials, v);
  return cudaGetLastError();
}

cudaError_t launch_corr_f64(const double* in, int iz, int iy, int ix, double* out, int oz, int oy,
                            int ox, const double* taps, int KZ, int KY, int KX, int dz, int dy,
                            int dx, const double* lam_prev, double2* partials, long long* nblocks,
                            cudaStream_t s) {
  const long long n = static_cast<long long>(oz) * oy * ox;
  const long long nb = (n + 255) / 256;
  if (nblocks) *nblocks = nb;
  corr_f64_kernel<<<static_cast<unsigned>(nb), 256, 0, s>>>(in, iz, iy, ix, out, oz, oy, ox, taps, KZ,
                                                            KY, KX, dz, dy, dx, lam_prev, partials);
  return cudaGetLastError();
}

cudaError_t launch_fill_f64(double* dst, double value, long long n, cudaStream_t s) {
  fill_f64_kernel<<<static_cast<unsigned>(std::min<long long>((n + 255) / 256, 4096)), 256, 0, s>>>(dst, value,
                                                                                               n);
  return cudaGetLastError();
}

cudaError_t launch_fill(float* dst, float value, int batch, const Geo& v, cudaStream_t s) {
  dim3 grid(row_blocks(static_cast<long long>(v.ez) * v.ey), batch);
  fill_kernel<<<grid, 256, 0, s>>>(dst, value, v);
  return cudaGetLastError();
}

cudaError_t launch_pack_f64(const double* dense, float* pitched, int batch, const Geo& v,
                            cudaStream_t s) {
  dim3 grid(row_blocks(static_cast<long long>(v.ez) * v.ey), batch);
  repack_kernel<double, float, true><<<grid, 256, 0, s>>>(dense, pitched, v);
  return cudaGetLastError();
}

cudaError_t launch_unpack_f64(const float* pitched, double* dense, int batch, const Geo& v,
                              cudaStream_t s) {
  dim3 grid(row_blocks(static_cast<long long>(v.ez) * v.ey), batch);
  repack_kernel<float, double, false><<<grid, 256, 0, s>>>(pitched, dense, v);
  return cudaGetLastError();
}

cudaError_t launch_pack_f32(const float* dense, float* pitched, int batch, const Geo& v,
                            cudaStream_t s) {
  dim3 grid(row_blocks(static_cast<long long>(v.ez) * v.ey), batch);
  repack_kernel<float, float, true><<<grid, 256, 0, s>>>(dense, pitched, v);
  return cudaGetLastError();
}

cudaError_t launch_unpack_f32(const float* pitched, float* dense, int batch, const Geo& v,
                              cudaStream_t s) {
  dim3 grid(row_blocks(static_cast<long long>(v.ez) * v.ey), batch);
  repack_kernel<float, float, false><<<grid, 256, 0, s>>>(pitched, dense, v);
  return cudaGetLastError();
}

// cuTensorMapEncodeTiled through cudaGetDriverEntryPoint (no link-time libcuda).
CUresult encode_tensor_map(CUtensorMap* map, const float* base, int ex, int ey, long long zcount,
                           long long pitch, long long plane, int box_x, int box_y) {
  using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static EncodeFn fn = nullptr;
  if (fn == nullptr) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        p == nullptr)
      return CUDA_ERROR_NOT_FOUND;
    fn = reinterpret_cast<EncodeFn>(p);
  }
  const cuuint64_t dims[3] = {static_cast<cuuint64_t>(ex), static_cast<cuuint64_t>(ey),
                              static_cast<cuuint64_t>(zcount)};
  const cuuint64_t strides[2] = {static_cast<cuuint64_t>(pitch) * 4,
                                 static_cast<cuuint64_t>(plane) * 4};
  const cuuint32_t box[3] = {static_cast<cuuint32_t>(box_x), static_cast<cuuint32_t>(box_y), 1};
  const cuuint32_t elem[3] = {1, 1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides, box,
            elem, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
}

}  // namespace ndc
