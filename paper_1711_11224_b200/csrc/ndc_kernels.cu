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

#include "ndc_internal.h"

namespace ndc {
namespace {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!done);
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                            int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void prefetch_map(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

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

__host__ __device__ constexpr int window_quads(int kx) { return (kRX + kx - 1 + 3) / 4; }

__host__ __device__ constexpr int stage_bytes_aligned(int rows, int pitch_s) {
  return ((rows * pitch_s * 4) + 127) / 128 * 128;
}

// p0 combines with max for the KKT-style epilogues, with + otherwise.
__device__ __forceinline__ bool p0_is_max(int mode) { return mode == kEpiPG || mode == kEpiKKT; }

template <int KX>
__global__ void __launch_bounds__(kThreads, 2)
    correlate_kernel(const __grid_constant__ CUtensorMap map, const CorrGeom g, const CorrArgs a,
                     const __grid_constant__ TapBlock taps) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ double red0[kThreads / 32], red1[kThreads / 32];

  const int b = blockIdx.z;
  if (a.active != nullptr && a.active[b] == 0) return;
  const int oz = blockIdx.y;
  const int tile = blockIdx.x;
  const int tx0 = (tile % g.tiles_x) * kTileX;
  const int ty0 = (tile / g.tiles_x) * kTileY;
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int wx = warp & 3;
  const int wy = warp >> 2;

  // Tap slices whose input plane iz = oz + kz + off_z exists (out-of-range planes are
  // skipped, which also balances edge z-slabs).
  const int kzA = max(g.kz0, -oz - g.off_z);
  const int kzB = min(g.kz1, g.in_ez - oz - g.off_z);
  const int n = kzB - kzA;

  const int sbytes = stage_bytes_aligned(g.rows, g.pitch_s);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + g.stages * sbytes);
  const uint32_t tx_bytes = static_cast<uint32_t>(g.rows * g.pitch_s * 4);

  if (tid == 0) {
    prefetch_map(&map);
    for (int s = 0; s < g.stages; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) {
    const int pre = min(n, g.stages);
    for (int i = 0; i < pre; ++i) {
      const int iz = oz + kzA + i + g.off_z;
      mbar_expect_tx(&bars[i], tx_bytes);
      tma_load_3d(smem_raw + i * sbytes, &map, &bars[i], tx0 + g.off_x, ty0 + g.off_y,
                  b * g.in_ez + iz);
    }
  }

  float acc[kRX];
#pragma unroll
  for (int c = 0; c < kRX; ++c) acc[c] = 0.f;

  const int row_l = wy * 32 + lane;
  constexpr int NQ = window_quads(KX);
  for (int i = 0; i < n; ++i) {
    const int s = i % g.stages;
    mbar_wait(&bars[s], static_cast<uint32_t>((i / g.stages) & 1));
    const float* base =
        reinterpret_cast<const float*>(smem_raw + s * sbytes) + row_l * g.pitch_s + wx * kRX;
    const float* trow = taps.t + (kzA + i - g.kz0) * g.KY * KX;
    for (int ky = 0; ky < g.KY; ++ky) {
      const float* rp = base + ky * g.pitch_s;
      float win[NQ * 4];
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const float4 v = *reinterpret_cast<const float4*>(rp + 4 * q);
        win[4 * q + 0] = v.x;
        win[4 * q + 1] = v.y;
        win[4 * q + 2] = v.z;
        win[4 * q + 3] = v.w;
      }
      const float* w = trow + ky * KX;
#pragma unroll
      for (int kx = 0; kx < KX; ++kx) {
        const float t = w[kx];
#pragma unroll
        for (int c = 0; c < kRX; ++c) acc[c] = fmaf(t, win[c + kx], acc[c]);
      }
    }
    __syncthreads();  // every warp is done with stage s
    if (tid == 0 && i + g.stages < n) {
      const int iz = oz + kzA + i + g.stages + g.off_z;
      mbar_expect_tx(&bars[s], tx_bytes);
      tma_load_3d(smem_raw + s * sbytes, &map, &bars[s], tx0 + g.off_x, ty0 + g.off_y,
                  b * g.in_ez + iz);
    }
  }

  // ---- epilogue --------------------------------------------------------------------
  const int oy = ty0 + row_l;
  const int ox0 = tx0 + wx * kRX;
  const bool row_ok = oy < g.out_ey;
  const long long o = static_cast<long long>(b) * g.out_image +
                      static_cast<long long>(g.out_z0 + oz) * g.out_plane +
                      static_cast<long long>(oy) * g.out_pitch + ox0;
  if (g.accum && row_ok) {
#pragma unroll
    for (int q = 0; q < kRX / 4; ++q) {
      const float4 p = *reinterpret_cast<const float4*>(a.accum_in + o + 4 * q);
      acc[4 * q + 0] += p.x;
      acc[4 * q + 1] += p.y;
      acc[4 * q + 2] += p.z;
      acc[4 * q + 3] += p.w;
    }
  }
  if (!g.final_chunk) {
    if (row_ok) {
#pragma unroll
      for (int q = 0; q < kRX / 4; ++q)
        *reinterpret_cast<float4*>(a.out + o + 4 * q) =
            make_float4(acc[4 * q], acc[4 * q + 1], acc[4 * q + 2], acc[4 * q + 3]);
    }
    return;
  }

  const int mode = g.mode;
  double p0 = 0.0, p1 = 0.0;
  if (row_ok) {
    const float sc = (a.scale != nullptr) ? a.scale[b] : 1.0f;
    float res[kRX];
    float aux[kRX];
    float in[kRX];
    if (mode == kEpiResid || mode == kEpiPG || mode == kEpiKKT || mode == kEpiRLRatio ||
        mode == kEpiRLUpdate) {
#pragma unroll
      for (int q = 0; q < kRX / 4; ++q) {
        const float4 v = *reinterpret_cast<const float4*>(a.aux_in + o + 4 * q);
        in[4 * q] = v.x;
        in[4 * q + 1] = v.y;
        in[4 * q + 2] = v.z;
        in[4 * q + 3] = v.w;
      }
    } else {
#pragma unroll
      for (int c = 0; c < kRX; ++c) in[c] = 0.f;
    }
    const float step = (mode == kEpiPG) ? static_cast<float>(a.step[b]) : 0.f;
#pragma unroll
    for (int c = 0; c < kRX; ++c) {
      const bool ok = ox0 + c < g.out_ex;
      float v = 0.f, ax = 0.f;
      switch (mode) {
        case kEpiStore:
          v = acc[c] * sc;
          break;
        case kEpiResid:
          v = acc[c] - in[c];
          if (ok) p0 += static_cast<double>(v) * static_cast<double>(v);
          break;
        case kEpiNorm:
          v = acc[c] * sc;
          if (ok) p0 += static_cast<double>(v) * static_cast<double>(v);
          break;
        case kEpiPG: {
          // solvers.hpp:180-191: g, kkt = max|min(x,g)|, trial = max(x - step*g, 0),
          // and the bitwise fixed-point test trial == x.
          const float gg = acc[c];
          const float xv = in[c];
          float t = __fsub_rn(xv, __fmul_rn(gg, step));
          t = t < 0.f ? 0.f : t;
          v = t;
          ax = gg;
          if (ok) {
            p0 = fmax(p0, fabs(static_cast<double>(fminf(xv, gg))));
            p1 += (t != xv) ? 1.0 : 0.0;
          }
          break;
        }
        case kEpiKKT:
          if (ok) p0 = fmax(p0, fabs(static_cast<double>(fminf(in[c], acc[c]))));
          break;
        case kEpiClamp:
          v = acc[c] < 0.f ? 0.f : acc[c];
          break;
        case kEpiRLRatio: {
          // tensor.hpp:112-116 guarded_div(y, A x) fused with the residual A x - y.
          const float ax_v = acc[c] * sc;
          v = fabsf(ax_v) < 1e-12f ? 0.f : in[c] / ax_v;
          ax = ax_v - in[c];
          if (ok) p0 += static_cast<double>(ax) * static_cast<double>(ax);
          break;
        }
        case kEpiRLUpdate: {
          // solvers.hpp:290-291: x_next = x .* A^T(ratio); relative change terms.
          const float xn = in[c] * acc[c];
          v = xn;
          if (ok) {
            const double d = static_cast<double>(xn) - static_cast<double>(in[c]);
            p0 += d * d;
            p1 += static_cast<double>(in[c]) * static_cast<double>(in[c]);
          }
          break;
        }
        default:
          break;
      }
      res[c] = ok ? v : 0.f;
      aux[c] = ok ? ax : 0.f;
    }
    if (mode != kEpiKKT) {
#pragma unroll
      for (int q = 0; q < kRX / 4; ++q)
        *reinterpret_cast<float4*>(a.out + o + 4 * q) =
            make_float4(res[4 * q], res[4 * q + 1], res[4 * q + 2], res[4 * q + 3]);
    }
    if (mode == kEpiPG || mode == kEpiRLRatio) {
#pragma unroll
      for (int q = 0; q < kRX / 4; ++q)
        *reinterpret_cast<float4*>(a.aux_out + o + 4 * q) =
            make_float4(aux[4 * q], aux[4 * q + 1], aux[4 * q + 2], aux[4 * q + 3]);
    }
  }

  if (a.partials != nullptr) {
    const bool pmax = p0_is_max(mode);
    p0 = pmax ? warp_max(p0) : warp_sum(p0);
    p1 = warp_sum(p1);
    if (lane == 0) {
      red0[warp] = p0;
      red1[warp] = p1;
    }
    __syncthreads();
    if (tid == 0) {
      double s0 = red0[0], s1 = red1[0];
      for (int w = 1; w < kThreads / 32; ++w) {
        s0 = pmax ? fmax(s0, red0[w]) : s0 + red0[w];
        s1 += red1[w];
      }
      const long long idx =
          (static_cast<long long>(b) * gridDim.y + oz) * (g.tiles_x * g.tiles_y) + tile;
      a.partials[idx] = make_double2(s0, s1);
    }
  }
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

// Row-parallel elementwise kernels over pitched volumes: grid (blocks_per_image, batch),
// each block takes rows (z*ey + y) strided by gridDim.x, threads stride over x.
__global__ void pg_trial_kernel(const float* __restrict__ x, const float* __restrict__ g,
                                float* __restrict__ trial, const double* step, const int* active,
                                double2* partials, int ez, int ey, int ex, long long pitch) {
  __shared__ double red[32];
  const int b = blockIdx.y;
  if (active != nullptr && active[b] == 0) return;
  const float d = static_cast<float>(step[b]);
  const long long img = static_cast<long long>(ez) * ey * pitch * b;
  double changed = 0.0;
  for (long long r = blockIdx.x; r < static_cast<long long>(ez) * ey; r += gridDim.x) {
    const long long base = img + r * pitch;
    for (int c = threadIdx.x; c < ex; c += blockDim.x) {
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
                                   double2* partials, int ez, int ey, int ex, long long pitch) {
  __shared__ double red[32];
  const int b = blockIdx.y;
  const long long img = static_cast<long long>(ez) * ey * pitch * b;
  double neg = 0.0, total = 0.0;
  for (long long r = blockIdx.x; r < static_cast<long long>(ez) * ey; r += gridDim.x) {
    const long long base = img + r * pitch;
    for (int c = threadIdx.x; c < ex; c += blockDim.x) {
      const float v = src[base + c];
      const float cv = v < 0.f ? 0.f : v;
      dst[base + c] = cv;
      neg += (v < 0.f) ? 1.0 : 0.0;
      total += static_cast<double>(cv);
    }
  }
  neg = warp_sum(neg);
  total = warp_sum(total);
  __shared__ double red2[32];
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

__global__ void fill_kernel(float* dst, float value, int ez, int ey, int ex, long long pitch) {
  const int b = blockIdx.y;
  const long long img = static_cast<long long>(ez) * ey * pitch * b;
  for (long long r = blockIdx.x; r < static_cast<long long>(ez) * ey; r += gridDim.x) {
    const long long base = img + r * pitch;
    for (long long c = threadIdx.x; c < pitch; c += blockDim.x) dst[base + c] = c < ex ? value : 0.f;
  }
}

template <class Src, class Dst, bool kToPitched>
__global__ void repack_kernel(const Src* __restrict__ src, Dst* __restrict__ dst, int ez, int ey,
                              int ex, long long pitch) {
  const int b = blockIdx.y;
  const long long rows = static_cast<long long>(ez) * ey;
  for (long long r = blockIdx.x; r < rows; r += gridDim.x) {
    const long long pr = (static_cast<long long>(b) * rows + r) * pitch;
    const long long dr = (static_cast<long long>(b) * rows + r) * ex;
    if (kToPitched) {
      for (long long c = threadIdx.x; c < pitch; c += blockDim.x)
        dst[pr + c] = c < ex ? static_cast<Dst>(src[dr + c]) : Dst(0);
    } else {
      for (long long c = threadIdx.x; c < ex; c += blockDim.x) dst[dr + c] = static_cast<Dst>(src[pr + c]);
    }
  }
}

int row_blocks(long long rows) {
  long long nb = rows < 4096 ? rows : 4096;
  return static_cast<int>(nb < 1 ? 1 : nb);
}

}  // namespace

int shared_pitch_for(int kx) {
  // Row pitch of the staged tile: covers the 4 warps' 16-wide strips plus the KX-1
  // halo, rounded so pitch/4 is odd -> a quarter-warp's LDS.128 at consecutive rows
  // hits 8 disjoint bank quads (conflict-free).
  int need = (kTileX - kRX) + 4 * window_quads(kx);
  int p = (need + 3) / 4 * 4;
  while ((p / 4) % 2 == 0) p += 4;
  return p;
}

size_t correlate_smem_bytes(const CorrGeom& g) {
  return static_cast<size_t>(g.stages) * stage_bytes_aligned(g.rows, g.pitch_s) +
         static_cast<size_t>(kMaxStages) * 8;
}

template <int KX>
static cudaError_t launch_kx(const CUtensorMap& map, const CorrGeom& g, const CorrArgs& a,
                             const TapBlock& taps, int batch, int nz_out, cudaStream_t s) {
  const size_t smem = correlate_smem_bytes(g);
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(correlate_kernel<KX>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  dim3 grid(g.tiles_x * g.tiles_y, nz_out, batch);
  correlate_kernel<KX><<<grid, kThreads, smem, s>>>(map, g, a, taps);
  return cudaGetLastError();
}

cudaError_t launch_correlate(int kx, const CUtensorMap& map, const CorrGeom& g, const CorrArgs& a,
                             const TapBlock& taps, int batch, int nz_out, cudaStream_t s) {
  switch (kx) {
#define NDC_KX(K) \
  case K:         \
    return launch_kx<K>(map, g, a, taps, batch, nz_out, s);
    NDC_KX(1)
    NDC_KX(3)
    NDC_KX(5)
    NDC_KX(7)
    NDC_KX(9)
    NDC_KX(11)
    NDC_KX(13)
    NDC_KX(15)
    NDC_KX(17)
    NDC_KX(19)
    NDC_KX(21)
    NDC_KX(23)
    NDC_KX(25)
    NDC_KX(27)
    NDC_KX(29)
    NDC_KX(31)
    NDC_KX(33)
#undef NDC_KX
    default:
      return cudaErrorInvalidValue;
  }
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
                            const int* active, double2* partials, int batch, long long,
                            int ez, int ey, int ex, long long pitch, int blocks_per_image,
                            cudaStream_t s) {
  dim3 grid(blocks_per_image, batch);
  pg_trial_kernel<<<grid, 256, 0, s>>>(x, g, trial, step, active, partials, ez, ey, ex, pitch);
  return cudaGetLastError();
}

cudaError_t launch_clamp_count(const float* src, float* dst, double2* partials, int batch, int ez,
                               int ey, int ex, long long pitch, int blocks_per_image,
                               cudaStream_t s) {
  dim3 grid(blocks_per_image, batch);
  clamp_count_kernel<<<grid, 256, 0, s>>>(src, dst, partials, ez, ey, ex, pitch);
  return cudaGetLastError();
}

cudaError_t launch_fill(float* dst, float value, int batch, int ez, int ey, int ex, long long pitch,
                        cudaStream_t s) {
  dim3 grid(row_blocks(static_cast<long long>(ez) * ey), batch);
  fill_kernel<<<grid, 256, 0, s>>>(dst, value, ez, ey, ex, pitch);
  return cudaGetLastError();
}

cudaError_t launch_pack_f64(const double* dense, float* pitched, int batch, int ez, int ey, int ex,
                            long long pitch, cudaStream_t s) {
  dim3 grid(row_blocks(static_cast<long long>(ez) * ey), batch);
  repack_kernel<double, float, true><<<grid, 256, 0, s>>>(dense, pitched, ez, ey, ex, pitch);
  return cudaGetLastError();
}

cudaError_t launch_unpack_f64(const float* pitched, double* dense, int batch, int ez, int ey, int ex,
                              long long pitch, cudaStream_t s) {
  dim3 grid(row_blocks(static_cast<long long>(ez) * ey), batch);
  repack_kernel<float, double, false><<<grid, 256, 0, s>>>(pitched, dense, ez, ey, ex, pitch);
  return cudaGetLastError();
}

cudaError_t launch_pack_f32(const float* dense, float* pitched, int batch, int ez, int ey, int ex,
                            long long pitch, cudaStream_t s) {
  dim3 grid(row_blocks(static_cast<long long>(ez) * ey), batch);
  repack_kernel<float, float, true><<<grid, 256, 0, s>>>(dense, pitched, ez, ey, ex, pitch);
  return cudaGetLastError();
}

cudaError_t launch_unpack_f32(const float* pitched, float* dense, int batch, int ez, int ey, int ex,
                              long long pitch, cudaStream_t s) {
  dim3 grid(row_blocks(static_cast<long long>(ez) * ey), batch);
  repack_kernel<float, float, false><<<grid, 256, 0, s>>>(pitched, dense, ez, ey, ex, pitch);
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
