// Correlation kernel template (see the ndc_kernels.cu header comment for the operator
// mapping).  Instantiated in ndc_corr_sh{0,2}_ry{1,2}.cu.
//
// CTA = 8 warps over an output tile of (64*RY) rows x 64 columns of one output plane:
// warp w takes columns 16*(w&3).. and rows 32*RY*(w>>2)..; lane l owns RY rows
// (l, l+32, ...) x 16 consecutive columns.  Per staged input plane and tap row ky each
// thread loads its RY input windows (16+KX-1 floats, float4 LDS; the smem row pitch
// has pitch/4 odd so a quarter-warp of consecutive rows is bank-conflict free) and
// runs RY*16*KX FFMAs whose tap operand is a uniform register loaded from the kernel
// parameter bank (LDCU, shared by the RY rows).  Tap rows are padded to an even
// length (kTapPitch) so pairs load as 64-bit words.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include "ndc_internal.h"

namespace ndc {
namespace corr {

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

// float4 quads of the register window: SH (0 or 2) leading floats keep every TMA tile
// start 16-byte aligned (an unaligned innermost start coordinate traps).
__host__ __device__ constexpr int window_quads(int kx, int sh) { return (sh + kRX + kx - 1 + 3) / 4; }

__host__ __device__ constexpr int stage_bytes_aligned(int rows, int pitch_s) {
  return ((rows * pitch_s * 4) + 127) / 128 * 128;
}

// p0 combines with max for the KKT-style epilogues, with + otherwise.
__device__ __forceinline__ bool p0_is_max(int mode) { return mode == kEpiPG || mode == kEpiKKT; }

// Epilogue for one 16-wide output strip at buffer offset o (see EpiMode).
__device__ __forceinline__ void epilogue_strip(const CorrGeom& g, const CorrArgs& a, int b,
                                               long long o, int ox0, float* acc, double& p0,
                                               double& p1) {
  if (g.accum) {
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
#pragma unroll
    for (int q = 0; q < kRX / 4; ++q)
      *reinterpret_cast<float4*>(a.out + o + 4 * q) =
          make_float4(acc[4 * q], acc[4 * q + 1], acc[4 * q + 2], acc[4 * q + 3]);
    return;
  }
  const int mode = g.mode;
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
  // The mode is uniform per launch: one specialised loop per mode (no per-element
  // branching).  Columns past the valid extent are written as zero.
#define NDC_EPI_LOOP(BODY)                           \
  _Pragma("unroll") for (int c = 0; c < kRX; ++c) {  \
    const bool ok = ox0 + c < g.out_ex;              \
    float v = 0.f, ax = 0.f;                         \
    BODY;                                            \
    res[c] = ok ? v : 0.f;                           \
    aux[c] = ok ? ax : 0.f;                          \
  }
  switch (mode) {
    case kEpiStore:
      NDC_EPI_LOOP(v = acc[c] * sc)
      break;
    case kEpiResid:
      NDC_EPI_LOOP(v = acc[c] - in[c]; if (ok) p0 += static_cast<double>(v) * static_cast<double>(v))
      break;
    case kEpiNorm:
      NDC_EPI_LOOP(v = acc[c] * sc; if (ok) p0 += static_cast<double>(v) * static_cast<double>(v))
      break;
    case kEpiPG: {
      // solvers.hpp:180-191: g, kkt = max|min(x,g)|, trial = max(x - step*g, 0), and the
      // bitwise fixed-point test trial == x.
      const float step = static_cast<float>(a.step[b]);
      NDC_EPI_LOOP(const float gg = acc[c]; const float xv = in[c];
                   float t = __fsub_rn(xv, __fmul_rn(gg, step)); t = t < 0.f ? 0.f : t; v = t; ax = gg;
                   if (ok) {
                     p0 = fmax(p0, fabs(static_cast<double>(fminf(xv, gg))));
                     p1 += (t != xv) ? 1.0 : 0.0;
                   })
      break;
    }
    case kEpiKKT:
      NDC_EPI_LOOP(if (ok) p0 = fmax(p0, fabs(static_cast<double>(fminf(in[c], acc[c])))))
      break;
    case kEpiClamp:
      NDC_EPI_LOOP(v = acc[c] < 0.f ? 0.f : acc[c])
      break;
    case kEpiRLRatio:
      // tensor.hpp:112-116 guarded_div(y, A x) fused with the residual A x - y.
      NDC_EPI_LOOP(const float ax_v = acc[c] * sc; v = fabsf(ax_v) < 1e-12f ? 0.f : in[c] / ax_v;
                   ax = ax_v - in[c]; if (ok) p0 += static_cast<double>(ax) * static_cast<double>(ax))
      break;
    case kEpiRLUpdate:
      // solvers.hpp:290-291: x_next = x .* A^T(ratio); relative change terms.
      NDC_EPI_LOOP(const float xn = in[c] * acc[c]; v = xn;
                   if (ok) {
                     const double d = static_cast<double>(xn) - static_cast<double>(in[c]);
                     p0 += d * d;
                     p1 += static_cast<double>(in[c]) * static_cast<double>(in[c]);
                   })
      break;
    default:
      NDC_EPI_LOOP((void)0)
      break;
  }
#undef NDC_EPI_LOOP
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

// NR of the thread's RY row windows against every tap row of one staged plane.
template <int KX, int SH, int RY, int NR>
__device__ __forceinline__ void accumulate_rows(float (&acc)[RY][kRX], const float* base,
                                                const float* trow, int KY, int kyA, int kyB,
                                                int pitch_s) {
  constexpr int NQ = window_quads(KX, SH);
  constexpr int KXP = tap_pitch(KX);
  // ky from 0: a uniform induction variable keeps the tap loads on the uniform datapath
  // (LDCU -> FFMA R, R, UR); [kyA, kyB) is warp-uniform (see the caller).
  for (int ky = 0; ky < KY; ++ky) {
#if defined(NDC_KY_SKIP)
    if (ky < kyA || ky >= kyB) continue;
#endif
    const float* w = trow + ky * KXP;
#if defined(NDC_J_NOUNROLL)
#pragma unroll 1
#else
#pragma unroll
#endif
    for (int j = 0; j < NR; ++j) {
      const float* rp = base + (ky + 32 * j) * pitch_s;
      float win[NQ * 4];
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const float4 v = *reinterpret_cast<const float4*>(rp + 4 * q);
        win[4 * q + 0] = v.x;
        win[4 * q + 1] = v.y;
        win[4 * q + 2] = v.z;
        win[4 * q + 3] = v.w;
      }
#pragma unroll
      for (int kx = 0; kx < KX; ++kx) {
        const float t = w[kx];
#pragma unroll
        for (int c = 0; c < kRX; ++c) acc[j][c] = fmaf(t, win[SH + c + kx], acc[j][c]);
      }
    }
  }
}

#ifndef NDC_MIN_BLOCKS
#define NDC_MIN_BLOCKS 2
#endif
template <int KX, int SH, int RY>
__global__ void __launch_bounds__(kThreads, NDC_MIN_BLOCKS)
    correlate_kernel(const __grid_constant__ CUtensorMap map, const CorrGeom g, const CorrArgs a,
                     const __grid_constant__ TapBlock taps) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  constexpr int TY = 64 * RY;

  const int b = blockIdx.z;
  if (a.active != nullptr && a.active[b] == 0) return;
  const int oz = blockIdx.y;
  const int tile = blockIdx.x;
  const int tx0 = (tile % g.tiles_x) * kTileX;
  const int ty0 = (tile / g.tiles_x) * TY;
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  // warp index broadcast from lane 0 so the compiler treats per-warp decisions as
  // warp-uniform (keeps the tap loads on the uniform datapath under those branches)
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
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

  float acc[RY][kRX];
#pragma unroll
  for (int j = 0; j < RY; ++j)
#pragma unroll
    for (int c = 0; c < kRX; ++c) acc[j][c] = 0.f;

  const int row_l = wy * (32 * RY) + lane;
  // Rows blocks / column strips entirely outside the output (the last tiles of an
  // extent that is not a tile multiple) skip their FFMAs; the test is warp-uniform.
  int nrun = 0;
#pragma unroll
  for (int j = 0; j < RY; ++j)
    if (ty0 + wy * (32 * RY) + 32 * j < g.out_ey) nrun = j + 1;
  if (tx0 + wx * kRX >= g.out_ex) nrun = 0;
  // Tap rows whose input row lies outside the data for every row this warp computes
  // multiply only zero fill (forward pass near the y borders).  Data row of (output row
  // r, tap row ky) = r + ky + off_y - in_row0.
  int kyA = 0, kyB = g.KY;
#if defined(NDC_KY_SKIP)
  {
    const int rw = ty0 + wy * (32 * RY);
    const int dd = g.off_y - g.in_row0;
    const int span = 32 * (nrun > 0 ? nrun : 1);
    kyA = max(0, -dd - rw - span + 1);
    kyB = min(g.KY, g.in_ey - dd - rw);
  }
#endif
  for (int i = 0; i < n; ++i) {
    const int s = i % g.stages;
    mbar_wait(&bars[s], static_cast<uint32_t>((i / g.stages) & 1));
    const float* base =
        reinterpret_cast<const float*>(smem_raw + s * sbytes) + row_l * g.pitch_s + wx * kRX;
    const float* trow = taps.t + (kzA + i - g.kz0) * g.KY * tap_pitch(KX);
    if (nrun == RY)
      accumulate_rows<KX, SH, RY, RY>(acc, base, trow, g.KY, kyA, kyB, g.pitch_s);
    else if (RY > 1 && nrun == 1)
      accumulate_rows<KX, SH, RY, 1>(acc, base, trow, g.KY, kyA, kyB, g.pitch_s);
    if (i + g.stages < n) {
      __syncthreads();  // every warp is done with stage s before it is refilled
      if (tid == 0) {
        const int iz = oz + kzA + i + g.stages + g.off_z;
        mbar_expect_tx(&bars[s], tx_bytes);
        tma_load_3d(smem_raw + s * sbytes, &map, &bars[s], tx0 + g.off_x, ty0 + g.off_y,
                    b * g.in_ez + iz);
      }
    }
  }

  // ---- epilogue --------------------------------------------------------------------
  const int ox0 = tx0 + wx * kRX;
  double p0 = 0.0, p1 = 0.0;
#pragma unroll
  for (int j = 0; j < RY; ++j) {
    const int oy = ty0 + row_l + 32 * j;
    if (oy < g.out_ey && ox0 < g.out_ex) {
      const long long o = static_cast<long long>(b) * g.out_image +
                          static_cast<long long>(g.out_z0 + oz) * g.out_plane +
                          static_cast<long long>(oy) * g.out_pitch + ox0;
      epilogue_strip(g, a, b, o, ox0, acc[j], p0, p1);
    }
  }

  if (a.partials != nullptr) {
    // one partial per warp, written without a CTA barrier (finalize reduces them in a
    // fixed order, so the result stays deterministic)
    const bool pmax = p0_is_max(g.mode);
    p0 = pmax ? warp_max(p0) : warp_sum(p0);
    p1 = warp_sum(p1);
    if (lane == 0) {
      const long long idx =
          ((static_cast<long long>(b) * gridDim.y + oz) * (g.tiles_x * g.tiles_y) + tile) *
              (kThreads / 32) + warp;
      a.partials[idx] = make_double2(p0, p1);
    }
  }
}

template <int KX, int SH, int RY>
cudaError_t launch_kx(const CUtensorMap& map, const CorrGeom& g, const CorrArgs& a,
                      const TapBlock& taps, int batch, int nz_out, cudaStream_t s) {
  const size_t smem = correlate_smem_bytes(g);
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(correlate_kernel<KX, SH, RY>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  dim3 grid(g.tiles_x * g.tiles_y, nz_out, batch);
  correlate_kernel<KX, SH, RY><<<grid, kThreads, smem, s>>>(map, g, a, taps);
  return cudaGetLastError();
}

#define NDC_KX_SWITCH(SH, RY)                                              \
  switch (kx) {                                                            \
    case 1: return launch_kx<1, SH, RY>(map, g, a, taps, batch, nz_out, s);   \
    case 3: return launch_kx<3, SH, RY>(map, g, a, taps, batch, nz_out, s);   \
    case 5: return launch_kx<5, SH, RY>(map, g, a, taps, batch, nz_out, s);   \
    case 7: return launch_kx<7, SH, RY>(map, g, a, taps, batch, nz_out, s);   \
    case 9: return launch_kx<9, SH, RY>(map, g, a, taps, batch, nz_out, s);   \
    case 11: return launch_kx<11, SH, RY>(map, g, a, taps, batch, nz_out, s); \
    case 13: return launch_kx<13, SH, RY>(map, g, a, taps, batch, nz_out, s); \
    case 15: return launch_kx<15, SH, RY>(map, g, a, taps, batch, nz_out, s); \
    case 17: return launch_kx<17, SH, RY>(map, g, a, taps, batch, nz_out, s); \
    case 19: return launch_kx<19, SH, RY>(map, g, a, taps, batch, nz_out, s); \
    case 21: return launch_kx<21, SH, RY>(map, g, a, taps, batch, nz_out, s); \
    case 23: return launch_kx<23, SH, RY>(map, g, a, taps, batch, nz_out, s); \
    case 25: return launch_kx<25, SH, RY>(map, g, a, taps, batch, nz_out, s); \
    case 27: return launch_kx<27, SH, RY>(map, g, a, taps, batch, nz_out, s); \
    case 29: return launch_kx<29, SH, RY>(map, g, a, taps, batch, nz_out, s); \
    case 31: return launch_kx<31, SH, RY>(map, g, a, taps, batch, nz_out, s); \
    case 33: return launch_kx<33, SH, RY>(map, g, a, taps, batch, nz_out, s); \
    default: return cudaErrorInvalidValue;                                 \
  }

}  // namespace corr
}  // namespace ndc
