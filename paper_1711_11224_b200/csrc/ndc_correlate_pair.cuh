// Two output planes per CTA (narrow 3-D PSFs: config 4's 21 x 9 x 9).
//
// The general kernel (ndc_correlate.cuh) gives a CTA one output plane and streams that
// plane's KZ input planes through the stage ring.  With 9 taps per row its tap loop issues
// 12 window LDS.128 + 5 tap LDCU.64 + loop control per 288 FFMA: 92.3 % FFMA in an
// issue-bound loop (profiles/r02e_tap_loop_probes.md).  Here a CTA owns the output planes
// (oz0, oz0 + 1): a staged input plane iz meets plane oz0 with tap slice kz = iz - oz0 - off_z
// and plane oz0 + 1 with slice kz - 1, so every window load feeds both planes' accumulators
// (12 LDS + 10 LDCU per 576 FFMA: 96 % FFMA), every staged plane, barrier and TMA load is
// shared by two output planes, and a tile position stages KZ + 1 planes instead of 2 KZ.
// Full tiles only (the edge tiles keep the general kernel), scalar FFMA, 128-row tiles
// (RY = 2), same epilogues and per-warp partial layout: results are bit-identical to the
// general kernel's (each accumulator still sums its taps in the same order).
#pragma once

#include "ndc_correlate.cuh"

namespace ndc {
namespace corr {

// NR of the thread's RY row windows against tap row ky of TWO tap slices (tA, tB) of one
// staged plane; one window load per row feeds both planes' accumulators.
template <int KX, int SH, int RY, int NR>
__device__ __forceinline__ void accumulate_rows_pair(RowAcc<false> (&accA)[RY], RowAcc<false> (&accB)[RY],
                                                     const float* base, const float* tA, int slice_back, int KY,
                                                     int pitch_s) {
  constexpr int NQ = window_quads(KX, SH);
  constexpr int KXP = tap_pitch(KX);
#pragma unroll 1
  for (int ky = 0; ky < KY; ++ky) {
    const float* wA = tA + ky * KXP;
    const float* wB = wA - slice_back;  // the previous tap slice (an even offset: 64-bit tap pairs)
#pragma unroll
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
        const float t = wA[kx];
#pragma unroll
        for (int c = 0; c < kRX; ++c) accA[j].v[c] = fmaf(t, win[SH + c + kx], accA[j].v[c]);
      }
#pragma unroll
      for (int kx = 0; kx < KX; ++kx) {
        const float t = wB[kx];
#pragma unroll
        for (int c = 0; c < kRX; ++c) accB[j].v[c] = fmaf(t, win[SH + c + kx], accB[j].v[c]);
      }
    }
  }
}

template <int KX, int SH, int RY>
__global__ void __launch_bounds__(kThreads, 2)
    correlate_pair_kernel(const __grid_constant__ CUtensorMap map, const CorrGeom g, const CorrArgs a,
                          const __grid_constant__ TapBlock taps, int nz) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  constexpr int TY = 64 * RY;
  constexpr bool kStagedEpi = KX <= NDC_STAGED_KX || KX <= NDC_PREFETCH_KX;

  const int b = blockIdx.z;
  if (a.active != nullptr && a.active[b] == 0) return;
  // output-plane-pair fastest CTA order (see NDC_Z_FAST in the general kernel)
  const int lin = blockIdx.y * gridDim.x + blockIdx.x;
  const int oz0 = 2 * (lin % gridDim.y);
  const int t = lin / gridDim.y;
  const bool has2 = oz0 + 1 < nz;
  const int txi = t % g.full_tx, tyi = t / g.full_tx;
  const int tile = tyi * g.tiles_x + txi;
  const int tx0 = txi * kTileX, ty0 = tyi * TY;
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);  // warp-uniform for the compiler
  const int wx = warp & 3, wy = warp >> 2;

  // Input planes [a0, a1) meet plane oz0 (slice iz - oz0 - off_z), [b0, b1) meet plane
  // oz0 + 1 (one slice lower); b0 is a0 or a0 + 1 and b1 is a1 or a1 + 1, so their union is
  // the contiguous range [a0, max(a1, b1)) (out-of-range planes skipped as in the general kernel).
  const int a0 = max(oz0 + g.off_z + g.kz0, 0);
  const int a1 = min(oz0 + g.off_z + g.kz1, g.in_ez);
  const int b0 = has2 ? max(oz0 + 1 + g.off_z + g.kz0, 0) : a1;
  const int b1 = has2 ? min(oz0 + 1 + g.off_z + g.kz1, g.in_ez) : a1;
  const int lo = a0 < a1 ? a0 : b0;
  const int hi = b0 < b1 ? b1 : a1;
  const int n = hi - lo;

  const int sbytes = stage_bytes_aligned(g.rows, g.pitch_s);
  constexpr bool kStaging = kStagedEpi || !NDC_NOSTAGING_DIRECT;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + barrier_offset(g.stages, sbytes, kStaging));
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
      mbar_expect_tx(&bars[i], tx_bytes);
      tma_load_3d(smem_raw + i * sbytes, &map, &bars[i], tx0 + g.off_x, ty0 + g.off_y, b * g.in_ez + lo + i);
    }
  }

  RowAcc<false> accA[RY], accB[RY];
#pragma unroll
  for (int j = 0; j < RY; ++j) {
    row_zero(accA[j]);
    row_zero(accB[j]);
  }
  const float* const base0 = reinterpret_cast<const float*>(smem_raw) + (wy * (32 * RY) + lane) * g.pitch_s + wx * kRX;
  const int slice_taps = 2 * (g.KY * (tap_pitch(KX) / 2));  // visibly even: both slices' tap pairs load as 64-bit words
  for (int i = 0; i < n; ++i) {
    int s;
    uint32_t parity;
    if (g.stages == 2) {
      s = i & 1;
      parity = static_cast<uint32_t>(i >> 1) & 1u;
    } else {
      s = i % g.stages;
      parity = static_cast<uint32_t>(i / g.stages) & 1u;
    }
    mbar_wait(&bars[s], parity);
    const int iz = lo + i;
    const bool useA = iz >= a0 && iz < a1, useB = iz >= b0 && iz < b1;
    const float* base = base0 + s * (sbytes / 4);
    // tap slice of plane oz0 for this input plane (plane oz0 + 1 takes the one before it)
    const float* tA = taps.t + (iz - oz0 - g.off_z - g.kz0) * slice_taps;
    if (useA && useB)
      accumulate_rows_pair<KX, SH, RY, RY>(accA, accB, base, tA, slice_taps, g.KY, g.pitch_s);
    else if (useA)
      accumulate_rows<KX, SH, RY, RY, false, false>(accA, base, tA, g.KY, 0, 1, g.pitch_s);
    else if (useB)
      accumulate_rows<KX, SH, RY, RY, false, false>(accB, base, tA - slice_taps, g.KY, 0, 1, g.pitch_s);
    if (i + g.stages < n) {
      __syncthreads();  // every warp is done with stage s before it is refilled
      if (tid == 0) {
        mbar_expect_tx(&bars[s], tx_bytes);
        tma_load_3d(smem_raw + s * sbytes, &map, &bars[s], tx0 + g.off_x, ty0 + g.off_y,
                    b * g.in_ez + iz + g.stages);
      }
    }
  }

  float* wst = reinterpret_cast<float*>(smem_raw + g.stages * sbytes) + warp * (32 * kRX);
#pragma unroll
  for (int p = 0; p < 2; ++p) {
    if (p == 1 && !has2) break;
    float acc[RY][kRX];
#pragma unroll
    for (int j = 0; j < RY; ++j) row_value(p == 0 ? accA[j] : accB[j], acc[j]);
    const int oz = oz0 + p;
    double p0 = 0.0, p1 = 0.0;
#define NDC_PEPI(M) \
  epilogue_tile<M, RY, kStagedEpi>(g, a, b, oz, tx0 + wx * kRX, ty0 + wy * (32 * RY), lane, acc, wst, 0, nullptr, p0, p1)
    switch (g.final_chunk ? g.mode : -1) {
      case kEpiStore: NDC_PEPI(kEpiStore); break;
      case kEpiResid: NDC_PEPI(kEpiResid); break;
      case kEpiNorm: NDC_PEPI(kEpiNorm); break;
      case kEpiPG: NDC_PEPI(kEpiPG); break;
      case kEpiKKT: NDC_PEPI(kEpiKKT); break;
      case kEpiClamp: NDC_PEPI(kEpiClamp); break;
      case kEpiRLRatio: NDC_PEPI(kEpiRLRatio); break;
      case kEpiRLUpdate: NDC_PEPI(kEpiRLUpdate); break;
      case -1: NDC_PEPI(-1); break;
      default: break;
    }
#undef NDC_PEPI
    if (a.partials != nullptr) {
      const bool pmax = p0_is_max(g.mode);
      p0 = pmax ? warp_max(p0) : warp_sum(p0);
      if (!kStagedEpi || g.mode == kEpiPG || g.mode == kEpiRLUpdate) p1 = warp_sum(p1);
      if (lane == 0) {
        const long long idx =
            ((static_cast<long long>(b) * nz + oz) * (g.tiles_x * g.tiles_y) + tile) * (kThreads / 32) + warp;
        a.partials[idx] = make_double2(p0, p1);
      }
    }
  }
}

// The full tiles of one tap-chunk launch over nz_out output planes, two planes per CTA.
template <int KX, int SH, int RY>
cudaError_t launch_pair(const CUtensorMap& map, const CorrGeom& g, const CorrArgs& a, const TapBlock& taps,
                        int batch, int nz_out, cudaStream_t s) {
  auto* kern = correlate_pair_kernel<KX, SH, RY>;
  static bool configured = false;
  if (!configured) {
    const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  constexpr bool kStaging = KX <= NDC_STAGED_KX || KX <= NDC_PREFETCH_KX || !NDC_NOSTAGING_DIRECT;
  const size_t smem = correlate_smem_bytes(g, kStaging);
  kern<<<dim3(g.full_tx * g.full_ty, (nz_out + 1) / 2, batch), kThreads, smem, s>>>(map, g, a, taps, nz_out);
  return cudaGetLastError();
}

}  // namespace corr
}  // namespace ndc
