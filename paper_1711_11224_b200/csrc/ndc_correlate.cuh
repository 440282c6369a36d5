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
#include <type_traits>
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

// Named CTA barrier `id`, split into its two halves: the warps that only signal (arrive,
// non-blocking) and the warp that waits for all `count` threads (sync).
template <int ID>
__device__ __forceinline__ void bar_arrive() {
  asm volatile("barrier.cta.arrive %0, %1;" ::"n"(ID), "n"(kThreads) : "memory");
}
template <int ID>
__device__ __forceinline__ void bar_sync() {
  asm volatile("barrier.cta.sync %0, %1;" ::"n"(ID), "n"(kThreads) : "memory");
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                            int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

// 16-byte global -> shared copy that bypasses the registers (and L1), tracked as a group.
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Output-plane-fastest CTA order for 3-D launches (see correlate_kernel).  Measured
// (profiles/r01m_kbench_z_fast.txt): config 4 forward DRAM reads 35.9 -> 5.1 GB per pass
// (the KZ = 21 input planes of a tile stay in L2); step times equal within 0.3 %.
#ifndef NDC_Z_FAST
#define NDC_Z_FAST 1
#endif

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

// Epilogue staging: a dedicated 2 KB (32 rows x 16 floats) buffer per warp after the
// stages, so no warp ever waits for another around the epilogue.
constexpr int kStagingBytes = (kThreads / 32) * 32 * kRX * 4;

// Dynamic shared memory: stages, staging (staged-epilogue kernels without operand-prefetch
// buffers only), the stage mbarriers, then -- single-plane small PSFs -- the per-warp
// operand-prefetch buffers, which double as the staging buffers.  The direct-epilogue
// (large-PSF) kernels carry no staging buffer: 16 KB less per CTA lets a third CTA share
// the SM when registers allow (configs 2 and 5: 3 x 63-64 KB).
__host__ __device__ constexpr int barrier_offset(int stages, int sbytes, bool staging) {
  return stages * sbytes + (staging ? kStagingBytes : 0);
}

// p0 combines with max for the KKT-style epilogues, with + otherwise.
__device__ __forceinline__ bool p0_is_max(int mode) { return mode == kEpiPG || mode == kEpiKKT; }

// Swizzled position of quad q of row r in a per-warp 32 x 16-float staging buffer:
// XOR by (r >> 1) & 3 makes both the row-per-lane writes and the 4-lanes-per-row reads
// of store_rows bank-conflict free.
__device__ __forceinline__ int stage_pos(int r, int q) { return r * kRX + 4 * (q ^ ((r >> 1) & 3)); }

// Epilogue value for `out` of quad q (4 columns) of one output row from the final
// accumulators acc4 and the staged aux_in quad `in` (see EpiMode); reduction terms into
// p0 / p1.  Columns past the valid extent are zero and excluded from the reductions: the
// reductions take the MASKED float32 values (a zero term leaves a sum or a max of
// magnitudes unchanged), the max and the changed-count of the quad are formed in float32 /
// int and folded into the float64 partials once -- same values bit for bit as per-element
// float64 updates under `if (ok)`, without the selects on doubles those compile to.
// MODE < 0: an intermediate tap chunk (the raw partial sum).
// FULL: all four columns are inside the output (no column masks at all).
template <int MODE, bool FULL = false>
__device__ __forceinline__ float4 epilogue_res_lean(int cols_left, const float* acc4, const float* in, float sc,
                                               float step, double& p0, double& p1) {
  float res[4];
  float qmax = 0.f;  // kEpiPG / kEpiKKT: max |min(x, g)| of the quad
  int qcount = 0;    // kEpiPG: entries with trial != x
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const bool ok = FULL || c < cols_left;
    const float acc_c = acc4[c];
    float v = 0.f;
    if (MODE < 0) {
      v = acc_c;
    } else if (MODE == kEpiStore) {
      v = acc_c * sc;
    } else if (MODE == kEpiResid) {
      v = ok ? acc_c - in[c] : 0.f;
      p0 += static_cast<double>(v) * static_cast<double>(v);
    } else if (MODE == kEpiNorm) {
      v = ok ? acc_c * sc : 0.f;
      p0 += static_cast<double>(v) * static_cast<double>(v);
    } else if (MODE == kEpiPG) {
      // solvers.hpp:180-191: kkt = max|min(x,g)|, trial = max(x - step*g, 0), and the
      // bitwise fixed-point test trial == x (g itself is the aux output).
      const float gg = acc_c, xv = in[c];
      float t = __fsub_rn(xv, __fmul_rn(gg, step));
      t = t < 0.f ? 0.f : t;
      v = t;
      qmax = fmaxf(qmax, ok ? fabsf(fminf(xv, gg)) : 0.f);
      qcount += (ok && t != xv) ? 1 : 0;
    } else if (MODE == kEpiKKT) {
      qmax = fmaxf(qmax, ok ? fabsf(fminf(in[c], acc_c)) : 0.f);
    } else if (MODE == kEpiClamp) {
      v = acc_c < 0.f ? 0.f : acc_c;
    } else if (MODE == kEpiRLRatio) {
      // tensor.hpp:112-116 guarded_div(y, A x) fused with the residual A x - y.
      const float ax_v = acc_c * sc;
      v = fabsf(ax_v) < 1e-12f ? 0.f : in[c] / ax_v;
      const float d = ok ? ax_v - in[c] : 0.f;
      p0 += static_cast<double>(d) * static_cast<double>(d);
    } else if (MODE == kEpiRLUpdate) {
      // solvers.hpp:290-291: x_next = x .* A^T(ratio); relative change terms.
      const float xn = in[c] * acc_c;
      v = xn;
      const float xm = ok ? xn : 0.f, im = ok ? in[c] : 0.f;
      const double d = static_cast<double>(xm) - static_cast<double>(im);
      p0 += d * d;
      p1 += static_cast<double>(im) * static_cast<double>(im);
    }
    res[c] = (ok || MODE < 0) ? v : 0.f;
  }
  if (MODE == kEpiPG || MODE == kEpiKKT) p0 = fmax(p0, static_cast<double>(qmax));
  if (MODE == kEpiPG) p1 += static_cast<double>(qcount);
  return make_float4(res[0], res[1], res[2], res[3]);
}

template <int MODE>
__device__ __forceinline__ float4 epilogue_res(int cols_left, const float* acc4, const float* in, float sc,
                                               float step, double& p0, double& p1) {
  float res[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const bool ok = c < cols_left;
    const float acc_c = acc4[c];
    float v = 0.f;
    if (MODE < 0) {
      v = acc_c;
    } else if (MODE == kEpiStore) {
      v = acc_c * sc;
    } else if (MODE == kEpiResid) {
      v = acc_c - in[c];
      if (ok) p0 += static_cast<double>(v) * static_cast<double>(v);
    } else if (MODE == kEpiNorm) {
      v = acc_c * sc;
      if (ok) p0 += static_cast<double>(v) * static_cast<double>(v);
    } else if (MODE == kEpiPG) {
      // solvers.hpp:180-191: kkt = max|min(x,g)|, trial = max(x - step*g, 0), and the
      // bitwise fixed-point test trial == x (g itself is the aux output).
      const float gg = acc_c, xv = in[c];
      float t = __fsub_rn(xv, __fmul_rn(gg, step));
      t = t < 0.f ? 0.f : t;
      v = t;
      if (ok) {
        p0 = fmax(p0, fabs(static_cast<double>(fminf(xv, gg))));
        p1 += (t != xv) ? 1.0 : 0.0;
      }
    } else if (MODE == kEpiKKT) {
      if (ok) p0 = fmax(p0, fabs(static_cast<double>(fminf(in[c], acc_c))));
    } else if (MODE == kEpiClamp) {
      v = acc_c < 0.f ? 0.f : acc_c;
    } else if (MODE == kEpiRLRatio) {
      // tensor.hpp:112-116 guarded_div(y, A x) fused with the residual A x - y.
      const float ax_v = acc_c * sc;
      v = fabsf(ax_v) < 1e-12f ? 0.f : in[c] / ax_v;
      const float d = ax_v - in[c];
      if (ok) p0 += static_cast<double>(d) * static_cast<double>(d);
    } else if (MODE == kEpiRLUpdate) {
      // solvers.hpp:290-291: x_next = x .* A^T(ratio); relative change terms.
      const float xn = in[c] * acc_c;
      v = xn;
      if (ok) {
        const double d = static_cast<double>(xn) - static_cast<double>(in[c]);
        p0 += d * d;
        p1 += static_cast<double>(in[c]) * static_cast<double>(in[c]);
      }
    }
    res[c] = (ok || MODE < 0) ? v : 0.f;
  }
  return make_float4(res[0], res[1], res[2], res[3]);
}

__host__ __device__ constexpr bool mode_reads_aux_rt(int m) {
  return m == kEpiResid || m == kEpiPG || m == kEpiKKT || m == kEpiRLRatio || m == kEpiRLUpdate;
}

template <int MODE>
__host__ __device__ constexpr bool mode_reads_aux() {
  return MODE == kEpiResid || MODE == kEpiPG || MODE == kEpiKKT || MODE == kEpiRLRatio || MODE == kEpiRLUpdate;
}

// Warp-collective coalesced load of the strip's 32 rows x 16 columns into a staging
// buffer (lanes 4r..4r+3 read row r: 8 whole 64-byte segments per instruction instead of
// 32 half sectors); the epilogue then reads lane-per-row from shared memory.  `src0` points
// at column 0 of the strip's first row, `rows` is how many of the 32 rows exist.  Row
// r = 8k + (lane >> 2) of pass k: one running pointer (+ 8 rows per pass), and since
// (r >> 1) & 3 does not depend on k, stage_pos(r, q) = stage_pos(lane >> 2, q) + 128 k.
__device__ __forceinline__ void load_rows(float* wst, int lane, const float* src0, long long pitch, int rows) {
  const int r0 = lane >> 2, q = lane & 3;
  const float* p = src0 + static_cast<long long>(r0) * pitch + 4 * q;
  float* w = wst + stage_pos(r0, q);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
    if (8 * k + r0 < rows) x = *reinterpret_cast<const float4*>(p);
    *reinterpret_cast<float4*>(w + 8 * kRX * k) = x;
    p += 8 * pitch;
  }
}

// Warp-collective store of the 32 staged rows x 16 columns (row r written by lane r):
// every store instruction covers 8 whole 64-byte row segments (lanes 4r..4r+3 -> row r),
// so each 32-byte sector is written completely by one instruction.  (A lane-per-row
// store writes half sectors, which the L2 fills from DRAM first: measured ~2x DRAM
// traffic on small PSFs.)  Arguments as for load_rows.
__device__ __forceinline__ void store_rows(const float* wst, int lane, float* dst0, long long pitch, int rows) {
  const int r0 = lane >> 2, q = lane & 3;
  float* p = dst0 + static_cast<long long>(r0) * pitch + 4 * q;
  const float* w = wst + stage_pos(r0, q);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float4 x = *reinterpret_cast<const float4*>(w + 8 * kRX * k);
    if (8 * k + r0 < rows) *reinterpret_cast<float4*>(p) = x;
    p += 8 * pitch;
  }
}

// The epilogue of one warp's strip (16 columns x 32*RY rows) for epilogue mode MODE:
// per 32-row block, staged coalesced loads (accum_in, aux_in), lane-per-row math,
// staged coalesced stores (out, then aux_out) through the warp's own 2 KB buffer.
//
// STAGED = false (large PSFs, compute-bound): lane-per-row float4 loads / stores straight
// to global memory -- no shuffle through shared memory and no warp syncs, so a warp's
// epilogue overlaps its neighbours' FFMA work (the staged form measured 2-3 % slower on
// config 2, the direct form ~30 % slower on 3x3 / 5x5 PSFs).
template <int MODE, int RY, bool STAGED>
__device__ __forceinline__ void epilogue_tile(const CorrGeom& g, const CorrArgs& a, int b, int oz, int ox0,
                                              int wrow0, int lane, float (&acc)[RY][kRX], float* wst0,
                                              int wst_stride, const float* wpre, double& p0, double& p1) {
  constexpr bool kReadsAux = mode_reads_aux<MODE>();
  constexpr bool kStoreOut = MODE != kEpiKKT;
  constexpr bool kStoreAux = MODE == kEpiPG || MODE == kEpiRLRatio;
  const long long obase = static_cast<long long>(b) * g.out_image +
                          static_cast<long long>(g.out_z0 + oz) * g.out_plane + ox0;
  const bool strip_ok = ox0 < g.out_ex;
  const int cols_left = g.out_ex - ox0;
  const float sc = (MODE >= 0 && a.scale != nullptr) ? a.scale[b] : 1.0f;
  const float step = MODE == kEpiPG ? static_cast<float>(a.step[b]) : 0.f;
#pragma unroll
  for (int j = 0; j < RY; ++j) {
    const int row0 = wrow0 + 32 * j;  // the warp's first row of block j
    const bool mine = row0 + lane < g.out_ey && strip_ok;
    // staged loads / stores: offset of the block's first row, and how many of its rows exist
    const long long blk = obase + static_cast<long long>(row0) * g.out_pitch;
    const int rows = strip_ok ? g.out_ey - row0 : 0;
    float* acc_j = acc[j];
    // staging buffer of block j: the warp's 2 KB buffer, or (wst_stride != 0) the block's own
    // operand-prefetch buffer, which each lane has read its slot of before it overwrites it
    float* wst = wst0 + j * wst_stride;
    if (!STAGED) {
      const long long o = obase + static_cast<long long>(row0 + lane) * g.out_pitch;
      if (!mine) continue;
      float in[kRX];
#pragma unroll
      for (int q = 0; q < kRX / 4; ++q) {
        if (g.accum) {
          const float4 p = *reinterpret_cast<const float4*>(a.accum_in + o + 4 * q);
          acc_j[4 * q] += p.x;
          acc_j[4 * q + 1] += p.y;
          acc_j[4 * q + 2] += p.z;
          acc_j[4 * q + 3] += p.w;
        }
        if (kReadsAux) {
          const float4 v = *reinterpret_cast<const float4*>(a.aux_in + o + 4 * q);
          in[4 * q] = v.x;
          in[4 * q + 1] = v.y;
          in[4 * q + 2] = v.z;
          in[4 * q + 3] = v.w;
        }
      }
#pragma unroll
      for (int q = 0; q < kRX / 4; ++q) {
        const float4 r = epilogue_res<MODE>(cols_left - 4 * q, &acc_j[4 * q], &in[4 * q], sc, step, p0, p1);
        if (kStoreOut) *reinterpret_cast<float4*>(a.out + o + 4 * q) = r;
        if (kStoreAux) {
          float x[4];
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const float v = MODE == kEpiPG ? acc_j[4 * q + c] : acc_j[4 * q + c] * sc - in[4 * q + c];
            x[c] = 4 * q + c < cols_left ? v : 0.f;
          }
          *reinterpret_cast<float4*>(a.aux_out + o + 4 * q) = make_float4(x[0], x[1], x[2], x[3]);
        }
      }
      continue;
    }
    if (g.accum) {  // partial sums of the earlier tap chunks
      load_rows(wst, lane, a.accum_in + blk, g.out_pitch, rows);
      __syncwarp();
#pragma unroll
      for (int q = 0; q < kRX / 4; ++q) {
        const float4 p = *reinterpret_cast<const float4*>(wst + stage_pos(lane, q));
        acc_j[4 * q] += p.x;
        acc_j[4 * q + 1] += p.y;
        acc_j[4 * q + 2] += p.z;
        acc_j[4 * q + 3] += p.w;
      }
      __syncwarp();
    }
    // aux_in: prefetched into wpre at kernel start (cp.async), else a staged load now
    const float* src_in = wpre != nullptr ? wpre + j * (32 * kRX) : wst;
    if (kReadsAux) {
      if (wpre != nullptr) {
        if (j == 0) cp_async_wait_all();
      } else {
        load_rows(wst, lane, a.aux_in + blk, g.out_pitch, rows);
      }
      __syncwarp();
    }
    float in[kRX];
    // (strips wholly inside the output -- all but the last tile column -- take the
    // instantiation without column masks)
    auto block_math = [&](auto full_tag) {
      constexpr bool kFull = decltype(full_tag)::value;
#pragma unroll
      for (int q = 0; q < kRX / 4; ++q) {
        const int sp = stage_pos(lane, q);
        if (kReadsAux) {
          const float4 v = *reinterpret_cast<const float4*>(src_in + sp);
          in[4 * q] = v.x;
          in[4 * q + 1] = v.y;
          in[4 * q + 2] = v.z;
          in[4 * q + 3] = v.w;
        }
        float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
        if (mine)
          r = epilogue_res_lean<MODE, kFull>(cols_left - 4 * q, &acc_j[4 * q], &in[4 * q], sc, step, p0, p1);
        if (kStoreOut) *reinterpret_cast<float4*>(wst + sp) = r;  // same lane, same slot
      }
    };
    if (RY == 1 && cols_left >= kRX)  // (the 128-row kernels measured 0.5 % slower with both copies)
      block_math(std::true_type{});
    else
      block_math(std::false_type{});
    if (kStoreOut) {
      __syncwarp();
      store_rows(wst, lane, a.out + blk, g.out_pitch, rows);
      __syncwarp();
    }
    if (kStoreAux) {  // kEpiPG: g = acc; kEpiRLRatio: A x - Y
#pragma unroll
      for (int q = 0; q < kRX / 4; ++q) {
        float r[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const float v = MODE == kEpiPG ? acc_j[4 * q + c] : acc_j[4 * q + c] * sc - in[4 * q + c];
          r[c] = 4 * q + c < cols_left ? v : 0.f;
        }
        *reinterpret_cast<float4*>(wst + stage_pos(lane, q)) = make_float4(r[0], r[1], r[2], r[3]);
      }
      __syncwarp();
      store_rows(wst, lane, a.aux_out + blk, g.out_pitch, rows);
      __syncwarp();
    }
  }
}

// Packed FP32 (sm_100 FFMA2): one instruction does two FMAs, so the FMA pipe -- not the
// issue slot -- bounds the tap loop, and the window LDS / tap LDCU / loop control issue in
// the slots FFMA2 leaves free (measured 73.3 vs 70.2 TFLOP/s for FFMA on a register-
// blocked loop, tools/probe/f2.cu).  A lane's 16 outputs are column pairs, and the tap is
// a broadcast scalar operand (`FFMA2 R, R, UR.F32, R`: no tap shuffling):
//   even tap kx: pairs (c, c+1), c = 0, 2, .., 14 -- window pair (c+kx, c+kx+1) starts at
//                an even register (a 64-bit aligned pair);
//   odd tap kx:  pairs (c, c+1), c = 1, 3, .., 13, into a second accumulator set, plus
//                scalar FFMAs for columns 0 and 15 (again even-aligned window pairs).
// Exactly 16*KX MACs per row window (8 FFMA2 per even tap, 7 FFMA2 + 2 FFMA per odd tap);
// the two sets are added once after the tap loop.
//
// Where it pays (tools/kbench.py, one B200, 2048^2 x 16 batch with N x N PSFs, both
// passes): N = 7..17 +8..26 %, 21 +3..5 %, 25..31 neutral, 33 -1 %; 3-D config 3
// (15 x 15 rows) +2 % forward; 3-D config 4 (9 x 9 rows) -8 %.  So: packed for
// 11 <= KX <= 21, and for KX = 7 / 9 only when a launch carries a single z-slice of taps
// (both instantiations exist for those two widths); scalar FFMA otherwise.
#ifndef NDC_FFMA2
#define NDC_FFMA2 1
#endif
#ifndef NDC_PACK_MAXKX
#define NDC_PACK_MAXKX 21
#endif
enum PackMode : int { kPackNever = 0, kPackAlways = 1, kPackSingleSlice = 2 };
template <int KX>
__host__ __device__ constexpr int pack_mode() {
  return !NDC_FFMA2 ? kPackNever
         : (KX >= 11 && KX <= NDC_PACK_MAXKX) ? kPackAlways
         : (KX == 7 || KX == 9) ? kPackSingleSlice : kPackNever;
}

template <bool PK>
struct RowAcc {  // scalar: one partial sum per output column
  float v[kRX];
};
template <>
struct RowAcc<true> {  // packed: even-tap pairs a, odd-tap pairs b (columns 1..14), b0, b15
  float2 a[kRX / 2];
  float2 b[kRX / 2 - 1];
  float b0, b15;
};

__device__ __forceinline__ void row_zero(RowAcc<false>& r) {
#pragma unroll
  for (int c = 0; c < kRX; ++c) r.v[c] = 0.f;
}
__device__ __forceinline__ void row_zero(RowAcc<true>& r) {
#pragma unroll
  for (int c = 0; c < kRX / 2; ++c) r.a[c] = make_float2(0.f, 0.f);
#pragma unroll
  for (int c = 0; c < kRX / 2 - 1; ++c) r.b[c] = make_float2(0.f, 0.f);
  r.b0 = r.b15 = 0.f;
}
__device__ __forceinline__ void row_value(const RowAcc<false>& r, float (&o)[kRX]) {
#pragma unroll
  for (int c = 0; c < kRX; ++c) o[c] = r.v[c];
}
__device__ __forceinline__ void row_value(const RowAcc<true>& r, float (&o)[kRX]) {
#pragma unroll
  for (int c = 0; c < kRX / 2; ++c) {
    o[2 * c] = r.a[c].x;
    o[2 * c + 1] = r.a[c].y;
  }
  o[0] += r.b0;
#pragma unroll
  for (int c = 0; c < kRX / 2 - 1; ++c) {
    o[2 * c + 1] += r.b[c].x;
    o[2 * c + 2] += r.b[c].y;
  }
  o[kRX - 1] += r.b15;
}

// NR of the thread's RY row windows against every tap row of one staged plane.
template <int KX, int SH, int RY, int NR, bool STRIDED, bool PK>
__device__ __forceinline__ void accumulate_rows(RowAcc<PK> (&acc)[RY], const float* base,
                                                const float* trow, int KY, int ky0, int kys,
                                                int pitch_s) {
  constexpr int NQ = window_quads(KX, SH);
  constexpr int KXP = tap_pitch(KX);
  // Tap rows 0..KY-1 (STRIDED, edge tiles only: ky0, ky0 + kys, ...).  In the interior
  // kernel the induction variable is uniform, which keeps the tap loads on the uniform
  // datapath (LDCU -> FFMA R, R, UR).  Measured and not kept: unrolling this
  // loop (taps leave the uniform datapath, -10..30 %), a uniform loop with per-phase skips
  // for edge tiles (+3 % on config 3's forward).
#pragma unroll 1
  for (int ky = STRIDED ? ky0 : 0; ky < KY; ky += STRIDED ? kys : 1) {
    const float* w = trow + ky * KXP;
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
      if constexpr (PK) {
      static_assert(SH % 2 == 0, "window pairs must start at even registers");
      static_assert(kRX == 16, "column pairing assumes 16-column strips");
#pragma unroll
      for (int kx = 0; kx < KX; ++kx) {
        const float t = w[kx];
        const float* wv = win + SH + kx;
        if (kx % 2 == 0) {
#pragma unroll
          for (int c = 0; c < kRX / 2; ++c)
            acc[j].a[c] = __ffma2_rn(make_float2(t, t), make_float2(wv[2 * c], wv[2 * c + 1]), acc[j].a[c]);
        } else {
          acc[j].b0 = fmaf(t, wv[0], acc[j].b0);
#pragma unroll
          for (int c = 0; c < kRX / 2 - 1; ++c)
            acc[j].b[c] = __ffma2_rn(make_float2(t, t), make_float2(wv[2 * c + 1], wv[2 * c + 2]), acc[j].b[c]);
          acc[j].b15 = fmaf(t, wv[kRX - 1], acc[j].b15);
        }
      }
      } else {
#pragma unroll
      for (int kx = 0; kx < KX; ++kx) {
        const float t = w[kx];
#pragma unroll
        for (int c = 0; c < kRX; ++c) acc[j].v[c] = fmaf(t, win[SH + c + kx], acc[j].v[c]);
      }
      }
    }
  }
}

#ifndef NDC_MIN_BLOCKS
#define NDC_MIN_BLOCKS 2
#endif
#ifndef NDC_SMALL_MIN_BLOCKS
#define NDC_SMALL_MIN_BLOCKS 5
#endif
#ifndef NDC_STAGED_KX
#define NDC_STAGED_KX kStagedMaxKX  // staged (coalesced) epilogue up to this kernel x-extent
#endif
#ifndef NDC_SMALL_KX
#define NDC_SMALL_KX kSmallMaxKX
#endif
#ifndef NDC_NOSTAGING_DIRECT
#define NDC_NOSTAGING_DIRECT 1  // direct-epilogue kernels allocate no staging buffer
#endif
#ifndef NDC_PREFETCH_KX
#define NDC_PREFETCH_KX kPrefetchMaxKX  // cp.async aux_in prefetch (single-plane PSFs) up to this KX
#endif
// Small kernels (KX <= NDC_SMALL_KX) are HBM-bound: more resident CTAs per SM keep more
// tile loads in flight.
template <int KX>
constexpr int min_blocks_for() { return KX <= NDC_SMALL_KX ? NDC_SMALL_MIN_BLOCKS : NDC_MIN_BLOCKS; }
#ifndef NDC_DIRECT_MIN_BLOCKS
#define NDC_DIRECT_MIN_BLOCKS 3
#endif
// Residency target per instantiation: the scalar direct-epilogue 128-row (RY = 2) kernels
// of large PSFs (config 2) ask for 3 CTAs / SM -- 80 registers, no spills, and their shared
// memory carries no staging buffer (3 x 63 KB).  Measured (tools/kbench.py): config 2
// +0.4..0.8 %, 2048^2 x 16 with 25 x 25 taps +1..5 %; the 64-row 3-D kernels (config 5)
// lose 0.8 % at 3 and keep 2.
template <int KX, int RY, bool EDGE, bool PK>
constexpr int min_blocks_of() {
  return (RY == 2 && !PK && !EDGE && KX > NDC_STAGED_KX && KX > NDC_PREFETCH_KX) ? NDC_DIRECT_MIN_BLOCKS
                                                                                 : min_blocks_for<KX>();
}

// EDGE = false: the full tiles (tx < full_tx, ty < full_ty).  EDGE = true: the partial
// tiles of extents that are not tile multiples (last tile column / row).  An edge tile has
// only S < 4 column strips / R < 2 row blocks with outputs; its 8 warps are spread over
// the S*R active (strip, block) pairs and the warps sharing a pair split the tap rows
// (phase, nph), folded through shared memory before the epilogue -- an edge CTA then
// finishes in proportion to its work instead of holding an SM slot for a full tile's
// time with idle warps (config 3 forward: 47 -> 52 TFLOP/s).  Two instantiations keep the
// interior kernel's code free of the edge logic (sharing it moved the taps off the
// uniform datapath: -12 % on config 4).
template <int KX, int SH, int RY, bool EDGE, bool PK>
__global__ void __launch_bounds__(kThreads, (min_blocks_of<KX, RY, EDGE, PK>()))
    correlate_kernel(const __grid_constant__ CUtensorMap map, const CorrGeom g, const CorrArgs a,
                     const __grid_constant__ TapBlock taps) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  constexpr int TY = 64 * RY;
  constexpr bool kStagedEpi = KX <= NDC_STAGED_KX || KX <= NDC_PREFETCH_KX;
  // 64-row staged kernels (the HBM-bound small PSFs): single-plane launches come as a 2-D
  // grid of tiles (bit 1 of g.aux_prefetch; no tile-index division) and skip the plane ring
  constexpr bool kLean2D = kStagedEpi && RY == 1 && !EDGE;
  const bool grid2d = kLean2D && (g.aux_prefetch & 2) != 0;

  const int b = blockIdx.z;
  if (a.active != nullptr && a.active[b] == 0) return;
  int oz = blockIdx.y;
  int txi, tyi;
  if (!EDGE && grid2d) {
    oz = 0;
    txi = blockIdx.x;
    tyi = blockIdx.y;
  } else if (!EDGE) {
    int t = blockIdx.x;
    if (NDC_Z_FAST && gridDim.y > 1) {
      // 3-D: consecutive CTAs take consecutive output planes of one tile position, so the
      // KZ input planes they stage are shared in L2 instead of re-read from DRAM.
      const int lin = blockIdx.y * gridDim.x + blockIdx.x;
      oz = lin % gridDim.y;
      t = lin / gridDim.y;
    }
    txi = t % g.full_tx;
    tyi = t / g.full_tx;
  } else {
    const int ncol = g.tiles_x - g.full_tx;  // 0 or 1 partial tile columns
    const int e = blockIdx.x;
    if (e < ncol * g.tiles_y) {
      txi = g.full_tx + e / g.tiles_y;
      tyi = e % g.tiles_y;
    } else {
      const int e2 = e - ncol * g.tiles_y;
      tyi = g.full_ty + e2 / g.full_tx;
      txi = e2 % g.full_tx;
    }
  }
  const int tile = tyi * g.tiles_x + txi;
  const int tx0 = txi * kTileX;
  const int ty0 = tyi * TY;
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  // warp index broadcast from lane 0 so the compiler treats per-warp decisions as
  // warp-uniform (keeps the tap loads on the uniform datapath under those branches)
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  int wx = warp & 3, wy = warp >> 2, pw = warp, phase = 0, nph = 1, P = 8;
  // Per-lane placement: output row offset within the tile and column offset of the lane's
  // 16-column strip.  Normally a warp is 32 consecutive rows of one strip; in a COMPACT
  // edge tile (<= 16 rows left: the bottom tile row of e.g. config 3's 270-row or config
  // 4's 1032-row forward output) a warp is LR = 8 or 16 rows x 32/LR strips, so its lanes
  // are not idle on rows past the extent.  A quarter-warp is still 8 consecutive rows of
  // one strip (bank-conflict-free loads).
  int lane_row = 0, lane_col = 0;
  bool compact = false;
  if constexpr (EDGE) {
    const int S = min(4, (g.out_ex - tx0 + kRX - 1) / kRX);
    const int rows_left = g.out_ey - ty0;
    compact = rows_left <= 16;
    if (compact) {
      const int LR = rows_left <= 8 ? 8 : 16;
      const int spw = 32 / LR;             // strips per warp
      P = (S + spw - 1) / spw;             // warp units
      pw = __shfl_sync(0xffffffffu, warp % P, 0);
      phase = __shfl_sync(0xffffffffu, warp / P, 0);
      nph = (7 - pw) / P + 1;
      wx = 0;
      wy = 0;
      lane_row = lane % LR;
      lane_col = (pw * spw + lane / LR) * kRX;
    } else {
      const int R = min(2, (rows_left + 32 * RY - 1) / (32 * RY));
      P = S * R;
      pw = __shfl_sync(0xffffffffu, warp % P, 0);
      phase = __shfl_sync(0xffffffffu, warp / P, 0);
      nph = (7 - pw) / P + 1;
      wx = __shfl_sync(0xffffffffu, pw % S, 0);
      wy = __shfl_sync(0xffffffffu, pw / S, 0);
    }
  }
  if constexpr (EDGE) {
    if (!compact) {
      lane_row = wy * (32 * RY) + lane;
      lane_col = wx * kRX;
    }
  }

  // Tap slices whose input plane iz = oz + kz + off_z exists (out-of-range planes are
  // skipped, which also balances edge z-slabs).
  const int kzA = max(g.kz0, -oz - g.off_z);
  const int kzB = min(g.kz1, g.in_ez - oz - g.off_z);
  const int n = kzB - kzA;

  const int sbytes = stage_bytes_aligned(g.rows, g.pitch_s);
  constexpr bool kStaging = KX <= NDC_STAGED_KX || KX <= NDC_PREFETCH_KX || !NDC_NOSTAGING_DIRECT;
  // Launches that prefetch the epilogue operand (single-plane small PSFs) carry per-warp
  // prefetch buffers after the barriers; those double as the staging buffers, so such a
  // launch has no separate staging area (16 KB less per CTA).
  const bool prebuf = KX <= NDC_PREFETCH_KX && (g.aux_prefetch & 1) != 0;
  const int bar_off = barrier_offset(g.stages, sbytes, kStaging && !prebuf);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + bar_off);
  float* const wbuf = reinterpret_cast<float*>(smem_raw + bar_off + 128) + warp * (RY * 32 * kRX);
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

  // Small PSFs: prefetch the epilogue's aux_in strip (Y or x) into shared memory now,
  // so it arrives during the FFMA loop instead of stalling the epilogue.
  const float* wpre = nullptr;
  // (not with earlier tap chunks to add: their partial sums are staged through the same buffer)
  if (prebuf && g.final_chunk && !g.accum && mode_reads_aux_rt(g.mode) && phase == 0 && !(EDGE && compact)) {
    float* pre = wbuf;
    const int ox0 = tx0 + wx * kRX;
    const long long obase = static_cast<long long>(b) * g.out_image +
                            static_cast<long long>(g.out_z0 + oz) * g.out_plane + ox0;
    if (ox0 < g.out_ex) {
      // row 8k + (lane >> 2) of block j: one running pointer, stage_pos(r, q) = stage_pos(r0, q) + 128 k
      const int r0 = lane >> 2, q = lane & 3;
      const int row_first = ty0 + wy * (32 * RY) + r0;
      const float* src = a.aux_in + obase + static_cast<long long>(row_first) * g.out_pitch + 4 * q;
      float* dst = pre + stage_pos(r0, q);
#pragma unroll
      for (int k = 0; k < 4 * RY; ++k) {
        if (row_first + 8 * k < g.out_ey) cp_async16(dst + 8 * kRX * k, src);
        src += 8 * g.out_pitch;
      }
    }
    cp_async_commit();
    wpre = pre;
  }

  RowAcc<PK> acc2[RY];
#pragma unroll
  for (int j = 0; j < RY; ++j) row_zero(acc2[j]);

  // Rows blocks / column strips entirely outside the output (the last tiles of an
  // extent that is not a tile multiple) skip their FFMAs; the test is warp-uniform.
  int nrun = 0;
#pragma unroll
  for (int j = 0; j < RY; ++j)
    if (ty0 + wy * (32 * RY) + 32 * j < g.out_ey) nrun = j + 1;
  if (tx0 + wx * kRX >= g.out_ex) nrun = 0;
  if (EDGE && compact) nrun = 1;  // rows 0..15 of block 0 only; inactive lanes are masked at the end
  if (grid2d) {  // one plane, one stage
    mbar_wait(&bars[0], 0u);
    if (nrun != 0) {
      const float* base = reinterpret_cast<const float*>(smem_raw) + (wy * (32 * RY) + lane) * g.pitch_s + wx * kRX;
      accumulate_rows<KX, SH, RY, RY, EDGE, PK>(acc2, base, taps.t, g.KY, phase, nph, g.pitch_s);
    }
  } else
  for (int i = 0; i < n; ++i) {
    // ring slot and mbarrier parity of staged plane i (a runtime i % stages and i / stages
    // cost ~40 instructions per plane; plans use one or two stages)
    int s;
    uint32_t parity;
    if (g.stages == 2) {
      s = i & 1;
      parity = static_cast<uint32_t>(i >> 1) & 1u;
    } else if (g.stages == 1) {
      s = 0;
      parity = static_cast<uint32_t>(i) & 1u;
    } else {
      s = i % g.stages;
      parity = static_cast<uint32_t>(i / g.stages) & 1u;
    }
    mbar_wait(&bars[s], parity);
    const float* base =
        EDGE ? reinterpret_cast<const float*>(smem_raw + s * sbytes) + lane_row * g.pitch_s + lane_col
             : reinterpret_cast<const float*>(smem_raw + s * sbytes) + (wy * (32 * RY) + lane) * g.pitch_s + wx * kRX;
    const float* trow = taps.t + (kzA + i - g.kz0) * g.KY * tap_pitch(KX);
    if (nrun == RY)
      accumulate_rows<KX, SH, RY, RY, EDGE, PK>(acc2, base, trow, g.KY, phase, nph, g.pitch_s);
    else if (RY > 1 && nrun == 1)
      accumulate_rows<KX, SH, RY, 1, EDGE, PK>(acc2, base, trow, g.KY, phase, nph, g.pitch_s);
    if (i + g.stages < n) {
      // Every warp is done with stage s before it is refilled.  Edge tiles: their warps split
      // the tap rows unevenly (15 rows over 4 phases: 4 / 4 / 4 / 3), so only warp 0, which
      // issues the refill, waits (named barrier 1 + s); the others signal and go on to the
      // next stage (ncu, config 3 edge launch: barrier stalls 1.2 per issued instruction).
      // The full-tile kernels keep the plain barrier: with any split form ptxas moves
      // config 4's tap loads off the uniform datapath (profiles/r02e_tap_loop_probes.md).
      if constexpr (EDGE) {
        // (literal barrier ids: with a register id ptxas reserves all 16 barriers per CTA)
        if (s == 0) {
          if (warp != 0) bar_arrive<1>(); else bar_sync<1>();
        } else if (s == 1) {
          if (warp != 0) bar_arrive<2>(); else bar_sync<2>();
        } else {
          if (warp != 0) bar_arrive<3>(); else bar_sync<3>();
        }
      } else {
        __syncthreads();
      }
      if (tid == 0) {
        const int iz = oz + kzA + i + g.stages + g.off_z;
        mbar_expect_tx(&bars[s], tx_bytes);
        tma_load_3d(smem_raw + s * sbytes, &map, &bars[s], tx0 + g.off_x, ty0 + g.off_y,
                    b * g.in_ez + iz);
      }
    }
  }

  float acc[RY][kRX];
#pragma unroll
  for (int j = 0; j < RY; ++j) row_value(acc2[j], acc[j]);

  if (EDGE && P < 8) {
    // fold the tap-row phases of each (strip, block) pair into its phase-0 warp, in
    // phase order (deterministic), through the now idle stage buffers
    __syncthreads();  // every warp is past its last staged plane
    float* red = reinterpret_cast<float*>(smem_raw);
    if (phase > 0) {
#pragma unroll
      for (int j = 0; j < RY; ++j)
#pragma unroll
        for (int q = 0; q < kRX / 4; ++q)
          *reinterpret_cast<float4*>(red + (warp * RY + j) * (32 * kRX) + stage_pos(lane, q)) =
              make_float4(acc[j][4 * q], acc[j][4 * q + 1], acc[j][4 * q + 2], acc[j][4 * q + 3]);
    }
    __syncthreads();
    if (phase == 0) {
      for (int k = 1; k < nph; ++k) {
        const int w2 = pw + k * P;
#pragma unroll
        for (int j = 0; j < RY; ++j)
#pragma unroll
          for (int q = 0; q < kRX / 4; ++q) {
            const float4 v =
                *reinterpret_cast<const float4*>(red + (w2 * RY + j) * (32 * kRX) + stage_pos(lane, q));
            acc[j][4 * q] += v.x;
            acc[j][4 * q + 1] += v.y;
            acc[j][4 * q + 2] += v.z;
            acc[j][4 * q + 3] += v.w;
          }
      }
    }
  }

  // ---- epilogue (one instantiation per mode: the dispatch happens once per tile) --------
  float* wst = prebuf ? wbuf : reinterpret_cast<float*>(smem_raw + g.stages * sbytes) + warp * (32 * kRX);
  const int wst_stride = prebuf ? 32 * kRX : 0;
  double p0 = 0.0, p1 = 0.0;
  // (compact edge tiles: per-lane row / strip, so the lane-per-row direct epilogue; its
  // row is wrow0 + lane, hence the per-lane wrow0)
#define NDC_EPI(M)                                                                                      \
  if (EDGE && compact)                                                                                \
    epilogue_tile<M, RY, false>(g, a, b, oz, tx0 + lane_col, ty0 + lane_row - lane, lane, acc, wst, 0, nullptr, \
                                p0, p1);                                                                \
  else                                                                                                \
    epilogue_tile<M, RY, (KX <= NDC_STAGED_KX || KX <= NDC_PREFETCH_KX)>(g, a, b, oz, tx0 + wx * kRX, ty0 + wy * (32 * RY), lane, acc, \
                                               wst, wst_stride, wpre, p0, p1)
  switch (phase != 0 ? -2 : g.final_chunk ? g.mode : -1) {  // -2: folded into a phase-0 warp
    case kEpiStore: NDC_EPI(kEpiStore); break;
    case kEpiResid: NDC_EPI(kEpiResid); break;
    case kEpiNorm: NDC_EPI(kEpiNorm); break;
    case kEpiPG: NDC_EPI(kEpiPG); break;
    case kEpiKKT: NDC_EPI(kEpiKKT); break;
    case kEpiClamp: NDC_EPI(kEpiClamp); break;
    case kEpiRLRatio: NDC_EPI(kEpiRLRatio); break;
    case kEpiRLUpdate: NDC_EPI(kEpiRLUpdate); break;
    case -1: NDC_EPI(-1); break;
    default: break;
  }
#undef NDC_EPI

  if (a.partials != nullptr) {
    // one partial per warp, written without a CTA barrier (finalize reduces them in a
    // fixed order, so the result stays deterministic)
    const bool pmax = p0_is_max(g.mode);
    p0 = pmax ? warp_max(p0) : warp_sum(p0);
    // (staged kernels: only the modes that produce p1 reduce it; the others leave it 0)
    if (!kStagedEpi || g.mode == kEpiPG || g.mode == kEpiRLUpdate) p1 = warp_sum(p1);
    if (lane == 0) {
      const long long idx =
          ((static_cast<long long>(b) * (grid2d ? 1 : gridDim.y) + oz) * (g.tiles_x * g.tiles_y) + tile) *
              (kThreads / 32) + warp;
      a.partials[idx] = make_double2(p0, p1);
    }
  }
}

template <int KX, int SH, int RY>
cudaError_t launch_kx(const CUtensorMap& map, const CorrGeom& g, const CorrArgs& a,
                      const TapBlock& taps, int batch, int nz_out, cudaStream_t s, cudaStream_t s_edge) {
  // staged (small-PSF) kernels add the per-warp aux_in prefetch buffers
  constexpr bool kStaging = KX <= NDC_STAGED_KX || KX <= NDC_PREFETCH_KX || !NDC_NOSTAGING_DIRECT;
  // (launches with the per-warp operand-prefetch buffers stage their stores through them)
  const bool prebuf = KX <= NDC_PREFETCH_KX && (g.aux_prefetch & 1) != 0;
  const size_t smem = correlate_smem_bytes(g, kStaging && !prebuf) +
                      (prebuf ? 128 + (kThreads / 32) * RY * 32 * kRX * 4 : 0);
  // packed FFMA2 tap loop (see pack_mode): edge tiles only where it is always on
  constexpr int kPM = pack_mode<KX>();
  constexpr bool kPkFull = kPM != kPackNever, kPkEdge = kPM == kPackAlways;
  const bool pk = kPM == kPackAlways || (kPM == kPackSingleSlice && g.kz1 - g.kz0 == 1);
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(correlate_kernel<KX, SH, RY, false, false>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e == cudaSuccess && kPkFull)
      e = cudaFuncSetAttribute(correlate_kernel<KX, SH, RY, false, kPkFull>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(correlate_kernel<KX, SH, RY, true, kPkEdge>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    // 3-CTA kernels (min_blocks_of): full shared-memory carveout so the third CTA fits
    // (the 64-row 3-D kernels keep the default: config 5 measured -1 % with it)
    if (e == cudaSuccess && min_blocks_of<KX, RY, false, false>() >= 3)
      e = cudaFuncSetAttribute(correlate_kernel<KX, SH, RY, false, false>,
                               cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  // full tiles, then the partial last tile column / row
  const int n_full = g.full_tx * g.full_ty;
  const int n_edge = g.tiles_x * g.tiles_y - n_full;
  // narrow 3-D PSFs: two output planes per CTA (ndc_correlate_pair.cuh)
  constexpr bool kPairKernel = RY == 2 && (KX == 7 || KX == 9);
  if (kPairKernel && n_full > 0 && nz_out >= 2 && g.kz1 - g.kz0 >= 2 && !pk) {
    if (cudaError_t e = launch_correlate_pair(KX, SH, map, g, a, taps, batch, nz_out, s); e != cudaSuccess) return e;
  } else if (n_full > 0) {
    dim3 grid(n_full, nz_out, batch);
    // 64-row staged kernels, single-plane launch: a 2-D grid of tiles (see kLean2D)
    constexpr bool kLean2D = (KX <= NDC_STAGED_KX || KX <= NDC_PREFETCH_KX) && RY == 1;
    CorrGeom g2 = g;
    // (exactly one staged plane per tile: kzA = 0, n = 1 in the kernel)
    if (kLean2D && nz_out == 1 && g.in_ez == 1 && g.kz0 == 0 && g.kz1 == 1 && g.stages == 1 && g.off_z == 0 &&
        g.full_ty <= 65535) {
      g2.aux_prefetch |= 2;
      grid = dim3(g.full_tx, g.full_ty, batch);
    }
    if (pk)
      correlate_kernel<KX, SH, RY, false, kPkFull><<<grid, kThreads, smem, s>>>(map, g2, a, taps);
    else
      correlate_kernel<KX, SH, RY, false, false><<<grid, kThreads, smem, s>>>(map, g2, a, taps);
    if (cudaError_t e = cudaGetLastError(); e != cudaSuccess) return e;
  }
  if (n_edge > 0)
    correlate_kernel<KX, SH, RY, true, kPkEdge><<<dim3(n_edge, nz_out, batch), kThreads, smem, s_edge>>>(map, g, a,
                                                                                                      taps);
  return cudaGetLastError();
}

#define NDC_KX_SWITCH(SH, RY)                                              \
  switch (kx) {                                                            \
    case 1: return launch_kx<1, SH, RY>(map, g, a, taps, batch, nz_out, s, s_edge);   \
    case 3: return launch_kx<3, SH, RY>(map, g, a, taps, batch, nz_out, s, s_edge);   \
    case 5: return launch_kx<5, SH, RY>(map, g, a, taps, batch, nz_out, s, s_edge);   \
    case 7: return launch_kx<7, SH, RY>(map, g, a, taps, batch, nz_out, s, s_edge);   \
    case 9: return launch_kx<9, SH, RY>(map, g, a, taps, batch, nz_out, s, s_edge);   \
    case 11: return launch_kx<11, SH, RY>(map, g, a, taps, batch, nz_out, s, s_edge); \
    case 13: return launch_kx<13, SH, RY>(map, g, a, taps, batch, nz_out, s, s_edge); \
    case 15: return launch_kx<15, SH, RY>(map, g, a, taps, batch, nz_out, s, s_edge); \
    case 17: return launch_kx<17, SH, RY>(map, g, a, taps, batch, nz_out, s, s_edge); \
    case 19: return launch_kx<19, SH, RY>(map, g, a, taps, batch, nz_out, s, s_edge); \
    case 21: return launch_kx<21, SH, RY>(map, g, a, taps, batch, nz_out, s, s_edge); \
    case 23: return launch_kx<23, SH, RY>(map, g, a, taps, batch, nz_out, s, s_edge); \
    case 25: return launch_kx<25, SH, RY>(map, g, a, taps, batch, nz_out, s, s_edge); \
    case 27: return launch_kx<27, SH, RY>(map, g, a, taps, batch, nz_out, s, s_edge); \
    case 29: return launch_kx<29, SH, RY>(map, g, a, taps, batch, nz_out, s, s_edge); \
    case 31: return launch_kx<31, SH, RY>(map, g, a, taps, batch, nz_out, s, s_edge); \
    case 33: return launch_kx<33, SH, RY>(map, g, a, taps, batch, nz_out, s, s_edge); \
    default: return cudaErrorInvalidValue;                                 \
  }

}  // namespace corr
}  // namespace ndc
