// Internal declarations shared by the device kernels (ndc_kernels.cu), the plan /
// projected-gradient driver (ndc_plan.cu) and the C-ABI (ndc_capi.cu).
//
// Device layout: every volume is stored as
// [image b][plane z][row y][pitch x] float32, with the x pitch rounded up to a
// multiple of kTileX floats so every output tile lies inside its row and every
// row starts 256-byte aligned.  Pad columns are kept at zero.  1-D and 2-D problems
// are the 3-D case with leading extents 1; the batch of independent images (BASELINE
// config 2) is the outermost index.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

namespace ndc {

// Output tile owned by one CTA: kTileY rows x kTileX columns of one output plane.
// 256 threads = 8 warps; warp w covers columns 16*(w&3).. and rows 32*(w>>2)..;
// lane l owns output row 32*(w>>2)+l and 16 consecutive columns (kRX).
constexpr int kTileX = 64;
constexpr int kTileY = 64;
constexpr int kRX = 16;
constexpr int kThreads = 256;
constexpr int kMaxKX = 33;        // largest x-extent with a register-window instantiation
constexpr int kMaxRows = 256;     // TMA box limit on rows: kTileY + KY - 1 <= 256
#ifndef NDC_TAP_CAP
#define NDC_TAP_CAP 7680
#endif
constexpr int kTapCap = NDC_TAP_CAP;  // taps per launch carried in the kernel parameter block
constexpr int kMaxStages = 3;
constexpr int kMaxDims = 8;  // tensor dimensions accepted (4+ merge into the plane axis)
// HBM-bound small PSFs (ndc_correlate.cuh): kernel x-extents up to kStagedMaxKX use the
// staged, sector-complete epilogue (and, for single-plane problems, a cp.async prefetch
// of the epilogue's aux_in strip); up to kSmallMaxKX also 64-row tiles at 5 CTAs / SM.
constexpr int kStagedMaxKX = 9;
constexpr int kSmallMaxKX = 5;
// Single-plane PSFs up to kPrefetchMaxKX prefetch the epilogue's aux_in strip with
// cp.async at kernel start (its global-load latency otherwise stalls every warp at the
// end of a tile).
#ifndef NDC_PREFETCH_MAXKX
#define NDC_PREFETCH_MAXKX 9
#endif
constexpr int kPrefetchMaxKX = NDC_PREFETCH_MAXKX;

// Epilogue selector (uniform per launch).
enum EpiMode : int {
  kEpiStore = 0,   // out = acc * scale[b]
  kEpiResid = 1,   // out = acc - Y ; part0 += out^2            (forward, objective)
  kEpiNorm = 2,    // out = acc * scale[b] ; part0 += out^2     (power iteration)
  kEpiPG = 3,      // g = acc ; trial = max(x - step[b]*g, 0) -> out ; g -> aux_out ;
                   //   part0 = max |min(x,g)| ; part1 += (trial != x)
  kEpiKKT = 4,     // part0 = max |min(x, acc)|                (final KKT, kkt_residual)
  kEpiClamp = 5,   // out = max(acc, 0)                          (x0 = clamp(A^T y))
  kEpiRLRatio = 6, // v = acc*scale ; out = |v| < 1e-12 ? 0 : Y / v ; part0 += (v - Y)^2
                   //   (Richardson-Lucy: forward pass fused with guarded_div)
  kEpiRLUpdate = 7 // u = acc ; xn = x * u -> out ; part0 += (xn - x)^2 ; part1 += x^2
};

// Correlation geometry for one launch (grid.y = number of computed output planes):
//   out[b][out_z0+oz][oy][ox] =
//     sum_{kz,ky,kx} taps[kz][ky][kx] * in[b][oz+kz+off_z][oy+ky+off_y][ox+kx+off_x]
// with `in` read as zero outside its extents (TMA out-of-bounds fill; planes outside
// [0, in_ez) are skipped).
struct CorrGeom {
  int in_ez, in_ey, in_ex;   // input buffer extents (planes held locally, rows, columns)
  int in_row0;               // tensor row of input data row 0 (zero margin above it)
  int out_ey, out_ex;        // output rows / columns (valid region)
  int out_z0;                // buffer plane of computed output plane 0 (z-slab offset)
  int off_z, off_y, off_x;   // input coordinate = computed index + tap + off
  int KY;              // tap rows per z-slice
  int kz0, kz1;        // z-slices of the taps carried by this launch
  int tiles_x, tiles_y;
  int full_tx, full_ty;  // tile columns / rows wholly inside the output
  int rows, pitch_s;   // shared tile: rows x pitch_s floats per stage
  int stages;
  int aux_prefetch;    // bit 0: cp.async the epilogue's aux_in strip at kernel start (small PSFs);
                       // bit 1 (set by the launcher): single-plane launch as a 2-D grid of tiles
  int accum;           // add the partial sum held in `accum_in`
  int mode;            // EpiMode (ignored unless final)
  int final_chunk;     // last tap chunk: apply the epilogue
  long long out_pitch, out_plane, out_image;  // in floats
};
// (a launch covering a subset of a pass's planes shifts out_z0 / off_z and the partials
// pointer on the host; the kernel's plane index stays blockIdx.y -- measured: reading a
// plane offset from the parameters costs the small-PSF kernels ~1.5 %)

struct CorrArgs {
  float* out;             // main output (x- or y-shaped per direction)
  float* aux_out;         // kEpiPG: gradient g
  const float* aux_in;    // Y (resid / RL ratio) or x (PG / KKT / RL update)
  const float* accum_in;  // partial sums of earlier tap chunks
  const float* scale;     // per-image scale (kEpiStore/kEpiNorm/kEpiRLRatio) or null
  const double* step;     // per-image PG step (kEpiPG)
  const int* active;      // per-image active flag, null = all
  double2* partials;      // per-CTA reduction partials [b][oz][tile]
};

struct TapBlock {
  float t[kTapCap];
};

// Tap rows are stored with an even pitch (64-bit aligned pairs in the parameter bank).
__host__ __device__ constexpr int tap_pitch(int kx) { return (kx + 1) & ~1; }

// Launch the correlation kernel for one tap chunk; sh (0 or 2) is the register-window
// shift that keeps the TMA tile start 16-byte aligned, ry (1 or 2) the output rows per
// thread (tile height 64*ry).  The full tiles run on stream s, the partial edge tiles
// (a second launch) on s_edge, which may be a different stream so the edge CTAs fill the
// SMs freed by the full-tile launch's last wave.
cudaError_t launch_correlate(int kx, int sh, int ry, const CUtensorMap& map, const CorrGeom& g,
                             const CorrArgs& a, const TapBlock& taps, int batch, int nz_out,
                             cudaStream_t s, cudaStream_t s_edge);
#define NDC_DECL_CORR(SH, RY)                                                               \
  cudaError_t launch_correlate_sh##SH##_ry##RY(int kx, const CUtensorMap& map,             \
                                               const CorrGeom& g, const CorrArgs& a,       \
                                               const TapBlock& taps, int batch, int nz_out, \
                                               cudaStream_t s, cudaStream_t s_edge);
NDC_DECL_CORR(0, 1)
NDC_DECL_CORR(0, 2)
NDC_DECL_CORR(2, 1)
NDC_DECL_CORR(2, 2)
#undef NDC_DECL_CORR
// Full tiles of a 3-D launch with two output planes per CTA (ndc_correlate_pair.cuh):
// narrow PSFs (kx = 7, 9) on 128-row tiles.
cudaError_t launch_correlate_pair(int kx, int sh, const CUtensorMap& map, const CorrGeom& g, const CorrArgs& a,
                                  const TapBlock& taps, int batch, int nz_out, cudaStream_t s);
size_t correlate_smem_bytes(const CorrGeom& g, bool staging);
int shared_pitch_for(int kx, int sh);

// Small kernels.
enum FinalizeOp : int {
  kFinHalfSum = 0,   // out0 = 0.5*sum(p0)                 (objective)
  kFinNorm = 1,      // out0 = sqrt(sum(p0)) ; scale = 1/out0 (power iteration)
  kFinMaxSum = 2,    // out0 = max(p0) ; out1 = sum(p1)     (kkt, changed count)
  kFinSumSum = 3     // out0 = sum(p0) ; out1 = sum(p1)
};
cudaError_t launch_finalize(const double2* partials, long long per_image, int batch, int op,
                            double* out0, double* out1, float* scale_out, const int* active,
                            cudaStream_t s);
cudaError_t launch_combine(const double* gathered, int world, int op, double* out0, double* out1,
                           float* scale_out, cudaStream_t s);
// Interior view of a pitched volume (pointers passed alongside are at the interior
// origin): ez planes of ey rows of ex valid floats; strides in floats.
struct Geo {
  int ez, ey, ex;
  long long pitch, plane, image;
};
cudaError_t launch_pg_trial(const float* x, const float* g, float* trial, const double* step,
                            const int* active, double2* partials, int batch, const Geo& v,
                            int blocks_per_image, cudaStream_t s);
cudaError_t launch_fill(float* dst, float value, int batch, const Geo& v, cudaStream_t s);
// float64 dense correlation (small-problem reference-exact power iteration)
cudaError_t launch_corr_f64(const double* in, int iz, int iy, int ix, double* out, int oz, int oy,
                            int ox, const double* taps, int KZ, int KY, int KX, int dz, int dy,
                            int dx, const double* lam_prev, double2* partials, long long* nblocks,
                            cudaStream_t s);
cudaError_t launch_fill_f64(double* dst, double value, long long n, cudaStream_t s);
cudaError_t launch_pack_f64(const double* dense, float* pitched, int batch, const Geo& v,
                            cudaStream_t s);
cudaError_t launch_unpack_f64(const float* pitched, double* dense, int batch, const Geo& v,
                              cudaStream_t s);
cudaError_t launch_pack_f32(const float* dense, float* pitched, int batch, const Geo& v,
                            cudaStream_t s);
cudaError_t launch_unpack_f32(const float* pitched, float* dense, int batch, const Geo& v,
                              cudaStream_t s);
cudaError_t launch_clamp_count(const float* src, float* dst, double2* partials, int batch,
                               const Geo& v, int blocks_per_image, cudaStream_t s);

// Driver-API entry for TMA descriptor encoding (resolved through the runtime, no -lcuda).
CUresult encode_tensor_map(CUtensorMap* map, const float* base, int ex, int ey, long long zcount,
                           long long pitch, long long plane, int box_x, int box_y);

}  // namespace ndc
