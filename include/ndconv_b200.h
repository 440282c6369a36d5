/*
 * ndconv_b200.h -- C-ABI drop-in boundary for the ndconv projected-gradient hot path
 * on NVIDIA B200 (sm_100a).  Library: paper_1711_11224_b200/libndconv_b200.so.
 *
 * Every entry point replaces one function of the reference's header-only C++ API
 * (/root/reference/proj/include/ndconv/, cited per declaration).  Plain pointers and
 * sizes only: host tensors are dense row-major (first index slowest, shape.hpp:55-64)
 * arrays of double exactly as the reference's Tensor stores them (tensor.hpp:22-66);
 * kernels are dense arrays with odd extents (kernel.hpp:15-37).  The device path
 * computes in float32 with float64 reductions; results match the
 * reference within the parity tolerances stated there (1e-5 relative L2 per
 * convolution, 1e-4 after the full iteration count).
 *
 * Errors: every function returns an ndc_status.  NDC_ERR_CONFIG, NDC_ERR_SHAPE,
 * NDC_ERR_NUMERIC and NDC_ERR_BOUNDS correspond one to one to the reference's
 * ndconv::Error, ShapeError, NumericError and BoundsError (error.hpp:8-30);
 * ndc_last_error() returns the thread's last message.  There is no CPU fallback:
 * without a usable B200 the compute entry points return NDC_ERR_NO_DEVICE.
 *
 * Supported operands on the device path: 1 <= ndim <= 3 (plus the batch index of
 * the *_batch entry points) and odd kernels of any size (PSFs beyond one launch's tap
 * block -- 33 columns, the rows of one TMA box, 7680 taps -- run as several accumulated
 * launches).
 */
#ifndef NDCONV_B200_H
#define NDCONV_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

typedef enum ndc_status {
  NDC_OK = 0,
  NDC_ERR_CONFIG = 1,      /* ndconv::Error        (solvers.hpp:65-76)          */
  NDC_ERR_SHAPE = 2,       /* ndconv::ShapeError   (kernel.hpp:20, convolution.hpp:31,169) */
  NDC_ERR_NUMERIC = 3,     /* ndconv::NumericError (solvers.hpp:130-139, 159-160) */
  NDC_ERR_BOUNDS = 4,      /* ndconv::BoundsError  (shape.hpp:68-76)             */
  NDC_ERR_UNSUPPORTED = 5, /* shape/kernel outside the device path's limits       */
  NDC_ERR_CUDA = 6,
  NDC_ERR_NCCL = 7,
  NDC_ERR_NO_DEVICE = 8,
  NDC_ERR_ARGUMENT = 9,    /* null pointer / capacity too small                    */
  NDC_ERR_FORMAT = 10      /* ndconv::FormatError  (imageio.hpp: bad / truncated files) */
} ndc_status;

/* solvers.hpp:37-46 */
typedef enum ndc_stop_reason {
  NDC_STOP_CONVERGED = 0,
  NDC_STOP_MAX_ITERS = 1,
  NDC_STOP_STALLED = 2
} ndc_stop_reason;

/* ndconv::DeconvConfig (solvers.hpp:20-28).  has_initial_step == 0 is the
 * reference's empty std::optional (step estimated by power iteration). */
typedef struct ndc_deconv_config {
  size_t max_iters;          /* default 500  */
  double tol_rel_objective;  /* default 1e-6 */
  int has_initial_step;      /* default 0    */
  double initial_step;
  double backtrack_factor;   /* default 0.5  */
  size_t max_backtracks;     /* default 50   */
  size_t power_iters;        /* default 30   */
} ndc_deconv_config;

/* ndconv::RlConfig (solvers.hpp:30-35) */
typedef struct ndc_rl_config {
  size_t max_iters;       /* default 500 */
  double tol_rel_change;  /* default 0.0 */
} ndc_rl_config;

/* ndconv::DeconvReport (solvers.hpp:48-61) minus the tensors, which the caller
 * passes as arrays.  trace_len == objective_trace.size() == kkt_trace.size(). */
typedef struct ndc_deconv_report {
  size_t iterations_run;
  int stop_reason;               /* ndc_stop_reason */
  double wall_time_seconds;
  size_t negative_pixels_clamped;
  size_t trace_len;
  size_t backtracks;             /* rejected trial steps (diagnostic, not in the reference) */
  double step0;                  /* the step actually used (1/lambda or initial_step) */
} ndc_deconv_report;

void ndc_deconv_config_default(ndc_deconv_config* cfg);
void ndc_rl_config_default(ndc_rl_config* cfg);

const char* ndc_last_error(void);
const char* ndc_version(void);
const char* ndc_stop_reason_name(int reason);   /* solvers.hpp:39-46 to_string */

/* Number of usable sm_100 devices; 0 when none (status still NDC_OK). */
ndc_status ndc_device_count(int* count);
/* Device used by the one-shot entry points of the calling thread (default 0). */
ndc_status ndc_set_device(int device);

/* convolution.hpp:26-27.  Recorded for API parity; the device path's parallelism is
 * the CUDA grid, so the value does not change results or launch shapes. */
void ndc_set_max_threads(unsigned n);
unsigned ndc_max_threads(void);

/* convolution.hpp:30-38: out_ext[i] = x_ext[i] + k_ext[i] - 1 (= d + 2p). */
ndc_status ndc_conv_output_shape(int ndim, const size_t* x_ext, const size_t* k_ext,
                                 size_t* out_ext);

/* convolution.hpp:81-123 conv_full: y (shape x+2p) = x (*) h, zero padding. */
ndc_status ndc_conv_full_f64(int ndim, const size_t* x_ext, const double* x, const size_t* k_ext,
                             const double* h, double* y);

/* convolution.hpp:166-174 adjoint_apply: x_out (x_ext) = A^T y (y_ext == x_ext + 2p). */
/* Batched float32 operators (a leading batch index of independent images): y[b] = A x[b]
 * and x[b] = A^T y[b] -- for callers that keep float data (no f64 round trip). */
ndc_status ndc_conv_full_batch_f32(size_t batch, int ndim, const size_t* x_ext, const float* x,
                                   const size_t* k_ext, const double* h, float* y);
ndc_status ndc_adjoint_apply_batch_f32(size_t batch, int ndim, const size_t* y_ext, const float* y,
                                       const size_t* k_ext, const double* h, const size_t* x_ext,
                                       float* x_out);
ndc_status ndc_adjoint_apply_f64(int ndim, const size_t* y_ext, const double* y,
                                 const size_t* k_ext, const double* h, const size_t* x_ext,
                                 double* x_out);

/* convolution.hpp:178-185 normal_gradient: g = A^T A x - A^T y. */
ndc_status ndc_normal_gradient_f64(int ndim, const size_t* x_ext, const double* x, const double* y,
                                   const size_t* k_ext, const double* h, double* g);

/* solvers.hpp:119-122 objective: 0.5 ||A x - y||^2. */
ndc_status ndc_objective_f64(int ndim, const size_t* x_ext, const double* x, const double* y,
                             const size_t* k_ext, const double* h, double* f);

/* solvers.hpp:127-143 estimate_step: 1/lambda_max(A^T A) by power iteration. */
ndc_status ndc_estimate_step_f64(int ndim, const size_t* k_ext, const double* h,
                                 const size_t* x_ext, size_t power_iters, double* step);

/* solvers.hpp:147-149 kkt_residual: max |min(x_i, g_i)|. */
ndc_status ndc_kkt_residual_f64(int ndim, const size_t* x_ext, const double* x, const double* y,
                                const size_t* k_ext, const double* h, double* kkt);

/* solvers.hpp:155-238 deconv_pg.  obj_trace / kkt_trace need trace_cap >=
 * cfg->max_iters + 1 entries; report->trace_len entries are written.  cfg == NULL
 * means ndc_deconv_config_default(). */
ndc_status ndc_deconv_pg_f64(int ndim, const size_t* y_ext, const double* y, const size_t* k_ext,
                             const double* h, const size_t* x_ext, const ndc_deconv_config* cfg,
                             double* x_out, double* obj_trace, double* kkt_trace, size_t trace_cap,
                             ndc_deconv_report* report);

/* Batched deconv_pg: `batch` independent observations of one shape (y is
 * [batch][y_ext...]), every scalar of the reference -- step, objective, KKT,
 * backtracking, stop reason -- kept per image (BASELINE config 2).  Traces are
 * [batch][trace_cap]; reports[batch]. */
ndc_status ndc_deconv_pg_batch_f64(size_t batch, int ndim, const size_t* y_ext, const double* y,
                                   const size_t* k_ext, const double* h, const size_t* x_ext,
                                   const ndc_deconv_config* cfg, double* x_out, double* obj_trace,
                                   double* kkt_trace, size_t trace_cap, ndc_deconv_report* reports);
ndc_status ndc_deconv_pg_batch_f32(size_t batch, int ndim, const size_t* y_ext, const float* y,
                                   const size_t* k_ext, const double* h, const size_t* x_ext,
                                   const ndc_deconv_config* cfg, float* x_out, double* obj_trace,
                                   double* kkt_trace, size_t trace_cap, ndc_deconv_report* reports);

/* solvers.hpp:245-305 deconv_rl (Richardson-Lucy baseline on the same operators). */
ndc_status ndc_deconv_rl_f64(int ndim, const size_t* y_ext, const double* y, const size_t* k_ext,
                             const double* h, const size_t* x_ext, const ndc_rl_config* cfg,
                             double* x_out, double* obj_trace, double* kkt_trace, size_t trace_cap,
                             ndc_deconv_report* report);

/* ---- tensor files (imageio.hpp) ----
 * NDTENSOR: "NDTENSOR <ndim> <d_1> ... <d_n>\n" + little-endian f64 payload
 * (imageio.hpp:24-125).  info: header only (ndim <= 16; extents into ext[16]). */
ndc_status ndc_ndtensor_info(const char* path, int* ndim, size_t* ext16);
ndc_status ndc_ndtensor_read_f64(const char* path, double* out, size_t capacity);
ndc_status ndc_ndtensor_write_f64(const char* path, int ndim, const size_t* ext, const double* data);
/* PGM P5/P2 (imageio.hpp:126-265): samples as doubles, shape (height, width); writes
 * 8-bit P5 with round-half-even, clamping to [0,255] when clamp != 0. */
ndc_status ndc_pgm_info(const char* path, size_t* height, size_t* width);
ndc_status ndc_pgm_read_f64(const char* path, double* out, size_t capacity);
ndc_status ndc_pgm_write_f64(const char* path, size_t height, size_t width, const double* data,
                             int clamp);

/* ---- simulation generators (simulation.hpp:36-191) ----
 * Image-sized work runs on the device (phantoms bit-identical to the reference; the
 * mt19937_64 stream bit-identical, Box-Muller within a few ulp); kernels on the host.
 * Errors as the reference: size < 3x3 -> SHAPE, no lines -> CONFIG (ndconv::Error),
 * sigma <= 0 or std_dev < 0 -> NUMERIC, even kernel extent -> SHAPE. */
ndc_status ndc_sim_phantom_lines_f64(size_t rows, size_t cols, size_t n_lines, double intensity,
                                     double* out);                     /* simulation.hpp:36-70 */
ndc_status ndc_sim_phantom_texture_f64(size_t rows, size_t cols, double* out);  /* :72-94 */
ndc_status ndc_sim_gaussian_psf_f64(int ndim, const size_t* ext, double sigma, double* out);  /* :98-122 */
ndc_status ndc_sim_delta_psf_f64(int ndim, const size_t* ext, double* out);  /* :124-131 */
ndc_status ndc_sim_add_gaussian_noise_f64(size_t n, const double* in, double mean, double std_dev,
                                          uint64_t seed, double* out);  /* :154-191 */
/* Raw std::mt19937_64(seed) words [skip, skip+n), generated on the device. */
ndc_status ndc_sim_mt19937_64(uint64_t seed, size_t skip, size_t n, uint64_t* out);

/* ---- device-resident plan (same operators, buffers kept in HBM between calls) ----
 * A plan owns the device buffers for `batch` images of one (x_ext, k_ext) problem, a
 * CUDA stream, and -- for z-slab sharded runs -- an NCCL communicator.  All calls on
 * one plan are serialised on its stream and synchronous at the API edge. */
typedef struct ndc_plan ndc_plan;

ndc_status ndc_plan_create(ndc_plan** plan, int device, size_t batch, int ndim,
                           const size_t* x_ext, const size_t* k_ext, const double* h);
ndc_status ndc_plan_destroy(ndc_plan* plan);
/* y: [batch][y_ext...] dense host array. */
ndc_status ndc_plan_set_observation_f64(ndc_plan* plan, const double* y);
ndc_status ndc_plan_set_observation_f32(ndc_plan* plan, const float* y);
/* PG split into begin (validation, step, x0 = max(A^T y, 0), objective), iterate
 * (up to n more iterations per image) and end (final KKT).  ndc_plan_pg_run does
 * all three. */
ndc_status ndc_plan_pg_begin(ndc_plan* plan, const ndc_deconv_config* cfg);
ndc_status ndc_plan_pg_iterate(ndc_plan* plan, size_t n, size_t* images_active);
ndc_status ndc_plan_pg_end(ndc_plan* plan);
ndc_status ndc_plan_pg_run(ndc_plan* plan, const ndc_deconv_config* cfg);
/* Richardson-Lucy (deconv_rl, solvers.hpp:245-305) on the resident observation, which it
 * leaves unchanged (the clamped copy lives in plan scratch for the run); per-image
 * results through ndc_plan_get_report / ndc_plan_get_estimate_*. */
ndc_status ndc_plan_rl_run(ndc_plan* plan, const ndc_rl_config* cfg);
/* Per-image results after pg_end; traces need trace_cap entries per image. */
ndc_status ndc_plan_get_report(ndc_plan* plan, size_t image, ndc_deconv_report* report,
                               double* obj_trace, double* kkt_trace, size_t trace_cap);
ndc_status ndc_plan_get_estimate_f64(ndc_plan* plan, double* x_out);
ndc_status ndc_plan_get_estimate_f32(ndc_plan* plan, float* x_out);
/* The resident observation (float32 on the device), owned planes when sharded. */
ndc_status ndc_plan_get_observation_f64(ndc_plan* plan, double* y_out);
/* Stream an NDTENSOR observation file straight into the plan (pinned 16 MB chunks, no
 * full host copy; a batch plan reads [batch, y_ext...] or, for batch 1, [y_ext...];
 * a sharded plan reads only its own planes), and stream the estimate back out
 * (sharded ranks each write their planes into one file; rank 0 writes the header). */
ndc_status ndc_plan_load_observation_ndtensor(ndc_plan* plan, const char* path);
ndc_status ndc_plan_save_estimate_ndtensor(ndc_plan* plan, const char* path);
/* add_gaussian_noise (simulation.hpp:184-191) to the resident observation in place: the
 * mt19937_64 stream of `seed` runs over the dense [batch, y...] storage order, generated
 * on the device; a sharded rank applies its own planes' samples. */
ndc_status ndc_plan_add_gaussian_noise(ndc_plan* plan, double mean, double std_dev, uint64_t seed);
/* One forward (A x) / adjoint (A^T y) pass on resident buffers, for kernel timing. */
ndc_status ndc_plan_forward(ndc_plan* plan);
ndc_status ndc_plan_adjoint(ndc_plan* plan);

/* Launch bookkeeping for the bench: kind 0 = forward correlation, 1 = adjoint
 * correlation, 2 = all kernels.  With timing enabled, forward/adjoint launches are
 * bracketed by CUDA events on the plan's stream. */
ndc_status ndc_plan_set_timing(ndc_plan* plan, int enabled);
ndc_status ndc_plan_reset_stats(ndc_plan* plan);
ndc_status ndc_plan_stats(ndc_plan* plan, int kind, uint64_t* launches, double* total_ms);
ndc_status ndc_plan_stream(ndc_plan* plan, void** cuda_stream);
/* Measured FP32 FMA throughput of `device` in TFLOP/s (best of 4 runs of a register-only
 * packed-FMA kernel on every SM): the roofline denominator the bench reports against. */
ndc_status ndc_probe_fp32_peak(int device, double* tflops);
/* Guard-band debugging (environment NDC_GUARD_BANDS=1 when the process starts): every plan
 * allocation carries 1 MB fill-pattern guards on both sides, checked here (bad_bytes =
 * changed guard bytes of this plan's live allocations) and when a plan is destroyed
 * (accumulated process-wide into *total_bad by ndc_debug_guard_violations). */
ndc_status ndc_plan_check_guards(ndc_plan* plan, size_t* bad_bytes);
ndc_status ndc_debug_guard_violations(unsigned long long* total_bad);
/* The checker's own test: writes 16 bytes into the guard after the plan's observation
 * buffer (guard-band mode only; NDC_ERR_ARGUMENT otherwise). */
ndc_status ndc_plan_debug_corrupt_guard(ndc_plan* plan);

/* ---- z-slab sharding across processes (one GPU per rank, NCCL over NVLink) ----
 * Rank r of `world` owns x planes [a_r, b_r) of the slowest axis (ndc_slab_range)
 * plus the matching y planes; every pass exchanges p_z-plane halos with its
 * neighbours and combines per-rank f64 partials in rank order. */
ndc_status ndc_slab_range(size_t mz, size_t pz, int rank, int world, size_t* x_begin,
                          size_t* x_end, size_t* y_begin, size_t* y_end);
ndc_status ndc_nccl_unique_id(unsigned char id[128]);
ndc_status ndc_plan_create_sharded(ndc_plan** plan, int device, int ndim, const size_t* x_ext,
                                   const size_t* k_ext, const double* h, int rank, int world,
                                   const unsigned char nccl_id[128]);
/* Sharded plans take and return only the rank's own planes (y planes
 * [y_begin, y_end), x planes [x_begin, x_end)). */

/* In-process slab group: `world` ranks of one process, each driven by its own host
 * thread (any device each), halos moved by device-to-device copies.  Same
 * partitioning and combine order as the NCCL path; used for testing the sharded
 * driver on fewer GPUs than ranks. */
typedef struct ndc_local_group ndc_local_group;
ndc_status ndc_local_group_create(ndc_local_group** group, int world);
ndc_status ndc_local_group_destroy(ndc_local_group* group);
ndc_status ndc_plan_create_local(ndc_plan** plan, ndc_local_group* group, int rank, int device,
                                 int ndim, const size_t* x_ext, const size_t* k_ext,
                                 const double* h);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif

#endif /* NDCONV_B200_H */
