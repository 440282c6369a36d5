// TEST INFRASTRUCTURE ONLY -- C-ABI shim around the UNMODIFIED reference headers.
//
// Compiled by oracle/Makefile straight from /root/reference/proj/include (never
// copied into this repo) into oracle/_ref/libndconv_ref.so, with the reference's
// own Release flags (-O3 -DNDEBUG, proj/CMakeLists.txt:8-10).  Used to pin the C
// restatement (oracle/ndconv_oracle.c), to generate tests/golden/ fixtures, and as
// the CPU baseline (bench.py cpu_baseline / --impl reference).
//
// Every entry point has the same signature as its oc_* twin in ndconv_oracle.c so
// the Python loader (oracle/oracle.py) can swap them.  Symbols other than the
// ref_* entry points are hidden, so the reference's inline ndconv:: functions can
// never interpose on (or be interposed by) anything else in the process.
#include <cstddef>
#include <cstring>
#include <cstdint>
#include <exception>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "ndconv/ndconv.hpp"

#define REF_API extern "C" __attribute__((visibility("default")))

namespace {

enum { RC_OK = 0, RC_ERROR = 1, RC_SHAPE = 2, RC_NUMERIC = 3, RC_BOUNDS = 4, RC_FORMAT = 5, RC_OTHER = 9 };

struct PgCfg {  // layout shared with oc_pg_config / ndc_deconv_config
  std::size_t max_iters;
  double tol_rel_objective;
  int has_initial_step;
  double initial_step;
  double backtrack_factor;
  std::size_t max_backtracks;
  std::size_t power_iters;
};

struct RlCfg {
  std::size_t max_iters;
  double tol_rel_change;
};

ndconv::Shape shape_of(int ndim, const std::size_t* ext) {
  return ndconv::Shape(std::vector<std::size_t>(ext, ext + ndim));
}

ndconv::Tensor tensor_of(int ndim, const std::size_t* ext, const double* v) {
  ndconv::Shape s = shape_of(ndim, ext);
  return ndconv::Tensor(s, std::vector<double>(v, v + s.element_count()));
}

ndconv::Kernel kernel_of(int ndim, const std::size_t* ext, const double* v) {
  return ndconv::Kernel(tensor_of(ndim, ext, v));
}

template <class F>
int guard(F&& f) {
  try {
    f();
    return RC_OK;
  } catch (const ndconv::ShapeError&) {
    return RC_SHAPE;
  } catch (const ndconv::NumericError&) {
    return RC_NUMERIC;
  } catch (const ndconv::BoundsError&) {
    return RC_BOUNDS;
  } catch (const ndconv::FormatError&) {
    return RC_FORMAT;
  } catch (const ndconv::Error&) {
    return RC_ERROR;
  } catch (...) {
    return RC_OTHER;
  }
}

void put(const ndconv::Tensor& t, double* out) {
  std::memcpy(out, t.data().data(), t.size() * sizeof(double));
}

int stop_code(ndconv::StopReason r) {
  switch (r) {
    case ndconv::StopReason::converged: return 0;
    case ndconv::StopReason::max_iters: return 1;
    case ndconv::StopReason::stalled: return 2;
  }
  return -1;
}

}  // namespace

REF_API void ref_set_threads(int n) { ndconv::set_max_threads(n < 1 ? 1u : unsigned(n)); }

REF_API int ref_conv_output_shape(int ndim, const std::size_t* xext, const std::size_t* hext,
                                  std::size_t* yext) {
  return guard([&] {
    std::vector<double> hv(shape_of(ndim, hext).element_count(), 0.0);
    const auto s = ndconv::conv_output_shape(shape_of(ndim, xext), kernel_of(ndim, hext, hv.data()));
    for (int i = 0; i < ndim; ++i) yext[i] = s.extent(i);
  });
}

REF_API int ref_conv_full(int ndim, const std::size_t* xext, const double* x,
                          const std::size_t* hext, const double* h, double* y) {
  return guard([&] { put(ndconv::conv_full(tensor_of(ndim, xext, x), kernel_of(ndim, hext, h)), y); });
}

REF_API int ref_adjoint_apply(int ndim, const std::size_t* yext, const double* y,
                              const std::size_t* hext, const double* h, const std::size_t* xext,
                              double* out) {
  return guard([&] {
    put(ndconv::adjoint_apply(tensor_of(ndim, yext, y), kernel_of(ndim, hext, h),
                              shape_of(ndim, xext)),
        out);
  });
}

REF_API int ref_objective(int ndim, const std::size_t* xext, const double* x, const double* y,
                          const std::size_t* hext, const double* h, double* f) {
  return guard([&] {
    const auto k = kernel_of(ndim, hext, h);
    const auto ys = ndconv::conv_output_shape(shape_of(ndim, xext), k);
    *f = ndconv::objective(tensor_of(ndim, xext, x),
                           ndconv::Tensor(ys, std::vector<double>(y, y + ys.element_count())), k);
  });
}

REF_API int ref_normal_gradient(int ndim, const std::size_t* xext, const double* x,
                                const double* y, const std::size_t* hext, const double* h,
                                double* g) {
  return guard([&] {
    const auto k = kernel_of(ndim, hext, h);
    const auto ys = ndconv::conv_output_shape(shape_of(ndim, xext), k);
    put(ndconv::normal_gradient(tensor_of(ndim, xext, x),
                                ndconv::Tensor(ys, std::vector<double>(y, y + ys.element_count())),
                                k),
        g);
  });
}

REF_API int ref_estimate_step(int ndim, const std::size_t* hext, const double* h,
                              const std::size_t* xext, std::size_t iters, double* step) {
  return guard([&] { *step = ndconv::estimate_step(kernel_of(ndim, hext, h), shape_of(ndim, xext), iters); });
}

REF_API int ref_kkt_residual(int ndim, const std::size_t* xext, const double* x, const double* y,
                             const std::size_t* hext, const double* h, double* kkt) {
  return guard([&] {
    const auto k = kernel_of(ndim, hext, h);
    const auto ys = ndconv::conv_output_shape(shape_of(ndim, xext), k);
    *kkt = ndconv::kkt_residual(tensor_of(ndim, xext, x),
                                ndconv::Tensor(ys, std::vector<double>(y, y + ys.element_count())), k);
  });
}

REF_API int ref_deconv_pg(int ndim, const std::size_t* yext, const double* y,
                          const std::size_t* hext, const double* h, const std::size_t* xext,
                          const PgCfg* c, double* x_out, double* obj_trace, double* kkt_trace,
                          std::size_t* trace_len, std::size_t* iters_run, int* stop_reason,
                          std::size_t* backtracks) {
  return guard([&] {
    ndconv::DeconvConfig cfg;
    cfg.max_iters = c->max_iters;
    cfg.tol_rel_objective = c->tol_rel_objective;
    if (c->has_initial_step) cfg.initial_step = c->initial_step;
    cfg.backtrack_factor = c->backtrack_factor;
    cfg.max_backtracks = c->max_backtracks;
    cfg.power_iters = c->power_iters;
    const auto rep = ndconv::deconv_pg(tensor_of(ndim, yext, y), kernel_of(ndim, hext, h),
                                       shape_of(ndim, xext), cfg);
    put(rep.estimate, x_out);
    std::memcpy(obj_trace, rep.objective_trace.data(), rep.objective_trace.size() * sizeof(double));
    std::memcpy(kkt_trace, rep.kkt_trace.data(), rep.kkt_trace.size() * sizeof(double));
    *trace_len = rep.objective_trace.size();
    *iters_run = rep.iterations_run;
    *stop_reason = stop_code(rep.stop_reason);
    if (backtracks) *backtracks = static_cast<std::size_t>(-1);  // not observable from the API
  });
}

REF_API int ref_deconv_rl(int ndim, const std::size_t* yext, const double* y,
                          const std::size_t* hext, const double* h, const std::size_t* xext,
                          const RlCfg* c, double* x_out, double* obj_trace, double* kkt_trace,
                          std::size_t* trace_len, std::size_t* iters_run, int* stop_reason,
                          std::size_t* clamped) {
  return guard([&] {
    ndconv::RlConfig cfg;
    cfg.max_iters = c->max_iters;
    cfg.tol_rel_change = c->tol_rel_change;
    const auto rep = ndconv::deconv_rl(tensor_of(ndim, yext, y), kernel_of(ndim, hext, h),
                                       shape_of(ndim, xext), cfg);
    put(rep.estimate, x_out);
    std::memcpy(obj_trace, rep.objective_trace.data(), rep.objective_trace.size() * sizeof(double));
    std::memcpy(kkt_trace, rep.kkt_trace.data(), rep.kkt_trace.size() * sizeof(double));
    *trace_len = rep.objective_trace.size();
    *iters_run = rep.iterations_run;
    *stop_reason = stop_code(rep.stop_reason);
    *clamped = rep.negative_pixels_clamped;
  });
}

// Sampled forward values through the reference's own per-voxel routine
// (detail::conv_element, convolution.hpp:55-74): bitwise equal to conv_full.
REF_API int ref_conv_full_sample(int ndim, const std::size_t* xext, const double* x,
                                 const std::size_t* hext, const double* h, std::size_t n,
                                 const std::size_t* flat_idx, double* values) {
  return guard([&] {
    const auto k = kernel_of(ndim, hext, h);
    const auto xs = shape_of(ndim, xext);
    const auto ys = ndconv::conv_output_shape(xs, k);
    const auto xst = ndconv::strides_of(xs);
    const auto hst = ndconv::strides_of(k.tensor().shape());
    const ndconv::detail::ConvView view{x, k.tensor().data().data(), xs.extents().data(),
                                        k.tensor().shape().extents().data(), xst.data(),
                                        hst.data(), xs.ndim()};
    for (std::size_t s = 0; s < n; ++s) {
      const auto idx = ndconv::unflatten(ys, flat_idx[s]);
      values[s] = ndconv::detail::conv_element(view, idx.data(), 0, 0, 0);
    }
  });
}

// Sampled adjoint values: conv_element over (y, flip h) at output index k + 2p,
// i.e. the entry adjoint_apply's crop_m keeps (convolution.hpp:151-174).
REF_API int ref_adjoint_sample(int ndim, const std::size_t* yext, const double* y,
                               const std::size_t* hext, const double* h, const std::size_t* xext,
                               std::size_t n, const std::size_t* flat_idx, double* values) {
  return guard([&] {
    const auto kf = ndconv::flip(kernel_of(ndim, hext, h));
    const auto ysh = shape_of(ndim, yext);
    const auto xs = shape_of(ndim, xext);
    const auto yst = ndconv::strides_of(ysh);
    const auto hst = ndconv::strides_of(kf.tensor().shape());
    const ndconv::detail::ConvView view{y, kf.tensor().data().data(), ysh.extents().data(),
                                        kf.tensor().shape().extents().data(), yst.data(),
                                        hst.data(), ysh.ndim()};
    for (std::size_t s = 0; s < n; ++s) {
      auto idx = ndconv::unflatten(xs, flat_idx[s]);
      for (int i = 0; i < ndim; ++i) idx[i] += 2 * kf.radius(i);
      values[s] = ndconv::detail::conv_element(view, idx.data(), 0, 0, 0);
    }
  });
}

// CPU-baseline replay of deconv_pg's loop body (solvers.hpp:179-228) using only
// the reference's own operators, so one accepted iteration can be timed without
// the per-call setup (power iteration, A^T y, x0, final KKT).  `state` holds
// x (in/out) and ax (in/out); aty and f are passed in.  Returns the number of
// accepted iterations actually run.
REF_API int ref_pg_iterations(int ndim, const std::size_t* yext, const double* y,
                              const std::size_t* hext, const double* h, const std::size_t* xext,
                              double step0, double backtrack_factor, std::size_t max_backtracks,
                              std::size_t iters, double* x_io, double* ax_io, const double* aty_in,
                              double* f_io, std::size_t* accepted_out) {
  return guard([&] {
    using namespace ndconv;
    const Kernel k = kernel_of(ndim, hext, h);
    const Shape xs = shape_of(ndim, xext);
    const Tensor yt = tensor_of(ndim, yext, y);
    const Tensor aty = tensor_of(ndim, xext, aty_in);
    Tensor x = tensor_of(ndim, xext, x_io);
    Tensor ax = tensor_of(ndim, yext, ax_io);
    double f = *f_io;
    std::size_t accepted_total = 0;
    for (std::size_t it = 0; it < iters; ++it) {
      const Tensor g = sub(adjoint_apply(ax, k, xs), aty);
      (void)detail::kkt_from_gradient(x, g);
      double step = step0;
      bool accepted = false;
      for (std::size_t b = 0; b <= max_backtracks; ++b) {
        Tensor trial = clamp_nonneg(sub(x, scale(g, step)));
        if (trial == x) break;
        Tensor ax_trial = conv_full(trial, k);
        Tensor r = sub(ax_trial, yt);
        const double f_trial = 0.5 * dot(r, r);
        if (f_trial < f) {
          x = std::move(trial);
          ax = std::move(ax_trial);
          f = f_trial;
          accepted = true;
          break;
        }
        step *= backtrack_factor;
      }
      if (!accepted) break;
      ++accepted_total;
    }
    put(x, x_io);
    put(ax, ax_io);
    *f_io = f;
    *accepted_out = accepted_total;
  });
}

// ---- tensor file formats (imageio.hpp), over in-memory byte strings ---------------------
// Parsing and serialising through the reference's own istream/ostream entry points pins
// the B200 library's NDTENSOR / PGM readers and writers byte for byte (tests/test_io.py).
namespace {
int emit(const std::string& s, char* out, std::size_t cap, std::size_t* n) {
  *n = s.size();
  if (out && cap >= s.size()) std::memcpy(out, s.data(), s.size());
  return RC_OK;
}

void take(const ndconv::Tensor& t, int* ndim, std::size_t* ext, double* out, std::size_t cap) {
  *ndim = static_cast<int>(t.shape().ndim());
  for (std::size_t i = 0; i < t.shape().ndim() && i < 16; ++i) ext[i] = t.shape().extent(i);
  if (out && cap >= t.size()) put(t, out);
}
}  // namespace

REF_API int ref_io_parse_tensor(const char* bytes, std::size_t nbytes, int* ndim, std::size_t* ext,
                                double* out, std::size_t cap) {
  return guard([&] {
    std::istringstream in(std::string(bytes, nbytes), std::ios::binary);
    take(ndconv::io::read_tensor(in), ndim, ext, out, cap);
  });
}

REF_API int ref_io_serialize_tensor(int ndim, const std::size_t* ext, const double* v, char* out,
                                    std::size_t cap, std::size_t* n) {
  return guard([&] {
    std::ostringstream os(std::ios::binary);
    ndconv::io::write_tensor(tensor_of(ndim, ext, v), os);
    emit(os.str(), out, cap, n);
  });
}

REF_API int ref_io_parse_pgm(const char* bytes, std::size_t nbytes, int* ndim, std::size_t* ext,
                             double* out, std::size_t cap) {
  return guard([&] {
    std::istringstream in(std::string(bytes, nbytes), std::ios::binary);
    take(ndconv::io::read_pgm(in), ndim, ext, out, cap);
  });
}

REF_API int ref_io_serialize_pgm(int ndim, const std::size_t* ext, const double* v, int clamp,
                                 char* out, std::size_t cap, std::size_t* n) {
  return guard([&] {
    std::ostringstream os(std::ios::binary);
    ndconv::io::write_pgm(tensor_of(ndim, ext, v), os, clamp != 0);
    emit(os.str(), out, cap, n);
  });
}

REF_API int ref_snr_db(int ndim, const std::size_t* ext, const double* a, const double* b, double* out) {
  return guard([&] { *out = ndconv::sim::snr_db(tensor_of(ndim, ext, a), tensor_of(ndim, ext, b)); });
}

// ---- simulation generators (simulation.hpp) ---------------------------------------------
REF_API int ref_sim_phantom_lines(std::size_t rows, std::size_t cols, std::size_t n, double intensity,
                                  double* out) {
  return guard([&] { put(ndconv::sim::phantom_lines(rows, cols, n, intensity), out); });
}

REF_API int ref_sim_phantom_texture(std::size_t rows, std::size_t cols, double* out) {
  return guard([&] { put(ndconv::sim::phantom_texture(rows, cols), out); });
}

REF_API int ref_sim_gaussian_psf(int ndim, const std::size_t* ext, double sigma, double* out) {
  return guard([&] {
    put(ndconv::sim::gaussian_psf(std::vector<std::size_t>(ext, ext + ndim), sigma).tensor(), out);
  });
}

REF_API int ref_sim_delta_psf(int ndim, const std::size_t* ext, double* out) {
  return guard([&] { put(ndconv::sim::delta_psf(std::vector<std::size_t>(ext, ext + ndim)).tensor(), out); });
}

REF_API int ref_sim_add_gaussian_noise(std::size_t n, const double* in, double mean, double std_dev,
                                       std::uint64_t seed, double* out) {
  return guard([&] {
    const std::size_t ext[1] = {n};
    put(ndconv::sim::add_gaussian_noise(tensor_of(1, ext, in), {mean, std_dev, seed}), out);
  });
}

// The raw engine the reference's GaussianSource wraps (simulation.hpp:175).
REF_API int ref_mt19937_64(std::uint64_t seed, std::size_t skip, std::size_t n, std::uint64_t* out) {
  return guard([&] {
    std::mt19937_64 rng(seed);
    rng.discard(skip);
    for (std::size_t i = 0; i < n; ++i) out[i] = rng();
  });
}
