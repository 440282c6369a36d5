// ndconv_b200/ndconv.hpp -- C++ drop-in for the reference's header-only ndconv API
// (/root/reference/proj/include/ndconv/*.hpp) on top of the B200 C-ABI
// (include/ndconv_b200.h, libndconv_b200.so).
//
// Swap `#include "ndconv/ndconv.hpp"` for `#include "ndconv_b200/ndconv.hpp"`, link
// libndconv_b200.so, and the same `ndconv::` code runs its convolutions and the
// projected-gradient solver on the GPU:
//   conv_full / adjoint_apply / normal_gradient / objective / estimate_step /
//   kkt_residual / deconv_pg / deconv_rl   -> device (float32, f64 reductions)
//   Shape / Tensor / Kernel / flip / crop_center / crop_m / elementwise helpers
//                                           -> host value types, as in the reference
// Errors surface as the reference's exception classes (error.hpp:8-30); a CUDA or
// NCCL failure, or no usable B200, throws DeviceError (derived from Error).  Include
// either this header or the reference's, never both (same namespace).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <initializer_list>
#include <limits>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "ndconv_b200.h"

namespace ndconv {

// ---- errors (error.hpp:8-30) ------------------------------------------------------------
struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ShapeError : Error {
  using Error::Error;
};
struct BoundsError : Error {
  using Error::Error;
};
struct FormatError : Error {
  using Error::Error;
};
struct NumericError : Error {
  using Error::Error;
};
// Device-side failure (CUDA / NCCL / no sm_100 GPU / unsupported operand).
struct DeviceError : Error {
  using Error::Error;
};

namespace b200 {
inline void check(ndc_status s) {
  if (s == NDC_OK) return;
  const std::string msg = ndc_last_error();
  switch (s) {
    case NDC_ERR_CONFIG: throw Error(msg);
    case NDC_ERR_SHAPE: throw ShapeError(msg);
    case NDC_ERR_NUMERIC: throw NumericError(msg);
    case NDC_ERR_BOUNDS: throw BoundsError(msg);
    case NDC_ERR_FORMAT: throw FormatError(msg);
    case NDC_ERR_ARGUMENT: throw std::invalid_argument(msg);
    default: throw DeviceError(msg);
  }
}
}  // namespace b200

// ---- Shape (shape.hpp:17-98) -----------------------------------------------------------
class Shape {
 public:
  explicit Shape(std::vector<std::size_t> extents) : ext_(std::move(extents)) {
    if (ext_.empty()) throw ShapeError("Shape: need at least one dimension");
    std::size_t n = 1;
    for (std::size_t e : ext_) {
      if (e == 0) throw ShapeError("Shape: extents must be positive");
      if (e > std::numeric_limits<std::size_t>::max() / n)
        throw ShapeError("Shape: element count overflows");
      n *= e;
    }
    count_ = n;
  }
  Shape(std::initializer_list<std::size_t> e) : Shape(std::vector<std::size_t>(e)) {}
  std::size_t ndim() const { return ext_.size(); }
  std::size_t extent(std::size_t d) const { return ext_[d]; }
  const std::vector<std::size_t>& extents() const { return ext_; }
  std::size_t element_count() const { return count_; }
  bool operator==(const Shape& o) const { return ext_ == o.ext_; }
  std::string to_string() const {
    std::string s;
    for (std::size_t i = 0; i < ext_.size(); ++i) s += (i ? "x" : "") + std::to_string(ext_[i]);
    return s;
  }

 private:
  std::vector<std::size_t> ext_;
  std::size_t count_ = 0;
};

inline std::vector<std::size_t> strides_of(const Shape& s) {
  std::vector<std::size_t> st(s.ndim());
  std::size_t acc = 1;
  for (std::size_t i = s.ndim(); i-- > 0;) {
    st[i] = acc;
    acc *= s.extent(i);
  }
  return st;
}

inline std::size_t flat_index(const Shape& s, std::span<const std::size_t> idx) {
  if (idx.size() != s.ndim()) throw BoundsError("flat_index: index rank does not match shape");
  std::size_t f = 0;
  for (std::size_t i = 0; i < s.ndim(); ++i) {
    if (idx[i] >= s.extent(i)) throw BoundsError("flat_index: index out of range");
    f = f * s.extent(i) + idx[i];
  }
  return f;
}

inline std::vector<std::size_t> unflatten(const Shape& s, std::size_t flat) {
  std::vector<std::size_t> idx(s.ndim());
  for (std::size_t i = s.ndim(); i-- > 0;) {
    idx[i] = flat % s.extent(i);
    flat /= s.extent(i);
  }
  return idx;
}

inline bool next_index(const Shape& s, std::span<std::size_t> idx) {
  for (std::size_t i = s.ndim(); i-- > 0;) {
    if (++idx[i] < s.extent(i)) return true;
    idx[i] = 0;
  }
  return false;
}

// ---- Tensor (tensor.hpp:22-144) -------------------------------------------------------
inline constexpr double kDivEpsilon = 1e-12;

class Tensor {
 public:
  Tensor(Shape shape, std::vector<double> data) : shape_(std::move(shape)), data_(std::move(data)) {
    if (data_.size() != shape_.element_count())
      throw ShapeError("Tensor: got " + std::to_string(data_.size()) + " values for shape " +
                       shape_.to_string());
  }
  static Tensor zeros(const Shape& s) { return Tensor(s, std::vector<double>(s.element_count(), 0.0)); }
  static Tensor filled(const Shape& s, double v) {
    return Tensor(s, std::vector<double>(s.element_count(), v));
  }
  const Shape& shape() const { return shape_; }
  std::size_t size() const { return data_.size(); }
  const std::vector<double>& data() const { return data_; }
  double operator[](std::size_t f) const { return data_[f]; }
  double& operator[](std::size_t f) { return data_[f]; }
  double at(std::span<const std::size_t> idx) const { return data_[flat_index(shape_, idx)]; }
  double& at(std::span<const std::size_t> idx) { return data_[flat_index(shape_, idx)]; }
  double at(std::initializer_list<std::size_t> idx) const {
    return at(std::span<const std::size_t>(idx.begin(), idx.size()));
  }
  double& at(std::initializer_list<std::size_t> idx) {
    return at(std::span<const std::size_t>(idx.begin(), idx.size()));
  }
  bool operator==(const Tensor& o) const { return shape_ == o.shape_ && data_ == o.data_; }

 private:
  Shape shape_;
  std::vector<double> data_;
};

inline const std::vector<double>& vectorize(const Tensor& t) { return t.data(); }
inline Tensor devectorize(const Shape& s, std::vector<double> d) { return Tensor(s, std::move(d)); }
inline bool all_finite(const Tensor& t) {
  return std::all_of(t.data().begin(), t.data().end(), [](double v) { return std::isfinite(v); });
}

namespace detail {
inline void check_same_shape(const Tensor& a, const Tensor& b, const char* what) {
  if (!(a.shape() == b.shape()))
    throw ShapeError(std::string(what) + ": shape " + a.shape().to_string() + " vs " +
                     b.shape().to_string());
}
template <class F>
Tensor zip(const Tensor& a, const Tensor& b, const char* what, F f) {
  check_same_shape(a, b, what);
  std::vector<double> out(a.size());
  for (std::size_t i = 0; i < a.size(); ++i) out[i] = f(a[i], b[i]);
  return Tensor(a.shape(), std::move(out));
}
}  // namespace detail

inline Tensor add(const Tensor& a, const Tensor& b) {
  return detail::zip(a, b, "add", [](double x, double y) { return x + y; });
}
inline Tensor sub(const Tensor& a, const Tensor& b) {
  return detail::zip(a, b, "sub", [](double x, double y) { return x - y; });
}
inline Tensor mul(const Tensor& a, const Tensor& b) {
  return detail::zip(a, b, "mul", [](double x, double y) { return x * y; });
}
inline Tensor guarded_div(const Tensor& a, const Tensor& b) {
  return detail::zip(a, b, "guarded_div",
                     [](double x, double y) { return std::abs(y) < kDivEpsilon ? 0.0 : x / y; });
}
inline Tensor scale(const Tensor& t, double f) {
  std::vector<double> out(t.size());
  for (std::size_t i = 0; i < t.size(); ++i) out[i] = t[i] * f;
  return Tensor(t.shape(), std::move(out));
}
inline Tensor clamp_nonneg(const Tensor& t) {
  std::vector<double> out(t.size());
  for (std::size_t i = 0; i < t.size(); ++i) out[i] = t[i] < 0.0 ? 0.0 : t[i];
  return Tensor(t.shape(), std::move(out));
}
inline double sum(const Tensor& t) {
  double s = 0.0;
  for (double v : t.data()) s += v;
  return s;
}
inline double dot(const Tensor& a, const Tensor& b) {
  detail::check_same_shape(a, b, "dot");
  double s = 0.0;
  for (std::size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
  return s;
}
inline double norm2(const Tensor& t) { return std::sqrt(dot(t, t)); }

// ---- Kernel (kernel.hpp:15-45) ---------------------------------------------------------
class Kernel {
 public:
  explicit Kernel(Tensor t) : t_(std::move(t)) {
    for (std::size_t e : t_.shape().extents()) {
      if (e % 2 == 0) throw ShapeError("Kernel: extents must be odd, got " + t_.shape().to_string());
      r_.push_back((e - 1) / 2);
    }
    if (!all_finite(t_)) throw NumericError("Kernel: values must be finite");
  }
  const Tensor& tensor() const { return t_; }
  const Shape& shape() const { return t_.shape(); }
  std::size_t ndim() const { return t_.shape().ndim(); }
  const std::vector<std::size_t>& radii() const { return r_; }
  std::size_t radius(std::size_t d) const { return r_[d]; }

 private:
  Tensor t_;
  std::vector<std::size_t> r_;
};

inline Kernel flip(const Kernel& h) {
  std::vector<double> d = h.tensor().data();
  std::reverse(d.begin(), d.end());
  return Kernel(Tensor(h.shape(), std::move(d)));
}

// ---- operators (convolution.hpp) --------------------------------------------------------
inline void set_max_threads(unsigned n) { ndc_set_max_threads(n); }
inline unsigned max_threads() { return ndc_max_threads(); }

inline Shape conv_output_shape(const Shape& x, const Kernel& h) {
  if (x.ndim() != h.ndim())
    throw ShapeError("conv_full: " + std::to_string(x.ndim()) + "-d input vs " +
                     std::to_string(h.ndim()) + "-d kernel");
  std::vector<std::size_t> out(x.ndim());
  b200::check(ndc_conv_output_shape(static_cast<int>(x.ndim()), x.extents().data(),
                                    h.shape().extents().data(), out.data()));
  return Shape(std::move(out));
}

inline Tensor conv_full(const Tensor& x, const Kernel& h) {
  const Shape out = conv_output_shape(x.shape(), h);
  std::vector<double> y(out.element_count());
  b200::check(ndc_conv_full_f64(static_cast<int>(x.shape().ndim()), x.shape().extents().data(),
                                x.data().data(), h.shape().extents().data(),
                                h.tensor().data().data(), y.data()));
  return Tensor(out, std::move(y));
}

inline Tensor crop_center(const Tensor& t, const Shape& target) {
  if (t.shape().ndim() != target.ndim()) throw ShapeError("crop_center: dimension count mismatch");
  std::vector<std::size_t> off(target.ndim());
  for (std::size_t i = 0; i < target.ndim(); ++i) {
    const std::size_t te = t.shape().extent(i), ge = target.extent(i);
    if (te < ge || (te - ge) % 2 != 0)
      throw ShapeError("crop_center: cannot center " + target.to_string() + " inside " +
                       t.shape().to_string());
    off[i] = (te - ge) / 2;
  }
  const std::vector<std::size_t> st = strides_of(t.shape());
  Tensor out = Tensor::zeros(target);
  std::vector<std::size_t> idx(target.ndim(), 0);
  for (std::size_t f = 0; f < target.element_count(); ++f) {
    std::size_t src = 0;
    for (std::size_t i = 0; i < idx.size(); ++i) src += (idx[i] + off[i]) * st[i];
    out[f] = t[src];
    next_index(target, idx);
  }
  return out;
}

inline Tensor crop_m(const Tensor& t, std::span<const std::size_t> radii, const Shape& target) {
  if (t.shape().ndim() != target.ndim() || radii.size() != target.ndim())
    throw ShapeError("crop_m: dimension count mismatch");
  for (std::size_t i = 0; i < target.ndim(); ++i)
    if (t.shape().extent(i) != target.extent(i) + 4 * radii[i])
      throw ShapeError("crop_m: extent is not target + 4p");
  return crop_center(t, target);
}

inline Tensor adjoint_apply(const Tensor& y, const Kernel& h, const Shape& x_shape) {
  if (y.shape().ndim() != h.ndim() || x_shape.ndim() != h.ndim())
    throw ShapeError("adjoint_apply: dimension count mismatch");
  for (std::size_t i = 0; i < x_shape.ndim(); ++i)
    if (y.shape().extent(i) != x_shape.extent(i) + 2 * h.radius(i))
      throw ShapeError("adjoint_apply: observation shape " + y.shape().to_string() + " is not " +
                       x_shape.to_string() + " + 2p");
  std::vector<double> x(x_shape.element_count());
  b200::check(ndc_adjoint_apply_f64(static_cast<int>(y.shape().ndim()), y.shape().extents().data(),
                                    y.data().data(), h.shape().extents().data(),
                                    h.tensor().data().data(), x_shape.extents().data(), x.data()));
  return Tensor(x_shape, std::move(x));
}

namespace detail {
inline void check_forward_shapes(const Tensor& y, const Kernel& h, const Shape& x_shape,
                                 const char* what) {
  const Shape expected = conv_output_shape(x_shape, h);
  if (!(y.shape() == expected))
    throw ShapeError(std::string(what) + ": observation shape " + y.shape().to_string() +
                     " does not match forward model output " + expected.to_string());
}
}  // namespace detail

inline Tensor normal_gradient(const Tensor& x, const Tensor& y, const Kernel& h) {
  detail::check_forward_shapes(y, h, x.shape(), "normal_gradient");
  std::vector<double> g(x.size());
  b200::check(ndc_normal_gradient_f64(static_cast<int>(x.shape().ndim()), x.shape().extents().data(),
                                      x.data().data(), y.data().data(), h.shape().extents().data(),
                                      h.tensor().data().data(), g.data()));
  return Tensor(x.shape(), std::move(g));
}

// ---- solvers (solvers.hpp) ----------------------------------------------------------------
struct DeconvConfig {
  std::size_t max_iters = 500;
  double tol_rel_objective = 1e-6;
  std::optional<double> initial_step{};
  double backtrack_factor = 0.5;
  std::size_t max_backtracks = 50;
  std::size_t power_iters = 30;
};

struct RlConfig {
  std::size_t max_iters = 500;
  double tol_rel_change = 0.0;
};

enum class StopReason { converged, max_iters, stalled };

inline const char* to_string(StopReason r) {
  switch (r) {
    case StopReason::converged: return "converged";
    case StopReason::max_iters: return "max_iters";
    case StopReason::stalled: return "stalled";
  }
  return "unknown";
}

struct DeconvReport {
  Tensor estimate;
  std::vector<double> objective_trace;
  std::vector<double> kkt_trace;
  std::size_t iterations_run = 0;
  StopReason stop_reason = StopReason::max_iters;
  double wall_time_seconds = 0.0;
  std::size_t negative_pixels_clamped = 0;
};

inline double objective(const Tensor& x, const Tensor& y, const Kernel& h) {
  detail::check_forward_shapes(y, h, x.shape(), "objective");
  double f = 0.0;
  b200::check(ndc_objective_f64(static_cast<int>(x.shape().ndim()), x.shape().extents().data(),
                                x.data().data(), y.data().data(), h.shape().extents().data(),
                                h.tensor().data().data(), &f));
  return f;
}

inline double estimate_step(const Kernel& h, const Shape& x_shape, std::size_t power_iters) {
  if (x_shape.ndim() != h.ndim()) throw ShapeError("estimate_step: dimension count mismatch");
  double s = 0.0;
  b200::check(ndc_estimate_step_f64(static_cast<int>(h.ndim()), h.shape().extents().data(),
                                    h.tensor().data().data(), x_shape.extents().data(), power_iters,
                                    &s));
  return s;
}

inline double kkt_residual(const Tensor& x, const Tensor& y, const Kernel& h) {
  detail::check_forward_shapes(y, h, x.shape(), "kkt_residual");
  double k = 0.0;
  b200::check(ndc_kkt_residual_f64(static_cast<int>(x.shape().ndim()), x.shape().extents().data(),
                                   x.data().data(), y.data().data(), h.shape().extents().data(),
                                   h.tensor().data().data(), &k));
  return k;
}

namespace b200 {
inline ndc_deconv_config to_c(const DeconvConfig& c) {
  ndc_deconv_config r;
  r.max_iters = c.max_iters;
  r.tol_rel_objective = c.tol_rel_objective;
  r.has_initial_step = c.initial_step ? 1 : 0;
  r.initial_step = c.initial_step ? *c.initial_step : 0.0;
  r.backtrack_factor = c.backtrack_factor;
  r.max_backtracks = c.max_backtracks;
  r.power_iters = c.power_iters;
  return r;
}
inline DeconvReport report_of(const Shape& xs, std::vector<double> x, const ndc_deconv_report& r,
                              const double* obj, const double* kkt) {
  DeconvReport rep{Tensor(xs, std::move(x)),
                   std::vector<double>(obj, obj + r.trace_len),
                   std::vector<double>(kkt, kkt + r.trace_len),
                   r.iterations_run,
                   static_cast<StopReason>(r.stop_reason),
                   r.wall_time_seconds,
                   r.negative_pixels_clamped};
  return rep;
}
}  // namespace b200

inline DeconvReport deconv_pg(const Tensor& y, const Kernel& h, const Shape& x_shape,
                              const DeconvConfig& cfg = {}) {
  detail::check_forward_shapes(y, h, x_shape, "deconv_pg");
  const ndc_deconv_config c = b200::to_c(cfg);
  const std::size_t cap = cfg.max_iters + 1;
  std::vector<double> x(x_shape.element_count()), obj(cap), kkt(cap);
  ndc_deconv_report r{};
  b200::check(ndc_deconv_pg_f64(static_cast<int>(h.ndim()), y.shape().extents().data(),
                                y.data().data(), h.shape().extents().data(), h.tensor().data().data(),
                                x_shape.extents().data(), &c, x.data(), obj.data(), kkt.data(), cap,
                                &r));
  return b200::report_of(x_shape, std::move(x), r, obj.data(), kkt.data());
}

// Extension: `ys` independent observations of one shape, each with its own scalars.
inline std::vector<DeconvReport> deconv_pg_batch(const std::vector<Tensor>& ys, const Kernel& h,
                                                 const Shape& x_shape, const DeconvConfig& cfg = {}) {
  if (ys.empty()) return {};
  for (const Tensor& y : ys) detail::check_forward_shapes(y, h, x_shape, "deconv_pg");
  const std::size_t B = ys.size(), ny = ys[0].size(), nx = x_shape.element_count();
  std::vector<double> yv(B * ny);
  for (std::size_t b = 0; b < B; ++b) std::copy(ys[b].data().begin(), ys[b].data().end(), yv.begin() + b * ny);
  const ndc_deconv_config c = b200::to_c(cfg);
  const std::size_t cap = cfg.max_iters + 1;
  std::vector<double> x(B * nx), obj(B * cap), kkt(B * cap);
  std::vector<ndc_deconv_report> r(B);
  b200::check(ndc_deconv_pg_batch_f64(B, static_cast<int>(h.ndim()), ys[0].shape().extents().data(),
                                      yv.data(), h.shape().extents().data(), h.tensor().data().data(),
                                      x_shape.extents().data(), &c, x.data(), obj.data(), kkt.data(),
                                      cap, r.data()));
  std::vector<DeconvReport> out;
  for (std::size_t b = 0; b < B; ++b)
    out.push_back(b200::report_of(x_shape, std::vector<double>(x.begin() + b * nx, x.begin() + (b + 1) * nx),
                                  r[b], obj.data() + b * cap, kkt.data() + b * cap));
  return out;
}

inline DeconvReport deconv_rl(const Tensor& y, const Kernel& h, const Shape& x_shape,
                              const RlConfig& cfg = {}) {
  detail::check_forward_shapes(y, h, x_shape, "deconv_rl");
  ndc_rl_config c{cfg.max_iters, cfg.tol_rel_change};
  const std::size_t cap = cfg.max_iters + 1;
  std::vector<double> x(x_shape.element_count()), obj(cap), kkt(cap);
  ndc_deconv_report r{};
  b200::check(ndc_deconv_rl_f64(static_cast<int>(h.ndim()), y.shape().extents().data(),
                                y.data().data(), h.shape().extents().data(), h.tensor().data().data(),
                                x_shape.extents().data(), &c, x.data(), obj.data(), kkt.data(), cap,
                                &r));
  return b200::report_of(x_shape, std::move(x), r, obj.data(), kkt.data());
}

// ---- tensor files (imageio.hpp) ----------------------------------------------------------
namespace io {

inline Tensor read_tensor(const std::string& path) {
  int nd = 0;
  std::size_t ext[16];
  b200::check(ndc_ndtensor_info(path.c_str(), &nd, ext));
  Shape s(std::vector<std::size_t>(ext, ext + nd));
  std::vector<double> v(s.element_count());
  b200::check(ndc_ndtensor_read_f64(path.c_str(), v.data(), v.size()));
  return Tensor(std::move(s), std::move(v));
}

inline void write_tensor(const Tensor& t, const std::string& path) {
  b200::check(ndc_ndtensor_write_f64(path.c_str(), static_cast<int>(t.shape().ndim()),
                                     t.shape().extents().data(), t.data().data()));
}

inline Tensor read_pgm(const std::string& path) {
  std::size_t h = 0, w = 0;
  b200::check(ndc_pgm_info(path.c_str(), &h, &w));
  std::vector<double> v(h * w);
  b200::check(ndc_pgm_read_f64(path.c_str(), v.data(), v.size()));
  return Tensor(Shape{h, w}, std::move(v));
}

inline void write_pgm(const Tensor& t, const std::string& path, bool clamp) {
  if (t.shape().ndim() != 2)
    throw ShapeError("write_pgm: need a 2-d tensor, got " + t.shape().to_string());
  b200::check(ndc_pgm_write_f64(path.c_str(), t.shape().extent(0), t.shape().extent(1),
                                t.data().data(), clamp ? 1 : 0));
}

}  // namespace io

// ---- simulation (simulation.hpp:20-208; image-sized generation on the device) -------------
namespace sim {
struct NoiseSpec {
  double mean = 0.0;
  double std_dev = 0.0;
  std::uint64_t seed = 0;
};

struct PsfSpec {
  enum class Kind { gaussian, delta, custom };
  Kind kind = Kind::gaussian;
  std::vector<std::size_t> size{5, 5};
  double sigma = 1.0;
  std::optional<Tensor> values{};
};

inline Tensor phantom_lines(std::size_t rows, std::size_t cols, std::size_t n_lines, double intensity) {
  std::vector<double> v(rows * cols);
  b200::check(ndc_sim_phantom_lines_f64(rows, cols, n_lines, intensity, v.data()));
  return Tensor(Shape{rows, cols}, std::move(v));
}

inline Tensor phantom_texture(std::size_t rows, std::size_t cols) {
  std::vector<double> v(rows * cols);
  b200::check(ndc_sim_phantom_texture_f64(rows, cols, v.data()));
  return Tensor(Shape{rows, cols}, std::move(v));
}

inline Kernel gaussian_psf(const std::vector<std::size_t>& extents, double sigma) {
  std::size_t n = 1;
  for (std::size_t e : extents) n *= e;
  std::vector<double> v(extents.empty() ? 1 : n);
  b200::check(ndc_sim_gaussian_psf_f64(static_cast<int>(extents.size()), extents.data(), sigma, v.data()));
  return Kernel(Tensor(Shape(std::vector<std::size_t>(extents)), std::move(v)));
}

inline Kernel delta_psf(const std::vector<std::size_t>& extents) {
  std::size_t n = 1;
  for (std::size_t e : extents) n *= e;
  std::vector<double> v(extents.empty() ? 1 : n);
  b200::check(ndc_sim_delta_psf_f64(static_cast<int>(extents.size()), extents.data(), v.data()));
  return Kernel(Tensor(Shape(std::vector<std::size_t>(extents)), std::move(v)));
}

inline Kernel make_psf(const PsfSpec& spec) {
  switch (spec.kind) {
    case PsfSpec::Kind::gaussian:
      return gaussian_psf(spec.size, spec.sigma);
    case PsfSpec::Kind::delta:
      return delta_psf(spec.size);
    case PsfSpec::Kind::custom: {
      if (!spec.values) throw Error("make_psf: custom PSF needs values");
      for (double v : spec.values->data())
        if (v < 0.0) throw NumericError("make_psf: PSF values must be nonnegative");
      return Kernel(*spec.values);
    }
  }
  throw Error("make_psf: unknown kind");
}

inline Tensor add_gaussian_noise(const Tensor& t, const NoiseSpec& spec) {
  std::vector<double> v(t.size());
  b200::check(ndc_sim_add_gaussian_noise_f64(t.size(), t.data().data(), spec.mean, spec.std_dev, spec.seed,
                                             v.data()));
  return Tensor(t.shape(), std::move(v));
}

// ---- metrics (simulation.hpp:195-208) ------------------------------------------------------
inline double snr_db(const Tensor& reference, const Tensor& estimate) {
  ndconv::detail::check_same_shape(reference, estimate, "snr_db");
  double ref = 0.0, err = 0.0;
  for (std::size_t i = 0; i < reference.size(); ++i) {
    ref += reference[i] * reference[i];
    const double e = estimate[i] - reference[i];
    err += e * e;
  }
  if (ref == 0.0) throw NumericError("snr_db: reference is all zero, metric undefined");
  if (err == 0.0) return std::numeric_limits<double>::infinity();
  return 10.0 * std::log10(ref / err);
}
}  // namespace sim

}  // namespace ndconv
