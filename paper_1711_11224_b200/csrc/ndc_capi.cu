// extern "C" boundary (include/ndconv_b200.h).  Converts the reference's f64 dense
// tensors at the edge, maps internal failures to ndc_status codes that correspond to
// the reference's exception types, and keeps the message per thread.
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "ndc_io.h"
#include "ndc_plan.h"
#include "ndc_sim.h"

struct ndc_plan {
  std::unique_ptr<ndc::Plan> p;
};


namespace {

thread_local std::string g_last_error;
thread_local int g_device = 0;
unsigned g_max_threads = 1;

template <class F>
ndc_status guard(F&& f) {
  try {
    f();
    g_last_error.clear();
    return NDC_OK;
  } catch (const ndc::Error& e) {
    g_last_error = e.msg;
    return static_cast<ndc_status>(e.code);
  } catch (const std::bad_alloc&) {
    g_last_error = "host allocation failed";
    return NDC_ERR_ARGUMENT;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return NDC_ERR_ARGUMENT;
  }
}

void need(const void* p, const char* what) {
  if (p == nullptr) ndc::fail(NDC_ERR_ARGUMENT, std::string(what) + " is null");
}

size_t count_of(int ndim, const size_t* ext) {
  size_t n = 1;
  for (int i = 0; i < ndim; ++i) n *= ext[i];
  return n;
}

// Shape checks with the reference's messages and exception classes.
void check_ndim(int ndim) {
  if (ndim < 1) ndc::fail(NDC_ERR_SHAPE, "Shape: need at least one dimension");
}

void check_forward(int ndim, const size_t* y_ext, const size_t* k_ext, const size_t* x_ext,
                   const char* what) {
  for (int i = 0; i < ndim; ++i) {
    if (k_ext[i] % 2 == 0) ndc::fail(NDC_ERR_SHAPE, "Kernel: extents must be odd");
    if (x_ext[i] == 0 || y_ext[i] == 0) ndc::fail(NDC_ERR_SHAPE, "Shape: extents must be positive");
    if (y_ext[i] != x_ext[i] + k_ext[i] - 1)
      ndc::fail(NDC_ERR_SHAPE, std::string(what) + ": observation shape does not match forward model output");
  }
}

std::unique_ptr<ndc::Plan> one_shot(size_t batch, int ndim, const size_t* x_ext, const size_t* k_ext,
                                    const double* h) {
  return std::make_unique<ndc::Plan>(g_device, batch, ndim, x_ext, k_ext, h);
}

bool early_estimate() {
  static const bool on = [] {
    const char* e = std::getenv("NDC_EARLY_ESTIMATE");
    return e == nullptr || std::atoi(e) != 0;
  }();
  return on;
}

ndc_deconv_config default_cfg() {
  ndc_deconv_config c;
  ndc_deconv_config_default(&c);
  return c;
}

}  // namespace

extern "C" {

void ndc_deconv_config_default(ndc_deconv_config* c) {
  if (!c) return;
  c->max_iters = 500;
  c->tol_rel_objective = 1e-6;
  c->has_initial_step = 0;
  c->initial_step = 0.0;
  c->backtrack_factor = 0.5;
  c->max_backtracks = 50;
  c->power_iters = 30;
}

void ndc_rl_config_default(ndc_rl_config* c) {
  if (!c) return;
  c->max_iters = 500;
  c->tol_rel_change = 0.0;
}

const char* ndc_last_error(void) { return g_last_error.c_str(); }
const char* ndc_version(void) { return "ndconv_b200 0.1.0 (sm_100a)"; }

const char* ndc_stop_reason_name(int r) {
  switch (r) {
    case NDC_STOP_CONVERGED: return "converged";
    case NDC_STOP_MAX_ITERS: return "max_iters";
    case NDC_STOP_STALLED: return "stalled";
  }
  return "unknown";
}

ndc_status ndc_device_count(int* count) {
  return guard([&] {
    need(count, "count");
    int n = 0;
    *count = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
      cudaGetLastError();
      return;
    }
    for (int d = 0; d < n; ++d) {
      cudaDeviceProp p;
      if (cudaGetDeviceProperties(&p, d) == cudaSuccess && p.major == 10) ++*count;
    }
  });
}

ndc_status ndc_set_device(int device) {
  return guard([&] {
    if (device < 0) ndc::fail(NDC_ERR_ARGUMENT, "device ordinal must be >= 0");
    g_device = device;
  });
}

void ndc_set_max_threads(unsigned n) { g_max_threads = n == 0 ? 1 : n; }
unsigned ndc_max_threads(void) { return g_max_threads; }

ndc_status ndc_conv_output_shape(int ndim, const size_t* x_ext, const size_t* k_ext, size_t* out_ext) {
  return guard([&] {
    check_ndim(ndim);
    need(x_ext, "x_ext");
    need(k_ext, "k_ext");
    need(out_ext, "out_ext");
    for (int i = 0; i < ndim; ++i) {
      if (x_ext[i] == 0 || k_ext[i] == 0) ndc::fail(NDC_ERR_SHAPE, "Shape: extents must be positive");
      if (k_ext[i] % 2 == 0) ndc::fail(NDC_ERR_SHAPE, "Kernel: extents must be odd");
      out_ext[i] = x_ext[i] + k_ext[i] - 1;
    }
  });
}

ndc_status ndc_conv_full_f64(int ndim, const size_t* x_ext, const double* x, const size_t* k_ext,
                             const double* h, double* y) {
  return guard([&] {
    check_ndim(ndim);
    need(x, "x");
    need(h, "h");
    need(y, "y");
    auto p = one_shot(1, ndim, x_ext, k_ext, h);
    p->set_x_f64(x);
    p->op_conv_full();
    p->get_y_buffer_f64(y);
  });
}

ndc_status ndc_conv_full_batch_f32(size_t batch, int ndim, const size_t* x_ext, const float* x,
                                   const size_t* k_ext, const double* h, float* y) {
  return guard([&] {
    check_ndim(ndim);
    need(x, "x");
    need(h, "h");
    need(y, "y");
    auto p = one_shot(batch, ndim, x_ext, k_ext, h);
    p->set_x_f32(x);
    p->op_conv_full();
    p->get_y_buffer_f32(y);
  });
}
ndc_status ndc_adjoint_apply_batch_f32(size_t batch, int ndim, const size_t* y_ext, const float* y,
                                       const size_t* k_ext, const double* h, const size_t* x_ext,
                                       float* x_out) {
  return guard([&] {
    check_ndim(ndim);
    need(y, "y");
    need(h, "h");
    need(x_out, "x_out");
    for (int i = 0; i < ndim; ++i)
      if (y_ext[i] != x_ext[i] + k_ext[i] - 1)
        ndc::fail(NDC_ERR_SHAPE, "adjoint_apply: observation shape is not x_shape + 2p");
    check_forward(ndim, y_ext, k_ext, x_ext, "adjoint_apply");
    auto p = one_shot(batch, ndim, x_ext, k_ext, h);
    p->set_observation_f32(y);
    p->op_adjoint_of_y();
    p->get_x_buffer_f32(x_out);
  });
}
ndc_status ndc_adjoint_apply_f64(int ndim, const size_t* y_ext, const double* y, const size_t* k_ext,
                                 const double* h, const size_t* x_ext, double* x_out) {
  return guard([&] {
    check_ndim(ndim);
    need(y, "y");
    need(h, "h");
    need(x_out, "x_out");
    for (int i = 0; i < ndim; ++i)
      if (y_ext[i] != x_ext[i] + k_ext[i] - 1)
        ndc::fail(NDC_ERR_SHAPE, "adjoint_apply: observation shape is not x_shape + 2p");
    check_forward(ndim, y_ext, k_ext, x_ext, "adjoint_apply");
    auto p = one_shot(1, ndim, x_ext, k_ext, h);
    p->set_observation_f64(y);
    p->op_adjoint_of_y();
    p->get_x_buffer_f64(x_out, 0);
  });
}

ndc_status ndc_normal_gradient_f64(int ndim, const size_t* x_ext, const double* x, const double* y,
                                   const size_t* k_ext, const double* h, double* g) {
  return guard([&] {
    check_ndim(ndim);
    need(x, "x");
    need(y, "y");
    need(h, "h");
    need(g, "g");
    auto p = one_shot(1, ndim, x_ext, k_ext, h);
    p->set_x_f64(x);
    p->set_observation_f64(y);
    p->op_normal_gradient();
    p->get_x_buffer_f64(g, 1);
  });
}

ndc_status ndc_objective_f64(int ndim, const size_t* x_ext, const double* x, const double* y,
                             const size_t* k_ext, const double* h, double* f) {
  return guard([&] {
    check_ndim(ndim);
    need(x, "x");
    need(y, "y");
    need(h, "h");
    need(f, "f");
    auto p = one_shot(1, ndim, x_ext, k_ext, h);
    p->set_x_f64(x);
    p->set_observation_f64(y);
    *f = p->op_objective();
  });
}

ndc_status ndc_estimate_step_f64(int ndim, const size_t* k_ext, const double* h, const size_t* x_ext,
                                 size_t power_iters, double* step) {
  return guard([&] {
    check_ndim(ndim);
    need(h, "h");
    need(step, "step");
    if (power_iters == 0) ndc::fail(NDC_ERR_CONFIG, "estimate_step: power_iters must be positive");
    auto p = one_shot(1, ndim, x_ext, k_ext, h);
    *step = p->estimate_step(power_iters);
  });
}

ndc_status ndc_kkt_residual_f64(int ndim, const size_t* x_ext, const double* x, const double* y,
                                const size_t* k_ext, const double* h, double* kkt) {
  return guard([&] {
    check_ndim(ndim);
    need(x, "x");
    need(y, "y");
    need(h, "h");
    need(kkt, "kkt");
    auto p = one_shot(1, ndim, x_ext, k_ext, h);
    p->set_x_f64(x);
    p->set_observation_f64(y);
    *kkt = p->op_kkt_residual();
  });
}

ndc_status ndc_deconv_pg_f64(int ndim, const size_t* y_ext, const double* y, const size_t* k_ext,
                             const double* h, const size_t* x_ext, const ndc_deconv_config* cfg,
                             double* x_out, double* obj_trace, double* kkt_trace, size_t trace_cap,
                             ndc_deconv_report* report) {
  return ndc_deconv_pg_batch_f64(1, ndim, y_ext, y, k_ext, h, x_ext, cfg, x_out, obj_trace,
                                 kkt_trace, trace_cap, report);
}

ndc_status ndc_deconv_pg_batch_f64(size_t batch, int ndim, const size_t* y_ext, const double* y,
                                   const size_t* k_ext, const double* h, const size_t* x_ext,
                                   const ndc_deconv_config* cfg, double* x_out, double* obj_trace,
                                   double* kkt_trace, size_t trace_cap, ndc_deconv_report* reports) {
  return guard([&] {
    check_ndim(ndim);
    need(y, "y");
    need(h, "h");
    need(x_out, "x_out");
    need(reports, "report");
    const ndc_deconv_config c = cfg ? *cfg : default_cfg();
    if (c.max_iters == 0) ndc::fail(NDC_ERR_CONFIG, "DeconvConfig: max_iters must be positive");
    check_forward(ndim, y_ext, k_ext, x_ext, "deconv_pg");
    if ((obj_trace || kkt_trace) && trace_cap < c.max_iters + 1)
      ndc::fail(NDC_ERR_ARGUMENT, "trace_cap must be at least max_iters + 1");
    auto p = one_shot(batch, ndim, x_ext, k_ext, h);
    if (early_estimate() && !c.has_initial_step && c.power_iters > 0 && !p->kernel_all_zero())
      p->estimate_launch(c.power_iters);  // overlaps the upload below
    p->set_observation_f64(y);
    p->pg_begin(c);
    p->pg_iterate(c.max_iters);
    p->pg_end();
    p->get_estimate_f64(x_out);
    for (size_t b = 0; b < batch; ++b)
      p->get_report(b, reports + b, obj_trace ? obj_trace + b * trace_cap : nullptr,
                    kkt_trace ? kkt_trace + b * trace_cap : nullptr, trace_cap);
  });
}

ndc_status ndc_deconv_pg_batch_f32(size_t batch, int ndim, const size_t* y_ext, const float* y,
                                   const size_t* k_ext, const double* h, const size_t* x_ext,
                                   const ndc_deconv_config* cfg, float* x_out, double* obj_trace,
                                   double* kkt_trace, size_t trace_cap, ndc_deconv_report* reports) {
  return guard([&] {
    check_ndim(ndim);
    need(y, "y");
    need(h, "h");
    need(x_out, "x_out");
    need(reports, "report");
    const ndc_deconv_config c = cfg ? *cfg : default_cfg();
    if (c.max_iters == 0) ndc::fail(NDC_ERR_CONFIG, "DeconvConfig: max_iters must be positive");
    check_forward(ndim, y_ext, k_ext, x_ext, "deconv_pg");
    if ((obj_trace || kkt_trace) && trace_cap < c.max_iters + 1)
      ndc::fail(NDC_ERR_ARGUMENT, "trace_cap must be at least max_iters + 1");
    auto p = one_shot(batch, ndim, x_ext, k_ext, h);
    if (early_estimate() && !c.has_initial_step && c.power_iters > 0 && !p->kernel_all_zero())
      p->estimate_launch(c.power_iters);  // overlaps the upload below
    p->set_observation_f32(y);
    p->pg_begin(c);
    p->pg_iterate(c.max_iters);
    p->pg_end();
    p->get_estimate_f32(x_out);
    for (size_t b = 0; b < batch; ++b)
      p->get_report(b, reports + b, obj_trace ? obj_trace + b * trace_cap : nullptr,
                    kkt_trace ? kkt_trace + b * trace_cap : nullptr, trace_cap);
  });
}

ndc_status ndc_deconv_rl_f64(int ndim, const size_t* y_ext, const double* y, const size_t* k_ext,
                             const double* h, const size_t* x_ext, const ndc_rl_config* cfg,
                             double* x_out, double* obj_trace, double* kkt_trace, size_t trace_cap,
                             ndc_deconv_report* report) {
  return guard([&] {
    check_ndim(ndim);
    need(y, "y");
    need(h, "h");
    need(x_out, "x_out");
    need(report, "report");
    ndc_rl_config c;
    ndc_rl_config_default(&c);
    if (cfg) c = *cfg;
    if (c.max_iters == 0) ndc::fail(NDC_ERR_CONFIG, "RlConfig: max_iters must be positive");
    if (!(c.tol_rel_change >= 0)) ndc::fail(NDC_ERR_CONFIG, "RlConfig: tol_rel_change must be >= 0");
    check_forward(ndim, y_ext, k_ext, x_ext, "deconv_rl");
    if ((obj_trace || kkt_trace) && trace_cap < c.max_iters + 1)
      ndc::fail(NDC_ERR_ARGUMENT, "trace_cap must be at least max_iters + 1");
    auto p = one_shot(1, ndim, x_ext, k_ext, h);
    p->set_observation_f64(y);
    p->rl_run(c);
    p->get_estimate_f64(x_out);
    p->get_report(0, report, obj_trace, kkt_trace, trace_cap);
  });
}

// ---- plan API ---------------------------------------------------------------------------
ndc_status ndc_plan_create(ndc_plan** plan, int device, size_t batch, int ndim, const size_t* x_ext,
                           const size_t* k_ext, const double* h) {
  return guard([&] {
    need(plan, "plan");
    check_ndim(ndim);
    need(x_ext, "x_ext");
    need(k_ext, "k_ext");
    need(h, "h");
    auto* w = new ndc_plan;
    try {
      w->p = std::make_unique<ndc::Plan>(device, batch, ndim, x_ext, k_ext, h);
    } catch (...) {
      delete w;
      throw;
    }
    *plan = w;
  });
}

ndc_status ndc_plan_destroy(ndc_plan* plan) {
  return guard([&] { delete plan; });
}

#define NDC_PLAN(expr)                    \
  return guard([&] {                      \
    need(plan, "plan");                   \
    expr;                                 \
  })

ndc_status ndc_plan_set_observation_f64(ndc_plan* plan, const double* y) {
  NDC_PLAN(need(y, "y"); plan->p->set_observation_f64(y));
}
ndc_status ndc_plan_set_observation_f32(ndc_plan* plan, const float* y) {
  NDC_PLAN(need(y, "y"); plan->p->set_observation_f32(y));
}
ndc_status ndc_plan_pg_begin(ndc_plan* plan, const ndc_deconv_config* cfg) {
  NDC_PLAN(plan->p->pg_begin(cfg ? *cfg : default_cfg()));
}
ndc_status ndc_plan_pg_iterate(ndc_plan* plan, size_t n, size_t* images_active) {
  NDC_PLAN(const size_t a = plan->p->pg_iterate(n); if (images_active) *images_active = a);
}
ndc_status ndc_plan_pg_end(ndc_plan* plan) { NDC_PLAN(plan->p->pg_end()); }
ndc_status ndc_plan_pg_run(ndc_plan* plan, const ndc_deconv_config* cfg) {
  NDC_PLAN(const ndc_deconv_config c = cfg ? *cfg : default_cfg(); plan->p->pg_begin(c);
           plan->p->pg_iterate(c.max_iters); plan->p->pg_end());
}
ndc_status ndc_plan_rl_run(ndc_plan* plan, const ndc_rl_config* cfg) {
  NDC_PLAN(ndc_rl_config c; ndc_rl_config_default(&c); if (cfg) c = *cfg; plan->p->rl_run(c));
}
ndc_status ndc_plan_get_report(ndc_plan* plan, size_t image, ndc_deconv_report* report,
                               double* obj_trace, double* kkt_trace, size_t trace_cap) {
  NDC_PLAN(need(report, "report"); plan->p->get_report(image, report, obj_trace, kkt_trace, trace_cap));
}
ndc_status ndc_plan_get_estimate_f64(ndc_plan* plan, double* x_out) {
  NDC_PLAN(need(x_out, "x_out"); plan->p->get_estimate_f64(x_out));
}
ndc_status ndc_plan_get_estimate_f32(ndc_plan* plan, float* x_out) {
  NDC_PLAN(need(x_out, "x_out"); plan->p->get_estimate_f32(x_out));
}
ndc_status ndc_plan_get_observation_f64(ndc_plan* plan, double* y_out) {
  NDC_PLAN(need(y_out, "y_out"); plan->p->get_observation_f64(y_out));
}
ndc_status ndc_plan_load_observation_ndtensor(ndc_plan* plan, const char* path) {
  NDC_PLAN(need(path, "path"); plan->p->load_observation_ndtensor(path));
}
ndc_status ndc_plan_save_estimate_ndtensor(ndc_plan* plan, const char* path) {
  NDC_PLAN(need(path, "path"); plan->p->save_estimate_ndtensor(path));
}
ndc_status ndc_plan_add_gaussian_noise(ndc_plan* plan, double mean, double std_dev, uint64_t seed) {
  NDC_PLAN(plan->p->add_gaussian_noise(mean, std_dev, seed));
}

// ---- simulation generators (ndc_sim.cu) -----------------------------------------------------
ndc_status ndc_sim_phantom_lines_f64(size_t rows, size_t cols, size_t n_lines, double intensity, double* out) {
  return guard([&] {
    need(out, "out");
    ndc::sim_phantom_lines(g_device, rows, cols, n_lines, intensity, out);
  });
}
ndc_status ndc_sim_phantom_texture_f64(size_t rows, size_t cols, double* out) {
  return guard([&] {
    need(out, "out");
    ndc::sim_phantom_texture(g_device, rows, cols, out);
  });
}
ndc_status ndc_sim_gaussian_psf_f64(int ndim, const size_t* ext, double sigma, double* out) {
  return guard([&] {
    need(ext, "ext");
    need(out, "out");
    ndc::sim_gaussian_psf(ndim, ext, sigma, out);
  });
}
ndc_status ndc_sim_delta_psf_f64(int ndim, const size_t* ext, double* out) {
  return guard([&] {
    need(ext, "ext");
    need(out, "out");
    ndc::sim_delta_psf(ndim, ext, out);
  });
}
ndc_status ndc_sim_add_gaussian_noise_f64(size_t n, const double* in, double mean, double std_dev, uint64_t seed,
                                          double* out) {
  return guard([&] {
    if (n) {
      need(in, "in");
      need(out, "out");
    }
    ndc::sim_add_gaussian_noise(g_device, n, in, mean, std_dev, seed, out);
  });
}
ndc_status ndc_sim_mt19937_64(uint64_t seed, size_t skip, size_t n, uint64_t* out) {
  return guard([&] {
    if (n) need(out, "out");
    ndc::sim_mt19937_64(g_device, seed, skip, n, out);
  });
}

// ---- tensor files ---------------------------------------------------------------------------
ndc_status ndc_ndtensor_info(const char* path, int* ndim, size_t* ext16) {
  return guard([&] {
    need(path, "path");
    need(ndim, "ndim");
    need(ext16, "ext");
    const ndc::NdtHeader h = ndc::read_ndtensor_header(path);
    *ndim = static_cast<int>(h.ext.size());
    for (size_t i = 0; i < h.ext.size(); ++i) ext16[i] = h.ext[i];
  });
}

ndc_status ndc_ndtensor_read_f64(const char* path, double* out, size_t capacity) {
  return guard([&] {
    need(path, "path");
    need(out, "out");
    ndc::read_ndtensor(path, out, capacity, nullptr);
  });
}

ndc_status ndc_ndtensor_write_f64(const char* path, int ndim, const size_t* ext, const double* data) {
  return guard([&] {
    need(path, "path");
    need(ext, "ext");
    need(data, "data");
    check_ndim(ndim);
    for (int i = 0; i < ndim; ++i)
      if (ext[i] == 0) ndc::fail(NDC_ERR_SHAPE, "Shape: extents must be positive");
    ndc::write_ndtensor(path, std::vector<size_t>(ext, ext + ndim), data);
  });
}

ndc_status ndc_pgm_info(const char* path, size_t* height, size_t* width) {
  return guard([&] {
    need(path, "path");
    need(height, "height");
    need(width, "width");
    std::vector<double> d;
    ndc::read_pgm(path, &d, height, width);
  });
}

ndc_status ndc_pgm_read_f64(const char* path, double* out, size_t capacity) {
  return guard([&] {
    need(path, "path");
    need(out, "out");
    std::vector<double> d;
    size_t h = 0, w = 0;
    ndc::read_pgm(path, &d, &h, &w);
    if (capacity < d.size()) ndc::fail(NDC_ERR_ARGUMENT, "read_pgm: output capacity too small");
    std::memcpy(out, d.data(), d.size() * 8);
  });
}

ndc_status ndc_pgm_write_f64(const char* path, size_t height, size_t width, const double* data,
                             int clamp) {
  return guard([&] {
    need(path, "path");
    need(data, "data");
    if (height == 0 || width == 0) ndc::fail(NDC_ERR_SHAPE, "Shape: extents must be positive");
    ndc::write_pgm(path, height, width, data, clamp != 0);
  });
}

ndc_status ndc_plan_forward(ndc_plan* plan) { NDC_PLAN(plan->p->bench_forward()); }
ndc_status ndc_plan_adjoint(ndc_plan* plan) { NDC_PLAN(plan->p->bench_adjoint()); }
ndc_status ndc_plan_set_timing(ndc_plan* plan, int enabled) {
  NDC_PLAN(plan->p->set_timing(enabled != 0));
}
ndc_status ndc_plan_reset_stats(ndc_plan* plan) { NDC_PLAN(plan->p->reset_stats()); }
ndc_status ndc_plan_stats(ndc_plan* plan, int kind, uint64_t* launches, double* total_ms) {
  NDC_PLAN(const ndc::KernelStats s = plan->p->stats(kind); if (launches) *launches = s.launches;
           if (total_ms) *total_ms = s.ms);
}
ndc_status ndc_plan_stream(ndc_plan* plan, void** cuda_stream) {
  NDC_PLAN(need(cuda_stream, "cuda_stream"); *cuda_stream = plan->p->stream());
}

// ---- z-slab sharding ----------------------------------------------------------------------
ndc_status ndc_slab_range(size_t mz, size_t pz, int rank, int world, size_t* x_begin, size_t* x_end,
                          size_t* y_begin, size_t* y_end) {
  return guard([&] {
    if (world < 1 || rank < 0 || rank >= world) ndc::fail(NDC_ERR_ARGUMENT, "bad rank / world");
    if (mz == 0) ndc::fail(NDC_ERR_SHAPE, "Shape: extents must be positive");
    const size_t w = static_cast<size_t>(world), r = static_cast<size_t>(rank);
    const size_t base = mz / w, rem = mz % w;
    const size_t a = r * base + (r < rem ? r : rem);
    const size_t b = a + base + (r < rem ? 1 : 0);
    if (x_begin) *x_begin = a;
    if (x_end) *x_end = b;
    if (y_begin) *y_begin = (r == 0) ? 0 : a + pz;
    if (y_end) *y_end = (r + 1 == w) ? mz + 2 * pz : b + pz;
  });
}

ndc_status ndc_plan_create_sharded(ndc_plan** plan, int device, int ndim, const size_t* x_ext,
                                   const size_t* k_ext, const double* h, int rank, int world,
                                   const unsigned char nccl_id[128]) {
  return guard([&] {
    need(plan, "plan");
    need(nccl_id, "nccl_id");
    auto comm = ndc::make_nccl_transport(device, rank, world, nccl_id);
    auto* w = new ndc_plan;
    try {
      w->p = std::make_unique<ndc::Plan>(device, 1, ndim, x_ext, k_ext, h, std::move(comm));
    } catch (...) {
      delete w;
      throw;
    }
    *plan = w;
  });
}

ndc_status ndc_plan_check_guards(ndc_plan* plan, size_t* bad_bytes) {
  NDC_PLAN(need(bad_bytes, "bad_bytes"); *bad_bytes = plan->p->check_guards());
}
ndc_status ndc_plan_debug_corrupt_guard(ndc_plan* plan) { NDC_PLAN(plan->p->debug_corrupt_guard()); }
ndc_status ndc_debug_guard_violations(unsigned long long* total_bad) {
  return guard([&] {
    need(total_bad, "total_bad");
    *total_bad = ndc::guard_violations();
  });
}

ndc_status ndc_probe_fp32_peak(int device, double* tflops) {
  return guard([&] {
    need(tflops, "tflops");
    *tflops = ndc::probe_fp32_peak(device);
  });
}

ndc_status ndc_nccl_unique_id(unsigned char id[128]) {
  return guard([&] {
    need(id, "id");
    ndc::nccl_unique_id(id);
  });
}

ndc_status ndc_local_group_create(ndc_local_group** group, int world) {
  return guard([&] {
    need(group, "group");
    if (world < 1) ndc::fail(NDC_ERR_ARGUMENT, "world must be >= 1");
    *group = reinterpret_cast<ndc_local_group*>(ndc::new_local_group(world));
  });
}

ndc_status ndc_local_group_destroy(ndc_local_group* group) {
  return guard([&] { ndc::delete_local_group(reinterpret_cast<ndc::LocalGroup*>(group)); });
}

ndc_status ndc_plan_create_local(ndc_plan** plan, ndc_local_group* group, int rank, int device,
                                 int ndim, const size_t* x_ext, const size_t* k_ext,
                                 const double* h) {
  return guard([&] {
    need(plan, "plan");
    need(group, "group");
    check_ndim(ndim);
    auto comm = ndc::make_local_transport(reinterpret_cast<ndc::LocalGroup*>(group), rank);
    auto* w = new ndc_plan;
    try {
      w->p = std::make_unique<ndc::Plan>(device, 1, ndim, x_ext, k_ext, h, std::move(comm));
    } catch (...) {
      delete w;
      throw;
    }
    *plan = w;
  });
}

}  // extern "C"

