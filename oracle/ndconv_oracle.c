/*
 * TEST INFRASTRUCTURE ONLY -- CPU oracle for the ndconv projected-gradient hot path.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load this file's library, and only as the checker or the reported CPU
 * baseline.  The product (paper_1711_11224_b200/libndconv_b200.so) never links it.
 *
 * This is a plain-C restatement of the reference algorithm in f64.  Every routine
 * keeps the reference's summation order so results are bitwise equal to the
 * reference (pinned by tests/test_oracle.py against tests/golden/ fixtures that
 * oracle/_ref -- the reference compiled from /root/reference -- produced).
 *
 * Reference map (paths under /root/reference/proj/include/ndconv/):
 *   conv_output_shape      convolution.hpp:30-38
 *   conv_element           convolution.hpp:55-74   (per-dimension tap clipping)
 *   conv_full              convolution.hpp:81-123
 *   crop_center / crop_m   convolution.hpp:126-162
 *   adjoint_apply          convolution.hpp:166-174 (flip + conv_full + crop_m)
 *   normal_gradient        convolution.hpp:178-185
 *   objective              solvers.hpp:119-122
 *   estimate_step          solvers.hpp:127-143
 *   kkt_from_gradient      solvers.hpp:98-103
 *   deconv_pg              solvers.hpp:155-238
 *   deconv_rl              solvers.hpp:245-305
 *   tensor ops             tensor.hpp:99-144 (sequential f64 dot / norm2 / sum)
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OC_MAXDIM 8

enum { OC_OK = 0, OC_ERROR = 1, OC_SHAPE = 2, OC_NUMERIC = 3, OC_ALLOC = 9 };

typedef struct {
  size_t max_iters;
  double tol_rel_objective;
  int has_initial_step;
  double initial_step;
  double backtrack_factor;
  size_t max_backtracks;
  size_t power_iters;
} oc_pg_config;

typedef struct {
  size_t max_iters;
  double tol_rel_change;
} oc_rl_config;

/* stop reasons, solvers.hpp:37 order */
enum { OC_CONVERGED = 0, OC_MAX_ITERS = 1, OC_STALLED = 2 };

static int g_threads = 1; /* informational: the restatement is single-threaded */
void oc_set_threads(int n) { g_threads = n < 1 ? 1 : n; }

static size_t count_of(int ndim, const size_t* ext) {
  size_t n = 1;
  for (int i = 0; i < ndim; ++i) n *= ext[i];
  return n;
}

static void strides(int ndim, const size_t* ext, size_t* st) {
  size_t acc = 1;
  for (int i = ndim - 1; i >= 0; --i) {
    st[i] = acc;
    acc *= ext[i];
  }
}

typedef struct {
  const double* x;
  const double* h;
  const size_t* xext;
  const size_t* hext;
  size_t xst[OC_MAXDIM];
  size_t hst[OC_MAXDIM];
  int ndim;
} view_t;

/* convolution.hpp:55-74: taps j with s-j inside the input, innermost dimension a
 * reversed contiguous dot; recursion order over dimensions fixes the sum order. */
static double element(const view_t* v, const size_t* s_idx, int dim, size_t xoff, size_t hoff) {
  const size_t s = s_idx[dim];
  const size_t d = v->xext[dim];
  const size_t jlo = s >= d ? s - d + 1 : 0;
  const size_t jhi = (v->hext[dim] - 1) < s ? (v->hext[dim] - 1) : s;
  double acc = 0.0;
  if (dim + 1 == v->ndim) {
    const double* xp = v->x + xoff + (s - jlo);
    const double* hp = v->h + hoff + jlo;
    const size_t n = jhi - jlo + 1;
    for (size_t k = 0; k < n; ++k) acc += xp[-(ptrdiff_t)k] * hp[k];
  } else {
    for (size_t j = jlo; j <= jhi; ++j)
      acc += element(v, s_idx, dim + 1, xoff + (s - j) * v->xst[dim], hoff + j * v->hst[dim]);
  }
  return acc;
}

static int check_kernel(int ndim, const size_t* hext) {
  if (ndim < 1 || ndim > OC_MAXDIM) return OC_SHAPE;
  for (int i = 0; i < ndim; ++i)
    if (hext[i] == 0 || hext[i] % 2 == 0) return OC_SHAPE; /* kernel.hpp:18-22 */
  return OC_OK;
}

int oc_conv_output_shape(int ndim, const size_t* xext, const size_t* hext, size_t* yext) {
  int rc = check_kernel(ndim, hext);
  if (rc) return rc;
  for (int i = 0; i < ndim; ++i) {
    if (xext[i] == 0) return OC_SHAPE;
    yext[i] = xext[i] + (hext[i] - 1); /* d + 2p */
  }
  return OC_OK;
}

/* convolution.hpp:81-123 */
int oc_conv_full(int ndim, const size_t* xext, const double* x, const size_t* hext,
                 const double* h, double* y) {
  size_t yext[OC_MAXDIM];
  int rc = oc_conv_output_shape(ndim, xext, hext, yext);
  if (rc) return rc;
  view_t v;
  v.x = x;
  v.h = h;
  v.xext = xext;
  v.hext = hext;
  v.ndim = ndim;
  strides(ndim, xext, v.xst);
  strides(ndim, hext, v.hst);
  const long long total = (long long)count_of(ndim, yext);
  for (long long f = 0; f < total; ++f) {
    size_t idx[OC_MAXDIM];
    size_t rem = (size_t)f;
    for (int i = ndim - 1; i >= 0; --i) {
      idx[i] = rem % yext[i];
      rem /= yext[i];
    }
    y[f] = element(&v, idx, 0, 0, 0);
  }
  return OC_OK;
}

/* convolution.hpp:126-149 (offset (te-ge)/2 per dimension) */
static void crop_center(int ndim, const size_t* text, const double* t, const size_t* gext,
                        double* out) {
  size_t off[OC_MAXDIM], tst[OC_MAXDIM], idx[OC_MAXDIM];
  strides(ndim, text, tst);
  for (int i = 0; i < ndim; ++i) {
    off[i] = (text[i] - gext[i]) / 2;
    idx[i] = 0;
  }
  const size_t total = count_of(ndim, gext);
  for (size_t f = 0; f < total; ++f) {
    size_t src = 0;
    for (int i = 0; i < ndim; ++i) src += (idx[i] + off[i]) * tst[i];
    out[f] = t[src];
    for (int i = ndim - 1; i >= 0; --i) {
      if (++idx[i] < gext[i]) break;
      idx[i] = 0;
    }
  }
}

/* convolution.hpp:166-174: crop_m(conv_full(y, flip(h)), radii, x_shape) */
int oc_adjoint_apply(int ndim, const size_t* yext, const double* y, const size_t* hext,
                     const double* h, const size_t* xext, double* out) {
  int rc = check_kernel(ndim, hext);
  if (rc) return rc;
  for (int i = 0; i < ndim; ++i)
    if (xext[i] == 0 || yext[i] != xext[i] + (hext[i] - 1)) return OC_SHAPE;
  const size_t K = count_of(ndim, hext);
  double* hf = (double*)malloc(K * sizeof(double));
  size_t bigext[OC_MAXDIM];
  for (int i = 0; i < ndim; ++i) bigext[i] = yext[i] + (hext[i] - 1); /* m + 4p */
  double* big = (double*)malloc(count_of(ndim, bigext) * sizeof(double));
  if (!hf || !big) {
    free(hf);
    free(big);
    return OC_ALLOC;
  }
  for (size_t i = 0; i < K; ++i) hf[i] = h[K - 1 - i]; /* kernel.hpp:41-45 */
  rc = oc_conv_full(ndim, yext, y, hext, hf, big);
  if (!rc) crop_center(ndim, bigext, big, xext, out);
  free(hf);
  free(big);
  return rc;
}

static double dot(const double* a, const double* b, size_t n) { /* tensor.hpp:137-142 */
  double acc = 0.0;
  for (size_t i = 0; i < n; ++i) acc += a[i] * b[i];
  return acc;
}

static double half_sq_resid(const double* ax, const double* y, double* r, size_t n) {
  for (size_t i = 0; i < n; ++i) r[i] = ax[i] - y[i];
  return 0.5 * dot(r, r, n);
}

/* solvers.hpp:119-122 */
int oc_objective(int ndim, const size_t* xext, const double* x, const double* y,
                 const size_t* hext, const double* h, double* f) {
  size_t yext[OC_MAXDIM];
  int rc = oc_conv_output_shape(ndim, xext, hext, yext);
  if (rc) return rc;
  const size_t ny = count_of(ndim, yext);
  double* ax = (double*)malloc(ny * sizeof(double));
  double* r = (double*)malloc(ny * sizeof(double));
  if (!ax || !r) {
    free(ax);
    free(r);
    return OC_ALLOC;
  }
  rc = oc_conv_full(ndim, xext, x, hext, h, ax);
  if (!rc) *f = half_sq_resid(ax, y, r, ny);
  free(ax);
  free(r);
  return rc;
}

/* convolution.hpp:178-185: adjoint(conv(x)) - adjoint(y) */
int oc_normal_gradient(int ndim, const size_t* xext, const double* x, const double* y,
                       const size_t* hext, const double* h, double* g) {
  size_t yext[OC_MAXDIM];
  int rc = oc_conv_output_shape(ndim, xext, hext, yext);
  if (rc) return rc;
  const size_t ny = count_of(ndim, yext), nx = count_of(ndim, xext);
  double* ax = (double*)malloc(ny * sizeof(double));
  double* aty = (double*)malloc(nx * sizeof(double));
  if (!ax || !aty) {
    free(ax);
    free(aty);
    return OC_ALLOC;
  }
  rc = oc_conv_full(ndim, xext, x, hext, h, ax);
  if (!rc) rc = oc_adjoint_apply(ndim, yext, ax, hext, h, xext, g);
  if (!rc) rc = oc_adjoint_apply(ndim, yext, y, hext, h, xext, aty);
  if (!rc)
    for (size_t i = 0; i < nx; ++i) g[i] = g[i] - aty[i];
  free(ax);
  free(aty);
  return rc;
}

static int kernel_all_zero(const double* h, size_t K) {
  for (size_t i = 0; i < K; ++i)
    if (h[i] != 0.0) return 0;
  return 1;
}

/* solvers.hpp:127-143 */
int oc_estimate_step(int ndim, const size_t* hext, const double* h, const size_t* xext,
                     size_t power_iters, double* step) {
  if (power_iters == 0) return OC_ERROR;
  size_t yext[OC_MAXDIM];
  int rc = oc_conv_output_shape(ndim, xext, hext, yext);
  if (rc) return rc;
  if (kernel_all_zero(h, count_of(ndim, hext))) return OC_NUMERIC;
  const size_t nx = count_of(ndim, xext), ny = count_of(ndim, yext);
  double* v = (double*)malloc(nx * sizeof(double));
  double* w = (double*)malloc(nx * sizeof(double));
  double* u = (double*)malloc(ny * sizeof(double));
  if (!v || !w || !u) {
    rc = OC_ALLOC;
    goto done;
  }
  for (size_t i = 0; i < nx; ++i) v[i] = 1.0;
  {
    const double s = 1.0 / sqrt(dot(v, v, nx));
    for (size_t i = 0; i < nx; ++i) v[i] = v[i] * s;
  }
  double lambda = 0.0;
  for (size_t it = 0; it < power_iters; ++it) {
    rc = oc_conv_full(ndim, xext, v, hext, h, u);
    if (!rc) rc = oc_adjoint_apply(ndim, yext, u, hext, h, xext, w);
    if (rc) goto done;
    lambda = sqrt(dot(w, w, nx));
    if (!(lambda > 0.0) || !isfinite(lambda)) {
      rc = OC_NUMERIC;
      goto done;
    }
    const double s = 1.0 / lambda;
    for (size_t i = 0; i < nx; ++i) v[i] = w[i] * s;
  }
  *step = 1.0 / lambda;
done:
  free(v);
  free(w);
  free(u);
  return rc;
}

/* solvers.hpp:98-103 */
static double kkt_from_gradient(const double* x, const double* g, size_t n) {
  double worst = 0.0;
  for (size_t i = 0; i < n; ++i) {
    const double m = fabs(x[i] < g[i] ? x[i] : g[i]);
    if (m > worst) worst = m;
  }
  return worst;
}

/* solvers.hpp:147-149 */
int oc_kkt_residual(int ndim, const size_t* xext, const double* x, const double* y,
                    const size_t* hext, const double* h, double* kkt) {
  const size_t nx = count_of(ndim, xext);
  double* g = (double*)malloc(nx * sizeof(double));
  if (!g) return OC_ALLOC;
  int rc = oc_normal_gradient(ndim, xext, x, y, hext, h, g);
  if (!rc) *kkt = kkt_from_gradient(x, g, nx);
  free(g);
  return rc;
}

/* solvers.hpp:65-76 */
static int validate_pg(const oc_pg_config* c) {
  if (c->max_iters == 0) return OC_ERROR;
  if (!(c->tol_rel_objective >= 0)) return OC_ERROR;
  if (c->has_initial_step && !(c->initial_step > 0)) return OC_ERROR;
  if (!(c->backtrack_factor > 0) || !(c->backtrack_factor < 1)) return OC_ERROR;
  if (c->max_backtracks == 0) return OC_ERROR;
  if (c->power_iters == 0) return OC_ERROR;
  return OC_OK;
}

/* solvers.hpp:155-238.  Traces are written into caller arrays of capacity
 * max_iters + 1; *trace_len receives the objective-trace length (== kkt length). */
int oc_deconv_pg(int ndim, const size_t* yext, const double* y, const size_t* hext,
                 const double* h, const size_t* xext, const oc_pg_config* cfg, double* x_out,
                 double* obj_trace, double* kkt_trace, size_t* trace_len, size_t* iters_run,
                 int* stop_reason, size_t* backtracks_out) {
  int rc = validate_pg(cfg);
  if (rc) return rc;
  size_t want[OC_MAXDIM];
  rc = oc_conv_output_shape(ndim, xext, hext, want);
  if (rc) return rc;
  for (int i = 0; i < ndim; ++i)
    if (want[i] != yext[i]) return OC_SHAPE; /* solvers.hpp:83-90 */
  if (kernel_all_zero(h, count_of(ndim, hext))) return OC_NUMERIC;

  double step0 = 0.0;
  if (cfg->has_initial_step)
    step0 = cfg->initial_step;
  else if ((rc = oc_estimate_step(ndim, hext, h, xext, cfg->power_iters, &step0)))
    return rc;

  const size_t nx = count_of(ndim, xext), ny = count_of(ndim, yext);
  double *aty = malloc(nx * 8), *x = malloc(nx * 8), *g = malloc(nx * 8),
         *trial = malloc(nx * 8), *ax = malloc(ny * 8), *ax_t = malloc(ny * 8),
         *r = malloc(ny * 8);
  if (!aty || !x || !g || !trial || !ax || !ax_t || !r) {
    rc = OC_ALLOC;
    goto done;
  }
  if ((rc = oc_adjoint_apply(ndim, yext, y, hext, h, xext, aty))) goto done;
  for (size_t i = 0; i < nx; ++i) x[i] = aty[i] < 0.0 ? 0.0 : aty[i];
  if ((rc = oc_conv_full(ndim, xext, x, hext, h, ax))) goto done;
  double f = half_sq_resid(ax, y, r, ny);

  size_t tlen = 0, klen = 0, iterations = 0, backtracks = 0;
  int reason = OC_MAX_ITERS;
  obj_trace[tlen++] = f;
  for (size_t k = 1; k <= cfg->max_iters; ++k) {
    /* g = adjoint(ax) - aty  (solvers.hpp:180) */
    if ((rc = oc_adjoint_apply(ndim, yext, ax, hext, h, xext, g))) goto done;
    for (size_t i = 0; i < nx; ++i) g[i] = g[i] - aty[i];
    kkt_trace[klen++] = kkt_from_gradient(x, g, nx);

    double step = step0;
    int accepted = 0, fixed_point = 0;
    double f_next = f;
    for (size_t b = 0; b <= cfg->max_backtracks; ++b) {
      int same = 1;
      for (size_t i = 0; i < nx; ++i) {
        const double t = x[i] - g[i] * step; /* sub(x, scale(g, step)) */
        trial[i] = t < 0.0 ? 0.0 : t;
        if (trial[i] != x[i]) same = 0;
      }
      if (same) {
        fixed_point = 1;
        break;
      }
      if ((rc = oc_conv_full(ndim, xext, trial, hext, h, ax_t))) goto done;
      const double f_trial = half_sq_resid(ax_t, y, r, ny);
      if (f_trial < f) {
        f_next = f_trial;
        accepted = 1;
        break;
      }
      ++backtracks;
      step *= cfg->backtrack_factor;
    }
    if (fixed_point) {
      reason = OC_CONVERGED;
      break;
    }
    if (!accepted) {
      reason = OC_STALLED;
      break;
    }
    const double drop = f - f_next;
    double* tmp = x;
    x = trial;
    trial = tmp;
    tmp = ax;
    ax = ax_t;
    ax_t = tmp;
    f = f_next;
    obj_trace[tlen++] = f;
    iterations = k;
    if (drop <= cfg->tol_rel_objective * obj_trace[tlen - 2]) {
      reason = OC_CONVERGED;
      break;
    }
  }
  if (klen < tlen) { /* solvers.hpp:230-233 */
    if ((rc = oc_adjoint_apply(ndim, yext, ax, hext, h, xext, g))) goto done;
    for (size_t i = 0; i < nx; ++i) g[i] = g[i] - aty[i];
    kkt_trace[klen++] = kkt_from_gradient(x, g, nx);
  }
  memcpy(x_out, x, nx * 8);
  *trace_len = tlen;
  *iters_run = iterations;
  *stop_reason = reason;
  if (backtracks_out) *backtracks_out = backtracks;
done:
  free(aty);
  free(x);
  free(g);
  free(trial);
  free(ax);
  free(ax_t);
  free(r);
  return rc;
}

/* solvers.hpp:245-305 (Richardson-Lucy with guarded division, tensor.hpp:112-116) */
int oc_deconv_rl(int ndim, const size_t* yext, const double* y, const size_t* hext,
                 const double* h, const size_t* xext, const oc_rl_config* cfg, double* x_out,
                 double* obj_trace, double* kkt_trace, size_t* trace_len, size_t* iters_run,
                 int* stop_reason, size_t* clamped_out) {
  if (cfg->max_iters == 0 || !(cfg->tol_rel_change >= 0)) return OC_ERROR;
  size_t want[OC_MAXDIM];
  int rc = oc_conv_output_shape(ndim, xext, hext, want);
  if (rc) return rc;
  for (int i = 0; i < ndim; ++i)
    if (want[i] != yext[i]) return OC_SHAPE;
  const size_t K = count_of(ndim, hext);
  for (size_t i = 0; i < K; ++i)
    if (h[i] < 0.0) return OC_NUMERIC;
  double hsum = 0.0;
  for (size_t i = 0; i < K; ++i) hsum += h[i];
  if (!(hsum > 0.0)) return OC_NUMERIC;

  const size_t nx = count_of(ndim, xext), ny = count_of(ndim, yext);
  double *hn = malloc(K * 8), *yc = malloc(ny * 8), *aty = malloc(nx * 8), *x = malloc(nx * 8),
         *xn = malloc(nx * 8), *ax = malloc(ny * 8), *ratio = malloc(ny * 8),
         *g = malloc(nx * 8), *r = malloc(ny * 8);
  if (!hn || !yc || !aty || !x || !xn || !ax || !ratio || !g || !r) {
    rc = OC_ALLOC;
    goto done;
  }
  {
    const double s = 1.0 / hsum;
    for (size_t i = 0; i < K; ++i) hn[i] = h[i] * s;
  }
  size_t clamped = 0;
  for (size_t i = 0; i < ny; ++i) {
    if (y[i] < 0.0) ++clamped;
    yc[i] = y[i] < 0.0 ? 0.0 : y[i];
  }
  if ((rc = oc_adjoint_apply(ndim, yext, yc, hext, hn, xext, aty))) goto done;
  double total = 0.0;
  for (size_t i = 0; i < ny; ++i) total += yc[i];
  size_t tlen = 0, iterations = 0;
  int reason = OC_MAX_ITERS;
  if (!(total > 0.0)) {
    memset(x, 0, nx * 8);
    if ((rc = oc_conv_full(ndim, xext, x, hext, hn, ax))) goto done;
    obj_trace[0] = half_sq_resid(ax, yc, r, ny);
    if ((rc = oc_adjoint_apply(ndim, yext, ax, hext, hn, xext, g))) goto done;
    for (size_t i = 0; i < nx; ++i) g[i] -= aty[i];
    kkt_trace[0] = kkt_from_gradient(x, g, nx);
    memcpy(x_out, x, nx * 8);
    *trace_len = 1;
    *iters_run = 0;
    *stop_reason = OC_CONVERGED;
    *clamped_out = clamped;
    goto done;
  }
  for (size_t i = 0; i < nx; ++i) x[i] = total / (double)nx;
  if ((rc = oc_conv_full(ndim, xext, x, hext, hn, ax))) goto done;
#define RL_RECORD()                                                                  \
  do {                                                                               \
    obj_trace[tlen] = half_sq_resid(ax, yc, r, ny);                                  \
    if ((rc = oc_adjoint_apply(ndim, yext, ax, hext, hn, xext, g))) goto done;       \
    for (size_t i = 0; i < nx; ++i) g[i] -= aty[i];                                  \
    kkt_trace[tlen] = kkt_from_gradient(x, g, nx);                                   \
    ++tlen;                                                                          \
  } while (0)
  RL_RECORD();
  for (size_t k = 1; k <= cfg->max_iters; ++k) {
    for (size_t i = 0; i < ny; ++i) ratio[i] = fabs(ax[i]) < 1e-12 ? 0.0 : yc[i] / ax[i];
    if ((rc = oc_adjoint_apply(ndim, yext, ratio, hext, hn, xext, xn))) goto done;
    double dd = 0.0, xx = 0.0;
    for (size_t i = 0; i < nx; ++i) xn[i] = x[i] * xn[i];
    for (size_t i = 0; i < nx; ++i) {
      const double d = xn[i] - x[i];
      dd += d * d;
    }
    for (size_t i = 0; i < nx; ++i) xx += x[i] * x[i];
    const double nrm = sqrt(xx);
    const double rel = sqrt(dd) / (nrm > 1e-300 ? nrm : 1e-300);
    double* tmp = x;
    x = xn;
    xn = tmp;
    if ((rc = oc_conv_full(ndim, xext, x, hext, hn, ax))) goto done;
    RL_RECORD();
    iterations = k;
    if (rel < cfg->tol_rel_change) {
      reason = OC_CONVERGED;
      break;
    }
  }
#undef RL_RECORD
  memcpy(x_out, x, nx * 8);
  *trace_len = tlen;
  *iters_run = iterations;
  *stop_reason = reason;
  *clamped_out = clamped;
done:
  free(hn);
  free(yc);
  free(aty);
  free(x);
  free(xn);
  free(ax);
  free(ratio);
  free(g);
  free(r);
  return rc;
}

/* Sampled per-voxel forward value, convolution.hpp:55-74 evaluated at one output
 * index (for parity at sizes where the full oracle is infeasible). */
int oc_conv_full_sample(int ndim, const size_t* xext, const double* x, const size_t* hext,
                        const double* h, size_t n_samples, const size_t* flat_out_idx,
                        double* values) {
  size_t yext[OC_MAXDIM];
  int rc = oc_conv_output_shape(ndim, xext, hext, yext);
  if (rc) return rc;
  view_t v;
  v.x = x;
  v.h = h;
  v.xext = xext;
  v.hext = hext;
  v.ndim = ndim;
  strides(ndim, xext, v.xst);
  strides(ndim, hext, v.hst);
  for (long long s = 0; s < (long long)n_samples; ++s) {
    size_t idx[OC_MAXDIM];
    size_t rem = flat_out_idx[s];
    for (int i = ndim - 1; i >= 0; --i) {
      idx[i] = rem % yext[i];
      rem /= yext[i];
    }
    values[s] = element(&v, idx, 0, 0, 0);
  }
  return OC_OK;
}

/* Sampled adjoint value: valid correlation g[k] = sum_j h[j] r[k+j]; equal to
 * adjoint_apply's crop of conv_full(r, flip h) (convolution.hpp:166-174). */
int oc_adjoint_sample(int ndim, const size_t* yext, const double* y, const size_t* hext,
                      const double* h, const size_t* xext, size_t n_samples,
                      const size_t* flat_x_idx, double* values) {
  int rc = check_kernel(ndim, hext);
  if (rc) return rc;
  for (int i = 0; i < ndim; ++i)
    if (yext[i] != xext[i] + hext[i] - 1) return OC_SHAPE;
  const size_t K = count_of(ndim, hext);
  double* hf = (double*)malloc(K * sizeof(double));
  if (!hf) return OC_ALLOC;
  for (size_t i = 0; i < K; ++i) hf[i] = h[K - 1 - i];
  view_t v;
  v.x = y;
  v.h = hf;
  v.xext = yext;
  v.hext = hext;
  v.ndim = ndim;
  strides(ndim, yext, v.xst);
  strides(ndim, hext, v.hst);
  for (long long s = 0; s < (long long)n_samples; ++s) {
    size_t idx[OC_MAXDIM];
    size_t rem = flat_x_idx[s];
    for (int i = ndim - 1; i >= 0; --i) {
      idx[i] = rem % xext[i] + (hext[i] - 1); /* crop offset 2p into the m+4p output */
      rem /= xext[i];
    }
    values[s] = element(&v, idx, 0, 0, 0);
  }
  free(hf);
  return OC_OK;
}
