/*
 * TEST INFRASTRUCTURE ONLY -- multi-threaded float64 CPU oracle for config-scale parity.
 *
 * Only tests/ may load this library (as the checker); the product never links it.
 *
 * The same algorithm as oracle/ndconv_oracle.c (the bitwise restatement of the
 * reference), with the two convolutions evaluated in a different -- vectorised and
 * threaded -- summation order, so that full-size BASELINE configs (config 2's 2048^2
 * images, config 3's 128x256x256 volume, config 4/5 replicas at full PSF depth) run in
 * seconds instead of hours.  Reordering a float64 sum of K terms moves it by
 * ~K * 2^-53 relative, ~1e-12 at config 5's 70,785 taps: seven orders of magnitude
 * inside the 1e-5 / 1e-4 parity bars.  tests/test_oracle.py pins this library against
 * ndconv_oracle.c (itself bitwise equal to the compiled reference, oracle/_ref) to
 * 1e-12 on operators, step estimates and whole PG runs.
 *
 * Reference map (paths under /root/reference/proj/include/ndconv/):
 *   conv_full          convolution.hpp:81-123 (per-element sum convolution.hpp:55-74)
 *   adjoint_apply      convolution.hpp:166-174 = the valid correlation
 *                      g[k] = sum_j h[j] r[k+j] (flip + (m+4p) conv_full + crop_m
 *                      computes exactly these sums)
 *   estimate_step      solvers.hpp:127-143
 *   kkt_from_gradient  solvers.hpp:98-103
 *   deconv_pg          solvers.hpp:155-238 (control flow as in ndconv_oracle.c)
 *
 * Tensors have 1 to 3 dimensions (row-major, first index slowest, shape.hpp:55-64).
 * Both operators reduce to one row primitive, acc[o] += sum_j t[j] src[o + j]
 * (correlation form): the forward pass reads a zero-padded copy of x with reversed
 * tap rows, the adjoint reads r directly.  Threads split the output rows in blocks of
 * kRows rows of one plane.
 */
#include <math.h>
#include <pthread.h>
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { OF_OK = 0, OF_ERROR = 1, OF_SHAPE = 2, OF_NUMERIC = 3, OF_ALLOC = 9 };
enum { OF_CONVERGED = 0, OF_MAX_ITERS = 1, OF_STALLED = 2 };

typedef struct {
  size_t max_iters;
  double tol_rel_objective;
  int has_initial_step;
  double initial_step;
  double backtrack_factor;
  size_t max_backtracks;
  size_t power_iters;
} of_pg_config; /* same layout as oc_pg_config / ndc_deconv_config */

static int g_threads = 1;
void of_set_threads(int n) { g_threads = n < 1 ? 1 : (n > 256 ? 256 : n); }

/* ---- row primitive ---------------------------------------------------------------- */

/* acc[o] += sum_{j<k} t[j] * src[o + j] for o in [0, n).  Blocks of 64 / 32 / 8 outputs
 * live in registers across the tap loop (one load per FMA). */
__attribute__((target_clones("avx512f", "avx2", "default")))
static void row_corr(double* restrict acc, const double* restrict src, const double* restrict t, long n,
                     long k) {
  long o = 0;
  for (; o + 64 <= n; o += 64) { /* 8 independent AVX-512 FMA chains: latency hidden */
    double a[64];
    for (int i = 0; i < 64; ++i) a[i] = acc[o + i];
    for (long j = 0; j < k; ++j) {
      const double tv = t[j];
      const double* s = src + o + j;
      for (int i = 0; i < 64; ++i) a[i] += tv * s[i];
    }
    for (int i = 0; i < 64; ++i) acc[o + i] = a[i];
  }
  for (; o + 32 <= n; o += 32) {
    double a[32];
    for (int i = 0; i < 32; ++i) a[i] = acc[o + i];
    for (long j = 0; j < k; ++j) {
      const double tv = t[j];
      const double* s = src + o + j;
      for (int i = 0; i < 32; ++i) a[i] += tv * s[i];
    }
    for (int i = 0; i < 32; ++i) acc[o + i] = a[i];
  }
  for (; o + 8 <= n; o += 8) {
    double a[8];
    for (int i = 0; i < 8; ++i) a[i] = acc[o + i];
    for (long j = 0; j < k; ++j) {
      const double tv = t[j];
      const double* s = src + o + j;
      for (int i = 0; i < 8; ++i) a[i] += tv * s[i];
    }
    for (int i = 0; i < 8; ++i) acc[o + i] = a[i];
  }
  for (; o < n; ++o) {
    double a = acc[o];
    for (long j = 0; j < k; ++j) a += t[j] * src[o + j];
    acc[o] = a;
  }
}

/* ---- thread fan-out ------------------------------------------------------------------ */

typedef void (*row_fn)(void* ctx, long row);
typedef struct {
  row_fn fn;
  void* ctx;
  long rows;
  long next; /* atomic work counter */
} pool_job;

static void* pool_worker(void* arg) {
  pool_job* j = (pool_job*)arg;
  for (;;) {
    const long r = __atomic_fetch_add(&j->next, 1, __ATOMIC_RELAXED);
    if (r >= j->rows) break;
    j->fn(j->ctx, r);
  }
  return NULL;
}

static void parallel_rows(long rows, row_fn fn, void* ctx) {
  pool_job job = {fn, ctx, rows, 0};
  int nt = g_threads;
  if (nt > rows) nt = (int)(rows < 1 ? 1 : rows);
  pthread_t th[256];
  int started = 0;
  for (int i = 1; i < nt; ++i)
    if (pthread_create(&th[started], NULL, pool_worker, &job) == 0) ++started;
  pool_worker(&job);
  for (int i = 0; i < started; ++i) pthread_join(th[i], NULL);
}

/* ---- shapes ----------------------------------------------------------------------- */

typedef struct {
  long mz, my, mx; /* x extents (leading 1s) */
  long kz, ky, kx; /* kernel extents */
  long oz, oy, ox; /* y extents = m + k - 1 */
} geo3;

static int make_geo(int ndim, const size_t* xext, const size_t* hext, geo3* g) {
  if (ndim < 1 || ndim > 3) return OF_SHAPE;
  long m[3] = {1, 1, 1}, k[3] = {1, 1, 1};
  for (int i = 0; i < ndim; ++i) {
    if (xext[i] == 0 || hext[i] == 0 || hext[i] % 2 == 0) return OF_SHAPE; /* kernel.hpp:18-22 */
    m[3 - ndim + i] = (long)xext[i];
    k[3 - ndim + i] = (long)hext[i];
  }
  g->mz = m[0], g->my = m[1], g->mx = m[2];
  g->kz = k[0], g->ky = k[1], g->kx = k[2];
  g->oz = m[0] + k[0] - 1, g->oy = m[1] + k[1] - 1, g->ox = m[2] + k[2] - 1;
  return OF_OK;
}

static size_t nx_of(const geo3* g) { return (size_t)g->mz * g->my * g->mx; }
static size_t ny_of(const geo3* g) { return (size_t)g->oz * g->oy * g->ox; }

/* ---- forward: y[o] = sum_j h[j] x[o - j] (convolution.hpp:81-123) -------------------- */

typedef struct {
  const geo3* g;
  const double* xp;   /* x rows zero-padded by kx-1 on both sides, row pitch px */
  long px;
  const double* hrev; /* h with every x-row reversed */
  double* y;
} fwd_ctx;

/* Work unit: kRows consecutive output rows of one plane, so every source row read for
 * them is reused from L1 by each of the kRows accumulators it contributes to. */
enum { kRows = 4 };

static void fwd_rows(void* c, long unit) {
  const fwd_ctx* f = (const fwd_ctx*)c;
  const geo3* g = f->g;
  const long per_plane = (g->oy + kRows - 1) / kRows;
  const long oz = unit / per_plane, oy0 = (unit % per_plane) * kRows;
  const long nr = g->oy - oy0 < kRows ? g->oy - oy0 : kRows;
  double* acc0 = f->y + ((size_t)oz * g->oy + oy0) * g->ox;
  memset(acc0, 0, (size_t)nr * g->ox * sizeof(double));
  const long jz0 = oz - g->mz + 1 > 0 ? oz - g->mz + 1 : 0, jz1 = oz < g->kz - 1 ? oz : g->kz - 1;
  for (long jz = jz0; jz <= jz1; ++jz) {
    const long iz = oz - jz;
    /* source row iy feeds output row oy = iy + jy for every valid tap row jy */
    const long iy0 = oy0 - (g->ky - 1) > 0 ? oy0 - (g->ky - 1) : 0;
    const long iy1 = oy0 + nr - 1 < g->my - 1 ? oy0 + nr - 1 : g->my - 1;
    for (long iy = iy0; iy <= iy1; ++iy) {
      const double* src = f->xp + ((size_t)iz * g->my + iy) * f->px;
      for (long r = 0; r < nr; ++r) {
        const long jy = oy0 + r - iy;
        if (jy < 0 || jy >= g->ky) continue;
        row_corr(acc0 + (size_t)r * g->ox, src, f->hrev + ((size_t)jz * g->ky + jy) * g->kx, g->ox, g->kx);
      }
    }
  }
}

int of_conv_full(int ndim, const size_t* xext, const double* x, const size_t* hext, const double* h,
                 double* y) {
  geo3 g;
  int rc = make_geo(ndim, xext, hext, &g);
  if (rc) return rc;
  const long px = g.mx + 2 * (g.kx - 1);
  const size_t nrows = (size_t)g.mz * g.my;
  double* xp = (double*)calloc(nrows * (size_t)px, sizeof(double));
  double* hrev = (double*)malloc((size_t)g.kz * g.ky * g.kx * sizeof(double));
  if (!xp || !hrev) {
    free(xp);
    free(hrev);
    return OF_ALLOC;
  }
  for (size_t r = 0; r < nrows; ++r) memcpy(xp + r * px + (g.kx - 1), x + r * g.mx, (size_t)g.mx * sizeof(double));
  for (long r = 0; r < g.kz * g.ky; ++r)
    for (long j = 0; j < g.kx; ++j) hrev[r * g.kx + j] = h[r * g.kx + (g.kx - 1 - j)];
  fwd_ctx c = {&g, xp, px, hrev, y};
  parallel_rows(g.oz * ((g.oy + kRows - 1) / kRows), fwd_rows, &c);
  free(xp);
  free(hrev);
  return OF_OK;
}

/* ---- adjoint: g[k] = sum_j h[j] r[k + j] (convolution.hpp:166-174) -------------------- */

typedef struct {
  const geo3* g;
  const double* r;
  const double* h;
  double* out;
} adj_ctx;

static void adj_rows(void* c, long unit) {
  const adj_ctx* a = (const adj_ctx*)c;
  const geo3* g = a->g;
  const long per_plane = (g->my + kRows - 1) / kRows;
  const long z = unit / per_plane, y0 = (unit % per_plane) * kRows;
  const long nr = g->my - y0 < kRows ? g->my - y0 : kRows;
  double* acc0 = a->out + ((size_t)z * g->my + y0) * g->mx;
  memset(acc0, 0, (size_t)nr * g->mx * sizeof(double));
  for (long jz = 0; jz < g->kz; ++jz)
    /* source row sy feeds output row y = sy - jy */
    for (long sy = y0; sy < y0 + nr + g->ky - 1; ++sy) {
      const double* src = a->r + ((size_t)(z + jz) * g->oy + sy) * g->ox;
      for (long r = 0; r < nr; ++r) {
        const long jy = sy - (y0 + r);
        if (jy < 0 || jy >= g->ky) continue;
        row_corr(acc0 + (size_t)r * g->mx, src, a->h + ((size_t)jz * g->ky + jy) * g->kx, g->mx, g->kx);
      }
    }
}

int of_adjoint_apply(int ndim, const size_t* yext, const double* r, const size_t* hext, const double* h,
                     const size_t* xext, double* out) {
  geo3 g;
  int rc = make_geo(ndim, xext, hext, &g);
  if (rc) return rc;
  for (int i = 0; i < ndim; ++i)
    if (yext[i] != xext[i] + hext[i] - 1) return OF_SHAPE; /* convolution.hpp:169-172 */
  adj_ctx c = {&g, r, h, out};
  parallel_rows(g.mz * ((g.my + kRows - 1) / kRows), adj_rows, &c);
  return OF_OK;
}

/* ---- solvers (solvers.hpp) ----------------------------------------------------------- */

static double dot(const double* a, const double* b, size_t n) {
  double acc = 0.0;
  for (size_t i = 0; i < n; ++i) acc += a[i] * b[i];
  return acc;
}

static int all_zero(const double* h, size_t n) {
  for (size_t i = 0; i < n; ++i)
    if (h[i] != 0.0) return 0;
  return 1;
}

/* solvers.hpp:127-143 */
int of_estimate_step(int ndim, const size_t* hext, const double* h, const size_t* xext, size_t power_iters,
                     double* step) {
  if (power_iters == 0) return OF_ERROR;
  geo3 g;
  int rc = make_geo(ndim, xext, hext, &g);
  if (rc) return rc;
  if (all_zero(h, (size_t)g.kz * g.ky * g.kx)) return OF_NUMERIC;
  size_t yext[3];
  for (int i = 0; i < ndim; ++i) yext[i] = xext[i] + hext[i] - 1;
  const size_t nx = nx_of(&g), ny = ny_of(&g);
  double *v = malloc(nx * 8), *w = malloc(nx * 8), *u = malloc(ny * 8);
  if (!v || !w || !u) {
    rc = OF_ALLOC;
    goto done;
  }
  for (size_t i = 0; i < nx; ++i) v[i] = 1.0;
  {
    const double s = 1.0 / sqrt(dot(v, v, nx));
    for (size_t i = 0; i < nx; ++i) v[i] *= s;
  }
  double lambda = 0.0;
  for (size_t it = 0; it < power_iters; ++it) {
    if ((rc = of_conv_full(ndim, xext, v, hext, h, u))) goto done;
    if ((rc = of_adjoint_apply(ndim, yext, u, hext, h, xext, w))) goto done;
    lambda = sqrt(dot(w, w, nx));
    if (!(lambda > 0.0) || !isfinite(lambda)) {
      rc = OF_NUMERIC;
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

static double kkt_from_gradient(const double* x, const double* g, size_t n) { /* solvers.hpp:98-103 */
  double worst = 0.0;
  for (size_t i = 0; i < n; ++i) {
    const double m = fabs(x[i] < g[i] ? x[i] : g[i]);
    if (m > worst) worst = m;
  }
  return worst;
}

static double half_sq_resid(const double* ax, const double* y, size_t n) {
  double acc = 0.0;
  for (size_t i = 0; i < n; ++i) {
    const double r = ax[i] - y[i];
    acc += r * r;
  }
  return 0.5 * acc;
}

/* solvers.hpp:155-238, the control flow of ndconv_oracle.c's oc_deconv_pg. */
int of_deconv_pg(int ndim, const size_t* yext, const double* y, const size_t* hext, const double* h,
                 const size_t* xext, const of_pg_config* cfg, double* x_out, double* obj_trace,
                 double* kkt_trace, size_t* trace_len, size_t* iters_run, int* stop_reason,
                 size_t* backtracks_out, double* step_out) {
  /* solvers.hpp:65-76 */
  if (cfg->max_iters == 0 || !(cfg->tol_rel_objective >= 0) ||
      (cfg->has_initial_step && !(cfg->initial_step > 0)) || !(cfg->backtrack_factor > 0) ||
      !(cfg->backtrack_factor < 1) || cfg->max_backtracks == 0 || cfg->power_iters == 0)
    return OF_ERROR;
  geo3 g;
  int rc = make_geo(ndim, xext, hext, &g);
  if (rc) return rc;
  for (int i = 0; i < ndim; ++i)
    if (yext[i] != xext[i] + hext[i] - 1) return OF_SHAPE; /* solvers.hpp:83-90 */
  if (all_zero(h, (size_t)g.kz * g.ky * g.kx)) return OF_NUMERIC;
  double step0 = 0.0;
  if (cfg->has_initial_step)
    step0 = cfg->initial_step;
  else if ((rc = of_estimate_step(ndim, hext, h, xext, cfg->power_iters, &step0)))
    return rc;
  if (step_out) *step_out = step0;

  const size_t nx = nx_of(&g), ny = ny_of(&g);
  double *aty = malloc(nx * 8), *x = malloc(nx * 8), *gr = malloc(nx * 8), *trial = malloc(nx * 8),
         *ax = malloc(ny * 8), *ax_t = malloc(ny * 8);
  if (!aty || !x || !gr || !trial || !ax || !ax_t) {
    rc = OF_ALLOC;
    goto done;
  }
  if ((rc = of_adjoint_apply(ndim, yext, y, hext, h, xext, aty))) goto done; /* :166 */
  for (size_t i = 0; i < nx; ++i) x[i] = aty[i] < 0.0 ? 0.0 : aty[i];      /* :167 */
  if ((rc = of_conv_full(ndim, xext, x, hext, h, ax))) goto done;            /* :168 */
  double f = half_sq_resid(ax, y, ny);                                       /* :169-172 */

  size_t tlen = 0, klen = 0, iterations = 0, backtracks = 0;
  int reason = OF_MAX_ITERS;
  obj_trace[tlen++] = f;
  for (size_t k = 1; k <= cfg->max_iters; ++k) {
    if ((rc = of_adjoint_apply(ndim, yext, ax, hext, h, xext, gr))) goto done; /* :180 */
    for (size_t i = 0; i < nx; ++i) gr[i] = gr[i] - aty[i];
    kkt_trace[klen++] = kkt_from_gradient(x, gr, nx); /* :181 */
    double step = step0;
    int accepted = 0, fixed_point = 0;
    double f_next = f;
    for (size_t b = 0; b <= cfg->max_backtracks; ++b) { /* :189 */
      int same = 1;
      for (size_t i = 0; i < nx; ++i) {
        const double t = x[i] - gr[i] * step; /* :190 */
        trial[i] = t < 0.0 ? 0.0 : t;
        if (trial[i] != x[i]) same = 0;
      }
      if (same) { /* :191-194 */
        fixed_point = 1;
        break;
      }
      if ((rc = of_conv_full(ndim, xext, trial, hext, h, ax_t))) goto done; /* :195 */
      const double f_trial = half_sq_resid(ax_t, y, ny);                   /* :196-197 */
      if (f_trial < f) {                                                   /* :198 */
        f_next = f_trial;
        accepted = 1;
        break;
      }
      ++backtracks;
      step *= cfg->backtrack_factor; /* :205 */
    }
    if (fixed_point) {
      reason = OF_CONVERGED;
      break;
    }
    if (!accepted) {
      reason = OF_STALLED;
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
    if (drop <= cfg->tol_rel_objective * obj_trace[tlen - 2]) { /* :224-227 */
      reason = OF_CONVERGED;
      break;
    }
  }
  if (klen < tlen) { /* :230-233 */
    if ((rc = of_adjoint_apply(ndim, yext, ax, hext, h, xext, gr))) goto done;
    for (size_t i = 0; i < nx; ++i) gr[i] = gr[i] - aty[i];
    kkt_trace[klen++] = kkt_from_gradient(x, gr, nx);
  }
  memcpy(x_out, x, nx * 8);
  *trace_len = tlen;
  *iters_run = iterations;
  *stop_reason = reason;
  if (backtracks_out) *backtracks_out = backtracks;
done:
  free(aty);
  free(x);
  free(gr);
  free(trial);
  free(ax);
  free(ax_t);
  return rc;
}
