"""TEST INFRASTRUCTURE ONLY -- deconv_pg (solvers.hpp:155-238) restated in float32.

The same control flow as the reference (and oracle/ndconv_oracle.c), with the gradient
in the device's form A^T(A x - y), and every tensor and every convolution in numpy float32 (scipy.signal direct convolution / correlation, float32
accumulators; the objective reduced in float64 as the device does).  It measures how far
float32 arithmetic ITSELF can follow the float64 reference on a given problem: on small
problems whose last iterations move x by less than float32 can resolve (the residual
falls below the rounding of the data, the bitwise fixed-point test trial == x fires
early), the float32 estimate settles up to ~1e-4 from the f64 one whatever the
implementation.  tests/test_gpu_pg.py holds the device to max(1e-4, 2 x this deviation).
Only tests/ use it; the product never does.
"""
from __future__ import annotations

import numpy as np
from scipy.signal import convolve, correlate


def deconv_pg_f32(y, h, x_shape, step: float, max_iters: int, tol_rel_objective: float = 0.0,
                  backtrack_factor: float = 0.5, max_backtracks: int = 50):
    f32 = np.float32
    y = np.asarray(y, f32)
    h = np.asarray(h, f32)

    def A(x):  # conv_full (convolution.hpp:81-123)
        return convolve(x, h, mode="full", method="direct").astype(f32)

    def At(r):  # adjoint_apply = valid correlation (convolution.hpp:166-174)
        return correlate(r, h, mode="valid", method="direct").astype(f32)

    def obj(r):
        return 0.5 * float(np.sum(r.astype(np.float64) ** 2))

    aty = At(y)
    x = np.maximum(aty, 0).astype(f32)                      # :166-167
    ax = A(x)
    fval = obj(ax - y)                                      # :168-172
    trace = [fval]
    reason, iters = "max_iters", 0
    for k in range(1, max_iters + 1):
        # :180 computes A^T(A x) - A^T y; equal in exact arithmetic to A^T(A x - y), the
        # form the device uses, which loses less to cancellation in float32 (golden case 6:
        # 1.3e-4 from the f64 estimate against 2.2e-4 with the reference's form)
        g = At((ax - y).astype(f32))
        st = step
        accepted = fixed = False
        for _ in range(max_backtracks + 1):                 # :189
            trial = np.maximum(x - f32(st) * g, 0).astype(f32)   # :190
            if np.array_equal(trial, x):                    # :191
                fixed = True
                break
            ax_t = A(trial)
            ft = obj(ax_t - y)
            if ft < fval:                                   # :198
                accepted = True
                break
            st *= backtrack_factor
        if fixed:
            reason = "converged"
            break
        if not accepted:
            reason = "stalled"
            break
        drop = fval - ft
        x, ax, fval = trial, ax_t, ft
        trace.append(fval)
        iters = k
        if drop <= tol_rel_objective * trace[-2]:
            reason = "converged"
            break
    return x.astype(np.float64), np.asarray(trace), iters, reason
