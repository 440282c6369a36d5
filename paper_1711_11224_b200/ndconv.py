"""Python mirror of the reference's ndconv API over the B200 C-ABI.

Same function names, argument meaning and error classes as the header-only C++ API in
/root/reference/proj/include/ndconv/ (cited per function), with numpy float64 arrays in
place of ndconv::Tensor (row-major, first index slowest -- shape.hpp:55-64) and a numpy
array with odd extents in place of ndconv::Kernel (kernel.hpp:15-37).  Every call goes
through libndconv_b200.so; nothing here computes on the CPU.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _native as N

# --- error classes (error.hpp:8-30) ------------------------------------------------------


class Error(RuntimeError):
    """ndconv::Error"""


class ShapeError(Error):
    """ndconv::ShapeError"""


class BoundsError(Error):
    """ndconv::BoundsError"""


class FormatError(Error):
    """ndconv::FormatError"""


class NumericError(Error):
    """ndconv::NumericError"""


class UnsupportedError(Error):
    """Operand outside the device path's limits (NDC_ERR_UNSUPPORTED)."""


class DeviceError(Error):
    """CUDA / NCCL failure or no usable B200 (NDC_ERR_CUDA / _NCCL / _NO_DEVICE)."""


_RC = {1: Error, 2: ShapeError, 3: NumericError, 4: BoundsError, 5: UnsupportedError,
       6: DeviceError, 7: DeviceError, 8: DeviceError, 9: ValueError, 10: FormatError}


def _check(rc: int):
    if rc != 0:
        msg = N.lib().ndc_last_error().decode(errors="replace")
        raise _RC.get(rc, Error)(msg)


def _ext(shape):
    return (C.c_size_t * len(shape))(*[int(s) for s in shape])


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _p(a: np.ndarray):
    return a.ctypes.data_as(N.dbl_p)


def _pf(a: np.ndarray):
    return a.ctypes.data_as(N.flt_p)


def _kernel(h) -> np.ndarray:
    h = _f64(h)
    if h.ndim < 1:
        raise ShapeError("Shape: need at least one dimension")
    return h


# --- configuration / report (solvers.hpp:20-61) ------------------------------------------


@dataclass
class DeconvConfig:
    """ndconv::DeconvConfig (solvers.hpp:20-28)."""
    max_iters: int = 500
    tol_rel_objective: float = 1e-6
    initial_step: float | None = None
    backtrack_factor: float = 0.5
    max_backtracks: int = 50
    power_iters: int = 30

    def to_c(self) -> N.DeconvConfig:
        return N.DeconvConfig(int(self.max_iters), float(self.tol_rel_objective),
                              0 if self.initial_step is None else 1,
                              0.0 if self.initial_step is None else float(self.initial_step),
                              float(self.backtrack_factor), int(self.max_backtracks),
                              int(self.power_iters))


@dataclass
class RlConfig:
    """ndconv::RlConfig (solvers.hpp:30-35)."""
    max_iters: int = 500
    tol_rel_change: float = 0.0


STOP_REASONS = {0: "converged", 1: "max_iters", 2: "stalled"}


@dataclass
class DeconvReport:
    """ndconv::DeconvReport (solvers.hpp:48-61); stop_reason is to_string(StopReason)."""
    estimate: np.ndarray
    objective_trace: np.ndarray
    kkt_trace: np.ndarray
    iterations_run: int
    stop_reason: str
    wall_time_seconds: float
    negative_pixels_clamped: int = 0
    extra: dict = field(default_factory=dict)


def _report(est, rep: N.Report, obj, kkt) -> DeconvReport:
    n = rep.trace_len
    return DeconvReport(est, obj[:n].copy(), kkt[:n].copy(), rep.iterations_run,
                        STOP_REASONS.get(rep.stop_reason, "unknown"), rep.wall_time_seconds,
                        rep.negative_pixels_clamped,
                        {"backtracks": rep.backtracks, "step0": rep.step0})


# --- operators (convolution.hpp) ---------------------------------------------------------


def set_max_threads(n: int) -> None:
    """convolution.hpp:26 (recorded only: the device grid is the parallelism)."""
    N.lib().ndc_set_max_threads(int(n))


def max_threads() -> int:
    return int(N.lib().ndc_max_threads())


def device_count() -> int:
    n = C.c_int()
    _check(N.lib().ndc_device_count(C.byref(n)))
    return n.value


def conv_output_shape(x_shape, h) -> tuple:
    """convolution.hpp:30-38: extents d + 2p."""
    h = _kernel(h)
    if len(x_shape) != h.ndim:
        raise ShapeError(f"conv_full: {len(x_shape)}-d input vs {h.ndim}-d kernel")
    out = (C.c_size_t * h.ndim)()
    _check(N.lib().ndc_conv_output_shape(h.ndim, _ext(x_shape), _ext(h.shape), out))
    return tuple(int(v) for v in out)


def conv_full(x, h) -> np.ndarray:
    """convolution.hpp:81-123: full n-d convolution with zero padding."""
    x, h = _f64(x), _kernel(h)
    out_shape = conv_output_shape(x.shape, h)
    y = np.empty(out_shape, np.float64)
    _check(N.lib().ndc_conv_full_f64(x.ndim, _ext(x.shape), _p(x), _ext(h.shape), _p(h), _p(y)))
    return y


def conv_full_batch(x, h) -> np.ndarray:
    """y[b] = conv_full(x[b], h) for a float32 batch x[b, ...] (ndc_conv_full_batch_f32)."""
    h = _kernel(h)
    x = np.ascontiguousarray(x, np.float32)
    if x.ndim != h.ndim + 1:
        raise ShapeError("conv_full: dimension count mismatch")
    ys = conv_output_shape(x.shape[1:], h)
    y = np.empty((x.shape[0],) + ys, np.float32)
    _check(N.lib().ndc_conv_full_batch_f32(x.shape[0], h.ndim, _ext(x.shape[1:]), _pf(x), _ext(h.shape), _p(h),
                                           _pf(y)))
    return y


def adjoint_apply_batch(y, h, x_shape) -> np.ndarray:
    """x[b] = adjoint_apply(y[b], h, x_shape) for a float32 batch (ndc_adjoint_apply_batch_f32)."""
    h = _kernel(h)
    y = np.ascontiguousarray(y, np.float32)
    if y.ndim != h.ndim + 1 or len(x_shape) != h.ndim:
        raise ShapeError("adjoint_apply: dimension count mismatch")
    x = np.empty((y.shape[0],) + tuple(int(v) for v in x_shape), np.float32)
    _check(N.lib().ndc_adjoint_apply_batch_f32(y.shape[0], h.ndim, _ext(y.shape[1:]), _pf(y), _ext(h.shape), _p(h),
                                               _ext(x_shape), _pf(x)))
    return x


def flip(h) -> np.ndarray:
    """kernel.hpp:41-45: reversal along every axis (the reversed flat buffer)."""
    h = _kernel(h)
    return h.reshape(-1)[::-1].reshape(h.shape).copy()


def adjoint_apply(y, h, x_shape) -> np.ndarray:
    """convolution.hpp:166-174: A^T y, computed on the device as a valid correlation."""
    y, h = _f64(y), _kernel(h)
    if y.ndim != h.ndim or len(x_shape) != h.ndim:
        raise ShapeError("adjoint_apply: dimension count mismatch")
    for i in range(h.ndim):
        if y.shape[i] != x_shape[i] + h.shape[i] - 1:
            raise ShapeError(f"adjoint_apply: observation shape {y.shape} is not {tuple(x_shape)} + 2p")
    out = np.empty(tuple(int(s) for s in x_shape), np.float64)
    _check(N.lib().ndc_adjoint_apply_f64(y.ndim, _ext(y.shape), _p(y), _ext(h.shape), _p(h),
                                         _ext(x_shape), _p(out)))
    return out


def _check_obs(x_shape, y, h, what):
    expected = conv_output_shape(x_shape, h)
    if tuple(y.shape) != expected:
        raise ShapeError(f"{what}: observation shape {y.shape} does not match forward model "
                         f"output {expected}")


def normal_gradient(x, y, h) -> np.ndarray:
    """convolution.hpp:178-185: A^T A x - A^T y."""
    x, y, h = _f64(x), _f64(y), _kernel(h)
    _check_obs(x.shape, y, h, "normal_gradient")
    g = np.empty(x.shape, np.float64)
    _check(N.lib().ndc_normal_gradient_f64(x.ndim, _ext(x.shape), _p(x), _p(y), _ext(h.shape), _p(h),
                                           _p(g)))
    return g


# --- solvers (solvers.hpp) ---------------------------------------------------------------


def objective(x, y, h) -> float:
    """solvers.hpp:119-122: 0.5 ||x (*) h - y||^2."""
    x, y, h = _f64(x), _f64(y), _kernel(h)
    _check_obs(x.shape, y, h, "objective")
    f = C.c_double()
    _check(N.lib().ndc_objective_f64(x.ndim, _ext(x.shape), _p(x), _p(y), _ext(h.shape), _p(h),
                                     C.byref(f)))
    return f.value


def estimate_step(h, x_shape, power_iters: int = 30) -> float:
    """solvers.hpp:127-143: 1 / lambda_max(A^T A) by power iteration from all-ones."""
    h = _kernel(h)
    if len(x_shape) != h.ndim:
        raise ShapeError("estimate_step: dimension count mismatch")
    s = C.c_double()
    _check(N.lib().ndc_estimate_step_f64(h.ndim, _ext(h.shape), _p(h), _ext(x_shape), int(power_iters),
                                         C.byref(s)))
    return s.value


def kkt_residual(x, y, h) -> float:
    """solvers.hpp:147-149: max_i |min(x_i, g_i)|."""
    x, y, h = _f64(x), _f64(y), _kernel(h)
    _check_obs(x.shape, y, h, "kkt_residual")
    k = C.c_double()
    _check(N.lib().ndc_kkt_residual_f64(x.ndim, _ext(x.shape), _p(x), _p(y), _ext(h.shape), _p(h),
                                        C.byref(k)))
    return k.value


def deconv_pg(y, h, x_shape, cfg: DeconvConfig | None = None) -> DeconvReport:
    """solvers.hpp:155-238: projected-gradient deconvolution."""
    return deconv_pg_batch(_f64(y)[None], h, x_shape, cfg)[0]


def deconv_pg_batch(y, h, x_shape, cfg: DeconvConfig | None = None, dtype=np.float64):
    """deconv_pg over a batch y[b, ...] of independent observations with per-image
    scalars (BASELINE config 2).  Returns one DeconvReport per image."""
    cfg = cfg or DeconvConfig()
    h = _kernel(h)
    y = np.ascontiguousarray(y, dtype=dtype)
    if y.ndim != h.ndim + 1:
        raise ShapeError("deconv_pg: dimension count mismatch")
    if len(x_shape) != h.ndim:
        raise ShapeError("deconv_pg: dimension count mismatch")
    B = y.shape[0]
    _check_obs(x_shape, y[0], h, "deconv_pg")
    cap = int(cfg.max_iters) + 1
    x = np.empty((B,) + tuple(int(s) for s in x_shape), dtype)
    obj = np.empty((B, cap), np.float64)
    kkt = np.empty((B, cap), np.float64)
    reps = (N.Report * B)()
    c = cfg.to_c()
    fn = N.lib().ndc_deconv_pg_batch_f64 if dtype == np.float64 else N.lib().ndc_deconv_pg_batch_f32
    ptr = _p if dtype == np.float64 else _pf
    _check(fn(B, h.ndim, _ext(y.shape[1:]), ptr(y), _ext(h.shape), _p(h), _ext(x_shape), C.byref(c),
              ptr(x), _p(obj), _p(kkt), cap, reps))
    return [_report(x[b], reps[b], obj[b], kkt[b]) for b in range(B)]


def deconv_rl(y, h, x_shape, cfg: RlConfig | None = None) -> DeconvReport:
    """solvers.hpp:245-305: Richardson-Lucy on the same operators."""
    cfg = cfg or RlConfig()
    y, h = _f64(y), _kernel(h)
    _check_obs(x_shape, y, h, "deconv_rl")
    cap = int(cfg.max_iters) + 1
    x = np.empty(tuple(int(s) for s in x_shape), np.float64)
    obj = np.empty(cap, np.float64)
    kkt = np.empty(cap, np.float64)
    rep = N.Report()
    c = N.RlConfig(int(cfg.max_iters), float(cfg.tol_rel_change))
    _check(N.lib().ndc_deconv_rl_f64(y.ndim, _ext(y.shape), _p(y), _ext(h.shape), _p(h), _ext(x_shape),
                                     C.byref(c), _p(x), _p(obj), _p(kkt), cap, C.byref(rep)))
    return _report(x, rep, obj, kkt)


# --- tensor files (imageio.hpp) -------------------------------------------------------------


def _path(p) -> bytes:
    return str(p).encode()


def read_tensor(path) -> np.ndarray:
    """imageio.hpp:84-125 NDTENSOR reader (strict header / payload validation)."""
    nd_ = C.c_int()
    ext = (C.c_size_t * 16)()
    _check(N.lib().ndc_ndtensor_info(_path(path), C.byref(nd_), ext))
    shape = tuple(int(ext[i]) for i in range(nd_.value))
    out = np.empty(shape, np.float64)
    _check(N.lib().ndc_ndtensor_read_f64(_path(path), _p(out), out.size))
    return out


def write_tensor(t, path) -> None:
    """imageio.hpp:63-81 NDTENSOR writer (refuses non-finite values)."""
    t = _f64(t)
    _check(N.lib().ndc_ndtensor_write_f64(_path(path), t.ndim, _ext(t.shape), _p(t)))


def read_pgm(path) -> np.ndarray:
    """imageio.hpp:186-238: P5/P2 samples as doubles, shape (height, width)."""
    h, w = C.c_size_t(), C.c_size_t()
    _check(N.lib().ndc_pgm_info(_path(path), C.byref(h), C.byref(w)))
    out = np.empty((h.value, w.value), np.float64)
    _check(N.lib().ndc_pgm_read_f64(_path(path), _p(out), out.size))
    return out


def write_pgm(t, path, clamp: bool = True) -> None:
    """imageio.hpp:240-265: 8-bit P5, round half to even, optional clamp."""
    t = _f64(t)
    if t.ndim != 2:
        raise ShapeError(f"write_pgm: need a 2-d tensor, got {t.shape}")
    _check(N.lib().ndc_pgm_write_f64(_path(path), t.shape[0], t.shape[1], _p(t), 1 if clamp else 0))


# --- simulation generators (simulation.hpp:36-208; image-sized work on the device) ----------


def phantom_lines(rows: int, cols: int, n_lines: int, intensity: float) -> np.ndarray:
    """simulation.hpp:36-70, bit-identical to the reference."""
    out = np.empty((int(rows), int(cols)), np.float64)
    _check(N.lib().ndc_sim_phantom_lines_f64(int(rows), int(cols), int(n_lines), float(intensity), _p(out)))
    return out


def phantom_texture(rows: int, cols: int) -> np.ndarray:
    """simulation.hpp:72-94, bit-identical to the reference."""
    out = np.empty((int(rows), int(cols)), np.float64)
    _check(N.lib().ndc_sim_phantom_texture_f64(int(rows), int(cols), _p(out)))
    return out


def gaussian_psf(extents, sigma: float) -> np.ndarray:
    """simulation.hpp:98-122: sampled isotropic Gaussian, unit sum."""
    ext = tuple(int(e) for e in extents)
    out = np.empty(ext, np.float64)
    _check(N.lib().ndc_sim_gaussian_psf_f64(len(ext), _ext(ext), float(sigma), _p(out)))
    return out


def delta_psf(extents) -> np.ndarray:
    """simulation.hpp:124-131: centred unit impulse."""
    ext = tuple(int(e) for e in extents)
    out = np.empty(ext, np.float64)
    _check(N.lib().ndc_sim_delta_psf_f64(len(ext), _ext(ext), _p(out)))
    return out


def add_gaussian_noise(t, mean: float = 0.0, std_dev: float = 0.0, seed: int = 0) -> np.ndarray:
    """simulation.hpp:184-191: t + mean + std_dev * N(0,1) from mt19937_64(seed) + Box-Muller,
    drawn in flat storage order on the device."""
    t = _f64(t)
    out = np.empty_like(t)
    _check(N.lib().ndc_sim_add_gaussian_noise_f64(t.size, _p(t), float(mean), float(std_dev),
                                                  C.c_uint64(int(seed) & (2**64 - 1)), _p(out)))
    return out


def mt19937_64(seed: int, n: int, skip: int = 0) -> np.ndarray:
    """Raw std::mt19937_64(seed) words [skip, skip+n), generated on the device."""
    out = np.empty(int(n), np.uint64)
    _check(N.lib().ndc_sim_mt19937_64(C.c_uint64(int(seed) & (2**64 - 1)), int(skip), int(n),
                                      out.ctypes.data_as(C.POINTER(C.c_uint64))))
    return out


def snr_db(reference, estimate) -> float:
    """simulation.hpp:195-208: 10 log10(|ref|^2 / |est - ref|^2); inf for an exact match."""
    a, b = _f64(reference), _f64(estimate)
    if a.shape != b.shape:
        raise ShapeError(f"snr_db: shape {a.shape} vs {b.shape}")
    ref = float(np.sum(a * a))
    err = float(np.sum((b - a) ** 2))
    if ref == 0.0:
        raise NumericError("snr_db: reference is all zero, metric undefined")
    return float("inf") if err == 0.0 else 10.0 * float(np.log10(ref / err))


# --- device-resident plan ----------------------------------------------------------------


def slab_range(mz: int, pz: int, rank: int, world: int):
    """z-slab ownership (ndc_slab_range): (x_begin, x_end, y_begin, y_end)."""
    v = [C.c_size_t() for _ in range(4)]
    _check(N.lib().ndc_slab_range(int(mz), int(pz), int(rank), int(world), *[C.byref(t) for t in v]))
    return tuple(t.value for t in v)


def probe_fp32_peak(device: int = 0) -> float:
    """Measured FP32 FMA throughput of the device, TFLOP/s (ndc_probe_fp32_peak)."""
    v = C.c_double()
    _check(N.lib().ndc_probe_fp32_peak(int(device), C.byref(v)))
    return v.value


def guard_violations() -> int:
    """Guard bytes found changed so far in this process (NDC_GUARD_BANDS=1 only)."""
    v = C.c_ulonglong()
    _check(N.lib().ndc_debug_guard_violations(C.byref(v)))
    return v.value


def _nccl_preload() -> None:
    """Load the NCCL that torch.distributed uses (the nvidia-nccl wheel) before the library
    opens libnccl.so.2: one libnccl.so.2 per process (shared by soname), so the plan's
    communicator and the plumbing's must be the same build.  No-op without the wheel."""
    global _NCCL_PRELOADED
    if _NCCL_PRELOADED:
        return
    _NCCL_PRELOADED = True
    import importlib.util
    import os
    try:
        spec = importlib.util.find_spec("nvidia.nccl")
    except (ImportError, ValueError):
        spec = None
    for d in (spec.submodule_search_locations if spec else []) or []:
        path = os.path.join(d, "lib", "libnccl.so.2")
        if os.path.exists(path):
            C.CDLL(path, mode=getattr(os, "RTLD_LOCAL", 0) | getattr(os, "RTLD_NOW", 2))
            os.environ.setdefault("NDC_NCCL_LIBRARY", path)
            return


_NCCL_PRELOADED = False


def nccl_unique_id() -> bytes:
    _nccl_preload()
    buf = C.create_string_buffer(128)
    _check(N.lib().ndc_nccl_unique_id(buf))
    return buf.raw


class Plan:
    """Device-resident problem (ndc_plan_*): `batch` images of one (x_shape, h), or one
    z-slab of a sharded volume (Plan.sharded / Plan.local)."""

    def __init__(self, x_shape, h, batch: int = 1, device: int = 0, _handle=None):
        self.h = _kernel(h)
        self.x_shape = tuple(int(s) for s in x_shape)
        self.y_shape = conv_output_shape(self.x_shape, self.h)
        self.batch = int(batch)
        self.handle = C.c_void_p()
        if _handle is not None:
            self.handle = _handle
        else:
            _check(N.lib().ndc_plan_create(C.byref(self.handle), int(device), self.batch, self.h.ndim,
                                           _ext(self.x_shape), _ext(self.h.shape), _p(self.h)))
        self.rank, self.world = 0, 1
        self.x_range = (0, self.x_shape[0])
        self.y_range = (0, self.y_shape[0])

    @classmethod
    def sharded(cls, x_shape, h, rank: int, world: int, nccl_id: bytes, device: int = 0):
        h = _kernel(h)
        _nccl_preload()
        handle = C.c_void_p()
        _check(N.lib().ndc_plan_create_sharded(C.byref(handle), int(device), h.ndim, _ext(x_shape),
                                               _ext(h.shape), _p(h), int(rank), int(world), nccl_id))
        return cls._wrap_slab(handle, x_shape, h, rank, world)

    @classmethod
    def local(cls, group: "LocalGroup", rank: int, x_shape, h, device: int = 0):
        h = _kernel(h)
        handle = C.c_void_p()
        _check(N.lib().ndc_plan_create_local(C.byref(handle), group.handle, int(rank), int(device), h.ndim,
                                             _ext(x_shape), _ext(h.shape), _p(h)))
        return cls._wrap_slab(handle, x_shape, h, rank, group.world)

    @classmethod
    def _wrap_slab(cls, handle, x_shape, h, rank, world):
        p = cls(x_shape, h, 1, _handle=handle)
        p.rank, p.world = int(rank), int(world)
        xa, xb, ya, yb = slab_range(x_shape[0], (h.shape[0] - 1) // 2, rank, world)
        p.x_range, p.y_range = (xa, xb), (ya, yb)
        return p

    def close(self):
        if self.handle:
            N.lib().ndc_plan_destroy(self.handle)
            self.handle = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # local (owned) shapes
    def owned_x_shape(self):
        return (self.x_range[1] - self.x_range[0],) + self.x_shape[1:]

    def owned_y_shape(self):
        return (self.y_range[1] - self.y_range[0],) + self.y_shape[1:]

    def set_observation(self, y):
        y = np.asarray(y)
        want = (self.batch,) + self.owned_y_shape()
        if y.size != int(np.prod(want)):
            raise ShapeError(f"set_observation: expected {want}, got {y.shape}")
        if y.dtype == np.float32:
            y = np.ascontiguousarray(y)
            _check(N.lib().ndc_plan_set_observation_f32(self.handle, _pf(y)))
        else:
            y = _f64(y)
            _check(N.lib().ndc_plan_set_observation_f64(self.handle, _p(y)))

    def load_observation(self, path):
        """Stream an NDTENSOR observation file into the plan (owned planes only)."""
        _check(N.lib().ndc_plan_load_observation_ndtensor(self.handle, _path(path)))

    def save_estimate(self, path):
        _check(N.lib().ndc_plan_save_estimate_ndtensor(self.handle, _path(path)))

    def add_gaussian_noise(self, mean: float = 0.0, std_dev: float = 0.0, seed: int = 0):
        """add_gaussian_noise on the resident observation (device mt19937_64 stream over the
        dense [batch, y...] order; a sharded rank applies its own planes' samples)."""
        _check(N.lib().ndc_plan_add_gaussian_noise(self.handle, float(mean), float(std_dev),
                                                   C.c_uint64(int(seed) & (2**64 - 1))))

    def pg_begin(self, cfg: DeconvConfig | None = None):
        c = (cfg or DeconvConfig()).to_c()
        _check(N.lib().ndc_plan_pg_begin(self.handle, C.byref(c)))

    def pg_iterate(self, n: int) -> int:
        a = C.c_size_t()
        _check(N.lib().ndc_plan_pg_iterate(self.handle, int(n), C.byref(a)))
        return a.value

    def pg_end(self):
        _check(N.lib().ndc_plan_pg_end(self.handle))

    def pg_run(self, cfg: DeconvConfig | None = None):
        c = (cfg or DeconvConfig()).to_c()
        _check(N.lib().ndc_plan_pg_run(self.handle, C.byref(c)))

    def rl_run(self, cfg: RlConfig | None = None):
        """deconv_rl (solvers.hpp:245-305) on the resident observation (left unchanged)."""
        cfg = cfg or RlConfig()
        c = N.RlConfig(int(cfg.max_iters), float(cfg.tol_rel_change))
        _check(N.lib().ndc_plan_rl_run(self.handle, C.byref(c)))

    def check_guards(self) -> int:
        """Changed guard bytes around this plan's allocations (NDC_GUARD_BANDS=1 only)."""
        v = C.c_size_t()
        _check(N.lib().ndc_plan_check_guards(self.handle, C.byref(v)))
        return v.value

    def estimate(self, dtype=np.float64) -> np.ndarray:
        x = np.empty((self.batch,) + self.owned_x_shape(), dtype)
        if dtype == np.float32:
            _check(N.lib().ndc_plan_get_estimate_f32(self.handle, _pf(x)))
        else:
            _check(N.lib().ndc_plan_get_estimate_f64(self.handle, _p(x)))
        return x

    def observation(self) -> np.ndarray:
        """The resident observation (float32 on the device) as float64, owned planes."""
        y = np.empty((self.batch,) + self.owned_y_shape(), np.float64)
        _check(N.lib().ndc_plan_get_observation_f64(self.handle, _p(y)))
        return y

    def report(self, image: int, cap: int) -> DeconvReport:
        rep = N.Report()
        obj = np.empty(cap, np.float64)
        kkt = np.empty(cap, np.float64)
        _check(N.lib().ndc_plan_get_report(self.handle, int(image), C.byref(rep), _p(obj), _p(kkt), int(cap)))
        return _report(None, rep, obj, kkt)

    def forward(self):
        _check(N.lib().ndc_plan_forward(self.handle))

    def adjoint(self):
        _check(N.lib().ndc_plan_adjoint(self.handle))

    def set_timing(self, on: bool):
        _check(N.lib().ndc_plan_set_timing(self.handle, 1 if on else 0))

    def reset_stats(self):
        _check(N.lib().ndc_plan_reset_stats(self.handle))

    def stats(self, kind: int):
        n = C.c_uint64()
        ms = C.c_double()
        _check(N.lib().ndc_plan_stats(self.handle, int(kind), C.byref(n), C.byref(ms)))
        return n.value, ms.value

    def stream(self) -> int:
        s = C.c_void_p()
        _check(N.lib().ndc_plan_stream(self.handle, C.byref(s)))
        return s.value or 0


class LocalGroup:
    """In-process slab group (ndc_local_group_*): drive each rank's Plan from its own thread."""

    def __init__(self, world: int):
        self.world = int(world)
        self.handle = C.c_void_p()
        _check(N.lib().ndc_local_group_create(C.byref(self.handle), self.world))

    def close(self):
        if self.handle:
            N.lib().ndc_local_group_destroy(self.handle)
            self.handle = C.c_void_p()
