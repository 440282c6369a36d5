"""TEST INFRASTRUCTURE ONLY -- ctypes front end for the CPU oracles.

Two interchangeable back ends with identical signatures:

* ``"c"``   -- ``oracle/_build/libndconv_oracle.so``, the plain-C restatement of the
  reference algorithm (``oracle/ndconv_oracle.c``);
* ``"ref"`` -- ``oracle/_ref/libndconv_ref.so``, the unmodified reference headers
  (``/root/reference/proj/include``) compiled behind a C shim (``oracle/ref_shim.cpp``).
* ``"fast"`` -- ``oracle/_build/libndconv_fast.so``, the same algorithm with threaded,
  vectorised float64 convolutions (``oracle/ndconv_fast.c``) for config-scale parity:
  conv_full / adjoint_apply / estimate_step / deconv_pg only, pinned to the "c" oracle
  to ~1e-12 by tests/test_oracle.py.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline legs may import
this module.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIBS = {
    "c": os.path.join(HERE, "_build", "libndconv_oracle.so"),
    "ref": os.path.join(HERE, "_ref", "libndconv_ref.so"),
    "fast": os.path.join(HERE, "_build", "libndconv_fast.so"),
}
PREFIX = {"c": "oc_", "ref": "ref_", "fast": "of_"}

RC_NAMES = {1: "Error", 2: "ShapeError", 3: "NumericError", 4: "BoundsError", 5: "FormatError", 9: "Other"}
STOP_NAMES = {0: "converged", 1: "max_iters", 2: "stalled"}


class OracleError(RuntimeError):
    def __init__(self, rc: int, what: str):
        super().__init__(f"{what}: {RC_NAMES.get(rc, rc)}")
        self.rc = rc
        self.kind = RC_NAMES.get(rc, str(rc))


class _PgCfg(C.Structure):
    _fields_ = [
        ("max_iters", C.c_size_t),
        ("tol_rel_objective", C.c_double),
        ("has_initial_step", C.c_int),
        ("initial_step", C.c_double),
        ("backtrack_factor", C.c_double),
        ("max_backtracks", C.c_size_t),
        ("power_iters", C.c_size_t),
    ]


class _RlCfg(C.Structure):
    _fields_ = [("max_iters", C.c_size_t), ("tol_rel_change", C.c_double)]


@dataclass
class Report:
    estimate: np.ndarray
    objective_trace: np.ndarray
    kkt_trace: np.ndarray
    iterations_run: int
    stop_reason: str
    extra: dict = field(default_factory=dict)


def available(kind: str) -> bool:
    return os.path.exists(LIBS[kind])


def _ext(shape) -> C.Array:
    return (C.c_size_t * len(shape))(*[int(s) for s in shape])


def _f64(a: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


class Oracle:
    def __init__(self, kind: str = "c"):
        path = LIBS[kind]
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library {path} not built (run make -C oracle)")
        self.kind = kind
        self.lib = C.CDLL(path)
        self.p = PREFIX[kind]

    def _fn(self, name):
        return getattr(self.lib, self.p + name)

    def _call(self, name, *args):
        fn = self._fn(name)
        fn.restype = C.c_int
        rc = fn(*args)
        if rc:
            raise OracleError(rc, name)

    def set_threads(self, n: int):
        self._fn("set_threads")(C.c_int(int(n)))

    # -- operators ---------------------------------------------------------------
    def conv_full(self, x, h):
        x, h = _f64(x), _f64(h)
        y = np.empty([a + b - 1 for a, b in zip(x.shape, h.shape)], np.float64)
        self._call("conv_full", C.c_int(x.ndim), _ext(x.shape), _ptr(x), _ext(h.shape), _ptr(h), _ptr(y))
        return y

    def adjoint_apply(self, y, h, x_shape):
        y, h = _f64(y), _f64(h)
        out = np.empty(tuple(x_shape), np.float64)
        self._call("adjoint_apply", C.c_int(y.ndim), _ext(y.shape), _ptr(y), _ext(h.shape), _ptr(h),
                   _ext(x_shape), _ptr(out))
        return out

    def objective(self, x, y, h):
        x, y, h = _f64(x), _f64(y), _f64(h)
        f = C.c_double()
        self._call("objective", C.c_int(x.ndim), _ext(x.shape), _ptr(x), _ptr(y), _ext(h.shape), _ptr(h),
                   C.byref(f))
        return f.value

    def normal_gradient(self, x, y, h):
        x, y, h = _f64(x), _f64(y), _f64(h)
        g = np.empty(x.shape, np.float64)
        self._call("normal_gradient", C.c_int(x.ndim), _ext(x.shape), _ptr(x), _ptr(y), _ext(h.shape),
                   _ptr(h), _ptr(g))
        return g

    def estimate_step(self, h, x_shape, power_iters=30):
        h = _f64(h)
        s = C.c_double()
        self._call("estimate_step", C.c_int(h.ndim), _ext(h.shape), _ptr(h), _ext(x_shape),
                   C.c_size_t(power_iters), C.byref(s))
        return s.value

    def kkt_residual(self, x, y, h):
        x, y, h = _f64(x), _f64(y), _f64(h)
        k = C.c_double()
        self._call("kkt_residual", C.c_int(x.ndim), _ext(x.shape), _ptr(x), _ptr(y), _ext(h.shape),
                   _ptr(h), C.byref(k))
        return k.value

    def conv_full_sample(self, x, h, flat_idx):
        x, h = _f64(x), _f64(h)
        idx = np.ascontiguousarray(flat_idx, dtype=np.uint64)
        out = np.empty(idx.size, np.float64)
        self._call("conv_full_sample", C.c_int(x.ndim), _ext(x.shape), _ptr(x), _ext(h.shape), _ptr(h),
                   C.c_size_t(idx.size), idx.ctypes.data_as(C.POINTER(C.c_size_t)), _ptr(out))
        return out

    def adjoint_sample(self, y, h, x_shape, flat_idx):
        y, h = _f64(y), _f64(h)
        idx = np.ascontiguousarray(flat_idx, dtype=np.uint64)
        out = np.empty(idx.size, np.float64)
        self._call("adjoint_sample", C.c_int(y.ndim), _ext(y.shape), _ptr(y), _ext(h.shape), _ptr(h),
                   _ext(x_shape), C.c_size_t(idx.size), idx.ctypes.data_as(C.POINTER(C.c_size_t)),
                   _ptr(out))
        return out

    # -- solvers -----------------------------------------------------------------
    def deconv_pg(self, y, h, x_shape, max_iters=500, tol_rel_objective=1e-6, initial_step=None,
                  backtrack_factor=0.5, max_backtracks=50, power_iters=30) -> Report:
        y, h = _f64(y), _f64(h)
        cfg = _PgCfg(max_iters, tol_rel_objective, 0 if initial_step is None else 1,
                     0.0 if initial_step is None else float(initial_step), backtrack_factor,
                     max_backtracks, power_iters)
        x = np.empty(tuple(x_shape), np.float64)
        ot = np.empty(max_iters + 1, np.float64)
        kt = np.empty(max_iters + 1, np.float64)
        tl, it, bt = C.c_size_t(), C.c_size_t(), C.c_size_t()
        sr = C.c_int()
        st = C.c_double()
        more = (C.byref(st),) if self.kind == "fast" else ()
        self._call("deconv_pg", C.c_int(y.ndim), _ext(y.shape), _ptr(y), _ext(h.shape), _ptr(h),
                   _ext(x_shape), C.byref(cfg), _ptr(x), _ptr(ot), _ptr(kt), C.byref(tl), C.byref(it),
                   C.byref(sr), C.byref(bt), *more)
        n = tl.value
        extra = {} if self.kind == "ref" else {"backtracks": bt.value}
        if self.kind == "fast":
            extra["step0"] = st.value
        return Report(x, ot[:n].copy(), kt[:n].copy(), it.value, STOP_NAMES[sr.value], extra)

    def deconv_rl(self, y, h, x_shape, max_iters=500, tol_rel_change=0.0) -> Report:
        y, h = _f64(y), _f64(h)
        cfg = _RlCfg(max_iters, tol_rel_change)
        x = np.empty(tuple(x_shape), np.float64)
        ot = np.empty(max_iters + 1, np.float64)
        kt = np.empty(max_iters + 1, np.float64)
        tl, it, cl = C.c_size_t(), C.c_size_t(), C.c_size_t()
        sr = C.c_int()
        self._call("deconv_rl", C.c_int(y.ndim), _ext(y.shape), _ptr(y), _ext(h.shape), _ptr(h),
                   _ext(x_shape), C.byref(cfg), _ptr(x), _ptr(ot), _ptr(kt), C.byref(tl), C.byref(it),
                   C.byref(sr), C.byref(cl))
        n = tl.value
        return Report(x, ot[:n].copy(), kt[:n].copy(), it.value, STOP_NAMES[sr.value],
                      {"negative_pixels_clamped": cl.value})

    def pg_iterations(self, y, h, x_shape, step0, iters, x, ax, aty, f,
                      backtrack_factor=0.5, max_backtracks=50):
        """Reference-only: replay ``iters`` accepted PG iterations with the
        reference's operators (ref_shim.cpp ref_pg_iterations).  x/ax are updated
        in place; returns (f, accepted)."""
        if self.kind != "ref":
            raise NotImplementedError("pg_iterations is a reference-shim entry point")
        y, h = _f64(y), _f64(h)
        fo = C.c_double(f)
        acc = C.c_size_t()
        self._call("pg_iterations", C.c_int(y.ndim), _ext(y.shape), _ptr(y), _ext(h.shape), _ptr(h),
                   _ext(x_shape), C.c_double(step0), C.c_double(backtrack_factor),
                   C.c_size_t(max_backtracks), C.c_size_t(iters), _ptr(x), _ptr(ax), _ptr(_f64(aty)),
                   C.byref(fo), C.byref(acc))
        return fo.value, acc.value

    # --- tensor file formats (reference only: ref_shim.cpp ref_io_*) -------------------
    def _ref_only(self, what):
        if self.kind != "ref":
            raise NotImplementedError(f"{what} is a reference-shim entry point")

    def _parse(self, name, data: bytes) -> np.ndarray:
        self._ref_only(name)
        nd = C.c_int()
        ext = (C.c_size_t * 16)()
        self._call(name, data, C.c_size_t(len(data)), C.byref(nd), ext, None, C.c_size_t(0))
        out = np.empty(tuple(int(ext[i]) for i in range(nd.value)), np.float64)
        self._call(name, data, C.c_size_t(len(data)), C.byref(nd), ext, _ptr(out), C.c_size_t(out.size))
        return out

    def parse_tensor(self, data: bytes) -> np.ndarray:
        """imageio.hpp:78-120 read_tensor(std::istream&) on ``data``."""
        return self._parse("io_parse_tensor", data)

    def parse_pgm(self, data: bytes) -> np.ndarray:
        """imageio.hpp:184-231 read_pgm(std::istream&) on ``data``."""
        return self._parse("io_parse_pgm", data)

    def _serialize(self, name, t, *extra) -> bytes:
        self._ref_only(name)
        t = _f64(t)
        n = C.c_size_t()
        self._call(name, C.c_int(t.ndim), _ext(t.shape), _ptr(t), *extra, None, C.c_size_t(0), C.byref(n))
        buf = C.create_string_buffer(n.value)
        self._call(name, C.c_int(t.ndim), _ext(t.shape), _ptr(t), *extra, buf, C.c_size_t(n.value), C.byref(n))
        return buf.raw[: n.value]

    def serialize_tensor(self, t) -> bytes:
        """imageio.hpp:63-71 write_tensor(t, std::ostream&)."""
        return self._serialize("io_serialize_tensor", t)

    def serialize_pgm(self, t, clamp: bool = False) -> bytes:
        """imageio.hpp:238-260 write_pgm(t, std::ostream&, clamp)."""
        return self._serialize("io_serialize_pgm", t, C.c_int(1 if clamp else 0))

    def snr_db(self, a, b) -> float:
        """simulation.hpp:195-208."""
        self._ref_only("snr_db")
        a, b = _f64(a), _f64(b)
        out = C.c_double()
        self._call("snr_db", C.c_int(a.ndim), _ext(a.shape), _ptr(a), _ptr(b), C.byref(out))
        return out.value

    # --- simulation generators (reference only: ref_shim.cpp ref_sim_*) ------------------
    def phantom_lines(self, rows, cols, n_lines, intensity):
        self._ref_only("phantom_lines")
        out = np.empty((rows, cols), np.float64)
        self._call("sim_phantom_lines", C.c_size_t(rows), C.c_size_t(cols), C.c_size_t(n_lines),
                   C.c_double(intensity), _ptr(out))
        return out

    def phantom_texture(self, rows, cols):
        self._ref_only("phantom_texture")
        out = np.empty((rows, cols), np.float64)
        self._call("sim_phantom_texture", C.c_size_t(rows), C.c_size_t(cols), _ptr(out))
        return out

    def gaussian_psf(self, extents, sigma):
        self._ref_only("gaussian_psf")
        out = np.empty(tuple(extents), np.float64)
        self._call("sim_gaussian_psf", C.c_int(len(extents)), _ext(extents), C.c_double(sigma), _ptr(out))
        return out

    def delta_psf(self, extents):
        self._ref_only("delta_psf")
        out = np.empty(tuple(extents), np.float64)
        self._call("sim_delta_psf", C.c_int(len(extents)), _ext(extents), _ptr(out))
        return out

    def add_gaussian_noise(self, t, mean, std_dev, seed):
        self._ref_only("add_gaussian_noise")
        t = _f64(t)
        out = np.empty_like(t)
        self._call("sim_add_gaussian_noise", C.c_size_t(t.size), _ptr(t), C.c_double(mean), C.c_double(std_dev),
                   C.c_uint64(seed), _ptr(out))
        return out

    def mt19937_64(self, seed, n, skip=0):
        self._ref_only("mt19937_64")
        out = np.empty(n, np.uint64)
        self._call("mt19937_64", C.c_uint64(seed), C.c_size_t(skip), C.c_size_t(n),
                   out.ctypes.data_as(C.POINTER(C.c_uint64)))
        return out
