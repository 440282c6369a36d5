"""Benchmark of the convolution-only deconvolution hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c5]

Metric (BASELINE.json): voxel-iterations/s of the projected-gradient iteration (forward
full conv + residual + adjoint valid correlation + projected update + reductions) and
its fraction of the FP32 roofline, at 1/2/4/8 B200.

Default workload, at every N: BASELINE config 5 -- the largest 3-D volume, 256 x 2048 x
2048 voxels (1.07 G), the 65x33x33 widefield 3-Gaussian PSF (70,785 taps), filaments +
5000 blobs, Poisson noise at peak 200, 20 iterations -- the config north_star's ">= 85 %
parallel efficiency at 8 GPUs on the largest 3D volume" names.  At N = 1 it runs on one
GPU; at N > 1 the volume is z-slab sharded across the N ranks (p_z = 32-plane halos over
NCCL, rank-order scalar combine), so `scaling` is "strong" (the total volume is fixed)
and BENCH N=1 is SCALE N=1.  Every rank generates only its own slab's observation (the
x planes it depends on, seeded per object and per plane, bit-identical to the full
volume's planes).  `--config c2` (16 x 2048^2 images, 31x31 PSF; N > 1 = independent
replicas), c3, c4 and c2s (small-PSF HBM case) select the other configs.

A "step" is one PG iteration over the whole volume (or batch).  Inputs are resident in
HBM before the timed region and larger than the 126 MB L2 (no flush needed).  One JSON
line on rank 0.  `value` is device time (CUDA events on the plan's stream, max over
ranks); `e2e` is the same metric through the public C-ABI with host f64 buffers: the
upload of the observation, a whole deconv_pg run of the config's iteration count, the
download of the estimate and traces inside the timed region (max over ranks);
`roofline` is the dominant pass's algorithmic FLOP rate against the FP32 FFMA peak;
`cpu_baseline` is the reference (oracle/_ref, the unmodified reference compiled from
/root/reference) on this host's cores.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_SM = 148
FFMA_PER_SM_CLK = 128


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None, help="timed PG iterations (default per config)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c5")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-iters", type=int, default=1)
    return ap.parse_args(argv)


# --- distributed plumbing -------------------------------------------------------------------

def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class Dist:
    def __init__(self, backend="nccl"):
        self.rank, self.world, self.local = dist_env()
        self.pg = None
        self.backend = backend
        if self.world > 1:
            if backend == "nccl":
                # communicator lines (rank, nranks, transport) for the run log, on stderr so
                # the JSON line stays the only line on stdout
                os.environ.setdefault("NCCL_DEBUG", "INFO")
                os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
                os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
            import torch
            import torch.distributed as dist
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            if backend == "nccl":
                torch.cuda.set_device(self.local)
            dist.init_process_group(backend=backend)
            self.dist = dist
            self.torch = torch

    def barrier(self):
        """Device-wide sync first (no plan NCCL operation is in flight when the plumbing
        communicator's barrier runs), then the rank barrier."""
        if self.world > 1:
            if self.backend == "nccl":
                self.torch.cuda.synchronize()
            self.dist.barrier()

    def allmax(self, v: float) -> float:
        return self.max(v)

    def max(self, v: float) -> float:
        if self.world == 1:
            return v
        dev = f"cuda:{self.local}" if self.backend == "nccl" else "cpu"
        t = self.torch.tensor([v], dtype=self.torch.float64, device=dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.world > 1:
            self.dist.destroy_process_group()


# --- clocks sampler -----------------------------------------------------------------------

class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []  # (host arrival time, csv line)
        self.window = None

    def start(self, wait_first: float = 5.0):
        """Start sampling every 50 ms; return once the first sample has arrived so the
        timed region is covered (start it before the warm-up)."""
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t_end = time.time() + wait_first
            while not self.lines and time.time() < t_end:
                time.sleep(0.01)
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def mark(self, t0: float, t1: float):
        self.window = (t0, t1)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.12)  # let the sample after the window arrive
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=2)
        sel = self.lines
        basis = "all samples"
        if self.window:
            t0, t1 = self.window
            inside = [l for l in self.lines if t0 <= l[0] <= t1 + 0.06]
            if inside:
                sel, basis = inside, "samples inside the timed region"
            else:  # region shorter than the sampling period: nearest samples around it
                near = sorted(self.lines, key=lambda l: min(abs(l[0] - t0), abs(l[0] - t1)))[:2]
                sel, basis = near, "nearest samples to a timed region shorter than 50 ms"
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for _, ln in sel:
            f = [s.strip() for s in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm), "basis": basis}


# --- workloads --------------------------------------------------------------------------------

# Per-config defaults: iterations per e2e solve (the config's BASELINE iteration count),
# timed steps, explicit step size.  The 3-D configs use initial_step = 1 (their PSFs
# are nonnegative with unit sum, so ||A|| <= 1 and 1 is a valid gradient step; the auto
# step at these sizes is checked against the reference in tests/test_gpu_config_scale.py);
# the 2-D batches estimate the step (untimed setup).
WORK = {
    "c2": dict(e2e_iters=100, steps=30, step=None, desc="16x2048x2048 2D batch, PSF 31x31 sigma 4, Poisson 1000"),
    "c3": dict(e2e_iters=50, steps=20, step=1.0, desc="3D 256x256x128, PSF 15x15x31 sigma_xy 1.5 sigma_z 4"),
    "c4": dict(e2e_iters=30, steps=5, step=1.0, desc="3D 1024x1024x512, PSF 9x9x21, Poisson 500"),
    "c5": dict(e2e_iters=20, steps=3, step=1.0,
               desc="3D 2048x2048x256 (filaments + 5000 blobs), 33x33x65 3-Gaussian widefield PSF, Poisson 200"),
    # HBM-bound small-PSF case (not a BASELINE config; north_star's ">= 70 % HBM" target)
    "c2s": dict(e2e_iters=100, steps=500, step=None,
                desc="16x2048x2048 2D batch, PSF 5x5 sigma 1 (reference acceptance PSF), Poisson 1000"),
}
HBM_BOUND = ("c2s",)


VOLUME = ("c3", "c4", "c5")


def inputs_2d(config: str, rank: int):
    """A 2-D batch (independent images; each rank of a replica run its own seed)."""
    from paper_1711_11224_b200 import synth
    _, y, h = synth.make(config, seed=synth.SEED + 100003 * rank)
    return y.astype(np.float32), h


def inputs_volume(config: str, y0: int, y1: int, d, device, shape=None, n_objects=None):
    """Observation planes [y0, y1) of a 3-D config, float32: the rank generates the x
    planes they depend on (synth.clean_observation_planes), the noise is seeded per plane
    and scaled by the whole volume's maximum (all-reduced), so every plane equals the
    unsharded volume's."""
    from paper_1711_11224_b200 import synth
    yc = synth.clean_observation_planes(config, y0, y1, shape=shape, n_objects=n_objects)
    if config == "c3":
        y = synth.gaussian_planes(yc, 0.005, synth.SEED + 1000, y0)
    else:
        peak = {"c4": 500.0, "c5": 200.0}[config]
        m = d.allmax(float(yc.max()))
        y = synth.poisson_planes(yc, peak, m, synth.SEED + 1000, y0, device=device)
    del yc
    return y.astype(np.float32)[None]


# --- CPU baseline (reference compiled from /root/reference: oracle/_ref) --------------------

class RefRunner:
    """The reference's own CPU path on ONE image of the config (configs 3-5: a reduced
    volume with the same PSF), all host threads.  setup() builds A^T y, x0 and
    A x0 untimed; step() times one PG loop-body iteration (ref_pg_iterations = the
    reference's operators in solvers.hpp:179-228 order)."""

    def __init__(self, config: str):
        from oracle.oracle import Oracle, available
        from paper_1711_11224_b200 import synth
        self.kind = "reference" if available("ref") else "port"
        self.orc = Oracle("ref" if self.kind == "reference" else "c")
        self.cores = os.cpu_count() or 1
        self.orc.set_threads(self.cores)
        if config in ("c2", "c2s"):
            _, y, h = synth.make(config, batch=1)
            self.y, self.h, self.xs = y[0], h, (2048, 2048)
        elif config == "c1":
            x, self.y, self.h = synth.make("c1")
            self.xs = x.shape
        else:
            shape = {"c3": (128, 256, 256), "c4": (64, 128, 128), "c5": (64, 96, 96)}[config]
            x, self.y, self.h = synth.make(config, shape=shape, n_objects=200)
            self.xs = x.shape
        self.sample = f"{'1 image' if config in ('c1', 'c2', 'c2s') else 'volume'} {self.xs}, PSF {self.h.shape}"
        self.voxels = int(np.prod(self.xs))
        self.step0 = 1.0  # unit-sum PSFs: ||A|| <= 1; loop-body cost does not depend on it

    def setup(self):
        self.aty = self.orc.adjoint_apply(self.y, self.h, self.xs)
        self.x = np.maximum(self.aty, 0.0)
        self.ax = self.orc.conv_full(self.x, self.h)
        self.f = 0.5 * float(np.sum((self.ax - self.y) ** 2))

    def step(self, iters: int = 1) -> float:
        t0 = time.perf_counter()
        if self.kind == "reference":
            self.f, _ = self.orc.pg_iterations(self.y, self.h, self.xs, self.step0, iters, self.x, self.ax,
                                               self.aty, self.f)
        else:
            self.orc.deconv_pg(self.y, self.h, self.xs, max_iters=iters, tol_rel_objective=0.0,
                               initial_step=self.step0)
        return time.perf_counter() - t0


def cpu_reference_sample(config: str, iters: int):
    r = RefRunner(config)
    r.setup()
    dt = r.step(iters)
    return {"value": r.voxels * iters / dt, "unit": "voxel-iterations/s", "cores": r.cores, "kind": r.kind,
            "sample": f"{r.sample}, {iters} PG iterations (loop body only), {dt:.2f} s"}, dt


# --- our arm ------------------------------------------------------------------------------------

def measured_hbm_peak():
    """(GB/s, basis): MEASURED_PEAKS.json's driver-measured copy bandwidth, else the
    profiling guide's B200 fallback."""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        v = float(json.load(open(p))["hbm_gbs"])
        return v, f"MEASURED_PEAKS.json hbm_gbs (torch copy, read+write bytes): {v:.1f} GB/s"
    except (OSError, ValueError, KeyError):
        return 7700.0, "fallback: B200 HBM3e nominal 7.7 TB/s (MEASURED_PEAKS.json absent)"


def make_plan(nd, d, x_shape, h, B, local, sharded):
    if not sharded:
        return nd.Plan(x_shape, h, batch=B, device=local)
    uid = nd.nccl_unique_id() if d.rank == 0 else None
    obj = [uid]
    d.dist.broadcast_object_list(obj, src=0)
    return nd.Plan.sharded(x_shape, h, d.rank, d.world, obj[0], device=local)


def run_ours(a):
    rank, world, local = dist_env()
    d = Dist("nccl")
    import torch  # plumbing only: external-stream CUDA events and the rank collectives
    from paper_1711_11224_b200 import ndconv as nd, synth
    if nd.device_count() < 1:
        raise SystemExit("no B200 visible")
    torch.cuda.set_device(local)
    work = WORK[a.config]
    steps = a.steps if a.steps is not None else work["steps"]
    volume = a.config in VOLUME
    sharded = world > 1 and volume
    t_gen = time.perf_counter()
    if volume:
        x_shape = tuple(synth.CONFIGS[a.config]["shape"])
        h = synth.psf_for(a.config)
        B = 1
        _, _, ya, yb = nd.slab_range(x_shape[0], (h.shape[0] - 1) // 2, rank, world) if sharded \
            else (0, 0, 0, x_shape[0] + h.shape[0] - 1)
        y_own = inputs_volume(a.config, ya, yb, d, f"cuda:{local}")
    else:
        y_own, h = inputs_2d(a.config, rank)
        B = y_own.shape[0]
        x_shape = tuple(s - k + 1 for s, k in zip(y_own.shape[1:], h.shape))
    t_gen = time.perf_counter() - t_gen
    K = int(np.prod(h.shape))
    plan = make_plan(nd, d, x_shape, h, B, local, sharded)
    xa, xb = plan.x_range if sharded else (0, x_shape[0])
    vox_rank = B * (xb - xa) * int(np.prod(x_shape[1:]))
    vox_job = B * int(np.prod(x_shape)) * (1 if (sharded or volume) else world)
    cfg = nd.DeconvConfig(max_iters=a.warmup + steps + 1, tol_rel_objective=0.0, initial_step=work["step"])

    plan.set_observation(y_own)
    plan.pg_begin(cfg)
    clocks = Clocks(local)
    clocks.start()  # sampling runs through warm-up and the timed steps
    for _ in range(a.warmup):
        plan.pg_iterate(1)
    stream = torch.cuda.ExternalStream(plan.stream(), device=f"cuda:{local}")
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    plan.reset_stats()
    plan.set_timing(True)
    d.barrier()
    torch.cuda.synchronize()
    t0 = time.time()
    e0.record(stream)
    for _ in range(steps):
        plan.pg_iterate(1)
    e1.record(stream)
    torch.cuda.synchronize()
    clocks.mark(t0, time.time())
    d.barrier()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    ms_max = d.max(ms)
    n_fwd, ms_fwd = plan.stats(0)
    n_adj, ms_adj = plan.stats(1)
    n_all, _ = plan.stats(2)
    plan.set_timing(False)
    plan.pg_end()
    rep = plan.report(0, cfg.max_iters + 1)

    value = vox_job * steps / (ms_max / 1e3)
    # Dominant pass: algorithmic FLOPs per pass = 2 K per x voxel of this rank (forward:
    # every x voxel meets K taps; adjoint: every output meets K taps).  A pass is one
    # launch, or several tap-chunk launches for PSFs beyond the 7680-tap parameter block
    # (config 5: 11) -- the roofline uses the pass time.
    flops_pass = 2.0 * K * vox_rank
    passes = steps  # one forward and one adjoint per accepted iteration without backtracks
    dom, n_dom, ms_dom = ("adjoint", n_adj, ms_adj) if ms_adj >= ms_fwd else ("forward", n_fwd, ms_fwd)
    avg_s = ms_dom / max(passes, 1) / 1e3
    achieved = flops_pass / avg_s / 1e12
    smax = clk.get("sm_max_mhz") or 1965.0
    peak_theory = N_SM * FFMA_PER_SM_CLK * 2 * smax * 1e6 / 1e12
    # measured FP32 FMA peak on this GPU, right after the timed region (same clocks):
    # a register-only packed-FMA kernel on every SM (ndc_probe_fp32_peak)
    try:
        peak_meas = nd.probe_fp32_peak(local)
    except nd.Error:
        peak_meas = None
    peak = peak_meas or peak_theory
    if a.config in HBM_BOUND:
        hbm_peak = measured_hbm_peak()
    # DRAM bytes of the dominant pass from the ncu capture at HEAD (tools/ncu_traffic.py:
    # dram__bytes_read.sum + dram__bytes_write.sum over every launch of one pass, whole
    # volume / batch on one GPU); a z-slab rank's share scales with its planes
    traffic, traffic_basis = None, None
    tf = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tf):
        try:
            t = json.load(open(tf)).get(a.config, {})
            if t.get(dom):
                traffic = float(t[dom]) * (vox_rank / (B * int(np.prod(x_shape))) if sharded else 1.0)
                traffic_basis = t.get("source", "") + (" (scaled to this rank's planes)" if sharded else "")
        except (OSError, ValueError):
            traffic = None
    # algorithmic bytes of the pass (float32): forward reads x and Y, writes r; adjoint
    # reads r and x, writes trial and g (this rank's planes)
    y_plane = int(np.prod([s + k - 1 for s, k in zip(x_shape[1:], h.shape[1:])]))
    ny_rank = B * y_plane * ((yb - ya) if volume else (x_shape[0] + h.shape[0] - 1))
    alg_bytes = 4.0 * ((ny_rank + 3 * vox_rank) if dom == "adjoint" else (vox_rank + 2 * ny_rank))
    par = "single" if world == 1 else (f"z-slab{world}" if sharded else f"replicas{world}")
    line = {
        "metric": "voxel-iterations/sec (fwd+adjoint conv) and % of FP32/HBM roofline @1/2/4/8 B200",
        "value": value, "unit": "voxel-iterations/s", "n_gpus": world, "steps": steps,
        "warmup": a.warmup, "ms_per_step": ms_max / steps, "higher_is_better": True,
        "scaling": "strong" if volume else "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": f"{a.config}: {work['desc']}",
                   "batch_per_gpu": B, "x_shape": list(x_shape), "psf": list(h.shape), "taps": K,
                   "parallelism": par, "x_planes_per_rank": xb - xa if volume else None,
                   "l2": "inputs larger than L2 (no flush)",
                   "step": "one PG iteration over the whole " + ("volume" if volume else "batch"),
                   "tol_rel_objective": 0.0,
                   "step_size": "auto (power iteration, untimed setup)" if work["step"] is None
                   else f"initial_step={work['step']} (unit-sum PSF)",
                   "input_generation_s": round(t_gen, 2)},
        "roofline": ({"bound": "hbm", "kernel": dom, "achieved": alg_bytes / avg_s / 1e9, "peak": hbm_peak[0],
                      "unit": "GB/s", "frac": alg_bytes / avg_s / 1e9 / hbm_peak[0], "traffic": traffic,
                      "traffic_basis": traffic_basis,
                      "peak_basis": hbm_peak[1], "algorithmic_bytes_per_pass": alg_bytes,
                      "pass_ms": avg_s * 1e3, "launches_per_pass": n_dom / max(passes, 1),
                      "fp32_tflops": achieved,
                      "forward": {"launches": n_fwd, "ms": ms_fwd}, "adjoint": {"launches": n_adj, "ms": ms_adj}}
                     if a.config in HBM_BOUND else
                     {"bound": "fp32", "kernel": dom, "achieved": achieved, "peak": peak,
                     "unit": "TFLOP/s", "frac": achieved / peak, "traffic": traffic,
                     "peak_basis": ("measured on this GPU after the timed region: register-only FFMA2 "
                                    "probe on all SMs (ndc_probe_fp32_peak); MEASURED_PEAKS.json has no "
                                    "FP32 figure" if peak_meas else
                                    f"{N_SM} SMs x 128 FFMA x 2 x {smax:.0f} MHz (probe unavailable)"),
                     "peak_theoretical": peak_theory, "frac_theoretical": achieved / peak_theory,
                     "traffic_basis": traffic_basis, "algorithmic_bytes_per_pass": alg_bytes,
                     "algorithmic_flops_per_pass": flops_pass, "pass_ms": avg_s * 1e3,
                     "launches_per_pass": n_dom / max(passes, 1),
                     "frac_at_observed_clock": (achieved / (N_SM * FFMA_PER_SM_CLK * 2 * clk["sm_mhz"] * 1e6 / 1e12)
                                                if clk.get("sm_mhz") else None),
                     "forward": {"launches": n_fwd, "ms": ms_fwd}, "adjoint": {"launches": n_adj, "ms": ms_adj}}),
        "gpu_launches": int(n_all),
        "clocks": clk,
        "iterations_accepted": int(rep.iterations_run),
        "backtracks": int(rep.extra.get("backtracks", 0)),
    }
    if not a.no_e2e:
        if volume:
            line["e2e"] = e2e_plan(nd, plan, y_own, work, vox_job, d)
        else:
            line["e2e"] = e2e_batch(nd, y_own, h, x_shape, B, work, world, d)
    plan.close()
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        cb, _ = cpu_reference_sample(a.config, a.cpu_iters)
        line["cpu_baseline"] = cb
    d.close()
    if rank == 0:
        print(json.dumps(line), flush=True)


def e2e_plan(nd, plan, y32, work, vox_job, d):
    """The public plan C-ABI with host f64 buffers, one whole solve per step: upload of
    this rank's observation planes (f64 -> f32 on the host pool, pinned ring, H2D),
    deconv_pg over the config's iteration count (ndc_plan_pg_run), download of the
    estimate planes as f64 and of the traces.  Max over ranks."""
    iters = work["e2e_iters"]
    yh = np.ascontiguousarray(y32, dtype=np.float64)
    cfg = nd.DeconvConfig(max_iters=iters, tol_rel_objective=0.0, initial_step=work["step"])
    d.barrier()
    t0 = time.perf_counter()
    plan.set_observation(yh)
    plan.pg_run(cfg)
    x = plan.estimate()
    rep = plan.report(0, iters + 1)
    dt = d.max(time.perf_counter() - t0)
    return {"value": vox_job * iters / dt, "unit": "voxel-iterations/s",
            "h2d_bytes_per_step": int(yh.nbytes),
            "d2h_bytes_per_step": int(x.nbytes + rep.objective_trace.nbytes + rep.kkt_trace.nbytes),
            "step": f"one full deconv_pg solve through the plan C-ABI (set_observation_f64, pg_run, "
                    f"get_estimate_f64, get_report): {iters} iterations, initial_step={work['step']}",
            "seconds_per_step": dt, "iterations_run": int(rep.iterations_run)}


def e2e_batch(nd, y32, h, x_shape, B, work, world, d):
    """Public C-ABI call (ndc_deconv_pg_batch_f64) with host f64 buffers: a whole solve
    per step -- H2D of Y, step estimate, all iterations, D2H of estimate and traces."""
    import ctypes as C
    from paper_1711_11224_b200 import _native as N
    iters = work["e2e_iters"]
    yh = np.ascontiguousarray(y32, dtype=np.float64)
    xo = np.empty((B,) + tuple(x_shape), np.float64)
    cap = iters + 1
    obj = np.empty((B, cap))
    kkt = np.empty((B, cap))
    reps = (N.Report * B)()
    cfg = nd.DeconvConfig(max_iters=iters, tol_rel_objective=0.0, initial_step=work["step"]).to_c()
    ext = (C.c_size_t * len(x_shape))(*x_shape)
    yext = (C.c_size_t * len(x_shape))(*yh.shape[1:])
    hext = (C.c_size_t * h.ndim)(*h.shape)
    hh = np.ascontiguousarray(h, np.float64)

    def call():
        rc = N.lib().ndc_deconv_pg_batch_f64(B, h.ndim, yext, yh.ctypes.data_as(N.dbl_p), hext,
                                             hh.ctypes.data_as(N.dbl_p), ext, C.byref(cfg),
                                             xo.ctypes.data_as(N.dbl_p), obj.ctypes.data_as(N.dbl_p),
                                             kkt.ctypes.data_as(N.dbl_p), cap, reps)
        if rc:
            raise RuntimeError(N.lib().ndc_last_error().decode())

    t0 = time.perf_counter()
    call()  # warm-up (module load, allocator)
    first = time.perf_counter() - t0
    reps_t = []
    # best of 3 (2 for solves over 2 s): the host side of the transfers is noisy
    for _ in range(3 if first < 2.0 else 2):
        d.barrier()
        t0 = time.perf_counter()
        call()
        reps_t.append(time.perf_counter() - t0)
    dt = d.max(min(reps_t))
    voxels = B * int(np.prod(x_shape))
    return {"value": world * voxels * iters / dt, "unit": "voxel-iterations/s",
            "h2d_bytes_per_step": int(yh.nbytes + hh.nbytes), "d2h_bytes_per_step": int(xo.nbytes + obj.nbytes + kkt.nbytes),
            "step": f"one full deconv_pg_batch_f64 call: {B} image(s), {iters} iterations, "
                    + ("auto step" if work["step"] is None else f"initial_step={work['step']}"),
            "seconds_per_step": dt}


def run_reference(a):
    """The reference's CPU implementation on the box's host cores (oracle/_ref: the
    unmodified reference headers compiled by oracle/Makefile), same config and metric;
    rank 0 only."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    steps = a.steps if a.steps is not None else 10
    r = RefRunner(a.config)
    r.setup()
    for _ in range(a.warmup):
        r.step(1)
    times = [r.step(1) for _ in range(steps)]
    per = float(np.sum(times))
    value = r.voxels * steps / per
    cb = {"value": value, "unit": "voxel-iterations/s", "cores": r.cores, "kind": r.kind,
          "sample": f"{r.sample}, {steps} timed steps of 1 PG iteration (loop body), {per:.2f} s"}
    line = {
        "metric": "voxel-iterations/sec (fwd+adjoint conv) and % of FP32/HBM roofline @1/2/4/8 B200",
        "impl": "reference", "value": value, "unit": "voxel-iterations/s", "n_gpus": world,
        "steps": steps, "warmup": a.warmup, "ms_per_step": per / steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{a.config}: {WORK[a.config]['desc']} (reference CPU path, "
                               f"{r.sample} per step)", "parallelism": f"{r.cores} cpu threads"},
        "cpu_baseline": cb,
        "e2e": {"value": value, "unit": "voxel-iterations/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)


if __name__ == "__main__":
    main()
