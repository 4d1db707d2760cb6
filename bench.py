"""bench.py -- backtraced point-steps/s (FP64) and wall time to t_end (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config ts1|wl1|sl1|wl2|wl3] [--impl reference]

A bench "step" is ONE FULL RUN of the configured workload to t_end (ts1: the
n = 0..1600 loop, P * N(N+1)/2 = 4.197e10 point-steps), all time steps on the
GPU: trace + f0 + v-reduction kernel, fixed-order block combine, single-CTA
Poisson / spline / append / energy kernel.  `value` = point-steps / device time
of the run (CUDA events on the library stream, outputs left in HBM; L2 flushed
between runs); `ms_per_step` = wall time to t_end of one run.  `e2e` = the same
metric through the public API call a user makes (Simulation(...).run() with
host numpy outputs: per-step rho / E / W / stats copied device -> host inside
the timed region).  `api_step` = the same again through the reference-shaped
per-step loop (compute_rho + advance per step).  N > 1 ranks
(torchrun): velocity-block sharding (paper_2301_05581_b200/dist.py; the
`parallelism` key records which exchange ran), device time = max over ranks.

`--impl reference` and `cpu_baseline`: the UNMODIFIED reference (vpflow, numba
backend, every host thread), pip-installed into the git-ignored baseline/_ref,
timed on this host at steps spread over the run with a t(n) = a + b*n fit
extrapolated to t_end (ReferenceTimer); rank 0 only.  When
baseline/_ref is absent, the oracle port (oracle/: C trace + numpy) stands in
(kind = "port").
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="ts1")
    ap.add_argument("--impl", default="nufi", choices=["nufi", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-api-step", action="store_true", help="skip the per-step drop-in loop leg")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="bounded CPU sample length")
    ap.add_argument("--force-dist", action="store_true",
                    help="test hook: take the multi-rank (NCCL) code path even with one rank")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# clocks (nvidia-smi sampled during the timed region)
# ---------------------------------------------------------------------------

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _loop(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                self.rows.append([x.strip() for x in out.stdout.strip().split(",")])
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._t = threading.Thread(target=self._loop, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        sm = [float(r[0]) for r in self.rows if len(r) >= 8 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 8 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            if len(r) >= 8:
                for nm, v in zip(names, r[4:8]):
                    if v.lower() == "active":
                        reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


# ---------------------------------------------------------------------------
# CPU baseline: the unmodified reference (vpflow, numba backend) on the host cores
# ---------------------------------------------------------------------------

METRIC = "backtraced point-steps/s (FP64) & wall time to t_end"  # both arms print exactly this
REF_DIR = os.path.join(ROOT, "baseline", "_ref")  # pip install --target of /root/reference/pkg (git-ignored)


def cpu_model() -> str:
    try:
        return [l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name")][0]
    except Exception:  # pragma: no cover
        return "unknown"


def import_reference():
    """The reference package as installed into baseline/_ref (unmodified; numba backend, every
    host thread).  None when it is not installed or numba is unavailable."""
    if not os.path.isdir(os.path.join(REF_DIR, "vpflow")):
        return None
    from oracle.oracle import max_threads

    os.environ.setdefault("NUMBA_NUM_THREADS", str(max_threads()))
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    try:
        import vpflow.density  # noqa: F401
        import vpflow.kernels as K
        if K.get_backend() != "numba":
            return None
        return sys.modules["vpflow"]
    except Exception:
        return None


class ReferenceTimer:
    """Times the reference's own per-step path (density.compute_rho, density.py:72-91 ->
    kernels.trace_backward numba, kernels.py:184-387; then solve_poisson / fit_spline /
    electric_energy / eval_E_many, the §3.1 tail) at steps spread over the run, and fits
    t(n) = a + b*n to extrapolate the whole run to t_end.

    The history is the reference's own PotentialHistory holding the golden slabs of this
    config (steps 0..50 of the unmodified reference, tests/golden; wl3 may use the wl3r
    slabs, same 16^3 x-grid) repeated up to step N: the numba trace's cost does not depend
    on the coefficient values.  Grids whose full
    compute_rho at step N would exceed ~2.5e9 point-steps (wl3) take the survey's plan:
    a = compute_rho at n = 0 on the full grid (f0 + copies + reduce, measured once),
    b from trace_backward on a node slice at the sample steps."""

    SLICE_LIMIT = 2.5e9

    def __init__(self, name: str):
        from paper_2301_05581_b200.configs import workload

        vp = import_reference()
        if vp is None:
            raise RuntimeError("reference not installed in baseline/_ref")
        from vpflow import density, kernels, poisson, spline
        from vpflow.flow import FlowContext
        from vpflow.grids import GridSpec, x_node_matrix
        from vpflow.initial import InitialCondition, VelocityProfile

        self.vp = dict(density=density, kernels=kernels, poisson=poisson, spline=spline)
        w = workload(name)
        self.w = w
        g = GridSpec(d=w.grid.d, L=w.grid.L, Nx=w.grid.Nx, Nv=w.grid.Nv, vmax=w.grid.vmax)
        ic = InitialCondition(benchmark=w.ic.benchmark, d=w.ic.d, L=w.ic.L, alpha=w.ic.alpha, k=w.ic.k, v0=w.ic.v0,
                              profiles=tuple(VelocityProfile(centers=p.centers, weights=p.weights, power=p.power)
                                             for p in w.ic.profiles))
        self.g = g
        N = w.n_steps
        # any reference history on the same x-grid will do (the trace cost is value-independent):
        # the config's own golden, else the reduced-velocity golden of the same Nx^d
        src = [f for f in (name, {"wl3": "wl3r"}.get(name)) if f and
               os.path.exists(os.path.join(ROOT, "tests", "golden", f"{f}.npz"))]
        z = np.load(os.path.join(ROOT, "tests", "golden", f"{src[0]}.npz"))
        slabs = z["coeffs"].reshape((-1,) + g.shape_x)
        hist = spline.PotentialHistory(g, w.tau)
        for m in range(N + 1):
            hist.append(spline.SplineField(grid=g, coeffs=np.ascontiguousarray(slabs[m % len(slabs)])))
        self.hist = hist
        self.ctx = FlowContext(history=hist, ic=ic, tau=w.tau, grid=g)
        self.Xn = x_node_matrix(g)
        P = g.n_nodes * g.n_cells
        self.P = P
        self.slice = P * N > self.SLICE_LIMIT
        self.samples = sorted({1, max(1, N // 4), max(1, N // 2), max(1, 3 * N // 4), N})
        self.a_full = None
        if self.slice:
            # node-aligned slice of the quadrature points (density.py:32-42 order)
            from vpflow.grids import v_mid_matrix

            nodes = max(1, g.n_nodes // 64)
            X = np.repeat(self.Xn[:nodes], g.n_cells, axis=0)
            V = np.tile(v_mid_matrix(g), (nodes, 1))
            self.slice_pts = (X, V)
        # JIT warm-up of the numba trace for this d (not timed)
        Xw = np.zeros((8, g.d))
        Vw = np.zeros((8, g.d))
        kernels.trace_backward(hist.stacked()[:2], g.L, 2, w.tau, Xw, Vw, False)
        self.cores = int(__import__("numba").get_num_threads())

    def _tail(self, r):
        P, S, K = self.vp["poisson"], self.vp["spline"], self.vp["kernels"]
        t0 = time.perf_counter()
        phi, spec = P.solve_poisson(r.density)
        fit = S.fit_spline(phi, self.g)
        P.electric_energy(spec)
        K.eval_E_many(fit.coeffs, self.g.L, self.Xn)
        return time.perf_counter() - t0

    def one_pass(self) -> dict:
        """compute_rho (or the slice trace) at every sample step + one tail; returns the fit."""
        D, K = self.vp["density"], self.vp["kernels"]
        t_pass = time.perf_counter()
        ts = []
        tail = 0.0
        if not self.slice:
            for n in self.samples:
                t0 = time.perf_counter()
                r = D.compute_rho(self.ctx, n)
                ts.append(time.perf_counter() - t0)
            tail = self._tail(r)
            b, a = np.polyfit(np.array(self.samples, float), np.array(ts), 1)
        else:
            if self.a_full is None:
                t0 = time.perf_counter()
                r = D.compute_rho(self.ctx, 0)
                self.a_full = time.perf_counter() - t0
                self.tail_full = self._tail(r)
            X0, V0 = self.slice_pts
            stack = self.hist.stacked()
            for n in self.samples:
                X, V = X0.copy(), V0.copy()
                t0 = time.perf_counter()
                K.trace_backward(stack[:n], self.g.L, n, self.w.tau, X, V, False)
                ts.append(time.perf_counter() - t0)
            bs, _ = np.polyfit(np.array(self.samples, float), np.array(ts), 1)
            b = bs * self.P / X0.shape[0]
            a = self.a_full
            tail = self.tail_full
        N = self.w.n_steps
        T = (N + 1) * (a + tail) + b * N * (N + 1) / 2
        return {"value": self.w.point_steps / T, "a_s": a, "b_s": b, "tail_s": tail, "T_run_s": T,
                "pass_s": time.perf_counter() - t_pass,
                "sample_ps": (self.P if not self.slice else X0.shape[0]) * sum(self.samples)}

    def describe(self, fit: dict) -> str:
        how = ("compute_rho" if not self.slice else
               f"compute_rho at n=0 (full grid) + trace_backward on a 1/64 node slice")
        return (f"{self.w.name}: unmodified reference (vpflow, numba backend, {self.cores} threads, {cpu_model()}); "
                f"{how} at n = {self.samples} of {self.w.n_steps} + one Poisson/spline/E tail; "
                f"fit t(n) = a + b*n: a = {fit['a_s'] * 1e3:.2f} ms, b = {fit['b_s'] * 1e6:.2f} us/step "
                f"({self.P / fit['b_s']:.3e} point-steps/s marginal), tail = {fit['tail_s'] * 1e3:.2f} ms; "
                f"extrapolated to t_end: {fit['T_run_s']:.1f} s for {self.w.point_steps:.3e} point-steps")


def cpu_sample_port(name: str, seconds: float):
    """Fallback when the reference is not installed: the oracle port (C trace with every host
    thread + numpy, oracle/) from n = 2 on, until `seconds` elapse."""
    from oracle import oracle as O
    from paper_2301_05581_b200.configs import workload

    w = workload(name)
    c = O.case(name)
    threads = O.max_threads()
    run = O.OracleRun(c, threads=threads)
    run.step(0)  # warm-up (not timed)
    run.step(1)
    t0 = time.perf_counter()
    n = 2
    while n <= w.n_steps:
        run.step(n)
        n += 1
        if time.perf_counter() - t0 > seconds:
            break
    dt = time.perf_counter() - t0
    ps = c.n_nodes * c.n_cells * (sum(range(2, n)))
    return {"value": ps / dt, "unit": "point-steps/s", "cores": threads, "kind": "port",
            "sample": f"{name} steps 2..{n - 1} of {w.n_steps} (whole loop: trace + f0 + reduce + Poisson/spline), "
                      f"{ps:.3e} point-steps in {dt:.1f} s; oracle C trace (OpenMP) + numpy (reference not installed)",
            "seconds": dt}


def cpu_baseline(name: str, seconds: float) -> dict:
    """One bounded sample of the reference's CPU path (rank 0, N = 1)."""
    try:
        rt = ReferenceTimer(name)
        fits = [rt.one_pass()]
        t0 = time.perf_counter()
        while time.perf_counter() - t0 < seconds and len(fits) < 8:
            fits.append(rt.one_pass())
    except Exception:  # the reference cannot run here: the oracle port stands in (kind "port")
        return cpu_sample_port(name, seconds)
    fit = sorted(fits, key=lambda f: f["value"])[len(fits) // 2]
    return {"value": fit["value"], "unit": "point-steps/s", "cores": rt.cores, "kind": "reference",
            "extrapolated": True, "sample": rt.describe(fit) + f"; median of {len(fits)} passes"}


def reference_arm(args, rank: int):
    """--impl reference: the reference's own CPU path on this host (rank 0 only).  A bench step
    is one pass of ReferenceTimer (compute_rho at 5 steps spread over the run + the tail);
    `ms_per_step` is that pass's measured wall time, `value` the whole-run rate the pass's
    t(n) = a + b*n fit extrapolates to t_end (labelled)."""
    from paper_2301_05581_b200.configs import workload

    if rank != 0:
        return
    w = workload(args.config)
    try:
        rt = ReferenceTimer(args.config)
    except Exception as exc:
        rt = None
        why = str(exc)
    if rt is None:  # the oracle port, same line shape
        per = max(2.0, min(20.0, 150.0 / max(1, args.steps + args.warmup)))
        for _ in range(args.warmup):
            cpu_sample_port(args.config, per / 4)
        runs = [cpu_sample_port(args.config, per) for _ in range(args.steps)]
        v = statistics.median(r["value"] for r in runs)
        ms = 1e3 * statistics.mean(r["seconds"] for r in runs)
        cb = {"value": v, "unit": "point-steps/s", "cores": runs[-1]["cores"], "kind": "port",
              "sample": runs[-1]["sample"] + f" ({why})"}
    else:
        for _ in range(args.warmup):
            rt.one_pass()
        fits = [rt.one_pass() for _ in range(args.steps)]  # a failure here is a real error: no silent switch
        v = statistics.median(f["value"] for f in fits)
        ms = 1e3 * statistics.mean(f["pass_s"] for f in fits)
        mid = sorted(fits, key=lambda f: f["value"])[len(fits) // 2]
        cb = {"value": v, "unit": "point-steps/s", "cores": rt.cores, "kind": "reference", "extrapolated": True,
              "sample": rt.describe(mid)}
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "point-steps/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (deterministic BASELINE config, no dataset)",
        "config": {"workload": args.config, "description": w.description, "point_steps_per_run": w.point_steps},
        "cpu_baseline": cb,
        "e2e": {"value": v, "unit": "point-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": ("a bench step is one measured sampling pass (ms_per_step = its wall time); value = the "
                 "point-steps of the whole run to t_end / the run time extrapolated from that pass's "
                 "t(n) = a + b*n fit (cpu_baseline.sample)"),
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

def smem_roofline(torch, dev, d, trace_ps, trace_ms):
    """The co-limiter of the gather stencil: algorithmic coefficient bytes (4^d doubles
    per point-step) over the shared-memory crossbar, 128 B/clk/SM
    (B300_MICROARCH.md LDS/STS table; no measured B200 figure exists) x SMs x max clock."""
    from paper_2301_05581_b200.configs import ALGO_BYTES

    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    mhz = 1965.0
    try:
        mhz = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["sm_max_mhz"])
    except Exception:
        pass
    peak = 128.0 * sms * mhz * 1e6 / 1e9
    achieved = ALGO_BYTES[d] * trace_ps / (trace_ms * 1e-3) / 1e9 if trace_ms else None
    return {"bound": "smem", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak if achieved else None,
            "peak_source": f"nominal: 128 B/clk/SM x {sms} SMs x {mhz:.0f} MHz",
            "note": ("d=1 reads 24 B/point-step (A,B,C cell polynomial) against the 32 B algorithmic figure; "
                     "random late-time gathers cost ~3.75 wavefronts per 8-byte warp load (ncu, profiles/)")
            if d == 1 else
            (f"d={d} reads exactly the {ALGO_BYTES[d]} B of the 4^d stencil per point-step, conflict-free "
             "(2.0 wavefronts per 8-byte warp load, ncu, profiles/); co-bound with the FP64 pipe")}


def api_step_leg(nufi, w, dev, reps: int) -> dict:
    """The drop-in loop a vpflow caller writes: per step
    r = compute_rho(ctx, n); up = advance(ctx, r.density) -- the whole run to t_end,
    wall-clocked, every step's rho / W / E / coefficients reaching the host.  Two variants:
    W read every step (one host wait per step), and every result read after the loop (the
    calls only enqueue; pending.py)."""
    g = w.grid

    def loop(read_each):
        hist = nufi.PotentialHistory(g, w.tau, capacity=w.n_steps + 1, device=dev)
        ctx = nufi.FlowContext(history=hist, ic=w.ic, tau=w.tau, grid=g)
        t0 = time.perf_counter()
        res = []
        for n in range(w.n_steps + 1):
            r = nufi.compute_rho(ctx, n)
            up = nufi.advance(ctx, r.density)
            if read_each:
                _ = up.W
            res.append((r, up))
        for r, up in res:  # every output on the host
            _ = (r.density.values, r.f_max, up.W, up.E)
        return time.perf_counter() - t0

    out = {}
    for key, each in (("read_each_step", True), ("read_at_end", False)):
        times = [loop(each) for _ in range(reps + 1)][1:]  # first pass warms up
        t = float(np.median(times))
        out[key] = {"value": w.point_steps / t, "wall_s_to_t_end": t}
    return {"value": out["read_each_step"]["value"], "unit": "point-steps/s", "runs": reps, **out,
            "api": "for n in 0..N: r = compute_rho(ctx, n); up = advance(ctx, r.density) (host outputs)"}


def flush_l2(torch, buf):
    buf.add_(1.0)  # 256 MiB write > 126 MB L2


def gpu_arm(args, rank: int, world: int):
    dist_mode = world > 1 or args.force_dist
    import ctypes

    import torch

    import paper_2301_05581_b200 as nufi
    from paper_2301_05581_b200 import _lib
    from paper_2301_05581_b200.configs import ALGO_FLOPS, workload

    dev = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(dev)
    w = workload(args.config)
    g = w.grid
    N = w.n_steps
    steps_per_run = N + 1
    lib = _lib.load()
    flush = torch.empty(32 * 1024 * 1024, dtype=torch.float64, device="cuda")
    # one dedicated (non-default) stream for the library, the collectives, the L2 flush and
    # the timing events: the events then bracket exactly the work they time
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)

    if dist_mode:
        import torch.distributed as dist

        from paper_2301_05581_b200.dist import DistributedSimulation

        sim = DistributedSimulation(g, w.ic, w.tau, N)
    else:
        sim = nufi.Simulation(g, w.ic, w.tau, N, device=dev, stream=stream.cuda_stream)
    dev_out = dict(rho=torch.empty((steps_per_run, g.n_nodes), dtype=torch.float64, device="cuda"),
                   E=torch.empty((steps_per_run, g.n_nodes, g.d), dtype=torch.float64, device="cuda"),
                   W=torch.empty(steps_per_run, dtype=torch.float64, device="cuda"),
                   stats=torch.empty((steps_per_run, 3), dtype=torch.float64, device="cuda"))

    def one_run():
        sim.history.truncate(0)
        sim.run(outputs=dev_out)

    def barrier():
        if dist_mode:
            torch.distributed.barrier()

    for _ in range(args.warmup):
        one_run()
    torch.cuda.synchronize()

    # ---- timed runs: device time per run, L2 flushed between runs ----
    times = []
    wall = []
    with ClockSampler(dev) as clocks:
        for _ in range(args.steps):
            flush_l2(torch, flush)
            barrier()
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter()
            e0.record(stream)
            one_run()
            e1.record(stream)
            torch.cuda.synchronize()
            barrier()
            wall.append(time.perf_counter() - t0)
            times.append(e0.elapsed_time(e1) / 1e3)
    t_dev = float(np.sum(times))
    if dist_mode:
        tt = torch.tensor([t_dev], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        t_dev = float(tt.item())
    ps_run = w.point_steps
    value = args.steps * ps_run / t_dev
    ms_per_run = 1e3 * t_dev / args.steps

    # ---- e2e: the public API with host outputs (per-step D2H inside the timed region) ----
    e2e_times = []
    d2h = steps_per_run * (g.n_nodes * (1 + g.d) + 4) * 8
    h2d = ctypes.sizeof(_lib.NufiConfig)  # the run's configuration descriptor (nufi_create)
    if not dist_mode:
        for i in range(args.warmup + args.steps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            res = nufi.Simulation(g, w.ic, w.tau, N, device=dev).run()
            _ = float(res.W[-1])  # host-side read of the result
            if i >= args.warmup:
                e2e_times.append(time.perf_counter() - t0)
        e2e_value = args.steps * ps_run / float(np.sum(e2e_times))
    else:
        # every rank: DistributedSimulation(...).run() -> host arrays; max over ranks
        from paper_2301_05581_b200.dist import DistributedSimulation

        for i in range(args.warmup + args.steps):
            torch.cuda.synchronize()
            torch.distributed.barrier()
            t0 = time.perf_counter()
            res = DistributedSimulation(g, w.ic, w.tau, N).run()
            _ = float(res["W"][-1])
            t_run = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device="cuda")
            torch.distributed.all_reduce(t_run, op=torch.distributed.ReduceOp.MAX)
            if i >= args.warmup:
                e2e_times.append(float(t_run.item()))
        e2e_value = args.steps * ps_run / float(np.sum(e2e_times))

    # ---- the reference-shaped per-step loop: compute_rho + advance per
    # step through the public API, host outputs, W read every step ----
    api_step = None
    if not dist_mode and not args.no_api_step:
        reps = 1 if w.point_steps > 1e11 else max(1, min(args.steps, 3))  # wl3: one pass of each (~9 s)
        api_step = api_step_leg(nufi, w, dev, reps)

    # ---- roofline: one additional identical run with per-launch CUDA events ----
    h = sim.history.handle
    lib.nufi_profiling(h.h, 1)
    one_run()
    prof = np.zeros(8)
    lib.nufi_profiling_read(h.h, prof.ctypes.data)
    lib.nufi_profiling(h.h, 0)
    trace_ms, trace_launches, reduce_ms, reduce_launches, field_ms, field_launches, trace_ps, _ = prof
    launches_per_run = int(trace_launches + reduce_launches + field_launches)
    peak = ctypes.c_double()
    peak_ms = ctypes.c_double()
    lib.nufi_fp64_peak(dev, ctypes.byref(peak), ctypes.byref(peak_ms))
    achieved = ALGO_FLOPS[g.d] * trace_ps / (trace_ms * 1e-3) / 1e12
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath)).get(args.config)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    peak_nominal = sms * 64 * 2 * 1.965e9 / 1e12  # 64 DFMA / clk / SM at the 1965 MHz max clock
    roofline = {
        "bound": "fp64", "achieved": achieved, "peak": peak.value, "unit": "TFLOP/s",
        "frac": achieved / peak.value if peak.value else None,
        "peak_nominal": peak_nominal, "frac_nominal": achieved / peak_nominal,
        "traffic": traffic["traffic"] if traffic else None,
        "traffic_detail": traffic,
        "kernel": ("run_1d_kernel (persistent: all steps, trace + grid barrier + field tail)" if g.d == 1
                   else f"trace_rho_kernel<{g.d}>"), "algo_flops_per_point_step": ALGO_FLOPS[g.d],
        "trace_launches": int(trace_launches), "trace_ms_per_launch": trace_ms / max(1, trace_launches),
        "trace_share_of_run": trace_ms / (trace_ms + reduce_ms + field_ms) if trace_ms else None,
        "reduce_ms_per_launch": reduce_ms / reduce_launches if reduce_launches else None,
        "field_ms_per_launch": field_ms / field_launches if field_launches else None,
        "peak_source": "measured in-run: DFMA-chain kernel (nufi_fp64_peak); MEASURED_PEAKS.json has no FP64 entry",
        "secondary": smem_roofline(torch, dev, g.d, trace_ps, trace_ms),
        "note": "tensor cores not applicable (FP64 gather-stencil, no dense contraction); HBM ~0 (history L2-resident)",
    }

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args.config, args.cpu_seconds)

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": value, "unit": "point-steps/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_run, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (deterministic BASELINE config; no dataset)",
            "config": {"workload": args.config, "description": w.description, "time_steps_per_run": steps_per_run,
                       "point_steps_per_run": ps_run, "l2": "flushed (256 MiB write) between timed runs",
                       "parallelism": (f"v-block sharding x{world}, exchange: {sim.exchange}" if dist_mode
                                       else "single GPU")},
            "wall_s_to_t_end": ms_per_run / 1e3,
            "e2e": {"value": e2e_value, "unit": "point-steps/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h,
                    "inputs": "a run's only input is its nufi_config descriptor (host struct, copied into the "
                              "handle and kernel parameters inside the timed region); NuFI keeps no per-point "
                              "state, and every per-time-step output row (rho, E, W, stats) is copied back",
                    "api": ("Simulation(grid, ic, tau, N).run()" if not dist_mode else
                            "DistributedSimulation(grid, ic, tau, N).run() on every rank (max over ranks)")
                           + " -> host numpy rho/E/W/stats per time step"},
            "api_step": api_step,
            "gpu_launches": launches_per_run * args.steps,
            "roofline": roofline,
            "cpu_baseline": None if cpu is None else {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample",
                                                                           "extrapolated") if k in cpu},
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        reference_arm(args, rank)
        return
    dist_mode = world > 1 or args.force_dist
    if dist_mode:
        import torch
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29511")
        os.environ.setdefault("RANK", "0")
        os.environ.setdefault("WORLD_SIZE", "1")
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
        dist.init_process_group("nccl")
    gpu_arm(args, rank, world)
    if dist_mode:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
