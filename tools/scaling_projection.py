"""Strong-scaling projection for the sharded run, measured on ONE GPU (this pool has one).

For G = 1, 2, 4, 8 ranks, rank 0's share of the velocity blocks is traced by a handle with
block_range(B, 0, G) through the real history of the run (nufi_rho_partials: trace + fused
block reduce of that rank's blocks), timed with the library's per-launch CUDA events at steps
spread over the run and fitted t(n) = a + b n; the per-step tail every rank runs
(nufi_step_finish_async: combine + Poisson / spline / append) is timed the same way.  The
allreduce of the (B Nx^d + 2B)-double block table is NOT measured (one GPU): it enters as an
assumed per-step latency, reported as a parameter with the projection at two values.

    python tools/scaling_projection.py wl3 [allreduce_us ...]  -> JSON line
"""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2301_05581_b200 as nufi  # noqa: E402
from paper_2301_05581_b200.configs import workload  # noqa: E402
from paper_2301_05581_b200.dist import block_range  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "wl3"
ar_us = [float(x) for x in sys.argv[2:]] or [20.0, 50.0]
w = workload(name)
g = w.grid
N = w.n_steps
B = 8

sim = nufi.Simulation(g, w.ic, w.tau, N, v_blocks=B)
sim.run()
stack = sim.history.stacked()
samples = sorted({1, N // 4, N // 2, 3 * N // 4, N})


def prof(h, fn):
    h.call("nufi_profiling", 1)
    fn()
    out = np.zeros(8)
    h.call("nufi_profiling_read", out.ctypes.data)
    h.call("nufi_profiling", 0)
    return out  # trace_ms, trace_launches, reduce_ms, reduce_launches, field_ms, field_launches, ps, 0


res = {"workload": name, "n_steps": N, "allreduce_us_assumed": ar_us, "ranks": {}}
for G in (1, 2, 4, 8):
    hist = nufi.PotentialHistory(g, w.tau, capacity=N + 1, v_blocks=B, block_range=block_range(B, 0, G))
    nufi.FlowContext(history=hist, ic=w.ic, tau=w.tau, grid=g)
    hist.load_stack(stack)
    h = hist.handle
    part = torch.zeros(int(h.lib.nufi_partials_len(h.h)), dtype=torch.float64, device="cuda")
    ev = ctypes.c_int64(0)
    ts = []
    for n in samples:
        prof(h, lambda: h.call("nufi_rho_partials", n, part.data_ptr(), ctypes.byref(ev)))  # warm
        o = prof(h, lambda: h.call("nufi_rho_partials", n, part.data_ptr(), ctypes.byref(ev)))
        ts.append((o[0] + o[2]) * 1e-3)
    b, a = np.polyfit(np.array(samples, float), np.array(ts), 1)
    # the per-step tail on the full (allreduced) table: time it on a copy of the history
    rho = torch.empty(g.n_nodes, dtype=torch.float64, device="cuda")
    for _ in range(2):  # the first call pays one-time launch setup
        hist.truncate(N)
        o = prof(h, lambda: h.call("nufi_step_finish_async", N, part.data_ptr(), rho.data_ptr(), None, None, None))
        torch.cuda.synchronize()
    t_field = o[4] * 1e-3
    trace_total = (N + 1) * a + b * N * (N + 1) / 2
    res["ranks"][G] = {"trace_fit_a_s": a, "trace_fit_b_s": b, "trace_run_s": trace_total, "tail_step_s": t_field,
                       "projected_run_s": {str(x): trace_total + (N + 1) * (t_field + (x * 1e-6 if G > 1 else 0))
                                           for x in ar_us}}
T1 = res["ranks"][1]["projected_run_s"][str(ar_us[0])]
for G in (2, 4, 8):
    res["ranks"][G]["projected_efficiency"] = {x: T1 / (G * res["ranks"][G]["projected_run_s"][x])
                                               for x in res["ranks"][G]["projected_run_s"]}
res["note"] = ("one-GPU measurement of rank 0's share (trace + fused block reduce) and of the per-step tail; "
               "the allreduce is an assumed latency, not measured (single-GPU pool)")
print(json.dumps(res))
