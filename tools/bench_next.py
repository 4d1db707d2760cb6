"""Measurements for the SURVEY.md §8(f) "next" rows, on the GPU, each beside its CPU restatement
(oracle, every host thread) on the same box:

  (f)1 Psi observable sweep (nufi_moments / density.conserved_moments): point-steps/s at step n
  (f)2 point-level Psi (nufi_trace FAST / PARITY, device buffers; flow.psi_batch): point-steps/s
  (f)3 VPHIST01 checkpoint save + load of a full history: MB/s
  (f)4 FP32-history run (PotentialHistory(dtype=float32)): whole-run rate vs FP64

  python tools/bench_next.py > profiles/r01_next_rows.json
Device times are CUDA events around the call on its stream (warm-up first); one JSON document.
"""
import ctypes
import json
import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2301_05581_b200 as nufi  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2301_05581_b200 import _lib  # noqa: E402
from paper_2301_05581_b200.configs import ALGO_FLOPS, workload  # noqa: E402


def dev_time(fn, reps=3):
    s = torch.cuda.current_stream()
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        fn()
        e1.record(s)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    return min(ts)


def fp64_peak():
    peak, ms = ctypes.c_double(), ctypes.c_double()
    _lib.load().nufi_fp64_peak(0, ctypes.byref(peak), ctypes.byref(ms))
    return peak.value


def history_for(name, n):
    w = workload(name)
    s = torch.cuda.current_stream()
    sim = nufi.Simulation(w.grid, w.ic, w.tau, n, stream=s.cuda_stream)
    sim.run()
    return w, sim


def sweep(name, n, peak):
    w, sim = history_for(name, n)
    ctx = sim.ctx
    t = dev_time(lambda: nufi.conserved_moments(ctx, n))
    ps = w.grid.n_nodes * w.grid.n_cells * (n + 1)
    rate = ps / t
    return {"row": "(f)1 Psi observable sweep (nufi_moments)", "workload": name, "step": n, "seconds": t,
            "point_steps": ps, "point_steps_per_s": rate,
            "fp64_frac": rate * ALGO_FLOPS[w.grid.d] / (peak * 1e12)}


def point_trace(name, n, M, peak):
    w, sim = history_for(name, n)
    d = w.grid.d
    rng = np.random.default_rng(5)
    x0 = rng.uniform(0.0, w.grid.L, (M, d))
    v0 = rng.uniform(-w.grid.vmax, w.grid.vmax, (M, d))
    X = torch.tensor(x0, device="cuda")
    V = torch.tensor(v0, device="cuda")
    out = {"row": "(f)2 point-level Psi (nufi_trace)", "workload": name, "step": n, "points": M}
    for mode_name, mode in (("fast", nufi.TRACE_FAST), ("parity", nufi.TRACE_PARITY)):
        def call():  # in place on the device buffers (positions keep evolving; rate only)
            sim.history.handle.call("nufi_trace", n, X.data_ptr(), V.data_ptr(), M, 1, mode, None)
        t = dev_time(call)
        rate = M * (n + 1) / t
        out[mode_name] = {"seconds": t, "point_steps_per_s": rate,
                          "fp64_frac": rate * ALGO_FLOPS[d] / (peak * 1e12)}
    # CPU: the oracle's C restatement of the numba trace, every host thread, on a sample
    Ms = min(M, 200_000 if d == 1 else (20_000 if d == 2 else 4_000))
    stack = sim.history.stacked()
    Xc, Vc = x0[:Ms].copy(), v0[:Ms].copy()
    threads = O.max_threads()
    t0 = time.perf_counter()
    O.trace_backward(stack, w.grid.L, n, w.tau, Xc, Vc, True, threads=threads)
    tc = time.perf_counter() - t0
    out["cpu_oracle"] = {"points": Ms, "threads": threads, "seconds": tc, "point_steps_per_s": Ms * (n + 1) / tc}
    return out


def checkpoint(name):
    w, sim = history_for(name, workload(name).n_steps)
    with tempfile.TemporaryDirectory() as tmp:
        path = os.path.join(tmp, "h.vphist")
        t0 = time.perf_counter()
        sim.history.save(path)
        ts = time.perf_counter() - t0
        size = os.path.getsize(path)
        t0 = time.perf_counter()
        h2 = nufi.PotentialHistory.load(path, device=0)
        torch.cuda.synchronize()
        tl = time.perf_counter() - t0
    return {"row": "(f)3 VPHIST01 checkpoint", "workload": name, "bytes": size, "save_s": ts,
            "save_MB_per_s": size / ts / 1e6, "load_s": tl, "load_MB_per_s": size / tl / 1e6,
            "rows": len(h2), "note": "host file I/O (tmpfs/overlay on the GPU box) + one H2D/D2H copy"}


def fp32_run(name):
    w = workload(name)
    s = torch.cuda.current_stream()
    res = {}
    for dt in (np.float64, np.float32):
        sim = nufi.Simulation(w.grid, w.ic, w.tau, w.n_steps, stream=s.cuda_stream, dtype=dt)
        out = dict(W=torch.empty(w.n_steps + 1, dtype=torch.float64, device="cuda"))

        def run():
            sim.history.truncate(0)
            sim.run(outputs=out)
        t = dev_time(run, reps=2)
        res[np.dtype(dt).name] = {"seconds": t, "point_steps_per_s": w.point_steps / t,
                                  "W_end": float(out["W"][-1].item())}
    return {"row": "(f)4 FP32 history run", "workload": name, **res}


def main():
    torch.cuda.set_device(0)
    peak = fp64_peak()
    doc = {"what": __doc__.strip().splitlines()[0], "fp64_peak_TFs_measured": peak,
           "device": torch.cuda.get_device_name(0), "results": []}
    doc["results"].append(sweep("ts1", 800, peak))
    doc["results"].append(sweep("wl3", 40, peak))
    doc["results"].append(point_trace("ts1", 400, 1 << 20, peak))
    doc["results"].append(point_trace("wl2", 80, 1 << 20, peak))
    doc["results"].append(point_trace("wl3", 40, 1 << 18, peak))
    doc["results"].append(checkpoint("wl3"))
    doc["results"].append(fp32_run("ts1"))
    doc["results"].append(fp32_run("wl2"))
    print(json.dumps(doc, indent=1))


if __name__ == "__main__":
    main()
