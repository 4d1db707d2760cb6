"""Finer split of the e2e overhead of one public run (wl1): handle create, bind (f0 + rho_bar),
run, result read, destroy -- host wall times, 5 repetitions after 2 warm-ups."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2301_05581_b200 as nufi  # noqa: E402
from paper_2301_05581_b200.configs import workload  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "wl1"
w = workload(name)
for it in range(7):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    hist = nufi.PotentialHistory(w.grid, w.tau, capacity=w.n_steps + 1, device=0)
    t1 = time.perf_counter()
    ctx = nufi.FlowContext(history=hist, ic=w.ic, tau=w.tau, grid=w.grid)
    t2 = time.perf_counter()
    sim = nufi.Simulation.__new__(nufi.Simulation)
    sim.grid, sim.n_steps, sim.history, sim.ctx = w.grid, w.n_steps, hist, ctx
    res = sim.run()
    t3 = time.perf_counter()
    _ = float(res.W[-1])
    del sim, ctx, hist, res
    t4 = time.perf_counter()
    if it >= 2:
        print(f"{name}: create {1e6*(t1-t0):.0f} us  bind {1e6*(t2-t1):.0f} us  run {1e6*(t3-t2):.0f} us  "
              f"destroy {1e6*(t4-t3):.0f} us  total {1e3*(t4-t0):.3f} ms", flush=True)
