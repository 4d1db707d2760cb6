"""Host cost of the reference-shaped per-step loop (compute_rho + advance), wl1: wall time of the
loop with results read at the end, and a cProfile of one pass (top entries by own time)."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2301_05581_b200 as nufi  # noqa: E402
from paper_2301_05581_b200.configs import workload  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "wl1"
w = workload(name)


def loop():
    hist = nufi.PotentialHistory(w.grid, w.tau, capacity=w.n_steps + 1)
    ctx = nufi.FlowContext(history=hist, ic=w.ic, tau=w.tau, grid=w.grid)
    us = []
    for n in range(w.n_steps + 1):
        r = nufi.compute_rho(ctx, n)
        us.append(nufi.advance(ctx, r.density))
    return [u.W for u in us]


for _ in range(2):
    loop()
torch.cuda.synchronize()
t0 = time.perf_counter()
loop()
print(f"{name}: loop {1e3 * (time.perf_counter() - t0):.2f} ms for {w.n_steps + 1} steps")
pr = cProfile.Profile()
pr.enable()
loop()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
