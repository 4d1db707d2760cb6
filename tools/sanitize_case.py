"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck / synccheck):
d = 1 run (persistent kernel) + single steps + parity trace, d = 2 / 3 runs, the sweep."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2301_05581_b200 as nufi  # noqa: E402
from paper_2301_05581_b200.configs import workload  # noqa: E402

for name, N in (("kat_wl", 12), ("rag1", 6), ("tiny2", 5), ("tiny3", 4), ("rag3", 4)):
    w = workload(name)
    sim = nufi.Simulation(w.grid, w.ic, w.tau, N)
    res = sim.run()
    st = nufi.Simulation(w.grid, w.ic, w.tau, 2)
    for _ in range(3):
        st.step()
    m = nufi.conserved_moments(sim.ctx, N - 1)
    X = np.random.default_rng(0).uniform(0, w.grid.L, (37, w.grid.d))
    V = np.random.default_rng(1).uniform(-w.grid.vmax, w.grid.vmax, (37, w.grid.d))
    nufi.trace_backward(sim.history, N - 1, X, V, True, nufi.TRACE_PARITY)
    nufi.trace_backward(sim.history, N - 1, X, V, False, nufi.TRACE_FAST)
    print(name, "W[-1]", res.W[-1], "l1", m.l1)
print("sanitize case done")
