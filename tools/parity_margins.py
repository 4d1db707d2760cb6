"""Parity margins of the BASELINE runs against the unmodified reference's goldens: the largest
normwise rho / coefficient deviation over steps 0..50 and the largest relative W deviation up to
the checked horizon (tests/test_gpu_parity.py thresholds: 1e-10, 1e-10, 1e-6)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2301_05581_b200 as nufi  # noqa: E402
from paper_2301_05581_b200.configs import workload  # noqa: E402
from tests._util import golden, normwise  # noqa: E402

for name in sys.argv[1:] or ["wl1", "ts1", "sl1", "wl2", "wl3"]:
    g = golden(name)
    w = workload(name)
    N = len(g["W"]) - 1
    sim = nufi.Simulation(w.grid, w.ic, w.tau, N)
    res = sim.run()
    k = min(51, g["rho"].shape[0])
    r = normwise(res.rho[:k], g["rho"][:k]).max()
    c = normwise(sim.history.stacked().reshape(N + 1, -1)[:k], g["coeffs"][:k]).max()
    upto = 881 if name == "ts1" else N + 1
    relW = np.abs(res.W[:upto] - g["W"][:upto]) / np.abs(g["W"][:upto])
    print(f"{name}: rho {r:.2e}  coeffs {c:.2e}  W max rel (to step {upto - 1}) {relW.max():.2e}  "
          f"W rel at t_end {abs(res.W[-1] - g['W'][-1]) / abs(g['W'][-1]):.2e}")
