"""Run one NuFI simulation (for ncu captures):  python tools/profile_run.py ts1 [n_last]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2301_05581_b200 as nufi  # noqa: E402
from paper_2301_05581_b200.configs import workload  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "ts1"
w = workload(name)
n_last = int(sys.argv[2]) if len(sys.argv) > 2 else w.n_steps
sim = nufi.Simulation(w.grid, w.ic, w.tau, n_last)
res = sim.run()
print(name, "steps", n_last + 1, "W[-1]", res.W[-1])
