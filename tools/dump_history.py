"""Run a workload on the GPU and save its coefficient history (for offline analysis)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2301_05581_b200 as nufi  # noqa: E402
from paper_2301_05581_b200.configs import workload  # noqa: E402

name = sys.argv[1]
w = workload(name)
sim = nufi.Simulation(w.grid, w.ic, w.tau, w.n_steps)
sim.run()
os.makedirs("gpurun_out", exist_ok=True)
np.save(f"gpurun_out/{name}_hist.npy", sim.history.stacked())
print("saved", sim.history.stacked().shape)
