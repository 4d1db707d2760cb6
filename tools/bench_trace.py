"""Time compute_rho (trace + f0 + v-reduction) at a fixed step n:
   python tools/bench_trace.py wl3 40 [reps]
Builds the history with a short run, then times nufi_rho(n) with CUDA events."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2301_05581_b200 as nufi  # noqa: E402
from paper_2301_05581_b200.configs import ALGO_FLOPS, workload  # noqa: E402

name = sys.argv[1]
n = int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
w = workload(name)
s = torch.cuda.current_stream()
sim = nufi.Simulation(w.grid, w.ic, w.tau, n, stream=s.cuda_stream)
sim.run(n - 1)
h = sim.history.handle
rho = torch.empty(w.grid.n_nodes, dtype=torch.float64, device="cuda")
st = torch.empty(3, dtype=torch.float64, device="cuda")
ts = []
for r in range(reps + 1):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    h.call("nufi_rho", n, rho.data_ptr(), st.data_ptr(), None)
    e1.record(s)
    torch.cuda.synchronize()
    if r:
        ts.append(e0.elapsed_time(e1))
best = min(ts)
ps = w.grid.n_points * n
rate = ps / (best * 1e-3)
print(f"{name} n={n} env={ {k: v for k, v in os.environ.items() if k.startswith('NUFI_')} }: {best:.3f} ms  "
      f"{rate:.3e} point-steps/s  {rate * ALGO_FLOPS[w.grid.d] / 1e12:.2f} TF/s algorithmic")
