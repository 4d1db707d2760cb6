"""Time one compute_rho launch (trace + f0 + v-reduction) at step n on the reference's own
history (tests/golden/<name>.npz coefficients), so experiment builds that change which points
are traced still see the real slabs:  python tools/trace_golden.py wl3 50 [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2301_05581_b200 as nufi  # noqa: E402
from paper_2301_05581_b200.configs import ALGO_FLOPS, workload  # noqa: E402

name, n = sys.argv[1], int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
w = workload(name)
coeffs = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", f"{name}.npz"))["coeffs"]
hist = nufi.PotentialHistory(w.grid, w.tau, capacity=coeffs.shape[0] + 1)
nufi.FlowContext(history=hist, ic=w.ic, tau=w.tau, grid=w.grid)
hist.load_stack(coeffs[: n + 1])
h = hist.handle
s = torch.cuda.current_stream()
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
rate = w.grid.n_points * n / (best * 1e-3)
print(f"{name} n={n} lib={os.environ.get('NUFI_LIB_VARIANT', 'base')}: {best:.3f} ms  {rate:.3e} point-steps/s  "
      f"{rate * ALGO_FLOPS[w.grid.d] / 1e12:.2f} TF/s  rho[:3]={rho[:3].tolist()}")
