"""Time full NuFI runs with CUDA events:  python tools/time_run.py ts1 [n_last] [reps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2301_05581_b200 as nufi  # noqa: E402
from paper_2301_05581_b200.configs import workload  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "ts1"
w = workload(name)
n_last = int(sys.argv[2]) if len(sys.argv) > 2 else w.n_steps
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
s = torch.cuda.current_stream()
sim = nufi.Simulation(w.grid, w.ic, w.tau, n_last, stream=s.cuda_stream)
out = dict(W=torch.empty(n_last + 1, dtype=torch.float64, device="cuda"))
ts = []
for r in range(reps + 1):
    sim.history.truncate(0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    sim.run(outputs=out)
    e1.record(s)
    torch.cuda.synchronize()
    if r:
        ts.append(e0.elapsed_time(e1))
ps = w.grid.n_points * n_last * (n_last + 1) // 2
best = min(ts)
print(f"{name} n_last={n_last} stages={os.environ.get('NUFI_D1_STAGES', 'default')}: {best:.2f} ms "
      f"({ps / best * 1e3:.3e} point-steps/s)  W[-1]={out['W'][-1].item():.6e}")
