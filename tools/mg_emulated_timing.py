"""Per-step cost of the fused multi-rank exchange, measured with emulated ranks on one GPU:
the same total work traced either as one rank or as G virtual ranks.

  d = 1: the persistent run kernel with G rank groups of CTAs in one launch (nufi_run);
  d >= 2: nufi_mg_step_async per step (block sums stored into every virtual rank's table +
          arrival counters, the tail waiting on them), against the single-rank step loop.

  python tools/mg_emulated_timing.py ts1 [n_steps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2301_05581_b200 as nufi  # noqa: E402
from paper_2301_05581_b200.configs import workload  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "ts1"
w = workload(name)
N = int(sys.argv[2]) if len(sys.argv) > 2 else w.n_steps
g = w.grid
base = None
for G in (1, 2, 4, 8):
    s = torch.cuda.current_stream()
    sim = nufi.Simulation(g, w.ic, w.tau, N, v_blocks=8, stream=s.cuda_stream)
    h = sim.history.handle
    if G > 1:
        h.call("nufi_mg_setup", G, 0, 1, None)
    out = dict(rho=torch.empty((N + 1, g.n_nodes), dtype=torch.float64, device="cuda"),
               E=torch.empty((N + 1, g.n_nodes * g.d), dtype=torch.float64, device="cuda"),
               W=torch.empty(N + 1, dtype=torch.float64, device="cuda"),
               stats=torch.empty((N + 1, 3), dtype=torch.float64, device="cuda"))

    def run():
        sim.history.truncate(0)
        if g.d == 1 or G == 1:
            sim.run(outputs=out)
        else:
            for n in range(N + 1):
                h.call("nufi_mg_step_async", n, out["rho"][n].data_ptr(), out["E"][n].data_ptr(),
                       out["W"][n:].data_ptr(), out["stats"][n].data_ptr())
            h.call("nufi_check_status")

    ts = []
    for r in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        run()
        e1.record(s)
        torch.cuda.synchronize()
        if r:
            ts.append(e0.elapsed_time(e1))
    best = min(ts)
    if G == 1:
        base = best
    print(f"{name} (d={g.d}, {N} steps) emulated ranks {G}: {best:.2f} ms  "
          f"({(best - base) * 1e3 / (N + 1):+.2f} us/step vs 1)")
