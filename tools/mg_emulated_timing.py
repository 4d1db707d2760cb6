"""Per-step cost of the fused multi-rank exchange, measured with emulated ranks on one GPU:
the same total tiles traced either as one rank or as G rank groups of one launch."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2301_05581_b200 as nufi  # noqa: E402
from paper_2301_05581_b200.configs import workload  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "ts1"
w = workload(name)
for G in (1, 2, 4, 8):
    s = torch.cuda.current_stream()
    sim = nufi.Simulation(w.grid, w.ic, w.tau, w.n_steps, v_blocks=8, stream=s.cuda_stream)
    if G > 1:
        sim.history.handle.call("nufi_mg_setup", G, 0, 1, None)
    out = dict(W=torch.empty(w.n_steps + 1, dtype=torch.float64, device="cuda"))
    ts = []
    for r in range(4):
        sim.history.truncate(0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        sim.run(outputs=out)
        e1.record(s)
        torch.cuda.synchronize()
        if r:
            ts.append(e0.elapsed_time(e1))
    best = min(ts)
    print(f"{name} emulated ranks {G}: {best:.2f} ms  ({(best - (base if G > 1 else best)) * 1e3 / (w.n_steps + 1):+.2f} us/step vs 1)")
    if G == 1:
        base = best
