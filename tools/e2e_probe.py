"""Break the e2e (public API, host outputs) time of one run into create / run / destroy."""
import gc
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2301_05581_b200 as nufi  # noqa: E402
from paper_2301_05581_b200.configs import workload  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "ts1"
w = workload(name)
for it in range(5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sim = nufi.Simulation(w.grid, w.ic, w.tau, w.n_steps, device=0)
    t1 = time.perf_counter()
    res = sim.run()
    t2 = time.perf_counter()
    del sim, res  # refcount drop: nufi_destroy runs here (no gc.collect, like the bench loop)
    t3 = time.perf_counter()
    print(f"{name} it{it}: create {1e3*(t1-t0):.1f} ms  run {1e3*(t2-t1):.1f} ms  destroy {1e3*(t3-t2):.1f} ms", flush=True)
