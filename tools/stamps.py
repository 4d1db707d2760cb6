"""Per-step phase split of the persistent d=1 run kernel (NUFI_STAMPS debug hook):
   python tools/stamps.py ts1   -> trace / barrier / tail microseconds summed over the run."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
name = sys.argv[1] if len(sys.argv) > 1 else "ts1"
path = f"/tmp/stamps_{name}.txt"
os.environ["NUFI_STAMPS"] = path

import numpy as np  # noqa: E402

import paper_2301_05581_b200 as nufi  # noqa: E402
from paper_2301_05581_b200.configs import workload  # noqa: E402

w = workload(name)
for rep in range(2):
    sim = nufi.Simulation(w.grid, w.ic, w.tau, w.n_steps)
    sim.run()
rows = np.array([[float(x) for x in l.split()] for l in open(path) if not l.startswith("#")])
t0, t1, t2 = rows[:, 1], rows[:, 2], rows[:, 3]
trace = t0[1:] - t2[:-1]
barrier = t1 - t0
tail = t2 - t1
tot = (t2[-1] - t0[0]) / 1e3 + trace[0] / 1e3
print(f"{name}: steps {len(rows)} total {tot / 1e3:.2f} ms | trace {trace.sum() / 1e6:.2f} ms, "
      f"barrier(cta0 wait) {barrier.sum() / 1e6:.2f} ms, tail {tail.sum() / 1e6:.2f} ms | "
      f"per-step barrier {np.median(barrier) / 1e3:.2f} us tail {np.median(tail) / 1e3:.2f} us")
for q in (10, 100, 400, 800, 1200, len(rows) - 1):
    if q < len(rows) - 1:
        print(f"  n={q}: trace {trace[q - 1] / 1e3:.1f} us barrier {barrier[q] / 1e3:.1f} us tail {tail[q] / 1e3:.1f} us")
for l in open(path):
    if l.startswith("# tail phases"):
        print(l.strip())
    if l.startswith("# wait/total"):
        pairs = [tuple(map(int, x.split("/"))) for x in l.split(":")[1].split()]
        w = np.array([a for a, b in pairs], float)
        t = np.array([b for a, b in pairs], float)
        print(f"  TMA wait share of the trace (last step, per CTA): mean {np.mean(w / t):.3f} max {np.max(w / t):.3f}")
