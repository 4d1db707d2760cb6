"""Time the d=1 observable sweep (nufi_moments) of ts1 at n = 800: python tools/sweep_probe.py (for ncu -k trace_rho)."""
import sys, os
sys.path.insert(0, '/root/repo')
import torch
import paper_2301_05581_b200 as nufi
from paper_2301_05581_b200.configs import workload
w = workload("ts1")
sim = nufi.Simulation(w.grid, w.ic, w.tau, 800)
sim.run()
for _ in range(3):
    nufi.conserved_moments(sim.ctx, 800)
torch.cuda.synchronize()
