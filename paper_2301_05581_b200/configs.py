"""The BASELINE.json workloads mapped onto the reference's constructors
(SURVEY.md §8(d)), plus the small parity cases of tests/golden/make_golden.py."""

from __future__ import annotations

import math
from dataclasses import dataclass

from .grids import GridSpec
from .initial import InitialCondition, VelocityProfile, make_benchmark, weak_landau_3d

FOUR_PI = 4.0 * math.pi


@dataclass(frozen=True)
class Workload:
    name: str
    grid: GridSpec
    ic: InitialCondition
    tau: float
    n_steps: int
    description: str

    @property
    def point_steps(self) -> int:
        """P * N(N+1)/2 for the full run (equals the reference's field_evals)."""
        N = self.n_steps
        return self.grid.n_points * N * (N + 1) // 2


def workload(name: str) -> Workload:
    if name == "wl1":
        return Workload(name, GridSpec(1, FOUR_PI, 64, 256, 6.0), make_benchmark("weak_landau_1d"), 1 / 8, 240,
                        "d=1 weak Landau, Nx=64, Nv=256, vmax=6, dt=1/8, t_end=30")
    if name == "ts1":
        return Workload(name, GridSpec(1, FOUR_PI, 64, 512, 10.0), make_benchmark("two_stream_1d"), 1 / 16, 1600,
                        "d=1 two-stream, Nx=64, Nv=512, vmax=10, dt=1/16, t_end=100")
    if name == "sl1":
        return Workload(name, GridSpec(1, FOUR_PI, 256, 2048, 8.0), make_benchmark("weak_landau_1d", alpha=0.5),
                        1 / 16, 800, "d=1 strong Landau, Nx=256, Nv=2048, vmax=8, dt=1/16, t_end=50")
    if name == "wl2":
        return Workload(name, GridSpec(2, FOUR_PI, 32, 64, 6.0), make_benchmark("strong_landau_2d", alpha=0.01),
                        1 / 8, 160, "d=2 weak Landau, 32^2 x 64^2, vmax=6, dt=1/8, t_end=20")
    if name == "wl3":
        return Workload(name, GridSpec(3, FOUR_PI, 16, 32, 6.0), weak_landau_3d(), 1 / 8, 80,
                        "d=3 weak Landau, 16^3 x 32^3, vmax=6, dt=1/8, t_end=10")
    # parity cases (tests/golden)
    if name == "wl3r":
        return Workload(name, GridSpec(3, FOUR_PI, 16, 8, 6.0), weak_landau_3d(), 1 / 8, 80, "reduced wl3")
    if name == "kat_wl":
        return Workload(name, GridSpec(1, FOUR_PI, 32, 128, 10.0), make_benchmark("weak_landau_1d"), 1 / 16, 160,
                        "SPEC KAT weak Landau Nx=32 Nv=128 vmax=10")
    if name == "eq1":
        return Workload(name, GridSpec(1, FOUR_PI, 32, 128, 10.0), make_benchmark("weak_landau_1d", alpha=0.0),
                        1 / 16, 160, "equilibrium (alpha = 0)")
    if name == "tiny2":
        return Workload(name, GridSpec(2, FOUR_PI, 8, 8, 6.0), make_benchmark("strong_landau_2d"), 1 / 8, 24,
                        "d=2 strong Landau 8^2 x 8^2")
    if name == "tiny3":
        return Workload(name, GridSpec(3, 10.0 * math.pi, 8, 4, 6.0), make_benchmark("two_stream_3d"), 1 / 8, 12,
                        "d=3 two-stream 8^3 x 4^3")
    # ragged / non-power-of-two grids (generic-N paths)
    if name == "rag1":
        return Workload(name, GridSpec(1, FOUR_PI, 24, 40, 6.0), make_benchmark("weak_landau_1d", alpha=0.05), 1 / 8,
                        40, "d=1 weak Landau, Nx=24 (non-power-of-two), Nv=40")
    if name == "rag2":
        return Workload(name, GridSpec(2, FOUR_PI, 6, 10, 6.0), make_benchmark("strong_landau_2d", alpha=0.3), 1 / 8,
                        16, "d=2 Landau, 6^2 x 10^2")
    if name == "rag3":
        return Workload(name, GridSpec(3, FOUR_PI, 5, 3, 5.0), weak_landau_3d(alpha=0.05), 1 / 8, 8,
                        "d=3 Landau, 5^3 x 3^3")
    # grids beyond one CTA
    if name == "big1":
        return Workload(name, GridSpec(1, FOUR_PI, 5000, 16, 6.0), make_benchmark("weak_landau_1d", alpha=0.05), 1 / 8,
                        6, "d=1 Nx=5000")
    if name == "big2":
        return Workload(name, GridSpec(2, FOUR_PI, 72, 6, 6.0), make_benchmark("strong_landau_2d", alpha=0.2), 1 / 8,
                        6, "d=2 72^2 x 6^2")
    if name == "big2g":
        return Workload(name, GridSpec(2, FOUR_PI, 120, 4, 6.0), make_benchmark("strong_landau_2d", alpha=0.2), 1 / 8,
                        4, "d=2 120^2 x 4^2 (in-place trace)")
    if name == "big3":
        return Workload(name, GridSpec(3, FOUR_PI, 22, 3, 5.0), weak_landau_3d(alpha=0.05), 1 / 8, 4,
                        "d=3 22^3 x 3^3 (in-place trace)")
    raise KeyError(name)


BASELINE = ("wl1", "ts1", "sl1", "wl2", "wl3")
PARITY_CASES = ("kat_wl", "eq1", "tiny2", "tiny3", "wl3r", "rag1", "rag2", "rag3")

# flops per point-step counted on the reference's arithmetic as written
# (SURVEY.md §8(d)): d=1 25, d=2 148, d=3 478
ALGO_FLOPS = {1: 25, 2: 148, 3: 478}
# coefficient bytes read per point-step (4^d doubles)
ALGO_BYTES = {1: 32, 2: 128, 3: 512}

__all__ = ["Workload", "workload", "BASELINE", "PARITY_CASES", "ALGO_FLOPS", "ALGO_BYTES", "VelocityProfile"]
