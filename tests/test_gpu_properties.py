"""Seeded random configurations (the reference lists hypothesis-style testing as its test
extra, pyproject.toml:19-20): small grids of every dimension with random Nx (incl.
non-powers of two), Nv, vmax, tau, alpha, wavenumber and multi-centre / v^2 velocity
profiles, run on the GPU and through the pinned CPU oracle (the reference's algorithm).
Bar: rho and coefficients within 1e-10 normwise per step, W within 1e-8 relative, stats
within 1e-12 -- plus the step-API == run-API bit-identity on the same configurations."""

import math

import numpy as np
import pytest

import paper_2301_05581_b200 as nufi
from oracle import oracle as O
from tests._util import normwise

pytestmark = pytest.mark.gpu


def random_case(seed):
    rng = np.random.default_rng(seed)
    d = 1 + seed % 3  # every dimension equally often
    Nx = int(rng.choice([4, 5, 6, 8, 12, 16, 24, 32] if d == 1 else ([4, 6, 8, 10] if d == 2 else [4, 5, 6])))
    Nv = int(rng.choice([6, 8, 16, 40, 64] if d == 1 else ([4, 6, 8, 12] if d == 2 else [3, 4, 6])))
    turns = int(rng.integers(1, 3))
    if 2 * turns >= Nx:  # keep the seeded mode below Nyquist (Nyquist modes of phi are dropped, poisson.py:110)
        turns = 1
    L = float(rng.choice([2 * math.pi, 4 * math.pi, 10 * math.pi]))
    k = 2 * math.pi * turns / L
    alpha = float(rng.uniform(0.0, 0.9 / d))
    vmax = float(rng.uniform(4.0, 9.0))
    tau = float(rng.choice([1 / 8, 1 / 10, 1 / 16]))
    prof_o, prof_n = [], []
    for _ in range(d):
        nc = int(rng.integers(1, 3))
        centers = tuple(float(c) for c in rng.uniform(-2.5, 2.5, nc)) if nc > 1 else (0.0,)
        weights = tuple(float(w) for w in rng.uniform(0.3, 1.0, nc))
        power = int(rng.choice([0, 2]))
        prof_o.append(O.Profile(centers=centers, weights=weights, power=power))
        prof_n.append(nufi.VelocityProfile(centers=centers, weights=weights, power=power))
    case = O.Case(d, L, Nx, Nv, vmax, tau, alpha, k, tuple(prof_o))
    grid = nufi.GridSpec(d=d, L=L, Nx=Nx, Nv=Nv, vmax=vmax)
    ic = nufi.InitialCondition(benchmark=f"random{seed}", d=d, L=L, alpha=alpha, k=k, profiles=tuple(prof_n))
    steps = 12 if d == 3 else 20
    return case, grid, ic, tau, steps


@pytest.mark.parametrize("seed", list(range(15)))
def test_random_configuration_vs_oracle(seed):
    case, grid, ic, tau, N = random_case(seed)
    ref = O.OracleRun(case).run(N)
    sim = nufi.Simulation(grid, ic, tau, N)
    res = sim.run()
    coeffs = sim.history.stacked().reshape(N + 1, -1)
    assert normwise(res.rho, ref["rho"]).max() <= 1e-10
    assert normwise(coeffs, ref["coeffs"]).max() <= 1e-10
    W, Wr = res.W, ref["W"]
    assert np.all(np.abs(W - Wr) <= 1e-8 * np.maximum(np.abs(Wr), 1e-300) + 1e-300)
    stats = np.array(ref["stats"])
    assert np.abs(res.stats[:, 1:] - stats[:, 1:]).max() <= 1e-12 * max(1.0, np.abs(stats[:, 2]).max())
    # the single-step API gives the run's bits
    st = nufi.Simulation(grid, ic, tau, 5)
    outs = [st.step() for _ in range(6)]
    assert np.array_equal(np.stack([o.rho.reshape(-1) for o in outs]), res.rho[:6])


@pytest.mark.parametrize("Nx", [4, 8, 16, 32, 64, 128, 256, 512, 1024, 2048, 4096])
def test_d1_tail_every_power_of_two(Nx):
    """The d = 1 step tail has size-specific paths (blocked direct convolution on skewed
    operands for Nx <= 64, four-step FFT for 128 and 256, radix-2 FFT above, more nodes than
    threads from 512, the multi-CTA tail once one CTA cannot hold the work rows): each
    against the oracle, and the persistent run == the single-step API bit for bit."""
    L, tau, N = 4 * math.pi, 1 / 8, 12
    prof_o = (O.Profile(centers=(0.0,), weights=(1.0,), power=0),)
    case = O.Case(1, L, Nx, 16, 6.0, tau, 0.3, 0.5, prof_o)
    ref = O.OracleRun(case).run(N)
    grid = nufi.GridSpec(d=1, L=L, Nx=Nx, Nv=16, vmax=6.0)
    ic = nufi.InitialCondition(benchmark=f"tail{Nx}", d=1, L=L, alpha=0.3, k=0.5,
                               profiles=(nufi.VelocityProfile(),))
    sim = nufi.Simulation(grid, ic, tau, N)
    res = sim.run()
    coeffs = sim.history.stacked().reshape(N + 1, -1)
    assert normwise(res.rho, ref["rho"]).max() <= 1e-10
    assert normwise(coeffs, ref["coeffs"]).max() <= 1e-10
    assert np.all(np.abs(res.W - ref["W"]) <= 1e-8 * np.abs(ref["W"]) + 1e-300)
    st = nufi.Simulation(grid, ic, tau, N)
    outs = [st.step() for _ in range(N + 1)]
    assert np.array_equal(np.stack([o.rho.reshape(-1) for o in outs]), res.rho)
    assert np.array_equal(np.array([o.W for o in outs]), res.W)
