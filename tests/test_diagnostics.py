"""Diagnostics and the observable sweep (density.py:94-120).

CPU tests: the host logic (damping-rate fit KATs, W from a spline slab against the
reference's own W).  GPU tests (-m gpu): the fused sweep kernel (nufi_moments)
and the generic quadrature_sweep_many against goldens produced by the unmodified
reference (tests/golden/make_golden.py sweep_*), plus conservation properties.
Tolerance: moments within 1e-10 of the largest moment magnitude (the trace's
production arithmetic differs from the reference's at ~1e-13).
"""

import math

import numpy as np
import pytest

import paper_2301_05581_b200 as nufi
from paper_2301_05581_b200.configs import workload
from paper_2301_05581_b200.diagnostics import fit_damping_rate
from tests._util import golden

MOM_TOL = 1e-10


# ---------------------------------------------------------------------------
# host logic (CPU)
# ---------------------------------------------------------------------------

def test_fit_damping_rate_synthetic():
    """e^{-0.306718 t} cos^2(w t) on [0, 40] -> 0.306718 within 1e-3."""
    t = np.arange(0, 40.0 + 1e-12, 1.0 / 64)
    e = np.exp(-0.306718 * t) * np.cos(1.4156 * t) ** 2 + 1e-300
    assert abs(fit_damping_rate(t, e, (0.0, 40.0)) - 0.306718) < 1e-3


def test_fit_damping_rate_constant_and_errors():
    t = np.linspace(0, 10, 101)
    assert fit_damping_rate(t, np.full_like(t, 3.0), (0, 10)) == 0.0
    with pytest.raises(nufi.FitError):
        fit_damping_rate(t, np.exp(-t), (0, 10))  # monotone: no peaks
    with pytest.raises(nufi.UsageError):
        fit_damping_rate(t[::-1], np.exp(-t), (0, 10))


def test_electric_energy_from_coeffs_matches_reference_W():
    """Parseval W from the stored slab equals the reference's electric_energy(spec)."""
    z = golden("kat_wl")
    w = workload("kat_wl")
    for n in (0, 10, 40, 160):
        W = nufi.electric_energy_from_coeffs(w.grid, z["coeffs"][n])
        assert abs(W - z["W"][n]) <= 1e-12 * abs(z["W"][n]), (n, W, z["W"][n])


# ---------------------------------------------------------------------------
# GPU: the sweep kernel vs the reference
# ---------------------------------------------------------------------------

def _ctx(name, rows):
    w = workload(name)
    base = golden(name)
    h = nufi.PotentialHistory(w.grid, w.tau, capacity=rows)
    h.load_stack(base["coeffs"][:rows].reshape((rows,) + w.grid.shape_x))
    return w, nufi.FlowContext(history=h, ic=w.ic, tau=w.tau, grid=w.grid)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["kat_wl", "tiny2", "tiny3", "wl3r", "rag1", "rag2", "rag3"])
def test_conserved_moments_vs_reference(name):
    z = golden(f"sweep_{name}")
    steps = [int(n) for n in z["steps"]]
    w, ctx = _ctx(name, max(steps) + 1)
    for i, n in enumerate(steps):
        ctx.field_evals = 0
        m = nufi.conserved_moments(ctx, n)
        got = np.array([m.l1, m.f2, m.f_ln_f, m.kinetic] + list(m.momentum))
        ref = z["moments"][i]
        scale = np.abs(ref).max()
        assert np.abs(got - ref).max() <= MOM_TOL * scale, (n, got - ref)
        assert ctx.field_evals == int(z["field_evals"][i])
        assert 0.0 <= m.f_min <= m.f_max


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["kat_wl", "tiny2"])
def test_generic_sweep_vs_reference(name):
    from oracle import oracle as O

    z = golden(f"sweep_{name}")
    steps = [int(n) for n in z["steps"]]
    w, ctx = _ctx(name, max(steps) + 1)
    for i, n in enumerate(steps):
        f, f2, flnf, kin, mom = nufi.quadrature_sweep_many(ctx, n, O.conserved_weights(), chunk=1 << 14)
        got = np.array([f, f2, flnf, kin] + list(np.atleast_1d(mom)))
        ref = z["moments"][i]
        assert np.abs(got - ref).max() <= MOM_TOL * np.abs(ref).max(), (n, got - ref)
    assert nufi.quadrature_sweep(ctx, 0, lambda X, V, F: F) == pytest.approx(z["moments"][0][0], rel=1e-12)


@pytest.mark.gpu
def test_sweep_needs_field_n():
    w, ctx = _ctx("kat_wl", 5)
    with pytest.raises(nufi.UsageError):
        nufi.conserved_moments(ctx, 5)  # Psi at step 5 needs fields 0..5
    with pytest.raises(nufi.UsageError):
        nufi.quadrature_sweep(ctx, 5, lambda X, V, F: F)


@pytest.mark.gpu
def test_conserved_quantities_kats_and_conservation():
    """SPEC.md:408-410 examples and the conservation property of SPEC.md:424."""
    w = workload("wl1")
    sim = nufi.Simulation(w.grid, w.ic, w.tau, 80)
    res = sim.run()
    r0 = nufi.conserved_quantities(sim.ctx, 0, electric_energy=res.W[0])
    assert abs(r0.l1_norm - 4 * math.pi) <= 1e-8 * 4 * math.pi  # vmax = 6 tail truncation ~1e-9
    assert abs(r0.electric_energy - 0.01 ** 2 * 4 * math.pi / (4 * 0.25)) < 1e-8
    assert np.abs(r0.momentum).max() < 1e-12
    rec = [nufi.conserved_quantities(sim.ctx, n) for n in range(0, 81, 20)]
    for r in rec[1:]:
        for q in ("l1_norm", "l2_norm", "entropy"):
            a, b = getattr(r, q), getattr(rec[0], q)
            assert abs(a - b) <= 1e-3 * abs(b), (q, r.step, a, b)
        assert abs(r.electric_energy - res.W[r.step]) <= 1e-12 * max(res.W[r.step], 1e-30)
        assert 0.0 <= r.linf_observed <= 1.0 / math.sqrt(2 * math.pi) * 1.02 + 1e-12


@pytest.mark.gpu
def test_landau_damping_rate():
    """SPEC.md:417 / PAPER.md:343: gamma_energy = 0.306718 +- 5% (weak Landau, Nx=32, Nv=128, tau=1/16)."""
    w = workload("kat_wl")
    N = 640  # t_end = 40
    res = nufi.Simulation(w.grid, w.ic, w.tau, N).run()
    t = np.arange(N + 1) * w.tau
    rate = fit_damping_rate(t, res.W, (0.0, 40.0))
    assert abs(rate - 0.306718) <= 0.05 * 0.306718, rate
