"""GPU parity tests: libnufi_b200 (through the C-ABI) vs the reference goldens and the oracle.

Tolerance contract (BASELINE.json north_star):
  rho and spline coefficients: normwise relative error <= 1e-10 per step, steps 0..50;
  electric energy W: relative error <= 1e-6 to t_end (ts1: to t = 55, the
  reference's own 1-ulp predictability horizon is t ~ 57-61);
  trace in PARITY mode: bit-exact vs the numba kernels;
  trace in FAST mode (production arithmetic): <= 1e-11 relative to the point scale.
"""

import math

import numpy as np
import pytest

import paper_2301_05581_b200 as nufi
from oracle import oracle as O
from paper_2301_05581_b200.configs import workload
from tests._util import golden, normwise

pytestmark = pytest.mark.gpu

RHO_TOL = 1e-10
COEF_TOL = 1e-10
W_TOL = 1e-6


def _hist_from(name, coeffs, n_rows):
    w = workload(name)
    h = nufi.PotentialHistory(w.grid, w.tau, capacity=n_rows + 1)
    h.load_stack(coeffs[:n_rows].reshape((n_rows,) + w.grid.shape_x))
    return w, h


# ---------------------------------------------------------------------------
# trace_backward: bit-exact parity mode, fast mode within tolerance
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("name", ["kat_wl", "tiny2", "tiny3", "wl3r", "rag1", "rag2", "rag3", "big3"])
@pytest.mark.parametrize("hk", [0, 1])
def test_trace_parity_bit_exact(name, hk):
    t = golden(f"trace_{name}")
    if t is None:
        pytest.skip("trace golden missing")
    n = int(t["n"])
    w, h = _hist_from(name, t["coeffs"], n + 1)
    X, V = t["Xin"].copy(), t["Vin"].copy()
    ev = nufi.trace_backward(h, n, X, V, bool(hk), nufi.TRACE_PARITY)
    assert ev == int(t[f"evals{hk}"])
    assert np.array_equal(X, t[f"X{hk}"]), np.abs(X - t[f"X{hk}"]).max()
    assert np.array_equal(V, t[f"V{hk}"]), np.abs(V - t[f"V{hk}"]).max()


@pytest.mark.parametrize("name", ["kat_wl", "tiny2", "tiny3", "wl3r", "rag1", "rag2", "rag3", "big3"])
@pytest.mark.parametrize("hk", [0, 1])
def test_trace_fast_close(name, hk):
    t = golden(f"trace_{name}")
    if t is None:
        pytest.skip("trace golden missing")
    n = int(t["n"])
    w, h = _hist_from(name, t["coeffs"], n + 1)
    X, V = t["Xin"].copy(), t["Vin"].copy()
    nufi.trace_backward(h, n, X, V, bool(hk), nufi.TRACE_FAST)
    Xr, Vr = t[f"X{hk}"], t[f"V{hk}"]
    assert np.abs(X - Xr).max() <= 1e-11 * max(1.0, np.abs(Xr).max())
    assert np.abs(V - Vr).max() <= 1e-11 * max(1.0, np.abs(Vr).max())


def test_trace_device_buffers_in_place():
    torch = pytest.importorskip("torch")
    t = golden("trace_kat_wl")
    n = int(t["n"])
    w, h = _hist_from("kat_wl", t["coeffs"], n + 1)
    X = torch.tensor(t["Xin"], device="cuda")
    V = torch.tensor(t["Vin"], device="cuda")
    nufi.trace_backward(h, n, X, V, False, nufi.TRACE_PARITY)
    assert np.array_equal(X.cpu().numpy(), t["X0"]) and np.array_equal(V.cpu().numpy(), t["V0"])


def test_trace_errors_and_edge_cases():
    t = golden("trace_kat_wl")
    n = int(t["n"])
    w, h = _hist_from("kat_wl", t["coeffs"], n)  # rows 0..n-1 only
    X, V = t["Xin"].copy(), t["Vin"].copy()
    with pytest.raises(nufi.UsageError, match="need"):
        nufi.trace_backward(h, n, X, V, True)  # Psi needs n + 1 fields (kernels.py:399-402)
    assert nufi.trace_backward(h, 0, X, V, True) == 0  # n = 0: identity
    assert np.array_equal(X, t["Xin"])
    E = np.empty((0, 1))
    assert nufi.trace_backward(h, n, E, E.copy(), False) == 0  # M = 0


# ---------------------------------------------------------------------------
# compute_rho drop-in and the field update on golden histories
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("name", ["kat_wl", "tiny2", "tiny3", "wl1", "rag1", "rag2", "rag3", "big1", "big2g", "big3"])
def test_compute_rho_on_reference_history(name):
    g = golden(name)
    keep = g["rho"].shape[0]
    w, h = _hist_from(name, g["coeffs"], keep)
    ctx = nufi.FlowContext(history=h, ic=w.ic, tau=w.tau, grid=w.grid)
    assert abs(ctx.rho_bar - float(g["rho_bar"])) <= 1e-14
    steps = range(0, keep, max(1, keep // 8))
    for n in steps:
        r = nufi.compute_rho(ctx, n)  # reads rows 0..n-1 only
        err = normwise(r.density.values.reshape(1, -1), g["rho"][n : n + 1])[0]
        assert err <= RHO_TOL, (n, err)
        assert abs(r.f_min - g["stats"][n, 1]) <= 1e-12 and abs(r.f_max - g["stats"][n, 2]) <= 1e-12
        assert abs(r.neutralization - g["stats"][n, 0]) <= 1e-12


def test_compute_rho_requires_history():
    w = workload("kat_wl")
    h = nufi.PotentialHistory(w.grid, w.tau, capacity=8)
    ctx = nufi.FlowContext(history=h, ic=w.ic, tau=w.tau, grid=w.grid)
    with pytest.raises(nufi.UsageError, match="needs fields"):
        nufi.compute_rho(ctx, 1)
    r = nufi.compute_rho(ctx, 0)
    assert ctx.field_evals == 0 and r.density.values.shape == (32,)


@pytest.mark.parametrize("name", ["kat_wl", "tiny2", "tiny3", "rag1", "rag2", "rag3", "big1", "big2", "big3"])
def test_advance_matches_solve_fit_append(name):
    """solve_poisson + fit_spline + append + electric_energy + E from the reference's rho."""
    g = golden(name)
    w = workload(name)
    h = nufi.PotentialHistory(w.grid, w.tau, capacity=4)
    ctx = nufi.FlowContext(history=h, ic=w.ic, tau=w.tau, grid=w.grid)
    for n in range(3):
        rho = nufi.DensityGrid(w.grid, g["rho"][n].reshape(w.grid.shape_x))
        up = nufi.advance(ctx, rho)
        assert normwise(up.coeffs.reshape(1, -1), g["coeffs"][n : n + 1])[0] <= COEF_TOL
        assert normwise(up.E.reshape(1, -1), g["E"][n].reshape(1, -1))[0] <= COEF_TOL
        assert abs(up.W / g["W"][n] - 1) <= 1e-12
    assert len(h) == 3


def test_advance_rejects_non_neutral_density():
    w = workload("kat_wl")
    h = nufi.PotentialHistory(w.grid, w.tau, capacity=4)
    ctx = nufi.FlowContext(history=h, ic=w.ic, tau=w.tau, grid=w.grid)
    rho = nufi.DensityGrid(w.grid, np.full(w.grid.shape_x, 0.5))
    with pytest.raises(nufi.NumericalConsistencyError):
        nufi.advance(ctx, rho)
    assert len(h) == 0


# ---------------------------------------------------------------------------
# full runs vs the reference goldens
# ---------------------------------------------------------------------------

def _run(name, N=None):
    w = workload(name)
    N = w.n_steps if N is None else N
    sim = nufi.Simulation(w.grid, w.ic, w.tau, N)
    res = sim.run()
    return w, sim, res


def _check_run(name, g, sim, res, w_until=None, rho_tol=RHO_TOL):
    keep = min(g["rho"].shape[0], res.rho.shape[0], 51)
    assert normwise(res.rho[:keep], g["rho"][:keep]).max() <= rho_tol
    coeffs = sim.history.stacked().reshape(len(sim.history), -1)
    assert normwise(coeffs[:keep], g["coeffs"][:keep]).max() <= COEF_TOL
    assert normwise(res.E[:keep].reshape(keep, -1), g["E"][:keep].reshape(keep, -1)).max() <= COEF_TOL
    N = len(g["W"])
    upto = N if w_until is None else w_until
    relW = np.abs(res.W[:upto] - g["W"][:upto]) / np.abs(g["W"][:upto])
    assert relW.max() <= W_TOL, (relW.argmax(), relW.max())
    assert np.abs(res.stats[:upto, 1:] - g["stats"][:upto, 1:]).max() <= 1e-12 * max(1.0, np.abs(g["stats"][:, 2]).max())
    return relW


@pytest.mark.parametrize("name", ["kat_wl", "tiny2", "tiny3", "wl1", "rag1", "rag2", "rag3", "big1", "big2", "big2g",
                                  "big3"])
def test_run_vs_reference(name):
    g = golden(name)
    N = len(g["W"]) - 1
    w, sim, res = _run(name, N)
    _check_run(name, g, sim, res)
    assert res.field_evals == int(g["field_evals"][-1])


def test_equilibrium_energy_zero():
    """SPEC acceptance 1: alpha = 0 -> W < 1e-20 at every step."""
    w, sim, res = _run("eq1")
    assert np.all(res.W < 1e-20)


def test_run_deterministic():
    w, _, a = _run("kat_wl", 60)
    _, _, b = _run("kat_wl", 60)
    assert np.array_equal(a.rho, b.rho) and np.array_equal(a.W, b.W) and np.array_equal(a.E, b.E)


def test_step_api_matches_run():
    w = workload("kat_wl")
    sim = nufi.Simulation(w.grid, w.ic, w.tau, 30)
    outs = [sim.step() for _ in range(31)]
    _, _, res = _run("kat_wl", 30)
    assert np.array_equal(np.stack([o.rho.reshape(-1) for o in outs]), res.rho)
    assert np.array_equal(np.array([o.W for o in outs]), res.W)
    with pytest.raises(nufi.UsageError):
        sim.step()


def test_maximum_principle_two_stream():
    """SPEC acceptance 5 (exact, tolerance 0): 0 <= f <= sup f0 on every sample."""
    w = workload("ts1")
    sim = nufi.Simulation(w.grid, w.ic, w.tau, 400)
    res = sim.run()
    sup = (1 + w.ic.alpha) * 2 / (math.e * math.sqrt(2 * math.pi))
    assert res.stats[:, 1].min() >= 0.0
    assert res.stats[:, 2].max() <= sup


@pytest.mark.slow
def test_wl3r_full_run():
    g = golden("wl3r")
    if g is None:
        pytest.skip("golden missing")
    w, sim, res = _run("wl3r")
    _check_run("wl3r", g, sim, res)


@pytest.mark.slow
@pytest.mark.parametrize("name", ["ts1", "sl1", "wl2", "wl3"])
def test_baseline_config_vs_reference(name):
    g = golden(name)
    if g is None:
        pytest.skip("golden missing")
    N = len(g["W"]) - 1
    w, sim, res = _run(name, N)
    if name == "ts1":
        # W within 1e-6 up to t = 55 (step 880); beyond the reference's own
        # 1-ulp predictability horizon only the envelope / physics checks apply
        relW = _check_run(name, g, sim, res, w_until=881)
        t = np.arange(N + 1) * w.tau
        first_peak = next(i for i in range(1, N) if res.W[i] > 0.1 and res.W[i] >= res.W[i - 1] and res.W[i] >= res.W[i + 1])
        assert abs(t[first_peak] - 25) <= 5
        assert res.W[t > 30].min() > 0.1 and res.W.max() < 1.0
    else:
        _check_run(name, g, sim, res)


@pytest.mark.parametrize("hk", [0, 1])
def test_trace_fast_d1_cell_boundaries_and_rounding_ties(hk):
    """The d = 1 FAST lookup rounds 8 Y (Y = x N/L - 1/16, csrc/trace_common.cuh d1_locate);
    its ties fall exactly on cell boundaries.  Points on every node (boundaries), 1/16 and
    1/2 cell either side, and outside [0, L), with v = 0 (so the first lookups hit those
    positions exactly) and small v: FAST within 1e-11 of the reference's arithmetic (PARITY)."""
    t = golden("trace_kat_wl")
    if t is None:
        pytest.skip("trace golden missing")
    n = int(t["n"])
    w, h = _hist_from("kat_wl", t["coeffs"], n + 1)
    g = w.grid
    hx = g.L / g.Nx
    k = np.arange(-2, g.Nx + 3, dtype=np.float64)
    x = np.concatenate([k, k + 1 / 16, k - 1 / 16, k + 0.5, k + 15 / 16]) * hx
    v = np.concatenate([np.zeros_like(x), np.full_like(x, 1e-3), np.full_like(x, -0.37)])
    X0 = np.tile(x, 3)[:, None].copy()
    V0 = v[:, None].copy()
    Xp, Vp = X0.copy(), V0.copy()
    nufi.trace_backward(h, n, Xp, Vp, bool(hk), nufi.TRACE_PARITY)
    Xf, Vf = X0.copy(), V0.copy()
    nufi.trace_backward(h, n, Xf, Vf, bool(hk), nufi.TRACE_FAST)
    assert np.abs(Xf - Xp).max() <= 1e-11 * max(1.0, np.abs(Xp).max())
    assert np.abs(Vf - Vp).max() <= 1e-11 * max(1.0, np.abs(Vp).max())
