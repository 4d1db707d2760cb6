"""The reference's install_field test hook (flow.py:44-47) with UniformField
(spline.py:55-68): the constant-force closed form of SPEC.md:309,529 (measured on the
reference: abs err <= 2.8e-14 at n = 100), the generic trace order (flow.py:65-82) with
mixed spline / uniform slots bit for bit against the oracle, and the usage errors."""

import math

import numpy as np
import pytest

import paper_2301_05581_b200 as nufi
from oracle import oracle as O
from paper_2301_05581_b200.errors import UsageError
from paper_2301_05581_b200.flow import psi_batch, psi_tilde_batch

pytestmark = pytest.mark.gpu


def _ctx(d, Nx=8, Nv=4, tau=0.125, cap=128, L=4 * math.pi):
    grid = nufi.GridSpec(d=d, L=L, Nx=Nx, Nv=Nv, vmax=5.0)
    ic = nufi.InitialCondition(benchmark="hook", d=d, L=grid.L, alpha=0.0, k=2 * math.pi / L,
                               profiles=(nufi.VelocityProfile(),) * d)
    hist = nufi.PotentialHistory(grid, tau, capacity=cap)
    return nufi.FlowContext(history=hist, ic=ic, tau=tau, grid=grid), grid


@pytest.mark.parametrize("d,n", [(1, 100), (2, 60), (3, 30)])
def test_constant_force_closed_form(d, n):
    ctx, grid = _ctx(d)
    rng = np.random.default_rng(3 + d)
    E0 = rng.uniform(-0.5, 0.5, d)
    for k in range(n + 1):
        ctx.install_field(k, nufi.UniformField(E0))
    M = 257
    x = rng.uniform(0.0, grid.L, (M, d))
    v = rng.uniform(-5.0, 5.0, (M, d))
    X, V = psi_batch(ctx, n, x, v)
    T = n * ctx.tau
    # Psi with a constant force: x - v T - E0 T^2 / 2, v + E0 T (positions not wrapped)
    assert np.abs(X - (x - v * T - 0.5 * E0 * T * T)).max() <= 1e-12
    assert np.abs(V - (v + E0 * T)).max() <= 1e-13
    assert ctx.field_evals == M * (n + 1)
    # Psi-tilde: kicks (n - 1/2) tau E0 in total
    Xt, Vt = psi_tilde_batch(ctx, n, x, v)
    assert np.abs(Vt - (v + E0 * (T - 0.5 * ctx.tau))).max() <= 1e-13


@pytest.mark.parametrize("d", [1, 2, 3])
def test_mixed_fields_match_reference_generic_trace(d):
    ctx, grid = _ctx(d, Nx=6 if d == 3 else 8)
    rng = np.random.default_rng(11 * d)
    n = 6
    slabs = rng.normal(0.0, 0.3, (n + 1,) + grid.shape_x)
    ctx.history.load_stack(slabs)
    fields = {k: slabs[k] for k in range(n + 1)}
    for k in (2, 5):
        E0 = rng.uniform(-0.4, 0.4, d)
        ctx.install_field(k, nufi.UniformField(E0))
        fields[k] = ("uniform", E0)
    M = 300
    x = rng.uniform(-grid.L, 2 * grid.L, (M, d))  # images too
    v = rng.uniform(-5.0, 5.0, (M, d))
    for half in (True, False):
        X, V = (psi_batch if half else psi_tilde_batch)(ctx, n, x, v)
        Xr, Vr = x.copy(), v.copy()
        O.trace_generic(fields, grid.L, n, ctx.tau, Xr, Vr, half)
        assert np.array_equal(X, Xr) and np.array_equal(V, Vr)
    # removing the overrides restores the fused spline trace (FAST mode, 1e-11 of the point scale)
    ctx.install_field(2, None)
    ctx.install_field(5, None)
    X, V = psi_batch(ctx, n, x, v)
    Xr, Vr = x.copy(), v.copy()
    O.trace_numpy(slabs, grid.L, n, ctx.tau, Xr, Vr, True)
    assert np.abs(X - Xr).max() <= 1e-11 * max(1.0, np.abs(Xr).max())


def test_installed_field_usage_errors():
    ctx, grid = _ctx(1)
    ctx.install_field(3, nufi.UniformField([0.1]))
    # slots 0..2 are neither stored nor installed
    with pytest.raises(UsageError):
        psi_batch(ctx, 3, [[1.0]], [[0.5]])
    for k in range(3):
        ctx.install_field(k, nufi.UniformField([0.1]))
    psi_batch(ctx, 3, [[1.0]], [[0.5]])
    # the fused density / run kernels trace stored splines only
    with pytest.raises(UsageError):
        nufi.compute_rho(ctx, 3)
    with pytest.raises(UsageError):
        ctx.install_field(1, object())
    with pytest.raises(UsageError):
        ctx.install_field(1, nufi.UniformField([0.1, 0.2]))
    ctx.clear_fields()
    with pytest.raises(UsageError):
        psi_batch(ctx, 3, [[1.0]], [[0.5]])  # nothing stored


@pytest.mark.parametrize("base", ["kat_wl", "tiny2", "tiny3"])
def test_install_field_matches_reference_goldens(base):
    """Against the reference's own install_field runs (tests/golden/hook_*.npz), bit for bit."""
    from tests._util import golden

    z = golden(f"hook_{base}")
    ref = golden(base)
    c = O.case(base)
    n = int(z["n"])
    grid = nufi.GridSpec(d=c.d, L=c.L, Nx=c.Nx, Nv=c.Nv, vmax=c.vmax)
    ic = nufi.InitialCondition(benchmark=f"hook_{base}", d=c.d, L=c.L, alpha=0.0, k=2 * math.pi / c.L,
                               profiles=(nufi.VelocityProfile(),) * c.d)
    hist = nufi.PotentialHistory(grid, c.tau, capacity=n + 1)
    hist.load_stack(ref["coeffs"].reshape((-1,) + (c.Nx,) * c.d)[: n + 1])
    ctx = nufi.FlowContext(history=hist, ic=ic, tau=c.tau, grid=grid)
    for s, e in zip(z["slots"], z["E0"]):
        ctx.install_field(int(s), nufi.UniformField(e))
    X, V = psi_batch(ctx, n, z["x"], z["v"])
    assert np.array_equal(X, z["X_psi"]) and np.array_equal(V, z["V_psi"])
    X, V = psi_tilde_batch(ctx, n, z["x"], z["v"])
    assert np.array_equal(X, z["X_tilde"]) and np.array_equal(V, z["V_tilde"])
    assert ctx.field_evals == int(z["evals"])
    ctx_u, _ = _ctx(c.d, Nx=c.Nx, tau=c.tau, L=c.L)
    for k in range(n + 1):
        ctx_u.install_field(k, nufi.UniformField(z["E_uniform"]))
    X, V = psi_batch(ctx_u, n, z["x"], z["v"])
    assert np.array_equal(X, z["X_uniform"]) and np.array_equal(V, z["V_uniform"])


@pytest.mark.parametrize("d,Nx,n,M", [(2, 32, 30, 20000), (2, 6, 9, 3000), (3, 16, 12, 9000), (3, 5, 7, 1500)])
def test_staged_point_trace_matches_in_place_kernel(d, Nx, n, M, monkeypatch):
    """FAST point traces for d >= 2 run through a shared-memory slab ring (trace_points_ring);
    the in-place kernel (NUFI_TP_NORING) computes the same arithmetic: bit-identical, incl.
    partial last CTAs, multi-pass CTAs and non-power-of-two grids."""
    ctx, grid = _ctx(d, Nx=Nx, cap=n + 2)
    rng = np.random.default_rng(40 + d + Nx)
    ctx.history.load_stack(rng.normal(0.0, 0.2, (n + 1,) + grid.shape_x))
    x = rng.uniform(-grid.L, 2 * grid.L, (M, d))
    v = rng.uniform(-5.0, 5.0, (M, d))
    for half in (True, False):
        fn = psi_batch if half else psi_tilde_batch
        X1, V1 = fn(ctx, n, x, v)
        monkeypatch.setenv("NUFI_TP_NORING", "1")
        X0, V0 = fn(ctx, n, x, v)
        monkeypatch.delenv("NUFI_TP_NORING")
        assert np.array_equal(X1, X0) and np.array_equal(V1, V0)
