"""The reference's public API, called by its own module and function names, against this
package (the drop-in check: a vpflow caller swaps the import and nothing else).

`vpflow` below IS paper_2301_05581_b200.  The §3.1 loop is written exactly as the golden
generator runs it on the unmodified reference (tests/golden/make_golden.py run()), and the
module-level helpers are compared with goldens the reference produced on seeded inputs
(tests/golden/make_golden.py api / hooks_spline).
"""

import math

import numpy as np
import pytest

import paper_2301_05581_b200 as vpflow
from paper_2301_05581_b200 import density, flow, grids, initial, kernels, poisson, spline
from paper_2301_05581_b200.configs import workload

from tests._util import golden, normwise

pytestmark = pytest.mark.gpu


def _api():
    g = golden("api")
    if g is None:
        pytest.skip("api golden missing")
    return g


@pytest.mark.parametrize("name,N", [("kat_wl", 30), ("tiny2", 12), ("tiny3", 8), ("rag1", 20)])
def test_reference_call_sequence(name, N):
    """compute_rho -> solve_poisson -> fit_spline -> append -> electric_energy -> eval_E_many
    at the nodes, through the reference's names (density.py:72, poisson.py:90/115,
    spline.py:71/132, kernels.py:102, grids.py:104)."""
    w = workload(name)
    g = grids.GridSpec(d=w.grid.d, L=w.grid.L, Nx=w.grid.Nx, Nv=w.grid.Nv, vmax=w.grid.vmax)
    ic = w.ic
    hist = spline.PotentialHistory(g, w.tau)
    ctx = flow.FlowContext(history=hist, ic=ic, tau=w.tau, grid=g)
    Xn = grids.x_node_matrix(g)
    ref = golden(name)
    for n in range(N + 1):
        r = density.compute_rho(ctx, n)
        phi, spec = poisson.solve_poisson(r.density)
        fit = spline.fit_spline(phi, g)
        hist.append(fit)
        W = poisson.electric_energy(spec)
        E = kernels.eval_E_many(fit.coeffs, g.L, Xn)
        assert normwise(r.density.values.reshape(1, -1), ref["rho"][n:n + 1])[0] <= 1e-10
        assert normwise(np.asarray(hist.entry(n).coeffs).reshape(1, -1), ref["coeffs"][n:n + 1])[0] <= 1e-10
        assert normwise(E.reshape(1, -1), ref["E"][n].reshape(1, -1))[0] <= 1e-10
        assert abs(W - ref["W"][n]) <= 1e-6 * abs(ref["W"][n])
        assert abs(r.f_max - ref["stats"][n, 2]) <= 1e-12
    assert ctx.field_evals == int(ref["field_evals"][N])
    assert abs(ctx.rho_bar - float(ref["rho_bar"])) <= 1e-14


def _ic(name):
    if name == "weak_landau_3d":
        return initial.InitialCondition(benchmark=name, d=3, L=4 * math.pi, alpha=0.01, k=0.5,
                                        profiles=(initial.VelocityProfile(),) * 3)
    return initial.make_benchmark(name)


@pytest.mark.parametrize("name", ["weak_landau_1d", "two_stream_1d", "strong_landau_2d", "two_stream_3d",
                                  "weak_landau_3d"])
def test_eval_f0_reference_signature(name):
    """initial.eval_f0(ic, x, v) on (M, d) and (..., d) batches (initial.py:165-180); also
    reachable as flow.eval_f0 (the reference's flow module imports it, flow.py:21)."""
    a = _api()
    ic = _ic(name)
    F = initial.eval_f0(ic, a[f"f0_{name}_x"], a[f"f0_{name}_v"])
    ref = a[f"f0_{name}_F"]
    assert F.shape == ref.shape
    assert np.abs(F - ref).max() <= 4e-16 * max(1.0, np.abs(ref).max())
    Fb = flow.eval_f0(ic, a[f"f0b_{name}_x"], a[f"f0b_{name}_v"])
    assert Fb.shape == (3, 5)
    assert np.abs(Fb - a[f"f0b_{name}_F"]).max() <= 4e-16
    with pytest.raises(vpflow.UsageError):
        initial.eval_f0(ic, np.zeros((4, ic.d)), np.zeros((4, ic.d + 1)))


@pytest.mark.parametrize("cname", ["wl1", "ts1", "sl1", "wl2", "wl3", "wl3r", "tiny3", "rag2"])
def test_background_density_reference_signature(cname):
    a = _api()
    w = workload(cname)
    rb = initial.background_density(w.ic, w.grid)
    assert abs(rb - float(a[f"rhobar_{cname}"])) <= 1e-14
    other = workload("tiny2" if w.grid.d != 2 else "kat_wl")
    with pytest.raises(vpflow.UsageError):
        initial.background_density(w.ic, other.grid)


def test_bspline_weights_bit_identical():
    """kernels.bspline_weights / bspline_dweights (kernels.py:62-81), incl. t = 0, 1, tiny."""
    a = _api()
    assert np.array_equal(kernels.bspline_weights(a["bs_t"]), a["bs_w"])
    assert np.array_equal(kernels.bspline_dweights(a["bs_t"]), a["bs_dw"])
    w2 = kernels.bspline_weights(a["bs_t2"])
    assert w2.shape == (4, 7, 9) and np.array_equal(w2, a["bs_w2"])
    assert np.array_equal(kernels.bspline_dweights(a["bs_t2"]), a["bs_dw2"])


@pytest.mark.parametrize("base", ["kat_wl", "tiny2", "tiny3", "rag1", "rag2", "rag3"])
def test_kernels_eval_many_bit_identical(base):
    """kernels.eval_phi_many / eval_E_many(coeffs, L, X) (kernels.py:84-123) at the field
    goldens' points (the reference's SplineField methods call exactly these)."""
    f = golden(f"field_{base}")
    w = workload(base)
    c = golden(base)["coeffs"][int(f["slot"])].reshape((w.grid.Nx,) * w.grid.d)
    assert np.array_equal(kernels.eval_phi_many(c, w.grid.L, f["X"]), f["phi"])
    assert np.array_equal(kernels.eval_E_many(c, w.grid.L, f["X"]), f["E"])


@pytest.mark.parametrize("d,N", [(1, 32), (1, 5), (2, 8), (2, 6), (3, 8), (3, 5)])
def test_transforms(d, N):
    """poisson.transform_values / forward_transform / inverse_transform (poisson.py:72-87)."""
    a = _api()
    g = grids.GridSpec(d=d, L=4 * math.pi, Nx=N, Nv=4, vmax=6.0)
    vals = a[f"tr_{d}_{N}_in"]
    spec = poisson.transform_values(g, vals)
    ref = a[f"tr_{d}_{N}_spec"]
    assert spec.coeffs.shape == g.shape_x
    assert np.abs(spec.coeffs - ref).max() <= 1e-15 * max(1.0, np.abs(ref).max()) * N ** d
    rho = density.DensityGrid(g, vals)
    assert np.array_equal(poisson.forward_transform(rho).coeffs, spec.coeffs)
    inv = poisson.inverse_transform(poisson.SpectralField(grid=g, coeffs=a[f"tr_{d}_{N}_cin"]))
    refi = a[f"tr_{d}_{N}_inv"]
    assert inv.shape == g.shape_x
    assert np.abs(inv - refi).max() <= 1e-14 * np.abs(refi).max() * N ** d
    back = poisson.inverse_transform(spec)
    assert np.abs(back - vals).max() <= 1e-13 * np.abs(vals).max()
    with pytest.raises(vpflow.UsageError):
        poisson.transform_values(g, np.zeros(3))


@pytest.mark.parametrize("base", ["kat_wl", "tiny2", "tiny3"])
def test_install_spline_field(base):
    """FlowContext.install_field(step, SplineField) (flow.py:44-47): other steps' splines in
    two slots + a UniformField, psi / psi_tilde through the generic trace (flow.py:65-82),
    bit-identical to the reference's run of the same sequence."""
    z = golden(f"hookspline_{base}")
    w = workload(base)
    g = w.grid
    n = int(z["n"])
    stack = golden(base)["coeffs"].reshape((-1,) + (g.Nx,) * g.d)
    hist = spline.PotentialHistory(g, w.tau)
    hist.load_stack(stack[: n + 1])
    ctx = flow.FlowContext(history=hist, ic=w.ic, tau=w.tau, grid=g)
    for s_, k in zip(z["slots"], z["src"]):
        ctx.install_field(int(s_), spline.SplineField(grid=g, coeffs=np.ascontiguousarray(stack[int(k)])))
    ctx.install_field(n - 1, spline.UniformField(z["E_uniform"]))
    X1, V1 = flow.psi_batch(ctx, n, z["x"], z["v"])
    X0, V0 = flow.psi_tilde_batch(ctx, n, z["x"], z["v"])
    assert np.array_equal(X1, z["X_psi"]) and np.array_equal(V1, z["V_psi"])
    assert np.array_equal(X0, z["X_tilde"]) and np.array_equal(V0, z["V_tilde"])
    assert ctx.field_evals == int(z["evals"])
    with pytest.raises(vpflow.UsageError):
        ctx.install_field(1, object())
    with pytest.raises(vpflow.UsageError):
        density.compute_rho(ctx, n)  # the fused density kernel traces stored splines only
    ctx.install_field(0, None)


def test_abi_rejects_negative_counts_and_unreachable_override_steps():
    """C-ABI validation (include/nufi.h): a negative point count and an override step no
    history can reach are usage errors, never a huge allocation."""
    w = workload("kat_wl")
    hist = spline.PotentialHistory(w.grid, w.tau, capacity=4)
    flow.FlowContext(history=hist, ic=w.ic, tau=w.tau, grid=w.grid)
    h = hist.handle
    buf = np.zeros(64)
    p = buf.ctypes.data
    for fn, args in [("nufi_trace", (1, p, p, -1, 0, 0, None)),
                     ("nufi_eval_f0", (p, p, -1, p)),
                     ("nufi_bspline_weights", (p, -1, p, p))]:
        with pytest.raises(vpflow.UsageError):
            h.call(fn, *args)
    for fn in ("nufi_set_uniform_field", "nufi_set_spline_field"):
        with pytest.raises(vpflow.UsageError):
            h.call(fn, 1 << 40, p)
        with pytest.raises(vpflow.UsageError):
            h.call(fn, -1, p)
    h.call("nufi_set_uniform_field", 2, p)  # a step beyond the stored history is fine
    h.call("nufi_set_uniform_field", 2, None)
