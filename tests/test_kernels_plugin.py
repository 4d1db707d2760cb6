"""paper_2301_05581_b200.kernels: the reference's trace plug-in point (kernels.py:30-45,
390-412) served by the GPU -- same signature, in-place contract, evaluation count and
errors; the default backend is bit-identical to the reference's numba kernels."""

import numpy as np
import pytest

from paper_2301_05581_b200 import kernels as K
from paper_2301_05581_b200.errors import UsageError
from tests._util import golden

CASES = ["kat_wl", "tiny2", "tiny3", "wl3r", "rag1", "rag2", "rag3"]


def _stack(t, rows):
    n = int(t["n"])
    c = t["coeffs"][:rows]
    N = round(c.shape[1] ** (1.0 / t["Xin"].shape[1]))
    return c.reshape((rows,) + (N,) * t["Xin"].shape[1]), n


def test_contract_without_gpu():
    X = np.zeros((4, 1))
    V = np.zeros((4, 1))
    c = np.zeros((3, 8))
    assert K.trace_backward(c, 1.0, 0, 0.1, X, V, True) == 0  # n = 0: no-op (kernels.py:397)
    assert K.trace_backward(c, 1.0, 2, 0.1, X[:0], V[:0], False) == 0  # M = 0
    with pytest.raises(UsageError):
        K.trace_backward(c, 1.0, 3, 0.1, X, V, True)  # needs 4 fields
    with pytest.raises(UsageError):
        K.set_backend("numba")
    assert K.get_backend() in ("b200-parity", "b200")


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("hk", [0, 1])
def test_plugin_bit_exact_vs_numba(name, hk):
    t = golden(f"trace_{name}")
    n = int(t["n"])
    stack, _ = _stack(t, n + 1)
    X, V = t["Xin"].copy(), t["Vin"].copy()
    K.set_backend("b200-parity")
    ev = K.trace_backward(stack, float(t["L"]), n, float(t["tau"]), X, V, bool(hk))
    assert ev == int(t[f"evals{hk}"])
    assert np.array_equal(X, t[f"X{hk}"]) and np.array_equal(V, t[f"V{hk}"])


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["kat_wl", "tiny3"])
def test_plugin_fast_backend_close(name):
    t = golden(f"trace_{name}")
    n = int(t["n"])
    stack, _ = _stack(t, n + 1)
    X, V = t["Xin"].copy(), t["Vin"].copy()
    K.set_backend("b200")
    try:
        K.trace_backward(stack, float(t["L"]), n, float(t["tau"]), X, V, True)
    finally:
        K.set_backend("b200-parity")
    scale = max(np.abs(t["X1"]).max(), np.abs(t["V1"]).max())
    assert np.abs(X - t["X1"]).max() <= 1e-11 * scale and np.abs(V - t["V1"]).max() <= 1e-11 * scale


FIELD_CASES = ["kat_wl", "tiny2", "tiny3", "rag1", "rag2", "rag3"]


@pytest.mark.gpu
@pytest.mark.parametrize("name", FIELD_CASES)
def test_spline_field_eval_bit_exact(name):
    """SplineField.eval_phi_many / eval_E_many on the GPU vs the reference (numpy twin,
    kernels.py:84-123) at seeded points and edge positions (0, L, -tiny, nodes, images)."""
    import paper_2301_05581_b200 as nufi
    from paper_2301_05581_b200.configs import workload

    z = golden(f"field_{name}")
    base = golden(name)
    w = workload(name)
    slot = int(z["slot"])
    c = base["coeffs"][slot].reshape(w.grid.shape_x)
    free = nufi.SplineField(grid=w.grid, coeffs=c)  # uploaded into a scratch history
    assert np.array_equal(free.eval_phi_many(z["X"]), z["phi"])
    assert np.array_equal(free.eval_E_many(z["X"]), z["E"])
    h = nufi.PotentialHistory(w.grid, w.tau, capacity=slot + 1)
    h.load_stack(base["coeffs"][: slot + 1].reshape((slot + 1,) + w.grid.shape_x))
    entry = h.entry(slot)  # evaluated in place on the device history
    assert np.array_equal(entry.eval_E_many(z["X"]), z["E"])
    with pytest.raises(UsageError):
        entry.eval_E_many(np.zeros((3, w.grid.d + 1)))


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["kat_wl", "tiny2", "tiny3", "rag1", "rag2", "rag3", "wl3"])
def test_solve_poisson_fit_spline_vs_reference(name):
    """poisson.solve_poisson + spline.fit_spline + electric_energy one by one on the GPU vs
    the reference's outputs (golden coefficients / W) and the pinned oracle (phi, spectrum)."""
    import paper_2301_05581_b200 as nufi
    from oracle import oracle as O
    from paper_2301_05581_b200.configs import workload
    from tests._util import normwise

    g = golden(name)
    if g is None:
        pytest.skip("golden missing")
    w = workload(name)
    for n in (0, 1, min(5, g["rho"].shape[0] - 1)):
        rho = nufi.DensityGrid(w.grid, g["rho"][n].reshape(w.grid.shape_x))
        phi, spec = nufi.solve_poisson(rho)
        phi_o, hat_o = O.solve_poisson(O.case(name), g["rho"][n])
        assert normwise(phi.reshape(1, -1), np.asarray(phi_o).reshape(1, -1))[0] <= 1e-12
        assert np.abs(spec.coeffs.reshape(-1) - np.asarray(hat_o).reshape(-1)).max() <= 1e-12 * np.abs(hat_o).max()
        assert abs(nufi.electric_energy(spec) / g["W"][n] - 1) <= 1e-12
        fit = nufi.fit_spline(phi, w.grid)
        assert normwise(np.asarray(fit.coeffs).reshape(1, -1), g["coeffs"][n: n + 1])[0] <= 1e-10
    with pytest.raises(nufi.NumericalConsistencyError):
        nufi.solve_poisson(nufi.DensityGrid(w.grid, np.full(w.grid.shape_x, 0.3)))


@pytest.mark.gpu
def test_poisson_eigenfunction_kat():
    """rho = cos(2 pi x / L) -> phi = (L / 2 pi)^2 cos(2 pi x / L)."""
    import math

    import paper_2301_05581_b200 as nufi

    grid = nufi.GridSpec(d=1, L=4 * math.pi, Nx=32, Nv=8, vmax=1.0)
    x = np.arange(32) * grid.hx
    rho = np.cos(2 * math.pi * x / grid.L)
    phi, _ = nufi.solve_poisson(nufi.DensityGrid(grid, rho))
    ref = (grid.L / (2 * math.pi)) ** 2 * rho
    assert np.abs(phi - ref).max() <= 1e-14 * np.abs(ref).max()
