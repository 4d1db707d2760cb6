"""Pin the CPU oracle against the reference's golden vectors (CPU only).

tests/golden/*.npz were produced by tests/golden/make_golden.py running the
unmodified reference (vpflow, numba backend) in the build container.  The
oracle restates that arithmetic (oracle/nufi_oracle.c + oracle/oracle.py), so
on the same host it must reproduce the goldens bit for bit; across hosts numpy's
exp/cos may differ by 1 ulp, hence the 1e-12 fallback bound.
"""

import math

import numpy as np
import pytest

from oracle import oracle as O
from tests._util import golden, normwise

TRACE_CASES = ["kat_wl", "tiny2", "tiny3", "wl3r", "rag1", "rag2", "rag3", "big3"]
LOOP_CASES = ["kat_wl", "eq1", "tiny2", "tiny3", "wl1", "kat_wl_f32", "tiny2_f32", "rag1", "rag2", "rag3", "big1",
              "big2", "big2g", "big3"]


@pytest.fixture(scope="module", autouse=True)
def _oracle_built():
    O.max_threads()  # raises if liboracle_nufi.so is missing


@pytest.mark.parametrize("name", TRACE_CASES)
@pytest.mark.parametrize("hk", [0, 1])
def test_trace_bit_exact_vs_numba(name, hk):
    t = golden(f"trace_{name}")
    if t is None:
        pytest.skip("trace golden not generated")
    n = int(t["n"])
    coeffs = t["coeffs"]
    X = t["Xin"].copy()
    V = t["Vin"].copy()
    ev = O.trace_backward(coeffs[: n + 1] if hk else coeffs[:n], float(t["L"]), n, float(t["tau"]), X, V, hk)
    assert ev == int(t[f"evals{hk}"])
    assert np.array_equal(X, t[f"X{hk}"])
    assert np.array_equal(V, t[f"V{hk}"])


@pytest.mark.parametrize("name", ["kat_wl", "tiny2"])
def test_numpy_twin_vs_numba(name):
    """The reference's two backends (kernels.py:4-6): bit-identical in d=1, ~1e-16 in d=2."""
    t = golden(f"trace_{name}")
    for hk in (0, 1):
        assert np.abs(t[f"Xnp{hk}"] - t[f"X{hk}"]).max() <= 1e-13 * np.abs(t[f"X{hk}"]).max()
        assert np.abs(t[f"Vnp{hk}"] - t[f"V{hk}"]).max() <= 1e-13 * np.abs(t[f"V{hk}"]).max()


def test_trace_numpy_twin_matches_c():
    t = golden("trace_kat_wl")
    n = int(t["n"])
    coeffs = t["coeffs"]
    X, V = t["Xin"].copy(), t["Vin"].copy()
    O.trace_numpy(coeffs.reshape(n + 1, -1), float(t["L"]), n, float(t["tau"]), X, V, True)
    assert np.array_equal(X, t["X1"]) and np.array_equal(V, t["V1"])


@pytest.mark.parametrize("name", LOOP_CASES)
def test_loop_vs_reference(name):
    g = golden(name)
    if g is None:
        pytest.skip("golden not generated")
    N = len(g["W"]) - 1
    keep = g["rho"].shape[0]
    run = O.OracleRun(O.case(name), f32=name.endswith("_f32")).run(N, keep)
    assert normwise(run["rho"], g["rho"]).max() <= 1e-12
    assert normwise(run["coeffs"], g["coeffs"]).max() <= 1e-12
    assert normwise(run["E"], g["E"]).max() <= 1e-12
    W, Wg = run["W"], g["W"]
    assert np.all(np.abs(W - Wg) <= 1e-12 * np.maximum(np.abs(Wg), 1e-300))
    assert np.abs(run["stats"] - g["stats"]).max() <= 1e-12


def test_rho_bar_matches_reference():
    for name in ["kat_wl", "wl1", "tiny3"]:
        g = golden(name)
        assert abs(O.background_density(O.case(name)) - float(g["rho_bar"])) <= 1e-15


def test_field_evals_counter():
    """compute_rho adds P*n per step: total P*N(N+1)/2."""
    g = golden("wl1")
    c = O.case("wl1")
    assert int(g["field_evals"][-1]) == O.point_steps(c, 240) == 473_825_280


# ---- SPEC known-answer tests re-verified on the oracle ----

def test_kat_energy_t0():
    """W(0) = alpha^2 L / (4 k^2)."""
    exact = 0.01 ** 2 * 4 * math.pi / (4 * 0.25)
    assert abs(golden("kat_wl")["W"][0] / exact - 1) < 1e-12
    assert abs(golden("wl1")["W"][0] / exact - 1) < 1e-8


def test_kat_rho_t0():
    """rho(0, x_i) = -alpha cos(k x_i)."""
    c = O.case("kat_wl")
    x = O.x_node_matrix(c)[:, 0]
    assert np.abs(golden("kat_wl")["rho"][0] + 0.01 * np.cos(0.5 * x)).max() < 1e-12


def test_kat_poisson_eigenfunction():
    """rho = cos(2 pi x / L) => phi = (L / 2 pi)^2 cos(2 pi x / L)."""
    c = O.case("kat_wl")
    x = O.x_node_matrix(c)[:, 0]
    rho = np.cos(2 * np.pi * x / c.L)
    phi, _ = O.solve_poisson(c, rho)
    assert np.abs(phi - (c.L / (2 * np.pi)) ** 2 * rho).max() < 1e-12 * (c.L / (2 * np.pi)) ** 2


def test_kat_equilibrium():
    """alpha = 0: W < 1e-20 at every step."""
    assert np.all(golden("eq1")["W"] < 1e-20)


@pytest.mark.parametrize("name", ["kat_wl", "tiny2", "tiny3", "wl3r", "rag1", "rag2", "rag3"])
def test_sweep_vs_reference(name):
    """Oracle quadrature_sweep_many (Psi) vs the reference's, conserved-quantity weights."""
    z = golden(f"sweep_{name}")
    base = golden(name)
    if z is None or base is None:
        pytest.skip("sweep golden missing")
    c = O.case(name)
    run = O.OracleRun(c)
    stack = base["coeffs"]
    for i, n in enumerate(z["steps"]):
        run.field_evals = 0
        f, f2, flnf, kin, mom = run.quadrature_sweep_many(int(n), O.conserved_weights(), stack=stack)
        got = np.array([f, f2, flnf, kin] + list(np.atleast_1d(mom)))
        ref = z["moments"][i]
        scale = np.abs(ref[:4]).max()
        assert np.abs(got - ref).max() <= 1e-12 * scale, (n, got - ref)
        assert run.field_evals == int(z["field_evals"][i])


@pytest.mark.parametrize("base", ["kat_wl", "tiny2", "tiny3"])
def test_generic_trace_matches_reference_install_field(base):
    """flow.py:65-82 with UniformField overrides (flow.py:44-47): the oracle's restatement
    against the reference's own output (tests/golden/hook_*.npz), bit for bit."""
    z = golden(f"hook_{base}")
    ref = golden(base)
    c = O.case(base)
    n = int(z["n"])
    stack = ref["coeffs"].reshape((-1,) + (c.Nx,) * c.d)
    fields = {k: stack[k] for k in range(n + 1)}
    for s, e in zip(z["slots"], z["E0"]):
        fields[int(s)] = ("uniform", e)
    for half, kx, kv in ((True, "X_psi", "V_psi"), (False, "X_tilde", "V_tilde")):
        X, V = z["x"].copy(), z["v"].copy()
        O.trace_generic(fields, c.L, n, c.tau, X, V, half)
        assert np.array_equal(X, z[kx]) and np.array_equal(V, z[kv])
    Xu, Vu = z["x"].copy(), z["v"].copy()
    O.trace_generic({k: ("uniform", z["E_uniform"]) for k in range(n + 1)}, c.L, n, c.tau, Xu, Vu, True)
    assert np.array_equal(Xu, z["X_uniform"]) and np.array_equal(Vu, z["V_uniform"])


def test_wl3_full_size_golden_consistent():
    """The full-size d = 3 fixture (16^3 x 32^3, generated by the unmodified reference for all
    80 steps) against the oracle's Poisson / spline restatement on its own densities, the
    evaluation counter and the background density (no trace: 134M points per step)."""
    g = golden("wl3")
    if g is None:
        pytest.skip("golden not generated")
    c = O.case("wl3")
    N = len(g["W"]) - 1
    keep = g["rho"].shape[0]
    for n in range(0, keep, 5):
        phi, hat = O.solve_poisson(c, g["rho"][n].reshape((c.Nx,) * 3))
        coeffs = O.fit_spline(c, phi)
        assert normwise(np.asarray(coeffs).reshape(1, -1), g["coeffs"][n:n + 1])[0] <= 1e-12
        W = O.electric_energy(c, hat)
        assert abs(W - g["W"][n]) <= 1e-12 * abs(g["W"][n])
    assert int(g["field_evals"][-1]) == O.point_steps(c, N)
    assert abs(O.background_density(c) - float(g["rho_bar"])) <= 1e-15
