"""CPU oracle: a restatement of the reference's hot path (vpflow) in numpy + C.

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / `--impl reference` legs may import this module, and only as the
checker (or as the timed CPU baseline, cpu_baseline.kind = "port").  The
product path (paper_2301_05581_b200) never imports it.

Every function cites the reference file:line it restates
(/root/reference/pkg/src/vpflow/...).  The backward trace runs in
oracle/nufi_oracle.c (bit-exact restatement of the numba kernels); everything
else is the same numpy arithmetic the reference performs.

Pinning: tests/test_oracle.py checks this module against the golden fixtures
in tests/golden/ that tests/golden/make_golden.py produced by running the
unmodified reference in the build container (trace bit-exact; rho / spline
coefficients / E / W per step bit-exact or within 1e-13 on the same host).
"""

from __future__ import annotations

import ctypes
import itertools
import math
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
GAUSS_NORM = 1.0 / math.sqrt(2.0 * math.pi)  # initial.py:22
DEFAULT_CHUNK = 1 << 21  # density.py:27


# ---------------------------------------------------------------------------
# configuration (grids.py:18-59, initial.py:25-106)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class Profile:
    """initial.py:25-56 VelocityProfile (centers, weights, power)."""

    centers: tuple = (0.0,)
    weights: tuple = (1.0,)
    power: int = 0


@dataclass(frozen=True)
class Case:
    """GridSpec (grids.py:18-59) + InitialCondition (initial.py:72-106) + tau."""

    d: int
    L: float
    Nx: int
    Nv: int
    vmax: float
    tau: float
    alpha: float
    k: float
    profiles: tuple = field(default=())

    @property
    def hx(self) -> float:  # grids.py:37-38
        return self.L / self.Nx

    @property
    def hv(self) -> float:  # grids.py:41-42
        return 2.0 * self.vmax / self.Nv

    @property
    def n_nodes(self) -> int:
        return self.Nx ** self.d

    @property
    def n_cells(self) -> int:
        return self.Nv ** self.d


# BASELINE configs + small parity cases (tests/golden/make_golden.py)
_MAX = Profile()
_TS1 = Profile(power=2)
FOUR_PI = 4.0 * math.pi


def case(name: str) -> Case:
    if name.endswith("_f32"):  # FP32 history variants: same case, OracleRun(..., f32=True)
        return case(name[: -len("_f32")])
    if name == "wl1":
        return Case(1, FOUR_PI, 64, 256, 6.0, 1 / 8, 0.01, 0.5, (_MAX,))
    if name == "ts1":
        return Case(1, FOUR_PI, 64, 512, 10.0, 1 / 16, 0.01, 0.5, (_TS1,))
    if name == "sl1":
        return Case(1, FOUR_PI, 256, 2048, 8.0, 1 / 16, 0.5, 0.5, (_MAX,))
    if name == "wl2":
        return Case(2, FOUR_PI, 32, 64, 6.0, 1 / 8, 0.01, 0.5, (_MAX,) * 2)
    if name == "wl3":
        return Case(3, FOUR_PI, 16, 32, 6.0, 1 / 8, 0.01, 0.5, (_MAX,) * 3)
    if name == "wl3r":
        return Case(3, FOUR_PI, 16, 8, 6.0, 1 / 8, 0.01, 0.5, (_MAX,) * 3)
    if name == "kat_wl":
        return Case(1, FOUR_PI, 32, 128, 10.0, 1 / 16, 0.01, 0.5, (_MAX,))
    if name == "eq1":
        return Case(1, FOUR_PI, 32, 128, 10.0, 1 / 16, 0.0, 0.5, (_MAX,))
    if name == "tiny2":
        return Case(2, FOUR_PI, 8, 8, 6.0, 1 / 8, 0.5, 0.5, (_MAX,) * 2)
    if name == "tiny3":
        streams = Profile(centers=(-2.4, 2.4), weights=(0.5, 0.5))
        return Case(3, 10.0 * math.pi, 8, 4, 6.0, 1 / 8, 1e-3, 0.2, (_MAX, streams, _MAX))
    if name == "big1":
        return Case(1, FOUR_PI, 5000, 16, 6.0, 1 / 8, 0.05, 0.5, (_MAX,))
    if name == "big2":
        return Case(2, FOUR_PI, 72, 6, 6.0, 1 / 8, 0.2, 0.5, (_MAX,) * 2)
    if name == "big2g":
        return Case(2, FOUR_PI, 120, 4, 6.0, 1 / 8, 0.2, 0.5, (_MAX,) * 2)
    if name == "big3":
        return Case(3, FOUR_PI, 22, 3, 5.0, 1 / 8, 0.05, 0.5, (_MAX,) * 3)
    if name == "rag1":
        return Case(1, FOUR_PI, 24, 40, 6.0, 1 / 8, 0.05, 0.5, (_MAX,))
    if name == "rag2":
        return Case(2, FOUR_PI, 6, 10, 6.0, 1 / 8, 0.3, 0.5, (_MAX,) * 2)
    if name == "rag3":
        return Case(3, FOUR_PI, 5, 3, 5.0, 1 / 8, 0.05, 0.5, (_MAX,) * 3)
    raise KeyError(name)


# ---------------------------------------------------------------------------
# grids.py:104-115
# ---------------------------------------------------------------------------

def x_node_matrix(c: Case) -> np.ndarray:
    axes = [np.arange(c.Nx) * c.hx] * c.d
    mesh = np.meshgrid(*axes, indexing="ij")
    return np.stack([m.reshape(-1) for m in mesh], axis=-1)


def v_mid_matrix(c: Case) -> np.ndarray:
    ax = -c.vmax + (np.arange(c.Nv) + 0.5) * c.hv
    mesh = np.meshgrid(*([ax] * c.d), indexing="ij")
    return np.stack([m.reshape(-1) for m in mesh], axis=-1)


# ---------------------------------------------------------------------------
# initial.py
# ---------------------------------------------------------------------------

def velocity_factor(p: Profile, v: np.ndarray) -> np.ndarray:
    """initial.py:41-49"""
    v = np.asarray(v, dtype=np.float64)
    out = np.zeros_like(v)
    for cc, w in zip(p.centers, p.weights):
        out += w * np.exp(-0.5 * (v - cc) ** 2)
    out *= GAUSS_NORM
    if p.power:
        out = out * v ** p.power
    return out


def eval_f0(c: Case, x: np.ndarray, v: np.ndarray) -> np.ndarray:
    """initial.py:165-180 (x is NOT wrapped)."""
    vel = velocity_factor(c.profiles[0], v[..., 0])
    for a in range(1, c.d):
        vel = vel * velocity_factor(c.profiles[a], v[..., a])
    pert = np.cos(c.k * x[..., 0])
    for a in range(1, c.d):
        pert = pert + np.cos(c.k * x[..., a])
    return vel * (1.0 + c.alpha * pert)


def background_density(c: Case) -> float:
    """initial.py:187-208 (quadrature rho_bar, fixed once per run, flow.py:36-39)."""
    X = x_node_matrix(c)
    V = v_mid_matrix(c)
    vel = velocity_factor(c.profiles[0], V[:, 0])
    for a in range(1, c.d):
        vel = vel * velocity_factor(c.profiles[a], V[:, a])
    pert = np.cos(c.k * X[:, 0])
    for a in range(1, c.d):
        pert = pert + np.cos(c.k * X[:, a])
    sum_v = float(np.add.reduce(vel))
    sum_x = float(np.add.reduce(1.0 + c.alpha * pert))
    total = sum_x * sum_v * c.hx ** c.d * c.hv ** c.d
    return total / c.L ** c.d


# ---------------------------------------------------------------------------
# kernels.py: trace (C restatement) and the numpy twin
# ---------------------------------------------------------------------------

_LIB = None


def _lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(HERE, "liboracle_nufi.so")
        if not os.path.exists(path):
            raise RuntimeError(f"oracle library missing: run `make -C {HERE}`")
        lib = ctypes.CDLL(path)
        lib.oracle_trace.restype = ctypes.c_int64
        lib.oracle_trace.argtypes = [
            ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int64, ctypes.c_double,
            ctypes.c_int64, ctypes.c_double, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
            ctypes.c_int, ctypes.c_int,
        ]
        lib.oracle_max_threads.restype = ctypes.c_int
        _LIB = lib
    return _LIB


def max_threads() -> int:
    """Every host thread this process may run on (not OMP_NUM_THREADS: torchrun sets it to 1
    for each rank, and the CPU baseline should use the whole host)."""
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except (AttributeError, OSError):  # pragma: no cover - non-Linux
        return max(1, os.cpu_count() or int(_lib().oracle_max_threads()))


def trace_backward(coeffs, L, n, tau, X, V, half_kick, threads=0) -> int:
    """kernels.py:390-412 with the numba kernels _trace_1d/2d/3d (kernels.py:184-387)."""
    if n == 0:
        return 0
    coeffs = np.ascontiguousarray(coeffs, dtype=np.float64)
    rows = coeffs.shape[0]
    need = n + 1 if half_kick else n
    if rows < need:
        raise ValueError(f"need {need} stored fields for step {n}, have {rows}")
    assert X.flags.c_contiguous and V.flags.c_contiguous and X.dtype == np.float64
    M, d = X.shape
    if M == 0:
        return 0
    N = int(round(coeffs[0].size ** (1.0 / d)))
    assert N ** d == coeffs[0].size, "coefficient slab is not (Nx,)*d"
    r = _lib().oracle_trace(coeffs.ctypes.data, rows, d, N, float(L), int(n), float(tau),
                            X.ctypes.data, V.ctypes.data, M, int(bool(half_kick)), int(threads))
    if r < 0:
        raise ValueError("history too short")
    return int(r)


def _locate(x, L, N):
    """kernels.py:52-59"""
    u = np.mod(x, L)
    u[u >= L] = 0.0
    t = u * (N / L)
    i = t.astype(np.int64)
    np.minimum(i, N - 1, out=i)
    return i, t - i


def bspline_weights(t):
    """kernels.py:62-70"""
    s = 1.0 - t
    w = np.empty((4,) + t.shape)
    w[0] = s * s * s / 6.0
    w[1] = 2.0 / 3.0 - t * t * (1.0 - 0.5 * t)
    w[2] = 2.0 / 3.0 - s * s * (1.0 - 0.5 * s)
    w[3] = t * t * t / 6.0
    return w


def bspline_dweights(t):
    """kernels.py:73-81"""
    s = 1.0 - t
    w = np.empty((4,) + t.shape)
    w[0] = -0.5 * s * s
    w[1] = t * (1.5 * t - 2.0)
    w[2] = s * (2.0 - 1.5 * s)
    w[3] = 0.5 * t * t
    return w


def eval_E_many(coeffs, L, X):
    """kernels.py:102-123: minus the spline gradient (the per-step E-at-nodes output)."""
    d = X.shape[1]
    N = coeffs.shape[0]
    inv_h = N / L
    loc = [_locate(np.array(X[:, a], dtype=np.float64), L, N) for a in range(d)]
    wts = [bspline_weights(t) for _, t in loc]
    dwts = [bspline_dweights(t) for _, t in loc]
    flat = coeffs.reshape(-1)
    E = np.zeros((X.shape[0], d))
    for offs in itertools.product(range(4), repeat=d):
        idx = (loc[0][0] + (offs[0] - 1)) % N
        for a in range(1, d):
            idx = idx * N + (loc[a][0] + (offs[a] - 1)) % N
        cc = flat[idx]
        for g in range(d):
            w = cc
            for a in range(d):
                w = w * (dwts[a][offs[a]] if a == g else wts[a][offs[a]])
            E[:, g] -= w
    E *= inv_h
    return E


def eval_phi_many(coeffs, L, X):
    """kernels.py:84-99"""
    d = X.shape[1]
    N = coeffs.shape[0]
    loc = [_locate(np.array(X[:, a], dtype=np.float64), L, N) for a in range(d)]
    wts = [bspline_weights(t) for _, t in loc]
    flat = coeffs.reshape(-1)
    out = np.zeros(X.shape[0])
    for offs in itertools.product(range(4), repeat=d):
        idx = (loc[0][0] + (offs[0] - 1)) % N
        w = wts[0][offs[0]]
        for a in range(1, d):
            idx = idx * N + (loc[a][0] + (offs[a] - 1)) % N
            w = w * wts[a][offs[a]]
        out += flat[idx] * w
    return out


def trace_numpy(coeffs, L, n, tau, X, V, half_kick) -> int:
    """kernels.py:126-144 (the reference's vectorised twin)."""
    if n == 0:
        return 0
    M = X.shape[0]
    evals = 0
    half = 0.5 * tau
    if half_kick:
        V += half * eval_E_many(coeffs[n], L, X)
        evals += M
    k = n
    while k > 1:
        k -= 1
        X -= tau * V
        V += tau * eval_E_many(coeffs[k], L, X)
        evals += M
    X -= tau * V
    V += half * eval_E_many(coeffs[0], L, X)
    evals += M
    return evals


def trace_generic(fields, L, n, tau, X, V, half_kick) -> int:
    """flow.py:65-82 (_trace_generic), the reference's trace whenever a non-spline field is
    installed (flow.py:44-47): fields[k] is a stored coefficient slab (SplineField,
    eval_E_many = kernels.py:102-123) or ("uniform", E0) (UniformField, spline.py:55-68)."""
    if n == 0:
        return 0
    M = X.shape[0]

    def E(k):
        f = fields[k]
        if isinstance(f, tuple) and f[0] == "uniform":
            return np.broadcast_to(np.asarray(f[1], dtype=np.float64), (M, X.shape[1])).copy()
        return eval_E_many(f, L, X)

    evals = 0
    if half_kick:
        V += (0.5 * tau) * E(n)
        evals += M
    k = n
    while k > 1:
        k -= 1
        X -= tau * V
        V += tau * E(k)
        evals += M
    X -= tau * V
    V += (0.5 * tau) * E(0)
    evals += M
    return evals


# ---------------------------------------------------------------------------
# poisson.py / spline.py
# ---------------------------------------------------------------------------

def _mode_numbers(c: Case):
    """poisson.py:47-49"""
    return [np.fft.fftfreq(c.Nx, d=1.0 / c.Nx) for _ in range(c.d)]


def wavenumber_squared(c: Case) -> np.ndarray:
    """poisson.py:52-59"""
    scale = 2.0 * np.pi / c.L
    modes = np.meshgrid(*_mode_numbers(c), indexing="ij")
    k2 = np.zeros((c.Nx,) * c.d)
    for m in modes:
        k2 += (scale * m) ** 2
    return k2


def nyquist_mask(c: Case) -> np.ndarray:
    """poisson.py:62-69"""
    mask = np.zeros((c.Nx,) * c.d, dtype=bool)
    if c.Nx % 2 == 0:
        modes = np.meshgrid(*_mode_numbers(c), indexing="ij")
        for m in modes:
            mask |= np.abs(m) == c.Nx // 2
    return mask


def solve_poisson(c: Case, rho: np.ndarray):
    """poisson.py:90-112 -> (phi nodal values, phi spectrum); raises on non-neutral input."""
    rho = np.asarray(rho, dtype=np.float64).reshape((c.Nx,) * c.d)
    mean = float(rho.mean())
    tol = 1e-8 * float(np.max(np.abs(rho)))
    if abs(mean) > tol:
        raise ArithmeticError(f"density is not neutral: {mean:.3e} > {tol:.3e}")
    spec = np.fft.fftn(rho) / c.n_nodes  # poisson.py:72-78
    k2 = wavenumber_squared(c)
    phi_hat = np.zeros_like(spec)
    interior = k2 > 0
    phi_hat[interior] = spec[interior] / k2[interior]
    phi_hat[nyquist_mask(c)] = 0.0
    phi = np.fft.ifftn(phi_hat * c.n_nodes).real  # poisson.py:85-87
    return phi, phi_hat


def electric_energy(c: Case, phi_hat: np.ndarray) -> float:
    """poisson.py:115-120"""
    k2 = wavenumber_squared(c)
    total = np.add.reduce((k2 * np.abs(phi_hat) ** 2).reshape(-1))
    return 0.5 * c.L ** c.d * float(total)


def filter_symbol(N: int) -> np.ndarray:
    """spline.py:20-25"""
    k = np.arange(N)
    return (4.0 + 2.0 * np.cos(2.0 * np.pi * k / N)) / 6.0


def fit_spline(c: Case, phi: np.ndarray) -> np.ndarray:
    """spline.py:71-86 -> coefficient slab (Nx,)*d"""
    sym = filter_symbol(c.Nx)
    hat = np.fft.fftn(phi)
    for axis in range(c.d):
        shape = [1] * c.d
        shape[axis] = c.Nx
        hat = hat / sym.reshape(shape)
    return np.fft.ifftn(hat).real.astype(np.float64)


# ---------------------------------------------------------------------------
# density.py:72-91 and the per-step loop
# ---------------------------------------------------------------------------

class OracleRun:
    """The canonical loop: compute_rho -> solve_poisson -> fit_spline -> append."""

    def __init__(self, c: Case, threads: int = 0, chunk: int = DEFAULT_CHUNK, f32: bool = False):
        self.c = c
        self.f32 = f32  # PotentialHistory(dtype=float32): append casts the slab (spline.py:118-125, 140)
        self.threads = threads
        self.chunk = chunk
        self.rho_bar = background_density(c)
        self.hist = []  # coefficient slabs (Nx,)*d
        self.field_evals = 0
        self._X = x_node_matrix(c)
        self._V = v_mid_matrix(c)

    def stacked(self) -> np.ndarray:
        c = self.c
        if not self.hist:
            return np.zeros((0,) + (c.Nx,) * c.d)
        return np.ascontiguousarray(np.stack(self.hist))

    def compute_rho(self, n: int, node_range=None):
        """density.py:72-91; returns (rho, neutralization, f_min, f_max).

        node_range restricts the sweep to a sub-range of nodes (used for bounded
        CPU-baseline samples); rho is then returned un-neutralized for those nodes.
        """
        c = self.c
        if len(self.hist) < n:
            raise ValueError("history too short")
        hv_d = c.hv ** c.d
        n_cells = c.n_cells
        lo, hi = (0, c.n_nodes) if node_range is None else node_range
        rho = np.empty(hi - lo)
        f_min, f_max = np.inf, -np.inf
        stack = self.stacked()[:n].reshape(n, -1) if n > 0 else None
        nodes_per = max(1, self.chunk // n_cells)
        for start in range(lo, hi, nodes_per):  # density.py:45-61 (node-aligned chunks)
            stop = min(start + nodes_per, hi)
            Xb = np.repeat(self._X[start:stop], n_cells, axis=0)
            Vb = np.tile(self._V, (stop - start, 1))
            if n > 0:
                self.field_evals += trace_backward(stack, c.L, n, c.tau, Xb, Vb, False, self.threads)
            F = eval_f0(c, Xb, Vb)
            per_node = F.reshape(stop - start, n_cells)
            rho[start - lo:stop - lo] = self.rho_bar - hv_d * np.add.reduce(per_node, axis=1)
            f_min = min(f_min, float(per_node.min()))
            f_max = max(f_max, float(per_node.max()))
        if node_range is not None:
            return rho, 0.0, f_min, f_max
        constant = float(rho.mean())
        rho -= constant
        return rho, constant, f_min, f_max

    def quadrature_sweep_many(self, n: int, weights, stack=None):
        """density.py:104-120: Psi-traced (half kick, flow.py:106-112) node-aligned
        batches, weights at the untraced points (density.py:45-61), per-batch
        np.add.reduce, total times hx^d hv^d.  stack: (rows, Nx^d) history
        (default: this run's), needs rows >= n + 1 for n > 0."""
        c = self.c
        stack = self.stacked().reshape(len(self.hist), -1) if stack is None else np.asarray(stack)
        stack = stack.reshape(stack.shape[0], -1)
        if n > 0 and stack.shape[0] < n + 1:
            raise ValueError("history too short for psi")
        n_cells = c.n_cells
        nodes_per = max(1, self.chunk // n_cells)
        totals = [None] * len(weights)
        for start in range(0, c.n_nodes, nodes_per):
            stop = min(start + nodes_per, c.n_nodes)
            Xb = np.repeat(self._X[start:stop], n_cells, axis=0)
            Vb = np.tile(self._V, (stop - start, 1))
            Xt, Vt = Xb.copy(), Vb.copy()
            if n > 0:
                self.field_evals += trace_backward(np.ascontiguousarray(stack[: n + 1]), c.L, n, c.tau, Xt, Vt,
                                                   True, self.threads)
            F = eval_f0(c, Xt, Vt)
            for iw, w in enumerate(weights):
                part = np.add.reduce(np.asarray(w(Xb, Vb, F), dtype=np.float64), axis=0)
                totals[iw] = part if totals[iw] is None else totals[iw] + part
        measure = c.hx ** c.d * c.hv ** c.d
        return [t * measure for t in totals]

    def step(self, n: int):
        """One full step n; returns dict(rho, coeffs, E, W, stats)."""
        c = self.c
        rho, neut, fmin, fmax = self.compute_rho(n)
        phi, phi_hat = solve_poisson(c, rho)
        coeffs = fit_spline(c, phi)
        stored = coeffs.astype(np.float32).astype(np.float64) if self.f32 else coeffs
        self.hist.append(stored)
        W = electric_energy(c, phi_hat)
        E = eval_E_many(coeffs, c.L, self._X)
        return dict(rho=rho, coeffs=stored.reshape(-1), E=E, W=W, stats=(neut, fmin, fmax))

    def run(self, N: int, keep: int | None = None):
        keep = N + 1 if keep is None else keep
        out = dict(rho=[], coeffs=[], E=[], W=[], stats=[])
        for n in range(N + 1):
            s = self.step(n)
            out["W"].append(s["W"])
            out["stats"].append(s["stats"])
            if n < keep:
                out["rho"].append(s["rho"])
                out["coeffs"].append(s["coeffs"])
                out["E"].append(s["E"])
        return {k: np.array(v) for k, v in out.items()}


def conserved_weights():
    """SPEC.md:403-406 weights: f, f^2, f ln f (0 ln 0 := 0), |v|^2 f / 2, v f."""

    def f_ln_f(X, V, F):
        return np.where(F > 0, F * np.log(np.where(F > 0, F, 1.0)), 0.0)

    return [lambda X, V, F: F, lambda X, V, F: F * F, f_ln_f,
            lambda X, V, F: 0.5 * np.sum(V * V, axis=1) * F, lambda X, V, F: V * F[:, None]]


def point_steps(c: Case, N: int) -> int:
    """P * N(N+1)/2; equals the reference's field_evals after the loop."""
    return c.n_nodes * c.n_cells * N * (N + 1) // 2
