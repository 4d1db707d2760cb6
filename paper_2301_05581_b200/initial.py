"""Initial-condition descriptors (the IC "callback" of the drop-in API).

The reference evaluates f0 with numpy (initial.py:165-180).  Here an initial
condition is a *descriptor* of the same closed family — per-axis Gaussian
mixtures times v^0 or v^2, times 1 + alpha * sum_a cos(k x_a) — that is shipped
to the GPU in nufi_config and evaluated at the foot point inside the trace
kernel (nufi_internal.cuh eval_f0).  Same names, parameters and validation as
the reference: VelocityProfile (initial.py:25-56), InitialCondition
(initial.py:72-106), BENCHMARK_DEFAULTS / make_benchmark (initial.py:112-162).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .errors import UsageError

GAUSS_NORM = 1.0 / math.sqrt(2.0 * math.pi)  # initial.py:22
MAX_CENTERS = 4  # nufi.h NUFI_MAX_CENTERS


@dataclass(frozen=True)
class VelocityProfile:
    """One velocity axis: v^power * sum_m weights[m] * N(v; centers[m], 1)."""

    centers: tuple = (0.0,)
    weights: tuple = (1.0,)
    power: int = 0

    def __post_init__(self):
        object.__setattr__(self, "centers", tuple(float(c) for c in self.centers))
        object.__setattr__(self, "weights", tuple(float(w) for w in self.weights))
        if not self.centers or len(self.centers) != len(self.weights):
            raise UsageError("centers and weights must be non-empty and equal-length")
        if self.power not in (0, 2):
            raise UsageError(f"velocity power must be 0 or 2, got {self.power}")
        if min(self.weights) <= 0:
            raise UsageError("mixture weights must be positive")
        if len(self.centers) > MAX_CENTERS:
            raise UsageError(f"at most {MAX_CENTERS} mixture centers per axis")

    def moment0(self) -> float:
        """Exact integral over the real line (initial.py:51-56)."""
        if self.power == 0:
            return float(sum(self.weights))
        return float(sum(w * (1.0 + c * c) for c, w in zip(self.centers, self.weights)))


@dataclass(frozen=True)
class InitialCondition:
    """f0 = prod_a profile_a(v_a) * (1 + alpha * sum_a cos(k x_a)) on [0, L)^d."""

    benchmark: str
    d: int
    L: float
    alpha: float
    k: float
    profiles: tuple
    v0: float | None = None
    rho_bar: float = field(init=False)

    def __post_init__(self):
        # initial.py:89-106
        if len(self.profiles) != self.d:
            raise UsageError(f"need {self.d} velocity profiles, got {len(self.profiles)}")
        if self.alpha < 0:
            raise UsageError(f"perturbation amplitude must be >= 0, got {self.alpha}")
        if self.alpha * self.d > 1.0 + 1e-12:
            raise UsageError(f"alpha*d = {self.alpha * self.d} > 1 makes f0 negative")
        turns = self.k * self.L / (2.0 * math.pi)
        if abs(turns - round(turns)) > 1e-9:
            raise UsageError(f"k*L = {self.k * self.L} is not a multiple of 2*pi; f0 would not be x-periodic")
        rb = math.prod(p.moment0() for p in self.profiles)
        if not rb > 0:
            raise UsageError("background density must be positive")
        object.__setattr__(self, "rho_bar", rb)


# initial.py:112-117
BENCHMARK_DEFAULTS: dict = {
    "weak_landau_1d": dict(d=1, L=4.0 * math.pi, alpha=0.01, k=0.5, v0=None),
    "two_stream_1d": dict(d=1, L=4.0 * math.pi, alpha=0.01, k=0.5, v0=None),
    "strong_landau_2d": dict(d=2, L=4.0 * math.pi, alpha=0.5, k=0.5, v0=None),
    "two_stream_3d": dict(d=3, L=10.0 * math.pi, alpha=1e-3, k=0.2, v0=2.4),
}


def _profiles(name: str, d: int, v0):
    if name == "two_stream_1d":
        return (VelocityProfile(power=2),)
    if name == "two_stream_3d":
        return (VelocityProfile(), VelocityProfile(centers=(-v0, v0), weights=(0.5, 0.5)), VelocityProfile())
    return (VelocityProfile(),) * d


def make_benchmark(name: str, *, L=None, alpha=None, k=None, v0=None) -> InitialCondition:
    """Named benchmark with optional overrides (initial.py:132-162)."""
    if name not in BENCHMARK_DEFAULTS:
        raise UsageError(f"unknown benchmark {name!r}; known: {', '.join(sorted(BENCHMARK_DEFAULTS))}")
    prm = dict(BENCHMARK_DEFAULTS[name])
    for key, val in (("L", L), ("alpha", alpha), ("k", k), ("v0", v0)):
        if val is not None:
            prm[key] = val
    return InitialCondition(benchmark=name, d=prm["d"], L=prm["L"], alpha=prm["alpha"], k=prm["k"],
                            v0=prm["v0"], profiles=_profiles(name, prm["d"], prm["v0"]))


def weak_landau_3d(alpha: float = 0.01, k: float = 0.5, L: float = 4.0 * math.pi) -> InitialCondition:
    """The BASELINE 'd=3 weak Landau' case: not a reference built-in, built the
    way SURVEY.md §8(d) maps it onto InitialCondition (initial.py:72-106)."""
    return InitialCondition(benchmark="weak_landau_3d", d=3, L=L, alpha=alpha, k=k,
                            profiles=(VelocityProfile(),) * 3)


# ---------------------------------------------------------------------------
# f0 and the background density on the device (the reference's module functions)
# ---------------------------------------------------------------------------

_f0_handles: dict = {}
_rho_bar_cache: dict = {}


def _f0_history(ic: InitialCondition):
    """A 1-slab device handle carrying ic's f0 descriptor (cached per initial condition)."""
    h = _f0_handles.get(ic)
    if h is None:
        from .grids import GridSpec
        from .spline import PotentialHistory

        g = GridSpec(d=ic.d, L=ic.L, Nx=4, Nv=2, vmax=1.0)  # only d and L matter for f0
        h = PotentialHistory(g, 1.0, capacity=1)
        h.bind(ic, rho_bar=ic.rho_bar)
        _f0_handles[ic] = h
    return h


def eval_f0(ic: InitialCondition, x, v) -> np.ndarray:
    """f0 at positions x and velocities v of shape (..., d) (initial.py:165-180), evaluated by
    the device kernel (nufi_eval_f0) on the unwrapped x.  Returns shape (...)."""
    x = np.asarray(x, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    if x.shape != v.shape or x.shape[-1:] != (ic.d,):
        raise UsageError(f"x and v must both end in a length-{ic.d} axis")
    X = np.ascontiguousarray(x.reshape(-1, ic.d))
    V = np.ascontiguousarray(v.reshape(-1, ic.d))
    F = np.empty(X.shape[0])
    if F.size:
        _f0_history(ic).handle.call("nufi_eval_f0", X.ctypes.data, V.ctypes.data, int(X.shape[0]), F.ctypes.data)
    return F.reshape(x.shape[:-1])


def f0_at(ic: InitialCondition, p) -> float:
    """f0 at one PhasePoint (initial.py:183-184)."""
    return float(eval_f0(ic, p.x, p.v))


def background_density(ic: InitialCondition, grid) -> float:
    """Midpoint-quadrature background density on the run's phase grid (initial.py:187-208),
    computed by the device's rho_bar kernel (the reference's factorised x-sum x v-sum)."""
    if grid.d != ic.d:
        raise UsageError(f"grid dimension {grid.d} does not match benchmark dimension {ic.d}")
    key = (ic, grid)
    if key not in _rho_bar_cache:
        from .spline import PotentialHistory

        h = PotentialHistory(grid, 1.0, capacity=1)
        _rho_bar_cache[key] = h.bind(ic)
    return _rho_bar_cache[key]
