"""Conserved / tracked quantities per step and the damping-rate fit.

The reference package declares this module in SPEC but does not ship it; its
building block is density.quadrature_sweep_many (density.py:104-120).  Here
the phase-space integrals come from one fused GPU sweep (conserved_moments ->
nufi_moments, csrc/trace_rho.cu MOM variant): Psi trace of every quadrature
point, f0 at the foot point, fixed-order sums of f, f^2, f ln f, |v|^2 f / 2,
v f.  electric_energy is the Parseval sum of poisson.py:115-120 evaluated from
the stored coefficient slab of step n (Nx^d values).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .density import conserved_moments
from .errors import FitError, UsageError
from .flow import FlowContext
from .grids import GridSpec


@dataclass(frozen=True)
class DiagnosticsRecord:
    """SPEC.md:399-402.  entropy is int f ln f (the SPEC weight, 0 ln 0 := 0);
    linf_observed is the max over quadrature points (an underestimate of sup f)."""

    step: int
    t: float
    electric_energy: float
    kinetic_energy: float
    total_energy: float
    l1_norm: float
    l2_norm: float
    linf_observed: float
    entropy: float
    momentum: np.ndarray
    neutralization_constant: float


def _wavenumber_squared(grid: GridSpec) -> np.ndarray:
    """|2 pi alpha / L|^2 on the FFT grid (poisson.py:52-59)."""
    m = np.fft.fftfreq(grid.Nx, d=1.0 / grid.Nx)
    k = 2.0 * np.pi * m / grid.L
    k2 = np.zeros((grid.Nx,) * grid.d)
    for a in range(grid.d):
        shape = [1] * grid.d
        shape[a] = grid.Nx
        k2 = k2 + (k * k).reshape(shape)
    return k2


def electric_energy_from_coeffs(grid: GridSpec, coeffs: np.ndarray) -> float:
    """W = 1/2 L^d sum_alpha k^2 |phi_hat_alpha|^2 (poisson.py:115-120) from a spline slab.

    fit_spline divides the spectrum of phi by prod_a sym(alpha_a) (spline.py:20-25,
    78-84) and phi's spectrum is phi_hat N^d (poisson.py:85-87), so
    phi_hat = fft(c) prod_a sym / N^d."""
    c = np.asarray(coeffs, dtype=np.float64).reshape((grid.Nx,) * grid.d)
    N = grid.Nx
    sym1 = (4.0 + 2.0 * np.cos(2.0 * np.pi * np.arange(N) / N)) / 6.0
    sym = np.ones((N,) * grid.d)
    for a in range(grid.d):
        shape = [1] * grid.d
        shape[a] = N
        sym = sym * sym1.reshape(shape)
    phi_hat = np.fft.fftn(c) * sym / float(N ** grid.d)
    return float(0.5 * grid.L ** grid.d * np.add.reduce((_wavenumber_squared(grid) * np.abs(phi_hat) ** 2).ravel()))


def conserved_quantities(ctx: FlowContext, n: int, electric_energy: float | None = None,
                         neutralization: float = 0.0) -> DiagnosticsRecord:
    """SPEC.md:403-410 conserved_quantities(ctx, n): needs step n completed (field n stored)."""
    if len(ctx.history) < n + 1:
        raise UsageError(f"conserved_quantities at step {n} needs fields 0..{n}; history holds {len(ctx.history)}")
    m = conserved_moments(ctx, n)
    if electric_energy is None:
        electric_energy = electric_energy_from_coeffs(ctx.grid, ctx.history.entry(n).coeffs)
    W = float(electric_energy)
    return DiagnosticsRecord(step=int(n), t=n * ctx.tau, electric_energy=W, kinetic_energy=m.kinetic,
                             total_energy=m.kinetic + W, l1_norm=m.l1, l2_norm=math.sqrt(max(m.f2, 0.0)),
                             linf_observed=m.f_max, entropy=m.f_ln_f, momentum=m.momentum,
                             neutralization_constant=float(neutralization))


def fit_damping_rate(t, energy, window) -> float:
    """negated least-squares slope of log(energy) through its local
    maxima inside window [t_lo, t_hi]; a sample is a maximum if strictly greater than
    both neighbours (ties broken toward the earlier sample).  Fewer than 3 peaks ->
    FitError."""
    t = np.asarray(t, dtype=np.float64)
    e = np.asarray(energy, dtype=np.float64)
    if t.shape != e.shape or t.ndim != 1:
        raise UsageError("t and energy must be 1-d arrays of equal length")
    if np.any(np.diff(t) <= 0):
        raise UsageError("times must be strictly increasing")
    lo, hi = window
    inside = (t >= lo) & (t <= hi)
    if inside.sum() >= 3 and np.all(e[inside] == e[inside][0]):
        return 0.0  # constant series: all peaks equal
    with np.errstate(divide="ignore"):
        y = np.log(e)
    peaks = []
    i = 1
    while i < len(y) - 1:
        if lo <= t[i] <= hi and y[i] > y[i - 1]:
            # plateau: extend while equal, a maximum if it then falls (earliest sample kept)
            j = i
            while j + 1 < len(y) and y[j + 1] == y[i]:
                j += 1
            if j + 1 < len(y) and y[j + 1] < y[i]:
                peaks.append(i)
            i = j + 1
            continue
        i += 1
    if len(peaks) < 3:
        raise FitError(f"need at least 3 local maxima in the window, found {len(peaks)}")
    tp, yp = t[peaks], y[peaks]
    slope = np.polyfit(tp, yp, 1)[0]
    return float(-slope)
