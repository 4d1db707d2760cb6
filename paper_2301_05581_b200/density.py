"""Charge density on the x-grid: the drop-in for density.compute_rho.

compute_rho(ctx, n) -> RhoResult has the reference's signature and result type
(density.py:64-91).  The whole quadrature — Psi-tilde trace of all
Nx^d * Nv^d points through history rows 0..n-1, f0 at the foot points, the
v-sum and the neutralisation — runs in libnufi_b200 (nufi_rho ->
csrc/trace_rho.cu + csrc/field_update.cu); only the Nx^d densities and three
scalars come back to the host.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from .errors import UsageError
from .flow import FlowContext
from .grids import GridSpec

DEFAULT_CHUNK = 1 << 21  # density.py:27 (accepted for signature parity; the GPU path does not chunk)


@dataclass(frozen=True)
class DensityGrid:
    """rho at the Nx^d nodes, row-major (poisson.py:19-32)."""

    grid: GridSpec
    values: np.ndarray

    def __post_init__(self):
        vals = np.asarray(self.values, dtype=np.float64)
        if vals.shape != self.grid.shape_x:
            raise UsageError(f"values must have shape {self.grid.shape_x}, got {vals.shape}")
        if not np.isfinite(vals).all():
            raise UsageError("density values must be finite")
        object.__setattr__(self, "values", vals)


@dataclass(frozen=True)
class RhoResult:
    """density.py:64-69"""

    density: DensityGrid
    neutralization: float
    f_min: float
    f_max: float


def compute_rho(ctx: FlowContext, n: int, chunk: int = DEFAULT_CHUNK) -> RhoResult:
    """Charge density at step n, neutralised to zero nodal mean (density.py:72-91)."""
    grid = ctx.grid
    rho = np.empty(grid.n_nodes)
    stats = np.empty(3)
    evals = ctypes.c_int64(0)
    ctx.history.handle.call("nufi_rho", int(n), rho.ctypes.data, stats.ctypes.data, ctypes.byref(evals))
    ctx.field_evals += int(evals.value)
    return RhoResult(density=DensityGrid(grid=grid, values=rho.reshape(grid.shape_x)),
                     neutralization=float(stats[0]), f_min=float(stats[1]), f_max=float(stats[2]))
