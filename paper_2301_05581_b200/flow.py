"""Backward numerical flows through the device-resident history.

Same API as the reference's flow module (flow.py:25-141): FlowContext,
psi_batch / psi_tilde_batch (Psi with / without the leading half kick),
eval_f_batch, point versions, and the field_evals counter.  The trace itself
runs in libnufi_b200 (nufi_trace -> csrc/trace_points.cu); f0 is evaluated on
the device (nufi_eval_f0).

`install_field` (flow.py:44-47, the reference's test hook that overrides a stored
field) takes UniformField (spline.py:55-68) and SplineField objects: while any is
installed, the point-level trace follows the reference's generic path (flow.py:65-82)
on the GPU (csrc/trace_points.cu trace_points_generic), for the constant-force
closed-form tests and field-substitution experiments.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import UsageError
from .grids import GridSpec, PhasePoint
from .initial import InitialCondition, background_density, eval_f0  # noqa: F401  (flow.py:21 re-exports)
from .spline import PotentialHistory

TRACE_FAST = _lib.NUFI_TRACE_FAST
TRACE_PARITY = _lib.NUFI_TRACE_PARITY


@dataclass(eq=False)
class FlowContext:
    """History + initial condition + tau + grid, and the evaluation counter (flow.py:25-53)."""

    history: PotentialHistory
    ic: InitialCondition
    tau: float
    grid: GridSpec
    field_evals: int = 0

    def __post_init__(self):
        if self.grid != self.history.grid:
            raise UsageError("context grid does not match the history grid")
        if float(self.tau) != self.history.tau:
            raise UsageError("context tau does not match the history tau")
        if self.history.ic is not self.ic:
            self.history.bind(self.ic)

    @property
    def rho_bar(self) -> float:
        """Background density from the t = 0 quadrature (flow.py:36-39), computed on the GPU."""
        return self.history.rho_bar

    def reset_counter(self) -> None:
        self.field_evals = 0

    def install_field(self, step: int, fld) -> None:
        """Override the stored field at one step (flow.py:44-47, testing hook).  Accepts a
        UniformField (spline.py:55-68) or a SplineField on this grid (spline.py:28-52; its
        coefficient slab is uploaded and evaluated on the device like eval_E_many), or None
        to remove the override.  The override lives on the history (its device handle), so
        every context over that history sees it.  Other Python field objects cannot be
        evaluated by the device trace and raise UsageError."""
        from .spline import SplineField, UniformField

        if int(step) < 0:
            raise UsageError("step index must be >= 0")
        if fld is None:
            self.history.handle.call("nufi_set_uniform_field", int(step), None)
            return
        if isinstance(fld, SplineField):
            if fld.grid.d != self.grid.d or fld.grid.Nx != self.grid.Nx or fld.grid.L != self.grid.L:
                raise UsageError("SplineField grid (d, Nx, L) does not match the context grid")
            c = np.ascontiguousarray(fld.coeffs, dtype=np.float64).reshape(-1)
            self.history.handle.call("nufi_set_spline_field", int(step), c.ctypes.data)
            return
        if not isinstance(fld, UniformField):
            raise UsageError("the GPU trace accepts UniformField or SplineField overrides only, got "
                             f"{type(fld).__name__}")
        if fld.d != self.grid.d:
            raise UsageError(f"UniformField has {fld.d} components, the grid has d = {self.grid.d}")
        E0 = np.ascontiguousarray(fld.E0, dtype=np.float64)
        self.history.handle.call("nufi_set_uniform_field", int(step), E0.ctypes.data)

    def clear_fields(self) -> None:
        """Remove every installed override."""
        self.history.handle.call("nufi_clear_fields")


def _batch(x, v, d: int):
    X = np.array(np.atleast_2d(np.asarray(x, dtype=np.float64)), copy=True, order="C")
    V = np.array(np.atleast_2d(np.asarray(v, dtype=np.float64)), copy=True, order="C")
    if X.shape != V.shape or X.shape[1] != d:
        raise UsageError(f"x and v must both have shape (M, {d})")
    return X, V


def trace_backward(history: PotentialHistory, n: int, X, V, half_kick: bool, mode: int = TRACE_FAST) -> int:
    """kernels.trace_backward (kernels.py:390-412) on the GPU, in place.

    X, V: (M, d) float64 numpy arrays (host) or CUDA tensors (device).
    Returns the number of field evaluations.
    """
    evals = _lib.ctypes.c_int64(0)
    M = X.shape[0]
    history.handle.call("nufi_trace", int(n), _lib.ptr(X), _lib.ptr(V), int(M), int(bool(half_kick)), int(mode),
                        _lib.ctypes.byref(evals))
    return int(evals.value)


def _trace(ctx: FlowContext, n: int, X, V, half_kick: bool, mode: int) -> None:
    if n == 0:
        return
    ctx.field_evals += trace_backward(ctx.history, n, X, V, half_kick, mode)


def psi_batch(ctx: FlowContext, n: int, x, v, mode: int = TRACE_FAST):
    """Backward flow from step n to t = 0 (flow.py:106-112); needs fields 0..n."""
    X, V = _batch(x, v, ctx.grid.d)
    _trace(ctx, n, X, V, True, mode)
    return X, V


def psi_tilde_batch(ctx: FlowContext, n: int, x, v, mode: int = TRACE_FAST):
    """Half-kick-free backward flow (flow.py:115-121); needs fields 0..n-1."""
    X, V = _batch(x, v, ctx.grid.d)
    _trace(ctx, n, X, V, False, mode)
    return X, V


def psi(ctx: FlowContext, n: int, p: PhasePoint) -> PhasePoint:
    X, V = psi_batch(ctx, n, p.x[None, :], p.v[None, :])
    return PhasePoint(x=X[0], v=V[0])


def psi_tilde(ctx: FlowContext, n: int, p: PhasePoint) -> PhasePoint:
    X, V = psi_tilde_batch(ctx, n, p.x[None, :], p.v[None, :])
    return PhasePoint(x=X[0], v=V[0])


def eval_f_batch(ctx: FlowContext, n: int, x, v) -> np.ndarray:
    """f(n tau, x, v) = f0(Psi(x, v)) (flow.py:134-137)."""
    X, V = psi_batch(ctx, n, x, v)
    return eval_f0(ctx.ic, X, V)


def eval_f(ctx: FlowContext, n: int, p: PhasePoint) -> float:
    return float(eval_f_batch(ctx, n, p.x[None, :], p.v[None, :])[0])
