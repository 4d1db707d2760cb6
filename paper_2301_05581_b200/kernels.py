"""The reference's trace plug-in point, served by the GPU (kernels.py:30-45, 390-412).

`trace_backward(coeffs, L, n, tau, X, V, half_kick) -> int` has the reference's
signature and contract: coeffs is a caller-owned (rows, Nx, ..., Nx) float64
coefficient stack (read only), X and V are (M, d) float64 arrays mutated in
place, the return value is the number of field evaluations, a short history
raises UsageError, n = 0 or M = 0 is a no-op returning 0.  A vpflow
maintainer can bind it as a third backend of vpflow.kernels.

Backends (the reference's set_backend / get_backend switch, kernels.py:35-45):
  "b200-parity"  (default) the sm_100a trace with the reference's operation order
                 and no FMA: bit-identical to the numba kernels _trace_1d/2d/3d;
  "b200"         the production arithmetic (FMA, cell-centred polynomial form),
                 within 1e-11 of the point scale.
Every call uploads the stack into a cached device history (<= a few MB for the
BASELINE grids); for repeated steps keep the history on the device instead
(PotentialHistory / FlowContext / compute_rho).
"""

from __future__ import annotations

import os

import numpy as np

from . import _lib
from .errors import UsageError
from .grids import GridSpec
from .spline import PotentialHistory

_BACKENDS = {"b200-parity": _lib.NUFI_TRACE_PARITY, "b200": _lib.NUFI_TRACE_FAST}
_backend = os.environ.get("VPFLOW_BACKEND", "b200-parity")
if _backend not in _BACKENDS:
    _backend = "b200-parity"
_cache: dict = {}


def set_backend(name: str) -> None:
    """kernels.py:35-41 (accepted names here: "b200-parity", "b200")."""
    global _backend
    if name not in _BACKENDS:
        raise UsageError(f"unknown backend {name!r}; choose from {sorted(_BACKENDS)}")
    _backend = name


def get_backend() -> str:
    return _backend


def _history(d: int, N: int, L: float, tau: float, rows: int) -> PotentialHistory:
    key = (d, N, float(L), float(tau))
    h = _cache.get(key)
    if h is None or h.capacity < rows:
        grid = GridSpec(d=d, L=float(L), Nx=N, Nv=2, vmax=1.0)  # velocity grid unused by the trace
        h = PotentialHistory(grid, float(tau), capacity=max(rows, 16))
        _cache[key] = h
    return h


def trace_backward(coeffs, L: float, n: int, tau: float, X: np.ndarray, V: np.ndarray, half_kick: bool) -> int:
    """Trace points backward through the stored fields (kernels.py:390-412), in place."""
    c = np.asarray(coeffs)
    if X.ndim != 2 or X.shape != V.shape:
        raise UsageError("X and V must both have shape (M, d)")
    d = X.shape[1]
    if c.ndim != d + 1:
        raise UsageError(f"coefficient stack must have shape (rows,) + (Nx,)*{d}")
    rows = c.shape[0]
    need = n + 1 if half_kick else n
    if n == 0 or X.shape[0] == 0:
        return 0
    if rows < need:
        raise UsageError(f"trace needs {need} stored fields for step {n}, got {rows}")  # kernels.py:398-402
    if X.dtype != np.float64 or V.dtype != np.float64 or not (X.flags.c_contiguous and V.flags.c_contiguous):
        raise UsageError("X and V must be C-contiguous float64 arrays (they are updated in place)")
    h = _history(d, c.shape[1], L, tau, rows)
    h.load_stack(np.ascontiguousarray(c[:need], dtype=np.float64))
    evals = _lib.ctypes.c_int64(0)
    h.handle.call("nufi_trace", int(n), X.ctypes.data, V.ctypes.data, int(X.shape[0]), int(bool(half_kick)),
                  int(_BACKENDS[_backend]), _lib.ctypes.byref(evals))
    return int(evals.value)


# ---------------------------------------------------------------------------
# The reference's spline helpers (kernels.py:62-123), on the device
# ---------------------------------------------------------------------------

def _helper_history():
    from .spline import _scratch_history

    return _scratch_history(GridSpec(d=1, L=1.0, Nx=4, Nv=2, vmax=1.0))


def _weights(t, which: str) -> np.ndarray:
    t = np.ascontiguousarray(np.asarray(t, dtype=np.float64))
    out = np.empty((4,) + t.shape)
    if t.size:
        w = out.ctypes.data if which == "w" else None
        dw = out.ctypes.data if which == "dw" else None
        _helper_history().handle.call("nufi_bspline_weights", t.ctypes.data, int(t.size), w, dw)
    return out


def bspline_weights(t) -> np.ndarray:
    """Cubic B-spline values for the 4-node stencil, shape (4,) + t.shape (kernels.py:62-70);
    bit-identical (numpy's operation order, no FMA; nufi_bspline_weights)."""
    return _weights(t, "w")


def bspline_dweights(t) -> np.ndarray:
    """Stencil weights of d/dt, shape (4,) + t.shape (kernels.py:73-81)."""
    return _weights(t, "dw")


def _spline_field(coeffs, L: float, X):
    from .spline import SplineField

    c = np.asarray(coeffs, dtype=np.float64)
    X = np.asarray(X)
    if X.ndim != 2 or c.ndim != X.shape[1]:
        raise UsageError("X must have shape (M, d) and coeffs shape (N,)*d")
    return SplineField(grid=GridSpec(d=c.ndim, L=float(L), Nx=c.shape[0], Nv=2, vmax=1.0), coeffs=c)


def eval_phi_many(coeffs, L: float, X) -> np.ndarray:
    """Spline values at X (M, d) for a (N,)*d coefficient grid (kernels.py:84-99), on the device."""
    return _spline_field(coeffs, L, X).eval_phi_many(X)


def eval_E_many(coeffs, L: float, X) -> np.ndarray:
    """Minus the spline gradient at X, shape (M, d) (kernels.py:102-123), on the device."""
    return _spline_field(coeffs, L, X).eval_E_many(X)
