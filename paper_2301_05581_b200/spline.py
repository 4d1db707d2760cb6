"""Device-resident potential history (the entire NuFI state, Eq. 26).

PotentialHistory mirrors the reference's append-only history
(spline.py:108-155): one periodic cubic-B-spline coefficient slab per completed
step, contiguous (capacity, Nx^d) storage, growth by doubling, read-only
entries.  Here the buffer lives in GPU memory inside a libnufi_b200 handle,
next to the derived evaluation slabs the trace kernel streams (see
csrc/trace_common.cuh); `stacked()` / `entry()` copy rows back to the host.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import UsageError
from .grids import GridSpec
from .initial import InitialCondition, VelocityProfile


@dataclass(frozen=True)
class SplineField:
    """One stored potential: coefficient slab of shape grid.shape_x (spline.py:28-52)."""

    grid: GridSpec
    coeffs: np.ndarray

    @property
    def d(self) -> int:
        return self.grid.d


def _current_device() -> int:
    try:
        import torch

        if torch.cuda.is_available():
            return torch.cuda.current_device()
    except ImportError:  # pragma: no cover
        pass
    return 0


_PLACEHOLDER_IC = None


def _placeholder_ic(grid: GridSpec) -> InitialCondition:
    # f0 parameters are installed when a FlowContext binds the history
    return InitialCondition(benchmark="unbound", d=grid.d, L=grid.L, alpha=0.0, k=2.0 * np.pi / grid.L,
                            profiles=(VelocityProfile(),) * grid.d)


class PotentialHistory:
    """Append-only sequence of spline fields on the GPU (spline.py:108-155).

    capacity: slabs preallocated (grown by doubling on demand, like
    spline.py:136-139).  dtype: float64 only (the FP32 history mode of
    spline.py:118-125 is not implemented).
    """

    def __init__(self, grid: GridSpec, tau: float, dtype=np.float64, capacity: int = 16, device: int | None = None,
                 v_blocks: int = 0, block_range: tuple | None = None, stream: int | None = None):
        if tau <= 0:
            raise UsageError(f"time step must be positive, got {tau}")
        if np.dtype(dtype) != np.dtype(np.float64):
            raise UsageError("only float64 histories are supported on the GPU path")
        self.grid = grid
        self.tau = float(tau)
        self.dtype = np.dtype(np.float64)
        self.device = _current_device() if device is None else int(device)
        lo, hi = block_range if block_range is not None else (0, 0)
        cfg = _lib.make_config(grid, _placeholder_ic(grid), self.tau, max(1, int(capacity)) - 1, rho_bar=1.0,
                               v_blocks=v_blocks, block_lo=lo, block_hi=hi)
        self._handle = _lib.Handle(cfg, self.device, stream)
        self.ic = None

    # -- binding ------------------------------------------------------------

    @property
    def handle(self) -> _lib.Handle:
        return self._handle

    def bind(self, ic: InitialCondition, rho_bar: float | None = None) -> float:
        """Install f0 (and compute rho_bar on the device); returns rho_bar."""
        if ic.d != self.grid.d:
            raise UsageError(f"grid dimension {self.grid.d} does not match benchmark dimension {ic.d}")
        cfg = _lib.make_config(self.grid, ic, self.tau, self.capacity - 1, rho_bar=rho_bar)
        self._handle.call("nufi_set_initial_condition", ctypes.byref(cfg))
        self.ic = ic
        return self.rho_bar

    @property
    def rho_bar(self) -> float:
        out = ctypes.c_double()
        self._handle.call("nufi_rho_bar", ctypes.byref(out))
        return out.value

    # -- history API (spline.py:128-155) -----------------------------------

    @property
    def capacity(self) -> int:
        return int(self._handle.lib.nufi_capacity(self._handle.h))

    def reserve(self, slabs: int) -> None:
        if slabs > self.capacity:
            self._handle.call("nufi_reserve", int(slabs))

    def __len__(self) -> int:
        n = ctypes.c_int64()
        self._handle.call("nufi_history_len", ctypes.byref(n))
        return int(n.value)

    def append(self, field: SplineField) -> SplineField:
        """Copy a fitted field into the device history (spline.py:132-142)."""
        if field.grid != self.grid:
            raise UsageError("field grid does not match the history grid")
        n = len(self)
        if n >= self.capacity:
            self.reserve(2 * self.capacity)
        c = np.ascontiguousarray(field.coeffs, dtype=np.float64).reshape(-1)
        if c.size != self.grid.n_nodes:
            raise UsageError(f"coefficients must have shape {self.grid.shape_x}")
        self._handle.call("nufi_append_coeffs", c.ctypes.data)
        return self.entry(n)

    def entry(self, m: int) -> SplineField:
        n = len(self)
        if not 0 <= m < n:
            raise UsageError(f"history has {n} entries, requested {m}")
        out = np.empty(self.grid.n_nodes)
        self._handle.call("nufi_get_history", out.ctypes.data, int(m), 1)
        out = out.reshape(self.grid.shape_x)
        out.flags.writeable = False
        return SplineField(grid=self.grid, coeffs=out)

    def stacked(self) -> np.ndarray:
        """Host copy (len, Nx, ..., Nx) of all stored coefficients (spline.py:151-155)."""
        n = len(self)
        out = np.empty((n, self.grid.n_nodes))
        if n:
            self._handle.call("nufi_get_history", out.ctypes.data, 0, n)
        out = out.reshape((n,) + self.grid.shape_x)
        out.flags.writeable = False
        return out

    def load_stack(self, coeffs: np.ndarray) -> None:
        """Replace the history by a (count, Nx, ..) coefficient stack."""
        c = np.ascontiguousarray(coeffs, dtype=np.float64).reshape(-1, self.grid.n_nodes)
        if c.shape[0] > self.capacity:
            self.reserve(c.shape[0])
        self._handle.call("nufi_load_history", c.ctypes.data, int(c.shape[0]))

    def truncate(self, count: int) -> None:
        self._handle.call("nufi_truncate_history", int(count))
