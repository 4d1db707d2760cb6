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
import struct
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import UsageError
from .grids import GridSpec
from .initial import InitialCondition, VelocityProfile


@dataclass(frozen=True)
class SplineField:
    """One stored potential: coefficient slab of shape grid.shape_x (spline.py:28-52).

    eval_phi_many / eval_E_many run on the GPU (nufi_eval_field, the numpy twin's
    operation order: bit-identical to the reference).  An entry of a device history
    evaluates in place; a free-standing field is uploaded into a cached 1-slab history."""

    grid: GridSpec
    coeffs: np.ndarray
    _source: tuple | None = field(default=None, compare=False, repr=False)  # (PotentialHistory, slot)

    @property
    def d(self) -> int:
        return self.grid.d

    def nodal_values(self) -> np.ndarray:
        """Potential values at the grid nodes (exact B-spline filter, spline.py:38-44)."""
        phi = np.asarray(self.coeffs, dtype=np.float64)
        for axis in range(self.grid.d):
            phi = (np.roll(phi, 1, axis=axis) + 4.0 * phi + np.roll(phi, -1, axis=axis)) / 6.0
        return phi

    def _eval(self, X, want_phi: bool):
        X = np.ascontiguousarray(np.atleast_2d(np.asarray(X, dtype=np.float64)))
        if X.shape[1] != self.grid.d:
            raise UsageError(f"position must have {self.grid.d} components")
        if self._source is not None:
            hist, slot = self._source
        else:
            hist, slot = _scratch_history(self.grid), 0
            hist.load_stack(np.asarray(self.coeffs, dtype=np.float64).reshape((1,) + self.grid.shape_x))
        M = X.shape[0]
        out = np.empty(M) if want_phi else np.empty((M, self.grid.d))
        hist.handle.call("nufi_eval_field", int(slot), X.ctypes.data, int(M),
                         out.ctypes.data if want_phi else None, None if want_phi else out.ctypes.data)
        return out

    def eval_phi_many(self, X) -> np.ndarray:
        """Spline values at X (M, d) (spline.py:46-48)."""
        return self._eval(X, True)

    def eval_E_many(self, X) -> np.ndarray:
        """Minus the spline gradient at X (M, d) (spline.py:50-52)."""
        return self._eval(X, False)


class UniformField:
    """A spatially constant electric field (spline.py:55-68).  No periodic potential
    generates it; it exists for flow tests against the constant-force closed form and is
    installed with FlowContext.install_field.  Only E evaluation is defined."""

    def __init__(self, E0):
        self.E0 = np.atleast_1d(np.asarray(E0, dtype=np.float64))
        self.d = self.E0.shape[0]

    def eval_E_many(self, X) -> np.ndarray:
        X = np.atleast_2d(np.asarray(X, dtype=np.float64))
        return np.broadcast_to(self.E0, (X.shape[0], self.d)).copy()


def fit_spline(phi_nodes, grid: GridSpec, dtype=np.float64) -> SplineField:
    """Interpolating periodic cubic spline through nodal values (spline.py:71-86), on the GPU."""
    if grid.Nx < 4:
        raise UsageError(f"spline fitting needs Nx >= 4, got {grid.Nx}")
    phi = np.ascontiguousarray(np.asarray(phi_nodes, dtype=np.float64))
    if phi.shape != grid.shape_x:
        raise UsageError(f"phi_nodes must have shape {grid.shape_x}, got {phi.shape}")
    out = np.empty(grid.n_nodes)
    _scratch_history(grid).handle.call("nufi_fit_spline", phi.ctypes.data, out.ctypes.data)
    coeffs = out.reshape(grid.shape_x).astype(dtype)
    coeffs.flags.writeable = False
    return SplineField(grid=grid, coeffs=coeffs)


_scratch: dict = {}


def _scratch_history(grid: GridSpec) -> "PotentialHistory":
    h = _scratch.get(grid)
    if h is None:
        h = PotentialHistory(grid, 1.0, capacity=1)
        _scratch[grid] = h
    return h


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
    spline.py:136-139).  dtype: float64, or float32 -- the reference's FP32
    history mode (spline.py:118-125): every stored coefficient is rounded to
    float32 on append and read back as double by the trace
    (NUFI_FLAG_F32_HISTORY).
    """

    def __init__(self, grid: GridSpec, tau: float, dtype=np.float64, capacity: int = 16, device: int | None = None,
                 v_blocks: int = 0, block_range: tuple | None = None, stream: int | None = None):
        if tau <= 0:
            raise UsageError(f"time step must be positive, got {tau}")
        self.dtype = np.dtype(dtype)
        if self.dtype not in (np.dtype(np.float32), np.dtype(np.float64)):
            raise UsageError(f"history dtype must be float32 or float64, got {self.dtype}")  # spline.py:123-125
        self.grid = grid
        self.tau = float(tau)
        self.device = _current_device() if device is None else int(device)
        lo, hi = block_range if block_range is not None else (0, 0)
        self._flags = _lib.NUFI_FLAG_F32_HISTORY if self.dtype == np.float32 else 0
        cfg = _lib.make_config(grid, _placeholder_ic(grid), self.tau, max(1, int(capacity)) - 1, rho_bar=1.0,
                               v_blocks=v_blocks, block_lo=lo, block_hi=hi, flags=self._flags)
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
        cfg = _lib.make_config(self.grid, ic, self.tau, self.capacity - 1, rho_bar=rho_bar, flags=self._flags)
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
        out = out.reshape(self.grid.shape_x).astype(self.dtype, copy=False)
        out.flags.writeable = False
        return SplineField(grid=self.grid, coeffs=out, _source=(self, m))

    def stacked(self) -> np.ndarray:
        """Host copy (len, Nx, ..., Nx) of all stored coefficients (spline.py:151-155)."""
        n = len(self)
        out = np.empty((n, self.grid.n_nodes))
        if n:
            self._handle.call("nufi_get_history", out.ctypes.data, 0, n)
        out = out.reshape((n,) + self.grid.shape_x).astype(self.dtype, copy=False)
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

    # -- checkpoint: the reference's VPHIST01 format (spline.py:105, 157-194) --

    def save(self, path) -> None:
        """Write the device history as VPHIST01: little-endian header <8sBBIQdd
        (magic, d, itemsize, Nx, count, L, tau) + raw coefficient rows."""
        with open(path, "wb") as fh:
            fh.write(checkpoint_bytes(self.grid, self.dtype, self.tau, self.stacked()))

    @classmethod
    def load(cls, path, grid: GridSpec | None = None, capacity: int | None = None, device: int | None = None
             ) -> "PotentialHistory":
        """Reload a VPHIST01 file into a device history (spline.py:171-194); grid, when
        given, supplies Nv and vmax and must match d, Nx, L."""
        grid, dtype, tau, rows = read_checkpoint(path, grid)
        count = rows.shape[0]
        hist = cls(grid, tau, dtype=dtype, capacity=max(count, capacity or 0, 1), device=device)
        if count:
            hist.load_stack(rows.astype(np.float64).reshape((count,) + grid.shape_x))
        return hist


_MAGIC = b"VPHIST01"
_HEADER = "<8sBBIQdd"


def checkpoint_bytes(grid: GridSpec, dtype, tau: float, rows: np.ndarray) -> bytes:
    """VPHIST01 image of `rows` (count, Nx, ..): header + little-endian rows (spline.py:157-169)."""
    dtype = np.dtype(dtype)
    rows = np.asarray(rows).reshape(-1, grid.n_nodes) if np.size(rows) else np.zeros((0, grid.n_nodes))
    header = struct.pack(_HEADER, _MAGIC, grid.d, dtype.itemsize, grid.Nx, rows.shape[0], grid.L, float(tau))
    return header + rows.astype(dtype.newbyteorder("<"), copy=False).tobytes()


def read_checkpoint(path, grid: GridSpec | None = None):
    """Parse a VPHIST01 file (spline.py:171-194) -> (grid, dtype, tau, rows (count, Nx^d))."""
    with open(path, "rb") as fh:
        head = fh.read(struct.calcsize(_HEADER))
        if len(head) != struct.calcsize(_HEADER):
            raise UsageError(f"{path} is not a potential-history file")
        magic, d, itemsize, Nx, count, L, tau = struct.unpack(_HEADER, head)
        if magic != _MAGIC:
            raise UsageError(f"{path} is not a potential-history file")
        dtype = np.dtype("<f4") if itemsize == 4 else np.dtype("<f8")
        payload = np.frombuffer(fh.read(), dtype=dtype)
    if grid is None:
        grid = GridSpec(d=d, L=L, Nx=Nx, Nv=2, vmax=1.0)  # velocity grid unknown
    elif (grid.d, grid.Nx) != (d, Nx) or abs(grid.L - L) > 1e-12 * L:
        raise UsageError("checkpoint grid does not match the supplied grid")
    if payload.size != count * Nx ** d:
        raise UsageError(f"truncated history file: {path}")
    return grid, np.dtype(f"=f{itemsize}"), float(tau), payload.reshape(count, Nx ** d)
