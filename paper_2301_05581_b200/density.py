"""Charge density on the x-grid and phase-space quadrature sweeps.

Drop-ins for density.compute_rho / quadrature_sweep / quadrature_sweep_many.

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
from .flow import FlowContext, eval_f0, psi_batch
from .grids import GridSpec, v_mid_matrix, x_node_matrix

DEFAULT_CHUNK = 1 << 21  # density.py:27 (accepted for signature parity; the GPU path does not chunk)


class DensityGrid:
    """rho at the Nx^d nodes, row-major (poisson.py:19-32).

    A density returned by compute_rho is stream-ordered: its `values` are read from the
    device the first time they are accessed (pending.py), and advance() of it needs no
    host copy at all."""

    __slots__ = ("grid", "_values", "_entry")

    def __init__(self, grid: GridSpec, values=None, *, _entry=None):
        self.grid = grid
        self._entry = _entry
        self._values = None
        if _entry is None:
            vals = np.asarray(values, dtype=np.float64)
            if vals.shape != grid.shape_x:
                raise UsageError(f"values must have shape {grid.shape_x}, got {vals.shape}")
            if not np.isfinite(vals).all():
                raise UsageError("density values must be finite")
            self._values = vals

    @property
    def values(self) -> np.ndarray:
        if self._values is None:
            self._values = self._entry.materialize()["rho"].copy()  # the entry keeps the pristine copy
        return self._values

    def __repr__(self) -> str:
        return f"DensityGrid(grid={self.grid!r}, values={self.values!r})"


class RhoResult:
    """density.py:64-69: density, neutralization, f_min, f_max (the scalars of a
    stream-ordered result are read on first access)."""

    __slots__ = ("density", "_stats", "_entry")

    def __init__(self, density: DensityGrid, neutralization: float | None = None, f_min: float | None = None,
                 f_max: float | None = None, *, _entry=None):
        self.density = density
        self._entry = _entry
        self._stats = None if _entry is not None else (neutralization, f_min, f_max)

    def _s(self, i: int) -> float:
        if self._stats is None:
            st = self._entry.materialize()["stats"]
            self._stats = (float(st[0]), float(st[1]), float(st[2]))
        return self._stats[i]

    neutralization = property(lambda self: self._s(0))
    f_min = property(lambda self: self._s(1))
    f_max = property(lambda self: self._s(2))

    def __repr__(self) -> str:
        return (f"RhoResult(density={self.density!r}, neutralization={self.neutralization!r}, "
                f"f_min={self.f_min!r}, f_max={self.f_max!r})")


def compute_rho(ctx: FlowContext, n: int, chunk: int = DEFAULT_CHUNK) -> RhoResult:
    """Charge density at step n, neutralised to zero nodal mean (density.py:72-91).

    Enqueued on the device (nufi_rho_async: trace + f0 + v-reduction + neutralisation);
    the usage checks (short history) raise here, synchronously, like the reference."""
    from .pending import Entry, ring_of

    ring = ring_of(ctx.history)
    entry = Entry(ring, "step", int(n))
    evals = ctypes.c_int64(0)
    spec = ctypes.c_int(0)
    try:
        ctx.history.handle.call("nufi_rho_async", int(n), entry.slot, ctypes.byref(evals), ctypes.byref(spec))
    except Exception:
        entry.release()
        raise
    if not spec.value:
        entry.kind = "rho"
    ctx.field_evals += int(evals.value)
    ring.last_rho = entry
    return RhoResult(DensityGrid(ctx.grid, _entry=entry), _entry=entry)


# ---------------------------------------------------------------------------
# observable sweeps (density.py:94-120): full flow Psi, weights at the untraced points
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class ConservedMoments:
    """Midpoint-rule integrals over phase space at one step (nufi_moments).

    l1 = int f, f2 = int f^2, f_ln_f = int f ln f (0 ln 0 := 0),
    kinetic = int |v|^2 f / 2, momentum[a] = int v_a f; f_min / f_max over the
    quadrature points (the observed L-infinity bound)."""

    n: int
    l1: float
    f2: float
    f_ln_f: float
    kinetic: float
    momentum: np.ndarray
    f_min: float
    f_max: float


def conserved_moments(ctx: FlowContext, n: int) -> ConservedMoments:
    """quadrature_sweep_many(ctx, n, [f, f^2, f ln f, |v|^2 f / 2, v f]) fused on the GPU.

    One kernel traces every quadrature point with Psi (csrc/trace_rho.cu,
    MOM variant), evaluates f0 at the foot point and reduces the five weights
    in a fixed order; needs fields 0..n (flow.py:106-112)."""
    d = ctx.grid.d
    out = np.empty(6 + d)
    evals = ctypes.c_int64(0)
    ctx.history.handle.call("nufi_moments", int(n), out.ctypes.data, ctypes.byref(evals))
    ctx.field_evals += int(evals.value)
    return ConservedMoments(n=int(n), l1=float(out[0]), f2=float(out[1]), f_ln_f=float(out[2]),
                            kinetic=float(out[3]), momentum=out[4:4 + d].copy(), f_min=float(out[4 + d]),
                            f_max=float(out[5 + d]))


def _batches(ctx: FlowContext, n: int, chunk: int):
    """Node-aligned batches (density.py:45-61): untraced (X0, V0) and F = f0(Psi(X0, V0))."""
    grid = ctx.grid
    Xn = x_node_matrix(grid)
    Vm = v_mid_matrix(grid)
    n_cells = grid.n_cells
    nodes_per = max(1, chunk // n_cells)
    for start in range(0, grid.n_nodes, nodes_per):
        stop = min(start + nodes_per, grid.n_nodes)
        Xb = np.repeat(Xn[start:stop], n_cells, axis=0)
        Vb = np.tile(Vm, (stop - start, 1))
        Xt, Vt = psi_batch(ctx, n, Xb, Vb)  # GPU trace (nufi_trace)
        F = eval_f0(ctx.ic, Xt, Vt)  # GPU f0 (nufi_eval_f0)
        yield slice(start, stop), Xb, Vb, F


def quadrature_sweep(ctx: FlowContext, n: int, weight, chunk: int = DEFAULT_CHUNK):
    """Integrate weight(x, v, f) over phase space at step n (density.py:94-101)."""
    return quadrature_sweep_many(ctx, n, [weight], chunk=chunk)[0]


def quadrature_sweep_many(ctx: FlowContext, n: int, weights, chunk: int = DEFAULT_CHUNK):
    """Several weights sharing one traced batch (density.py:104-120).

    Arbitrary Python weights run on the host over batches traced on the GPU;
    for the conserved-quantity weights use conserved_moments (all on device)."""
    if n > 0 and len(ctx.history) < n + 1:
        raise UsageError(f"psi at step {n} needs fields 0..{n}; history holds {len(ctx.history)}")
    grid = ctx.grid
    measure = grid.hx ** grid.d * grid.hv ** grid.d
    totals = [None] * len(weights)
    for _, Xb, Vb, F in _batches(ctx, n, chunk):
        for iw, w in enumerate(weights):
            vals = np.asarray(w(Xb, Vb, F), dtype=np.float64)
            if vals.shape[0] != F.shape[0]:
                raise UsageError("weight must return one row per phase point")
            part = np.add.reduce(vals, axis=0)
            totals[iw] = part if totals[iw] is None else totals[iw] + part
    out = []
    for t in totals:
        t = t * measure
        out.append(float(t) if np.ndim(t) == 0 else t)
    return out
