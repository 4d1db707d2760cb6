"""The NuFI time loop (run driver) and the per-step field update.

The reference package ships no driver; SPEC.md:465-468 and SURVEY.md §3.1 give
the canonical loop

    for n in 0..N:  r = compute_rho(ctx, n); phi, spec = solve_poisson(r.density)
                    history.append(fit_spline(phi)); W = electric_energy(spec)

Simulation runs exactly that loop with every step on the GPU (nufi_step /
nufi_run): the trace + f0 + v-reduction kernel, then the single-CTA
Poisson / spline / append / energy / E kernel, the history never leaving the
device.  Per-step outputs are rho (Nx^d), E at the nodes (Nx^d x d), the
electric energy W and (neutralization, f_min, f_max).

advance(ctx, density) is the drop-in for the loop's tail
(solve_poisson + fit_spline + append + electric_energy + E at the nodes).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from .density import DensityGrid
from .errors import UsageError
from .flow import FlowContext
from .grids import GridSpec
from .initial import InitialCondition
from .spline import PotentialHistory


@dataclass(frozen=True)
class StepOutput:
    n: int
    rho: np.ndarray          # shape_x
    E: np.ndarray            # (Nx^d, d)
    W: float
    neutralization: float
    f_min: float
    f_max: float


@dataclass(frozen=True)
class RunResult:
    first_step: int
    rho: np.ndarray          # (steps, Nx^d)
    E: np.ndarray            # (steps, Nx^d, d)
    W: np.ndarray            # (steps,)
    stats: np.ndarray        # (steps, 3): neutralization, f_min, f_max
    field_evals: int

    @property
    def times(self) -> np.ndarray:
        return np.arange(self.first_step, self.first_step + len(self.W))


class FieldUpdate:
    """W, E at the nodes and the appended coefficients of one tail (read on first access)."""

    __slots__ = ("_vals", "_entry")

    def __init__(self, W: float | None = None, E: np.ndarray | None = None, coeffs: np.ndarray | None = None,
                 *, _entry=None):
        self._entry = _entry
        self._vals = None if _entry is not None else {"W": W, "E": E, "coeffs": coeffs}

    def _get(self, key):
        if self._vals is None:
            self._vals = self._entry.materialize()
        return self._vals[key]

    W = property(lambda self: self._get("W"))
    E = property(lambda self: self._get("E"))
    coeffs = property(lambda self: self._get("coeffs"))


def advance(ctx: FlowContext, density: DensityGrid) -> FieldUpdate:
    """solve_poisson (poisson.py:90-112) + fit_spline (spline.py:71-86) + append
    (spline.py:132-142) + electric_energy (poisson.py:115-120) + E at the nodes,
    enqueued on the GPU (nufi_field_update_async).  A host density is checked for
    neutrality here with the reference's own test (poisson.py:97-104) and raises
    NumericalConsistencyError before anything is appended; a density that compute_rho
    left on the device is passed without a copy (its tail re-checks on the device, and a
    failure surfaces when a later result is read)."""
    from .errors import NumericalConsistencyError
    from .pending import Entry, ring_of

    g = ctx.grid
    if density.grid is not g and density.grid != g:
        raise UsageError("density grid does not match the context grid")
    h = ctx.history
    ring = ring_of(h)
    e = density._entry
    if e is not None and e is ring.last_rho:
        ring.last_rho = None
        # unmodified values of the step compute_rho just enqueued (never read, or read and
        # still equal to the device's output)
        pristine = density._values is None or np.array_equal(density._values, e.materialize()["rho"])
        if e.kind == "step" and pristine:
            try:
                h.handle.call("nufi_commit_async", e.n)  # its tail already ran: commit slot n
                return FieldUpdate(_entry=e)
            except UsageError:  # the speculation was discarded by another call
                pass
        elif e.kind == "rho" and pristine:
            entry = Entry(ring, "field")
            try:
                h.handle.call("nufi_field_update_async", None, entry.slot)
                return FieldUpdate(_entry=entry)
            except UsageError:  # another call replaced the device density: pass the host values
                entry.release()
    if len(h) >= h.capacity:
        h.reserve(2 * h.capacity)  # PotentialHistory grows by doubling (spline.py:136-139)
    vals = density.values
    mean = float(vals.mean())
    tol = 1e-8 * float(np.max(np.abs(vals)))
    if abs(mean) > tol:
        raise NumericalConsistencyError(
            f"density is not neutral: nodal mean {mean:.3e} exceeds tolerance {tol:.3e}; "
            "subtract the mean before solving")
    rho = np.ascontiguousarray(vals, dtype=np.float64).reshape(-1)
    entry = Entry(ring, "field")
    try:
        h.handle.call("nufi_field_update_async", rho.ctypes.data, entry.slot)
    except Exception:
        entry.release()
        raise
    return FieldUpdate(_entry=entry)


class Simulation:
    """NuFI run state: device history + initial condition + tau, stepping to n_steps."""

    def __init__(self, grid: GridSpec, ic: InitialCondition, tau: float, n_steps: int, device: int | None = None,
                 v_blocks: int = 0, stream: int | None = None, dtype=np.float64):
        if n_steps < 0:
            raise UsageError("n_steps must be >= 0")
        self.grid = grid
        self.n_steps = int(n_steps)
        self.history = PotentialHistory(grid, tau, dtype=dtype, capacity=n_steps + 1, device=device,
                                        v_blocks=v_blocks, stream=stream)
        self.ctx = FlowContext(history=self.history, ic=ic, tau=tau, grid=grid)

    @classmethod
    def resume(cls, path, grid: GridSpec, ic: InitialCondition, n_steps: int, device: int | None = None,
               v_blocks: int = 0, stream: int | None = None) -> "Simulation":
        """Continue a run from a VPHIST01 checkpoint (PotentialHistory.save, spline.py:157-194):
        the history is the entire NuFI state (Eq. 26), so step len(history) is next."""
        from .spline import read_checkpoint

        grid_ck, dtype, tau, rows = read_checkpoint(path, grid)
        if rows.shape[0] > n_steps + 1:
            raise UsageError(f"checkpoint holds {rows.shape[0]} fields, more than n_steps + 1 = {n_steps + 1}")
        sim = cls(grid, ic, tau, n_steps, device=device, v_blocks=v_blocks, stream=stream, dtype=dtype)
        if rows.shape[0]:
            sim.history.load_stack(rows.astype(np.float64).reshape((rows.shape[0],) + grid.shape_x))
        return sim

    @property
    def n(self) -> int:
        """Next step index (= number of stored fields)."""
        return len(self.history)

    def step(self) -> StepOutput:
        n = self.n
        if n > self.n_steps:
            raise UsageError(f"simulation already reached n_steps = {self.n_steps}")
        g = self.grid
        rho = np.empty(g.n_nodes)
        E = np.empty((g.n_nodes, g.d))
        W = np.empty(1)
        st = np.empty(3)
        ev = ctypes.c_int64(0)
        self.history.handle.call("nufi_step", n, rho.ctypes.data, E.ctypes.data, W.ctypes.data, st.ctypes.data,
                                 ctypes.byref(ev))
        self.ctx.field_evals += int(ev.value)
        return StepOutput(n=n, rho=rho.reshape(g.shape_x), E=E, W=float(W[0]), neutralization=float(st[0]),
                          f_min=float(st[1]), f_max=float(st[2]))

    def run(self, n_last: int | None = None, outputs=None) -> RunResult:
        """Steps self.n .. n_last (default n_steps) on the device.

        outputs: optional dict of preallocated buffers (numpy host arrays or CUDA
        tensors) 'rho', 'E', 'W', 'stats' with leading dimension = steps."""
        n_last = self.n_steps if n_last is None else int(n_last)
        first = self.n
        steps = max(0, n_last - first + 1)
        g = self.grid
        if outputs is None:
            outputs = dict(rho=np.empty((steps, g.n_nodes)), E=np.empty((steps, g.n_nodes, g.d)),
                           W=np.empty(steps), stats=np.empty((steps, 3)))
        ev = ctypes.c_int64(0)
        from . import _lib

        self.history.handle.call("nufi_run", n_last, _lib.ptr(outputs.get("rho")), _lib.ptr(outputs.get("E")),
                                 _lib.ptr(outputs.get("W")), _lib.ptr(outputs.get("stats")), ctypes.byref(ev))
        self.ctx.field_evals += int(ev.value)
        return RunResult(first_step=first, rho=outputs.get("rho"), E=outputs.get("E"), W=outputs.get("W"),
                         stats=outputs.get("stats"), field_evals=int(ev.value))


def run_simulation(grid: GridSpec, ic: InitialCondition, tau: float, n_steps: int, device: int | None = None
                   ) -> RunResult:
    """The whole loop n = 0..n_steps on the GPU."""
    return Simulation(grid, ic, tau, n_steps, device=device).run()


def point_steps(grid: GridSpec, n_first: int, n_last: int) -> int:
    """Backtraced point-steps of steps n_first..n_last: P * sum n."""
    s = (n_last * (n_last + 1) - (n_first - 1) * n_first) // 2 if n_last >= n_first else 0
    return grid.n_points * s
