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


@dataclass(frozen=True)
class FieldUpdate:
    W: float
    E: np.ndarray
    coeffs: np.ndarray


def advance(ctx: FlowContext, density: DensityGrid) -> FieldUpdate:
    """solve_poisson (poisson.py:90-112) + fit_spline (spline.py:71-86) + append
    (spline.py:132-142) + electric_energy (poisson.py:115-120) + E at the nodes,
    on the GPU.  Raises NumericalConsistencyError for a non-neutral density."""
    g = ctx.grid
    if density.grid != g:
        raise UsageError("density grid does not match the context grid")
    h = ctx.history
    if len(h) >= h.capacity:
        h.reserve(2 * h.capacity)
    rho = np.ascontiguousarray(density.values, dtype=np.float64).reshape(-1)
    W = np.empty(1)
    E = np.empty((g.n_nodes, g.d))
    C = np.empty(g.n_nodes)
    h.handle.call("nufi_field_update", rho.ctypes.data, W.ctypes.data, E.ctypes.data, C.ctypes.data)
    return FieldUpdate(W=float(W[0]), E=E, coeffs=C.reshape(g.shape_x))


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
