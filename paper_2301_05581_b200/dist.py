"""Multi-GPU NuFI: quadrature points sharded by velocity blocks, one exchange per step.

One process per GPU (torch.distributed, NCCL over NVLink for the plumbing).
The Nv^d velocity rows are cut into B fixed blocks (default 8, independent of
the rank count); rank r traces blocks [r*B/G, (r+1)*B/G) for every x node
(v-row sharding; d >= 2 blocks are contiguous row ranges,
d = 1 blocks are residue classes j mod B so every rank -- and every CTA tile --
mixes trapped and passing particles, csrc/trace_common.cuh d1_row).  Each rank's
nufi_rho_partials writes its blocks' per-node v-sums into a
(B*Nx^d + 2B)-double buffer and zeros elsewhere, so one SUM allreduce gives
every rank the complete block table exactly (one non-zero contributor per
element).  Every rank then runs the same fixed-order combine + Poisson /
spline / append (nufi_step_finish) and therefore holds a bit-identical full
history.  Because the combine order over blocks does not depend on G, the
result is bit-identical for G = 1, 2, 4, 8.

The exchange is either the per-step NCCL allreduce of that table (default) or,
with NUFI_MG=1, fused into our own kernels over CUDA-IPC peer memory (the d = 1
persistent run kernel / the d >= 2 block reduce store the block sums straight into
every peer's table); the fused path is opt-in until it has run on more than one
physical GPU.  `exchange` names the path a run took.
"""

from __future__ import annotations

import ctypes
import functools
import os
from dataclasses import dataclass

import numpy as np

from .errors import NumericalConsistencyError, UsageError


def block_range(B: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous share of the B velocity blocks for `rank` of `world`."""
    if world < 1 or not 0 <= rank < world:
        raise UsageError("invalid rank / world size")
    lo = (B * rank) // world
    hi = (B * (rank + 1)) // world
    return lo, hi


def _on_stream(fn):
    """Run a DistributedSimulation method with its stream current, so torch collectives and
    tensor ops are ordered with the library's kernels."""

    @functools.wraps(fn)
    def wrapper(self, *args, **kwargs):
        cur = self.torch.cuda.current_stream(self.stream.device)
        if cur != self.stream:
            self.stream.wait_stream(cur)
        with self.torch.cuda.stream(self.stream):
            out = fn(self, *args, **kwargs)
        if cur != self.stream:
            cur.wait_stream(self.stream)
        return out

    return wrapper


@dataclass
class ShardedStep:
    """The exchange + combine logic of one sharded step, independent of the device."""

    B: int
    nodes: int

    @property
    def length(self) -> int:
        return self.B * self.nodes + 2 * self.B

    def combine(self, table: np.ndarray, rho_bar: float, hv_d: float):
        """Fixed-order combine of an allreduced block table (host restatement of
        field_update.cu's prologue) -> (rho neutralised, neutralization, f_min, f_max).
        Used by the CPU tests of the exchange; the GPU path does this on the device."""
        sums = table[: self.B * self.nodes].reshape(self.B, self.nodes)
        S = np.zeros(self.nodes)
        for b in range(self.B):
            S = S + sums[b]
        rho = rho_bar - hv_d * S
        mm = table[self.B * self.nodes:].reshape(self.B, 2)
        c = rho.mean()
        return rho - c, c, mm[:, 0].min(), mm[:, 1].max()


class DistributedSimulation:
    """Sharded NuFI run on one GPU per rank (requires an initialised NCCL process group)."""

    def __init__(self, grid, ic, tau, n_steps, v_blocks: int = 8, group=None):
        import torch
        import torch.distributed as dist

        from .driver import Simulation

        self.torch = torch
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        V = grid.n_cells
        B = v_blocks
        while B > 1 and V % B:
            B -= 1
        if B < self.world:
            raise UsageError(f"{B} velocity blocks cannot be shared by {self.world} ranks")
        self.B = B
        lo, hi = block_range(B, self.rank, self.world)
        device = torch.cuda.current_device()
        # The library and the collectives must share ONE stream.  The legacy default stream
        # (cuda_stream == 0) cannot be handed to the library (NULL means "private stream"),
        # so a run started on it gets a dedicated stream, made current around every step.
        cur = torch.cuda.current_stream(device)
        self.stream = cur if cur.cuda_stream != 0 else torch.cuda.Stream(device)
        from .flow import FlowContext
        from .spline import PotentialHistory

        self.grid = grid
        self.n_steps = int(n_steps)
        self.history = PotentialHistory(grid, tau, capacity=n_steps + 1, device=device, v_blocks=B,
                                        block_range=(lo, hi), stream=self.stream.cuda_stream)
        self.ctx = FlowContext(history=self.history, ic=ic, tau=tau, grid=grid)
        n = int(self.history.handle.lib.nufi_partials_len(self.history.handle.h))
        with torch.cuda.stream(self.stream):
            self.partials = torch.zeros(n, dtype=torch.float64, device=f"cuda:{device}")
        self.stream.wait_stream(cur)  # the caller's pending work (e.g. output allocation) first
        self.block_lo, self.block_hi = lo, hi
        self.fused = False
        # The fused peer-memory exchange is opt-in (NUFI_MG=1) until it has run on more
        # than one physical GPU; the default is the per-step NCCL allreduce loop.
        if self.world > 1 and B % self.world == 0 and os.environ.get("NUFI_MG", "0") == "1":
            self._connect_fused(device)

    @property
    def exchange(self) -> str:
        """The exchange the next run takes: "fused-ipc" or "nccl-allreduce" (single rank: "none")."""
        if self.world == 1:
            return "none"
        return "fused-ipc" if self.fused else "nccl-allreduce"

    @_on_stream
    def _connect_fused(self, device: int) -> None:
        """The exchange fused into our own kernels (nufi_mg_*): d = 1 the persistent run
        kernel, d = 2, 3 the block reduce (nufi_mg_step_async).  Every rank exports its
        exchange buffer (CUDA IPC), the handles are all-gathered over the process group,
        every rank opens its peers'.  The ranks decide TOGETHER: every rank reaches the
        all_gather (with an ok byte in front of its handle, 0 if its setup failed) and the
        final all_reduce(MIN) of the connect outcome, so either all ranks run fused or all
        fall back to the per-step NCCL loop (with a warning) -- never a split decision
        that would leave the ranks in mismatched collectives."""
        import warnings

        t = self.torch
        h = self.history.handle
        size = int(h.lib.nufi_mg_handle_size())
        buf = ctypes.create_string_buffer(size)
        ok = 1
        why = None
        try:
            h.call("nufi_mg_setup", self.world, self.rank, 0, buf)
        except Exception as exc:  # pragma: no cover - depends on the machine's peer access
            ok, why = 0, exc
        set_up = ok == 1  # this rank holds multi-rank resources to release on a fallback
        # NCCL gathers device tensors; gloo (CPU-side test groups) gathers host tensors
        where = f"cuda:{device}" if self.dist.get_backend(self.group) == "nccl" else "cpu"
        mine = t.tensor([ok] + list(buf.raw), dtype=t.uint8, device=where)
        allh = [t.empty_like(mine) for _ in range(self.world)]
        self.dist.all_gather(allh, mine, group=self.group)
        rows = [bytes(x.cpu().tolist()) for x in allh]
        if all(r[0] == 1 for r in rows):
            try:
                h.call("nufi_mg_connect", b"".join(r[1:] for r in rows))
            except Exception as exc:  # pragma: no cover
                ok, why = 0, exc
        else:
            ok = 0
            why = why or "a peer's peer-memory setup failed"
        flag = t.tensor([ok], dtype=t.int32, device=where)
        self.dist.all_reduce(flag, op=self.dist.ReduceOp.MIN, group=self.group)
        self.fused = int(flag.item()) == 1
        if not self.fused:
            warnings.warn(f"fused multi-rank kernel unavailable ({why or 'on a peer'}); "
                          "using the per-step NCCL loop")
            if set_up:
                h.call("nufi_mg_teardown")

    def _run_exchange_steps(self, first: int, outputs: dict, ev) -> None:
        """d = 2, 3 fused loop: nufi_mg_step_async per step (trace own blocks -> block sums
        stored into every rank's table over peer memory -> tail waiting on the arrival
        counters), device outputs, one status check at the end."""
        t = self.torch
        g = self.grid
        h = self.history.handle
        dev = f"cuda:{self.partials.device.index}"
        steps = self.n_steps + 1 - first
        host = {k: v for k, v in outputs.items() if v is not None and not hasattr(v, "data_ptr")}
        dout = {k: (v if hasattr(v, "data_ptr") else None) for k, v in outputs.items()}
        shapes = dict(rho=(steps, g.n_nodes), E=(steps, g.n_nodes, g.d), W=(steps,), stats=(steps, 3))
        for k in host:
            dout[k] = t.empty(shapes[k], dtype=t.float64, device=dev)

        def row(k, n):
            a = dout.get(k)
            if a is None:
                return None
            width = int(np.prod(shapes[k][1:])) if len(shapes[k]) > 1 else 1
            return a.data_ptr() + (n - first) * width * 8

        for n in range(first, self.n_steps + 1):
            h.call("nufi_mg_step_async", n, row("rho", n), row("E", n), row("W", n), row("stats", n))
        h.call("nufi_check_status")
        for k, a in host.items():
            a[...] = dout[k].cpu().numpy().reshape(a.shape)
        # this rank traced its share of the blocks: P_rank * sum_n n
        per_step = g.n_nodes * g.n_cells * (self.block_hi - self.block_lo) // self.B
        ev.value += per_step * sum(range(first, self.n_steps + 1))

    @_on_stream
    def step(self, outputs: dict | None = None, row: int = 0, sync: bool = True):
        """One step: trace own blocks -> allreduce -> redundant field update."""
        h = self.history.handle
        n = len(self.history)
        ev = ctypes.c_int64(0)
        h.call("nufi_rho_partials", n, self.partials.data_ptr(), ctypes.byref(ev))
        self.dist.all_reduce(self.partials, group=self.group)  # NCCL on the same stream order
        o = outputs or {}

        def rowptr(key, width):
            a = o.get(key)
            if a is None:
                return None
            return a.data_ptr() + row * width * 8 if hasattr(a, "data_ptr") else a.ctypes.data + row * width * 8

        g = self.grid
        args = (n, self.partials.data_ptr(), rowptr("rho", g.n_nodes), rowptr("E", g.n_nodes * g.d),
                rowptr("W", 1), rowptr("stats", 3))
        if sync:
            h.call("nufi_step_finish", *args)
        else:
            h.call("nufi_step_finish_async", *args)  # stream-ordered, device outputs
        self.ctx.field_evals += int(ev.value)
        return n

    @_on_stream
    def run(self, outputs: dict | None = None):
        """The whole loop.  With device (CUDA tensor) outputs every step is enqueued
        without a host synchronisation (trace -> NCCL allreduce -> field update, all on
        one stream) and the status is checked once at the end.  outputs=None: the same,
        into internal device buffers, returning host numpy arrays (the public call,
        like Simulation.run)."""
        first = len(self.history)
        steps = self.n_steps + 1 - first
        if self.fused:
            # one persistent kernel per rank, exchanging over peer memory every step
            from . import _lib

            self.dist.barrier(group=self.group)  # start together (the kernels wait on each other)
            g = self.grid
            if outputs is None:
                outputs = dict(rho=np.empty((steps, g.n_nodes)), E=np.empty((steps, g.n_nodes, g.d)),
                               W=np.empty(steps), stats=np.empty((steps, 3)))
            ev = ctypes.c_int64(0)
            err = None
            try:
                if g.d == 1:
                    self.history.handle.call("nufi_run", self.n_steps, _lib.ptr(outputs.get("rho")),
                                             _lib.ptr(outputs.get("E")), _lib.ptr(outputs.get("W")),
                                             _lib.ptr(outputs.get("stats")), ctypes.byref(ev))
                else:
                    self._run_exchange_steps(first, outputs, ev)
            except NumericalConsistencyError:
                raise  # the physics, not the transport: same on every rank
            except Exception as exc:  # a peer timed out (watchdog) or the launch failed
                err = exc
            # every rank agrees on the outcome before anyone trusts its history
            flag = self.torch.tensor([0 if err is None else 1], dtype=self.torch.int32,
                                     device=self.partials.device)
            self.dist.all_reduce(flag, group=self.group)
            if int(flag.item()) == 0:
                if g.d == 1:  # nufi_run counts the whole grid; this rank traced its share of the blocks
                    self.ctx.field_evals += int(ev.value) * (self.block_hi - self.block_lo) // self.B
                else:
                    self.ctx.field_evals += int(ev.value)
                return outputs
            import warnings

            warnings.warn(f"fused multi-rank run failed ({err or 'on a peer'}); rerunning with the per-step NCCL loop")
            self.fused = False
            self.history.handle.call("nufi_mg_teardown")
            self.history.truncate(first)
        host = outputs is None
        if host:
            g = self.grid
            t = self.torch
            dev = f"cuda:{self.partials.device.index}"
            outputs = dict(rho=t.empty((steps, g.n_nodes), dtype=t.float64, device=dev),
                           E=t.empty((steps, g.n_nodes, g.d), dtype=t.float64, device=dev),
                           W=t.empty(steps, dtype=t.float64, device=dev),
                           stats=t.empty((steps, 3), dtype=t.float64, device=dev))
        on_device = all(v is None or hasattr(v, "data_ptr") for v in outputs.values())
        for n in range(first, self.n_steps + 1):
            self.step(outputs, n - first, sync=not on_device)
        if on_device:
            self.history.handle.call("nufi_check_status")
        if host:
            return {k: v.cpu().numpy() for k, v in outputs.items()}
        return outputs
