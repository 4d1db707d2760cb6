"""Multi-rank exchange logic on CPU ranks (gloo, world size 2).

The GPU path (dist.DistributedSimulation) shards the velocity blocks, writes each
rank's block sums into a zero-padded (B*Nx^d + 2B) table, SUM-allreduces it and
runs the same fixed-order combine on every rank.  Here the per-block sums come
from the oracle (test-only) so the sharding / exchange / combine logic runs on
CPU: the combined rho must be bit-identical for world sizes 1 and 2, identical
on every rank, and equal to the oracle's compute_rho to roundoff.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_2301_05581_b200.dist import ShardedStep, block_range

B = 8


def block_table(c, run, n, blocks):
    """Zero-padded (B*nodes + 2B) table with the per-block v-sums of `blocks` (oracle)."""
    nodes, cells = c.n_nodes, c.n_cells
    per = cells // B
    tab = np.zeros(B * nodes + 2 * B)
    stack = run.stacked()[:n].reshape(n, -1) if n > 0 else None
    X0 = O.x_node_matrix(c)
    V0 = O.v_mid_matrix(c)
    for b in blocks:
        # d = 1: block b is the residue class {j : j mod B == b} (csrc/trace_common.cuh
        # d1_row); d >= 2: contiguous rows
        rows = np.arange(b, cells, B) if c.d == 1 else np.arange(b * per, (b + 1) * per)
        V = np.tile(V0[rows], (nodes, 1))
        X = np.repeat(X0, per, axis=0)
        if n > 0:
            O.trace_backward(stack, c.L, n, c.tau, X, V, False)
        F = O.eval_f0(c, X, V).reshape(nodes, per)
        S = np.zeros(nodes)
        for j in range(per):  # fixed order within the block
            S = S + F[:, j]
        tab[b * nodes:(b + 1) * nodes] = S
        tab[B * nodes + 2 * b] = F.min()
        tab[B * nodes + 2 * b + 1] = F.max()
    return tab


def sharded_rho(rank, world, name, steps):
    c = O.case(name)
    run = O.OracleRun(c)
    out = []
    lo, hi = block_range(B, rank, world)
    st = ShardedStep(B=B, nodes=c.n_nodes)
    for n in range(steps + 1):
        t = torch.from_numpy(block_table(c, run, n, range(lo, hi)))
        if world > 1:
            dist.all_reduce(t)
        rho, neut, fmn, fmx = st.combine(t.numpy(), run.rho_bar, c.hv ** c.d)
        out.append(rho)
        # advance the (oracle) history with the combined rho
        phi, _ = O.solve_poisson(c, rho)
        run.hist.append(O.fit_spline(c, phi))
    return np.array(out)


def _worker(rank, world, port, name, steps, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, sharded_rho(rank, world, name, steps)))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_block_range_covers_all_blocks():
    for world in (1, 2, 4, 8):
        seen = []
        for r in range(world):
            lo, hi = block_range(B, r, world)
            seen += list(range(lo, hi))
        assert seen == list(range(B))


@pytest.mark.parametrize("name,steps", [("kat_wl", 6), ("tiny2", 3)])
def test_two_rank_exchange_bit_identical(name, steps):
    ref = sharded_rho(0, 1, name, steps)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, steps, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert np.array_equal(res[0], res[1]), "ranks disagree"
    assert np.array_equal(res[0], ref), "world size changed the result"
    # and the combine equals the oracle's compute_rho to roundoff
    run = O.OracleRun(O.case(name)).run(steps)
    scale = np.abs(run["rho"]).max(axis=1, keepdims=True)
    assert (np.abs(ref - run["rho"]) / scale).max() < 1e-12


# ---------------------------------------------------------------------------
# the fused-exchange decision is collective (dist.DistributedSimulation._connect_fused)
# ---------------------------------------------------------------------------

class _FakeHandle:
    """Stands in for the library handle: records the calls, fails nufi_mg_setup on request."""

    def __init__(self, fail_setup, fail_connect=False):
        self.fail_setup = fail_setup
        self.fail_connect = fail_connect
        self.calls = []

        class _Lib:
            @staticmethod
            def nufi_mg_handle_size():
                return 64

        self.lib = _Lib()

    def call(self, name, *args):
        self.calls.append(name)
        if name == "nufi_mg_setup" and self.fail_setup:
            raise RuntimeError("setup failed on this rank")
        if name == "nufi_mg_connect" and self.fail_connect:
            raise RuntimeError("connect failed on this rank")


def _agree_worker(rank, world, port, fail_rank, fail_what, q):
    import types

    from paper_2301_05581_b200.dist import DistributedSimulation

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        obj = DistributedSimulation.__new__(DistributedSimulation)
        obj.torch, obj.dist, obj.group = torch, dist, None
        obj.rank, obj.world = rank, world
        h = _FakeHandle(fail_setup=(rank == fail_rank and fail_what == "setup"),
                        fail_connect=(rank == fail_rank and fail_what == "connect"))
        obj.history = types.SimpleNamespace(handle=h)
        DistributedSimulation._connect_fused.__wrapped__(obj, 0)  # the undecorated body (no CUDA stream)
        q.put((rank, obj.fused, h.calls))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("fail_rank,fail_what", [(-1, None), (1, "setup"), (0, "connect")])
def test_fused_exchange_decision_is_collective(fail_rank, fail_what):
    """a rank whose peer-memory setup or connect fails must not leave its peers in
    mismatched collectives -- every rank reaches the all_gather and the all_reduce, and all
    ranks take the same decision (fused, or all fall back and tear down)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_agree_worker, args=(r, 2, port, fail_rank, fail_what, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((r, (f, c)) for r, f, c in (q.get(timeout=120) for _ in procs))
    for p in procs:
        p.join(timeout=60)
    fused = {r: v[0] for r, v in res.items()}
    assert fused[0] == fused[1] == (fail_rank < 0)
    for r, (_, calls) in res.items():
        assert calls[0] == "nufi_mg_setup"
        if fail_rank >= 0 and not (fail_what == "setup" and r == fail_rank):
            # a rank whose own setup succeeded leaves multi-rank mode again
            assert calls[-1] == "nufi_mg_teardown"
