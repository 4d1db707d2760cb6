"""The multi-rank device path on one GPU, ranks emulated in one process.

Each emulated rank owns a handle tracing its velocity blocks (nufi_rho_partials);
the allreduce is emulated by summing the ranks' zero-padded block tables (exact:
one non-zero contributor per element, x + 0 = x); every rank then runs the
redundant combine + field update (nufi_step_finish).  The ranks' launches are
independent and sequential (no kernel waits on another rank).  Required:
per-step rho / W and the full coefficient history bit-identical across ranks and
to the single-GPU run (the block combine order does not depend on the rank count).
"""

import ctypes

import numpy as np
import pytest
import torch

import paper_2301_05581_b200 as nufi
from paper_2301_05581_b200.configs import workload
from paper_2301_05581_b200.dist import block_range

pytestmark = pytest.mark.gpu


def sharded_run(name, N, world, B=8, asynchronous=False):
    w = workload(name)
    g = w.grid
    ranks = []
    for r in range(world):
        h = nufi.PotentialHistory(g, w.tau, capacity=N + 1, v_blocks=B, block_range=block_range(B, r, world))
        nufi.FlowContext(history=h, ic=w.ic, tau=w.tau, grid=g)  # binds f0
        n_part = int(h.handle.lib.nufi_partials_len(h.handle.h))
        ranks.append((h, torch.zeros(n_part, dtype=torch.float64, device="cuda")))
    rho = np.empty((world, N + 1, g.n_nodes))
    W = np.empty((world, N + 1))
    evals = 0
    for n in range(N + 1):
        for h, part in ranks:
            ev = ctypes.c_int64(0)
            h.handle.call("nufi_rho_partials", n, part.data_ptr(), ctypes.byref(ev))
            evals += ev.value
        torch.cuda.synchronize()
        table = sum(p for _, p in ranks)  # the allreduce
        torch.cuda.synchronize()
        for r, (h, _) in enumerate(ranks):
            if asynchronous:  # device outputs, stream-ordered (DistributedSimulation.run)
                d_rho = torch.empty(g.n_nodes, dtype=torch.float64, device="cuda")
                d_W = torch.empty(1, dtype=torch.float64, device="cuda")
                h.handle.call("nufi_step_finish_async", n, table.data_ptr(), d_rho.data_ptr(), None,
                              d_W.data_ptr(), None)
                h.handle.call("nufi_sync")
                rho[r, n] = d_rho.cpu().numpy()
                W[r, n] = float(d_W[0])
            else:
                out_rho = np.empty(g.n_nodes)
                out_W = np.empty(1)
                h.handle.call("nufi_step_finish", n, table.data_ptr(), out_rho.ctypes.data, None,
                              out_W.ctypes.data, None)
                rho[r, n] = out_rho
                W[r, n] = out_W[0]
    if asynchronous:
        for h, _ in ranks:
            h.handle.call("nufi_check_status")
    hists = [h.stacked().reshape(N + 1, -1) for h, _ in ranks]
    return rho, W, hists, evals


@pytest.mark.parametrize("name,N", [("kat_wl", 40), ("tiny2", 12), ("tiny3", 8), ("rag1", 20), ("ts1", 80),
                                    ("wl1", 40), ("sl1", 16)])
@pytest.mark.parametrize("world", [2, 4, 8])
def test_sharded_bit_identical_to_single_gpu(name, N, world):
    """Also on the BASELINE d = 1 grids, whose tile height the single-GPU run picks from the
    grid (ts1 8 rows, wl1 4, sl1 16): a rank must tile the same way although it traces
    only 1/world of the rows, else its block sums group rows differently."""
    w = workload(name)
    sim = nufi.Simulation(w.grid, w.ic, w.tau, N, v_blocks=8)
    ref = sim.run()
    rho, W, hists, evals = sharded_run(name, N, world)
    ref_hist = sim.history.stacked().reshape(N + 1, -1)
    for r in range(world):
        assert np.array_equal(rho[r], ref.rho), (r, np.abs(rho[r] - ref.rho).max())
        assert np.array_equal(W[r], ref.W)
        assert np.array_equal(hists[r], ref_hist)
    assert evals == ref.field_evals


@pytest.mark.parametrize("name,N", [("kat_wl", 30), ("tiny2", 10)])
def test_sharded_async_finish_bit_identical(name, N):
    w = workload(name)
    ref = nufi.Simulation(w.grid, w.ic, w.tau, N, v_blocks=8).run()
    rho, W, hists, _ = sharded_run(name, N, 2, asynchronous=True)
    for r in range(2):
        assert np.array_equal(rho[r], ref.rho) and np.array_equal(W[r], ref.W)



@pytest.mark.parametrize("name,N", [("kat_wl", 30), ("tiny3", 6)])
def test_distributed_simulation_nccl_single_rank(name, N):
    """The real torch.distributed / NCCL plumbing of dist.DistributedSimulation with one
    rank (no other rank to wait for): async device-output loop, bit-identical to one GPU."""
    import socket

    import torch.distributed as dist

    from paper_2301_05581_b200.dist import DistributedSimulation

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        w = workload(name)
        g = w.grid
        ds = DistributedSimulation(g, w.ic, w.tau, N)
        out = dict(rho=torch.empty((N + 1, g.n_nodes), dtype=torch.float64, device="cuda"),
                   W=torch.empty(N + 1, dtype=torch.float64, device="cuda"))
        ds.run(outputs=out)
        torch.cuda.synchronize()
        ref = nufi.Simulation(g, w.ic, w.tau, N, v_blocks=ds.B).run()
        assert np.array_equal(out["rho"].cpu().numpy(), ref.rho)
        assert np.array_equal(out["W"].cpu().numpy(), ref.W)
        assert len(ds.history) == N + 1
        host = DistributedSimulation(g, w.ic, w.tau, N).run()  # public call: host arrays
        assert np.array_equal(host["rho"], ref.rho) and np.array_equal(host["W"], ref.W)
    finally:
        dist.destroy_process_group()


def _emulated_mg_run(name, N, world, repeat=1):
    w = workload(name)
    sim = nufi.Simulation(w.grid, w.ic, w.tau, N, v_blocks=8)
    h = sim.history.handle
    h.call("nufi_mg_setup", world, 0, 1, None)  # all ranks as CTA groups of one launch
    res = None
    for _ in range(repeat):  # repeated runs: the arrival flags keep counting across runs
        sim.history.truncate(0)
        res = sim.run()
    return sim, res


@pytest.mark.parametrize("name,N", [("kat_wl", 60), ("ts1", 200), ("rag1", 20), ("sl1", 24)])
@pytest.mark.parametrize("world", [2, 4, 8])
def test_fused_multirank_kernel_emulated(name, N, world):
    """The fused multi-rank persistent kernel (exchange over peer memory + arrival flags,
    run_1d.cu) with `world` ranks emulated as CTA groups of one cooperative launch:
    bit-identical to the single-GPU run (same tiles, same block-combine order)."""
    w = workload(name)
    if (w.grid.n_cells % 8) or (8 % world):
        pytest.skip("needs 8 velocity blocks divisible by the rank count")
    ref_sim = nufi.Simulation(w.grid, w.ic, w.tau, N, v_blocks=8)
    ref = ref_sim.run()
    sim, res = _emulated_mg_run(name, N, world, repeat=2)
    assert np.array_equal(res.rho, ref.rho), np.abs(res.rho - ref.rho).max()
    assert np.array_equal(res.W, ref.W)
    assert np.array_equal(sim.history.stacked(), ref_sim.history.stacked())


def test_fused_multirank_setup_errors():
    w = workload("kat_wl")
    h = nufi.PotentialHistory(w.grid, w.tau, capacity=4, v_blocks=8, block_range=(0, 4))
    with pytest.raises(nufi.UsageError):
        h.handle.call("nufi_mg_setup", 2, 1, 0, None)  # rank 1's share is blocks 4..8
    with pytest.raises(nufi.UsageError):
        h.handle.call("nufi_mg_setup", 2, 0, 1, None)  # emulation needs all blocks
    w2 = workload("tiny2")
    h2 = nufi.PotentialHistory(w2.grid, w2.tau, capacity=4, v_blocks=8)
    with pytest.raises(nufi.UsageError):
        h2.handle.call("nufi_mg_step_async", 0, None, None, None, None)  # no nufi_mg_setup yet
    wb = workload("big2")
    hb = nufi.PotentialHistory(wb.grid, wb.tau, capacity=4, v_blocks=6)
    with pytest.raises(nufi.UsageError):
        hb.handle.call("nufi_mg_setup", 2, 0, 1, None)  # grids beyond one CTA's tail


@pytest.mark.parametrize("name,N", [("tiny2", 12), ("tiny3", 8), ("rag2", 10), ("wl3r", 6)])
@pytest.mark.parametrize("world", [2, 4, 8])
def test_fused_exchange_d23_emulated(name, N, world):
    """d >= 2 steps with the exchange fused into the block reduce (nufi_mg_step_async:
    block sums stored into every rank's table over peer memory + arrival counters, the
    step tail waiting on them; no NCCL), `world` ranks emulated on this device: rho, W,
    E, stats and the history bit-identical to the single-GPU run, over repeated runs."""
    import torch

    w = workload(name)
    g = w.grid
    if (g.n_cells % 8) or (8 % world):
        pytest.skip("needs 8 velocity blocks divisible by the rank count")
    ref_sim = nufi.Simulation(g, w.ic, w.tau, N, v_blocks=8)
    ref = ref_sim.run()
    sim = nufi.Simulation(g, w.ic, w.tau, N, v_blocks=8)
    h = sim.history.handle
    h.call("nufi_mg_setup", world, 0, 1, None)
    for _ in range(2):  # the arrival counters keep counting across runs
        sim.history.truncate(0)
        out = dict(rho=torch.empty((N + 1, g.n_nodes), dtype=torch.float64, device="cuda"),
                   E=torch.empty((N + 1, g.n_nodes * g.d), dtype=torch.float64, device="cuda"),
                   W=torch.empty(N + 1, dtype=torch.float64, device="cuda"),
                   stats=torch.empty((N + 1, 3), dtype=torch.float64, device="cuda"))
        for n in range(N + 1):
            h.call("nufi_mg_step_async", n, out["rho"][n].data_ptr(), out["E"][n].data_ptr(),
                   out["W"][n:].data_ptr(), out["stats"][n].data_ptr())
        h.call("nufi_check_status")
        res = {k: v.cpu().numpy() for k, v in out.items()}
        assert np.array_equal(res["rho"], ref.rho.reshape(N + 1, -1))
        assert np.array_equal(res["W"], ref.W)
        assert np.array_equal(res["E"], ref.E.reshape(N + 1, -1))
        assert np.array_equal(res["stats"], ref.stats)
        assert np.array_equal(sim.history.stacked(), ref_sim.history.stacked())
