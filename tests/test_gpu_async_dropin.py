"""The stream-ordered drop-in pair compute_rho / advance (pending.py, nufi_rho_async /
nufi_field_update_async): same results as the whole-run kernel and the reference goldens,
results readable in any order and long after the ring slot was reused, usage errors still
synchronous, a non-neutral host density still rejected before anything is appended."""

import numpy as np
import pytest

import paper_2301_05581_b200 as nufi
from paper_2301_05581_b200.configs import workload
from tests._util import golden, normwise

pytestmark = pytest.mark.gpu


def _loop(name, N, read_each_step=True):
    w = workload(name)
    hist = nufi.PotentialHistory(w.grid, w.tau, capacity=N + 1)
    ctx = nufi.FlowContext(history=hist, ic=w.ic, tau=w.tau, grid=w.grid)
    rs, us = [], []
    for n in range(N + 1):
        r = nufi.compute_rho(ctx, n)
        u = nufi.advance(ctx, r.density)
        if read_each_step:
            _ = u.W
        rs.append(r)
        us.append(u)
    return w, ctx, rs, us


@pytest.mark.parametrize("name,N", [("kat_wl", 100), ("tiny2", 20), ("tiny3", 10), ("rag1", 30)])
@pytest.mark.parametrize("read_each_step", [True, False])
def test_async_loop_matches_run_and_reference(name, N, read_each_step):
    w, ctx, rs, us = _loop(name, N, read_each_step)
    ref = nufi.Simulation(w.grid, w.ic, w.tau, N).run()
    rho = np.stack([r.density.values.reshape(-1) for r in rs])  # read after the ring wrapped (N > 64)
    W = np.array([u.W for u in us])
    assert normwise(rho, ref.rho.reshape(N + 1, -1)).max() <= 1e-14
    assert np.abs(W - ref.W).max() <= 1e-13 * np.abs(ref.W).max()
    g = golden(name)
    k = min(len(g["rho"]), N + 1)
    assert normwise(rho[:k], g["rho"][:k]).max() <= 1e-10
    coeffs = np.stack([u.coeffs.reshape(-1) for u in us])
    assert np.array_equal(coeffs, ctx.history.stacked().reshape(N + 1, -1))
    E = np.stack([u.E.reshape(-1) for u in us])
    assert normwise(E[:k], g["E"][:k].reshape(k, -1)).max() <= 1e-10
    st = np.array([[r.neutralization, r.f_min, r.f_max] for r in rs])
    assert np.abs(st[:, 1:] - ref.stats[:, 1:]).max() <= 1e-13
    assert ctx.field_evals == ref.field_evals
    assert len(ctx.history) == N + 1


def test_async_usage_errors_stay_synchronous():
    w = workload("kat_wl")
    hist = nufi.PotentialHistory(w.grid, w.tau, capacity=8)
    ctx = nufi.FlowContext(history=hist, ic=w.ic, tau=w.tau, grid=w.grid)
    with pytest.raises(nufi.UsageError):
        nufi.compute_rho(ctx, 3)  # history holds 0 fields (flow.py:55-62)
    r = nufi.compute_rho(ctx, 0)
    bad = nufi.DensityGrid(w.grid, np.full(w.grid.shape_x, 0.5))
    with pytest.raises(nufi.NumericalConsistencyError):
        nufi.advance(ctx, bad)
    assert len(hist) == 0
    u = nufi.advance(ctx, r.density)
    assert len(hist) == 1 and u.W > 0


def test_device_density_replaced_falls_back_to_host_values():
    """compute_rho, then another call that overwrites the device density, then advance of
    the first result: the tail must use the first result's values."""
    w = workload("kat_wl")
    N = 12
    hist = nufi.PotentialHistory(w.grid, w.tau, capacity=N + 1)
    ctx = nufi.FlowContext(history=hist, ic=w.ic, tau=w.tau, grid=w.grid)
    ref = nufi.Simulation(w.grid, w.ic, w.tau, N).run()
    for n in range(N + 1):
        r = nufi.compute_rho(ctx, n)
        if n % 3 == 1:
            nufi.compute_rho(ctx, n)  # a second density replaces the device copy
        u = nufi.advance(ctx, r.density)
        assert abs(u.W - ref.W[n]) <= 1e-13 * abs(ref.W[n])


def test_device_side_failure_reconciles_the_length_after_truncate():
    """A tail that fails its neutrality check on the device reports the history length as
    its own slot (nothing appended), so the host length is reconciled correctly even when
    the device's previous length is stale (a truncate, or an uncommitted speculative step)."""
    from paper_2301_05581_b200.pending import Entry, ring_of

    w = workload("kat_wl")
    sim = nufi.Simulation(w.grid, w.ic, w.tau, 10)
    sim.run()
    hist = sim.history
    assert len(hist) == 11
    hist.truncate(5)
    r = nufi.compute_rho(sim.ctx, 5)  # speculative whole step 5 (uncommitted)
    _ = r.density.values
    ring = ring_of(hist)
    e = Entry(ring, "field")
    bad = np.ones(w.grid.n_nodes)  # not neutral: the device check fails (the host check is bypassed)
    hist.handle.call("nufi_field_update_async", bad.ctypes.data, e.slot)
    with pytest.raises(nufi.NumericalConsistencyError):
        e.materialize()
    assert len(hist) == 5
    u = nufi.advance(sim.ctx, nufi.compute_rho(sim.ctx, 5).density)  # the loop carries on
    assert len(hist) == 6 and u.W > 0


def test_entries_after_a_device_failure_raise_too():
    """Steps enqueued after one whose tail failed are skipped on the device; reading any of
    them raises (not stale values), also after the first failure was reported."""
    from paper_2301_05581_b200.pending import Entry, ring_of

    w = workload("kat_wl")
    hist = nufi.PotentialHistory(w.grid, w.tau, capacity=16)
    ctx = nufi.FlowContext(history=hist, ic=w.ic, tau=w.tau, grid=w.grid)
    for n in range(3):
        nufi.advance(ctx, nufi.compute_rho(ctx, n).density)
    ring = ring_of(hist)
    bad = np.ones(w.grid.n_nodes)  # not neutral: the device check fails (host check bypassed)
    e1 = Entry(ring, "field")
    hist.handle.call("nufi_field_update_async", bad.ctypes.data, e1.slot)
    good = nufi.compute_rho(ctx, 3)  # enqueued behind the failure: skipped on the device
    u2 = nufi.advance(ctx, good.density)
    with pytest.raises(nufi.NumericalConsistencyError):
        e1.materialize()
    with pytest.raises(nufi.NumericalConsistencyError):
        _ = u2.W
    assert len(hist) == 3
    u = nufi.advance(ctx, nufi.compute_rho(ctx, 3).density)  # the loop recovers
    assert len(hist) == 4 and u.W > 0
