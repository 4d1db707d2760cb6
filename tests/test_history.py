"""PotentialHistory extras: the VPHIST01 checkpoint
(spline.py:105, 157-194) and the FP32 history mode (spline.py:118-125).

CPU: the checkpoint codec against files written by the unmodified reference
(tests/golden/make_golden.py checkpoints) -- byte-identical.
GPU: device history save / load / resume, FP32-history runs vs the reference's
FP32 goldens.  FP32 tolerance: a stored coefficient is a float32 rounding, so a
1e-13 difference in the fit can flip one float32 ulp (2^-24 relative); the bar is
two ulps of the slab scale for coefficients and 1e-7 for rho (the whole FP32
effect is ~2e-6), and W within 1e-6.
"""

import os

import numpy as np
import pytest

import paper_2301_05581_b200 as nufi
from paper_2301_05581_b200.configs import workload
from paper_2301_05581_b200.spline import checkpoint_bytes, read_checkpoint
from tests._util import GOLDEN, golden, normwise

CKPTS = [("kat_wl", 20, np.float64), ("tiny2_f32", 10, np.float32)]


def _base(name):
    return name[: -len("_f32")] if name.endswith("_f32") else name


@pytest.mark.parametrize("name,rows,dtype", CKPTS)
def test_checkpoint_codec_matches_reference_file(name, rows, dtype):
    path = os.path.join(GOLDEN, f"{name}_{rows}.vphist")
    w = workload(_base(name))
    grid, dt, tau, data = read_checkpoint(path, w.grid)
    assert dt == np.dtype(dtype) and tau == w.tau and data.shape == (rows, w.grid.n_nodes)
    ref = golden(name)["coeffs"][:rows]
    assert np.array_equal(data.astype(np.float64), ref)
    assert checkpoint_bytes(w.grid, dt, tau, data) == open(path, "rb").read()


def test_checkpoint_errors(tmp_path):
    w = workload("kat_wl")
    bad = tmp_path / "bad.vphist"
    bad.write_bytes(b"NOTAHIST" + bytes(30))
    with pytest.raises(nufi.UsageError):
        read_checkpoint(bad)
    good = open(os.path.join(GOLDEN, "kat_wl_20.vphist"), "rb").read()
    trunc = tmp_path / "trunc.vphist"
    trunc.write_bytes(good[:-8])
    with pytest.raises(nufi.UsageError):
        read_checkpoint(trunc)
    with pytest.raises(nufi.UsageError):
        read_checkpoint(os.path.join(GOLDEN, "kat_wl_20.vphist"), workload("wl1").grid)  # Nx mismatch
    g, _, _, _ = read_checkpoint(os.path.join(GOLDEN, "kat_wl_20.vphist"))
    assert (g.d, g.Nx, g.L) == (1, 32, w.grid.L)


def test_history_dtype_validation():
    w = workload("kat_wl")
    with pytest.raises(nufi.UsageError):
        nufi.PotentialHistory(w.grid, w.tau, dtype=np.int32)


# ---------------------------------------------------------------------------
# GPU
# ---------------------------------------------------------------------------

@pytest.mark.gpu
@pytest.mark.parametrize("name,rows,dtype", CKPTS)
def test_device_checkpoint_roundtrip(name, rows, dtype, tmp_path):
    src = os.path.join(GOLDEN, f"{name}_{rows}.vphist")
    w = workload(_base(name))
    h = nufi.PotentialHistory.load(src, w.grid)
    assert len(h) == rows and h.dtype == np.dtype(dtype)
    assert np.array_equal(h.stacked().reshape(rows, -1).astype(np.float64), golden(name)["coeffs"][:rows])
    out = tmp_path / "out.vphist"
    h.save(out)
    assert out.read_bytes() == open(src, "rb").read()


@pytest.mark.gpu
def test_resume_is_bit_identical(tmp_path):
    w = workload("kat_wl")
    full = nufi.Simulation(w.grid, w.ic, w.tau, 60).run()
    a = nufi.Simulation(w.grid, w.ic, w.tau, 60)
    a.run(29)
    ck = tmp_path / "a.vphist"
    a.history.save(ck)
    b = nufi.Simulation.resume(ck, w.grid, w.ic, 60)
    assert b.n == 30
    rest = b.run()
    assert np.array_equal(rest.rho, full.rho[30:])
    assert np.array_equal(rest.W, full.W[30:])


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["kat_wl_f32", "tiny2_f32"])
def test_f32_history_vs_reference(name):
    g = golden(name)
    g64 = golden(_base(name))
    w = workload(_base(name))
    keep = g["rho"].shape[0]
    N = len(g["W"]) - 1
    sim = nufi.Simulation(w.grid, w.ic, w.tau, N, dtype=np.float32)
    res = sim.run()
    coeffs = sim.history.stacked().reshape(N + 1, -1)
    assert coeffs.dtype == np.float32
    e_rho = normwise(res.rho[:keep], g["rho"])
    e_c = normwise(coeffs[:keep].astype(np.float64), g["coeffs"])
    e_W = np.abs(res.W - g["W"]) / np.abs(g["W"])
    assert e_c.max() <= 2 * 2.0 ** -24, e_c.max()
    assert e_rho.max() <= 1e-7, e_rho.max()
    assert e_W.max() <= 1e-6, e_W.max()
    # the mode is really active: the FP64 run differs from the FP32 reference far more
    e64 = normwise(g64["rho"][:keep], g["rho"]).max()
    assert e_rho.max() < 0.1 * e64, (e_rho.max(), e64)
