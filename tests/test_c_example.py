"""The C-ABI used from plain C (tools/c_example/nufi_run.c): it compiles and links
against libnufi_b200.so here; on the GPU it runs and reproduces the reference's
energy series (tests/golden/kat_wl.npz) -- no Python or torch on that path."""

import os
import subprocess

import numpy as np
import pytest

from tests._util import golden

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2301_05581_b200")


def _build(tmp_path):
    exe = str(tmp_path / "nufi_run")
    cc = "/usr/bin/gcc" if os.path.exists("/usr/bin/gcc") else "gcc"
    subprocess.run([cc, "-O2", "-I", os.path.join(ROOT, "include"), os.path.join(ROOT, "tools", "c_example", "nufi_run.c"),
                    "-L", LIBDIR, "-lnufi_b200", "-lm", "-Wl,-rpath," + LIBDIR, "-o", exe], check=True)
    return exe


def test_c_example_links(tmp_path):
    assert os.path.exists(_build(tmp_path))


@pytest.mark.gpu
def test_c_example_runs_and_matches_reference(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe, "40"], capture_output=True, text=True)
    assert r.returncode == 0, (r.returncode, r.stderr[-2000:], r.stdout[-500:])
    out = r.stdout
    W = np.array([float(l.split()[1]) for l in out.splitlines() if l and not l.startswith("#")])
    ref = golden("kat_wl")["W"][:41]
    assert W.shape == ref.shape
    assert np.max(np.abs(W - ref) / np.abs(ref)) <= 1e-6
