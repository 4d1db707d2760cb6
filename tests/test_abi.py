"""The C-ABI boundary (CPU only): the library loads, exports every symbol that
include/nufi.h declares, and the ctypes structs match the C layout."""

import ctypes
import os
import re
import subprocess
import tempfile

import pytest

from paper_2301_05581_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "nufi.h")


def header_functions():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z0-9_]+\s*\*?\s*(nufi_[a-z0-9_]+)\s*\(", src, re.M)))


def test_header_declares_expected_entry_points():
    names = header_functions()
    for must in ("nufi_create", "nufi_rho", "nufi_field_update", "nufi_step", "nufi_run", "nufi_trace",
                 "nufi_rho_partials", "nufi_rho_finish", "nufi_load_history", "nufi_get_history"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    missing = [n for n in header_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_covers_header():
    assert set(header_functions()) == set(_lib.EXPORTS)


def test_abi_version():
    assert _lib.load().nufi_abi_version() == 1


def test_struct_layout_matches_c():
    probe = r"""
#include <stddef.h>
#include <stdio.h>
#include "nufi.h"
int main(void) {
  printf("%zu %zu %zu %zu %zu %zu\n", sizeof(nufi_config), sizeof(nufi_profile),
         offsetof(nufi_config, rho_bar), offsetof(nufi_config, profiles),
         offsetof(nufi_config, v_blocks), offsetof(nufi_config, flags));
  return 0;
}
"""
    cc = "/usr/bin/gcc" if os.path.exists("/usr/bin/gcc") else "gcc"
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "p.c")
        exe = os.path.join(d, "p")
        open(c, "w").write(probe)
        subprocess.run([cc, "-I", os.path.dirname(HEADER), c, "-o", exe], check=True)
        got = list(map(int, subprocess.run([exe], check=True, capture_output=True, text=True).stdout.split()))
    C = _lib.NufiConfig
    want = [ctypes.sizeof(C), ctypes.sizeof(_lib.NufiProfile), C.rho_bar.offset, C.profiles.offset,
            C.v_blocks.offset, C.flags.offset]
    assert got == want


def test_create_without_gpu_fails_loudly():
    """No silent CPU fallback: without a device the create call returns an error."""
    try:
        import torch

        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    from paper_2301_05581_b200.configs import workload

    w = workload("kat_wl")
    cfg = _lib.make_config(w.grid, w.ic, w.tau, 10)
    with pytest.raises(Exception):
        _lib.Handle(cfg, 0)


def test_validation_errors_without_gpu():
    """Config validation runs before any device call and maps to UsageError."""
    from paper_2301_05581_b200.configs import workload
    from paper_2301_05581_b200.errors import UsageError

    w = workload("kat_wl")
    cfg = _lib.make_config(w.grid, w.ic, -1.0, 10)
    with pytest.raises(UsageError, match="time step must be positive"):
        _lib.Handle(cfg, 0)
    cfg = _lib.make_config(w.grid, w.ic, w.tau, 10)
    cfg.Nx = 3
    with pytest.raises(UsageError, match="Nx >= 4"):
        _lib.Handle(cfg, 0)
    cfg = _lib.make_config(w.grid, w.ic, w.tau, 10)
    cfg.k = 0.3
    with pytest.raises(UsageError, match="multiple of 2\\*pi"):
        _lib.Handle(cfg, 0)


def test_size_limits_without_gpu():
    """Maximum sizes: grids up to Nx^d = 2^21 (128^3) are accepted (beyond 4096 nodes the
    tail runs multi-CTA, field_large.cu); larger grids are refused with ConfigError before
    any device work, as are unknown flags."""
    from paper_2301_05581_b200.configs import workload
    from paper_2301_05581_b200.errors import ConfigError, UsageError

    w = workload("wl3")
    cfg = _lib.make_config(w.grid, w.ic, w.tau, 10)
    cfg.Nx = 129  # 2 146 689 nodes
    with pytest.raises(ConfigError, match="supported grid size"):
        _lib.Handle(cfg, 0)
    w2 = workload("wl2")
    cfg = _lib.make_config(w2.grid, w2.ic, w2.tau, 10)
    cfg.flags = 8
    with pytest.raises(UsageError, match="flags"):
        _lib.Handle(cfg, 0)
