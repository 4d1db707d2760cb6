"""ctypes binding of libnufi_b200.so (C-ABI declared in include/nufi.h).

The shared library is built in-tree (paper_2301_05581_b200/libnufi_b200.so) by
`__graft_entry__.build()` / `make -C paper_2301_05581_b200/csrc`.  There is no
fallback: if the library (or a CUDA device) is missing, every call raises.
"""

from __future__ import annotations

import ctypes
import math
import os

from .errors import ConfigError, NumericalConsistencyError, UsageError, VpflowError

HERE = os.path.dirname(os.path.abspath(__file__))
# experiment builds of the same sources with other compile-time options live beside it
# (make EXTRA=... LIB=../libnufi_b200_<tag>.so BUILD=build_<tag>); NUFI_LIB_VARIANT=<tag> loads one
_VARIANT = "".join(ch for ch in os.environ.get("NUFI_LIB_VARIANT", "") if ch.isalnum() or ch == "_")
LIB_PATH = os.path.join(HERE, f"libnufi_b200_{_VARIANT}.so" if _VARIANT else "libnufi_b200.so")

NUFI_OK = 0
NUFI_ERR_USAGE = 1
NUFI_ERR_NUMERICAL = 2
NUFI_ERR_CONFIG = 3
NUFI_ERR_CUDA = 4
NUFI_ERR_COMM = 5
NUFI_MAX_CENTERS = 4
NUFI_TRACE_FAST = 0
NUFI_TRACE_PARITY = 1
NUFI_FLAG_F32_HISTORY = 1


class CudaError(VpflowError):
    """A CUDA runtime failure inside libnufi_b200."""


class CommError(VpflowError):
    """A collective-communication failure."""


class NufiProfile(ctypes.Structure):
    _fields_ = [
        ("n_centers", ctypes.c_int32),
        ("power", ctypes.c_int32),
        ("centers", ctypes.c_double * NUFI_MAX_CENTERS),
        ("weights", ctypes.c_double * NUFI_MAX_CENTERS),
    ]


class NufiConfig(ctypes.Structure):
    _fields_ = [
        ("d", ctypes.c_int32),
        ("Nx", ctypes.c_int32),
        ("Nv", ctypes.c_int32),
        ("n_max", ctypes.c_int32),
        ("L", ctypes.c_double),
        ("vmax", ctypes.c_double),
        ("tau", ctypes.c_double),
        ("alpha", ctypes.c_double),
        ("k", ctypes.c_double),
        ("rho_bar", ctypes.c_double),
        ("profiles", NufiProfile * 3),
        ("v_blocks", ctypes.c_int32),
        ("block_lo", ctypes.c_int32),
        ("block_hi", ctypes.c_int32),
        ("flags", ctypes.c_int32),
    ]


_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I64P = ctypes.POINTER(ctypes.c_int64)
_D = ctypes.c_double

# name -> argtypes (all return int status unless listed in _RESTYPE)
_SIGS = {
    "nufi_create": [ctypes.POINTER(NufiConfig), ctypes.c_int, _P, ctypes.POINTER(_P)],
    "nufi_destroy": [_P],
    "nufi_last_error": [],
    "nufi_abi_version": [],
    "nufi_sync": [_P],
    "nufi_rho_bar": [_P, ctypes.POINTER(_D)],
    "nufi_set_initial_condition": [_P, ctypes.POINTER(NufiConfig)],
    "nufi_reserve": [_P, _I64],
    "nufi_capacity": [_P],
    "nufi_history_len": [_P, _I64P],
    "nufi_load_history": [_P, _P, _I64],
    "nufi_get_history": [_P, _P, _I64, _I64],
    "nufi_append_coeffs": [_P, _P],
    "nufi_truncate_history": [_P, _I64],
    "nufi_rho": [_P, _I64, _P, _P, _I64P],
    "nufi_rho_partials": [_P, _I64, _P, _I64P],
    "nufi_rho_finish": [_P, _P, _P, _P],
    "nufi_step_finish": [_P, _I64, _P, _P, _P, _P, _P],
    "nufi_step_finish_async": [_P, _I64, _P, _P, _P, _P, _P],
    "nufi_check_status": [_P],
    "nufi_mg_setup": [_P, ctypes.c_int, ctypes.c_int, ctypes.c_int, _P],
    "nufi_mg_connect": [_P, _P],
    "nufi_mg_handle_size": [],
    "nufi_mg_teardown": [_P],
    "nufi_mg_step_async": [_P, _I64, _P, _P, _P, _P],
    "nufi_partials_len": [_P],
    "nufi_field_update": [_P, _P, _P, _P, _P],
    "nufi_async_slots": [_P, ctypes.c_int],
    "nufi_rho_async": [_P, _I64, ctypes.c_int, _I64P, ctypes.POINTER(ctypes.c_int)],
    "nufi_commit_async": [_P, _I64],
    "nufi_field_update_async": [_P, _P, ctypes.c_int],
    "nufi_async_wait": [_P, ctypes.c_int, ctypes.POINTER(ctypes.POINTER(ctypes.c_double))],
    "nufi_async_ring": [_P, ctypes.POINTER(ctypes.POINTER(ctypes.c_double)), ctypes.POINTER(ctypes.c_int64)],
    "nufi_step": [_P, _I64, _P, _P, _P, _P, _I64P],
    "nufi_run": [_P, _I64, _P, _P, _P, _P, _I64P],
    "nufi_trace": [_P, _I64, _P, _P, _I64, ctypes.c_int, ctypes.c_int, _I64P],
    "nufi_eval_f0": [_P, _P, _P, _I64, _P],
    "nufi_bspline_weights": [_P, _P, _I64, _P, _P],
    "nufi_eval_field": [_P, _I64, _P, _I64, _P, _P],
    "nufi_set_uniform_field": [_P, _I64, _P],
    "nufi_set_spline_field": [_P, _I64, _P],
    "nufi_clear_fields": [_P],
    "nufi_solve_poisson": [_P, _P, _P, _P, _P, _P],
    "nufi_fit_spline": [_P, _P, _P],
    "nufi_transform_values": [_P, _P, _P, _P],
    "nufi_inverse_transform": [_P, _P, _P, _P],
    "nufi_moments": [_P, _I64, _P, _I64P],
    "nufi_profiling": [_P, ctypes.c_int],
    "nufi_profiling_read": [_P, _P],
    "nufi_fp64_peak": [ctypes.c_int, ctypes.POINTER(_D), ctypes.POINTER(_D)],
}
_RESTYPE = {"nufi_last_error": ctypes.c_char_p, "nufi_partials_len": _I64, "nufi_capacity": _I64}
EXPORTS = tuple(_SIGS)

_lib = None


def load():
    """Load the CUDA library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU fallback)"
            )
        lib = ctypes.CDLL(LIB_PATH)
        for name, args in _SIGS.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = _RESTYPE.get(name, ctypes.c_int)
        _lib = lib
    return _lib


def check(rc: int) -> None:
    if rc == NUFI_OK:
        return
    msg = load().nufi_last_error().decode(errors="replace")
    if rc == NUFI_ERR_USAGE:
        raise UsageError(msg)
    if rc == NUFI_ERR_NUMERICAL:
        raise NumericalConsistencyError(msg)
    if rc == NUFI_ERR_CONFIG:
        raise ConfigError(msg)
    if rc == NUFI_ERR_COMM:
        raise CommError(msg)
    raise CudaError(msg)


def make_config(grid, ic, tau: float, n_max: int, rho_bar: float | None = None, v_blocks: int = 0,
                block_lo: int = 0, block_hi: int = 0, flags: int = 0) -> NufiConfig:
    c = NufiConfig()
    c.d = grid.d
    c.Nx = grid.Nx
    c.Nv = grid.Nv
    c.n_max = int(n_max)
    c.L = float(grid.L)
    c.vmax = float(grid.vmax)
    c.tau = float(tau)
    c.alpha = float(ic.alpha)
    c.k = float(ic.k)
    c.rho_bar = math.nan if rho_bar is None else float(rho_bar)
    for a, p in enumerate(ic.profiles):
        if len(p.centers) > NUFI_MAX_CENTERS:
            raise ConfigError(f"at most {NUFI_MAX_CENTERS} mixture centers per axis")
        c.profiles[a].n_centers = len(p.centers)
        c.profiles[a].power = int(p.power)
        for m, (cc, w) in enumerate(zip(p.centers, p.weights)):
            c.profiles[a].centers[m] = float(cc)
            c.profiles[a].weights[m] = float(w)
    c.v_blocks = int(v_blocks)
    c.block_lo = int(block_lo)
    c.block_hi = int(block_hi)
    c.flags = int(flags)
    return c


def ptr(a) -> int | None:
    """Raw address of a numpy array or torch tensor (None passes NULL)."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    return a.ctypes.data


class Handle:
    """Owns one nufi_handle (one GPU / rank)."""

    def __init__(self, cfg: NufiConfig, device: int = 0, stream: int | None = None):
        lib = load()
        h = _P()
        check(lib.nufi_create(ctypes.byref(cfg), int(device), stream, ctypes.byref(h)))
        self._h = h
        self.cfg = cfg
        self.device = device
        self.lib = lib

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                self.lib.nufi_destroy(h)
            except Exception:  # pragma: no cover - interpreter shutdown
                pass
            self._h = None

    @property
    def h(self):
        return self._h

    def call(self, name: str, *args) -> None:
        check(getattr(self.lib, name)(self._h, *args))
