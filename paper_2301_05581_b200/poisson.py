"""The reference's poisson module (poisson.py:19-120) with the transforms on the GPU.

solve_poisson(rho) -> (phi nodal values, phi spectrum) and spline.fit_spline(phi, grid)
run as single-CTA sm_100a kernels (nufi_solve_poisson / nufi_fit_spline: separable
shared-memory DFTs, csrc/field_update.cu poisson_fit_kernel).  The per-step loop does not
use them -- it runs the fused tail (driver.advance / nufi_field_update / the run kernels);
these are the one-by-one reference operations for callers that use them directly.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .density import DensityGrid
from .errors import UsageError
from .grids import GridSpec
from .spline import _scratch_history


@dataclass(frozen=True)
class SpectralField:
    """Complex mode amplitudes in numpy FFT layout (poisson.py:35-44):
    values(x_i) = sum_alpha c_alpha exp(i 2 pi alpha.x_i / L)."""

    grid: GridSpec
    coeffs: np.ndarray
    _W: float | None = field(default=None, compare=False, repr=False)  # energy computed with the spectrum


def wavenumber_squared(grid: GridSpec) -> np.ndarray:
    """|2 pi alpha / L|^2 on the FFT grid (poisson.py:52-59)."""
    m = np.fft.fftfreq(grid.Nx, d=1.0 / grid.Nx)
    k2 = np.zeros(grid.shape_x)
    for a in range(grid.d):
        shape = [1] * grid.d
        shape[a] = grid.Nx
        k2 = k2 + ((2.0 * np.pi / grid.L) * m).reshape(shape) ** 2
    return k2


def transform_values(grid: GridSpec, values) -> SpectralField:
    """Trigonometric interpolant coefficients fftn(values) / N^d of real nodal values
    (poisson.py:72-78), by the device's separable DFT passes (nufi_transform_values)."""
    values = np.asarray(values, dtype=np.float64)
    if values.shape != grid.shape_x:
        raise UsageError(f"values must have shape {grid.shape_x}, got {values.shape}")
    vals = np.ascontiguousarray(values).reshape(-1)
    re = np.empty(grid.n_nodes)
    im = np.empty(grid.n_nodes)
    _scratch_history(grid).handle.call("nufi_transform_values", vals.ctypes.data, re.ctypes.data, im.ctypes.data)
    return SpectralField(grid=grid, coeffs=(re + 1j * im).reshape(grid.shape_x))


def forward_transform(rho: DensityGrid) -> SpectralField:
    """poisson.py:81-82."""
    return transform_values(rho.grid, rho.values)


def inverse_transform(spectrum: SpectralField) -> np.ndarray:
    """Real nodal values Re ifftn(coeffs * N^d) of the interpolant (poisson.py:85-87), on the device."""
    g = spectrum.grid
    c = np.asarray(spectrum.coeffs)
    if c.shape != g.shape_x:
        raise UsageError(f"spectrum must have shape {g.shape_x}")
    re = np.ascontiguousarray(c.real, dtype=np.float64).reshape(-1)
    im = np.ascontiguousarray(c.imag if np.iscomplexobj(c) else np.zeros(c.shape), dtype=np.float64).reshape(-1)
    out = np.empty(g.n_nodes)
    _scratch_history(g).handle.call("nufi_inverse_transform", re.ctypes.data, im.ctypes.data, out.ctypes.data)
    return out.reshape(g.shape_x)


def solve_poisson(rho: DensityGrid) -> tuple[np.ndarray, SpectralField]:
    """-laplace(phi) = rho on the torus (poisson.py:90-112), on the GPU.  Raises
    NumericalConsistencyError when |mean rho| > 1e-8 max|rho|."""
    grid = rho.grid
    vals = np.ascontiguousarray(rho.values, dtype=np.float64).reshape(-1)
    phi = np.empty(grid.n_nodes)
    re = np.empty(grid.n_nodes)
    im = np.empty(grid.n_nodes)
    W = np.empty(1)
    h = _scratch_history(grid)
    h.handle.call("nufi_solve_poisson", vals.ctypes.data, phi.ctypes.data, re.ctypes.data, im.ctypes.data,
                  W.ctypes.data)
    spec = SpectralField(grid=grid, coeffs=(re + 1j * im).reshape(grid.shape_x), _W=float(W[0]))
    return phi.reshape(grid.shape_x), spec


def electric_energy(spectrum: SpectralField) -> float:
    """(1/2) L^d sum k^2 |phi_hat|^2 (poisson.py:115-120).  For a spectrum from
    solve_poisson this is the value its kernel computed on the GPU."""
    if spectrum._W is not None:
        return spectrum._W
    c = np.asarray(spectrum.coeffs)
    if c.shape != spectrum.grid.shape_x:
        raise UsageError(f"spectrum must have shape {spectrum.grid.shape_x}")
    g = spectrum.grid
    return 0.5 * g.L ** g.d * float(np.add.reduce((wavenumber_squared(g) * np.abs(c) ** 2).reshape(-1)))
