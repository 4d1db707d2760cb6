"""B200-native NuFI (numerical flow iteration for Vlasov-Poisson, arXiv 2301.05581).

Drop-in for the reference package's (vpflow) per-step rho loop, with the hot
path — backward characteristic trace -> f0 at the foot point -> v-reduction to
rho, plus the per-step Poisson / spline append — in hand-written sm_100a CUDA
(libnufi_b200.so, C-ABI in include/nufi.h).  Host code mirrors the reference's
module names: grids, initial, spline, flow, density, driver.
"""

from .density import (DEFAULT_CHUNK, ConservedMoments, DensityGrid, RhoResult, compute_rho, conserved_moments,
                      quadrature_sweep, quadrature_sweep_many)
from .diagnostics import DiagnosticsRecord, conserved_quantities, electric_energy_from_coeffs, fit_damping_rate
from .driver import FieldUpdate, RunResult, Simulation, StepOutput, advance, point_steps, run_simulation
from .errors import ConfigError, FitError, NumericalConsistencyError, UsageError, VpflowError
from .flow import (TRACE_FAST, TRACE_PARITY, FlowContext, eval_f, eval_f0, eval_f_batch, psi, psi_batch,
                   psi_tilde, psi_tilde_batch, trace_backward)
from .grids import GridSpec, PhasePoint, v_mid, v_mid_matrix, x_node, x_node_matrix
from .initial import (BENCHMARK_DEFAULTS, InitialCondition, VelocityProfile, background_density, make_benchmark,
                      weak_landau_3d)
from .poisson import (SpectralField, electric_energy, forward_transform, inverse_transform, solve_poisson,
                      transform_values, wavenumber_squared)
from .spline import PotentialHistory, SplineField, UniformField, fit_spline

__version__ = "0.1.0"
