"""B200-native (sm_100a) pseudo-spectral Navier-Stokes RHS + RK integrator hot path.

Drop-in for the hot path of the ``spectralrk`` reference (arxiv/paper_1810_10197):
the same public names for the grid, transforms, dealiasing, tendencies,
integrators, controller and driver, computing on the device through libsrk
(include/srk.h).  There is no CPU fallback: importing works anywhere, every
compute call needs a CUDA device and the built library.
"""

from .grid import Grid
from .spectral import (DealiasWorkspace, curl, dealiased_product, forward_transform, get_plan,
                       inverse_transform, pad_spectrum, symmetrize_real_planes, truncate_spectrum,
                       zero_nyquist, zero_self_conjugate_imag)
from .physics import (FlowRHS, FlowState, ForcingError, PhysParams, apply_forcing, boussinesq_rhs,
                      leray_project, ns_rhs)
from .integrators import (ButcherPair, NonFiniteStateError, StepOutcome, ab2_combine, ab2_step, make_bs5, make_dp5,
                          make_kcl5, make_pair, make_rk4, rk_step)
from .control import (AdvanceOutcome, ControllerConfig, ControllerState, StepSizeUnderflowError,
                      adaptive_advance, error_norm, error_norm_delta, propose_step, scale_vector)
from .diagnostics import (DiagnosticsRecord, SpectrumRecord, compare_series, dissipation_rate, energy_spectrum,
                          enstrophy, field_error_norms, kinetic_energy)
from .problems import ProblemSpec, hit_init, rayleigh_taylor_init, rt_tanh_init, taylor_green_init
from .simulation import (ADAPTIVE_CAPABLE, INTEGRATORS, ConfigError, RunConfig, SimulationResult,
                         default_lengths, make_initial_state, run_simulation)
from .checkpoint import (CheckpointData, CheckpointError, read_checkpoint, read_diagnostics_csv,
                         write_checkpoint, write_diagnostics_csv)
from .workprec import WorkPrecisionPoint, cell_config, work_precision, write_work_precision_csv
from .hostio import HostMirror, forcing_planes, plane_runs
from . import _native

__version__ = "0.1.0"

__all__ = [n for n in dir() if not n.startswith("_")]
