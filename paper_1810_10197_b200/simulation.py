"""Device-resident stepping loops (mirrors simulation.py:64-368 of the reference).

Same bookkeeping as the reference driver: cached tendency f_now, FSAL reuse,
evaluation accounting (RK4 4/step + 1, BS5 7/step + 1), lattice timestamps,
final-step clamping with the working-h restore, forcing after every accepted
step.  Additions: an initial-condition hook (``initial_state``) and an
accepted-step cap (``max_steps``) -- SURVEY D4 / D6.  Per accepted step there
is one device->host read (the fused error-norm + E/eps/Z sums).
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np
import torch

from .control import ControllerConfig, ControllerState, adaptive_advance
from .diagnostics import DiagnosticsRecord, diag_from_sums, reduce_sums
from .grid import Grid
from .integrators import NonFiniteStateError, make_pair, make_rk4, run_stages
from .physics import FlowRHS, FlowState, apply_forcing
from .problems import ProblemSpec, hit_init, rayleigh_taylor_init, taylor_green_init
from .spectral import to_device
from .checkpoint import CheckpointData, CheckpointError, write_checkpoint, write_diagnostics_csv

__all__ = ["RunConfig", "ConfigError", "default_lengths", "make_initial_state", "SimulationResult",
           "run_simulation", "INTEGRATORS", "ADAPTIVE_CAPABLE"]

INTEGRATORS = ("ab2", "rk4", "dp5", "kcl5", "bs5")
ADAPTIVE_CAPABLE = ("dp5", "kcl5", "bs5")


class ConfigError(ValueError):
    """Invalid or inconsistent configuration (config.py:16)."""


@dataclass
class RunConfig:
    """Same fields as the reference RunConfig (config.py:55-117)."""

    grid_shape: tuple
    problem: ProblemSpec
    integrator: str
    mode: str
    t_end: float
    lengths: tuple | None = None
    h: float | None = None
    tol_abs: float = 1e-6
    tol_rel: float = 1e-6
    h0: float = 1e-3
    output_dir: str | None = None
    checkpoint_interval: float | None = None
    forcing: bool = False
    k_f: float = 2.0
    controller: ControllerConfig = field(default_factory=ControllerConfig)

    def validate(self):
        if self.integrator not in INTEGRATORS:
            raise ConfigError(f"unknown integrator {self.integrator!r}")
        if self.mode not in ("fixed", "adaptive"):
            raise ConfigError(f"mode must be fixed or adaptive, got {self.mode!r}")
        if self.mode == "adaptive" and self.integrator not in ADAPTIVE_CAPABLE:
            raise ConfigError(f"integrator {self.integrator} has no embedded error estimate")
        if self.mode == "fixed" and (self.h is None or self.h <= 0.0):
            raise ConfigError("fixed mode requires a positive step size h")
        if self.mode == "adaptive":
            for name, tol in (("tol_abs", self.tol_abs), ("tol_rel", self.tol_rel)):
                if tol <= 0.0:
                    raise ConfigError(f"{name} must be positive, got {tol}")
                if not 1e-10 <= tol <= 1e-2:
                    warnings.warn(f"{name} = {tol:g} lies outside the tested range", stacklevel=2)
            if self.h0 <= 0.0:
                raise ConfigError("adaptive mode requires a positive initial step h0")
        if self.t_end <= 0.0:
            raise ConfigError(f"t_end must be positive, got {self.t_end}")
        if self.problem.kind not in ("taylor_green", "rayleigh_taylor", "hit"):
            raise ConfigError(f"unknown problem kind {self.problem.kind!r}")
        if self.problem.kind == "hit" and self.problem.seed is None:
            raise ConfigError("hit requires a seed")
        if self.forcing and self.problem.kind != "hit":
            raise ConfigError("forcing is only meaningful for the hit problem")
        self.controller.tol_abs = self.tol_abs
        self.controller.tol_rel = self.tol_rel
        return self

    @property
    def has_density(self):
        return self.problem.kind == "rayleigh_taylor"


def default_lengths(kind, shape):
    """config.py:142-152."""
    if kind == "rayleigh_taylor":
        base = 2.0 * np.pi
        return tuple([base] * (len(shape) - 1) + [base * shape[-1] / shape[0]])
    return (2.0 * np.pi,) * len(shape)


def make_initial_state(config) -> FlowState:
    """simulation.py:64-77."""
    lengths = config.lengths if config.lengths is not None else default_lengths(config.problem.kind,
                                                                                config.grid_shape)
    grid = Grid(config.grid_shape, lengths)
    kind = config.problem.kind
    if kind == "taylor_green":
        return taylor_green_init(grid)
    if kind == "rayleigh_taylor":
        return rayleigh_taylor_init(grid, config.problem)
    return hit_init(grid, config.problem)


@dataclass
class SimulationResult:
    records: list
    state: FlowState
    t: float
    rhs_evals: int
    rejections: int
    steps: int
    errs: list = field(default_factory=list)


def _rng_state_tuple(rng):
    st = rng.bit_generator.state["state"]
    return (st["state"], st["inc"])


def _rng_from_tuple(tup):
    rng = np.random.default_rng()
    state = rng.bit_generator.state
    state["state"]["state"], state["state"]["inc"] = tup
    rng.bit_generator.state = state
    return rng


class _Driver:
    """simulation.py:93-219 on device tensors (cached tendency, FSAL, accounting,
    resume, periodic SRKL checkpoints)."""

    def __init__(self, config, initial_state=None, resume=None):
        self.config = config
        if resume is not None:
            if tuple(resume.grid.shape) != tuple(config.grid_shape):
                raise CheckpointError(f"checkpoint grid {resume.grid.shape} does not match configured grid "
                                      f"{tuple(config.grid_shape)}")
            if resume.has_density != config.has_density:
                raise CheckpointError("checkpoint and configuration disagree on the presence of a density field")
            self.grid = resume.grid
            self.y = to_device(resume.fields, torch.complex128)[0].clone()
            self.t = resume.time
            self.evals = resume.rhs_evals
            self.rejections = resume.rejections
            self.steps = resume.steps
            self.f_now = None if resume.f_now is None else to_device(resume.f_now, torch.complex128)[0].clone()
            self.prev_rejected = resume.prev_rejected
            self.h_ctrl = resume.h
            self.rng = (_rng_from_tuple(resume.rng_state) if resume.rng_state is not None
                        else np.random.default_rng(config.problem.seed))
        else:
            if initial_state is None:
                st = make_initial_state(config)
            elif callable(initial_state):
                st = initial_state(config)
            else:
                st = initial_state
            if isinstance(st, FlowState):
                self.grid, y = st.grid, st.fields
            else:
                lengths = config.lengths or default_lengths(config.problem.kind, config.grid_shape)
                self.grid, y = Grid(config.grid_shape, lengths), st
            self.y = to_device(y, torch.complex128)[0].clone()
            self.t = 0.0
            self.evals = 0
            self.rejections = 0
            self.steps = 0
            self.f_now = None
            self.h_ctrl = config.h if config.mode == "fixed" else config.h0
            self.prev_rejected = False
            self.rng = np.random.default_rng(config.problem.seed)
        self.rhs = FlowRHS(self.grid, config.problem.params, density=config.has_density)
        if self.f_now is None:
            self.f_now = self.rhs(self.t, self.y)
            self.evals += 1
        self.records = []
        self.errs = []
        self.graphs = False  # run_simulation decides (CUDA-graph replay of attempts)
        self.second_input = self.refresh_sums = None
        out_dir = getattr(config, "output_dir", None)
        self.out_dir = Path(out_dir) if out_dir else None
        if self.out_dir is not None:
            self.out_dir.mkdir(parents=True, exist_ok=True)
        interval = getattr(config, "checkpoint_interval", None)
        self._next_checkpoint = None
        if interval is not None and self.out_dir is not None:
            self._next_checkpoint = (int(np.floor(self.t / interval + 1e-9)) + 1) * interval

    def maybe_checkpoint(self):
        """simulation.py:184-191."""
        if self._next_checkpoint is None:
            return
        if self.t + 1e-12 >= self._next_checkpoint:
            write_checkpoint(self.out_dir / f"checkpoint_t{self.t:.6f}.srkl", self.snapshot())
            while self._next_checkpoint <= self.t + 1e-12:
                self._next_checkpoint += self.config.checkpoint_interval

    def snapshot(self) -> CheckpointData:
        cfg = self.config
        return CheckpointData(grid=self.grid, fields=self.y, has_density=cfg.has_density, time=self.t,
                              h=self.h_ctrl, prev_rejected=self.prev_rejected, rhs_evals=self.evals,
                              rejections=self.rejections, steps=self.steps, f_now=self.f_now,
                              rng_state=_rng_state_tuple(self.rng), forcing=cfg.forcing, k_f=cfg.k_f,
                              forcing_energy=cfg.problem.energy)

    def record(self, h, sums=None):
        d = self.grid.dims
        if sums is None:
            # every component (density too) in the non-finite count; E / eps / Z stay
            # over the velocity components (the kernel's dvel = min(dims, ncomp))
            sums = reduce_sums(self.grid, self.y, fl=self.f_now, flags=2, ncomp=self.y.shape[0], host=True).tolist()
            if sums[6] > 0:
                raise NonFiniteStateError(f"non-finite state at t={self.t}")
        e, eps, z = diag_from_sums(sums, self.grid)
        self.records.append(DiagnosticsRecord(t=self.t, h=h, e_kin=e, eps=eps, rhs_evals=self.evals,
                                              rejections=self.rejections, enstrophy=z))

    def after_accept(self, last_stage, fsal_ok, energy_sum=None, next_coef=None):
        """simulation.py:165-182. Returns True when f_now is the FSAL stage.
        energy_sum: sum_w |u|^2 of the new state from the step reduction, if known.
        next_coef=(h, h a21): when f_now has to be recomputed, do it with
        FlowRHS.refresh -- the same f_now, plus the diagnostics sums of the new
        state (``refresh_sums``) and the next attempt's stage-2 input for step
        size h (``second_input``) from the same pass."""
        cfg = self.config
        forced = False
        if cfg.forcing:
            apply_forcing(self.y[: self.grid.dims], self.grid, cfg.problem.energy, cfg.k_f,
                          energy_sum=energy_sum)
            forced = True
        self.steps += 1
        self.second_input = self.refresh_sums = None
        if fsal_ok and not forced and last_stage is not None:
            self.f_now = last_stage
            return True
        if next_coef is not None:
            self.f_now, y2, sums = self.rhs.refresh(self.t, self.y, next_coef[1])
            if not all(np.isfinite(sums[k]) for k in (4, 5, 8)):
                raise NonFiniteStateError(f"non-finite state at t={self.t}")
            self.second_input, self.refresh_sums = (next_coef[0], y2), sums
        else:
            self.f_now = self.rhs(self.t, self.y)
        self.evals += 1
        return False

    def result(self):
        return SimulationResult(records=self.records, state=FlowState(grid=self.grid, fields=self.y), t=self.t,
                                rhs_evals=self.evals, rejections=self.rejections, steps=self.steps, errs=self.errs)


def _fixed_step_times(drv, h, t_end):
    """simulation.py:222-247."""
    t0 = drv.t
    remaining = t_end - t0
    n_full = int(np.floor(remaining / h + 1e-9))
    h_last = remaining - n_full * h
    if h_last < 1e-12 * h:
        h_last = 0.0
    base = drv.steps
    on_lattice = abs(t0 - base * h) <= 1e-9 * max(1.0, abs(t0))

    def time_at(i):
        if i >= n_full:
            return t_end
        if on_lattice:
            return (base + i + 1) * h
        return t0 + (i + 1) * h

    total = n_full + (1 if h_last > 0.0 else 0)
    return total, n_full, h_last, time_at


def _run_fixed(drv, max_steps=None):
    """simulation.py:250-271 (RK pairs; AB2 bootstraps with RK4, :274-310)."""
    cfg = drv.config
    h, t_end = cfg.h, cfg.t_end
    drv.record(h)
    if cfg.integrator == "ab2":
        return _run_ab2(drv, h, t_end, max_steps)
    pair = make_pair(cfg.integrator)
    total, n_full, h_last, time_at = _fixed_step_times(drv, h, t_end)
    if max_steps is not None:
        total = min(total, max_steps)
    graph = None
    if drv.graphs and not cfg.forcing and drv.y.numel() * drv.y.element_size() <= _graph_max_bytes():
        from .graphs import attempt_graph

        graph = attempt_graph(drv.rhs, pair, cfg.controller, drv.grid, fixed=True)
    for i in range(total):
        h_i = h if i < n_full else h_last
        if graph is not None:  # the whole step + the cached tendency + the record's sums, one replay
            drv.y, drv.f_now, sums = graph.step_fixed(drv.y, h_i, drv.f_now)
            if sums[6] > 0:
                raise NonFiniteStateError(f"non-finite state at t={time_at(i)}")
            drv.evals += pair.s - 1 + (0 if pair.fsal else 1)
            drv.t = time_at(i)
            drv.steps += 1
            drv.record(h_i, sums=sums)
            drv.maybe_checkpoint()
            continue
        stages, y_new, ev = run_stages(drv.rhs, drv.y, drv.t, h_i, pair, drv.f_now)
        drv.evals += ev
        drv.y = y_new
        drv.t = time_at(i)
        drv.after_accept(stages[-1] if pair.fsal else None, fsal_ok=pair.fsal)
        drv.record(h_i)
        drv.maybe_checkpoint()
    if graph is not None:  # hand back buffers the graph will not overwrite
        drv.y = drv.y.clone()
        drv.f_now = drv.f_now.clone()


def _run_ab2(drv, h, t_end, max_steps=None):
    from .integrators import ab2_combine

    total, n_full, h_last, time_at = _fixed_step_times(drv, h, t_end)
    if max_steps is not None:
        total = min(total, max_steps)
    if total == 0:
        return
    rk4 = make_rk4()
    f_prev = drv.f_now
    h0 = h if n_full > 0 else h_last
    _, y_new, ev = run_stages(drv.rhs, drv.y, drv.t, h0, rk4, f_prev)
    drv.evals += ev
    drv.y = y_new
    drv.t = time_at(0)
    drv.after_accept(None, fsal_ok=False)
    drv.record(h0)
    drv.maybe_checkpoint()
    for i in range(1, total):
        h_i = h if i < n_full else h_last
        if h_i != h:
            _, y_new, ev = run_stages(drv.rhs, drv.y, drv.t, h_i, rk4, drv.f_now)
            drv.evals += ev
            drv.y = y_new
        else:
            drv.y = ab2_combine(drv.y, h, drv.f_now, f_prev)  # reference association (integrators.py:361-363)
        f_prev = drv.f_now
        drv.t = time_at(i)
        drv.after_accept(None, fsal_ok=False)
        drv.record(h_i)
        drv.maybe_checkpoint()


def _run_adaptive(drv, max_steps=None):
    """simulation.py:313-347 (+ accepted-step cap)."""
    cfg = drv.config
    pair = make_pair(cfg.integrator)
    t_end = cfg.t_end
    ctrl = ControllerState(h=drv.h_ctrl, prev_rejected=drv.prev_rejected, rejections=drv.rejections)
    a21 = float(pair.A[1, 0])
    drv.record(drv.h_ctrl)
    # launch-bound sizes: replay each first attempt from a CUDA graph (graphs.py);
    # unforced FSAL runs only (forcing refreshes f_now every step)
    graph = None
    field_bytes = drv.y.numel() * drv.y.element_size()
    if drv.graphs and pair.fsal and not cfg.forcing:
        from .graphs import GRAPH_MAX_FIELD_BYTES, attempt_graph

        # only where launches matter: a graph holds ~s + 4 state-sized buffers of
        # its own, and at 256^3+ one RHS is milliseconds of kernels
        if field_bytes <= GRAPH_MAX_FIELD_BYTES:
            graph = attempt_graph(drv.rhs, pair, cfg.controller, drv.grid)
    n = 0
    while drv.t < t_end and (max_steps is None or n < max_steps):
        remaining = t_end - drv.t
        clamped = ctrl.h >= remaining
        h_saved = ctrl.h
        if clamped:
            ctrl.h = remaining
        if graph is not None and drv.second_input is None:
            out = graph.advance(drv.y, drv.t, ctrl, drv.f_now)
        else:
            out = adaptive_advance(drv.y, drv.t, pair, ctrl, cfg.controller, drv.rhs, first_stage=drv.f_now,
                                   grid=drv.grid, second_input=drv.second_input)
        drv.evals += out.rhs_evals
        drv.rejections += out.rejections
        drv.y = out.y_new
        if clamped and out.rejections == 0:
            drv.t = t_end
            ctrl.h = h_saved
        else:
            drv.t = out.t_new
            if clamped and out.t_new >= t_end - 1e-12 * t_end:
                drv.t = t_end
        drv.h_ctrl = ctrl.h
        drv.prev_rejected = ctrl.prev_rejected
        drv.errs.append(out.errs)
        fsal_used = drv.after_accept(out.last_stage, fsal_ok=pair.fsal,
                                     energy_sum=out.diag_sums[4] if out.diag_sums is not None else None,
                                     next_coef=(ctrl.h, ctrl.h * a21))
        drv.record(out.h_used, sums=out.diag_sums if fsal_used else drv.refresh_sums)
        drv.maybe_checkpoint()
        n += 1
    if graph is not None:  # hand back buffers the graph will not overwrite
        drv.y = drv.y.clone()
        drv.f_now = drv.f_now.clone()


USE_GRAPHS = True  # default for run_simulation(graphs=None)


def _graph_max_bytes():
    from .graphs import GRAPH_MAX_FIELD_BYTES

    return GRAPH_MAX_FIELD_BYTES


def run_simulation(config, resume=None, initial_state=None, max_steps=None, graphs=None):
    """simulation.py:350-368 on the device.

    ``resume``: CheckpointData (read_checkpoint) continuing a run bit-exactly.
    ``initial_state``: optional FlowState / array / callable(config) replacing
    make_initial_state (IC hook).  ``max_steps``: accepted-step cap
    (SURVEY D6).  With ``config.output_dir`` the diagnostics CSV, periodic and
    final SRKL checkpoints are written like the reference.  ``graphs``: replay
    each adaptive step's first attempt from a CUDA graph (default USE_GRAPHS;
    bit-identical to the eager path, graphs.py).
    """
    config.validate()
    drv = _Driver(config, initial_state, resume)
    drv.graphs = USE_GRAPHS if graphs is None else bool(graphs)
    if config.mode == "fixed":
        _run_fixed(drv, max_steps)
    else:
        _run_adaptive(drv, max_steps)
    if drv.out_dir is not None:
        write_diagnostics_csv(drv.records, drv.out_dir / "diagnostics.csv")
        write_checkpoint(drv.out_dir / "final.srkl", drv.snapshot())
    return drv.result()
