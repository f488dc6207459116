"""Work-precision sweep on the device (mirrors bench.py:26-128 of the reference).

Every cell (integrator, step size or tolerance) runs through run_simulation on
the GPU and is scored against a fixed-step RK4 reference run: max |eps(t) -
spline(eps_ref)(t)| over the cell's accepted times and the relative L2 error of
the final velocity field.  Evaluation counts include rejected attempts.  With
torch.distributed initialised the cells are dealt round-robin to the ranks
(independent replicas, one GPU each) and gathered on every rank.
"""

from __future__ import annotations

import copy
import warnings
from dataclasses import dataclass

import numpy as np

from .diagnostics import compare_series, field_error_norms
from .simulation import ConfigError, run_simulation
from .spectral import inverse_transform

__all__ = ["WorkPrecisionPoint", "cell_config", "work_precision", "write_work_precision_csv"]


@dataclass
class WorkPrecisionPoint:
    integrator: str
    mode: str
    setting: float
    rhs_evals: int
    error: float
    kind: str
    status: str = "ok"


def _eps_series(records):
    return np.array([r.t for r in records]), np.array([r.eps for r in records])


def cell_config(base, integrator, mode, setting):
    """bench.py:45-56."""
    cfg = copy.deepcopy(base)
    cfg.integrator = integrator
    cfg.mode = mode
    if mode == "fixed":
        cfg.h = setting
    else:
        cfg.tol_abs = cfg.tol_rel = setting
    cfg.output_dir = None
    cfg.checkpoint_interval = None
    return cfg.validate()


def work_precision(cells, reference, keep_states=False, initial_state=None):
    """bench.py:59-116 (+ optional IC hook and rank-parallel cells)."""
    if reference.integrator != "rk4" or reference.mode != "fixed":
        raise ConfigError("work-precision reference must be fixed-step rk4")
    fixed_h = [c.h for c in cells if c.mode == "fixed"]
    if fixed_h and reference.h > min(fixed_h) / 10.0 + 1e-15:
        raise ConfigError(f"reference h = {reference.h:g} exceeds a tenth of the smallest compared fixed "
                          f"step {min(fixed_h):g}")
    ref = run_simulation(reference, initial_state=initial_state)
    t_ref, eps_ref = _eps_series(ref.records)
    dims = ref.state.grid.dims
    u_ref = inverse_transform(ref.state.fields[:dims], ref.state.grid)

    rank, world = 0, 1
    try:
        import torch.distributed as dist

        if dist.is_available() and dist.is_initialized():
            rank, world = dist.get_rank(), dist.get_world_size()
    except Exception:
        pass

    points = []
    for i, cfg in enumerate(cells):
        if i % world != rank:
            continue
        setting = cfg.h if cfg.mode == "fixed" else cfg.tol_abs
        try:
            res = run_simulation(cfg, initial_state=initial_state)
            err_s = compare_series(_eps_series(res.records), (t_ref, eps_ref))
            u = inverse_transform(res.state.fields[:dims], res.state.grid)
            err_l2, _ = field_error_norms(u, u_ref, res.state.grid)
            for kind, err in (("eps_series", err_s), ("l2_final", err_l2)):
                points.append(WorkPrecisionPoint(cfg.integrator, cfg.mode, setting, res.rhs_evals, err, kind))
        except Exception as exc:  # cell failures are data, not aborts
            warnings.warn(f"cell {cfg.integrator}/{setting:g} failed: {exc}")
            for kind in ("eps_series", "l2_final"):
                points.append(WorkPrecisionPoint(cfg.integrator, cfg.mode, setting, 0, float("nan"), kind,
                                                 status=f"failed: {exc}"))
    if world > 1:
        import torch.distributed as dist

        gathered = [None] * world
        dist.all_gather_object(gathered, points)
        points = [p for part in gathered for p in part]
    points.sort(key=lambda p: (p.integrator, p.setting, p.kind))
    return (points, ref) if keep_states else (points, None)


def write_work_precision_csv(points, path):
    """bench.py:119-128."""
    with open(path, "w") as fh:
        fh.write("# rhs_evals include all evaluations spent on rejected steps\n")
        fh.write("integrator,mode,setting,rhs_evals,error,kind,status\n")
        for p in points:
            fh.write(f"{p.integrator},{p.mode},{p.setting:.16e},{p.rhs_evals},{p.error:.16e},{p.kind},{p.status}\n")
