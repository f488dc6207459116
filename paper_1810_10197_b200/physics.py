"""Device Navier-Stokes / Boussinesq tendencies (mirrors physics.py of the reference).

``FlowRHS(grid, params, density)`` is the drop-in operator: ``f(t, fields)``
evaluates physics.py:105-129 (ns_rhs) or :132-185 (boussinesq_rhs) with one
srk_rhs call (6 sm_100a kernels in 3D, 4 in 2D).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from .grid import Grid
from .spectral import from_device, get_plan, to_device

__all__ = ["ForcingError", "PhysParams", "FlowState", "FlowRHS", "ns_rhs", "boussinesq_rhs",
           "leray_project", "apply_forcing", "forcing_band"]


class ForcingError(RuntimeError):
    """The forcing band cannot reach the requested target energy (physics.py:23)."""


@dataclass
class PhysParams:
    reynolds: float
    richardson: float = 1.0
    prandtl: float = 1.0


@dataclass
class FlowState:
    grid: Grid
    fields: object

    @property
    def has_density(self):
        return self.fields.shape[0] == self.grid.dims + 1

    @property
    def velocity(self):
        return self.fields[: self.grid.dims]

    @property
    def density(self):
        if not self.has_density:
            raise ValueError("state carries no density component")
        return self.fields[self.grid.dims]


class FlowRHS:
    """Callable ``f(t, fields)`` (physics.py:188-206); returns a fresh caller-owned array."""

    def __init__(self, grid: Grid, params: PhysParams, density=False):
        self.grid = grid
        self.params = params
        self.density = bool(density)
        self.plan = get_plan(grid, density=self.density)
        self.ncomp = grid.dims + (1 if self.density else 0)
        self.calls = 0

    def __call__(self, t, fields, out=None):
        y, was_np = to_device(fields, torch.complex128)
        want = (self.ncomp,) + self.grid.kshape
        if tuple(y.shape) != want:
            raise ValueError(f"fields shape {tuple(y.shape)} != {want}")
        f = out if out is not None else torch.empty_like(y)
        p = self.params
        pl = self.plan
        with _native.nvtx("srk_rhs"):
            _native.check(pl.lib.srk_rhs(pl.bind(), _native.ptr(y), _native.ptr(f), 1.0 / p.reynolds,
                                         float(p.richardson), float(p.reynolds) * float(p.prandtl),
                                         _native.stream_ptr()), "srk_rhs")
        self.calls += 1
        _native.count(pl.lib.srk_rhs_launch_count(pl.h))
        return from_device(f, was_np)

    def eval_combine(self, t, fields, ybase, terms, coef_self):
        """``f(t, fields)`` plus the rk_step accumulation that consumes it
        (integrators.py:327-339): returns ``(f, ybase + sum c_j F_j + coef_self f)``,
        summed in ascending stage order with f last -- bitwise the unfused
        ``combine(ybase, terms + [(coef_self, f)])`` -- in one srk_rhs_combine call
        (the projection kernel forms the sum while f is in registers; 2D / 3D,
        with or without density)."""
        y, _ = to_device(fields, torch.complex128)
        yb, _ = to_device(ybase, torch.complex128)
        f = torch.empty_like(y)
        ynext = torch.empty_like(y)
        p = self.params
        pl = self.plan
        Fs = [F for _, F in terms]
        with _native.nvtx("srk_rhs_combine"):
            _native.check(pl.lib.srk_rhs_combine(pl.bind(), _native.ptr(y), _native.ptr(f), 1.0 / p.reynolds,
                                                 float(p.richardson), float(p.reynolds) * float(p.prandtl),
                                                 _native.ptr(yb), len(Fs), _native.ptr_array(Fs),
                                                 _native.dbl_array([c for c, _ in terms]), float(coef_self),
                                                 _native.ptr(ynext), _native.stream_ptr()), "srk_rhs_combine")
        self.calls += 1
        _native.count(pl.lib.srk_rhs_launch_count(pl.h))
        return f, ynext

    def refresh(self, t, fields, coef_self):
        """The after-accept refresh (simulation.py:165-182) fused with the next
        step's first stage sum: returns ``(f, y + coef_self f, sums)`` with ``f =
        self(t, y)`` and ``sums`` the 9 reduce_sums values of (y, f) for the
        diagnostics record (entries 4, 5, 8 = E, eps, Z sums; diag_from_sums).
        One projection pass (srk_rhs_refresh; E, eps, Z over the velocity
        components, density included in the stage sum)."""
        y, _ = to_device(fields, torch.complex128)
        f = torch.empty_like(y)
        ynext = torch.empty_like(y)
        p = self.params
        pl = self.plan
        out = _native.host_result(9)
        with _native.nvtx("srk_rhs_refresh"):
            _native.check(pl.lib.srk_rhs_refresh(pl.bind(), _native.ptr(y), _native.ptr(f), 1.0 / p.reynolds,
                                                 float(p.richardson), float(p.reynolds) * float(p.prandtl),
                                                 float(coef_self), _native.ptr(ynext), _native.ptr(out),
                                                 _native.stream_ptr()), "srk_rhs_refresh")
        self.calls += 1
        _native.count(pl.lib.srk_rhs_launch_count(pl.h))
        _native.wait_stream_point()
        return f, ynext, out.clone().tolist()

    def launches_per_call(self):
        return int(self.plan.lib.srk_rhs_launch_count(self.plan.h))


def ns_rhs(u_hat, grid: Grid, params: PhysParams, workspace=None):
    return FlowRHS(grid, params)(0.0, u_hat)


def boussinesq_rhs(fields, grid: Grid, params: PhysParams, workspace=None):
    return FlowRHS(grid, params, density=True)(0.0, fields)


def leray_project(u_hat, grid: Grid):
    """u - k (k.u)/|k|^2, k=0 untouched (physics.py:89-102)."""
    u, was_np = to_device(u_hat, torch.complex128)
    out = torch.empty_like(u)
    p = get_plan(grid)
    _native.check(p.lib.srk_leray_project(p.h, _native.ptr(u), _native.ptr(out), _native.stream_ptr()))
    return from_device(out, was_np)


_BANDS = {}


def forcing_band(grid: Grid, k_f, device):
    """Flat indices + Hermitian weights of the modes 0 < |k|^2 <= k_f^2 (1+1e-12)."""
    key = (grid.shape, grid.lengths, float(k_f), str(device))
    if key not in _BANDS:
        band = (grid.k2 > 0.0) & (grid.k2 <= k_f * k_f * (1.0 + 1e-12))
        idx = np.flatnonzero(band.ravel()).astype(np.int64)
        w = np.broadcast_to(grid.hermitian_weights, grid.kshape).ravel()[idx].astype(np.float64)
        _BANDS[key] = (torch.from_numpy(idx).to(device), torch.from_numpy(np.ascontiguousarray(w)).to(device),
                       len(idx))
    return _BANDS[key]


def forcing_band_slab(grid: Grid, k_f, device, rank, nranks):
    """Band modes of one y-slab (flat indices within the slab component)."""
    key = (grid.shape, grid.lengths, float(k_f), str(device), rank, nranks)
    if key not in _BANDS:
        ny = grid.shape[1] // nranks
        k2 = grid.k2[:, rank * ny:(rank + 1) * ny]
        band = (k2 > 0.0) & (k2 <= k_f * k_f * (1.0 + 1e-12))
        idx = np.flatnonzero(band.ravel()).astype(np.int64)
        w = np.broadcast_to(grid.hermitian_weights, k2.shape).ravel()[idx].astype(np.float64)
        _BANDS[key] = (torch.from_numpy(idx).to(device), torch.from_numpy(np.ascontiguousarray(w)).to(device),
                       len(idx))
    return _BANDS[key]


def apply_forcing(u_hat, grid: Grid, target_energy, k_f, plan=None, allreduce=None, slab=None,
                  energy_sum=None):
    """Rescale 0<|k|<=k_f in place to restore ``target_energy`` (physics.py:209-239).

    Slab runs pass the slab ``plan``, ``slab=(rank, nranks)`` and the rank-order
    ``allreduce``; E_total and E_band are then global sums.  ``energy_sum``: the
    (global) weighted sum sum_w |u|^2 of ``u_hat`` when the caller already has it
    -- e.g. ``AdvanceOutcome.diag_sums[4]`` of the step that produced u_hat, which
    the fused step reduction computes with the same arithmetic as the full pass
    this function would otherwise make -- so only the band is read."""
    from .diagnostics import reduce_sums

    u = u_hat
    if not (isinstance(u, torch.Tensor) and u.is_cuda and u.is_contiguous()):
        # host arrays (the reference rescales numpy arrays in place): force a device
        # copy and write the rescaled band back into the caller's array
        if slab is not None:
            raise TypeError("slab forcing works in place on the rank's CUDA slab")
        ud, _ = to_device(u_hat, torch.complex128)
        gamma = apply_forcing(ud, grid, target_energy, k_f, energy_sum=energy_sum)
        host = ud.cpu()
        if isinstance(u_hat, torch.Tensor):
            u_hat.copy_(host.to(u_hat.dtype))
        else:
            np.copyto(u_hat, host.numpy())
        return gamma
    if slab is None:
        idx, w, nb = forcing_band(grid, k_f, u.device)
        ph = get_plan(grid).h
    else:
        idx, w, nb = forcing_band_slab(grid, k_f, u.device, slab[0], slab[1])
        ph = plan
    lib = _native.load()
    ncomp = u.shape[0]
    pts2 = 2.0 * float(grid.points) ** 2
    q = reduce_sums(grid, u, flags=2, ncomp=ncomp, plan=plan, host=True) if energy_sum is None else None
    eb = _native.host_result(1)  # written by the kernel (pinned, mapped)
    eb.zero_()
    if nb > 0:
        _native.check(lib.srk_band_energy(ph, _native.ptr(u), ncomp, _native.ptr(idx), _native.ptr(w), nb,
                                          _native.ptr(eb), _native.stream_ptr()))
    _native.wait_stream_point()
    eb = eb.clone()  # the pinned buffer is reused by the next call
    if allreduce is not None:
        s = allreduce([q[4].item() if q is not None else 0.0, eb.item()])
        e_total = (s[0] if q is not None else float(energy_sum)) / pts2
        e_band = s[1] / pts2
    else:
        e_total = (q[4].item() if q is not None else float(energy_sum)) / pts2
        e_band = eb.item() / pts2
    e_rest = e_total - e_band
    if e_band <= 0.0:
        raise ForcingError("forcing band carries no energy")
    radicand = (target_energy - e_rest) / e_band
    if radicand < 0.0:
        raise ForcingError(f"energy outside the band ({e_rest:.6e}) exceeds target ({target_energy:.6e})")
    gamma = float(np.sqrt(radicand))
    if nb > 0:
        _native.check(lib.srk_band_scale(ph, _native.ptr(u), ncomp, _native.ptr(idx), nb, gamma,
                                         _native.stream_ptr()))
    _native.count(2)
    return gamma
