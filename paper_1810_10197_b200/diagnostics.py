"""Per-step diagnostics on the device (mirrors diagnostics.py:27-70 of the reference).

E_kin, eps and the enstrophy come from one deterministic fused
reduction kernel (csrc/pointwise.cu k_reduce, flags=2).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from .grid import Grid
from .spectral import get_plan, to_device

__all__ = ["DiagnosticsRecord", "SpectrumRecord", "kinetic_energy", "dissipation_rate", "enstrophy",
           "reduce_sums", "diag_from_sums", "energy_spectrum", "field_error_norms", "compare_series"]


@dataclass
class DiagnosticsRecord:
    """One per-step row (diagnostics.py:27-36) plus the enstrophy (D2)."""

    t: float
    h: float
    e_kin: float
    eps: float
    rhs_evals: int
    rejections: int
    enstrophy: float = float("nan")


def reduce_sums(grid: Grid, y1, fl=None, y0=None, terms=(), tol_abs=0.0, tol_rel=0.0, flags=2, ncomp=None,
                stream=None, plan=None, host=False):
    """Launch srk_step_reduce; returns the 9 device sums as a CUDA float64 tensor (no sync).

    ``plan``: a slab plan handle (paper_1810_10197_b200.slab) when y1 is a y-slab;
    the sums are then this rank's partials.  ``host=True``: the finishing kernel
    stores the sums straight into pinned host memory (no copy-engine transfer that
    could queue behind a large HostMirror copy); the call then waits for the
    stream and returns a CPU tensor."""
    lib = _native.load()
    h = get_plan(grid).h if plan is None else plan
    ncomp = y1.shape[0] if ncomp is None else ncomp
    out = _native.host_result(9) if host else torch.empty(9, dtype=torch.float64, device=y1.device)
    Fs = [t for _, t in terms]
    cs = [c for c, _ in terms]
    _native.check(lib.srk_step_reduce(
        h, _native.ptr(y0), _native.ptr(y1), len(Fs), _native.ptr_array(Fs), _native.dbl_array(cs),
        _native.ptr(fl if fl is not None else y1), ncomp, float(tol_abs), float(tol_rel), int(flags),
        _native.ptr(out), _native.stream_ptr(stream)), "srk_step_reduce")
    _native.count(2)
    if host:
        _native.wait_stream_point(stream)
        return out.clone()  # the pinned buffer is reused by the next call
    return out


def diag_from_sums(q, grid: Grid):
    """(E_kin, eps, Z) from reduce sums (diagnostics.py:48-70)."""
    pts2 = float(grid.points) ** 2
    return q[4] / (2.0 * pts2), -q[5] / pts2, q[8] / (2.0 * pts2)


def kinetic_energy(u_hat, grid: Grid):
    """E = sum_k w_k sum_j |u_kj|^2 / (2 points^2) (diagnostics.py:48-50)."""
    u, _ = to_device(u_hat, torch.complex128)
    q = reduce_sums(grid, u, flags=2, ncomp=u.shape[0], host=True).tolist()
    return q[4] / (2.0 * float(grid.points) ** 2)


def dissipation_rate(u_hat, f_hat, grid: Grid):
    """eps = -sum_k w_k sum_{j<d} Re(u conj f) / points^2 (diagnostics.py:53-70)."""
    u, _ = to_device(u_hat, torch.complex128)
    f, _ = to_device(f_hat, torch.complex128)
    if tuple(u.shape[1:]) != grid.kshape or tuple(f.shape) != tuple(u.shape):
        raise ValueError(f"shape mismatch: fields {tuple(u.shape)}, tendency {tuple(f.shape)}, "
                         f"grid modes {grid.kshape}")
    q = reduce_sums(grid, u, fl=f, flags=2, ncomp=min(u.shape[0], grid.dims), host=True).tolist()
    return -q[5] / float(grid.points) ** 2


def enstrophy(u_hat, grid: Grid):
    """Z = sum_k w_k |k|^2 sum_{j<d} |u_kj|^2 / (2 points^2)."""
    u, _ = to_device(u_hat, torch.complex128)
    q = reduce_sums(grid, u, flags=2, ncomp=min(u.shape[0], grid.dims), host=True).tolist()
    return q[8] / (2.0 * float(grid.points) ** 2)


@dataclass
class SpectrumRecord:
    """Shell-binned spectrum E(m), unit-width shells centred on integer |k| (diagnostics.py:20-24)."""

    k: object
    E: object


_SHELLS = {}


def _shell_index(grid: Grid, device):
    key = (grid.shape, grid.lengths, str(device))
    if key not in _SHELLS:
        kk = [torch.as_tensor(np.ascontiguousarray(k), dtype=torch.float64, device=device) for k in grid.k]
        k2 = torch.zeros(grid.kshape, dtype=torch.float64, device=device)
        for ka in kk:
            k2 = k2 + ka * ka
        bins = torch.floor(torch.sqrt(k2) + 0.5).to(torch.int64).reshape(-1)
        w = torch.full((grid.kshape[-1],), 2.0, dtype=torch.float64, device=device)
        w[0] = w[-1] = 1.0
        wf = torch.broadcast_to(w, grid.kshape).reshape(-1).contiguous()
        _SHELLS[key] = (bins, wf, int(bins.max().item()) + 1)
    return _SHELLS[key]


def energy_spectrum(u_hat, grid: Grid):
    """Shell energy spectrum on the device (diagnostics.py:73-91); shells sum to E_kin.

    Post-processing, not on the per-stage path: torch device reductions."""
    u, was_np = to_device(u_hat, torch.complex128)
    bins, w, nshell = _shell_index(grid, u.device)
    e = torch.zeros(nshell, dtype=torch.float64, device=u.device)
    for j in range(u.shape[0]):
        a = u[j].reshape(-1)
        e += torch.bincount(bins, weights=w * (a.real ** 2 + a.imag ** 2), minlength=nshell)
    e /= 2.0 * float(grid.points) ** 2
    k = np.arange(nshell, dtype=float)
    return SpectrumRecord(k=k, E=e.cpu().numpy())


def field_error_norms(u, u_ref, grid: Grid):
    """Relative L2 and max norms of a physical-space difference (diagnostics.py:94-103)."""
    a, _ = to_device(u, torch.float64)
    b, _ = to_device(u_ref, torch.float64)
    if tuple(a.shape) != tuple(b.shape):
        raise ValueError(f"shape mismatch: {tuple(a.shape)} vs {tuple(b.shape)}")
    if tuple(a.shape[-grid.dims:]) != grid.shape:
        raise ValueError(f"fields {tuple(a.shape)} do not live on grid {grid.shape}")
    diff = a - b
    l2 = float(torch.sqrt(torch.sum(diff ** 2) / torch.sum(b ** 2)))
    mx = float(torch.max(torch.abs(diff)) / torch.max(torch.abs(b)))
    return l2, mx


def compare_series(series, ref_series):
    """Max |series - quadratic-spline(ref)| at the series times (diagnostics.py:106-123); host."""
    from scipy.interpolate import make_interp_spline

    t, v = (np.asarray(x, dtype=float) for x in series)
    tr, vr = (np.asarray(x, dtype=float) for x in ref_series)
    if tr.size < 3:
        raise ValueError("reference series needs at least 3 points")
    if t.min() < tr[0] or t.max() > tr[-1]:
        raise ValueError(f"series times [{t.min():g}, {t.max():g}] extend beyond the reference range "
                         f"[{tr[0]:g}, {tr[-1]:g}]")
    return float(np.max(np.abs(v - make_interp_spline(tr, vr, k=2)(t))))
