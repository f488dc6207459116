"""Device transforms, curl and 3/2-rule dealiasing (mirrors spectral.py of the reference).

All compute goes through libsrk (sm_100a kernels).  Inputs may be torch CUDA
tensors (returned as tensors) or numpy arrays (copied to the current device
and returned as numpy, so reference call sites work unchanged).
"""

from __future__ import annotations

import ctypes
import itertools

import numpy as np
import torch

from . import _native
from .grid import Grid

__all__ = [
    "Plan", "get_plan", "forward_transform", "inverse_transform", "curl",
    "zero_nyquist", "zero_self_conjugate_imag", "symmetrize_real_planes",
    "pad_spectrum", "truncate_spectrum", "DealiasWorkspace", "dealiased_product",
    "to_device", "from_device",
]


def require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1810_10197_b200 needs a CUDA device (B200, sm_100a); there is no CPU path")


def to_device(x, dtype):
    """numpy/torch -> contiguous CUDA tensor of ``dtype``; returns (tensor, was_numpy)."""
    require_cuda()
    if isinstance(x, torch.Tensor):
        t = x
        if not t.is_cuda:
            t = t.to("cuda")
        if t.dtype != dtype:
            t = t.to(dtype)
        return t.contiguous(), False
    arr = np.ascontiguousarray(np.asarray(x))
    return torch.from_numpy(arr).to(device="cuda", dtype=dtype), True


def from_device(t, as_numpy):
    return t.cpu().numpy() if as_numpy else t


# ---------------------------------------------------------------------------
# plans + shared workspace arena
# ---------------------------------------------------------------------------
_ARENA = {}


def _arena(dev, nbytes):
    t = _ARENA.get(dev)
    if t is None or t.numel() < nbytes:
        _ARENA[dev] = None
        t = torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=dev)
        _ARENA[dev] = t
    return t


class Plan:
    """Owns an ``srk_plan`` (include/srk.h); binds the per-device workspace arena.

    Plans on one device share one workspace arena, so like the reference's
    FlowRHS / DealiasWorkspace they are not re-entrant across concurrent
    streams (physics.py:195-201).
    """

    def __init__(self, grid: Grid, density=False, max_comps=0, device=None):
        require_cuda()
        self.lib = _native.load()
        self.grid = grid
        self.density = bool(density)
        self.max_comps = int(max_comps)
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        shape = (ctypes.c_int64 * 3)(*grid.shape, *([0] * (3 - grid.dims)))
        lengths = (ctypes.c_double * 3)(*grid.lengths, *([0.0] * (3 - grid.dims)))
        h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _native.check(self.lib.srk_plan_create(ctypes.byref(h), grid.dims, shape, lengths,
                                                   int(self.density), self.max_comps), "srk_plan_create")
        self.h = h
        nb = ctypes.c_int64()
        _native.check(self.lib.srk_plan_workspace_bytes(h, ctypes.byref(nb)))
        self.need = nb.value
        self._bound = None

    def bind(self):
        t = _arena(self.device, self.need)
        if self._bound is not t:
            _native.check(self.lib.srk_plan_set_workspace(self.h, ctypes.c_void_p(t.data_ptr()), t.numel()))
            self._bound = t
        return self.h

    def __del__(self):
        try:
            if getattr(self, "h", None) is not None and self.h.value:
                self.lib.srk_plan_destroy(self.h)
        except Exception:
            pass


_PLANS = {}


def get_plan(grid: Grid, density=False, max_comps=0):
    require_cuda()
    dev = torch.cuda.current_device()
    key = (grid.shape, grid.lengths, bool(density), dev)
    p = _PLANS.get(key)
    if p is None or p.max_comps < max_comps:
        p = Plan(grid, density, max(max_comps, p.max_comps if p else 0), dev)
        _PLANS[key] = p
    return p


def _stream():
    return _native.stream_ptr()


def _stack(x, lead_rank_ok, trailing):
    """Reshape (..., *trailing) -> (c, *trailing)."""
    if tuple(x.shape[x.dim() - len(trailing):]) != tuple(trailing):
        raise ValueError(f"array shape {tuple(x.shape)} does not end in {tuple(trailing)}")
    lead = tuple(x.shape[: x.dim() - len(trailing)])
    c = int(np.prod(lead)) if lead else 1
    return x.reshape((c,) + tuple(trailing)), lead


# ---------------------------------------------------------------------------
# transforms (spectral.py:17-65)
# ---------------------------------------------------------------------------
def forward_transform(field, grid: Grid):
    """Unnormalised rfftn over the grid axes (spectral.py:17-30)."""
    x, was_np = to_device(field, torch.float64)
    if tuple(x.shape[-grid.dims:]) != grid.shape:
        raise ValueError(f"field shape {tuple(x.shape)} does not end in grid shape {grid.shape}")
    xs, lead = _stack(x, True, grid.shape)
    c = xs.shape[0]
    p = get_plan(grid, max_comps=c)
    out = torch.empty((c,) + grid.kshape, dtype=torch.complex128, device=x.device)
    _native.check(p.lib.srk_forward_transform(p.bind(), _native.ptr(xs), c, _native.ptr(out), _stream()))
    return from_device(out.reshape(lead + grid.kshape), was_np)


def inverse_transform(spec, grid: Grid):
    """irfftn with 1/points normalisation (spectral.py:33-44)."""
    s, was_np = to_device(spec, torch.complex128)
    if tuple(s.shape[-grid.dims:]) != grid.kshape:
        raise ValueError(f"spectrum shape {tuple(s.shape)} does not end in {grid.kshape}")
    ss, lead = _stack(s, True, grid.kshape)
    c = ss.shape[0]
    p = get_plan(grid, max_comps=c)
    out = torch.empty((c,) + grid.shape, dtype=torch.float64, device=s.device)
    _native.check(p.lib.srk_inverse_transform(p.bind(), _native.ptr(ss), c, _native.ptr(out), _stream()))
    return from_device(out.reshape(lead + grid.shape), was_np)


def curl(u_hat, grid: Grid, out=None):
    """Spectral curl i k x u (spectral.py:47-65); 2D returns the scalar vorticity."""
    u, was_np = to_device(u_hat, torch.complex128)
    p = get_plan(grid)
    nw = 3 if grid.dims == 3 else 1
    w = torch.empty((nw,) + grid.kshape, dtype=torch.complex128, device=u.device)
    _native.check(p.lib.srk_curl(p.h, _native.ptr(u), _native.ptr(w), _stream()))
    if grid.dims == 2:
        w = w[0]
    res = from_device(w, was_np)
    if out is not None:
        out[...] = res
        return out
    return res


# ---------------------------------------------------------------------------
# Hermitian bookkeeping helpers (spectral.py:73-171) -- host logic on tensors
# ---------------------------------------------------------------------------
def _lib_of(x):
    return torch if isinstance(x, torch.Tensor) else np


def zero_nyquist(spec, grid: Grid):
    lead = spec.ndim - grid.dims
    for ax, n in enumerate(grid.shape):
        sl = [slice(None)] * spec.ndim
        sl[lead + ax] = n // 2
        spec[tuple(sl)] = 0.0
    return spec


def zero_self_conjugate_imag(spec, grid: Grid):
    lead = (slice(None),) * (spec.ndim - grid.dims)
    for corner in itertools.product(*[(0, n // 2) for n in grid.shape]):
        idx = lead + corner
        spec[idx] = spec[idx].real
    return spec


def symmetrize_real_planes(spec, grid: Grid):
    xp = _lib_of(spec)
    lead = spec.ndim - grid.dims
    for kz in (0, grid.shape[-1] // 2):
        sl = [slice(None)] * spec.ndim
        sl[-1] = kz
        plane = spec[tuple(sl)]
        refl = plane
        for ax in range(lead, lead + grid.dims - 1):
            if xp is torch:
                refl = torch.roll(torch.flip(refl, dims=(ax,)), 1, dims=ax)
            else:
                refl = np.roll(np.flip(refl, axis=ax), 1, axis=ax)
        spec[tuple(sl)] = 0.5 * (plane + refl.conj())
    return spec


def _copy_blocks(src, dst, grid: Grid, widen: bool):
    lead = (slice(None),) * (dst.ndim - grid.dims)
    per_axis = []
    for n in grid.shape[:-1]:
        m = 3 * n // 2
        per_axis.append([(slice(0, n // 2 + 1), slice(0, n // 2 + 1)),
                         (slice(n // 2 + 1, n), slice(m - (n // 2 - 1), m))])
    nz = grid.shape[-1] // 2 + 1
    per_axis.append([(slice(0, nz), slice(0, nz))])
    for pick in itertools.product(*per_axis):
        coarse = lead + tuple(c for c, _ in pick)
        padded = lead + tuple(p for _, p in pick)
        if widen:
            dst[padded] = src[coarse]
        else:
            dst[coarse] = src[padded]


def pad_spectrum(spec, grid: Grid, out=None):
    xp = _lib_of(spec)
    shape = tuple(spec.shape[: spec.ndim - grid.dims]) + grid.padded_kshape
    if out is None:
        out = (torch.zeros(shape, dtype=torch.complex128, device=spec.device) if xp is torch
               else np.zeros(shape, dtype=np.complex128))
    else:
        out[...] = 0.0
    _copy_blocks(spec, out, grid, widen=True)
    return out


def truncate_spectrum(padded, grid: Grid, out=None):
    xp = _lib_of(padded)
    shape = tuple(padded.shape[: padded.ndim - grid.dims]) + grid.kshape
    if out is None:
        out = (torch.empty(shape, dtype=torch.complex128, device=padded.device) if xp is torch
               else np.empty(shape, dtype=np.complex128))
    _copy_blocks(padded, out, grid, widen=False)
    zero_nyquist(out, grid)
    zero_self_conjugate_imag(out, grid)
    return out


# ---------------------------------------------------------------------------
# dealiasing (spectral.py:174-337)
# ---------------------------------------------------------------------------
class DealiasWorkspace:
    """Factored 3/2-rule padded transforms on the device (spectral.py:174-304).

    ``widen`` returns a fresh float64 tensor (c, *padded_shape); ``narrow``
    returns the truncated spectrum (fresh unless ``out`` is given).
    """

    def __init__(self, grid: Grid, ncomp: int):
        self.grid = grid
        self.ncomp = int(ncomp)
        self.plan = get_plan(grid, max_comps=self.ncomp)

    def _pieces(self, specs):
        if isinstance(specs, (np.ndarray, torch.Tensor)):
            specs = [specs]
        out, any_np = [], False
        for p in specs:
            t, was_np = to_device(p, torch.complex128)
            any_np |= was_np
            out.append(t if t.dim() == self.grid.dims + 1 else t[None])
        return out, any_np

    def widen(self, specs):
        pieces, was_np = self._pieces(specs)
        spec = pieces[0] if len(pieces) == 1 else torch.cat(pieces, dim=0)
        spec = spec.contiguous()
        c = spec.shape[0]
        if c > self.ncomp:
            raise ValueError(f"{c} components exceed workspace size {self.ncomp}")
        out = torch.empty((c,) + self.grid.padded_shape, dtype=torch.float64, device=spec.device)
        p = self.plan
        _native.check(p.lib.srk_widen(p.bind(), _native.ptr(spec), c, _native.ptr(out), _stream()))
        return from_device(out, was_np)

    def narrow(self, fields, out=None):
        x, was_np = to_device(fields, torch.float64)
        c = x.shape[0]
        if c > self.ncomp:
            raise ValueError(f"{c} components exceed workspace size {self.ncomp}")
        res = torch.empty((c,) + self.grid.kshape, dtype=torch.complex128, device=x.device)
        p = self.plan
        _native.check(p.lib.srk_narrow(p.bind(), _native.ptr(x), c, _native.ptr(res), _stream()))
        res = from_device(res, was_np)
        if out is not None:
            out[...] = res
            return out
        return res


def dealiased_product(kernel, specs, grid: Grid, workspace=None, out=None):
    """narrow(kernel(widen(specs))) with the kernel applied to device tensors (spectral.py:307-337)."""
    if workspace is None:
        pieces = specs if not isinstance(specs, (np.ndarray, torch.Tensor)) else [specs]
        c = sum(1 if p.ndim == grid.dims else p.shape[0] for p in pieces)
        workspace = DealiasWorkspace(grid, c)
    was_np = any(isinstance(p, np.ndarray) for p in
                 (specs if not isinstance(specs, (np.ndarray, torch.Tensor)) else [specs]))
    fields = workspace.widen(specs)
    if was_np:
        fields = torch.from_numpy(fields).cuda()
    product = kernel(fields)
    res = workspace.narrow(product, out=None)
    res = from_device(res, was_np)
    if out is not None:
        out[...] = res
        return out
    return res
