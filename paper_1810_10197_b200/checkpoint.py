"""SRKL v1 checkpoints and the diagnostics CSV (mirrors simulation.py:371-516).

Byte-compatible with the reference format, so a run checkpointed on the GPU
resumes in the reference CPU code and vice versa
(tests/test_checkpoint.py pins this against a file written by the reference).
Device tensors are copied to the host for writing; restart is bit-exact
because every device kernel is deterministic.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np

from .diagnostics import DiagnosticsRecord
from .grid import Grid

__all__ = ["CheckpointError", "CheckpointData", "write_checkpoint", "read_checkpoint",
           "write_diagnostics_csv", "read_diagnostics_csv"]

MAGIC = b"SRKL"
VERSION = 1
_HDR_STATE = "<Bdd B QQQ"   # has_density, time, h, prev_rejected, rhs_evals, rejections, steps
_HDR_FORCE = "<Bdd"         # forcing, k_f, target energy
_HDR_RNG = "<BQQQQ"         # flag + PCG64 (state lo, hi, inc lo, hi)
_CSV_HEADER = "t,h,E_kin,eps,rhs_evals_cum,rejections_cum"


class CheckpointError(RuntimeError):
    """Unreadable, corrupt or incompatible checkpoint (simulation.py:28)."""


@dataclass
class CheckpointData:
    grid: Grid
    fields: object
    has_density: bool
    time: float
    h: float
    prev_rejected: bool
    rhs_evals: int
    rejections: int
    steps: int
    f_now: object
    rng_state: tuple | None
    forcing: bool
    k_f: float
    forcing_energy: float


def _host(a):
    if a is None:
        return None
    if hasattr(a, "detach"):
        a = a.detach().cpu().numpy()
    return np.ascontiguousarray(a, dtype=np.complex128)


def write_checkpoint(path, data: CheckpointData):
    g = data.grid
    out = bytearray(MAGIC)
    out += struct.pack("<II", VERSION, g.dims)
    out += struct.pack(f"<{g.dims}I", *g.shape)
    out += struct.pack(f"<{g.dims}d", *g.lengths)
    out += struct.pack(_HDR_STATE, bool(data.has_density), float(data.time), float(data.h),
                       bool(data.prev_rejected), int(data.rhs_evals), int(data.rejections), int(data.steps))
    out += struct.pack(_HDR_FORCE, bool(data.forcing), float(data.k_f), float(data.forcing_energy))
    if data.rng_state is not None:
        st, inc = data.rng_state
        m = (1 << 64) - 1
        out += struct.pack(_HDR_RNG, 1, st & m, st >> 64, inc & m, inc >> 64)
    else:
        out += struct.pack(_HDR_RNG, 0, 0, 0, 0, 0)
    f_now = _host(data.f_now)
    out += struct.pack("<B", f_now is not None)
    out += _host(data.fields).astype("<c16", copy=False).tobytes()
    if f_now is not None:
        out += f_now.astype("<c16", copy=False).tobytes()
    with open(path, "wb") as fh:
        fh.write(out)


def read_checkpoint(path) -> CheckpointData:
    with open(path, "rb") as fh:
        raw = fh.read()
    if len(raw) < 12 or raw[:4] != MAGIC:
        raise CheckpointError(f"{path}: not a checkpoint file (bad magic)")
    version, dims = struct.unpack_from("<II", raw, 4)
    off = 12
    if version != VERSION:
        raise CheckpointError(f"{path}: unsupported version {version}")
    if dims not in (2, 3):
        raise CheckpointError(f"{path}: invalid dimension count {dims}")
    shape = struct.unpack_from(f"<{dims}I", raw, off)
    off += 4 * dims
    lengths = struct.unpack_from(f"<{dims}d", raw, off)
    off += 8 * dims
    has_d, time, h, prev, evals, rej, steps = struct.unpack_from(_HDR_STATE, raw, off)
    off += struct.calcsize(_HDR_STATE)
    forcing, k_f, energy = struct.unpack_from(_HDR_FORCE, raw, off)
    off += struct.calcsize(_HDR_FORCE)
    has_rng, s_lo, s_hi, i_lo, i_hi = struct.unpack_from(_HDR_RNG, raw, off)
    off += struct.calcsize(_HDR_RNG)
    (has_f,) = struct.unpack_from("<B", raw, off)
    off += 1
    grid = Grid(shape, lengths)
    ncomp = grid.dims + (1 if has_d else 0)
    count = ncomp * grid.mode_count
    nbytes = 16 * count
    if len(raw) - off != nbytes * (2 if has_f else 1):
        raise CheckpointError(f"{path}: truncated payload ({len(raw) - off} bytes, "
                              f"expected {nbytes * (2 if has_f else 1)})")

    def take(o):
        return np.frombuffer(raw, dtype="<c16", count=count, offset=o).astype(np.complex128).reshape(
            (ncomp,) + grid.kshape)

    fields = take(off)
    f_now = take(off + nbytes) if has_f else None
    rng = ((s_hi << 64) | s_lo, (i_hi << 64) | i_lo) if has_rng else None
    return CheckpointData(grid=grid, fields=fields, has_density=bool(has_d), time=time, h=h,
                          prev_rejected=bool(prev), rhs_evals=evals, rejections=rej, steps=steps, f_now=f_now,
                          rng_state=rng, forcing=bool(forcing), k_f=k_f, forcing_energy=energy)


def write_diagnostics_csv(records, path):
    """17 significant digits (simulation.py:371-379)."""
    with open(path, "w") as fh:
        fh.write(_CSV_HEADER + "\n")
        for r in records:
            fh.write(f"{r.t:.16e},{r.h:.16e},{r.e_kin:.16e},{r.eps:.16e},{r.rhs_evals},{r.rejections}\n")


def read_diagnostics_csv(path):
    out = []
    with open(path) as fh:
        head = fh.readline().strip()
        if head != _CSV_HEADER:
            raise ValueError(f"unexpected CSV header {head!r}")
        for line in fh:
            t, h, e, eps, ev, rej = line.strip().split(",")
            out.append(DiagnosticsRecord(t=float(t), h=float(h), e_kin=float(e), eps=float(eps),
                                         rhs_evals=int(ev), rejections=int(rej)))
    return out
