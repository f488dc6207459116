"""Host-resident state: a pinned host copy of a device field kept in sync by chunked
asynchronous copies on two copy streams.

The reference keeps its state in host numpy arrays between steps
(`simulation.py:250-347`); a caller of the drop-in that does the same moves the
whole state over PCIe twice per step (3.2 GB each way at 512^3).  ``HostMirror``
makes that traffic overlap what it can:

* ``push`` (device -> host) runs on its own stream, ordered after the work
  already queued on the current stream, so it overlaps whatever is queued next.
  ``adaptive_advance(on_y_new=mirror.push)`` issues it the moment y_new exists,
  before the FSAL stage f(y_new) and the error reduction that decide whether the
  step is accepted (a rejected attempt pushes again; the last push wins).
* ``push(dev, planes=...)`` re-sends only some x-planes, e.g. the ones
  ``apply_forcing`` rescaled (``forcing_planes``).
* ``pull`` (host -> device) runs on a second stream, chunk by chunk, each chunk
  waiting only for the push that last wrote it -- device->host and host->device
  use both PCIe directions at once instead of one after the other
  (`tools/pcie_probe.py`: 3.23 GB push + pull 69 ms, either alone 58 ms).
  ``pull(wait=False)`` right after the speculative push starts the next step's
  input transfer under the FSAL stage too; ``pull(into=, planes=)`` then
  re-sends only the planes a later push changed.

Chunks are (component, x-plane range) blocks of the C-order ``(ncomp, n0, ...)``
state, ~``chunk_bytes`` each.  No arithmetic happens here: the copies are
``cudaMemcpyAsync`` through torch, the results are bitwise the device field.
"""

from __future__ import annotations

import numpy as np
import torch

from .grid import Grid


def plane_runs(planes):
    """Sorted x-plane indices -> list of contiguous half-open runs [(lo, hi), ...]."""
    p = sorted(set(int(i) for i in planes))
    runs = []
    for i in p:
        if runs and runs[-1][1] == i:
            runs[-1][1] = i + 1
        else:
            runs.append([i, i + 1])
    return [(a, b) for a, b in runs]


def forcing_planes(grid: Grid, k_f):
    """x-plane runs (first spectral axis) holding the forcing band 0 < |k|^2 <= k_f^2 (1+1e-12)
    that ``apply_forcing`` rescales (physics.py:209-239)."""
    band = (grid.k2 > 0.0) & (grid.k2 <= k_f * k_f * (1.0 + 1e-12))
    return plane_runs(np.flatnonzero(band.reshape(grid.kshape[0], -1).any(axis=1)))


class HostMirror:
    """Pinned host copy of a contiguous CUDA state tensor ``(ncomp, n0, ...)``."""

    def __init__(self, like: torch.Tensor, chunk_bytes: int = 128 << 20):
        if not (isinstance(like, torch.Tensor) and like.is_cuda and like.is_contiguous()):
            raise TypeError("HostMirror mirrors a contiguous CUDA tensor")
        self.shape, self.dtype, self.device = tuple(like.shape), like.dtype, like.device
        self.host = torch.empty(self.shape, dtype=self.dtype, pin_memory=True)
        ncomp, n0 = self.shape[0], self.shape[1]
        plane_bytes = like[0, 0].numel() * like.element_size()
        per = max(1, min(n0, chunk_bytes // max(1, plane_bytes)))
        self.chunks = [(c, lo, min(n0, lo + per)) for c in range(ncomp) for lo in range(0, n0, per)]
        self._d2h = torch.cuda.Stream(self.device)
        self._h2d = torch.cuda.Stream(self.device)
        # per chunk: disjoint x-plane segments [a, b) with the event and queue position
        # of the push that last wrote them (pull copies segments in that order)
        self._seg = [[(lo, hi, None, 0)] for (_, lo, hi) in self.chunks]
        self._n = 0
        self.d2h_bytes = 0
        self.h2d_bytes = 0

    def _check(self, dev):
        if tuple(dev.shape) != self.shape or dev.dtype != self.dtype or not dev.is_contiguous():
            raise ValueError(f"HostMirror holds {self.shape} {self.dtype}, got {tuple(dev.shape)} {dev.dtype}")

    def load_host(self, src):
        """Fill the host copy synchronously (numpy or CPU tensor); no push pending afterwards.
        The CPU write must not race queued copies on the mirror's own streams (a
        push still writing the host copy, a pull still reading it), so the host
        blocks on both before touching the pinned buffer."""
        self.wait()
        self._d2h.synchronize()
        self._h2d.synchronize()
        self.host.copy_(torch.as_tensor(src).reshape(self.shape))
        self._seg = [[(lo, hi, None, 0)] for (_, lo, hi) in self.chunks]

    def push(self, dev: torch.Tensor, planes=None):
        """Queue device -> host of ``dev`` (all of it, or the x-plane runs ``planes``) after the
        work already queued on the current stream; returns immediately."""
        self._check(dev)
        cur = torch.cuda.current_stream(self.device)
        self._d2h.wait_stream(cur)        # dev is complete
        self._d2h.wait_stream(self._h2d)  # a pull still reading the host copy finishes first
        dev.record_stream(self._d2h)
        with torch.cuda.stream(self._d2h):
            for i, (c, lo, hi) in enumerate(self.chunks):
                sel = [(lo, hi)] if planes is None else \
                    sorted((max(lo, a), min(hi, b)) for a, b in planes if max(lo, a) < min(hi, b))
                if not sel:
                    continue
                for a, b in sel:
                    self.host[c, a:b].copy_(dev[c, a:b], non_blocking=True)
                    self.d2h_bytes += self.host[c, a:b].numel() * self.host.element_size()
                ev = torch.cuda.Event()
                ev.record(self._d2h)
                self._n += 1
                keep = []
                for (sa, sb, sev, sq) in self._seg[i]:  # older segments minus the re-sent planes
                    cuts = [sa]
                    for a, b in sel:
                        cuts += [a, b]
                    cuts.append(sb)
                    for u, v in zip(cuts[::2], cuts[1::2]):
                        u, v = max(u, sa), min(v, sb)
                        if u < v:
                            keep.append((u, v, sev, sq))
                self._seg[i] = sorted(keep + [(a, b, ev, self._n) for a, b in sel])

    def pull(self, into=None, planes=None, wait=True) -> torch.Tensor:
        """Host -> device into a fresh tensor (or ``into``, optionally only its x-plane
        runs ``planes``); each segment starts once the push that last wrote it has
        landed.  Segments go in the order their pushes were queued (the h2d stream
        is in order: re-sent planes first in line would hold back all the others).
        ``wait``: the current stream waits for the copy before it can use the
        result; with ``wait=False`` the caller does that later (``wait_pull``), e.g.
        to pull the next step's input while the current stream still computes."""
        cur = torch.cuda.current_stream(self.device)
        with torch.cuda.stream(self._h2d):
            if into is None:
                dev = torch.empty(self.shape, dtype=self.dtype, device=self.device)
            else:
                self._check(into)
                self._h2d.wait_stream(cur)  # earlier work on ``into`` is done
                dev = into
            segs = [(sq, self.chunks[i][0], a, b, ev) for i in range(len(self.chunks))
                    for (a, b, ev, sq) in self._seg[i]]
            for sq, c, a, b, ev in sorted(segs, key=lambda x: (x[0], x[1], x[2])):
                if planes is not None:
                    sub = [(max(a, p), min(b, q)) for p, q in planes if max(a, p) < min(b, q)]
                else:
                    sub = [(a, b)]
                if not sub:
                    continue
                if ev is not None:
                    self._h2d.wait_event(ev)
                for u, v in sub:
                    dev[c, u:v].copy_(self.host[c, u:v], non_blocking=True)
                    self.h2d_bytes += dev[c, u:v].numel() * dev.element_size()
        dev.record_stream(cur)
        if wait:
            self.wait_pull()
        return dev

    def wait_pull(self):
        """Make the current stream wait for every queued pull."""
        torch.cuda.current_stream(self.device).wait_stream(self._h2d)

    def wait(self):
        """Make the current stream wait for every queued push (the host copy is then final
        once the current stream reaches this point)."""
        torch.cuda.current_stream(self.device).wait_stream(self._d2h)

    def synchronize(self):
        """Block the host until the host copy is final."""
        self._d2h.synchronize()
