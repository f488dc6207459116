"""CUDA-graph replay of one adaptive attempt.

At 32^3 (config 1) and 2D 1024^2 (config 4) one RHS is a few tens of
microseconds of kernels, so the stepping loop of the reference
(simulation.py:313-347 -> control.py:132-169 -> integrators.py:295-358) is bound
by kernel launches and host work, not by the GPU.  ``AttemptGraph`` captures one
whole attempt of an FSAL pair whose first stage is known -- the s - 1 RHS
evaluations with their fused stage sums, the embedded-error / diagnostics
reduction and its store into pinned host memory -- as one CUDA graph, and
replays it with the step size read from device memory (the *_scaled entry
points of include/srk.h: coefficients are tableau values baked into the graph,
multiplied by h on the device -- bitwise the host products h * a_ij of the
eager path, so the graphed run is bit-identical to the ungraphed one).

State buffers are static and ping-pong between two graphs: graph p reads the
state Y[p] and the FSAL stage FL[p] and writes y_new to Y[1-p] and the new FSAL
stage to FL[1-p], so an accepted step feeds the next replay without a copy.  A
rejected attempt (rare) continues on the eager path (control.adaptive_advance,
which recomputes F1 like the reference).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native
from .control import AdvanceOutcome, adaptive_advance, propose_step
from .integrators import _FUSED_MAX_TERMS

__all__ = ["AttemptGraph", "attempt_graph", "GRAPH_MAX_FIELD_BYTES"]

# captured graphs outlive one run_simulation call (a capture costs about two
# attempts): keyed by everything a graph bakes in -- plan, physics, tableau,
# tolerances, device; small states only (a graph holds ~s + 4 state-sized buffers)
_CACHE = {}
_CACHE_MAX = 4
GRAPH_MAX_FIELD_BYTES = 256 << 20  # run_simulation graphs states up to this size (128^3: 51 MB, 2D 1024^2: 25 MB)


def attempt_graph(rhs, pair, config, grid, fixed=False):
    """The cached AttemptGraph for this (plan, physics, pair, tolerances, mode, device)."""
    p = rhs.params
    tol = (0.0, 0.0) if fixed else (float(config.tol_abs), float(config.tol_rel))
    key = (rhs.plan.h.value if hasattr(rhs.plan.h, "value") else int(rhs.plan.h), tuple(grid.shape),
           tuple(grid.lengths), rhs.density, float(p.reynolds), float(p.richardson), float(p.prandtl), pair.name,
           tol, bool(fixed), torch.cuda.current_device())
    g = _CACHE.pop(key, None)
    if g is None:
        g = AttemptGraph(rhs, pair, config, grid, fixed=fixed)
    elif g.rhs is not rhs:
        g.rhs = rhs  # same plan and physics: the recorded launches are identical
    field_bytes = g.Y[0].numel() * g.Y[0].element_size()
    if field_bytes <= GRAPH_MAX_FIELD_BYTES:
        _CACHE[key] = g
        while len(_CACHE) > _CACHE_MAX:
            _CACHE.pop(next(iter(_CACHE)))
    g.cfg = config
    return g


class AttemptGraph:
    """One replayable adaptive attempt of ``pair`` (FSAL, embedded) on ``rhs``."""

    def __init__(self, rhs, pair, config, grid, fixed=False):
        if not fixed and not (pair.fsal and pair.b_hat is not None):
            raise ValueError("an adaptive AttemptGraph needs an FSAL pair with embedded weights")
        self.rhs, self.pair, self.cfg, self.grid = rhs, pair, config, grid
        self.fixed = bool(fixed)
        shape = (rhs.ncomp,) + tuple(grid.kshape)
        dev = torch.device("cuda", torch.cuda.current_device())
        self.Y = [torch.zeros(shape, dtype=torch.complex128, device=dev) for _ in range(2)]
        self.FL = [torch.zeros(shape, dtype=torch.complex128, device=dev) for _ in range(2)]
        self.h_pin = torch.zeros(1, dtype=torch.float64, pin_memory=True)
        self.h_dev = torch.zeros(1, dtype=torch.float64, device=dev)
        self.q_pin = torch.zeros(9, dtype=torch.float64, pin_memory=True)  # mapped: written by the graph
        self.graphs = [None, None]
        self.launches = [0, 0]
        self.replays = 0
        self._keep = []

    # -- the attempt, as recorded ------------------------------------------------
    def _record(self, p):
        lib = _native.load()
        pl = self.rhs.plan
        prm = self.rhs.params
        nu, ri, repr_ = 1.0 / prm.reynolds, float(prm.richardson), float(prm.reynolds) * float(prm.prandtl)
        A, b, s = self.pair.A, self.pair.b, self.pair.s
        hp = _native.ptr(self.h_dev)
        y = self.Y[p]
        self.h_dev.copy_(self.h_pin, non_blocking=True)
        stages = [self.FL[p]] + [None] * (s - 1)

        def combine(base, terms, out):
            Fs = [F for _, F in terms]
            _native.check(lib.srk_combine_scaled(out.numel(), _native.ptr(base), len(Fs), _native.ptr_array(Fs),
                                                 _native.dbl_array([a for a, _ in terms]), hp, _native.ptr(out),
                                                 _native.stream_ptr()), "srk_combine_scaled")
            _native.count(1)

        # stage 2 input y + (h a21) F1 (integrators.py:327-333)
        fsal = self.pair.fsal
        y_new = self.Y[1 - p]
        x = torch.empty_like(y) if s > 2 else y_new
        combine(y, [(A[1, j], stages[j]) for j in range(1) if A[1, j] != 0.0], x)
        for i in range(1, s):
            last = i == s - 1
            f = self.FL[1 - p] if (last and fsal) else torch.empty_like(y)
            # the accumulation that consumes stage i: the next stage input (FSAL: the
            # last stage's input is y_new) or, for non-FSAL pairs, y_new itself
            if i + 1 < s:
                row, nxt = A[i + 1], (y_new if (fsal and i + 1 == s - 1) else torch.empty_like(y))
            else:
                row, nxt = (None, None) if fsal else (b, y_new)
            if row is not None:
                terms = [(row[j], stages[j]) for j in range(i) if row[j] != 0.0]
                if row[i] != 0.0 and len(terms) <= _FUSED_MAX_TERMS:
                    Fs = [F for _, F in terms]
                    _native.check(lib.srk_rhs_combine_scaled(
                        pl.bind(), _native.ptr(x), _native.ptr(f), nu, ri, repr_, _native.ptr(y), len(Fs),
                        _native.ptr_array(Fs), _native.dbl_array([a for a, _ in terms]), float(row[i]), hp,
                        _native.ptr(nxt), _native.stream_ptr()), "srk_rhs_combine_scaled")
                    _native.count(pl.lib.srk_rhs_launch_count(pl.h))
                    stages[i] = f
                    x = nxt
                    continue
            self.rhs(0.0, x, out=f)
            stages[i] = f
            if row is not None:
                combine(y, [(row[j], stages[j]) for j in range(i + 1) if row[j] != 0.0], nxt)
                x = nxt
        fl = self.FL[1 - p]
        if self.fixed:
            # fixed step: the cached tendency of y_new (FSAL stage, or a fresh RHS --
            # simulation.py:165-182) and the diagnostics record's sums (diagnostics.py:48-70)
            if not fsal:
                self.rhs(0.0, y_new, out=fl)
            _native.check(lib.srk_step_reduce(
                pl.bind(), _native.ptr(y), _native.ptr(y_new), 0, _native.ptr_array([]), _native.dbl_array([]),
                _native.ptr(fl), y.shape[0], 0.0, 0.0, 2, _native.ptr(self.q_pin), _native.stream_ptr()),
                "srk_step_reduce")
            _native.count(2)
            return
        # embedded error + E / eps / Z sums (control.py:51-79, diagnostics.py:48-70)
        d = b - self.pair.b_hat
        terms = [(d[i], stages[i]) for i in range(s) if d[i] != 0.0]
        Fs = [F for _, F in terms]
        _native.check(lib.srk_step_reduce_scaled(
            pl.bind(), _native.ptr(y), _native.ptr(y_new), len(Fs), _native.ptr_array(Fs),
            _native.dbl_array([a for a, _ in terms]), hp, _native.ptr(fl), y.shape[0], float(self.cfg.tol_abs),
            float(self.cfg.tol_rel), 3, _native.ptr(self.q_pin), _native.stream_ptr()), "srk_step_reduce_scaled")
        _native.count(2)

    def _capture(self, p):
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):  # warm-up: twiddle tables, kernel attributes, plan workspace
            self._record(p)
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        l0 = _native.LAUNCHES
        with torch.cuda.graph(g):
            self._record(p)
        self.launches[p] = _native.LAUNCHES - l0
        _native.LAUNCHES = l0  # capture launched nothing; replays are counted
        self.graphs[p] = g
        # the graph writes the plan's workspace arena as bound at capture: keep that
        # memory alive even if a larger plan later replaces the device's arena
        self._keep.append(self.rhs.plan._bound)

    # -- one adaptive step -----------------------------------------------------------
    def _slot(self, y, f_now):
        for p in (0, 1):
            if y.data_ptr() == self.Y[p].data_ptr() and f_now.data_ptr() == self.FL[p].data_ptr():
                return p
        self.Y[0].copy_(y)
        self.FL[0].copy_(f_now)
        return 0

    def step_fixed(self, y, h, f_now):
        """One fixed step of run_simulation's loop (simulation.py:250-271): returns
        (y_new, f_new, sums) with f_new the cached tendency of y_new (FSAL stage or a
        fresh RHS) and sums the diagnostics record's reduce_sums values."""
        p = self._slot(y, f_now)
        if self.graphs[p] is None:
            self._capture(p)
        self.h_pin[0] = h
        self.graphs[p].replay()
        _native.count(self.launches[p])
        self.replays += 1
        torch.cuda.current_stream().synchronize()
        return self.Y[1 - p], self.FL[1 - p], self.q_pin.tolist()

    def advance(self, y, t, state, first_stage):
        """adaptive_advance(y, t, pair, state, config, rhs, first_stage) with the first
        attempt replayed from the graph; same outcome, same accounting."""
        p = self._slot(y, first_stage)
        if self.graphs[p] is None:
            self._capture(p)
        h = state.h
        self.h_pin[0] = h
        self.graphs[p].replay()
        _native.count(self.launches[p])
        self.replays += 1
        torch.cuda.current_stream().synchronize()
        q = self.q_pin.tolist()
        ncomp = self.Y[p].shape[0]
        modes = float(self.grid.mode_count)
        if q[6] > 0:
            err = np.inf
        else:
            if q[7] > 0:
                raise ValueError("error scales must be strictly positive")
            err = float(max(np.sqrt(q[c] / modes) for c in range(ncomp)))
        h_new, accepted = propose_step(err, state, self.cfg)
        state.h = h_new
        evals = self.pair.s - 1
        if accepted:
            return AdvanceOutcome(y_new=self.Y[1 - p], t_new=t + h, h_used=h, h_next=h_new, rhs_evals=evals,
                                  rejections=0, last_stage=self.FL[1 - p], errs=[err], diag_sums=q)
        # rejected: the retries run eagerly from the unchanged state (F1 recomputed)
        out = adaptive_advance(self.Y[p], t, self.pair, state, self.cfg, self.rhs, first_stage=None,
                               grid=self.grid)
        out.rhs_evals += evals
        out.rejections += 1
        out.errs = [err] + out.errs
        return out
