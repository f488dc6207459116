"""Explicit RK pairs and the device step executor (mirrors integrators.py of the reference).

Tableaux are built from exact rationals and converted once to float64
(integrators.py:107-131).  ``rk_step`` keeps the reference's stage order and
accumulation order (ascending j, zero coefficients skipped) but runs every
linear combination through the fused srk_combine kernel; for FSAL pairs the
stage-s input *is* y_new (bitwise equal in the reference too).
"""

from __future__ import annotations

from dataclasses import dataclass
from fractions import Fraction

import numpy as np
import torch

from . import _native
from .spectral import from_device, to_device

__all__ = ["NonFiniteStateError", "ButcherPair", "StepOutcome", "make_rk4", "make_dp5", "make_bs5",
           "make_kcl5", "make_pair", "rk_step", "combine", "ab2_combine", "ab2_step"]


class NonFiniteStateError(RuntimeError):
    """A stage or updated state contains NaN or Inf (integrators.py:17)."""


class ButcherPair:
    """Explicit RK tableau with optional embedded weights (integrators.py:21-88)."""

    def __init__(self, name, A, b, c, p, b_hat=None, q=None, exact=None):
        self.name = name
        self.A = np.asarray(A, dtype=np.float64)
        self.b = np.asarray(b, dtype=np.float64)
        self.c = np.asarray(c, dtype=np.float64)
        self.b_hat = None if b_hat is None else np.asarray(b_hat, dtype=np.float64)
        self.p, self.q = p, q
        self.s = len(self.b)
        if self.A.shape != (self.s, self.s):
            raise ValueError("A must be s x s")
        if np.any(np.triu(self.A) != 0.0):
            raise ValueError("A must be strictly lower triangular")
        if abs(self.b.sum() - 1.0) > 1e-15 * self.s:
            raise ValueError("advance weights must sum to 1")
        if self.b_hat is not None and abs(self.b_hat.sum() - 1.0) > 1e-15 * self.s:
            raise ValueError("error weights must sum to 1")
        if np.max(np.abs(self.A.sum(axis=1) - self.c)) > 1e-15 * self.s:
            raise ValueError("abscissae must equal tableau row sums")
        self.exact = exact
        self.fsal = (self.b_hat is not None and self.c[-1] == 1.0 and np.array_equal(self.A[-1], self.b))

    def __repr__(self):
        emb = f"({self.q})" if self.q is not None else ""
        return f"ButcherPair({self.name}, s={self.s}, order {self.p}{emb})"


@dataclass
class StepOutcome:
    y_new: object
    error_vector: object
    rhs_evals: int
    last_stage: object = None


def _from_rationals(name, rows, b, p, b_hat=None, q=None):
    s = len(b)
    A = [[Fraction(0)] * s for _ in range(s)]
    for i, row in enumerate(rows):
        for j, v in enumerate(row):
            A[i + 1][j] = Fraction(v)
    bq = [Fraction(v) for v in b]
    cq = [sum(row, Fraction(0)) for row in A]
    bh = None if b_hat is None else [Fraction(v) for v in b_hat]
    to_f = lambda seq: [float(v) for v in seq]
    return ButcherPair(name, [to_f(r) for r in A], to_f(bq), to_f(cq), p,
                       b_hat=None if bh is None else to_f(bh), q=q, exact=(A, bq, cq, bh))


def make_rk4():
    F = Fraction
    return _from_rationals("rk4", [[F(1, 2)], [0, F(1, 2)], [0, 0, 1]], [F(1, 6), F(1, 3), F(1, 3), F(1, 6)], 4)


def make_dp5():
    F = Fraction
    rows = [[F(1, 5)], [F(3, 40), F(9, 40)], [F(44, 45), F(-56, 15), F(32, 9)],
            [F(19372, 6561), F(-25360, 2187), F(64448, 6561), F(-212, 729)],
            [F(9017, 3168), F(-355, 33), F(46732, 5247), F(49, 176), F(-5103, 18656)],
            [F(35, 384), 0, F(500, 1113), F(125, 192), F(-2187, 6784), F(11, 84)]]
    b = [F(35, 384), 0, F(500, 1113), F(125, 192), F(-2187, 6784), F(11, 84), 0]
    bh = [F(5179, 57600), 0, F(7571, 16695), F(393, 640), F(-92097, 339200), F(187, 2100), F(1, 40)]
    return _from_rationals("dp5", rows, b, 5, bh, 4)


def make_bs5():
    F = Fraction
    rows = [[F(1, 6)], [F(2, 27), F(4, 27)], [F(183, 1372), F(-162, 343), F(1053, 1372)],
            [F(68, 297), F(-4, 11), F(42, 143), F(1960, 3861)],
            [F(597, 22528), F(81, 352), F(63099, 585728), F(58653, 366080), F(4617, 20480)],
            [F(174197, 959244), F(-30942, 79937), F(8152137, 19744439), F(666106, 1039181),
             F(-29421, 29068), F(482048, 414219)],
            [F(587, 8064), 0, F(4440339, 15491840), F(24353, 124800), F(387, 44800), F(2152, 5985),
             F(7267, 94080)]]
    b = [F(587, 8064), 0, F(4440339, 15491840), F(24353, 124800), F(387, 44800), F(2152, 5985),
         F(7267, 94080), 0]
    bh = [F(2479, 34992), 0, F(123, 416), F(612941, 3411720), F(43, 1440), F(2272, 6561),
          F(79937, 1113912), F(3293, 556956)]
    return _from_rationals("bs5", rows, b, 5, bh, 4)


_KCL5 = dict(
    sub1=(0.2449991650950331532633989, 0.3255876658223002585360424, 0.2953235221406422382001682,
          0.1193703593613548032956652, 0.06565483806981039962298386, 0.3616753624764124275144138,
          0.2005935320246650226379431),
    sub2=(0.05657291200262709074196688, -0.07667012917590769265730675, 0.01045572406422470259355013,
          0.1652065151174663332707352, 0.1661850667315458191199747, 0.1455019846988342566658738),
    b=(0.09790311694145986584975407, 0.05774510356579696240927496, 0.1660969888114508950148388,
       -0.06187775335289376452019296, 0.2526229419443198221985107, 0.1675798102960971615063023,
       -0.03604824961456221699888925, 0.3559780414083312745404014),
    bh=(0.09463592814099053839208871, 0.0815494393421897267245835, 0.1507872419642323929947585,
        -0.02888689228216589896931827, 0.2174837713302734535126134, 0.1527068641691501852170764,
        -0.003581175832029266818942221, 0.3353048231673588689471399),
)


def make_kcl5():
    """8-stage 5(4) pair with the 3R low-storage column pattern (integrators.py:219-284)."""
    s = 8
    b = list(_KCL5["b"])
    A = [[0.0] * s for _ in range(s)]
    for i in range(1, s):
        A[i][i - 1] = _KCL5["sub1"][i - 1]
        if i >= 2:
            A[i][i - 2] = _KCL5["sub2"][i - 2]
        for j in range(0, i - 2):
            A[i][j] = b[j]
    c = [float(np.sum(row)) for row in A]
    return ButcherPair("kcl5", A, b, c, p=5, b_hat=list(_KCL5["bh"]), q=4)


def make_pair(name):
    makers = {"rk4": make_rk4, "dp5": make_dp5, "bs5": make_bs5, "kcl5": make_kcl5}
    if name not in makers:
        raise ValueError(f"unknown integrator '{name}'")
    return makers[name]()


def combine(y, terms, out=None):
    """out = y + sum_j c_j F_j on the device (srk_combine); y may be None (zeros)."""
    ref = y if y is not None else terms[0][1]
    if out is None:
        out = torch.empty_like(ref)
    Fs = [t for _, t in terms]
    cs = [c for c, _ in terms]
    lib = _native.load()
    _native.check(lib.srk_combine(ref.numel(), _native.ptr(y), len(Fs), _native.ptr_array(Fs),
                                  _native.dbl_array(cs), _native.ptr(out), _native.stream_ptr()), "srk_combine")
    _native.count(1)
    return out


def _as_dev_fn(f):
    def g(t, y):
        r = f(t, y)
        if not isinstance(r, torch.Tensor):
            r = torch.from_numpy(np.ascontiguousarray(r)).to(y.device)
        return r
    if callable(getattr(f, "eval_combine", None)):
        g.eval_combine = f.eval_combine  # device operator: RHS + next accumulation in one call
    return g


# srk_rhs_combine carries at most this many earlier stages on its fused path
_FUSED_MAX_TERMS = 6


def run_stages(f, y, t, h, pair, first_stage=None, on_y_new=None, second_input=None):
    """Stage loop of integrators.py:322-339 on the device.

    Returns (stages, y_new, evals).  For FSAL pairs y_new is the last stage's
    input (identical arithmetic to y + sum h b_i F_i since A[-1] == b).  When
    ``f`` is a device operator with ``eval_combine`` (FlowRHS), each stage's
    RHS call also forms the accumulation that consumes it -- the next stage
    input (row i+1 of A) or, for non-FSAL pairs, y_new -- bitwise the same sums,
    without reading the new stage back (srk_rhs_combine).

    ``on_y_new(y_new)`` is called once y_new is queued: for FSAL pairs before the
    last stage's RHS (whose input it is), so a consumer such as
    ``HostMirror.push`` overlaps that evaluation.

    ``second_input``: the stage-2 input y + h a21 F1 already formed together with
    ``first_stage`` (FlowRHS.refresh); used as is (bitwise what the combine
    would give) -- the caller guarantees it was formed with this h.
    """
    A, b, c, s = pair.A, pair.b, pair.c, pair.s
    fused = getattr(f, "eval_combine", None)
    evals = 0
    stages = [None] * s
    pending = None  # input of stage i (or y_new) formed by the previous stage's call
    yi = None
    for i in range(s):
        if i == 0:
            if first_stage is not None:
                stages[0] = first_stage
                continue
            xi = y
        elif pending is not None:
            xi, pending = pending, None
        elif i == 1 and second_input is not None and stages[0] is first_stage:
            xi = second_input
        else:
            xi = combine(y, [(h * A[i, j], stages[j]) for j in range(i) if A[i, j] != 0.0])
        if i > 0:
            yi = xi
            if on_y_new is not None and pair.fsal and i == s - 1:
                on_y_new(xi)
        row = A[i + 1] if i + 1 < s else (None if pair.fsal else b)
        if fused is not None and row is not None and row[i] != 0.0:
            terms = [(h * row[j], stages[j]) for j in range(i) if row[j] != 0.0]
            if len(terms) <= _FUSED_MAX_TERMS:
                stages[i], pending = fused(t + c[i] * h, xi, y, terms, h * row[i])
                evals += 1
                continue
        stages[i] = f(t + c[i] * h, xi)
        evals += 1
    if pair.fsal and yi is not None:
        y_new = yi
    elif pending is not None:
        y_new = pending
    else:
        y_new = combine(y, [(h * b[i], stages[i]) for i in range(s) if b[i] != 0.0])
    if on_y_new is not None and not (pair.fsal and yi is not None):
        on_y_new(y_new)
    return stages, y_new, evals


def error_terms(h, pair, stages):
    d = pair.b - pair.b_hat
    return [(h * d[i], stages[i]) for i in range(pair.s) if d[i] != 0.0]


def rk_step(f, y, t, h, pair, first_stage=None):
    """One explicit RK step (integrators.py:295-358) with device arithmetic."""
    from .diagnostics import reduce_sums
    from .grid import Grid

    yd, was_np = to_device(y, torch.complex128)
    fd = _as_dev_fn(f)
    fs = None if first_stage is None else to_device(first_stage, torch.complex128)[0]
    stages, y_new, evals = run_stages(fd, yd, t, h, pair, fs)
    err = None
    terms = []
    if pair.b_hat is not None:
        terms = error_terms(h, pair, stages)
        err = combine(None, terms) if terms else torch.zeros_like(yd)
    kshape = tuple(yd.shape[1:])
    grid = Grid(kshape[:-1] + (2 * (kshape[-1] - 1),))
    q = reduce_sums(grid, y_new, y0=yd, terms=terms, tol_abs=1.0, tol_rel=0.0,
                    flags=1 if terms else 0, ncomp=yd.shape[0], host=True).tolist()
    if q[6] > 0:
        raise NonFiniteStateError(f"non-finite state at t={t}")
    return StepOutcome(y_new=from_device(y_new, was_np), error_vector=None if err is None else from_device(err, was_np),
                       rhs_evals=evals, last_stage=from_device(stages[-1], was_np) if pair.fsal else None)


def ab2_combine(y, h, f_curr, f_prev):
    """y + h (1.5 f_curr - 0.5 f_prev) on the device (integrators.py:361-363).

    Two srk_combine passes in the reference's association: g = 1.5 f_curr +
    (-0.5) f_prev (0 + 1.5 f is exact, x + (-y) == x - y), then y + h g --
    bitwise numpy's rounding of ``y + h * (1.5 * f_curr - 0.5 * f_prev)``.
    numpy inputs are moved to the device and the result comes back as numpy."""
    yd, was_np = to_device(y, torch.complex128)
    fc = to_device(f_curr, torch.complex128)[0]
    fp = to_device(f_prev, torch.complex128)[0]
    g = combine(None, [(1.5, fc), (-0.5, fp)])
    return from_device(combine(yd, [(float(h), g)], out=g), was_np)


def ab2_step(f, y, t, h, f_prev):
    """One AB2 step (integrators.py:366-381): returns (y_new, f_curr)."""
    from .diagnostics import reduce_sums
    from .grid import Grid

    if f_prev is None:
        raise ValueError("ab2_step requires the previous slope; bootstrap first")
    yd, was_np = to_device(y, torch.complex128)
    fd = _as_dev_fn(f)
    f_curr = fd(t, yd)
    y_new = ab2_combine(yd, h, f_curr, to_device(f_prev, torch.complex128)[0])
    kshape = tuple(yd.shape[1:])
    grid = Grid(kshape[:-1] + (2 * (kshape[-1] - 1),))
    q = reduce_sums(grid, y_new, flags=0, ncomp=yd.shape[0], host=True).tolist()
    if q[6] > 0:
        raise NonFiniteStateError(f"non-finite state at t={t}")
    return from_device(y_new, was_np), from_device(f_curr, was_np)
