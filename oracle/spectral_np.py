"""numpy/scipy restatement of the reference hot path (TEST INFRASTRUCTURE ONLY).

Every function cites the reference file:line it restates; paths are relative
to ``/root/reference/pkg/src/spectralrk/``.  Nothing here is imported by the
product package.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from fractions import Fraction

import numpy as np
import scipy.fft
from scipy.special import erf

__all__ = [
    "OGrid", "fwd", "inv", "curl", "zero_nyquist", "zero_self_conj_imag",
    "symmetrize_planes", "Dealias", "cross_kernel", "ns_rhs", "boussinesq_rhs",
    "leray", "OracleRHS", "apply_forcing", "kinetic_energy", "dissipation_rate",
    "enstrophy", "Tableau", "tableau", "rk_step", "scale_vector",
    "error_norm_delta", "propose_step", "Ctrl", "CtrlState", "adaptive_advance",
    "NonFinite", "Underflow", "ForcingErr", "taylor_green", "rayleigh_taylor",
    "hit", "rt_tanh_ic", "Record", "run_fixed", "run_adaptive", "replay_steps",
    "set_fft_workers", "ab2_combine", "run_ab2",
]

_WORKERS = 1


def set_fft_workers(n):
    """Threads for the scipy x/y C2C calls (bitwise-neutral)."""
    global _WORKERS
    _WORKERS = int(n)


class NonFinite(RuntimeError):
    """integrators.py:17 NonFiniteStateError."""


class Underflow(RuntimeError):
    """control.py:20 StepSizeUnderflowError."""


class ForcingErr(RuntimeError):
    """physics.py:23 ForcingError."""


# --------------------------------------------------------------------------
# geometry -- grid.py:53-121
# --------------------------------------------------------------------------
class OGrid:
    """Periodic grid in the rfftn layout (grid.py:53-121).

    The r2c axis is the LAST axis (grid.py:71).  Full-axis mode labels are
    fftfreq with the Nyquist slot relabelled +n/2 (grid.py:75-82).
    """

    def __init__(self, shape, lengths=None):
        shape = tuple(int(n) for n in shape)
        if len(shape) not in (2, 3):
            raise ValueError("grid must be 2D or 3D")
        if any(n < 4 or n % 2 for n in shape):
            raise ValueError("grid extents must be even and >= 4")
        d = len(shape)
        if lengths is None:
            lengths = (2.0 * np.pi,) * d
        self.lengths = tuple(float(v) for v in lengths)
        self.shape = shape
        self.dims = d
        self.kshape = shape[:-1] + (shape[-1] // 2 + 1,)
        self.points = math.prod(shape)
        self.mode_count = math.prod(self.kshape)
        self.pshape = tuple(3 * n // 2 for n in shape)
        ks = []
        for ax, n in enumerate(shape):
            if ax == d - 1:
                m = np.arange(n // 2 + 1, dtype=np.float64)
            else:
                m = np.concatenate([np.arange(0, n // 2 + 1), np.arange(-(n // 2) + 1, 0)]).astype(np.float64)
            view = [1] * d
            view[ax] = m.size
            ks.append((m * (2.0 * np.pi / self.lengths[ax])).reshape(view))
        self.k = tuple(ks)
        acc = np.zeros(self.kshape)
        for ka in ks:  # same accumulation order as grid.py:94-97
            acc = acc + ka * ka
        self.k2 = acc
        self.inv_k2 = np.where(acc == 0.0, 0.0, 1.0 / np.where(acc == 0.0, 1.0, acc))
        w = np.full(self.kshape[-1], 2.0)
        w[0] = w[-1] = 1.0
        self.w = w.reshape((1,) * (d - 1) + (-1,))
        self.x = tuple(
            (np.arange(n) * (self.lengths[ax] / n)).reshape([n if a == ax else 1 for a in range(d)])
            for ax, n in enumerate(shape)
        )


def _axes(g):
    return tuple(range(-g.dims, 0))


def fwd(field_, g):
    """forward_transform, spectral.py:17-30 (unnormalised rfftn)."""
    return scipy.fft.rfftn(np.asarray(field_), axes=_axes(g))


def inv(spec, g):
    """inverse_transform, spectral.py:33-44."""
    return scipy.fft.irfftn(np.asarray(spec), s=g.shape, axes=_axes(g))


def curl(u, g):
    """spectral.py:47-65: i k x u (3D vector, 2D scalar)."""
    k = g.k
    if g.dims == 3:
        w = np.empty_like(u)
        w[0] = 1j * (k[1] * u[2] - k[2] * u[1])
        w[1] = 1j * (k[2] * u[0] - k[0] * u[2])
        w[2] = 1j * (k[0] * u[1] - k[1] * u[0])
        return w
    return 1j * (k[0] * u[1] - k[1] * u[0])


def zero_nyquist(spec, g):
    """spectral.py:73-80: zero the n/2 slot of every axis (incl. the r2c one)."""
    lead = spec.ndim - g.dims
    for ax, n in enumerate(g.shape):
        idx = [slice(None)] * spec.ndim
        idx[lead + ax] = n // 2
        spec[tuple(idx)] = 0.0
    return spec


def zero_self_conj_imag(spec, g):
    """spectral.py:83-95: modes whose indices are all 0 or n/2 are real."""
    lead = (slice(None),) * (spec.ndim - g.dims)
    sel = np.ix_(*[np.array([0, n // 2]) for n in g.shape])
    spec[lead + sel] = spec[lead + sel].real
    return spec


def symmetrize_planes(spec, g):
    """spectral.py:98-115: Hermitian symmetrisation of the kz=0 and kz=n/2 planes."""
    lead = spec.ndim - g.dims
    for kz in (0, g.shape[-1] // 2):
        idx = [slice(None)] * spec.ndim
        idx[-1] = kz
        plane = spec[tuple(idx)]
        mirrored = plane
        for ax in range(lead, lead + g.dims - 1):
            mirrored = np.roll(np.flip(mirrored, axis=ax), 1, axis=ax)
        spec[tuple(idx)] = 0.5 * (plane + np.conj(mirrored))
    return spec


# --------------------------------------------------------------------------
# 3/2-rule factored transforms -- spectral.py:174-304
# --------------------------------------------------------------------------
class Dealias:
    """Restatement of DealiasWorkspace.widen / narrow (spectral.py:215-304).

    widen: for each full axis in order (x, then y): zero-band pad n -> m with
    the head 0..n/2 (incl. the Nyquist slot) and tail n/2+1..n-1 (x-pass also
    scales by 1.5**dims), scipy ifft along that axis; then numpy irfft(n=m)
    on the last axis.  narrow: numpy rfft on the last axis keeping n/2+1,
    scipy fft + truncation on the middle axis (y-Nyquist row zeroed), scipy fft
    on x with (1/1.5)**dims and truncation; then zero_nyquist and
    zero_self_conj_imag.
    """

    def __init__(self, g):
        self.g = g

    def widen(self, spec):
        g = self.g
        arr = np.asarray(spec)
        for ax in range(g.dims - 1):
            n, m = g.shape[ax], g.pshape[ax]
            a1 = 1 + ax
            shp = list(arr.shape)
            shp[a1] = m
            buf = np.zeros(shp, dtype=np.complex128)
            src_h = [slice(None)] * arr.ndim
            src_t = [slice(None)] * arr.ndim
            dst_t = [slice(None)] * arr.ndim
            src_h[a1] = slice(0, n // 2 + 1)
            src_t[a1] = slice(n // 2 + 1, n)
            dst_t[a1] = slice(m - (n // 2 - 1), m)
            if ax == 0:
                s = 1.5 ** g.dims
                buf[tuple(src_h)] = arr[tuple(src_h)] * s
                buf[tuple(dst_t)] = arr[tuple(src_t)] * s
            else:
                buf[tuple(src_h)] = arr[tuple(src_h)]
                buf[tuple(dst_t)] = arr[tuple(src_t)]
            arr = scipy.fft.ifft(buf, axis=a1, overwrite_x=True, workers=_WORKERS)
        return np.fft.irfft(arr, n=g.pshape[-1], axis=-1)

    def narrow(self, phys):
        g = self.g
        kz = g.kshape[-1]
        arr = np.fft.rfft(np.asarray(phys), axis=-1)[..., :kz]
        for ax in range(g.dims - 2, -1, -1):
            n = g.shape[ax]
            a1 = 1 + ax
            arr = scipy.fft.fft(arr, axis=a1, overwrite_x=True, workers=_WORKERS)
            m = arr.shape[a1]
            shp = list(arr.shape)
            shp[a1] = n
            out = np.empty(shp, dtype=np.complex128)
            h = [slice(None)] * arr.ndim
            t_src = [slice(None)] * arr.ndim
            t_dst = [slice(None)] * arr.ndim
            ny = [slice(None)] * arr.ndim
            h[a1] = slice(0, n // 2)
            t_src[a1] = slice(m - (n // 2 - 1), m)
            t_dst[a1] = slice(n // 2 + 1, n)
            ny[a1] = n // 2
            if ax == 0:
                s = (1.0 / 1.5) ** g.dims
                out[tuple(h)] = arr[tuple(h)] * s
                out[tuple(ny)] = 0.0
                out[tuple(t_dst)] = arr[tuple(t_src)] * s
            else:
                out[tuple(h)] = arr[tuple(h)]
                out[tuple(ny)] = 0.0
                out[tuple(t_dst)] = arr[tuple(t_src)]
            arr = out
        zero_nyquist(arr, g)
        zero_self_conj_imag(arr, g)
        return arr

    def product(self, kernel, specs):
        """dealiased_product, spectral.py:307-337."""
        if isinstance(specs, np.ndarray):
            specs = [specs]
        pieces = [p if p.ndim == self.g.dims + 1 else p[None] for p in specs]
        return self.narrow(kernel(self.widen(np.concatenate(pieces, axis=0))))


# --------------------------------------------------------------------------
# physics -- physics.py:62-239
# --------------------------------------------------------------------------
def cross_kernel(d):
    """physics.py:62-82: u x omega on the padded grid."""

    def kern(ph):
        u, w = ph[:d], ph[d:]
        out = np.empty((d,) + ph.shape[1:])
        if d == 3:
            out[0] = u[1] * w[2] - u[2] * w[1]
            out[1] = u[2] * w[0] - u[0] * w[2]
            out[2] = u[0] * w[1] - u[1] * w[0]
        else:
            out[0] = u[1] * w[0]
            out[1] = -(u[0] * w[0])
        return out

    return kern


def leray(u, g):
    """physics.py:89-102."""
    kd = np.zeros(g.kshape, dtype=np.complex128)
    for j in range(g.dims):
        kd += g.k[j] * u[j]
    kd *= g.inv_k2
    out = u.copy()
    for j in range(g.dims):
        out[j] -= g.k[j] * kd
    return out


def _project_viscous(G, u, g, nu):
    """physics.py:119-129 (and 168-178): P(G) - nu |k|^2 u."""
    d = g.dims
    kd = g.k[0] * G[0]
    for j in range(1, d):
        kd += g.k[j] * G[j]
    kd *= g.inv_k2
    out = np.empty((d,) + g.kshape, dtype=np.complex128)
    for j in range(d):
        out[j] = G[j]
        out[j] -= g.k[j] * kd
        out[j] -= (nu * g.k2) * u[j]
    return out


def ns_rhs(u, g, re, dl=None):
    """physics.py:105-129."""
    dl = dl or Dealias(g)
    w = curl(u, g)
    if g.dims == 2:
        w = w[None]
    G = dl.product(cross_kernel(g.dims), [u, w])
    return _project_viscous(G, u, g, 1.0 / re)


def boussinesq_rhs(fields, g, re, ri, pr, dl=None):
    """physics.py:132-185."""
    dl = dl or Dealias(g)
    d = g.dims
    u = fields[:d]
    rho = fields[d]
    w = curl(u, g)
    if d == 2:
        w = w[None]
    wc = w.shape[0]
    ck = cross_kernel(d)

    def kern(ph):
        out = np.empty((2 * d,) + ph.shape[1:])
        out[:d] = ck(ph[: d + wc])
        for j in range(d):
            out[d + j] = ph[d + wc] * ph[j]
        return out

    prod = dl.product(kern, [u, w, fields[d:d + 1]])
    G = prod[:d]
    flux = prod[d:]
    G[d - 1] -= ri * rho
    out = np.empty_like(fields)
    out[:d] = _project_viscous(G, u, g, 1.0 / re)
    div = g.k[0] * flux[0]
    for j in range(1, d):
        div += g.k[j] * flux[j]
    out[d] = -1j * div
    out[d] -= (g.k2 / (re * pr)) * rho
    return out


class OracleRHS:
    """FlowRHS, physics.py:188-206: callable f(t, y)."""

    def __init__(self, g, re, ri=1.0, pr=1.0, density=False):
        self.g, self.re, self.ri, self.pr, self.density = g, re, ri, pr, density
        self.dl = Dealias(g)
        self.calls = 0

    def __call__(self, t, y):
        self.calls += 1
        if self.density:
            return boussinesq_rhs(y, self.g, self.re, self.ri, self.pr, self.dl)
        return ns_rhs(y, self.g, self.re, self.dl)


def _wsum_abs2(a, g):
    tot = 0.0
    for j in range(a.shape[0]):
        tot += float(np.sum(g.w * (a[j].real ** 2 + a[j].imag ** 2)))
    return tot


def kinetic_energy(u, g):
    """diagnostics.py:48-50."""
    return _wsum_abs2(u, g) / (2.0 * g.points ** 2)


def dissipation_rate(u, f, g):
    """diagnostics.py:53-70 (velocity components only)."""
    tot = 0.0
    for j in range(g.dims):
        tot += float(np.sum(g.w * (u[j] * np.conj(f[j])).real))
    return -tot / g.points ** 2


def enstrophy(u, g):
    """Discrepancy D2: Z = sum_k w_k |k|^2 sum_j |u_kj|^2 / (2 points^2).

    Not in the reference; defined with the same Hermitian weights as
    kinetic_energy (diagnostics.py:39-50) so eps = 2 nu Z for pure NS.
    """
    tot = 0.0
    for j in range(g.dims):
        tot += float(np.sum(g.w * g.k2 * (u[j].real ** 2 + u[j].imag ** 2)))
    return tot / (2.0 * g.points ** 2)


def apply_forcing(u, g, target, k_f):
    """physics.py:209-239: rescale 0<|k|<=k_f to restore the target energy."""
    band = (g.k2 > 0.0) & (g.k2 <= k_f * k_f * (1.0 + 1e-12))
    e_tot = kinetic_energy(u, g)
    w = np.broadcast_to(g.w, g.kshape)
    e_band = 0.0
    for j in range(u.shape[0]):
        a = u[j]
        e_band += np.sum(w[band] * (a.real[band] ** 2 + a.imag[band] ** 2))
    e_band /= 2.0 * g.points ** 2
    e_rest = e_tot - e_band
    if e_band <= 0.0:
        raise ForcingErr("forcing band carries no energy")
    rad = (target - e_rest) / e_band
    if rad < 0.0:
        raise ForcingErr("energy outside the band exceeds the target")
    gamma = float(np.sqrt(rad))
    for j in range(u.shape[0]):
        u[j][band] *= gamma
    return gamma


# --------------------------------------------------------------------------
# tableaux -- integrators.py:107-292
# --------------------------------------------------------------------------
@dataclass
class Tableau:
    name: str
    A: np.ndarray
    b: np.ndarray
    c: np.ndarray
    b_hat: np.ndarray | None
    p: int
    q: int | None

    @property
    def s(self):
        return len(self.b)

    @property
    def fsal(self):  # integrators.py:80-84
        return (self.b_hat is not None and self.c[-1] == 1.0
                and np.array_equal(self.A[-1], self.b))


def _exact(name, rows, b, p, bh=None, q=None):
    """integrators.py:107-131: rationals -> float64 once."""
    s = len(b)
    A = [[Fraction(0)] * s for _ in range(s)]
    for i, r in enumerate(rows):
        for j, v in enumerate(r):
            A[i + 1][j] = Fraction(v)
    c = [sum(r, Fraction(0)) for r in A]
    f = lambda v: np.array([float(x) for x in v])
    return Tableau(name, np.array([[float(x) for x in r] for r in A]), f(map(Fraction, b)),
                   f(c), None if bh is None else f(map(Fraction, bh)), p, q)


def tableau(name):
    F = Fraction
    if name == "rk4":  # integrators.py:134-142
        return _exact("rk4", [[F(1, 2)], [0, F(1, 2)], [0, 0, 1]],
                      [F(1, 6), F(1, 3), F(1, 3), F(1, 6)], 4)
    if name == "dp5":  # integrators.py:145-166 (Dormand-Prince 5(4))
        rows = [[F(1, 5)], [F(3, 40), F(9, 40)], [F(44, 45), F(-56, 15), F(32, 9)],
                [F(19372, 6561), F(-25360, 2187), F(64448, 6561), F(-212, 729)],
                [F(9017, 3168), F(-355, 33), F(46732, 5247), F(49, 176), F(-5103, 18656)],
                [F(35, 384), 0, F(500, 1113), F(125, 192), F(-2187, 6784), F(11, 84)]]
        b = [F(35, 384), 0, F(500, 1113), F(125, 192), F(-2187, 6784), F(11, 84), 0]
        bh = [F(5179, 57600), 0, F(7571, 16695), F(393, 640), F(-92097, 339200),
              F(187, 2100), F(1, 40)]
        return _exact("dp5", rows, b, 5, bh, 4)
    if name == "bs5":  # integrators.py:169-216 (Bogacki-Shampine 5(4))
        rows = [[F(1, 6)], [F(2, 27), F(4, 27)], [F(183, 1372), F(-162, 343), F(1053, 1372)],
                [F(68, 297), F(-4, 11), F(42, 143), F(1960, 3861)],
                [F(597, 22528), F(81, 352), F(63099, 585728), F(58653, 366080), F(4617, 20480)],
                [F(174197, 959244), F(-30942, 79937), F(8152137, 19744439), F(666106, 1039181),
                 F(-29421, 29068), F(482048, 414219)],
                [F(587, 8064), 0, F(4440339, 15491840), F(24353, 124800), F(387, 44800),
                 F(2152, 5985), F(7267, 94080)]]
        b = [F(587, 8064), 0, F(4440339, 15491840), F(24353, 124800), F(387, 44800),
             F(2152, 5985), F(7267, 94080), 0]
        bh = [F(2479, 34992), 0, F(123, 416), F(612941, 3411720), F(43, 1440),
              F(2272, 6561), F(79937, 1113912), F(3293, 556956)]
        return _exact("bs5", rows, b, 5, bh, 4)
    if name == "kcl5":  # integrators.py:225-284 (float constants, low-storage pattern)
        sub1 = (0.2449991650950331532633989, 0.3255876658223002585360424,
                0.2953235221406422382001682, 0.1193703593613548032956652,
                0.06565483806981039962298386, 0.3616753624764124275144138,
                0.2005935320246650226379431)
        sub2 = (0.05657291200262709074196688, -0.07667012917590769265730675,
                0.01045572406422470259355013, 0.1652065151174663332707352,
                0.1661850667315458191199747, 0.1455019846988342566658738)
        b = np.array([0.09790311694145986584975407, 0.05774510356579696240927496,
                      0.1660969888114508950148388, -0.06187775335289376452019296,
                      0.2526229419443198221985107, 0.1675798102960971615063023,
                      -0.03604824961456221699888925, 0.3559780414083312745404014])
        bh = np.array([0.09463592814099053839208871, 0.0815494393421897267245835,
                       0.1507872419642323929947585, -0.02888689228216589896931827,
                       0.2174837713302734535126134, 0.1527068641691501852170764,
                       -0.003581175832029266818942221, 0.3353048231673588689471399])
        A = np.zeros((8, 8))
        for i in range(1, 8):
            A[i, i - 1] = sub1[i - 1]
            if i >= 2:
                A[i, i - 2] = sub2[i - 2]
            for j in range(0, i - 2):
                A[i, j] = b[j]
        c = np.array([float(np.sum(r)) for r in A])
        return Tableau("kcl5", A, b, c, bh, 5, 4)
    raise ValueError(f"unknown integrator {name!r}")


# --------------------------------------------------------------------------
# stepping -- integrators.py:295-358, control.py:24-169
# --------------------------------------------------------------------------
@dataclass
class StepOut:
    y_new: np.ndarray
    err_vec: np.ndarray | None
    evals: int
    last: np.ndarray | None


def rk_step(f, y, t, h, tab, first=None):
    """integrators.py:295-358 (ascending-j accumulation, zeros skipped)."""
    A, b, c, s = tab.A, tab.b, tab.c, tab.s
    ev = 0
    F = [None] * s
    if first is None:
        F[0] = f(t, y)
        ev += 1
    else:
        F[0] = first
    for i in range(1, s):
        yi = y.copy()
        for j in range(i):
            if A[i, j] != 0.0:
                yi += (h * A[i, j]) * F[j]
        F[i] = f(t + c[i] * h, yi)
        ev += 1
    y_new = y.copy()
    for i in range(s):
        if b[i] != 0.0:
            y_new += (h * b[i]) * F[i]
    ev_vec = None
    if tab.b_hat is not None:
        d = b - tab.b_hat
        ev_vec = np.zeros_like(y)
        for i in range(s):
            if d[i] != 0.0:
                ev_vec += (h * d[i]) * F[i]
        if not np.all(np.isfinite(ev_vec)):
            raise NonFinite(f"non-finite error estimate at t={t}")
    if not np.all(np.isfinite(y_new)):
        raise NonFinite(f"non-finite state at t={t}")
    return StepOut(y_new, ev_vec, ev, F[-1] if tab.fsal else None)


@dataclass
class Ctrl:
    """control.py:24-38."""
    tol_abs: float = 1e-6
    tol_rel: float = 1e-6
    safety: float = 0.8
    shrink_min: float = 0.01
    growth_max: float = 2.0
    embedded_order: int = 4
    h_min: float | None = None


@dataclass
class CtrlState:
    """control.py:41-47."""
    h: float
    prev_rejected: bool = False
    acceptances: int = 0
    rejections: int = 0


def scale_vector(y0, y1, cfg):
    """control.py:51-57."""
    return cfg.tol_abs + np.maximum(np.abs(y0), np.abs(y1)) * cfg.tol_rel


def error_norm_delta(delta, sc):
    """control.py:72-79: max over components of the RMS over stored modes."""
    if np.any(sc <= 0.0):
        raise ValueError("error scales must be strictly positive")
    nc = delta.shape[0] if delta.ndim > 1 else 1
    r2 = (np.abs(delta) / sc) ** 2
    return float(np.sqrt(r2.reshape(nc, -1).mean(axis=1)).max())


def propose_step(err, st, cfg):
    """control.py:82-116."""
    cap = 1.0 if st.prev_rejected else cfg.growth_max
    ex = 1.0 / (cfg.embedded_order + 1.0)
    if not np.isfinite(err):
        fac, ok = cfg.shrink_min, False
    else:
        fac = cap if err == 0.0 else min(cap, max(cfg.shrink_min, cfg.safety * err ** (-ex)))
        ok = err <= 1.0
    h_new = st.h * fac
    hmin = cfg.h_min if cfg.h_min is not None else 0.0
    if h_new < hmin:
        raise Underflow(f"proposed step {h_new:.3e} below minimum {hmin:.3e}")
    if ok:
        st.acceptances += 1
        st.prev_rejected = False
    else:
        st.rejections += 1
        st.prev_rejected = True
    return h_new, ok


@dataclass
class Advance:
    y_new: np.ndarray
    t_new: float
    h_used: float
    h_next: float
    evals: int
    rejections: int
    last: np.ndarray | None
    errs: list = field(default_factory=list)


def adaptive_advance(y, t, tab, st, cfg, f, first=None):
    """control.py:132-169 (retry loop; F1 recomputed after a rejection)."""
    ev = rej = 0
    errs = []
    while True:
        h = st.h
        try:
            o = rk_step(f, y, t, h, tab, first)
            ev += o.evals
            err = error_norm_delta(o.err_vec, scale_vector(y, o.y_new, cfg))
        except NonFinite:
            ev += tab.s - (1 if first is not None else 0)
            err = np.inf
        errs.append(err)
        h_new, ok = propose_step(err, st, cfg)
        st.h = h_new
        if ok:
            return Advance(o.y_new, t + h, h, h_new, ev, rej, o.last, errs)
        rej += 1
        first = None


# --------------------------------------------------------------------------
# initial conditions -- problems.py:37-108
# --------------------------------------------------------------------------
def taylor_green(g):
    """problems.py:37-62."""
    x = g.x
    z = np.zeros(g.shape)
    if g.dims == 3:
        u = np.stack([np.sin(x[0]) * np.cos(x[1]) * np.cos(x[2]) + z,
                      -np.cos(x[0]) * np.sin(x[1]) * np.cos(x[2]) + z, z])
    else:
        u = np.stack([np.sin(x[0]) * np.cos(x[1]) + z, -np.cos(x[0]) * np.sin(x[1]) + z])
    return fwd(u, g)


def rayleigh_taylor(g, delta_rho=0.1, z0=None, amplitude=0.01):
    """problems.py:65-82: quiescent velocity, erf density interface."""
    x = g.x
    z0 = 0.5 * g.lengths[-1] if z0 is None else z0
    zeta = amplitude * np.cos(x[0]) * np.cos(x[1]) if g.dims == 3 else -amplitude * np.cos(x[0])
    rho = 0.5 * delta_rho * erf(x[-1] - z0 + zeta) + np.zeros(g.shape)
    out = np.zeros((g.dims + 1,) + g.kshape, dtype=np.complex128)
    out[g.dims] = fwd(rho[None], g)[0]
    return out


def hit(g, a=9.5, energy=1.0, seed=None):
    """problems.py:85-108: random-phase solenoidal field, |k| exp(-|k|^2/a^2)."""
    if seed is None:
        raise ValueError("hit requires a seed")
    rng = np.random.default_rng(seed)
    mod = np.sqrt(g.k2) * np.exp(-g.k2 / a ** 2)
    ph = rng.uniform(0.0, 2.0 * np.pi, size=(g.dims,) + g.kshape)
    u = mod * np.exp(1j * ph)
    symmetrize_planes(u, g)
    zero_nyquist(u, g)
    u = leray(u, g)
    u *= np.sqrt(energy / kinetic_energy(u, g))
    return u


def rt_tanh_ic(g, width=0.05, amp=1e-3, kmax=8, seed=4, y0=None):
    """Config-4 IC (not in the reference): 2D Boussinesq state with
    rho = tanh((y - y0)/width) + amp * (seeded random modes with |k| <= kmax),
    u = 0.  The vertical axis is the last (r2c) axis as in physics.py:166."""
    x = g.x
    y0 = 0.5 * g.lengths[-1] if y0 is None else y0
    rho = np.tanh((x[-1] - y0) / width) + np.zeros(g.shape)
    rng = np.random.default_rng(seed)
    pert = rng.standard_normal((1,) + g.kshape) + 1j * rng.standard_normal((1,) + g.kshape)
    pert[:, (g.k2 > kmax * kmax)] = 0.0
    symmetrize_planes(pert, g)
    zero_nyquist(pert, g)
    pr = inv(pert, g)[0]
    pr *= amp / max(np.max(np.abs(pr)), 1e-300)
    out = np.zeros((g.dims + 1,) + g.kshape, dtype=np.complex128)
    out[g.dims] = fwd((rho + pr)[None], g)[0]
    return out


# --------------------------------------------------------------------------
# drivers -- simulation.py:151-347 (restated with a step cap)
# --------------------------------------------------------------------------
@dataclass
class Record:
    t: float
    h: float
    e_kin: float
    eps: float
    ens: float
    evals: int
    rejections: int


def _rec(t, h, y, fnow, g, ev, rej):
    d = g.dims
    return Record(t, h, kinetic_energy(y[:d], g), dissipation_rate(y[:d], fnow[:d], g),
                  enstrophy(y[:d], g), ev, rej)


def run_fixed(f, y, g, tab, h, t_end, max_steps=None):
    """_run_fixed + _fixed_step_times (simulation.py:222-271), t0 = 0, no forcing."""
    fnow = f(0.0, y)
    ev = 1
    t = 0.0
    recs = [_rec(t, h, y, fnow, g, ev, 0)]
    n_full = int(np.floor(t_end / h + 1e-9))
    h_last = t_end - n_full * h
    if h_last < 1e-12 * h:
        h_last = 0.0
    total = n_full + (1 if h_last > 0.0 else 0)
    if max_steps is not None:
        total = min(total, max_steps)
    for i in range(total):
        hi = h if i < n_full else h_last
        o = rk_step(f, y, t, hi, tab, fnow)
        ev += o.evals
        y = o.y_new
        t = t_end if i >= n_full else (i + 1) * h
        if tab.fsal and o.last is not None:
            fnow = o.last
        else:
            fnow = f(t, y)
            ev += 1
        recs.append(_rec(t, hi, y, fnow, g, ev, 0))
    return y, recs


def ab2_combine(y, h, f_curr, f_prev):
    """integrators.py:361-363 (numpy's association and rounding)."""
    return y + h * (1.5 * f_curr - 0.5 * f_prev)


def run_ab2(f, y, g, h, t_end, max_steps=None):
    """_run_ab2 (simulation.py:274-310), t0 = 0: one RK4 bootstrap step, then
    AB2 from the cached slopes; an uneven tail step restarts with RK4."""
    rk4 = tableau("rk4")
    fnow = f(0.0, y)
    ev = 1
    t = 0.0
    recs = [_rec(t, h, y, fnow, g, ev, 0)]
    n_full = int(np.floor(t_end / h + 1e-9))
    h_last = t_end - n_full * h
    if h_last < 1e-12 * h:
        h_last = 0.0
    total = n_full + (1 if h_last > 0.0 else 0)
    if max_steps is not None:
        total = min(total, max_steps)
    if total == 0:
        return y, recs

    def time_at(i):
        return t_end if i >= n_full else (i + 1) * h

    h0 = h if n_full > 0 else h_last
    o = rk_step(f, y, t, h0, rk4, fnow)
    ev += o.evals
    f_prev = fnow
    y = o.y_new
    t = time_at(0)
    fnow = f(t, y)
    ev += 1
    recs.append(_rec(t, h0, y, fnow, g, ev, 0))
    for i in range(1, total):
        hi = h if i < n_full else h_last
        if hi != h:
            o = rk_step(f, y, t, hi, rk4, fnow)
            ev += o.evals
            y = o.y_new
        else:
            y = ab2_combine(y, h, fnow, f_prev)  # no finiteness check here (as the reference)
        f_prev = fnow
        t = time_at(i)
        fnow = f(t, y)
        ev += 1
        recs.append(_rec(t, hi, y, fnow, g, ev, 0))
    return y, recs


def run_adaptive(f, y, g, tab, cfg, h0, t_end, max_steps=None, forcing=None):
    """_run_adaptive (simulation.py:313-347) with an optional accepted-step cap.

    ``forcing`` = (target_energy, k_f) applies apply_forcing after every
    accepted step and invalidates the FSAL cache (simulation.py:165-182).
    Returns (y, records, per-step err lists).
    """
    st = CtrlState(h=h0)
    fnow = f(0.0, y)
    ev, rej, t = 1, 0, 0.0
    recs = [_rec(t, h0, y, fnow, g, ev, rej)]
    errs = []
    n = 0
    while t < t_end and (max_steps is None or n < max_steps):
        rem = t_end - t
        clamped = st.h >= rem
        saved = st.h
        if clamped:
            st.h = rem
        o = adaptive_advance(y, t, tab, st, cfg, f, fnow)
        ev += o.evals
        rej += o.rejections
        y = o.y_new
        if clamped and o.rejections == 0:
            t = t_end
            st.h = saved
        else:
            t = o.t_new
            if clamped and o.t_new >= t_end - 1e-12 * t_end:
                t = t_end
        forced = False
        if forcing is not None:
            y = y.copy()
            apply_forcing(y[: g.dims], g, forcing[0], forcing[1])
            forced = True
        if tab.fsal and not forced and o.last is not None:
            fnow = o.last
        else:
            fnow = f(t, y)
            ev += 1
        recs.append(_rec(t, o.h_used, y, fnow, g, ev, rej))
        errs.append(o.errs)
        n += 1
    return y, recs, errs


def replay_steps(f, y, g, tab, hs):
    """Pinned step sequence: rk_step with the given accepted h list,
    FSAL first stage carried over.  Rejected attempts do not change the state."""
    fnow = f(0.0, y)
    t = 0.0
    for h in hs:
        o = rk_step(f, y, t, h, tab, fnow)
        y = o.y_new
        t = t + h
        fnow = o.last if (tab.fsal and o.last is not None) else f(t, y)
    return y
