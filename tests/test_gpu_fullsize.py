"""Full-size (BASELINE config 5 grid, 512^3) checks of the drop-in RHS.

The CPU oracle cannot run at 512^3 in test time, so parity at the
benchmark size is established two ways:

* against an independent fp64 device restatement of the reference's factored
  algorithm built on torch.fft (cuFFT) -- curl (spectral.py:47-65), the 3/2-rule
  widen / narrow (spectral.py:215-304) and the projection + viscous term
  (physics.py:105-129).  It is a checker only (test infrastructure, like the
  oracle), never the product path;
* through size-independent properties of the continuous operator that the
  reference's own suite checks at small sizes (test_physics.py:72-89): a
  divergence-free tendency and an energy-neutral convective term.

Needs a B200 (about 40 GB of device memory at 512^3).
"""

import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

srk = pytest.importorskip("paper_1810_10197_b200")

N = 512
RE = 1000.0


def _kvecs(n, dev, lengths=None):
    """Wavenumbers (grid.py:75-93): full axes fftfreq with n/2 relabelled +n/2, r2c axis 0..n/2,
    times 2 pi / L.  n: an int (cube) or (n0, n1, n2)."""
    ns = (n, n, n) if isinstance(n, int) else tuple(n)
    ls = lengths or (2 * math.pi,) * 3

    def full(m):
        return torch.cat([torch.arange(0, m // 2 + 1), torch.arange(-(m // 2) + 1, 0)]).to(dev, torch.float64)

    k0 = full(ns[0]).view(-1, 1, 1) * (2 * math.pi / ls[0])
    k1 = full(ns[1]).view(1, -1, 1) * (2 * math.pi / ls[1])
    k2 = torch.arange(0, ns[2] // 2 + 1, device=dev, dtype=torch.float64).view(1, 1, -1) * (2 * math.pi / ls[2])
    return k0, k1, k2


def _widen(s, n):
    """One component: x pad (x 1.5^3) + ifft, y pad + ifft, irfft(n=m) along z (spectral.py:215-261)."""
    n0, n1, n2 = (n, n, n) if isinstance(n, int) else n
    m0, m1, m2 = 3 * n0 // 2, 3 * n1 // 2, 3 * n2 // 2
    h0, h1 = n0 // 2, n1 // 2
    kz = n2 // 2 + 1
    b = torch.zeros((m0, n1, kz), dtype=torch.complex128, device=s.device)
    b[: h0 + 1] = s[: h0 + 1] * 1.5 ** 3
    b[m0 - (h0 - 1):] = s[h0 + 1:] * 1.5 ** 3
    a = torch.fft.ifft(b, dim=0)
    del b
    b = torch.zeros((m0, m1, kz), dtype=torch.complex128, device=s.device)
    b[:, : h1 + 1] = a[:, : h1 + 1]
    b[:, m1 - (h1 - 1):] = a[:, h1 + 1:]
    del a
    b = torch.fft.ifft(b, dim=1)
    return torch.fft.irfft(b, n=m2, dim=2)


def _narrow(p, n):
    """One component: rfft along z keeping n/2+1, fft + truncation on y then x (x (1/1.5)^3),
    Nyquist rows zeroed (spectral.py:263-304)."""
    n0, n1, n2 = (n, n, n) if isinstance(n, int) else n
    m0, m1 = 3 * n0 // 2, 3 * n1 // 2
    h0, h1, kz = n0 // 2, n1 // 2, n2 // 2 + 1
    a = torch.fft.rfft(p, dim=2)[:, :, :kz]
    a = torch.fft.fft(a, dim=1)
    o = torch.zeros((m0, n1, kz), dtype=torch.complex128, device=p.device)
    o[:, :h1] = a[:, :h1]
    o[:, h1 + 1:] = a[:, m1 - (h1 - 1):]
    del a
    a = torch.fft.fft(o, dim=0)
    del o
    s = (1.0 / 1.5) ** 3
    o = torch.zeros((n0, n1, kz), dtype=torch.complex128, device=p.device)
    o[:h0] = a[:h0] * s
    o[h0 + 1:] = a[m0 - (h0 - 1):] * s
    o[:, :, kz - 1] = 0.0
    o.imag[0, 0, 0] = 0.0
    return o


def torch_ns_rhs(u, n, re, lengths=None):
    """Independent device restatement of ns_rhs (physics.py:105-129) on torch.fft."""
    k0, k1, k2 = _kvecs(n, u.device, lengths)
    ks = (k0, k1, k2)
    w = torch.empty_like(u)
    w[0] = 1j * (k1 * u[2] - k2 * u[1])
    w[1] = 1j * (k2 * u[0] - k0 * u[2])
    w[2] = 1j * (k0 * u[1] - k1 * u[0])
    U = [_widen(u[j], n) for j in range(3)]
    W = [_widen(w[j], n) for j in range(3)]
    del w
    P = [U[1] * W[2] - U[2] * W[1], U[2] * W[0] - U[0] * W[2], U[0] * W[1] - U[1] * W[0]]
    del U, W
    G = torch.stack([_narrow(P[j], n) for j in range(3)])
    del P
    kk = k0 * k0 + k1 * k1 + k2 * k2
    inv = torch.where(kk == 0.0, torch.zeros_like(kk), 1.0 / torch.where(kk == 0.0, torch.ones_like(kk), kk))
    kd = (k0 * G[0] + k1 * G[1] + k2 * G[2]) * inv
    return torch.stack([G[j] - ks[j] * kd - (kk / re) * u[j] for j in range(3)])


def _hermitian_w(n, dev):
    w = torch.full((n // 2 + 1,), 2.0, dtype=torch.float64, device=dev)
    w[0] = w[-1] = 1.0
    return w.view(1, 1, -1)


@pytest.fixture(scope="module")
def state():
    torch.cuda.set_device(0)
    gen = torch.Generator(device="cuda").manual_seed(1810)
    g = srk.Grid((N, N, N))
    # band-limited random field with a decaying spectrum, projected solenoidal
    k0, k1, k2 = _kvecs(N, "cuda")
    kk = (k0 * k0 + k1 * k1 + k2 * k2)
    amp = torch.exp(-kk / (2 * 40.0 ** 2)).to(torch.complex128)
    u = torch.randn((3, N, N, N // 2 + 1), dtype=torch.complex128, device="cuda", generator=gen) * amp
    del kk, amp
    # unnormalised spectra (rfftn convention): scale to an O(1) physical rms velocity
    # so the convective term, not the trivially exact viscous term, dominates f
    u *= float(N) ** 3 / torch.linalg.vector_norm(u).item()
    u = srk.leray_project(u, g)
    f = srk.FlowRHS(g, srk.PhysParams(RE))(0.0, u)
    torch.cuda.synchronize()
    return g, u, f


def test_rhs_512_matches_cufft_restatement(state):
    g, u, f = state
    ref = torch_ns_rhs(u, N, RE)
    rel = (torch.linalg.vector_norm(f - ref) / torch.linalg.vector_norm(ref)).item()
    # the dealiased convective part alone (viscous term added back on both sides)
    k0, k1, k2 = _kvecs(N, "cuda")
    visc = ((k0 * k0 + k1 * k1 + k2 * k2) / RE) * u
    ref += visc
    conv = f + visc
    del visc
    rel_c = (torch.linalg.vector_norm(conv - ref) / torch.linalg.vector_norm(ref)).item()
    share = (torch.linalg.vector_norm(ref) / torch.linalg.vector_norm(f)).item()
    del ref, conv
    print(f"512^3 RHS vs torch.fft restatement: rel L2 {rel:.3e}, convective part {rel_c:.3e} "
          f"(|P(u x w)| / |f| = {share:.2f})")
    assert rel <= 1e-12, f"512^3 RHS vs torch.fft restatement: rel L2 {rel:.3e}"
    assert rel_c <= 1e-12, f"512^3 convective term vs torch.fft restatement: rel L2 {rel_c:.3e}"


def test_rhs_512_is_divergence_free(state):
    g, u, f = state
    k0, k1, k2 = _kvecs(N, "cuda")
    w = _hermitian_w(N, "cuda")
    div = k0 * f[0] + k1 * f[1] + k2 * f[2]
    kmag = torch.sqrt(k0 * k0 + k1 * k1 + k2 * k2)
    num = torch.sqrt((w * div.abs() ** 2).sum()).item()
    den = torch.sqrt((w * (kmag * torch.sqrt((f.abs() ** 2).sum(0))) ** 2).sum()).item()
    print(f"512^3 |k.f| / |k||f| = {num / den:.3e}")
    assert num <= 1e-13 * den, f"|k.f| / |k||f| = {num / den:.3e}"


def test_convective_term_512_is_energy_neutral(state):
    """sum_k w Re(conj(u) . (u x w)^) = 0 for the dealiased product (test_physics.py:79-89)."""
    g, u, f = state
    k0, k1, k2 = _kvecs(N, "cuda")
    w = _hermitian_w(N, "cuda")
    kk = k0 * k0 + k1 * k1 + k2 * k2
    conv = f + (kk / RE) * u  # add the viscous term back: P(u x w)^
    num = (w * (u.conj() * conv).real.sum(0)).sum().item()
    den = math.sqrt((w * (u.abs() ** 2).sum(0)).sum().item() * (w * (conv.abs() ** 2).sum(0)).sum().item())
    print(f"512^3 energy transfer / scale = {num / den:.3e}")
    assert abs(num) <= 1e-10 * den, f"energy transfer {num:.3e} vs scale {den:.3e}"


def test_rhs_512_bitwise_repeatable(state):
    g, u, f = state
    f2 = srk.FlowRHS(g, srk.PhysParams(RE))(0.0, u)
    assert torch.equal(f, f2)


def test_refresh_512_is_bitwise_the_separate_calls(state):
    """srk_rhs_refresh at the config-5 grid: f bitwise the plain RHS, y + c f bitwise
    the stage-sum kernel, the diagnostics sums equal to the step reduction's."""
    from paper_1810_10197_b200.diagnostics import reduce_sums
    from paper_1810_10197_b200.integrators import combine

    g, u, f = state
    rhs = srk.FlowRHS(g, srk.PhysParams(RE))
    c = 1.7e-3 * 0.2
    f2, y2, q = rhs.refresh(0.0, u, c)
    assert torch.equal(f2, f)
    assert torch.equal(y2, combine(u, [(c, f)]))
    del y2, f2
    q_ref = reduce_sums(g, u, fl=f, flags=2, ncomp=3, host=True).tolist()
    for k in (4, 5, 8):
        assert abs(q[k] - q_ref[k]) <= 1e-12 * abs(q_ref[k]), (k, q[k], q_ref[k])


@pytest.mark.parametrize("shape,lengths", [((64, 128, 512), (2 * math.pi, 3.0, 5.0)),
                                           ((128, 32, 512), (1.0, 2 * math.pi, 2 * math.pi))])
def test_rhs_anisotropic_z512_matches_cufft_restatement(shape, lengths):
    """The one-pencil z-pass (M = 768) on non-cubic grids / non-2 pi boxes."""
    gen = torch.Generator(device="cuda").manual_seed(7)
    g = srk.Grid(shape, lengths)
    u = torch.randn((3,) + g.kshape, dtype=torch.complex128, device="cuda", generator=gen)
    u *= float(np.prod(shape)) / torch.linalg.vector_norm(u).item()
    f = srk.FlowRHS(g, srk.PhysParams(700.0))(0.0, u)
    ref = torch_ns_rhs(u, shape, 700.0, lengths)
    rel = (torch.linalg.vector_norm(f - ref) / torch.linalg.vector_norm(ref)).item()
    assert rel <= 1e-12, f"{shape}: rel L2 {rel:.3e}"


@pytest.mark.parametrize("shape", [(32, 48, 1024), (1024, 32, 16), (16, 1024, 32), (64, 64, 1024)])
def test_rhs_1536_axes_match_cufft_restatement(shape):
    """M = 1536 passes (the 1024^3 slab configs' lengths) on each axis vs the torch.fft restatement."""
    gen = torch.Generator(device="cuda").manual_seed(11)
    g = srk.Grid(shape)
    u = torch.randn((3,) + g.kshape, dtype=torch.complex128, device="cuda", generator=gen)
    u *= float(np.prod(shape)) / torch.linalg.vector_norm(u).item()
    f = srk.FlowRHS(g, srk.PhysParams(700.0))(0.0, u)
    ref = torch_ns_rhs(u, shape, 700.0, g.lengths)
    rel = (torch.linalg.vector_norm(f - ref) / torch.linalg.vector_norm(ref)).item()
    assert rel <= 1e-12, f"{shape}: rel L2 {rel:.3e}"
