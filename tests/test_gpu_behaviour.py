"""Device-path versions of the reference suite's physics / integrator / acceptance
checks (pkg/tests/test_physics.py, test_integrators.py, test_acceptance.py),
restated against the drop-in API.  Needs a B200."""

import numpy as np
import pytest
import torch

import oracle as O

pytestmark = pytest.mark.gpu

srk = pytest.importorskip("paper_1810_10197_b200")


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(a):
    return a.cpu().numpy() if isinstance(a, torch.Tensor) else a


def band(og, rng, ncomp=1):
    """Spectra of real fields on the retained band (reference helpers.py:90-100 idea)."""
    s = rng.standard_normal((ncomp,) + og.kshape) + 1j * rng.standard_normal((ncomp,) + og.kshape)
    O.symmetrize_planes(s, og)
    O.zero_nyquist(s, og)
    ax = tuple(range(-og.dims, 0))
    return np.fft.rfftn(np.fft.irfftn(s, s=og.shape, axes=ax), axes=ax)


def solenoidal(og, rng):
    return O.leray(band(og, rng, og.dims), og)


def div_rel(u, og):
    u = host(u)
    d = sum(og.k[j] * u[j] for j in range(og.dims))
    sc = np.sqrt(np.sum(np.abs(u[: og.dims]) ** 2 * og.w))
    return float(np.sqrt(np.sum(np.abs(d) ** 2 * og.w)) / sc) if sc else 0.0


# ---------------------------------------------------------------- physics
def test_taylor_green_2d_is_an_eigenfunction():
    g = srk.Grid((32, 32))
    u = srk.taylor_green_init(g).fields
    f = srk.FlowRHS(g, srk.PhysParams(100.0))(0.0, u)
    assert torch.allclose(f, -(2.0 / 100.0) * u, rtol=0, atol=1e-13 * float(u.abs().max()))


def test_zero_field_gives_exact_zero():
    g = srk.Grid((8, 8, 8))
    f = srk.FlowRHS(g, srk.PhysParams(50.0))(0.0, torch.zeros((3,) + g.kshape, dtype=torch.complex128,
                                                                   device="cuda"))
    assert bool((f == 0).all())


@pytest.mark.parametrize("shape", [(16, 16), (12, 12, 12), (32, 32, 32)])
def test_tendency_is_divergence_free(shape, rng):
    og = O.OGrid(shape)
    u = solenoidal(og, rng)
    f = srk.FlowRHS(srk.Grid(shape), srk.PhysParams(100.0))(0.0, dev(u))
    assert div_rel(f, og) < 1e-12


def test_convective_term_is_energy_neutral(rng):
    og = O.OGrid((16, 16, 16))
    u = solenoidal(og, rng)
    f = host(srk.FlowRHS(srk.Grid(og.shape), srk.PhysParams(75.0))(0.0, dev(u)))
    total = np.sum(og.w * np.real(u * np.conj(f)))
    diffusion = -np.sum(og.w * og.k2 * np.abs(u) ** 2) / 75.0
    assert abs(total - diffusion) < 1e-8 * abs(diffusion)


def test_single_mode_viscous_decay():
    g = srk.Grid((16, 16))
    u = torch.zeros((2,) + g.kshape, dtype=torch.complex128, device="cuda")
    u[1, 2, 0] = 1.0 - 0.5j
    u[1, -2, 0] = 1.0 + 0.5j
    f = srk.FlowRHS(g, srk.PhysParams(10.0))(0.0, u)
    assert torch.allclose(f, -(4.0 / 10.0) * u, rtol=0, atol=1e-12)


def test_boussinesq_zero_density_reduces_to_ns(rng):
    og = O.OGrid((16, 16))
    g = srk.Grid(og.shape)
    p = srk.PhysParams(100.0, richardson=2.0, prandtl=0.7)
    u = solenoidal(og, rng)
    fields = np.concatenate([u, np.zeros_like(u[:1])])
    f = host(srk.FlowRHS(g, p, density=True)(0.0, dev(fields)))
    f_ns = host(srk.FlowRHS(g, p)(0.0, dev(u)))
    assert np.allclose(f[:2], f_ns, atol=1e-12 * np.max(np.abs(f_ns)))
    assert np.max(np.abs(f[2])) < 1e-12


def test_boussinesq_pure_density_diffusion():
    g = srk.Grid((16, 16, 16))
    p = srk.PhysParams(100.0, richardson=0.0, prandtl=2.0)
    y = torch.zeros((4,) + g.kshape, dtype=torch.complex128, device="cuda")
    y[3, 1, 2, 3] = 1.0 + 1.0j
    f = host(srk.FlowRHS(g, p, density=True)(0.0, y))
    k2 = g.k2[1, 2, 3]
    assert np.isclose(f[3, 1, 2, 3], -k2 / (100.0 * 2.0) * (1.0 + 1.0j), atol=1e-14)


def test_boussinesq_uniform_density_buoyancy_at_k0():
    g = srk.Grid((16, 16))
    p = srk.PhysParams(100.0, richardson=1.5)
    y = torch.zeros((3,) + g.kshape, dtype=torch.complex128, device="cuda")
    y[2, 0, 0] = 4.0
    f = host(srk.FlowRHS(g, p, density=True)(0.0, y))
    assert np.isclose(f[1, 0, 0], -1.5 * 4.0)
    f[1, 0, 0] = 0.0
    assert np.max(np.abs(f)) < 1e-14


def test_boussinesq_single_mode_buoyancy_projection():
    g = srk.Grid((16, 16))
    y = torch.zeros((3,) + g.kshape, dtype=torch.complex128, device="cuda")
    y[2, 3, 0] = 1.0
    y[2, -3, 0] = 1.0
    f = host(srk.FlowRHS(g, srk.PhysParams(100.0, richardson=1.0), density=True)(0.0, y))
    assert np.isclose(f[1, 3, 0], -1.0) and np.isclose(f[0, 3, 0], 0.0, atol=1e-14)


def test_boussinesq_velocity_tendency_divergence_free(rng):
    og = O.OGrid((12, 12, 12))
    y = np.concatenate([solenoidal(og, rng), band(og, rng)])
    f = srk.FlowRHS(srk.Grid(og.shape), srk.PhysParams(200.0), density=True)(0.0, dev(y))
    assert div_rel(f[:3], og) < 1e-12


def test_flowrhs_repeatable_bitwise(rng):
    og = O.OGrid((16, 16, 16))
    rhs = srk.FlowRHS(srk.Grid(og.shape), srk.PhysParams(100.0))
    u = dev(solenoidal(og, rng))
    first = rhs(0.0, u).clone()
    rhs(0.0, dev(solenoidal(og, rng)))
    assert torch.equal(rhs(0.0, u), first)


# ---------------------------------------------------------------- forcing
def _hit(g, seed=7, energy=1.0):
    return srk.hit_init(g, srk.ProblemSpec("hit", seed=seed, energy=energy)).fields


def test_forcing_restores_target_energy():
    g = srk.Grid((16, 16, 16))
    u = _hit(g) * 0.9
    before = srk.kinetic_energy(u, g)
    gamma = srk.apply_forcing(u, g, target_energy=1.0, k_f=2.0)
    assert gamma > 1.0
    assert np.isclose(srk.kinetic_energy(u, g), 1.0, rtol=1e-12) and srk.kinetic_energy(u, g) > before


def test_forcing_only_scales_the_band():
    g = srk.Grid((16, 16, 16))
    u = _hit(g)
    u0 = u.clone()
    srk.apply_forcing(u, g, target_energy=1.05, k_f=2.0)
    bandm = torch.from_numpy((g.k2 > 0) & (g.k2 <= 4.0 * (1 + 1e-12))).cuda()
    assert torch.equal(u[:, ~bandm], u0[:, ~bandm])
    assert not torch.equal(u[:, bandm], u0[:, bandm])


def test_forcing_errors():
    g = srk.Grid((16, 16, 16))
    u = torch.zeros((3,) + g.kshape, dtype=torch.complex128, device="cuda")
    u[0, 0, 0, 5] = 1.0
    u[1, 0, 0, 5] = 1.0
    with pytest.raises(srk.ForcingError):
        srk.apply_forcing(u, g, target_energy=1.0, k_f=2.0)
    u = _hit(g)
    with pytest.raises(srk.ForcingError):
        srk.apply_forcing(u, g, target_energy=1e-6, k_f=2.0)


def test_forcing_matches_oracle():
    g = srk.Grid((16, 16, 16))
    og = O.OGrid((16, 16, 16))
    u = _hit(g) * 0.8
    un = host(u).copy()
    gd = srk.apply_forcing(u, g, 1.0, 2.0)
    go = O.apply_forcing(un, og, 1.0, 2.0)
    assert abs(gd - go) <= 1e-14 * go
    assert np.abs(host(u) - un).max() <= 1e-15 * np.abs(un).max()


def test_forcing_numpy_in_place_like_reference():
    """physics.py:209-239 rescales a numpy array in place: same gamma and band as
    the device path, the caller's array updated."""
    g = srk.Grid((16, 16, 16))
    og = O.OGrid((16, 16, 16))
    un = host(_hit(g) * 0.8).copy()
    ref = un.copy()
    go = O.apply_forcing(ref, og, 1.0, 2.0)
    gd = srk.apply_forcing(un, g, 1.0, 2.0)
    assert abs(gd - go) <= 1e-14 * go
    assert np.abs(un - ref).max() <= 1e-15 * np.abs(ref).max()


# ---------------------------------------------------------------- rk_step known answers
def _ode_state(val):
    return torch.full((1, 4, 4, 3), val, dtype=torch.complex128, device="cuda")


def test_rk4_integrates_a_cubic_exactly():
    f = lambda t, y: torch.full_like(y, 3.0 * t * t)
    out = srk.rk_step(f, _ode_state(0.0), 0.0, 2.0, srk.make_rk4())
    assert torch.allclose(out.y_new, _ode_state(8.0), rtol=0, atol=1e-13)


@pytest.mark.parametrize("name", ["rk4", "dp5", "bs5", "kcl5"])
def test_complex_linear_ode_matches_oracle(name, rng):
    lam = -0.7 + 2.0j
    f = lambda t, y: lam * y
    y0 = rng.standard_normal((1, 4, 4, 3)) + 1j * rng.standard_normal((1, 4, 4, 3))
    out = srk.rk_step(f, dev(y0), 0.0, 0.05, srk.make_pair(name))
    ref = O.rk_step(lambda t, y: lam * y, y0, 0.0, 0.05, O.tableau(name))
    assert np.abs(host(out.y_new) - ref.y_new).max() <= 1e-15 * np.abs(ref.y_new).max()
    assert np.abs(host(out.y_new) - y0 * np.exp(lam * 0.05)).max() < 1e-6  # O((lam h)^5) local error
    if ref.err_vec is not None:
        assert np.abs(host(out.error_vector) - ref.err_vec).max() <= 1e-15


def test_first_stage_reuse_and_fsal():
    calls = []

    def f(t, y):
        calls.append(t)
        return -y

    y0 = _ode_state(1.0)
    p = srk.make_bs5()
    out = srk.rk_step(f, y0, 0.0, 0.1, p)
    assert out.rhs_evals == 8 and out.last_stage is not None
    assert torch.allclose(out.last_stage, -out.y_new, rtol=0, atol=1e-15)  # FSAL: f(y_new)
    calls.clear()
    out2 = srk.rk_step(f, out.y_new, 0.1, 0.1, p, first_stage=out.last_stage)
    assert out2.rhs_evals == 7 and len(calls) == 7


def test_nonfinite_step_raises():
    f = lambda t, y: y * float("nan")
    with pytest.raises(srk.NonFiniteStateError):
        srk.rk_step(f, _ode_state(1.0), 0.0, 0.1, srk.make_rk4())


# ---------------------------------------------------------------- acceptance
def test_invariants_over_200_adaptive_bs5_steps():
    """test_acceptance.py:198-246 on the device path (32^3 TG, Re = 280)."""
    g = srk.Grid((32, 32, 32))
    og = O.OGrid((32, 32, 32))
    rhs = srk.FlowRHS(g, srk.PhysParams(280.0))
    pair = srk.make_bs5()
    cfg = srk.ControllerConfig(tol_abs=1e-6, tol_rel=1e-6)
    st = srk.ControllerState(h=1e-3)
    y = srk.taylor_green_init(g).fields
    t = 0.0
    f_now = rhs(t, y)
    worst_div = worst_neu = worst_probe = 0.0
    kmax = np.sqrt(og.k2.max())
    for _ in range(200):
        out = srk.adaptive_advance(y, t, pair, st, cfg, rhs, first_stage=f_now, grid=g)
        y, t = out.y_new, out.t_new
        f_now = out.last_stage
        yh, fh = host(y), host(f_now)
        kdu = sum(og.k[j] * yh[j] for j in range(3))
        worst_div = max(worst_div, np.max(np.abs(kdu)) / (kmax * np.max(np.abs(yh))))
        total = sum(float(np.sum(og.w * (yh[j] * np.conj(fh[j])).real)) for j in range(3))
        diff = -sum(float(np.sum(og.w * og.k2 * np.abs(yh[j]) ** 2)) for j in range(3)) / 280.0
        worst_neu = max(worst_neu, abs(total - diff) / abs(diff))
        eps = srk.dissipation_rate(y, f_now, g)
        d = 1e-3
        fd = (srk.kinetic_energy(y + d * f_now, g) - srk.kinetic_energy(y - d * f_now, g)) / (2 * d)
        worst_probe = max(worst_probe, abs(fd + eps) / abs(eps))
    assert worst_div <= 1e-11 and worst_neu <= 1e-8 and worst_probe <= 1e-6


# ---------------------------------------------------------------- host-resident state (hostio)
@pytest.mark.parametrize("chunk_bytes", [1 << 30, 48 * 1024])
def test_host_mirror_loop_is_bitwise_the_device_loop(chunk_bytes):
    """Forced-HIT BS5 steps with the state kept on the host (HostMirror: y_new pushed
    before its FSAL stage, forcing planes re-sent, chunked pull) == the device-resident
    loop, bit for bit; h0 = 0.5 forces rejected attempts (each pushes again)."""
    g = srk.Grid((32, 32, 32))
    rhs = srk.FlowRHS(g, srk.PhysParams(2000.0))
    pair = srk.make_bs5()
    cfg = srk.ControllerConfig(tol_abs=1e-6, tol_rel=1e-6)
    y0 = _hit(g, seed=42, energy=0.5)
    planes = srk.forcing_planes(g, 2.0)

    def run(host_state):
        st = srk.ControllerState(h=0.5)
        t, y, pushes, rej = 0.0, y0.clone(), [], 0
        m, spec = None, {}
        if host_state:
            m = srk.HostMirror(y, chunk_bytes=chunk_bytes)
            m.load_host(y.cpu())
            y = m.pull()

        def hook(v):  # every attempt: push y_new, pull it back as the next input (speculative)
            pushes.append(1)
            m.push(v)
            spec["next"] = m.pull(wait=False)

        hist = []
        for _ in range(4):
            f = rhs(t, y)
            out = srk.adaptive_advance(y, t, pair, st, cfg, rhs, first_stage=f, grid=g,
                                       on_y_new=hook if host_state else None)
            srk.apply_forcing(out.y_new, g, 0.5, 2.0, energy_sum=out.diag_sums[4])
            rej += out.rejections
            t, y = out.t_new, out.y_new
            if host_state:
                m.push(out.y_new, planes=planes)
                y = m.pull(into=spec.pop("next"), planes=planes)
            hist.append((out.h_used, out.h_next))
        if host_state:
            m.synchronize()
            assert torch.equal(y.cpu(), m.host)  # the pulled input is the host copy
            return m.host.clone(), hist, len(pushes), rej
        return y.cpu(), hist, None, rej

    yh, hh, pushes, rej = run(True)
    yd, hd, _, rej_d = run(False)
    assert rej >= 1 and rej == rej_d
    assert pushes == 4 + rej  # one push per attempt
    assert hh == hd
    assert torch.equal(yh, yd)


def test_host_mirror_rejects_mismatched_tensors():
    m = srk.HostMirror(torch.zeros((2, 4, 4, 3), dtype=torch.complex128, device="cuda"))
    with pytest.raises(ValueError):
        m.push(torch.zeros((2, 4, 4, 2), dtype=torch.complex128, device="cuda"))
    with pytest.raises(TypeError):
        srk.HostMirror(torch.zeros(3))


@pytest.mark.gpu
def test_nvtx_ranges_wrap_rhs_calls(monkeypatch):
    """With SRK_NVTX on, RHS calls and attempts run inside NVTX ranges and give the same results."""
    from paper_1810_10197_b200 import _native

    g = srk.Grid((32, 32, 32))
    rhs = srk.FlowRHS(g, srk.PhysParams(1000.0))
    y = srk.hit_init(g, srk.ProblemSpec("hit", a=4.0, energy=0.5, seed=3)).fields
    f0 = rhs(0.0, y)
    monkeypatch.setattr(_native, "NVTX", True)
    f1 = rhs(0.0, y)
    out = srk.adaptive_advance(y, 0.0, srk.make_bs5(), srk.ControllerState(h=1e-3), srk.ControllerConfig(), rhs, grid=g)
    torch.cuda.synchronize()
    assert torch.equal(f0, f1) and out.rhs_evals >= 7


@pytest.mark.gpu
@pytest.mark.parametrize("shape, pitch, yblock", [
    ((512, 512, 512), 260, 64),   # x rows of 2.1 MB: y-blocked; K = 257 -> 260
    ((256, 256, 256), 132, 0),    # x rows of 528 KB: plain order; K = 129 -> 132
    ((128, 128, 128), 65, 0),     # short rows: reference pitch
    ((64, 512, 256), 132, 64),    # anisotropic: n1 * K * 16 B = 1 MB
    ((1024, 1024), 516, 0),       # 2D: pitch only
    ((16, 12, 10), 6, 0),         # runtime (generic) FFT plan: reference layout
])
def test_plan_layout_of_the_intermediates(shape, pitch, yblock):
    """srk_plan_layout: sector-aligned pitch for n_last >= 256 on the compile-time plans, y-blocked
    x-pass buffers once a plain x row reaches 1 MB."""
    import ctypes

    from paper_1810_10197_b200.spectral import get_plan

    pl = get_plan(srk.Grid(shape), density=False)
    kp, yb = ctypes.c_int(-1), ctypes.c_int(-1)
    assert pl.lib.srk_plan_layout(pl.h, ctypes.byref(kp), ctypes.byref(yb)) == 0
    assert (kp.value, yb.value) == (pitch, yblock)


@pytest.mark.gpu
def test_layout_switches_do_not_change_results(tmp_path):
    """SRK_KPAD=0 / SRK_YB=0 (reference pitch / plain order of the RHS intermediates) run the
    same arithmetic as the default sector-aligned, y-blocked layout: bitwise equal tendencies
    (the switches are read once per process, hence subprocesses)."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import sys, numpy as np, torch; sys.path.insert(0, %r)\n"
        "import paper_1810_10197_b200 as srk\n"
        "g = srk.Grid((64, 512, 256))\n"          # x rows of 1 MB: y-blocked by default, K = 129 -> 132
        "torch.manual_seed(7)\n"
        "y = torch.randn((3,) + g.kshape, dtype=torch.complex128, device='cuda')\n"
        "f = srk.FlowRHS(g, srk.PhysParams(500.0))(0.0, y)\n"
        "np.save(sys.argv[1], f.cpu().numpy())\n" % root
    )
    outs = []
    for name, env in (("default", {}), ("nopad", {"SRK_KPAD": "0"}), ("noyb", {"SRK_YB": "0"}),
                      ("plain", {"SRK_KPAD": "0", "SRK_YB": "0"})):
        out = str(tmp_path / f"{name}.npy")
        subprocess.run([sys.executable, "-c", code, out], check=True, env={**os.environ, **env}, timeout=300)
        outs.append(np.load(out))
    assert np.isfinite(outs[0]).all() and np.abs(outs[0]).max() > 0
    for o in outs[1:]:
        assert np.array_equal(outs[0], o)
