"""RHS + next-stage accumulation in one call (srk_rhs_combine, FlowRHS.eval_combine)
must be bitwise what the unfused srk_rhs + srk_combine produce, and the stage loop
(integrators.py:322-347) must give bitwise the same stages and y_new with and
without the fusion.  Needs a B200."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

srk = pytest.importorskip("paper_1810_10197_b200")
from paper_1810_10197_b200 import integrators  # noqa: E402


def _state(g, ncomp, seed):
    gen = torch.Generator(device="cuda").manual_seed(seed)
    y = torch.randn((ncomp,) + g.kshape, dtype=torch.complex128, device="cuda", generator=gen)
    return y * (float(np.prod(g.shape)) / torch.linalg.vector_norm(y).item())


CASES = [((32, 32, 32), False), ((16, 32, 48), False), ((64, 64, 64), False), ((256, 256, 256), False),
         ((64, 256), False), ((16, 32, 24), True), ((64, 128), True), ((1024, 1024), True), ((128, 128, 128), True)]


@pytest.mark.parametrize("shape,density", CASES)
@pytest.mark.parametrize("nt", [0, 1, 3, 6])
def test_rhs_combine_is_bitwise_rhs_then_combine(shape, density, nt):
    g = srk.Grid(shape)
    rhs = srk.FlowRHS(g, srk.PhysParams(800.0, 1.3, 0.7), density=density)
    nc = g.dims + (1 if density else 0)
    y = _state(g, nc, 1)
    yb = _state(g, nc, 2)
    Fs = [_state(g, nc, 10 + j) for j in range(nt)]
    cs = [0.013 * (j + 1) - 0.004 for j in range(nt)]
    terms = list(zip(cs, Fs))
    f_ref = rhs(0.0, y)
    yn_ref = integrators.combine(yb, terms + [(0.0271, f_ref)])
    f, yn = rhs.eval_combine(0.0, y, yb, terms, 0.0271)
    assert torch.equal(f, f_ref)
    assert torch.equal(yn, yn_ref)


def _unfused(rhs):
    return lambda t, y: rhs(t, y)  # plain callable: no eval_combine


@pytest.mark.parametrize("name", ["bs5", "rk4", "dp5", "kcl5"])
@pytest.mark.parametrize("shape", [(32, 32, 32), (128, 128, 128)])
def test_stage_loop_fused_equals_unfused(name, shape):
    g = srk.Grid(shape)
    y = srk.hit_init(g, srk.ProblemSpec("hit", a=4.0, energy=0.5, seed=42)).fields
    rhs = srk.FlowRHS(g, srk.PhysParams(1600.0))
    pair = srk.make_pair(name)
    h = 2e-3
    for first in (None, rhs(0.0, y)):
        st_a, yn_a, ev_a = integrators.run_stages(integrators._as_dev_fn(rhs), y, 0.0, h, pair, first)
        st_b, yn_b, ev_b = integrators.run_stages(_unfused(rhs), y, 0.0, h, pair, first)
        assert ev_a == ev_b
        assert torch.equal(yn_a, yn_b)
        for a, b in zip(st_a, st_b):
            assert torch.equal(a, b)


def test_adaptive_step_fused_equals_unfused_256():
    g = srk.Grid((256, 256, 256))
    y = srk.hit_init(g, srk.ProblemSpec("hit", a=4.0, energy=0.5, seed=42)).fields
    rhs = srk.FlowRHS(g, srk.PhysParams(2000.0))
    cfg = srk.ControllerConfig(tol_abs=1e-6, tol_rel=1e-6)
    f0 = rhs(0.0, y)
    outs = []
    for fn in (rhs, _unfused(rhs)):
        st = srk.ControllerState(h=1e-3)
        outs.append(srk.adaptive_advance(y, 0.0, srk.make_bs5(), st, cfg, fn, first_stage=f0, grid=g))
    a, b = outs
    assert a.h_next == b.h_next and a.errs == b.errs and a.rhs_evals == b.rhs_evals
    assert torch.equal(a.y_new, b.y_new) and torch.equal(a.last_stage, b.last_stage)


def test_rhs_combine_rejects_aliasing():
    g = srk.Grid((32, 32, 32))
    rhs = srk.FlowRHS(g, srk.PhysParams(800.0))
    y = _state(g, 3, 1)
    lib = rhs.plan.lib
    from paper_1810_10197_b200 import _native

    with pytest.raises(ValueError):  # SRK_ERR_INVALID -> ValueError (_native.check)
        f = torch.empty_like(y)
        _native.check(lib.srk_rhs_combine(rhs.plan.bind(), _native.ptr(y), _native.ptr(f), 1e-3, 1.0, 1.0,
                                          _native.ptr(y), 0, _native.ptr_array([]), _native.dbl_array([]), 0.5,
                                          _native.ptr(y), _native.stream_ptr()))


def test_forcing_with_step_energy_sum_is_bitwise_the_full_pass():
    """apply_forcing(energy_sum=AdvanceOutcome.diag_sums[4]) skips its own energy pass;
    the fused step reduction computes the same sum with the same arithmetic."""
    g = srk.Grid((64, 64, 64))
    y = srk.hit_init(g, srk.ProblemSpec("hit", a=4.0, energy=0.5, seed=42)).fields
    rhs = srk.FlowRHS(g, srk.PhysParams(2000.0))
    st = srk.ControllerState(h=1e-3)
    out = srk.adaptive_advance(y, 0.0, srk.make_bs5(), st, srk.ControllerConfig(), rhs, first_stage=rhs(0.0, y),
                               grid=g)
    a, b = out.y_new.clone(), out.y_new.clone()
    ga = srk.apply_forcing(a, g, 0.5, 2.0)
    gb = srk.apply_forcing(b, g, 0.5, 2.0, energy_sum=out.diag_sums[4])
    assert ga == gb
    assert torch.equal(a, b)


@pytest.mark.parametrize("shape,density", [((64, 64, 64), False), ((16, 32, 24), True), ((64, 128), True),
                                           ((64, 128), False), ((1024, 1024), True)])
def test_refresh_matches_separate_calls(shape, density):
    """srk_rhs_refresh: f and y + c f bitwise the separate calls, the diagnostics
    sums equal to srk_step_reduce's (different fixed summation order); 3D / 2D,
    NS / Boussinesq (sums over the velocity components)."""
    from paper_1810_10197_b200.diagnostics import reduce_sums
    from paper_1810_10197_b200.integrators import combine

    g = srk.Grid(shape)
    rhs = srk.FlowRHS(g, srk.PhysParams(700.0, 1.1, 0.9), density=density)
    if len(shape) == 3 and not density:
        y = srk.hit_init(g, srk.ProblemSpec("hit", a=4.0, energy=0.5, seed=9)).fields
    else:
        y = _state(g, g.dims + (1 if density else 0), 9)
    c = 1e-3 * 0.5
    f, y2, q = rhs.refresh(0.0, y, c)
    f_ref = rhs(0.0, y)
    assert torch.equal(f, f_ref)
    assert torch.equal(y2, combine(y, [(c, f_ref)]))
    q_ref = reduce_sums(g, y, fl=f_ref, flags=2, ncomp=g.dims, host=True).tolist()
    for k in (4, 5, 8):
        assert abs(q[k] - q_ref[k]) <= 1e-13 * abs(q_ref[k])
    assert all(q[k] == 0.0 for k in (0, 1, 2, 3, 6, 7))


def test_second_input_is_bitwise_the_stage_sum():
    """adaptive_advance(second_input=(h, y + h a21 F1)) == the unfused first stage sum."""
    g = srk.Grid((32, 32, 32))
    rhs = srk.FlowRHS(g, srk.PhysParams(900.0))
    pair = srk.make_bs5()
    cfg = srk.ControllerConfig(tol_abs=1e-6, tol_rel=1e-6)
    y = srk.hit_init(g, srk.ProblemSpec("hit", a=4.0, energy=0.5, seed=2)).fields
    h = 2e-3
    f, y2, _ = rhs.refresh(0.0, y, h * float(pair.A[1, 0]))
    a = srk.adaptive_advance(y, 0.0, pair, srk.ControllerState(h=h), cfg, rhs, first_stage=f, grid=g,
                             second_input=(h, y2))
    b = srk.adaptive_advance(y, 0.0, pair, srk.ControllerState(h=h), cfg, rhs, first_stage=f, grid=g)
    assert torch.equal(a.y_new, b.y_new) and a.h_next == b.h_next and a.rhs_evals == b.rhs_evals
