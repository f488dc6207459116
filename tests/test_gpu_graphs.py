"""CUDA-graph replay of adaptive attempts (graphs.py) is bit-identical to the
eager stepping loop: same records (t, h, E, eps, evaluation / rejection counts)
and the same final field, including runs with rejections (eager retries) and the
clamped final step; and the step-size-scaled entry points equal the host products."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

srk = pytest.importorskip("paper_1810_10197_b200")


def _records(res):
    return np.array([[r.t, r.h, r.e_kin, r.eps, r.enstrophy, r.rhs_evals, r.rejections] for r in res.records])


def _both(cfg, **kw):
    r0 = srk.run_simulation(cfg, graphs=False, **kw)
    r1 = srk.run_simulation(cfg, graphs=True, **kw)
    return r0, r1


@pytest.mark.parametrize("shape,kind,re,t_end,tol,h0", [
    ((32, 32, 32), "taylor_green", 1600.0, 1.0, 1e-6, 1e-3),      # config 1
    ((16, 16, 16), "hit", 1000.0, 0.2, 1e-6, 0.5),                # oversized h0: rejections
    ((64, 256), "rayleigh_taylor", 3000.0, 0.3, 1e-7, 1e-3),      # 2D Boussinesq
])
def test_graph_replay_bit_identical(shape, kind, re, t_end, tol, h0):
    lengths = srk.default_lengths(kind, shape)
    spec = srk.ProblemSpec(kind, params=srk.PhysParams(re), seed=3, a=4.0, energy=0.5)
    cfg = srk.RunConfig(grid_shape=shape, problem=spec, integrator="bs5", mode="adaptive", t_end=t_end,
                        tol_abs=tol, tol_rel=tol, h0=h0, lengths=lengths)
    r0, r1 = _both(cfg)
    assert r1.steps == r0.steps and r1.rhs_evals == r0.rhs_evals and r1.rejections == r0.rejections
    assert np.array_equal(_records(r0), _records(r1))
    assert torch.equal(r0.state.fields, r1.state.fields)
    if h0 == 0.5:
        assert r0.rejections > 0


def test_scaled_entry_points_equal_host_products():
    from paper_1810_10197_b200 import _native
    from paper_1810_10197_b200.integrators import combine

    rng = np.random.default_rng(4)
    shape = (3, 16, 16, 9)
    y, F0, F1 = (torch.from_numpy(rng.standard_normal(shape) + 1j * rng.standard_normal(shape)).cuda()
                 for _ in range(3))
    h = 0.0123456789
    a = [0.2, -0.4375]
    ref = combine(y, [(h * a[0], F0), (h * a[1], F1)])
    hd = torch.tensor([h], dtype=torch.float64, device="cuda")
    out = torch.empty_like(y)
    lib = _native.load()
    _native.check(lib.srk_combine_scaled(y.numel(), _native.ptr(y), 2, _native.ptr_array([F0, F1]),
                                         _native.dbl_array(a), _native.ptr(hd), _native.ptr(out),
                                         _native.stream_ptr()), "srk_combine_scaled")
    assert torch.equal(out, ref)


@pytest.mark.parametrize("shape,kind,integ,h,t_end", [
    ((32, 32, 32), "taylor_green", "rk4", 0.01, 0.305),   # config 1 RK4, uneven tail step
    ((64, 256), "rayleigh_taylor", "rk4", 2e-3, 0.05),    # 2D Boussinesq (config 4 family)
    ((16, 16, 16), "hit", "dp5", 0.02, 0.1),               # FSAL pair on fixed steps
])
def test_fixed_step_graph_bit_identical(shape, kind, integ, h, t_end):
    lengths = srk.default_lengths(kind, shape)
    spec = srk.ProblemSpec(kind, params=srk.PhysParams(1000.0), seed=5, a=4.0, energy=0.5)
    cfg = srk.RunConfig(grid_shape=shape, problem=spec, integrator=integ, mode="fixed", t_end=t_end, h=h,
                        lengths=lengths)
    r0, r1 = _both(cfg)
    assert r1.steps == r0.steps and r1.rhs_evals == r0.rhs_evals
    assert np.array_equal(_records(r0), _records(r1))
    assert torch.equal(r0.state.fields, r1.state.fields)
