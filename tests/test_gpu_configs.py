"""BASELINE.json configurations on the device path vs the CPU oracle, in
windows the oracle finishes in seconds to minutes.  Initial
states come from the oracle and enter through the IC hook
(run_simulation(initial_state=...)); adaptive runs use the
accepted-step cap (max_steps).

Bars (north_star): fields <= 1e-10 relative L2; t, h, E_kin, eps, enstrophy
histories <= 1e-9 relative; evaluation / rejection counts exact."""

import numpy as np
import pytest
import torch

import oracle as O

pytestmark = pytest.mark.gpu

srk = pytest.importorskip("paper_1810_10197_b200")


def rel(a, b):
    a = a.cpu().numpy() if isinstance(a, torch.Tensor) else np.asarray(a)
    return float(np.linalg.norm((a - b).ravel()) / np.linalg.norm(np.asarray(b).ravel()))


def compare(res, y_ref, recs_ref, tol_f=1e-10, tol_r=1e-9):
    mine = np.array([[r.t, r.h, r.e_kin, r.eps, r.enstrophy] for r in res.records])
    ref = np.array([[r.t, r.h, r.e_kin, r.eps, r.ens] for r in recs_ref])
    assert mine.shape == ref.shape
    assert [r.rhs_evals for r in res.records] == [r.evals for r in recs_ref]
    assert [r.rejections for r in res.records] == [r.rejections for r in recs_ref]
    np.testing.assert_allclose(mine, ref, rtol=tol_r, atol=1e-300)
    assert rel(res.state.fields, y_ref) <= tol_f


def cfg(shape, kind, re, integ, mode, t_end, lengths=None, a=9.5, energy=1.0, **kw):
    spec = srk.ProblemSpec(kind=kind, params=srk.PhysParams(re), seed=42, a=a, energy=energy)
    c = srk.RunConfig(grid_shape=shape, problem=spec, integrator=integ, mode=mode, t_end=t_end, lengths=lengths)
    for k, v in kw.items():
        setattr(c, k, v)
    return c


# C2: Taylor-Green 128^3, nu = 1/1600 -- RK4 h = 1e-3 and BS5 tol 1e-7 (windows)
def test_c2_tg128_rk4_window():
    og = O.OGrid((128,) * 3)
    y0 = O.taylor_green(og)
    y_ref, recs = O.run_fixed(O.OracleRHS(og, 1600.0), y0, og, O.tableau("rk4"), 1e-3, 2.0, max_steps=5)
    res = srk.run_simulation(cfg((128,) * 3, "taylor_green", 1600.0, "rk4", "fixed", 2.0, h=1e-3),
                             initial_state=y0, max_steps=5)
    compare(res, y_ref, recs)


def test_c2_tg128_bs5_window():
    og = O.OGrid((128,) * 3)
    y0 = O.taylor_green(og)
    y_ref, recs, _ = O.run_adaptive(O.OracleRHS(og, 1600.0), y0, og, O.tableau("bs5"),
                                    O.Ctrl(tol_abs=1e-7, tol_rel=1e-7), 1e-3, 2.0, max_steps=2)
    res = srk.run_simulation(cfg((128,) * 3, "taylor_green", 1600.0, "bs5", "adaptive", 2.0, tol_abs=1e-7,
                                 tol_rel=1e-7), initial_state=y0, max_steps=2)
    compare(res, y_ref, recs)


# C3: decaying HIT 256^3, a = 4, E = 0.5, nu = 1e-3, BS5 tol 1e-6 (1 accepted step vs oracle)
def test_c3_hit256_bs5_one_step():
    og = O.OGrid((256,) * 3)
    y0 = O.hit(og, a=4.0, energy=0.5, seed=42)
    y_ref, recs, _ = O.run_adaptive(O.OracleRHS(og, 1000.0), y0, og, O.tableau("bs5"), O.Ctrl(), 1e-3, 1e9,
                                    max_steps=1)
    res = srk.run_simulation(cfg((256,) * 3, "hit", 1000.0, "bs5", "adaptive", 1e9, a=4.0, energy=0.5),
                             initial_state=y0, max_steps=1)
    compare(res, y_ref, recs)


def test_c3_two_gpu_slab_equals_one_gpu():
    """C3 on 2 ranks (slab kernels, emulated exchange on one GPU) vs the unsplit RHS,
    through 3 accepted BS5 steps (SURVEY §8e transitive pinning)."""
    from paper_1810_10197_b200.slab import CudaSlabBackend, scatter_slab

    g = srk.Grid((256,) * 3)
    y0 = srk.hit_init(g, srk.ProblemSpec("hit", a=4.0, energy=0.5, seed=42)).fields
    P = 2
    params = srk.PhysParams(1000.0)
    backs = [CudaSlabBackend(g, params, r, P) for r in range(P)]
    from paper_1810_10197_b200.slab import slab_geometry

    geo = slab_geometry(g, P)

    def slab_rhs(t, y):  # y: full field; run the P slab pipelines with emulated all-to-alls
        ys = [scatter_slab(y, r, P) for r in range(P)]
        s1 = [b.empty(geo["send1"]) for b in backs]
        for r in range(P):
            backs[r].forward(ys[r], s1[r])
        blk = geo["send1"] // P
        r1 = [torch.cat([s1[q][r * blk:(r + 1) * blk] for q in range(P)]) for r in range(P)]
        s2 = [b.empty(geo["send2"]) for b in backs]
        for r in range(P):
            backs[r].middle(r1[r], s2[r])
        blk = geo["send2"] // P
        r2 = [torch.cat([s2[q][r * blk:(r + 1) * blk] for q in range(P)]) for r in range(P)]
        fs = [torch.empty_like(ys[r]) for r in range(P)]
        for r in range(P):
            backs[r].finish(r2[r], ys[r], fs[r])
        return torch.cat(fs, dim=2).contiguous()

    pair, ctrl_cfg = srk.make_bs5(), srk.ControllerConfig()
    one = srk.FlowRHS(g, params)
    ya, yb = y0.clone(), y0.clone()
    sa, sb = srk.ControllerState(h=1e-3), srk.ControllerState(h=1e-3)
    fa, fb = one(0.0, ya), slab_rhs(0.0, yb)
    ta = tb = 0.0
    for _ in range(3):
        oa = srk.adaptive_advance(ya, ta, pair, sa, ctrl_cfg, one, first_stage=fa, grid=g)
        ob = srk.adaptive_advance(yb, tb, pair, sb, ctrl_cfg, slab_rhs, first_stage=fb, grid=g)
        ya, fa, ta = oa.y_new, oa.last_stage, oa.t_new
        yb, fb, tb = ob.y_new, ob.last_stage, ob.t_new
        assert abs(oa.h_used - ob.h_used) <= 1e-12 * oa.h_used and oa.rhs_evals == ob.rhs_evals
    assert rel(yb, ya.cpu().numpy()) <= 1e-12


# C4: 2D Boussinesq Rayleigh-Taylor 1024^2, tanh interface + seeded perturbation
def _c4():
    shape = (1024, 1024)
    og = O.OGrid(shape)
    return og, O.rt_tanh_ic(og, width=0.05, amp=1e-3, kmax=8, seed=4)


def test_c4_rt1024_bs5_window():
    og, y0 = _c4()
    f = O.OracleRHS(og, 1e4, ri=1.0, pr=1.0, density=True)
    y_ref, recs, _ = O.run_adaptive(f, y0, og, O.tableau("bs5"), O.Ctrl(), 1e-3, 10.0, max_steps=3)
    c = cfg((1024, 1024), "rayleigh_taylor", 1e4, "bs5", "adaptive", 10.0, lengths=og.lengths)
    c.problem.params = srk.PhysParams(1e4, 1.0, 1.0)
    res = srk.run_simulation(c, initial_state=y0, max_steps=3)
    compare(res, y_ref, recs)


def test_c4_rt1024_rk4_window():
    og, y0 = _c4()
    f = O.OracleRHS(og, 1e4, ri=1.0, pr=1.0, density=True)
    y_ref, recs = O.run_fixed(f, y0, og, O.tableau("rk4"), 2e-3, 10.0, max_steps=3)
    c = cfg((1024, 1024), "rayleigh_taylor", 1e4, "rk4", "fixed", 10.0, lengths=og.lengths, h=2e-3)
    c.problem.params = srk.PhysParams(1e4, 1.0, 1.0)
    res = srk.run_simulation(c, initial_state=y0, max_steps=3)
    compare(res, y_ref, recs)


# C5: forced HIT (energy-restoring forcing on 0 < |k| <= 2, nu = 5e-4, BS5 tol 1e-6)
# at 64^3 (no CPU oracle exists at 1024^3)
def test_c5_forced_hit64_window():
    og = O.OGrid((64,) * 3)
    y0 = O.hit(og, a=4.0, energy=0.5, seed=42)
    y_ref, recs, _ = O.run_adaptive(O.OracleRHS(og, 2000.0), y0, og, O.tableau("bs5"), O.Ctrl(), 1e-3, 1e9,
                                    max_steps=5, forcing=(0.5, 2.0))
    c = cfg((64,) * 3, "hit", 2000.0, "bs5", "adaptive", 1e9, a=4.0, energy=0.5, forcing=True, k_f=2.0)
    res = srk.run_simulation(c, initial_state=y0, max_steps=5)
    compare(res, y_ref, recs)


def test_c4_rt_tanh_init_matches_oracle():
    """The product's config-4 IC generator (device transforms) vs the oracle's restatement."""
    og, y0 = _c4()
    st = srk.rt_tanh_init(srk.Grid((1024, 1024)), width=0.05, amp=1e-3, kmax=8, seed=4)
    assert rel(st.fields, y0) <= 1e-13
