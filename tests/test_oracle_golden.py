"""Pin the CPU oracle (oracle/spectral_np.py) to golden vectors produced by the
reference itself (oracle/make_golden.py).  CPU-only."""

import numpy as np
import pytest

import oracle as O
from conftest import load_golden


def rel(a, b):
    return float(np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-300))


RHS = load_golden("rhs_cases")


@pytest.mark.parametrize("case", sorted(RHS))
def test_oracle_rhs_matches_reference(case):
    c = RHS[case]
    g = O.OGrid(tuple(c["shape"]), tuple(c["lengths"]))
    f = O.OracleRHS(g, float(c["re"]), float(c["ri"]), float(c["pr"]), bool(c["density"]))(0.0, c["y"])
    assert rel(f, c["f"]) <= 1e-14


DEAL = load_golden("dealias_cases")


@pytest.mark.parametrize("case", sorted(DEAL))
def test_oracle_widen_narrow_match_reference(case):
    c = DEAL[case]
    g = O.OGrid(tuple(c["shape"]))
    dl = O.Dealias(g)
    assert rel(dl.widen(c["spec"]), c["phys"]) <= 1e-14
    assert rel(dl.narrow(c["pin"]), c["narrow"]) <= 1e-14


def test_oracle_ics_match_reference():
    ic = load_golden("ics")
    g = O.OGrid((16, 16, 16))
    assert np.array_equal(O.hit(g, a=4.0, energy=0.5, seed=42), ic["hit16_a4_s42"])
    assert rel(O.taylor_green(g), ic["tg16"]) <= 1e-15
    shape = (16, 64)
    g = O.OGrid(shape, (2 * np.pi, 2 * np.pi * 64 / 16))
    assert rel(O.rayleigh_taylor(g), ic["rt16x64"]) <= 1e-15


TRAJ = load_golden("trajectories")


def _check_traj(y, recs, gold, tol_y=1e-12, tol_rec=1e-10):
    rec = np.array([[r.t, r.h, r.e_kin, r.eps, r.evals, r.rejections] for r in recs])
    assert rec.shape == gold["rec"].shape
    assert np.array_equal(rec[:, 4:], gold["rec"][:, 4:])  # eval / rejection accounting
    np.testing.assert_allclose(rec[:, :4], gold["rec"][:, :4], rtol=tol_rec, atol=0)
    assert rel(y, gold["y"]) <= tol_y


def test_oracle_c1_rk4_trajectory():
    g = O.OGrid((32, 32, 32))
    f = O.OracleRHS(g, 1600.0)
    y, recs = O.run_fixed(f, O.taylor_green(g), g, O.tableau("rk4"), 0.01, 1.0)
    _check_traj(y, recs, TRAJ["c1_rk4"])


def test_oracle_c1_bs5_trajectory():
    g = O.OGrid((32, 32, 32))
    f = O.OracleRHS(g, 1600.0)
    y, recs, _ = O.run_adaptive(f, O.taylor_green(g), g, O.tableau("bs5"), O.Ctrl(), 1e-3, 1.0)
    _check_traj(y, recs, TRAJ["c1_bs5"])


def test_oracle_bs5_with_rejections():
    g = O.OGrid((16, 16, 16))
    f = O.OracleRHS(g, 1000.0)
    y0 = O.hit(g, a=4.0, energy=0.5, seed=3)
    y, recs, errs = O.run_adaptive(f, y0, g, O.tableau("bs5"), O.Ctrl(), 0.5, 0.2)
    assert recs[-1].rejections > 0
    _check_traj(y, recs, TRAJ["hit16_bs5_rej"])


def test_oracle_forced_hit():
    g = O.OGrid((16, 16, 16))
    f = O.OracleRHS(g, 2000.0)
    y0 = O.hit(g, a=4.0, energy=0.5, seed=5)
    y, recs, _ = O.run_adaptive(f, y0, g, O.tableau("bs5"), O.Ctrl(), 1e-3, 0.05, forcing=(0.5, 2.0))
    _check_traj(y, recs, TRAJ["hit16_forced"])


def test_oracle_rt2d_rk4():
    shape = (16, 64)
    g = O.OGrid(shape, (2 * np.pi, 2 * np.pi * 64 / 16))
    f = O.OracleRHS(g, 1600.0, density=True)
    y, recs = O.run_fixed(f, O.rayleigh_taylor(g), g, O.tableau("rk4"), 0.01, 0.2)
    _check_traj(y, recs, TRAJ["rt2d_rk4"])


def test_enstrophy_consistent_with_eps():
    # D2: for pure NS the convective term is energy neutral, so eps = 2 nu Z
    g = O.OGrid((16, 16, 16))
    y = O.hit(g, a=4.0, energy=0.5, seed=1)
    re = 500.0
    f = O.OracleRHS(g, re)(0.0, y)
    eps = O.dissipation_rate(y, f, g)
    assert abs(eps - 2.0 / re * O.enstrophy(y, g)) <= 1e-8 * abs(eps)


R2 = load_golden("r2_cases")


def test_oracle_ab2_tg_with_uneven_tail():
    """AB2 (simulation.py:274-310): RK4 bootstrap, AB2 steps, RK4 restart on the tail."""
    g = O.OGrid((32, 32, 32))
    y, recs = O.run_ab2(O.OracleRHS(g, 1600.0), O.taylor_green(g), g, 0.01, 0.105)
    _check_traj(y, recs, R2["ab2_tg32"])


def test_oracle_ab2_rt2d():
    shape = (16, 64)
    g = O.OGrid(shape, (2 * np.pi, 2 * np.pi * 64 / 16))
    y, recs = O.run_ab2(O.OracleRHS(g, 1600.0, density=True), O.rayleigh_taylor(g), g, 0.01, 0.2)
    _check_traj(y, recs, R2["ab2_rt2d"])


def test_oracle_ab2_update_is_the_reference_expression(rng):
    y, fc, fp = (rng.standard_normal((3, 8, 5)) + 1j * rng.standard_normal((3, 8, 5)) for _ in range(3))
    assert np.array_equal(O.ab2_combine(y, 0.013, fc, fp), y + 0.013 * (1.5 * fc - 0.5 * fp))


def test_oracle_rt3d_rhs():
    c = R2["rt3d_rhs"]
    g = O.OGrid(tuple(c["shape"]), tuple(c["lengths"]))
    f = O.OracleRHS(g, 800.0, ri=1.0, pr=0.7, density=True)(0.0, c["y"])
    assert rel(f, c["f"]) <= 1e-14


def test_oracle_rt3d_rk4_and_bs5_windows():
    shape = (32, 32, 64)
    g = O.OGrid(shape, (2 * np.pi, 2 * np.pi, 4 * np.pi))
    f = O.OracleRHS(g, 1600.0, density=True)
    y, recs = O.run_fixed(f, O.rayleigh_taylor(g), g, O.tableau("rk4"), 0.01, 0.05)
    _check_traj(y, recs, R2["rt3d_rk4"])
    y, recs, _ = O.run_adaptive(f, O.rayleigh_taylor(g), g, O.tableau("bs5"), O.Ctrl(), 1e-3, 0.3)
    _check_traj(y, recs, R2["rt3d_bs5"])
