"""Round-2 parity pins on the B200:

* AB2 (integrators.py:361-381, simulation.py:274-310): the device update in the
  reference's association (bitwise numpy's rounding), and AB2 runs through the
  drop-in driver vs trajectories the reference itself wrote (uneven tail step
  with the RK4 restart; a 2D Boussinesq run with density in the update);
* 3D Boussinesq (physics.py:132-185) at the fast-plan sizes (the 6-signal K1,
  the 7-column z-pass ZOP_B3) vs the oracle at M = 48 ... 384, a Rayleigh-Taylor
  state with z-Nyquist content vs the reference's own RHS, and 3D RT RK4 / BS5
  windows vs the reference driver.

Bars (north_star): one evaluation <= 1e-12 relative L2; trajectories: fields
<= 1e-10, t / h / E / eps <= 1e-9 relative, evaluation and rejection counts exact.
"""

import numpy as np
import pytest
import torch

import oracle as O
from conftest import load_golden

pytestmark = pytest.mark.gpu

srk = pytest.importorskip("paper_1810_10197_b200")

R2 = load_golden("r2_cases")


def rel(a, b):
    a = a.cpu().numpy() if isinstance(a, torch.Tensor) else np.asarray(a)
    b = b.cpu().numpy() if isinstance(b, torch.Tensor) else np.asarray(b)
    return float(np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-300))


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _check_records(res, gold, tol=1e-9):
    rec = np.array([[r.t, r.h, r.e_kin, r.eps, r.rhs_evals, r.rejections] for r in res.records])
    assert rec.shape == gold["rec"].shape
    assert np.array_equal(rec[:, 4:], gold["rec"][:, 4:])
    np.testing.assert_allclose(rec[:, :4], gold["rec"][:, :4], rtol=tol, atol=0)


# ---------------------------------------------------------------------------
# AB2
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("h", [0.01, 1e-3, 0.37])
def test_ab2_combine_bitwise_numpy(h):
    rng = np.random.default_rng(17)
    shape = (4, 24, 16, 9)
    y, fc, fp = (rng.standard_normal(shape) + 1j * rng.standard_normal(shape) for _ in range(3))
    want = y + h * (1.5 * fc - 0.5 * fp)  # integrators.py:361-363
    got = srk.ab2_combine(dev(y), h, dev(fc), dev(fp)).cpu().numpy()
    assert np.array_equal(got, want)
    # numpy in, numpy out (computed on the device)
    got_np = srk.ab2_combine(y, h, fc, fp)
    assert isinstance(got_np, np.ndarray) and np.array_equal(got_np, want)


def test_ab2_tg32_uneven_tail_vs_reference():
    spec = srk.ProblemSpec("taylor_green", params=srk.PhysParams(1600.0))
    c = srk.RunConfig(grid_shape=(32, 32, 32), problem=spec, integrator="ab2", mode="fixed", t_end=0.105, h=0.01)
    res = srk.run_simulation(c)
    gold = R2["ab2_tg32"]
    _check_records(res, gold)
    assert abs(res.records[-1].h - 0.005) < 1e-15  # the RK4 tail restart ran
    assert rel(res.state.fields, gold["y"]) <= 1e-10


def test_ab2_rt2d_vs_reference():
    shape = (16, 64)
    spec = srk.ProblemSpec("rayleigh_taylor", params=srk.PhysParams(1600.0))
    c = srk.RunConfig(grid_shape=shape, problem=spec, integrator="ab2", mode="fixed", t_end=0.2, h=0.01,
                      lengths=srk.default_lengths("rayleigh_taylor", shape))
    res = srk.run_simulation(c)
    gold = R2["ab2_rt2d"]
    _check_records(res, gold)
    assert rel(res.state.fields, gold["y"]) <= 1e-10


def test_ab2_step_api_vs_oracle():
    """ab2_step(f, y, t, h, f_prev) -> (y_new, f_curr) (integrators.py:366-381)."""
    og = O.OGrid((32, 32, 32))
    y = O.hit(og, a=4.0, energy=0.5, seed=21)
    fo = O.OracleRHS(og, 900.0)
    f_prev = fo(0.0, y)
    y1_ref = y + 1e-3 * f_prev
    f_curr_ref = fo(1e-3, y1_ref)
    y2_ref = O.ab2_combine(y1_ref, 1e-3, f_curr_ref, f_prev)
    rhs = srk.FlowRHS(srk.Grid(og.shape), srk.PhysParams(900.0))
    y2, f_curr = srk.ab2_step(rhs, dev(y1_ref), 1e-3, 1e-3, dev(f_prev))
    assert rel(f_curr, f_curr_ref) <= 1e-12
    assert rel(y2, y2_ref) <= 1e-13
    with pytest.raises(ValueError):
        srk.ab2_step(rhs, dev(y), 0.0, 1e-3, None)


# ---------------------------------------------------------------------------
# 3D Boussinesq at the fast-plan sizes
# ---------------------------------------------------------------------------
def _bq_state(og, seed):
    """HIT velocity + a random-phase density with content up to every Nyquist plane."""
    rng = np.random.default_rng(seed)
    u = O.hit(og, a=4.0, energy=0.5, seed=seed)
    rho = 0.05 * O.fwd(rng.standard_normal((1,) + og.shape), og)
    return np.concatenate([u, rho], axis=0)


@pytest.mark.parametrize("shape", [(32, 32, 32), (64, 64, 64), (128, 128, 128), (32, 64, 128)])
def test_boussinesq_3d_fast_plans_vs_oracle(shape):
    """M = 48, 96, 192 (and a mixed-axis grid): the 6-signal K1 (u, kx u1, kx u2, rho),
    the 7-signal K2 and the ZOP_B3 z-pass (u x w, rho u) vs physics.py:132-185."""
    og = O.OGrid(shape)
    y = _bq_state(og, 5)
    f_ref = O.OracleRHS(og, 650.0, ri=1.7, pr=0.8, density=True)(0.0, y)
    f = srk.FlowRHS(srk.Grid(shape), srk.PhysParams(650.0, 1.7, 0.8), density=True)(0.0, dev(y))
    assert rel(f, f_ref) <= 1e-12
    # velocity and density tendencies separately (the density part is much smaller)
    assert rel(f[3], f_ref[3]) <= 1e-12


def test_boussinesq_3d_256_one_rhs_vs_oracle():
    """M = 384 (config-3 geometry) with a density field (~20 s CPU oracle)."""
    shape = (256, 256, 256)
    og = O.OGrid(shape)
    y = _bq_state(og, 6)
    f_ref = O.OracleRHS(og, 1000.0, ri=1.0, pr=0.7, density=True)(0.0, y)
    f = srk.FlowRHS(srk.Grid(shape), srk.PhysParams(1000.0, 1.0, 0.7), density=True)(0.0, dev(y))
    assert rel(f, f_ref) <= 1e-12
    assert rel(f[3], f_ref[3]) <= 1e-12


def test_rt3d_rhs_vs_reference_golden():
    """3D Rayleigh-Taylor state (problems.py:65-82, erf interface: z-Nyquist
    content) + random velocity vs the reference's own FlowRHS."""
    c = R2["rt3d_rhs"]
    g = srk.Grid(tuple(int(v) for v in c["shape"]), tuple(float(v) for v in c["lengths"]))
    f = srk.FlowRHS(g, srk.PhysParams(800.0, 1.0, 0.7), density=True)(0.0, dev(c["y"]))
    assert rel(f, c["f"]) <= 1e-12


def test_rt3d_init_vs_oracle():
    shape = (32, 32, 64)
    L = srk.default_lengths("rayleigh_taylor", shape)
    g = srk.Grid(shape, L)
    y = srk.rayleigh_taylor_init(g, srk.ProblemSpec("rayleigh_taylor")).fields
    y_ref = O.rayleigh_taylor(O.OGrid(shape, L))
    assert rel(y, y_ref) <= 1e-14


@pytest.mark.parametrize("integ", ["rk4", "bs5"])
def test_rt3d_window_vs_reference(integ):
    shape = (32, 32, 64)
    spec = srk.ProblemSpec("rayleigh_taylor", params=srk.PhysParams(1600.0))
    kw = dict(h=0.01, t_end=0.05, mode="fixed") if integ == "rk4" else dict(t_end=0.3, mode="adaptive")
    c = srk.RunConfig(grid_shape=shape, problem=spec, integrator=integ,
                      lengths=srk.default_lengths("rayleigh_taylor", shape), **kw)
    if integ == "bs5":
        c.tol_abs = c.tol_rel = 1e-6
    res = srk.run_simulation(c)
    gold = R2[f"rt3d_{integ}"]
    _check_records(res, gold)
    assert rel(res.state.fields, gold["y"]) <= 1e-10


def test_spectrum_entry_point_vs_reference_cli(tmp_path):
    """`python -m paper_1810_10197_b200.spectrum CK` (reference cli.py:90-103) on a
    checkpoint the reference wrote: same text layout, values to 1e-13."""
    from paper_1810_10197_b200.spectrum import main, spectrum_text

    c = R2["spectrum_cli"]
    ck = tmp_path / "final.srkl"
    ck.write_bytes(bytes(c["srkl"]))
    want = bytes(c["text"]).decode().strip().splitlines()
    got = spectrum_text(ck).strip().splitlines()
    assert got[0] == want[0] == "k,E" and len(got) == len(want)
    a = np.array([[float(v) for v in ln.split(",")] for ln in got[1:]])
    b = np.array([[float(v) for v in ln.split(",")] for ln in want[1:]])
    assert np.array_equal(a[:, 0], b[:, 0])
    np.testing.assert_allclose(a[:, 1], b[:, 1], rtol=1e-13, atol=1e-30)
    out = tmp_path / "spec.csv"
    assert main([str(ck), "--out", str(out)]) == 0 and out.read_text().startswith("k,E\n")


@pytest.mark.parametrize("shape", [(6, 10, 512), (8, 8, 512), (4, 6, 512)])
def test_paired_zpass_pencil_counts_vs_oracle(shape):
    """The 512-point z axis runs the paired z-pass (two pencils per CTA, A's P2 packed
    into B's forward column): even and odd pencil counts (135 = 9 x 15: the last CTA
    pairs its pencil with a zero pencil) vs the oracle."""
    og = O.OGrid(shape)
    rng = np.random.default_rng(12)
    y = O.fwd(rng.standard_normal((3,) + shape), og)
    f_ref = O.OracleRHS(og, 300.0)(0.0, y)
    f = srk.FlowRHS(srk.Grid(shape), srk.PhysParams(300.0))(0.0, dev(y))
    assert rel(f, f_ref) <= 1e-12
