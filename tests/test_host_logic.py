"""Host-side logic of the drop-in API vs the oracle restatement (CPU-only)."""

import os
import numpy as np
import pytest

import oracle as O
import paper_1810_10197_b200 as srk
from paper_1810_10197_b200.simulation import _fixed_step_times


@pytest.mark.parametrize("name", ["rk4", "dp5", "bs5", "kcl5"])
def test_tableaux_match_oracle(name):
    a, b = srk.make_pair(name), O.tableau(name)
    assert np.array_equal(a.A, b.A) and np.array_equal(a.b, b.b) and np.array_equal(a.c, b.c)
    assert (a.b_hat is None) == (b.b_hat is None)
    if a.b_hat is not None:
        assert np.array_equal(a.b_hat, b.b_hat)
    assert a.fsal == b.fsal


def test_fsal_flags():
    assert srk.make_bs5().fsal and srk.make_dp5().fsal
    assert not srk.make_rk4().fsal and not srk.make_kcl5().fsal


def test_bs5_stage_sparsity():
    # non-zeros per A row [0,1,2,3,4,5,6,6]; b has 6; b - b_hat has 7
    p = srk.make_bs5()
    assert [int(np.count_nonzero(r)) for r in p.A] == [0, 1, 2, 3, 4, 5, 6, 6]
    assert np.count_nonzero(p.b) == 6 and np.count_nonzero(p.b - p.b_hat) == 7


@pytest.mark.parametrize("err", [0.0, 1e-12, 0.3, 0.999999, 1.0, 1.0000001, 7.0, 1e9, np.inf, np.nan])
@pytest.mark.parametrize("prev", [False, True])
def test_propose_step_matches_oracle(err, prev):
    s1 = srk.ControllerState(h=0.2, prev_rejected=prev)
    s2 = O.CtrlState(h=0.2, prev_rejected=prev)
    assert srk.propose_step(err, s1, srk.ControllerConfig()) == O.propose_step(err, s2, O.Ctrl())
    assert (s1.prev_rejected, s1.rejections, s1.acceptances) == (s2.prev_rejected, s2.rejections, s2.acceptances)


def test_propose_step_underflow():
    st = srk.ControllerState(h=1e-3)
    with pytest.raises(srk.StepSizeUnderflowError):
        srk.propose_step(np.inf, st, srk.ControllerConfig(h_min=1e-4))


def test_controller_exact_values():
    # test_acceptance.py:174-195 style: err=0.5 -> 0.8 * 0.5**-0.2; err=32 -> shrink 0.4
    st = srk.ControllerState(h=0.2)
    h, ok = srk.propose_step(0.5, st, srk.ControllerConfig())
    assert ok and h == 0.2 * min(2.0, 0.8 * 0.5 ** (-0.2))
    st = srk.ControllerState(h=0.2)
    h, ok = srk.propose_step(32.0, st, srk.ControllerConfig())
    assert not ok and h == 0.2 * 0.4


@pytest.mark.parametrize("shape,lengths", [((8, 6, 4), None), ((16, 64), (2 * np.pi, 8 * np.pi)),
                                           ((12, 10, 8), (1.0, 2.0, 3.0))])
def test_grid_geometry_matches_oracle(shape, lengths):
    g, og = srk.Grid(shape, lengths), O.OGrid(shape, lengths)
    assert g.kshape == og.kshape and g.mode_count == og.mode_count and g.points == og.points
    assert g.padded_shape == og.pshape
    for a, b in zip(g.k, og.k):
        assert np.array_equal(a, b)
    assert np.array_equal(g.k2, og.k2) and np.array_equal(g.inv_k2, og.inv_k2)
    assert np.array_equal(np.broadcast_to(g.hermitian_weights, g.kshape), np.broadcast_to(og.w, og.kshape))


@pytest.mark.parametrize("bad", [(7, 8, 8), (2, 8), (8,), (8, 8, 8, 8)])
def test_grid_rejects_bad_shapes(bad):
    with pytest.raises(ValueError):
        srk.Grid(bad)


def _cfg(**kw):
    base = dict(grid_shape=(16, 16), problem=srk.ProblemSpec("taylor_green"), integrator="rk4", mode="fixed",
                t_end=1.0, h=0.1)
    base.update(kw)
    return srk.RunConfig(**base)


@pytest.mark.parametrize("kw", [dict(integrator="euler"), dict(mode="sometimes"), dict(mode="adaptive"),
                                dict(h=None), dict(t_end=0.0),
                                dict(problem=srk.ProblemSpec("hit")),
                                dict(forcing=True)])
def test_config_validation(kw):
    with pytest.raises(srk.ConfigError):
        _cfg(**kw).validate()


class _D:
    def __init__(self, t, steps):
        self.t, self.steps = t, steps


def test_fixed_step_times_lattice_and_tail():
    total, n_full, h_last, time_at = _fixed_step_times(_D(0.0, 0), 0.3, 1.0)
    assert (total, n_full) == (4, 3) and abs(h_last - 0.1) < 1e-12
    assert [time_at(i) for i in range(4)] == [0.3, 0.6, 0.8999999999999999, 1.0]
    total, n_full, h_last, time_at = _fixed_step_times(_D(0.0, 0), 0.1, 1.0)
    assert total == 10 and h_last == 0.0 and [time_at(i) for i in range(10)] == [(i + 1) * 0.1 for i in range(10)]


def test_default_lengths():
    assert srk.default_lengths("rayleigh_taylor", (16, 64))[1] == 2 * np.pi * 4
    assert srk.default_lengths("hit", (8, 8, 8)) == (2 * np.pi,) * 3


def test_compute_without_cuda_fails_loudly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    with pytest.raises(RuntimeError, match="CUDA"):
        srk.FlowRHS(srk.Grid((8, 8, 8)), srk.PhysParams(10.0))


def test_plane_runs_and_forcing_planes():
    from paper_1810_10197_b200.hostio import forcing_planes, plane_runs

    assert plane_runs([]) == []
    assert plane_runs([5, 0, 1, 2, 7, 6, 2]) == [(0, 3), (5, 8)]
    g = srk.Grid((16, 16, 16))
    # k_f = 2 on L = 2pi: |k_x| <= 2 -> x-planes 0, 1, 2, 14, 15
    assert forcing_planes(g, 2.0) == [(0, 3), (14, 16)]
    og = O.OGrid((16, 12, 8), (2 * np.pi, 3.0, 4.0))
    g2 = srk.Grid((16, 12, 8), (2 * np.pi, 3.0, 4.0))
    band = (og.k2 > 0) & (og.k2 <= 2.5 ** 2 * (1 + 1e-12))
    want = sorted(set(np.nonzero(band)[0].tolist()))
    got = [i for a, b in forcing_planes(g2, 2.5) for i in range(a, b)]
    assert got == want


def test_bench_self_launches_n_ranks_dry_run():
    """`bench.py --gpus 2` without a torchrun environment re-launches itself with 2
    ranks (gloo, --dry-run: no GPU work) and rank 0's line reports n_gpus == 2."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    p = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--dry-run", "--steps", "2",
                        "--warmup", "1"], cwd=root, env=env, capture_output=True, text=True, timeout=240)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["ranks_seen"] == 2 and d["dry_run"]


def test_nvtx_ranges_are_a_noop_unless_enabled(monkeypatch):
    """SRK_NVTX gates the NVTX ranges around RHS calls / attempts (tracing)."""
    from paper_1810_10197_b200 import _native

    monkeypatch.setattr(_native, "NVTX", False)
    with _native.nvtx("srk_rhs") as r:
        assert r is _native._NO_RANGE
    monkeypatch.setattr(_native, "NVTX", True)
    assert isinstance(_native.nvtx("srk_rhs"), _native._Range)
    assert _native.nvtx("bs5_attempt").name == "bs5_attempt"
