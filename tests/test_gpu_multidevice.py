"""One process driving two GPUs (SURVEY §8e single-process layout, or a caller that
switches torch.cuda.set_device between plans): libsrk's launch settings are cached
per (device, kernel) -- the opt-in shared-memory attribute, SM count and resident
CTAs per SM (csrc/host_util.cuh) -- so plans on device 1 launch correctly after
plans on device 0.  Skips on a one-GPU box."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

srk = pytest.importorskip("paper_1810_10197_b200")


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two GPUs in one process")
@pytest.mark.parametrize("shape", [(64, 64, 64), (32, 32, 512)])
def test_plans_on_two_devices_in_one_process(shape):
    g = srk.Grid(shape)
    y0 = srk.hit_init(g, srk.ProblemSpec("hit", a=4.0, energy=0.5, seed=3)).fields
    outs = []
    for dev in (0, 1):
        with torch.cuda.device(dev):
            y = y0.to(f"cuda:{dev}")
            rhs = srk.FlowRHS(g, srk.PhysParams(800.0))
            f = rhs(0.0, y)
            st = srk.ControllerState(h=1e-3)
            out = srk.adaptive_advance(y, 0.0, srk.make_bs5(), st, srk.ControllerConfig(), rhs,
                                       first_stage=f, grid=g)
            torch.cuda.synchronize(dev)
            outs.append((f.cpu(), out.y_new.cpu(), out.h_next))
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])
    assert outs[0][2] == outs[1][2]


def test_launch_caches_are_per_device_single_gpu():
    """On one GPU the per-device caches still serve repeated plans of different sizes."""
    for shape in [(32, 32, 32), (32, 32, 512), (64, 64, 64)]:
        g = srk.Grid(shape)
        y = srk.hit_init(g, srk.ProblemSpec("hit", a=4.0, energy=0.5, seed=1)).fields
        f = srk.FlowRHS(g, srk.PhysParams(500.0))(0.0, y)
        assert bool(torch.isfinite(torch.view_as_real(f)).all())
    assert np.isfinite(1.0)
