"""Slab-decomposed RHS on CPU: gloo, world_size 2 and 3, numpy
restatement of the kernel groups, checked against the single-process oracle.
Also checks the distributed reduction protocol (rank-order sums) used for the
adaptive controller."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, shape, density, q, chunks=1):
    import sys

    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle as O
        from paper_1810_10197_b200 import Grid, PhysParams
        from paper_1810_10197_b200.slab import SlabFlowRHS, dist_sum_in_rank_order, scatter_slab
        from slab_numpy_backend import NumpySlabBackend

        og = O.OGrid(shape)
        rng = np.random.default_rng(3)
        nc = 4 if density else 3
        y = rng.standard_normal((nc,) + og.kshape) + 1j * rng.standard_normal((nc,) + og.kshape)
        y[:3] = O.leray(y[:3], og)
        params = PhysParams(reynolds=80.0, richardson=1.5, prandtl=0.7)
        g = Grid(shape)
        be = NumpySlabBackend(g, params, rank, world, density)
        rhs = SlabFlowRHS(g, params, rank, world, density=density, backend=be, chunks=chunks)
        assert rhs.pipelined == (chunks > 1)
        ys = torch.from_numpy(scatter_slab(y, rank, world))
        f = rhs(0.0, ys)
        parts = [torch.empty_like(f) for _ in range(world)]
        dist.all_gather(parts, f)
        # distributed kinetic-energy sum in rank order (the controller's protocol)
        w = np.full(og.kshape[-1], 2.0)
        w[0] = w[-1] = 1.0
        loc = float(np.sum(w * np.abs(ys.numpy()[:3]) ** 2))
        tot = dist_sum_in_rank_order()([loc])[0]
        if rank == 0:
            full = torch.cat(parts, dim=2).numpy()
            ref = O.OracleRHS(og, 80.0, 1.5, 0.7, density=density)(0.0, y)
            err = np.linalg.norm(full - ref) / np.linalg.norm(ref)
            e_ref = float(np.sum(w * np.abs(y[:3]) ** 2))
            q.put((err, abs(tot - e_ref) / e_ref))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,shape,density,chunks", [(2, (16, 16, 12), False, 1), (3, (16, 12, 8), False, 1),
                                                        (2, (8, 8, 8), True, 1),
                                                        # kz-chunk pipeline, async gloo exchanges
                                                        (2, (16, 16, 30), False, 3), (3, (12, 12, 34), True, 4)])
def test_slab_rhs_matches_oracle(world, shape, density, chunks):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, shape, density, q, chunks)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    assert all(p.exitcode == 0 for p in procs)
    err, e_err = q.get(timeout=5)
    assert err <= 1e-12
    assert e_err <= 1e-14


def test_slab_geometry_rules():
    from paper_1810_10197_b200 import Grid
    from paper_1810_10197_b200.slab import slab_geometry

    geo = slab_geometry(Grid((1024, 1024, 1024)), 8)
    assert geo["ny"] == 128 and geo["mx"] == 192
    # bytes per GPU per RHS crossing the fabric (~12.7 GB at P=8 with
    # 6 exchanged signals; the curl is completed after the exchange here -> 5)
    sent = (geo["send1"] + geo["send2"]) * 16 * (7 / 8)
    assert 10e9 < sent < 12e9
    with pytest.raises(ValueError):
        slab_geometry(Grid((16, 12, 8)), 5)
    with pytest.raises(ValueError):
        slab_geometry(Grid((16, 16)), 2)
