"""The peer-store slab exchange across real process boundaries: two ranks as two
processes (CUDA IPC handles all-gathered over gloo), both on cuda:0 -- the one
GPU gpurun grants.  The barrier between K1 / K4 and their readers is a host one
(device sync + gloo barrier) here, the NCCL all-reduce on multi-GPU boxes; no
kernel waits on another rank's kernel."""

import ctypes
import os
import random

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

SHAPE = (64, 64, 64)


def _worker(rank, world, port, out_dir):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import paper_1810_10197_b200 as srk
    from paper_1810_10197_b200 import _native
    from paper_1810_10197_b200.slab import (SlabFlowRHS, exchange_peer_tables, ipc_close, ipc_export,
                                            ipc_import, scatter_slab)

    # 1. raw IPC: rank 0 stores into rank 1's buffer through the imported pointer
    buf = torch.full((1000,), float(rank), dtype=torch.float64, device="cuda")
    mine = ipc_export(buf)
    allh = [None] * world
    dist.all_gather_object(allh, mine)
    if rank == 0:
        peer = ipc_import(*allh[1])
        src = torch.arange(1000, dtype=torch.float64, device="cuda")
        _native.check(_native.load().srk_store_mapped(_native.ptr(src), ctypes.c_void_p(peer), 1000,
                                                      _native.stream_ptr()))
        torch.cuda.synchronize()
        ipc_close(peer, allh[1][1])
    dist.barrier()
    ok_raw = bool(torch.equal(buf, torch.arange(1000, dtype=torch.float64, device="cuda"))) if rank == 1 else True

    # 2. the peer-store slab RHS over both processes vs the unsplit RHS
    g = srk.Grid(SHAPE)
    params = srk.PhysParams(300.0)
    y = srk.hit_init(g, srk.ProblemSpec("hit", a=4.0, energy=0.5, seed=5)).fields

    def barrier():
        torch.cuda.synchronize()
        dist.barrier()

    rhs = SlabFlowRHS(g, params, rank, world, peer=True, barrier=barrier)
    ys = scatter_slab(y, rank, world)
    f = rhs(0.0, ys)
    torch.cuda.synchronize()
    np.save(os.path.join(out_dir, f"f{rank}.npy"), f.cpu().numpy())
    if rank == 0:
        np.save(os.path.join(out_dir, "ref.npy"), srk.FlowRHS(g, params)(0.0, y).cpu().numpy())
    np.save(os.path.join(out_dir, f"raw{rank}.npy"), np.array([ok_raw]))
    dist.barrier()
    dist.destroy_process_group()


def test_peer_store_exchange_across_processes(tmp_path):
    world = 2
    port = random.randint(20000, 40000)
    mp.start_processes(_worker, args=(world, port, str(tmp_path)), nprocs=world, start_method="spawn", join=True)
    assert all(bool(np.load(tmp_path / f"raw{r}.npy")[0]) for r in range(world))
    f = np.concatenate([np.load(tmp_path / f"f{r}.npy") for r in range(world)], axis=2)
    ref = np.load(tmp_path / "ref.npy")
    assert np.linalg.norm(f - ref) / np.linalg.norm(ref) <= 1e-14
