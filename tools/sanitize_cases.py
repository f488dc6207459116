"""Small-N workload that reaches every sm_100a kernel family of libsrk, for
compute-sanitizer (memcheck / racecheck / synccheck, one tool per run):

    compute-sanitizer --tool racecheck --racecheck-report hazard python tools/sanitize_cases.py
    SRK_LIB_PATH=_lib_chk/libsrk.so python tools/sanitize_cases.py --dump chk.npz   (hazard-probe build)

Anisotropic grids put one long axis on each pass so the production plans run
on a handful of tiles: an axis of n = 512 gives M = 768 (the 512^3 kernels:
k_colpass<FastFFT1<768,...>> for x / y, the one-pencil z-pass k_zpass_ns3p<768>),
n = 1024 gives M = 1536 (the 1024^3-slab and 2D config-4 kernels), n = 256 /
128 / 64 / 32 the pencil-pair z-passes and the three-stage strided plans, and
odd small sizes the runtime (generic) engine.  Also: Boussinesq 2D / 3D, the
fused stage sums, the refresh, the step reduction, forcing, widen / narrow,
the CUDA-graph attempt replay, and the y-slab kernels with emulated ranks
(block-copy exchange and peer stores into the other ranks' receive buffers).
Prints one line per case; exits non-zero on a parity failure (the sanitizer
report is the point, but a wrong answer must not pass silently).
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_10197_b200 as srk  # noqa: E402
from paper_1810_10197_b200.integrators import combine  # noqa: E402

torch.cuda.init()
RNG = np.random.default_rng(11)
DUMP = {}


def state(g, ncomp, amp=1.0):
    """Band-limited random state (Hermitian by construction: forward transform of a real field)."""
    x = RNG.standard_normal((ncomp,) + tuple(g.shape))
    return srk.forward_transform(torch.from_numpy(x).cuda(), g) * amp


def rhs_case(shape, density=False, lengths=None):
    g = srk.Grid(shape, lengths)
    nc = g.dims + (1 if density else 0)
    y = state(g, nc, 1e-3)
    rhs = srk.FlowRHS(g, srk.PhysParams(500.0, 1.3, 0.7), density=density)
    f = rhs(0.0, y)
    # fused stage sum + refresh on the same plan
    f2, yn = rhs.eval_combine(0.0, y, y, [(0.1, f)], 0.2)
    ref = combine(y, [(0.1, f), (0.2, f2)])
    assert torch.equal(yn, ref), f"fused stage sum differs {shape}"
    _, y2, sums = rhs.refresh(0.0, y, 0.05)
    assert np.isfinite(sums[4])
    torch.cuda.synchronize()
    assert bool(torch.isfinite(torch.view_as_real(f)).all()), f"non-finite RHS {shape} (poisoned shared memory read?)"
    key = "x".join(map(str, shape)) + ("_b" if density else "")
    DUMP[key + "_f"] = f.cpu().numpy()
    DUMP[key + "_yn"] = yn.cpu().numpy()
    DUMP[key + "_y2"] = y2.cpu().numpy()
    DUMP[key + "_sums"] = np.array(sums)
    return float(f.abs().max())


def main():
    t0 = time.time()
    from paper_1810_10197_b200 import _native

    print(f"libsrk {_native.LIB_PATH} build_info={_native.load().srk_build_info()}", flush=True)
    cases = [
        ((512, 8, 8), False), ((8, 512, 8), False), ((8, 8, 512), False),       # M = 768 (512^3 kernels)
        ((1024, 8, 8), False), ((8, 8, 1024), False), ((1024, 16), True),       # M = 1536
        ((16, 16, 256), False), ((16, 256, 16), False), ((256, 16, 16), False),  # M = 384
        ((32, 32, 32), False), ((64, 64, 64), False), ((16, 16, 128), False),   # 48 / 96 / 192
        ((32, 32, 64), True), ((16, 16, 512), True), ((512, 16), True), ((64, 256), False),
        ((8, 12, 16), False), ((12, 10), False), ((8, 10, 6), True),            # runtime engine
    ]
    for shape, dens in cases:
        m = rhs_case(shape, dens)
        print(f"rhs {shape} density={dens} ok max|f|={m:.3e}", flush=True)
    # widen / narrow / transforms / forcing / reductions
    g = srk.Grid((16, 16, 16))
    y = state(g, 3)
    ph = srk.DealiasWorkspace(g, 3).widen(y)
    sp = srk.DealiasWorkspace(g, 3).narrow(ph)
    srk.apply_forcing(srk.hit_init(g, srk.ProblemSpec("hit", seed=3, a=4.0, energy=0.5)).fields, g, 0.5, 2.0)
    print("widen / narrow / forcing ok", float(sp.abs().max()), flush=True)
    # adaptive steps, eager and graphed (CUDA-graph replay of the attempt)
    for graphs in (False, True):
        cfg = srk.RunConfig(grid_shape=(32, 32, 32), problem=srk.ProblemSpec("taylor_green",
                            params=srk.PhysParams(1600.0)), integrator="bs5", mode="adaptive", t_end=0.05)
        res = srk.run_simulation(cfg, graphs=graphs)
        print(f"bs5 run graphs={graphs} steps={res.steps} evals={res.rhs_evals}", flush=True)
    # y-slab kernels, emulated ranks on one GPU (block copies and peer stores)
    from paper_1810_10197_b200.slab import CudaSlabBackend, scatter_slab, slab_geometry

    for shape, P in (((32, 32, 32), 2), ((32, 48, 16), 3)):
        g = srk.Grid(shape)
        prm = srk.PhysParams(321.0)
        yf = state(g, 3, 1e-3)
        f_ref = srk.FlowRHS(g, prm)(0.0, yf)
        geo = slab_geometry(g, P)
        backs = [CudaSlabBackend(g, prm, r, P) for r in range(P)]
        ys = [scatter_slab(yf, r, P).contiguous() for r in range(P)]
        s1 = [b.empty(geo["send1"]) for b in backs]
        r1 = [b.empty(geo["send1"]) for b in backs]
        s2 = [b.empty(geo["send2"]) for b in backs]
        r2 = [b.empty(geo["send2"]) for b in backs]
        fs = [torch.empty_like(v) for v in ys]
        for r in range(P):
            backs[r].forward(ys[r], s1[r])
        blk1 = geo["send1"] // P
        for r in range(P):
            for d in range(P):
                r1[d][r * blk1:(r + 1) * blk1].copy_(s1[r][d * blk1:(d + 1) * blk1])
        for r in range(P):
            backs[r].middle(r1[r], s2[r])
        blk2 = geo["send2"] // P
        for r in range(P):
            for d in range(P):
                r2[d][r * blk2:(r + 1) * blk2].copy_(s2[r][d * blk2:(d + 1) * blk2])
        for r in range(P):
            backs[r].finish(r2[r], ys[r], fs[r])
        torch.cuda.synchronize()
        got = torch.cat(fs, dim=2)
        err = float((got - f_ref).abs().max() / f_ref.abs().max())
        assert err < 1e-13, f"slab {shape} P={P}: {err}"
        # peer stores: each rank's K1 / K4 write straight into every rank's receive buffer
        for r in range(P):
            backs[r].set_peers([t.data_ptr() for t in r1], [t.data_ptr() for t in r2])
        K = g.kshape[2]
        for r in range(P):
            backs[r].forward_kz_peer(ys[r], 0, K)
        for r in range(P):
            backs[r].inverse_y_kz(r1[r], 0, K)
            backs[r].zpass()
            backs[r].forward_y_kz_peer(0, K)
        for r in range(P):
            backs[r].forward_x_kz(r2[r], 0, K)
            backs[r].project(ys[r], fs[r])
        torch.cuda.synchronize()
        err2 = float((torch.cat(fs, dim=2) - f_ref).abs().max() / f_ref.abs().max())
        assert err2 < 1e-13, f"slab peer {shape} P={P}: {err2}"
        print(f"slab {shape} P={P} ok {err:.1e} peer {err2:.1e}", flush=True)
    if len(sys.argv) > 2 and sys.argv[1] == "--dump":
        np.savez(sys.argv[2], **DUMP)
    print(f"all cases ok in {time.time() - t0:.1f} s", flush=True)


if __name__ == "__main__":
    main()
