"""Per-kernel cost per unit of work vs. working-set size: RHS on (n0, 512, 512)
grids with n0 = 4 .. 512 (the y/z passes of a few x planes fit in the 126 MB L2).
Prints ns per 768-point column FFT (K2, K4) and per z pencil (K3)."""
import ctypes, json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_10197_b200 as srk
from paper_1810_10197_b200 import _native

for n0 in [int(v) for v in (sys.argv[1:] or [4, 8, 16, 64, 512])]:
    g = srk.Grid((n0, 512, 512))
    y = torch.randn((3,) + g.kshape, dtype=torch.complex128, device="cuda")
    f = torch.empty_like(y)
    rhs = srk.FlowRHS(g, srk.PhysParams(1000.0))
    rhs(0.0, y)
    pl = rhs.plan
    acc = np.zeros(6)
    reps = 6
    for r in range(reps):
        ms = (ctypes.c_float * 16)()
        pl.lib.srk_rhs_timed(pl.bind(), _native.ptr(y), _native.ptr(f), 1e-3, 1.0, 1000.0, _native.stream_ptr(), ms, 16)
        if r:
            acc += np.array(ms[:6])
    acc /= reps - 1
    m0, m1, K = 3 * n0 // 2, 768, 257
    k2_cols, k3_pen, k4_cols = 6 * m0 * K, m0 * m1, 3 * m0 * K
    print(json.dumps({"n0": n0, "ms": acc.round(4).tolist(), "K2_ns_per_col": round(acc[1] * 1e6 / k2_cols, 3),
                      "K3_ns_per_pencil": round(acc[2] * 1e6 / k3_pen, 3), "K4_ns_per_col": round(acc[3] * 1e6 / k4_cols, 3),
                      "K3_in_MB": round(6 * k3_pen * K * 16 / 1e6, 1)}))
    del rhs, y, f
    torch.cuda.empty_cache()
