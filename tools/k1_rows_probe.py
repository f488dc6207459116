import ctypes, json, os, sys
import numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_1810_10197_b200 as srk
from paper_1810_10197_b200 import _native
for n0 in (64, 128, 256, 512):
    shape = (n0, 512, 512)
    g = srk.Grid(shape)
    y = torch.randn((3,) + g.kshape, dtype=torch.complex128, device="cuda")
    f = torch.empty_like(y)
    rhs = srk.FlowRHS(g, srk.PhysParams(1000.0))
    rhs(0.0, y); torch.cuda.synchronize()
    pl = rhs.plan
    acc = None
    for r in range(6):
        ms = (ctypes.c_float * 16)()
        rc = pl.lib.srk_rhs_timed(pl.bind(), _native.ptr(y), _native.ptr(f), 1e-3, 1.0, 1000.0, _native.stream_ptr(), ms, 16)
        v = np.array(ms[:-rc])
        if r > 0: acc = v if acc is None else acc + v
    acc /= 5
    sc = n0 * 512 * 257 * 16
    print(json.dumps({"n0": n0, "probe": os.environ.get("SRK_PROBE_INV", "0"), "K1_ms": round(float(acc[0]), 4), "K1_load_GBps_dram": round(3 * sc / acc[0] / 1e6, 1), "K5_ms": round(float(acc[4]), 4)}))
    del rhs, y, f
    torch.cuda.empty_cache()
