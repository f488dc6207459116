"""Bisect a process-level RHS slowdown: per-kernel times under variants (one per process)."""
import ctypes, json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_10197_b200 as srk
from paper_1810_10197_b200 import _native

v = sys.argv[1]
n = 512
g = srk.Grid((n, n, n))
extra = []
if "pre" in v:  # allocations before the plan
    extra = [torch.empty((3,) + g.kshape, dtype=torch.complex128, device="cuda") for _ in range(2)]
if "hit" in v:
    y = srk.hit_init(g, srk.ProblemSpec("hit", a=4.0, energy=0.5, seed=42)).fields
else:
    y = torch.randn((3,) + g.kshape, dtype=torch.complex128, device="cuda")
f = torch.empty_like(y)
rhs = srk.FlowRHS(g, srk.PhysParams(2000.0 if "re2k" in v else 1000.0))
rhs(0.0, y)
torch.cuda.synchronize()
pl = rhs.plan
acc = np.zeros(6)
for r in range(4):
    ms = (ctypes.c_float * 16)()
    pl.lib.srk_rhs_timed(pl.bind(), _native.ptr(y), _native.ptr(f), 1e-3, 1.0, 1000.0, _native.stream_ptr(), ms, 16)
    if r:
        acc += np.array(ms[:6])
from paper_1810_10197_b200.spectral import _arena
ws = pl._bound
print(json.dumps({"variant": v, "ms": (acc / 3).round(3).tolist(), "total": round(float(acc.sum() / 3), 2),
                  "y_ptr_mod_2M": y.data_ptr() % (2 << 20), "ws_ptr_mod_2M": ws.data_ptr() % (2 << 20),
                  "ws_gb": ws.numel() * ws.element_size() / 1e9, "alloc_gb": torch.cuda.memory_allocated() / 1e9,
                  "reserved_gb": torch.cuda.memory_reserved() / 1e9}))
