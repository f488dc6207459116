"""Per-kernel device times of one srk_rhs (CUDA events between launches).

    python tools/rhs_timing.py --n 512 [--reps 5] [--dims 3] [--density]
Device-side random input (FFT cost is data independent); prints one JSON line.
"""
import argparse
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_10197_b200 as srk  # noqa: E402
from paper_1810_10197_b200 import _native  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=512)
ap.add_argument("--dims", type=int, default=3)
ap.add_argument("--density", action="store_true")
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--chain", type=int, default=0,
                help="also time this many back-to-back RHS calls with events only around the chain "
                     "(per-kernel events serialise the launches and hide PDL overlap)")
a = ap.parse_args()
shape = (a.n,) * a.dims
g = srk.Grid(shape)
nc = a.dims + (1 if a.density else 0)
y = torch.randn((nc,) + g.kshape, dtype=torch.complex128, device="cuda")
f = torch.empty_like(y)
rhs = srk.FlowRHS(g, srk.PhysParams(1000.0), density=a.density)
rhs(0.0, y)
torch.cuda.synchronize()
pl = rhs.plan
acc = None
for r in range(a.reps):
    ms = (ctypes.c_float * 16)()
    rc = pl.lib.srk_rhs_timed(pl.bind(), _native.ptr(y), _native.ptr(f), 1e-3, 1.0, 1000.0, _native.stream_ptr(), ms, 16)
    n = -rc
    v = np.array(ms[:n])
    if r > 0:
        acc = v if acc is None else acc + v
acc /= (a.reps - 1)
m, k = 3 * a.n // 2, a.n // 2 + 1
sc, sx, sxy = a.n * a.n * k, m * a.n * k, m * m * k
model = [16 * (3 * sc + 6 * sx), 16 * (6 * sx + 6 * sxy), 16 * (9 * sxy), 16 * (3 * sxy + 3 * sx), 16 * (3 * sx + 3 * sc), 16 * 9 * sc]
out = {"n": a.n, "dims": a.dims, "ms": [round(x, 4) for x in acc], "total_ms": round(float(acc.sum()), 3)}
if a.chain:
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.chain):
        rhs(0.0, y, out=f)
    e1.record()
    e1.synchronize()
    out["chain_ms_per_rhs"] = round(e0.elapsed_time(e1) / a.chain, 4)
if a.dims == 3 and not a.density:
    out["GBps"] = [round(b / (t * 1e-3) / 1e9, 1) for b, t in zip(model, acc)]
    out["rhs_model_frac"] = round(16 * (9 * sc + 18 * sx + 18 * sxy) / (acc.sum() * 1e-3) / 6533.2e9, 4)
print(json.dumps(out))
