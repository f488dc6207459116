"""Per-phase cycle split of the RHS kernels (clock64 timestamps of every 97th CTA).

    python tools/phase_timing.py [n] [launch ...]     (launch 0 = K1 ... 4 = K5)
"""
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_10197_b200 as srk  # noqa: E402
from paper_1810_10197_b200 import _native  # noqa: E402

# K3 one-pencil 768 kernel: the last forward stage keeps its outputs in registers and stores them,
# so "forward_suffix" includes the extraction and "extraction" is empty there
NAMES = {2: ["tma_wait", "inverse_prefix", "fused_middle", "forward_suffix", "extraction"]}
COL = ["stage_wait", "fft_and_store"]
n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
launches = [int(v) for v in sys.argv[2:]] or [0, 1, 2, 3, 4]
g = srk.Grid((n, n, n))
y = torch.randn((3,) + g.kshape, dtype=torch.complex128, device="cuda")
rhs = srk.FlowRHS(g, srk.PhysParams(1000.0))
rhs(0.0, y)
pl = rhs.plan
buf = torch.zeros(1 << 24, dtype=torch.int64, device="cuda")
for li in launches:
    buf.zero_()
    _native.check(pl.lib.srk_debug_phase_buffer(pl.h, ctypes.c_void_p(buf.data_ptr()), li))
    rhs(0.0, y)
    torch.cuda.synchronize()
    _native.check(pl.lib.srk_debug_phase_buffer(pl.h, ctypes.c_void_p(0), -1))
    nts = 6 if li == 2 else 3
    names = NAMES.get(li, COL)
    t = buf.cpu().numpy()[: (1 << 24) // nts * nts].reshape(-1, nts).astype(np.float64)
    t = t[(t[:, 0] > 0) & (t[:, -1] > 0)]
    d = np.diff(t, axis=1)
    med = np.median(d, axis=0)
    # spread of CTA start times / durations: concurrency estimate
    dur = t[:, -1] - t[:, 0]
    print(json.dumps({"n": n, "launch": li, "ctas_sampled": len(t),
                      "median_cycles": dict(zip(names, med.round(0).tolist())),
                      "share": dict(zip(names, (med / med.sum()).round(3).tolist())),
                      "median_total_cycles": float(np.median(dur)),
                      "p10_p90_total": [float(np.percentile(dur, 10)), float(np.percentile(dur, 90))]}))
