"""Config C4 (2D Boussinesq Rayleigh-Taylor 1024^2, BS5 adaptive): device time per RHS vs
wall time per stage of the adaptive loop -- is the 2D path launch / host bound?"""
import json, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_10197_b200 as srk

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
g = srk.Grid((n, n))
rhs = srk.FlowRHS(g, srk.PhysParams(1e4, 1.0, 1.0), density=True)
y = srk.rayleigh_taylor_init(g, srk.ProblemSpec("rayleigh_taylor")).fields if hasattr(srk, "rayleigh_taylor_init") else None
y = torch.as_tensor(y).cuda() if not isinstance(y, torch.Tensor) else y
f = rhs(0.0, y)
torch.cuda.synchronize()
a, b = torch.cuda.Event(True), torch.cuda.Event(True)
a.record()
for _ in range(50):
    rhs(0.0, y)
b.record()
torch.cuda.synchronize()
rhs_ms = a.elapsed_time(b) / 50
t0 = time.perf_counter()
for _ in range(50):
    rhs(0.0, y)
host_ms = (time.perf_counter() - t0) / 50 * 1e3
torch.cuda.synchronize()
pair = srk.make_bs5()
cfg = srk.ControllerConfig(tol_abs=1e-7, tol_rel=1e-7)
st = srk.ControllerState(h=1e-3)
s = dict(y=y, t=0.0, f=f)
evals = 0
for it in range(30):
    if it == 10:
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        evals = 0
    o = srk.adaptive_advance(s["y"], s["t"], pair, st, cfg, rhs, first_stage=s["f"], grid=g)
    evals += o.rhs_evals
    s.update(y=o.y_new, t=o.t_new, f=o.last_stage)
torch.cuda.synchronize()
wall = time.perf_counter() - w0
print(json.dumps({"n": n, "rhs_device_ms": round(rhs_ms, 4), "rhs_host_enqueue_ms": round(host_ms, 4),
                  "stages_per_s": round(evals / wall, 1), "ms_per_stage_wall": round(wall / evals * 1e3, 4)}))
