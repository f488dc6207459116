"""A/B of the fused projection + next-stage sum on the density paths (srk_rhs_combine
through k_project_tma<DIMS, true, NT>) against the unfused K6 + k_combine
(SRK_NO_PCOMB=1 in the environment selects the latter): BS5 adaptive loop,
device-synchronised wall time per stage.  Usage: python tools/pcomb_ab.py [2d|3d]"""
import json, os, sys, time
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_10197_b200 as srk

case = sys.argv[1] if len(sys.argv) > 1 else "2d"
if case == "2d":
    g = srk.Grid((1024, 1024))
    rhs = srk.FlowRHS(g, srk.PhysParams(1e4, 1.0, 1.0), density=True)
    y = srk.rt_tanh_init(g).fields
    steps, h0 = 30, 1e-3
else:
    g = srk.Grid((256, 256, 256))
    rhs = srk.FlowRHS(g, srk.PhysParams(1e3, 1.0, 1.0), density=True)
    u = srk.hit_init(g, srk.ProblemSpec("hit", a=4.0, energy=0.5, seed=42)).fields
    y = torch.cat([u, 0.1 * u[:1]], 0).contiguous()
    steps, h0 = 12, 1e-3
y = torch.as_tensor(y).cuda()
pair = srk.make_bs5()
cfg = srk.ControllerConfig(tol_abs=1e-7, tol_rel=1e-7)
st = srk.ControllerState(h=h0)
s = dict(y=y, t=0.0, f=rhs(0.0, y))
evals = 0
for it in range(steps):
    if it == steps // 3:
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        evals = 0
    o = srk.adaptive_advance(s["y"], s["t"], pair, st, cfg, rhs, first_stage=s["f"], grid=g)
    evals += o.rhs_evals
    s.update(y=o.y_new, t=o.t_new, f=o.last_stage)
torch.cuda.synchronize()
wall = time.perf_counter() - w0
print(json.dumps({"case": case, "shape": list(g.shape), "fused": not os.environ.get("SRK_NO_PCOMB"),
                  "stages_per_s": round(evals / wall, 2), "ms_per_stage": round(wall / evals * 1e3, 4),
                  "t": s["t"], "energy_check": float(torch.linalg.vector_norm(s["y"]).item())}))
