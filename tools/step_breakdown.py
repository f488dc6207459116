"""Wall-clock breakdown of the bench step (steady state) into its public-API calls."""
import sys, os, time, json
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_10197_b200 as srk

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
g = srk.Grid((n, n, n))
y = srk.hit_init(g, srk.ProblemSpec("hit", a=4.0, energy=0.5, seed=42)).fields
rhs = srk.FlowRHS(g, srk.PhysParams(2000.0))
pair = srk.make_bs5()
cfg = srk.ControllerConfig(tol_abs=1e-6, tol_rel=1e-6)
st = srk.ControllerState(h=1e-3)
s = dict(y=y, t=0.0, f=rhs(0.0, y))
acc = {"advance": 0.0, "forcing": 0.0, "refresh_rhs": 0.0, "diag": 0.0}
evals = 0


def tick():
    torch.cuda.synchronize()
    return time.perf_counter()


for it in range(8):
    t0 = tick()
    o = srk.adaptive_advance(s["y"], s["t"], pair, st, cfg, rhs, first_stage=s["f"], grid=g)
    t1 = tick()
    srk.apply_forcing(o.y_new, g, 0.5, 2.0)
    t2 = tick()
    f = rhs(o.t_new, o.y_new)
    t3 = tick()
    q = srk.diagnostics.reduce_sums(g, o.y_new, fl=f, flags=2, ncomp=3).tolist()
    t4 = tick()
    s.update(y=o.y_new, t=o.t_new, f=f)
    if it >= 3:
        acc["advance"] += t1 - t0
        acc["forcing"] += t2 - t1
        acc["refresh_rhs"] += t3 - t2
        acc["diag"] += t4 - t3
        evals += o.rhs_evals + 1
steps = 5
res = {k: v / steps * 1e3 for k, v in acc.items()}
res["evals_per_step"] = evals / steps
res["ms_per_eval"] = sum(acc.values()) / evals * 1e3
# RHS alone
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    rhs(0.0, s["y"])
res["rhs_ms"] = (tick() - t0) / 10 * 1e3
print(json.dumps({k: round(v, 3) for k, v in res.items()}))
