"""Host-side cost of the public API calls (no device sync inside the timed loop)."""
import sys, os, time, json
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_10197_b200 as srk

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
g = srk.Grid((n, n, n))
y = srk.hit_init(g, srk.ProblemSpec("hit", a=4.0, energy=0.5, seed=42)).fields
rhs = srk.FlowRHS(g, srk.PhysParams(2000.0))
f = rhs(0.0, y)
torch.cuda.synchronize()
out = {}
# host enqueue time of one RHS (GPU may still be busy)
t0 = time.perf_counter()
for _ in range(20):
    rhs(0.0, y, out=f) if "out" in rhs.__call__.__code__.co_varnames else rhs(0.0, y)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
out["rhs_host_ms"] = (t1 - t0) / 20 * 1e3
out["rhs_wall_ms"] = (t2 - t0) / 20 * 1e3
pair = srk.make_bs5()
cfg = srk.ControllerConfig(tol_abs=1e-6, tol_rel=1e-6)
st = srk.ControllerState(h=1e-3)
torch.cuda.synchronize()
t0 = time.perf_counter()
o = srk.adaptive_advance(y, 0.0, pair, st, cfg, rhs, first_stage=f, grid=g)
torch.cuda.synchronize()
t1 = time.perf_counter()
out["advance_wall_ms"] = (t1 - t0) * 1e3
out["advance_evals"] = o.rhs_evals
yy = o.y_new
t0 = time.perf_counter()
srk.apply_forcing(yy, g, 0.5, 2.0)
torch.cuda.synchronize()
out["forcing_wall_ms"] = (time.perf_counter() - t0) * 1e3
t0 = time.perf_counter()
q = srk.diagnostics.reduce_sums(g, yy, fl=f, flags=2, ncomp=3).tolist()
out["diag_wall_ms"] = (time.perf_counter() - t0) * 1e3
print(json.dumps(out))
