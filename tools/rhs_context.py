"""RHS device time in different contexts at N^3 (CUDA events): isolated timed
calls, back-to-back public-API calls, random vs HIT input, and with a stage
combination in between.  Finds where a stage's time outside the kernels goes."""
import ctypes, json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_10197_b200 as srk
from paper_1810_10197_b200 import _native, integrators

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
g = srk.Grid((n, n, n))
rhs = srk.FlowRHS(g, srk.PhysParams(2000.0))
yh = srk.hit_init(g, srk.ProblemSpec("hit", a=4.0, energy=0.5, seed=42)).fields
yr = torch.randn_like(yh)
out = {}


def ev_time(fn, reps=4):
    fn()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def timed(y):
    pl = rhs.plan
    f = torch.empty_like(y)
    acc = np.zeros(6)
    for r in range(3):
        ms = (ctypes.c_float * 16)()
        rc = pl.lib.srk_rhs_timed(pl.bind(), _native.ptr(y), _native.ptr(f), 1 / 2000.0, 1.0, 2000.0, _native.stream_ptr(), ms, 16)
        acc += np.array(ms[:6])
    return (acc / 3).round(3).tolist()


out["timed_hit"] = timed(yh)
out["timed_rand"] = timed(yr)
out["api_hit_ms"] = ev_time(lambda: rhs(0.0, yh))
out["api_rand_ms"] = ev_time(lambda: rhs(0.0, yr))
fbuf = torch.empty_like(yh)
out["api_hit_out_ms"] = ev_time(lambda: rhs(0.0, yh, out=fbuf))
# evolved state: 3 BS5 steps
pair = srk.make_bs5()
cfg = srk.ControllerConfig(tol_abs=1e-6, tol_rel=1e-6)
st = srk.ControllerState(h=1e-3)
y, t, f = yh, 0.0, rhs(0.0, yh)
for _ in range(3):
    o = srk.adaptive_advance(y, t, pair, st, cfg, rhs, first_stage=f, grid=g)
    y, t, f = o.y_new, o.t_new, o.last_stage
out["timed_evolved"] = timed(y)
out["api_evolved_ms"] = ev_time(lambda: rhs(0.0, y))
# denormal census of the evolved state
v = torch.view_as_real(y).abs()
out["frac_zero"] = float((v == 0).double().mean())
out["frac_denormal"] = float(((v > 0) & (v < 2.2250738585072014e-308)).double().mean())
out["frac_below_1e-250"] = float(((v > 0) & (v < 1e-250)).double().mean())
vr = torch.view_as_real(yh).abs()
out["hit0_frac_zero"] = float((vr == 0).double().mean())
out["hit0_frac_denormal"] = float(((vr > 0) & (vr < 2.2250738585072014e-308)).double().mean())
print(json.dumps(out))
