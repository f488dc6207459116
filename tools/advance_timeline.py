"""GPU-time split of adaptive_advance at N^3: RHS, combine, reduce, gaps (CUDA events)."""
import sys, os, json, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_10197_b200 as srk
from paper_1810_10197_b200 import integrators, diagnostics, control

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
g = srk.Grid((n, n, n))
y = srk.hit_init(g, srk.ProblemSpec("hit", a=4.0, energy=0.5, seed=42)).fields
rhs0 = srk.FlowRHS(g, srk.PhysParams(2000.0))
ev = []


def mark(tag):
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    ev.append((tag, e))


class _Timed:
    """rhs0 with CUDA-event marks; keeps the fused RHS + accumulation entry."""

    def __call__(self, t, yy):
        mark("rhs<")
        out = rhs0(t, yy)
        mark("rhs>")
        return out

    def eval_combine(self, *a):
        mark("rhs<")
        out = rhs0.eval_combine(*a)
        mark("rhs>")
        return out


rhs = _Timed()


_comb = integrators.combine


def comb(*a, **k):
    mark("comb<")
    out = _comb(*a, **k)
    mark("comb>")
    return out


integrators.combine = comb
_red = diagnostics.reduce_sums


def red(*a, **k):
    mark("red<")
    out = _red(*a, **k)
    mark("red>")
    return out


diagnostics.reduce_sums = red
pair = srk.make_bs5()
cfg = srk.ControllerConfig(tol_abs=1e-6, tol_rel=1e-6)
st = srk.ControllerState(h=1e-3)
f = rhs0(0.0, y)
s = dict(y=y, t=0.0, f=f)
for it in range(4):
    ev.clear()
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    mark("start")
    o = srk.adaptive_advance(s["y"], s["t"], pair, st, cfg, rhs, first_stage=s["f"], grid=g)
    mark("end")
    torch.cuda.synchronize()
    wall = (time.perf_counter() - w0) * 1e3
    s.update(y=o.y_new, t=o.t_new, f=o.last_stage)
tot = {"rhs": 0.0, "comb": 0.0, "red": 0.0}
for (t0, e0), (t1, e1) in zip(ev, ev[1:]):
    if t0.endswith("<") and t1 == t0[:-1] + ">":
        tot[t0[:-1]] += e0.elapsed_time(e1)
span = ev[0][1].elapsed_time(ev[-1][1])
print(json.dumps({"n": n, "wall_ms": round(wall, 2), "gpu_span_ms": round(span, 2),
                  **{k: round(v, 2) for k, v in tot.items()},
                  "gaps_ms": round(span - sum(tot.values()), 2), "evals": o.rhs_evals, "rejections": o.rejections}))
