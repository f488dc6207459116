"""Device time of the fused RHS + next-stage sum (srk_rhs_combine) vs srk_rhs followed
by k_combine, per number of earlier stages nt, at N^3 (CUDA events)."""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_10197_b200 as srk
from paper_1810_10197_b200 import integrators

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
g = srk.Grid((n, n, n))
rhs = srk.FlowRHS(g, srk.PhysParams(1000.0))
y = torch.randn((3,) + g.kshape, dtype=torch.complex128, device="cuda")
yb = torch.randn_like(y)
Fs = [torch.randn_like(y) for _ in range(6)]


def t(fn, reps=4):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


base = t(lambda: rhs(0.0, y))
out = {"n": n, "rhs_ms": round(base, 3)}
F3 = 3 * g.mode_count * 16
for nt in range(0, 7):
    terms = [(0.01 * (j + 1), Fs[j]) for j in range(nt)]
    fused = t(lambda: rhs.eval_combine(0.0, y, yb, terms, 0.02))
    split = t(lambda: integrators.combine(yb, terms + [(0.02, rhs(0.0, y))]))
    extra = (nt + 2) * F3  # ybase + nt stages read, ynext written (f stays in registers)
    f0 = rhs(0.0, y)
    comb = t(lambda: integrators.combine(yb, terms + [(0.02, f0)]))
    out[f"nt{nt}"] = {"fused_ms": round(fused, 3), "split_ms": round(split, 3), "combine_only_ms": round(comb, 3),
                      "combine_GBps": round((nt + 3) * F3 / (comb * 1e-3) / 1e9, 1),
                      "fused_extra_GBps": round(extra / ((fused - base) * 1e-3) / 1e9, 1)}
print(json.dumps(out))
