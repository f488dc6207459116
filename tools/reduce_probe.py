"""Time / profile the fused error-norm + diagnostics reduction (k_reduce) at N^3 with BS5-like terms."""
import sys, os, json
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_10197_b200 as srk
from paper_1810_10197_b200.diagnostics import reduce_sums

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
nt = int(sys.argv[2]) if len(sys.argv) > 2 else 7
g = srk.Grid((n, n, n))
sh = (3,) + g.kshape
y0 = torch.randn(sh, dtype=torch.complex128, device="cuda")
y1 = torch.randn(sh, dtype=torch.complex128, device="cuda")
fl = torch.randn(sh, dtype=torch.complex128, device="cuda")
Fs = [torch.randn(sh, dtype=torch.complex128, device="cuda") for _ in range(nt)]
terms = [(1e-3 * (j + 1), F) for j, F in enumerate(Fs)]
for _ in range(2):
    q = reduce_sums(g, y1, fl=fl, y0=y0, terms=terms, tol_abs=1e-6, tol_rel=1e-6, flags=3, ncomp=3)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    q = reduce_sums(g, y1, fl=fl, y0=y0, terms=terms, tol_abs=1e-6, tol_rel=1e-6, flags=3, ncomp=3)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
nbytes = (3 + nt) * y0.numel() * 16
print(json.dumps({"n": n, "terms": nt, "ms": round(ms, 3), "GBps": round(nbytes / ms / 1e6, 1)}))
