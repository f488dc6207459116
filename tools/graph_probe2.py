"""Per-step wall times of run_simulation's adaptive loop with graphs on / off
(diagnostics for graphs.py): prints the slowest steps and the totals."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_10197_b200 as srk  # noqa: E402
from paper_1810_10197_b200 import graphs as G  # noqa: E402
from paper_1810_10197_b200 import simulation as S  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from graph_timing import case  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
orig = G.AttemptGraph.advance
log = []


def timed(self, *a, **k):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    cap = [g is None for g in self.graphs]
    out = orig(self, *a, **k)
    torch.cuda.synchronize()
    log.append((round((time.perf_counter() - t0) * 1e3, 3), out.rejections, cap))
    return out


G.AttemptGraph.advance = timed
cfg, ic = case(name)
st = ic if ic is not None else srk.make_initial_state(cfg)
for rep in range(2):
    log.clear()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = srk.run_simulation(cfg, initial_state=st, graphs=True)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    adv = sum(x[0] for x in log)
    print(json.dumps({"rep": rep, "wall_ms": round(wall * 1e3, 2), "advance_ms": round(adv, 2), "steps": len(log),
                      "slowest": sorted(log, reverse=True)[:5], "median_ms": sorted(x[0] for x in log)[len(log) // 2]}),
          flush=True)
