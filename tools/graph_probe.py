"""Diagnose CUDA-graph replay of one adaptive attempt (graphs.py): device time of
back-to-back replays vs the eager attempt, and per-step host time in the driver.

    python tools/graph_probe.py c4|c1
"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_10197_b200 as srk  # noqa: E402
from paper_1810_10197_b200.graphs import attempt_graph  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from graph_timing import case  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
cfg, ic = case(name)
st = ic if ic is not None else srk.make_initial_state(cfg)
g = srk.Grid(cfg.grid_shape, cfg.lengths or srk.default_lengths(cfg.problem.kind, cfg.grid_shape))
rhs = srk.FlowRHS(g, cfg.problem.params, density=cfg.has_density)
y = st.fields if hasattr(st, "fields") else st
y = torch.as_tensor(y).cuda() if not isinstance(y, torch.Tensor) else y
f = rhs(0.0, y)
pair = srk.make_bs5()
ag = attempt_graph(rhs, pair, cfg.controller, g)
ctrl = srk.ControllerState(h=1e-4)
out = ag.advance(y, 0.0, ctrl, f)  # captures graph 0
out = ag.advance(out.y_new, out.t_new, srk.ControllerState(h=1e-4), out.last_stage)  # graph 1
torch.cuda.synchronize()
res = {"case": name, "launches_per_replay": ag.launches}
for p in (0, 1):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ag.h_pin[0] = 1e-4
    e0.record()
    for _ in range(20):
        ag.graphs[p].replay()
    e1.record()
    e1.synchronize()
    res[f"replay_ms_graph{p}"] = round(e0.elapsed_time(e1) / 20, 4)
# eager attempt (same work) for comparison
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
yy, ff = y.clone(), f.clone()
e0.record()
for _ in range(10):
    srk.adaptive_advance(yy, 0.0, pair, srk.ControllerState(h=1e-4), cfg.controller, rhs, first_stage=ff, grid=g)
e1.record()
e1.synchronize()
res["eager_attempt_ms_incl_host"] = round(e0.elapsed_time(e1) / 10, 4)
t0 = time.perf_counter()
for _ in range(10):
    ag.h_pin[0] = 1e-4
    ag.graphs[0].replay()
    torch.cuda.current_stream().synchronize()
res["replay_plus_sync_wall_ms"] = round((time.perf_counter() - t0) / 10 * 1e3, 4)
print(json.dumps(res), flush=True)
