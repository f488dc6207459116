"""Adaptive runs through run_simulation with and without CUDA-graph replay of the
attempts (graphs.py): stages/s of both, and whether the trajectories are
bit-identical (records and final field).

    python tools/graph_timing.py [c1|c4|c2|all]

c1: TG 32^3 BS5 tol 1e-6 to t = 1 (config 1); c4: 2D RT 1024^2 BS5 tol 1e-6 to
t = 2 (config 4 window; tanh IC); c2: TG 128^3 BS5 tol 1e-7 to t = 2 (config 2).
Per mode: one full warm-up run (plan, twiddles, graph capture), then the best
of three timed runs (wall clock around run_simulation, synchronised).
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_10197_b200 as srk  # noqa: E402


def case(name):
    tg = srk.ProblemSpec("taylor_green", params=srk.PhysParams(1600.0))
    if name == "c1":
        return srk.RunConfig(grid_shape=(32,) * 3, problem=tg, integrator="bs5", mode="adaptive", t_end=1.0), None
    if name == "c2":
        return srk.RunConfig(grid_shape=(128,) * 3, problem=tg, integrator="bs5", mode="adaptive", t_end=2.0,
                             tol_abs=1e-7, tol_rel=1e-7), None
    if name == "c4":
        g = srk.Grid((1024, 1024))
        rt = srk.ProblemSpec("rayleigh_taylor", params=srk.PhysParams(1e4, 1.0, 1.0))
        cfg = srk.RunConfig(grid_shape=(1024, 1024), problem=rt, integrator="bs5", mode="adaptive", t_end=2.0,
                            lengths=g.lengths)
        return cfg, srk.rt_tanh_init(g, width=0.05, amp=1e-3, kmax=8, seed=4)
    if name == "c4full":  # config 4 as BASELINE states it: BS5 tol 1e-6 to t = 10
        g = srk.Grid((1024, 1024))
        rt = srk.ProblemSpec("rayleigh_taylor", params=srk.PhysParams(1e4, 1.0, 1.0))
        cfg = srk.RunConfig(grid_shape=(1024, 1024), problem=rt, integrator="bs5", mode="adaptive", t_end=10.0,
                            lengths=g.lengths)
        return cfg, srk.rt_tanh_init(g, width=0.05, amp=1e-3, kmax=8, seed=4)
    if name == "c1rk4":
        return srk.RunConfig(grid_shape=(32,) * 3, problem=tg, integrator="rk4", mode="fixed", t_end=1.0, h=0.01), None
    if name == "c2rk4":  # config 2's RK4 run, first quarter (t <= 0.5, 500 steps)
        return srk.RunConfig(grid_shape=(128,) * 3, problem=tg, integrator="rk4", mode="fixed", t_end=0.5,
                             h=1e-3), None
    if name == "c4rk4":  # config 4's RK4 h = 1e-3 run, first 1000 steps
        g = srk.Grid((1024, 1024))
        rt = srk.ProblemSpec("rayleigh_taylor", params=srk.PhysParams(1e4, 1.0, 1.0))
        cfg = srk.RunConfig(grid_shape=(1024, 1024), problem=rt, integrator="rk4", mode="fixed", t_end=1.0,
                            h=1e-3, lengths=g.lengths)
        return cfg, srk.rt_tanh_init(g, width=0.05, amp=1e-3, kmax=8, seed=4)
    raise SystemExit(name)


def run(name, graphs, reps=None):
    """Best of `reps` full runs after a full warm-up run (plans, twiddles, graph captures)."""
    cfg, ic = case(name)
    st = ic if ic is not None else srk.make_initial_state(cfg)
    reps = reps or (1 if name.endswith("full") else 3)
    srk.run_simulation(cfg, initial_state=st, graphs=graphs, max_steps=200 if name.endswith("full") else None)  # warm-up
    wall = None
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = srk.run_simulation(cfg, initial_state=st, graphs=graphs)
        torch.cuda.synchronize()
        w = time.perf_counter() - t0
        wall = w if wall is None else min(wall, w)
    rec = np.array([[r.t, r.h, r.e_kin, r.eps, r.rhs_evals, r.rejections] for r in res.records])
    return res, rec, wall


def main():
    names = (["c1", "c4", "c2", "c1rk4", "c4rk4", "c2rk4"] if len(sys.argv) < 2 or sys.argv[1] == "all"
             else sys.argv[1:])
    for name in names:
        r0, rec0, w0 = run(name, False)
        r1, rec1, w1 = run(name, True)
        same = bool(np.array_equal(rec0, rec1) and torch.equal(r0.state.fields, r1.state.fields))
        print(json.dumps({"case": name, "steps": r1.steps, "rhs_evals": r1.rhs_evals, "rejections": r1.rejections,
                          "eager_stages_per_s": round(r0.rhs_evals / w0, 1),
                          "graph_stages_per_s": round(r1.rhs_evals / w1, 1),
                          "speedup": round(w0 / w1, 3), "bit_identical": same}), flush=True)


if __name__ == "__main__":
    main()
