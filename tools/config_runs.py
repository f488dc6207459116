"""BASELINE.json configurations run end to end on the B200 through the drop-in
driver (run_simulation, reference simulation.py:350-368), at their full lengths:

  c1  TG 32^3, Re 1600: BS5 adaptive tol 1e-6 to t = 1, RK4 h = 0.01 (100 steps)
  c2  TG 128^3, Re 1600: RK4 h = 1e-3 to t = 2 (2000 steps), BS5 tol 1e-7 to t = 2
  c3  decaying HIT 256^3, Re 1000, E = 0.5, k0 = 4, seed 42: BS5 tol 1e-6, 200 steps
  c4  2D Boussinesq RT 1024^2 (tanh interface + seeded |k| <= 8 perturbation),
      Re 1e4, Ri = Pr = 1: BS5 tol 1e-6 and RK4 h = 2e-3 to t = 10
  c5  forced HIT 512^3, Re 2000: BS5 tol 1e-6, 50 steps (1-GPU size of config 5)

    python tools/config_runs.py CASE [OUTDIR]

Writes OUTDIR/CASE_<run>/diagnostics.csv (reference layout) and prints one JSON
line per run: steps, RHS evaluations, rejections, final t / E / eps / Z, and the
wall time of run_simulation (initial state generated before it; per-step host
record + accept/reject syncs included).
"""

import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_10197_b200 as srk  # noqa: E402


def spec(kind, re, **kw):
    return srk.ProblemSpec(kind=kind, params=srk.PhysParams(*re) if isinstance(re, tuple) else srk.PhysParams(re),
                           **kw)


def runs(case):
    tg = spec("taylor_green", 1600.0)
    if case == "c1":
        return [("bs5", dict(grid_shape=(32,) * 3, problem=tg, integrator="bs5", mode="adaptive", t_end=1.0,
                             tol_abs=1e-6, tol_rel=1e-6), None, None),
                ("rk4", dict(grid_shape=(32,) * 3, problem=tg, integrator="rk4", mode="fixed", t_end=1.0, h=0.01),
                 None, None)]
    if case == "c2":
        return [("rk4", dict(grid_shape=(128,) * 3, problem=tg, integrator="rk4", mode="fixed", t_end=2.0, h=1e-3),
                 None, None),
                ("bs5", dict(grid_shape=(128,) * 3, problem=tg, integrator="bs5", mode="adaptive", t_end=2.0,
                             tol_abs=1e-7, tol_rel=1e-7), None, None)]
    if case == "c3":
        hit = spec("hit", 1000.0, a=4.0, energy=0.5, seed=42)
        return [("bs5", dict(grid_shape=(256,) * 3, problem=hit, integrator="bs5", mode="adaptive", t_end=1e9,
                             tol_abs=1e-6, tol_rel=1e-6), None, 200)]
    if case == "c4":
        g = srk.Grid((1024, 1024))
        ic = lambda cfg: srk.rt_tanh_init(g, width=0.05, amp=1e-3, kmax=8, seed=4)  # noqa: E731
        rt = spec("rayleigh_taylor", (1e4, 1.0, 1.0))
        base = dict(grid_shape=(1024, 1024), problem=rt, t_end=10.0, lengths=g.lengths)
        return [("bs5", dict(base, integrator="bs5", mode="adaptive", tol_abs=1e-6, tol_rel=1e-6), ic, None),
                ("rk4_h2e-3", dict(base, integrator="rk4", mode="fixed", h=2e-3), ic, None),
                ("rk4_h1e-3", dict(base, integrator="rk4", mode="fixed", h=1e-3), ic, None)]
    if case == "c5":
        hit = spec("hit", 2000.0, a=4.0, energy=0.5, seed=42)
        return [("bs5", dict(grid_shape=(512,) * 3, problem=hit, integrator="bs5", mode="adaptive", t_end=1e9,
                             tol_abs=1e-6, tol_rel=1e-6, forcing=True, k_f=2.0), None, 50)]
    raise SystemExit(f"unknown case {case}")


def main():
    case = sys.argv[1]
    out = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/configs"
    for name, kw, ic, cap in runs(case):
        d = os.path.join(out, f"{case}_{name}")
        os.makedirs(d, exist_ok=True)
        cfg = srk.RunConfig(**kw)
        state = ic(cfg) if ic is not None else srk.make_initial_state(cfg)  # IC outside the timed region
        torch.cuda.synchronize()
        t0 = time.time()
        status = "ok"
        try:
            res = srk.run_simulation(cfg, initial_state=state, max_steps=cap)
        except srk.NonFiniteStateError as exc:  # a fixed step above the stability limit is data, not a crash
            print(json.dumps({"case": case, "run": name, "status": f"non-finite: {exc}"}), flush=True)
            continue
        torch.cuda.synchronize()
        wall = time.time() - t0
        srk.write_diagnostics_csv(res.records, os.path.join(d, "diagnostics.csv"))
        last = res.records[-1]
        print(json.dumps({"case": case, "run": name, "status": status, "grid": list(kw["grid_shape"]),
                          "steps": res.steps, "rhs_evals": res.rhs_evals, "rejections": res.rejections, "t": res.t,
                          "E_kin": last.e_kin, "eps": last.eps, "enstrophy": last.enstrophy,
                          "wall_s": round(wall, 2), "stages_per_s": round(res.rhs_evals / wall, 1),
                          "csv": os.path.join(d, "diagnostics.csv")}), flush=True)


if __name__ == "__main__":
    main()
