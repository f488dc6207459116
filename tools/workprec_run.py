"""Work-precision sweep on the B200 (the paper's headline comparison, reference
bench.py:26-128 via paper_1810_10197_b200.workprec): RK4 fixed steps vs the
adaptive embedded pairs (BS5, DP5, KCL5), scored against a fine fixed-step RK4
run, at the grid sizes the paper uses rather than desk scale.

    python tools/workprec_run.py CASE [OUTDIR]     CASE: tg128 | hit256 | tg512

Writes OUTDIR/workprec_CASE.csv (the reference's CSV layout) and prints one JSON
summary line: per integrator the (rhs_evals, error) points, and the RHS
evaluations BS5 needs for the error RK4 reaches at each of its step sizes
(log-log interpolation along the BS5 tolerance sweep) -> the evaluation savings.
"""

import json
import math
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_10197_b200 as srk  # noqa: E402

CASES = {
    # Taylor-Green, Re = 1600 (configs 1/2), to t = 1
    "tg128": dict(shape=(128,) * 3, problem=srk.ProblemSpec("taylor_green", srk.PhysParams(1600.0)), t_end=1.0,
                  rk4=(0.04, 0.02, 0.01), tols=(1e-3, 1e-4, 1e-5, 1e-6, 1e-7), ref_h=0.001),
    # decaying HIT (config 3 IC, Re = 1000), to t = 0.5
    "hit256": dict(shape=(256,) * 3,
                   problem=srk.ProblemSpec("hit", srk.PhysParams(1000.0), a=4.0, energy=0.5, seed=42), t_end=0.5,
                   rk4=(0.01, 0.005, 0.0025), tols=(1e-3, 1e-4, 1e-5, 1e-6), ref_h=0.00025),
    # Taylor-Green at the config-5 grid, to t = 0.5
    "tg512": dict(shape=(512,) * 3, problem=srk.ProblemSpec("taylor_green", srk.PhysParams(1600.0)), t_end=0.5,
                  rk4=(0.025, 0.0125, 0.00625), tols=(1e-4, 1e-5, 1e-6), ref_h=0.000625),
}


def main():
    case = sys.argv[1]
    out = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out"
    c = CASES[case]
    base = srk.RunConfig(grid_shape=c["shape"], problem=c["problem"], integrator="rk4", mode="fixed",
                         t_end=c["t_end"], h=c["rk4"][0])
    cells = [srk.cell_config(base, "rk4", "fixed", h) for h in c["rk4"]]
    for name in ("bs5", "dp5", "kcl5"):
        cells += [srk.cell_config(base, name, "adaptive", tol) for tol in c["tols"]]
    ref = srk.cell_config(base, "rk4", "fixed", c["ref_h"])
    t0 = time.time()
    points, _ = srk.work_precision(cells, ref)
    wall = time.time() - t0
    os.makedirs(out, exist_ok=True)
    srk.write_work_precision_csv(points, os.path.join(out, f"workprec_{case}.csv"))
    res = {"case": case, "shape": c["shape"], "t_end": c["t_end"], "ref_h": c["ref_h"], "wall_s": round(wall, 1)}
    for kind in ("l2_final", "eps_series"):
        pts = {}
        for p in points:
            if p.kind == kind and p.status == "ok":
                pts.setdefault(p.integrator, []).append((p.setting, p.rhs_evals, p.error))
        res[kind] = pts
        # BS5 evaluations for RK4's error levels (log-log interpolation over the tolerance sweep)
        bs = sorted((e, n) for _, n, e in pts.get("bs5", []) if e > 0)
        sav = []
        for h, n_rk4, e_rk4 in pts.get("rk4", []):
            if len(bs) < 2 or not (bs[0][0] <= e_rk4 <= bs[-1][0]):
                sav.append({"rk4_h": h, "rk4_evals": n_rk4, "error": e_rk4, "bs5_evals": None})
                continue
            le = [math.log(e) for e, _ in bs]
            ln = [math.log(n) for _, n in bs]
            n_bs = math.exp(float(np.interp(math.log(e_rk4), le, ln)))
            sav.append({"rk4_h": h, "rk4_evals": n_rk4, "error": e_rk4, "bs5_evals": round(n_bs, 1),
                        "rk4_over_bs5": round(n_rk4 / n_bs, 3)})
        res[f"{kind}_rk4_vs_bs5"] = sav
    print(json.dumps(res))


if __name__ == "__main__":
    main()
