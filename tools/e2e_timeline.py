"""Timeline of the host-resident e2e step (bench.py e2e loop) at N^3: CUDA events on
the compute stream and on HostMirror's two copy streams, ms from the step start.
    python tools/e2e_timeline.py [n] [steps]"""

import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_10197_b200 as srk  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    g = srk.Grid((n, n, n))
    rhs = srk.FlowRHS(g, srk.PhysParams(2000.0))
    pair, cfg = srk.make_bs5(), srk.ControllerConfig(tol_abs=1e-6, tol_rel=1e-6)
    y0 = srk.hit_init(g, srk.ProblemSpec("hit", a=4.0, energy=0.5, seed=42)).fields
    ctrl = srk.ControllerState(h=1e-3)
    m = srk.HostMirror(y0)
    m.load_host(y0.cpu())
    planes = srk.forcing_planes(g, 2.0)
    cur = torch.cuda.current_stream()
    marks = []

    def mark(name, stream=None):
        e = torch.cuda.Event(enable_timing=True)
        e.record(stream or cur)
        marks.append((name, e))

    spec = {}

    def hook(v):
        mark("y_new queued")
        m.push(v)
        mark("push done", m._d2h)
        spec["next"] = m.pull(wait=False)
        mark("pull done", m._h2d)

    t = 0.0
    yd = m.pull()
    rows = []
    for it in range(steps):
        marks.clear()
        mark("start")
        fd = rhs(t, yd)
        mark("refresh")
        srk.diagnostics.reduce_sums(g, yd, fl=fd, flags=2, ncomp=3, host=True).tolist()
        mark("record")
        out = srk.adaptive_advance(yd, t, pair, ctrl, cfg, rhs, first_stage=fd, grid=g, on_y_new=hook)
        mark("advance")
        srk.apply_forcing(out.y_new, g, 0.5, 2.0, energy_sum=out.diag_sums[4])
        mark("forcing")
        m.push(out.y_new, planes=planes)
        mark("patch push", m._d2h)
        t = out.t_new
        del yd, fd
        yd = m.pull(into=spec.pop("next"), planes=planes)
        mark("patch pull", m._h2d)
        mark("end")
        torch.cuda.synchronize()
        t0 = marks[0][1]
        rows.append({"step": it, "rej": out.rejections,
                     **{k: round(t0.elapsed_time(e), 2) for k, e in marks[1:]}})
        print(json.dumps(rows[-1]), flush=True)


if __name__ == "__main__":
    main()
