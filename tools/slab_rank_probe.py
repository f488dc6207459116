"""One rank of a P-way slab decomposition on one GPU: the rank's kernels timed for
real (CUDA events), the two all-to-alls replaced by no-ops and modelled from their
byte counts.  A projection for the multi-GPU configs gpurun cannot provide (config 5:
1024^3 on 4 / 8 B200), not a multi-GPU measurement.

    python tools/slab_rank_probe.py N P [steps]

Prints one JSON line: per-RHS kernel-group times of rank 0, BS5 step time of the
rank (7 RHS + stage sums + reduction, no forcing), the exchange bytes per rank per
RHS, and the per-stage time / strong-scaling efficiency implied with the exchanges
fully exposed and fully hidden at the measured 770 GB/s peer-copy rate
(B200_PROFILING.md), against the 1-GPU 512^3 stage time given by --t1 (ms).
"""

import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_10197_b200 as srk  # noqa: E402
from paper_1810_10197_b200.slab import SlabFlowRHS, hit_slab, slab_geometry  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("n", type=int)
ap.add_argument("P", type=int)
ap.add_argument("steps", type=int, nargs="?", default=3)
ap.add_argument("--t1", type=float, default=1000.0 / 37.3, help="1-GPU 512^3 ms per stage (bench value)")
ap.add_argument("--nvlink", type=float, default=770.0, help="GB/s per direction per GPU")
a = ap.parse_args()

n, P = a.n, a.P
g = srk.Grid((n, n, n))
params = srk.PhysParams(reynolds=2000.0)
geo = slab_geometry(g, P)
rhs = SlabFlowRHS(g, params, 0, P, exchange=lambda r, s: None)
rhs.recv1.zero_()
rhs.recv2.zero_()
y = hit_slab(g, 0, P, a=4.0, energy=0.5, seed=42)
f = torch.empty_like(y)
be = rhs.backend


def ev():
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    return e


for _ in range(2):
    rhs(0.0, y, out=f)
torch.cuda.synchronize()
grp = []
for _ in range(3):
    e = [ev()]
    be.forward(y, rhs.send1)
    e.append(ev())
    be.middle(rhs.recv1, rhs.send2)
    e.append(ev())
    be.finish(rhs.recv2, y, f)
    e.append(ev())
    torch.cuda.synchronize()
    grp.append([e[i].elapsed_time(e[i + 1]) for i in range(3)])
grp = [min(x[i] for x in grp) for i in range(3)]
K = geo["K"]
split = []
for _ in range(3):  # the middle group kernel by kernel (kz-chunk entry points over all kz)
    e = [ev()]
    be.inverse_y_kz(rhs.recv1, 0, K)
    e.append(ev())
    be.zpass()
    e.append(ev())
    be.forward_y_kz(rhs.send2, 0, K)
    e.append(ev())
    torch.cuda.synchronize()
    split.append([e[i].elapsed_time(e[i + 1]) for i in range(3)])
split = [round(min(x[i] for x in split), 3) for i in range(3)]

pair = srk.make_bs5()
cfg = srk.ControllerConfig(tol_abs=1e-6, tol_rel=1e-6)
st = srk.ControllerState(h=1e-3)
fs = rhs(0.0, y)
t = 0.0
out = srk.adaptive_advance(y, t, pair, st, cfg, rhs, first_stage=fs, grid=g, plan=be.h)  # warm-up
torch.cuda.synchronize()
e0 = ev()
evals = 0
for _ in range(a.steps):
    st.h = 1e-3  # fixed attempt size: the partial sums of one rank steer nothing real
    out = srk.adaptive_advance(out.y_new, out.t_new, pair, st, cfg, rhs, first_stage=out.last_stage, grid=g,
                               plan=be.h)
    evals += out.rhs_evals
e1 = ev()
torch.cuda.synchronize()
stage_ms = e0.elapsed_time(e1) / evals

xbytes = (geo["send1"] + geo["send2"]) * 16 * (P - 1) / P  # sent (= received) per rank per RHS
x_ms = xbytes / (a.nvlink * 1e9) * 1e3
m = 3 * n // 2
k = n // 2 + 1


def bstage(nn):
    mm, kk = 3 * nn // 2, nn // 2 + 1
    sc, sx, sxy = nn * nn * kk, mm * nn * kk, mm * mm * kk
    return 16 * (9 * sc + 18 * sx + 18 * sxy) + 50.0 / 7.0 * 3 * sc * 16


def eff(ms):  # per-GPU model bandwidth at P over the 1-GPU 512^3 one
    return (bstage(n) / (P * ms)) / (bstage(512) / a.t1)


res = {"n": n, "P": P, "rank_rhs_ms": {"forward": round(grp[0], 3), "middle": round(grp[1], 3),
                                        "finish": round(grp[2], 3), "sum": round(sum(grp), 3),
                                        "K2_K3_K4": split},
       "rank_stage_ms": round(stage_ms, 3), "exchange_GB_per_rank_per_rhs": round(xbytes / 1e9, 3),
       "exchange_ms_at_nvlink": round(x_ms, 3),
       "projected_stage_ms": {"exposed": round(stage_ms + x_ms, 3), "hidden": round(stage_ms, 3)},
       "projected_stages_per_s": {"exposed": round(1e3 / (stage_ms + x_ms), 2), "hidden": round(1e3 / stage_ms, 2)},
       "projected_E_P": {"exposed": round(eff(stage_ms + x_ms), 3), "hidden": round(eff(stage_ms), 3)},
       "t1_512_ms_per_stage": a.t1, "mem_GB": round(torch.cuda.max_memory_allocated() / 1e9, 1),
       "note": "one rank's kernels measured; all-to-alls modelled (no-op here), not a multi-GPU measurement"}
print(json.dumps(res))
