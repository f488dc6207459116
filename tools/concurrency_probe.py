"""Do the fp64-bound z-pass (K3) and the latency/DRAM-bound strided passes (K2, K4)
overlap when they run concurrently on two streams?  Two independent slab plans
(nranks = 1, own workspaces) at N^3; device times with CUDA events.
    python tools/concurrency_probe.py [n]"""

import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_10197_b200 as srk  # noqa: E402
from paper_1810_10197_b200.slab import CudaSlabBackend, slab_geometry  # noqa: E402


def timed(fn, reps=3):
    best = 1e30
    for _ in range(reps):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return round(best, 3)


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
    g = srk.Grid((n, n, n))
    geo = slab_geometry(g, 1)
    K = geo["K"]
    p = srk.PhysParams(1000.0)
    be = [CudaSlabBackend(g, p, 0, 1) for _ in range(2)]
    ys = [torch.randn((3,) + g.kshape, dtype=torch.complex128, device="cuda") for _ in range(2)]
    fs = [torch.empty_like(y) for y in ys]
    s1 = [be[i].empty(geo["send1"]) for i in range(2)]
    s2 = [be[i].empty(geo["send2"]) for i in range(2)]
    lo, hi = torch.cuda.Stream(priority=0), torch.cuda.Stream(priority=-1)

    def rhs(i):
        be[i].forward(ys[i], s1[i])
        be[i].middle(s1[i], s2[i])
        be[i].finish(s2[i], ys[i], fs[i])

    for i in range(2):
        rhs(i)
    torch.cuda.synchronize()
    res = {"n": n}

    def on(stream, fn):
        cur = torch.cuda.current_stream()
        stream.wait_stream(cur)
        with torch.cuda.stream(stream):
            fn()
        cur.wait_stream(stream)

    k2 = lambda i: be[i].inverse_y_kz(s1[i], 0, K)  # noqa: E731
    k3 = lambda i: be[i].zpass()  # noqa: E731
    k4 = lambda i: be[i].forward_y_kz(s2[i], 0, K)  # noqa: E731
    res["rhs"] = timed(lambda: rhs(0))
    res["rhs_x2_serial"] = timed(lambda: (rhs(0), rhs(1)))
    res["rhs_x2_concurrent"] = timed(lambda: (on(lo, lambda: rhs(0)), on(hi, lambda: rhs(1))))
    res["k2"] = timed(lambda: k2(1))
    res["k3"] = timed(lambda: k3(0))
    res["k4"] = timed(lambda: k4(1))
    res["k3_k2_serial"] = timed(lambda: (k3(0), k2(1)))
    res["k3_k2_concurrent"] = timed(lambda: (on(lo, lambda: k3(0)), on(hi, lambda: k2(1))))
    res["k3_k2_concurrent_k2first"] = timed(lambda: (on(hi, lambda: k2(1)), on(lo, lambda: k3(0))))
    res["k3_k4_concurrent"] = timed(lambda: (on(lo, lambda: k3(0)), on(hi, lambda: k4(1))))
    res["k3_k2k4_concurrent"] = timed(lambda: (on(lo, lambda: k3(0)), on(hi, lambda: (k2(1), k4(1)))))
    print(json.dumps(res))


if __name__ == "__main__":
    main()
