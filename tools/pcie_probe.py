"""PCIe probe for the host-resident e2e path: pinned H2D / D2H of one 512^3 state
(3.23 GB) alone, both directions at once (HostMirror chunks), and D2H under a
running RHS.  Prints one JSON line.   python tools/pcie_probe.py [n]"""

import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_10197_b200 as srk  # noqa: E402


def timed(fn, reps=3):
    st = torch.cuda.current_stream()
    out = []
    for _ in range(reps):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b))
    return min(out)


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
    g = srk.Grid((n, n, n))
    y = srk.hit_init(g, srk.ProblemSpec("hit", a=4.0, energy=0.5, seed=42)).fields
    nb = y.numel() * y.element_size()
    m = srk.HostMirror(y)
    m.load_host(y.cpu())
    h2 = torch.empty_like(m.host).pin_memory()
    res = {"bytes": nb}
    res["h2d_ms"] = timed(lambda: y.copy_(m.host, non_blocking=True))
    res["d2h_ms"] = timed(lambda: m.host.copy_(y, non_blocking=True))

    def both():
        m.push(y)
        z = m.pull()
        m.wait()
        del z
    res["push_then_pull_ms"] = timed(both)

    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    y2 = torch.empty_like(y)

    def duplex():
        cur = torch.cuda.current_stream()
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            m.host.copy_(y, non_blocking=True)
        with torch.cuda.stream(s2):
            y2.copy_(h2, non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)
    res["independent_duplex_ms"] = timed(duplex)

    rhs = srk.FlowRHS(g, srk.PhysParams(2000.0))
    f = rhs(0.0, y)
    res["rhs_ms"] = timed(lambda: rhs(0.0, y))

    def rhs_and_push():
        m.push(y)
        rhs(0.0, y)
        m.wait()
    res["rhs_with_push_ms"] = timed(rhs_and_push)
    res["gbs"] = {k: nb / (v * 1e-3) / 1e9 for k, v in res.items() if k.endswith("_ms") and "rhs" not in k}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
