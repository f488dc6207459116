"""Read-only / write-only / copy DRAM bandwidth on this GPU (torch kernels; CUDA events, best of 5).

    python tools/dram_rw_probe.py [GiB]
The strided passes are write-heavy (K1 71 %, K2 64 % writes) or read-heavy (K4, K5 60 % reads): their
byte rooflines differ if the two directions do.
"""
import json
import sys

import torch

gib = float(sys.argv[1]) if len(sys.argv) > 1 else 8.0
n = int(gib * (1 << 30) / 8)
a = torch.empty(n, dtype=torch.float64, device="cuda")
b = torch.empty(n, dtype=torch.float64, device="cuda")
a.fill_(1.0)


def best(fn, reps=5):
    t = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        t.append(e0.elapsed_time(e1))
    return min(t)


fn_w = lambda: b.fill_(2.0)
fn_r = lambda: a.sum()
fn_c = lambda: b.copy_(a)
fn_w(); fn_r(); fn_c()
tw, tr, tc = best(fn_w), best(fn_r), best(fn_c)
by = n * 8
print(json.dumps({"GiB": gib, "write_only_GBps": round(by / tw / 1e6, 1), "read_only_GBps": round(by / tr / 1e6, 1),
                  "copy_GBps_rw": round(2 * by / tc / 1e6, 1)}))
