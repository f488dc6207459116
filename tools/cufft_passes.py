"""Per-pass vendor comparison at 512^3 (NOT the product path): each axis pass of
srk_rhs against cuFFT fp64 (torch.fft) doing the same batched transforms on the
same shapes, timed with CUDA events on one box.

    python tools/cufft_passes.py [--n 512]

Pass-by-pass equivalents (M = 3N/2, K = N/2 + 1; padding / truncation left to
cuFFT's n= argument, which pads at the end instead of the 3/2-rule's middle band
-- same transform sizes and counts):
  K1  ifft(n=M) along x of 5 signals (N, N, K) -> (M, N, K)   [ours: + k_x u1, k_x u2 on load]
  K2  ifft(n=M) along y of 6 signals (M, N, K) -> (M, M, K)   [ours: + the curl on load]
  K3  irfft(n=M) along z of 6 signals + rfft of 3 signals      [ours: two-for-one, u x w in registers,
                                                                truncation to K modes]
  K4  fft along y of 3 signals (M, M, K), keep N rows         [ours: truncation + Nyquist zeroing]
  K5  fft along x of 3 signals (M, N, K), keep N rows          [ours: + scale, Nyquist / DC fixes]
cuFFT does no padding-aware pruning and no fusion; for K3 the separate cross
product (torch elementwise) is timed too.  One JSON line.
"""
import argparse
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_10197_b200 as srk  # noqa: E402
from paper_1810_10197_b200 import _native  # noqa: E402


def t(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=512)
    n = ap.parse_args().n
    m, k = 3 * n // 2, n // 2 + 1
    dev = "cuda"
    # ours: per-kernel event times of one srk_rhs (random input; FFT cost is data independent)
    g = srk.Grid((n, n, n))
    y = torch.randn((3,) + g.kshape, dtype=torch.complex128, device=dev)
    f = torch.empty_like(y)
    rhs = srk.FlowRHS(g, srk.PhysParams(1000.0))
    rhs(0.0, y)
    pl = rhs.plan
    acc = np.zeros(6)
    for _ in range(3):
        ms = (ctypes.c_float * 16)()
        rc = pl.lib.srk_rhs_timed(pl.bind(), _native.ptr(y), _native.ptr(f), 1e-3, 1.0, 1000.0,
                                  _native.stream_ptr(), ms, 16)
        acc += np.array(ms[:6])
    ours = acc / 3
    del y, f, rhs
    torch.cuda.empty_cache()
    out = {"n": n, "passes": {}}

    def rec(name, ours_ms, cufft_ms, extra=None):
        d = {"ours_ms": round(float(ours_ms), 3), "cufft_ms": round(float(cufft_ms), 3),
             "cufft_over_ours": round(float(cufft_ms / ours_ms), 2)}
        if extra:
            d.update(extra)
        out["passes"][name] = d
        print(name, d, file=sys.stderr, flush=True)

    x = torch.randn(5, n, n, k, dtype=torch.complex128, device=dev)
    rec("K1_x_inverse", ours[0], t(lambda: torch.fft.ifft(x, n=m, dim=1)))
    del x
    torch.cuda.empty_cache()
    x = torch.randn(6, m, n, k, dtype=torch.complex128, device=dev)
    rec("K2_y_inverse", ours[1], t(lambda: torch.fft.ifft(x, n=m, dim=2)))
    del x
    torch.cuda.empty_cache()
    z = torch.randn(6, m, m, k, dtype=torch.complex128, device=dev)
    ms_i = t(lambda: torch.fft.irfft(z, n=m, dim=3), reps=2)
    del z
    torch.cuda.empty_cache()
    r = torch.randn(6, m, m, m, dtype=torch.float64, device=dev)
    o = torch.empty(3, m, m, m, dtype=torch.float64, device=dev)

    def cross():
        torch.mul(r[1], r[5], out=o[0]).sub_(r[2] * r[4])
        torch.mul(r[2], r[3], out=o[1]).sub_(r[0] * r[5])
        torch.mul(r[0], r[4], out=o[2]).sub_(r[1] * r[3])

    ms_x = t(cross, reps=2)
    del r
    torch.cuda.empty_cache()
    ms_f = t(lambda: torch.fft.rfft(o, dim=3), reps=2)
    del o
    torch.cuda.empty_cache()
    rec("K3_z_c2r_cross_r2c", ours[2], ms_i + ms_x + ms_f,
        {"cufft_irfft6_ms": round(ms_i, 3), "torch_cross_ms": round(ms_x, 3), "cufft_rfft3_ms": round(ms_f, 3)})
    x = torch.randn(3, m, m, k, dtype=torch.complex128, device=dev)
    rec("K4_y_forward", ours[3], t(lambda: torch.fft.fft(x, dim=2)))
    del x
    torch.cuda.empty_cache()
    x = torch.randn(3, m, n, k, dtype=torch.complex128, device=dev)
    rec("K5_x_forward", ours[4], t(lambda: torch.fft.fft(x, dim=1)))
    del x
    tot_o = float(sum(ours[:5]))
    tot_c = sum(v["cufft_ms"] for v in out["passes"].values())
    out["sum_passes"] = {"ours_ms": round(tot_o, 3), "cufft_ms": round(tot_c, 3),
                         "cufft_over_ours": round(tot_c / tot_o, 2)}
    out["note"] = ("cuFFT via torch.fft, same batched transform sizes/counts per pass; cuFFT pads at the end "
                   "(n=) and returns all outputs (no truncation, no fusion). Ours: live srk_rhs_timed.")
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
