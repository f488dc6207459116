"""Measured on-chip ceilings of this B200 (srk_probe): fp64 FMA / add rates,
shared-memory 16 B load rate, warp-shuffle rate, and whether shuffles and
shared loads share one datapath.  One JSON line; used for the z-pass roofline.

    python tools/probe_peaks.py [--sustain-s 3]
Burst: best of 5 single launches.  Sustained: launches back to back for
--sustain-s seconds, the rate of the whole run (power-capped clocks).
"""
import argparse
import ctypes
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_10197_b200 import _native  # noqa: E402


def run(mode, iters, bps, scratch, reps=5):
    lib = _native.load()
    ops = ctypes.c_double(0)
    best = None
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _native.check(lib.srk_probe(mode, iters, bps, _native.ptr(scratch), _native.stream_ptr(), ctypes.byref(ops)),
                      "srk_probe")
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1)
        best = ms if best is None else min(best, ms)
    return ops.value, best


def sustained(mode, iters, bps, scratch, seconds):
    lib = _native.load()
    ops = ctypes.c_double(0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 0
    t0 = time.time()
    e0.record()
    while time.time() - t0 < seconds:
        for _ in range(4):
            lib.srk_probe(mode, iters, bps, _native.ptr(scratch), _native.stream_ptr(), ctypes.byref(ops))
            n += 1
        torch.cuda.current_stream().synchronize()
    e1.record()
    e1.synchronize()
    return ops.value * n, e0.elapsed_time(e1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sustain-s", type=float, default=3.0)
    a = ap.parse_args()
    torch.cuda.init()
    nsm = torch.cuda.get_device_properties(0).multi_processor_count
    scratch = torch.zeros(max(64 * nsm, 8192), dtype=torch.float64, device="cuda")
    out = {"sms": nsm}
    run(0, 1000, 4, scratch, reps=2)  # warm-up
    ops, ms = run(0, 20000, 4, scratch)
    out["fp64_fma_tflops_burst"] = round(2 * ops / (ms * 1e-3) / 1e12, 2)
    out["fp64_fma_per_clk_sm_at_1965"] = round(ops / (ms * 1e-3) / nsm / 1.965e9, 1)
    ops, ms = run(1, 20000, 4, scratch)
    out["fp64_add_gops_burst"] = round(ops / (ms * 1e-3) / 1e9, 1)
    ops, ms = sustained(0, 20000, 4, scratch, a.sustain_s)
    out["fp64_fma_tflops_sustained"] = round(2 * ops / (ms * 1e-3) / 1e12, 2)
    ops, ms = run(2, 4000, 4, scratch)
    out["lds128_TBps_burst"] = round(16 * ops / (ms * 1e-3) / 1e12, 2)
    out["lds128_B_per_clk_sm_at_1965"] = round(16 * ops / (ms * 1e-3) / nsm / 1.965e9, 1)
    ops, ms = run(3, 4000, 4, scratch)
    out["shfl32_per_clk_sm_at_1965"] = round(ops / (ms * 1e-3) / nsm / 1.965e9, 1)
    ops_mix, ms_mix = run(4, 4000, 4, scratch)
    # mixed: 2 LDS.128 (8 wavefronts / warp) + 8 SHFL per trip
    out["mix_ms"] = round(ms_mix, 4)
    _, ms_l = run(2, 1000, 4, scratch)  # 8 LDS per trip x 1000 = same LDS count as mix (2 x 4000)
    _, ms_s = run(3, 4000, 4, scratch)
    out["mix_lds_only_ms"] = round(ms_l, 4)
    out["mix_shfl_only_ms"] = round(ms_s, 4)
    out["shfl_shares_lds_path"] = bool(ms_mix > 0.8 * (ms_l + ms_s))
    # global loads served from L1 vs shared loads: separate or shared datapath?
    ops, ms = run(5, 4000, 4, scratch)
    out["ldg128_L1hit_B_per_clk_sm_at_1965"] = round(16 * ops / (ms * 1e-3) / nsm / 1.965e9, 1)
    _, ms_gl = run(6, 4000, 4, scratch)        # 2 LDG + 2 LDS per trip
    _, ms_g = run(5, 1000, 4, scratch)         # 8 LDG per trip x 1000 = the same LDG count
    _, ms_l2 = run(2, 1000, 4, scratch)        # 8 LDS per trip x 1000 = the same LDS count
    out["mix_ldg_lds_ms"] = round(ms_gl, 4)
    out["ldg_only_ms"] = round(ms_g, 4)
    out["lds_only_ms"] = round(ms_l2, 4)
    out["ldg_shares_lds_path"] = bool(ms_gl > 0.8 * (ms_g + ms_l2))
    out["device"] = torch.cuda.get_device_name(0)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
