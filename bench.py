"""Throughput bench: adaptive BS5 steps of the forced-HIT workload (BASELINE config 5)
at N^3 fp64 on the B200 path, one JSON line on rank 0.

A "step" = one accepted adaptive BS5 step through the drop-in API
(adaptive_advance + energy-restoring forcing + cached-tendency refresh +
diagnostics record), i.e. 8 RHS evaluations per accepted step (7 stages, FSAL
invalidated by the forcing, simulation.py:165-182).  The metric is RK stages
(RHS evaluations, the reference's rhs_evals accounting) per second.

    python bench.py                       # N=1, 512^3, K=10, W=3
    python bench.py --impl reference      # CPU oracle port (the reference's algorithm)
    python bench.py --gpus N              # re-launches itself under torchrun: N ranks, y-slab
                                          # decomposed N^3 (strong scaling); at N >= 4 also a
                                          # 1024^3 leg with SURVEY M4's E_P
    torchrun --nproc-per-node N bench.py --gpus N   # the same, launched by the caller
    python bench.py --gpus 2 --dry-run    # launcher check on CPU (gloo ranks, no GPU work)
    python bench.py --mode slab --grid 256  # the slab path on one GPU (NCCL world of 1)
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "RK stages/sec (BS5 adaptive, forced HIT, N^3 fp64)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--grid", dest="n", type=int, default=512, help="N of the N^3 grid")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--chunks", type=int, default=None,
                    help="slab mode: kz chunks of the pipelined RHS (exchange of chunk c overlaps chunk c+1); "
                         "default 4 for N > 1, 1 on a single GPU (nothing to overlap)")
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "peer"],
                    help="slab mode: nccl = all_to_all_single (kz-chunk pipelined); peer = the exchange fused "
                         "into K1 / K4 (row blocks stored into the peers' receive buffers over CUDA IPC)")
    ap.add_argument("--mode", default="auto", choices=["auto", "single", "slab", "replicas"],
                    help="auto: single GPU at N=1, slab decomposition (strong scaling) for N>1")
    ap.add_argument("--dry-run", action="store_true",
                    help="launcher / rank plumbing only: gloo ranks on the CPU, no GPU work (tests)")
    ap.add_argument("--no-1024", action="store_true", help="N >= 4: skip the 1024^3 E_P leg")
    ap.add_argument("--ep-test", type=int, nargs=2, default=None, metavar=("N_BIG", "N_BASE"),
                    help="slab mode: run the E_P leg at any world size with N_BIG^3 slabs and an N_BASE^3 "
                         "single-GPU baseline (exercises the 1024^3 code path on small grids)")
    return ap.parse_args()


def model_bytes(n):
    """SURVEY §8(d) M3 byte model (3/2-rule padded algorithm, complex128) for the
    stage fraction; per kernel, the bytes each launch of this implementation must
    move: K1 writes 5 x-padded signals [u0, u1, u2, kx u1, kx u2] (the curl is
    finished in K2), K2 reads those 5 and writes 6."""
    m, k = 3 * n // 2, n // 2 + 1
    sc, sx, sxy = n * n * k, m * n * k, m * m * k
    b_rhs = 16 * (9 * sc + 18 * sx + 18 * sxy)
    f = 3 * sc * 16
    per_kernel = {  # algorithmic bytes each kernel of srk_rhs must move
        "K1_xinv_curl": 16 * (3 * sc + 5 * sx),
        "K2_yinv": 16 * (5 * sx + 6 * sxy),
        "K3_z_c2r_cross_r2c": 16 * (6 * sxy + 3 * sxy),
        "K4_yfwd": 16 * (3 * sxy + 3 * sx),
        "K5_xfwd": 16 * (3 * sx + 3 * sc),
        "K6_project": 16 * (3 * sc + 3 * sc + 3 * sc),
    }
    return dict(b_rhs=b_rhs, b_stage_bs5=b_rhs + 50.0 / 7.0 * f, per_kernel=per_kernel)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def source_hash():
    """srk_source_hash() of the loaded libsrk: kernel sources + compile flags."""
    from paper_1810_10197_b200 import _native

    return _native.load().srk_source_hash().decode()


def ncu_counters(n, kernel):
    """Per-launch ncu counters of `kernel` at N = n from profiles/ncu_kernels.json,
    only if that capture was taken of a build of the same kernel sources and flags
    as the library loaded now (srk_source_hash match); otherwise None -- stale
    counters are never reported."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_kernels.json")) as fh:
            d = json.load(fh)
    except Exception:
        return None, "no profiles/ncu_kernels.json"
    if d.get("source_hash") != source_hash():
        return None, "profiles/ncu_kernels.json was captured from other kernel sources"
    e = d.get(str(n), {}).get(kernel)
    return e, d.get("report")


def probe_peaks():
    """Live on-chip ceilings (srk_probe, burst): fp64 FMA rate and the shared-memory
    datapath (16 B loads), for the z-pass's non-HBM roofline."""
    import ctypes

    import torch

    from paper_1810_10197_b200 import _native

    lib = _native.load()
    nsm = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    scratch = torch.zeros(64 * nsm, dtype=torch.float64, device="cuda")
    out = {}
    for mode, iters, key in ((0, 20000, "fp64"), (2, 4000, "smem")):
        ops = ctypes.c_double(0)
        best = None
        for _ in range(4):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            _native.check(lib.srk_probe(mode, iters, 4, _native.ptr(scratch), _native.stream_ptr(),
                                        ctypes.byref(ops)), "srk_probe")
            e1.record()
            e1.synchronize()
            ms = e0.elapsed_time(e1)
            best = ms if best is None else min(best, ms)
        out[key] = 2 * ops.value / (best * 1e-3) / 1e12 if mode == 0 else 16 * ops.value / (best * 1e-3) / 1e9
    return {"fp64_tflops": out["fp64"], "smem_GBps": out["smem"],
            "source": "srk_probe in this process: 8 independent DFMA chains / conflict-free 16 B shared loads, "
                      "4 CTAs x 256 threads per SM, best of 4 launches"}


class ClockSampler:
    """SM clocks / throttle reasons during the timed region, sampled every 0.2 s.

    Uses NVML in-process (no fork of the CUDA process: spawning nvidia-smi every
    0.2 s from a host-bound run measurably slowed the 256^3 steps); falls back
    to the nvidia-smi CLI when NVML is unavailable."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    BITS = (("hw_slowdown", 8), ("hw_thermal_slowdown", 64), ("sw_thermal_slowdown", 32), ("sw_power_cap", 4))

    def __init__(self, index):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._th = threading.Thread(target=self._run, daemon=True)
        self._nvml = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self._nvml = pynvml
        except Exception:
            self._nvml = None

    def _sample(self):
        if self._nvml is not None:
            p = self._nvml
            sm = p.nvmlDeviceGetClockInfo(self._h, p.NVML_CLOCK_SM)
            mx = p.nvmlDeviceGetMaxClockInfo(self._h, p.NVML_CLOCK_SM)
            r = p.nvmlDeviceGetCurrentClocksEventReasons(self._h)
            return [str(sm), str(mx), hex(r)] + ["Active" if r & b else "Not Active" for _, b in self.BITS]
        out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True,
                             timeout=5).stdout.strip()
        return [c.strip() for c in out.split(",")] if out else None

    def _run(self):
        if os.environ.get("SRK_BENCH_NO_CLOCKS"):  # diagnostics only: no sampling
            return
        while not self._stop.is_set():
            try:
                row = self._sample()
                if row:
                    self.rows.append(row)
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._th.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._th.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = [n for n, _ in self.BITS]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 3 + i and r[3 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows),
                "source": "nvml" if self._nvml is not None else "nvidia-smi"}


# ---------------------------------------------------------------------------
# CPU oracle leg (reference algorithm restated; bench-only use of oracle/)
# ---------------------------------------------------------------------------
def cpu_sample(n_target, steps=1, n_sample=128, workers=None):
    import oracle as O

    workers = workers or (os.cpu_count() or 1)
    O.set_fft_workers(workers)
    og = O.OGrid((n_sample,) * 3)
    y = O.hit(og, a=4.0, energy=0.5, seed=42)
    f = O.OracleRHS(og, 2000.0)
    tab = O.tableau("bs5")
    st = O.CtrlState(h=1e-3)
    fnow = f(0.0, y)
    t0 = time.perf_counter()
    evals = 0
    t = 0.0
    for _ in range(steps):
        o = O.adaptive_advance(y, t, tab, st, O.Ctrl(), f, fnow)
        y = o.y_new.copy()
        O.apply_forcing(y[:3], og, 0.5, 2.0)
        fnow = f(t, y)
        evals += o.evals + 1
        t = o.t_new
    dt = time.perf_counter() - t0
    pts = float(n_sample) ** 3
    value = evals / dt * pts / float(n_target) ** 3
    return dict(value=value, unit="stages/s", cores=workers, kind="port",
                sample=(f"oracle port (numpy/scipy, scipy.fft workers={workers}) on {n_sample}^3, {steps} BS5 "
                        f"forced step(s) = {evals} RHS in {dt:.1f} s; scaled by points to {n_target}^3 "
                        f"({evals / dt * pts / 1e9:.4f} Gpts*stage/s)"),
                gpts_stage_per_s=evals / dt * pts / 1e9)


CPU_SAMPLE_N = 128  # both CPU legs: one forced BS5 step on 128^3, scaled by points to N^3


def run_reference(args, rank, world):
    """The reference's own algorithm on the host cores (oracle port: the reference is
    Python, nothing to compile into oracle/_ref), all cores, each step one forced
    BS5 step at 128^3 (~6 s at 16 workers) scaled by points to the bench's N^3."""
    if rank != 0:
        return
    steps_per = 1
    vals = []
    for i in range(args.warmup + args.steps):
        r = cpu_sample(args.n, steps=steps_per, n_sample=min(args.n, CPU_SAMPLE_N))
        if i >= args.warmup:
            vals.append(r)
    v = statistics.median([r["value"] for r in vals])
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "stages/s", "n_gpus": 0,
        "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded HIT spectrum, a=4, E=0.5)",
        "config": {"workload": f"forced_hit_bs5_{args.n}^3", "n": args.n, "nu": 5e-4, "tol": 1e-6, "k_f": 2.0},
        "cpu_baseline": {"value": v, "unit": "stages/s", "cores": vals[-1]["cores"], "kind": "port",
                         "sample": vals[-1]["sample"], "scaled_from": f"{min(args.n, CPU_SAMPLE_N)}^3",
                         "gpts_stage_per_s": statistics.median([r["gpts_stage_per_s"] for r in vals])},
        "e2e": {"value": v, "unit": "stages/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU leg
# ---------------------------------------------------------------------------
def run_native(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_1810_10197_b200 as srk
    from paper_1810_10197_b200 import _native
    from paper_1810_10197_b200.diagnostics import diag_from_sums

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    n = args.n
    g = srk.Grid((n, n, n))
    params = srk.PhysParams(reynolds=2000.0)  # nu = 5e-4 (config 5)
    energy, k_f = 0.5, 2.0
    y0 = srk.hit_init(g, srk.ProblemSpec("hit", a=4.0, energy=energy, seed=42 + rank)).fields
    rhs = srk.FlowRHS(g, params)
    pair = srk.make_bs5()
    cfg = srk.ControllerConfig(tol_abs=1e-6, tol_rel=1e-6)

    def new_state():
        y = y0.clone()
        return dict(y=y, t=0.0, f=rhs(0.0, y), ctrl=srk.ControllerState(h=1e-3))

    a21 = float(pair.A[1, 0])

    def step(s):
        out = srk.adaptive_advance(s["y"], s["t"], pair, s["ctrl"], cfg, rhs, first_stage=s["f"], grid=g,
                                   second_input=s.get("y2"))
        y = out.y_new
        srk.apply_forcing(y, g, energy, k_f, energy_sum=out.diag_sums[4])
        # the cached tendency + diagnostics record of the forced state, with the
        # next step's first stage sum y + h a21 f formed in the same pass
        h = s["ctrl"].h
        f, y2, q = rhs.refresh(out.t_new, y, h * a21)
        s.update(y=y, t=out.t_new, f=f, y2=(h, y2))
        return out.rhs_evals + 1, diag_from_sums(q, g)

    def barrier():
        if world > 1:
            dist.barrier()

    s = new_state()
    for _ in range(args.warmup):
        step(s)
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    evals = 0
    l0 = _native.LAUNCHES
    with ClockSampler(local_rank) as clk:
        e0.record(st)
        per_step = []  # diagnostics (SRK_BENCH_STEPS=1): device time and RHS count of every step
        for _ in range(args.steps):
            if os.environ.get("SRK_BENCH_STEPS"):
                es = torch.cuda.Event(enable_timing=True)
                es.record(st)
            ev, diag = step(s)
            evals += ev
            if os.environ.get("SRK_BENCH_STEPS"):
                ee = torch.cuda.Event(enable_timing=True)
                ee.record(st)
                per_step.append((es, ee, ev))
        e1.record(st)
        torch.cuda.synchronize()
        if per_step:
            print("per-step ms/evals:", [(round(a.elapsed_time(b), 1), e) for a, b, e in per_step], file=sys.stderr)
    launches = _native.LAUNCHES - l0
    barrier()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    t_sec = torch.tensor([ms / 1e3], dtype=torch.float64, device=dev)
    ev_t = torch.tensor([float(evals)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_sec, op=dist.ReduceOp.MAX)
        dist.all_reduce(ev_t, op=dist.ReduceOp.SUM)
    T = t_sec.item()
    total_evals = ev_t.item()
    value = total_evals / T

    # ---- per-kernel live timing of the RHS (CUDA events between launches) ----
    import ctypes

    pl = rhs.plan
    kn = list(model_bytes(n)["per_kernel"].keys())
    acc = np.zeros(len(kn))
    reps = 3
    yk, fk = s["y"], torch.empty_like(s["y"])
    for _ in range(reps):
        ms_arr = (ctypes.c_float * 16)()
        rc = pl.lib.srk_rhs_timed(pl.bind(), _native.ptr(yk), _native.ptr(fk), 1.0 / params.reynolds, 1.0,
                                  params.reynolds, _native.stream_ptr(), ms_arr, 16)
        if rc > 0:
            _native.check(rc, "srk_rhs_timed")
        acc += np.array(ms_arr[: len(kn)])
    kms = acc / reps
    mb = model_bytes(n)
    shares = kms / kms.sum()
    dom = int(np.argmax(kms))
    peak, peak_src = peaks()
    achieved = mb["per_kernel"][kn[dom]] / (kms[dom] * 1e-3) / 1e9
    # ncu counters of the dominant kernel, only from a capture of this very binary
    cnt, cnt_src = ncu_counters(n, kn[dom])
    traffic = cnt.get("dram_bytes") if cnt else None
    # The z-pass is not bound by HBM: the SM's shared-memory datapath (128 B/clk,
    # shuffles included) and the fp64 pipe are its ceilings.  Live
    # probe peaks; the kernel's wavefront / fp64-instruction counts per launch come
    # from the sha-matched ncu capture.
    ceil = None
    try:
        pk = probe_peaks()
        ceil = {"probe": pk}
        if cnt and cnt.get("smem_wavefronts") is not None:
            sm_gbps = cnt["smem_wavefronts"] * 128 / (kms[dom] * 1e-3) / 1e9
            ceil["smem"] = {"achieved_GBps": sm_gbps, "peak_GBps": pk["smem_GBps"],
                            "frac": sm_gbps / pk["smem_GBps"], "wavefronts_per_launch": cnt["smem_wavefronts"]}
        if cnt and cnt.get("fp64_flops") is not None:
            tf = cnt["fp64_flops"] / (kms[dom] * 1e-3) / 1e12
            ceil["fp64"] = {"achieved_tflops": tf, "peak_tflops": pk["fp64_tflops"], "frac": tf / pk["fp64_tflops"],
                            "flops_per_launch": cnt["fp64_flops"],
                            "counted_as": "2 per DFMA + 1 per DADD/DMUL thread instruction (ncu sass counters)"}
    except Exception as exc:  # the probe is evidence, never a reason to lose the line
        ceil = {"error": str(exc)}

    # ---- e2e: through the public API with the state resident on the host ----
    # The state crosses PCIe every step (hostio.HostMirror, pinned): y is copied
    # host->device, the cached tendency f = rhs(t, y) (the refresh the
    # device-resident loop does at the end of the previous step, same count) and
    # the diagnostics record are computed from it, one adaptive step + forcing
    # runs, and y_new goes back to the host copy the next step reads -- issued as
    # soon as y_new exists, and the next step's host->device chunks follow the
    # device->host ones on the other PCIe direction, both under the FSAL stage and
    # the error reduction (a rejected attempt redoes both); after the accept and
    # the forcing rescale only the band's x-planes go down and up again.
    e2e = None
    if not args.no_e2e:
        s2 = new_state()
        mirror = srk.HostMirror(s2["y"])
        mirror.load_host(s2["y"].cpu())
        fplanes = srk.forcing_planes(g, k_f)
        torch.cuda.synchronize()
        barrier()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev2 = 0
        t2_ = s2["t"]
        n_e2e = max(2, args.steps // 2)
        b_in0, b_out0 = mirror.h2d_bytes, mirror.d2h_bytes
        spec = {}

        def on_y_new(v):  # every attempt: y_new -> host, and the host copy -> the next input
            mirror.push(v)
            spec["next"] = mirror.pull(wait=False)

        def e2e_step(yd, t):
            h = s2["ctrl"].h
            fd, y2, _ = rhs.refresh(t, yd, h * a21)
            out = srk.adaptive_advance(yd, t, pair, s2["ctrl"], cfg, rhs, first_stage=fd, grid=g,
                                       on_y_new=on_y_new, second_input=(h, y2))
            srk.apply_forcing(out.y_new, g, energy, k_f, energy_sum=out.diag_sums[4])
            mirror.push(out.y_new, planes=fplanes)
            ev, t = out.rhs_evals + 1, out.t_new
            del yd, fd, out
            return mirror.pull(into=spec.pop("next"), planes=fplanes), t, ev  # the re-sent planes, then wait

        yd = mirror.pull()
        for _ in range(max(1, min(args.warmup, 2))):  # untimed: first-use costs of the host path
            yd, t2_, _ = e2e_step(yd, t2_)
        mirror.wait()
        torch.cuda.synchronize()
        b_in0, b_out0 = mirror.h2d_bytes, mirror.d2h_bytes
        del yd  # the timed region pulls the (final) host copy itself
        a0.record(st)
        yd = mirror.pull()
        for _ in range(n_e2e):
            yd, t2_, ev = e2e_step(yd, t2_)
            ev2 += ev
        mirror.wait()
        a1.record(st)
        torch.cuda.synchronize()
        t2 = torch.tensor([a0.elapsed_time(a1) / 1e3], dtype=torch.float64, device=dev)
        e2t = torch.tensor([float(ev2)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t2, op=dist.ReduceOp.MAX)
            dist.all_reduce(e2t, op=dist.ReduceOp.SUM)
        e2e = {"value": e2t.item() / t2.item(), "unit": "stages/s",
               "h2d_bytes_per_step": (mirror.h2d_bytes - b_in0) // n_e2e,
               "d2h_bytes_per_step": (mirror.d2h_bytes - b_out0) // n_e2e + 9 * 8,
               "path": "per step: y host->device (pinned HostMirror), cached tendency + diagnostics record + "
                       "first stage sum (FlowRHS.refresh), adaptive_advance (BS5) + forcing through the Python "
                       "API, y_new device->host "
                       "(every attempt's y_new, issued before its FSAL stage, the next step's host->device behind it; "
                       "forcing band planes re-sent both ways); "
                       "same RHS count as the device-resident step; bytes include every attempt's copies"}

    if rank != 0:
        return
    cpu = None
    if world == 1 and not args.no_cpu:
        ns = min(n, CPU_SAMPLE_N)
        c_all = cpu_sample(n, steps=1, n_sample=ns)
        c_one = cpu_sample(n, steps=1, n_sample=ns, workers=1)
        cpu = {k: c_all[k] for k in ("value", "unit", "cores", "kind", "sample")}
        cpu["scaled_from"] = f"{ns}^3"
        cpu["one_core"] = {"value": c_one["value"], "unit": "stages/s", "cores": 1, "sample": c_one["sample"],
                           "note": "BASELINE.md primary: the reference is single-threaded by default"}
    stage_frac = mb["b_stage_bs5"] * (value / world) / (peak * 1e9)
    line = {
        "metric": METRIC, "value": value, "unit": "stages/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": T * 1e3 / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded HIT spectrum E(k)~k^4 exp(-2(k/4)^2), E=0.5, reference hit_init)",
        "config": {"workload": f"forced_hit_bs5_{n}^3", "n": n, "nu": 5e-4, "tol": 1e-6, "k_f": 2.0,
                   "parallelism": f"replicas x{world}" if world > 1 else "single GPU",
                   "l2": "inputs larger than L2 (each field %.2f GB)" % (3 * g.mode_count * 16 / 1e9)},
        "gpts_stage_per_s": value * n ** 3 / 1e9,
        "rhs_evals": total_evals,
        "stage_hbm_frac": stage_frac,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "kernel": kn[dom],
                     "peak_source": peak_src,
                     "kernel_ms": {k: round(float(v), 4) for k, v in zip(kn, kms)},
                     "kernel_share": {k: round(float(v), 4) for k, v in zip(kn, shares)},
                     "algorithmic_bytes_per_launch": mb["per_kernel"][kn[dom]],
                     "traffic_source": cnt_src,
                     "fp64_pipe_active": cnt.get("fp64_pipe") if cnt else None,
                     "on_chip_ceilings": ceil},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)


def run_slab(args, rank, world, local_rank):
    """N^3 grid y-slab decomposed over all ranks; strong scaling."""
    import torch
    import torch.distributed as dist

    import paper_1810_10197_b200 as srk
    from paper_1810_10197_b200 import _native
    from paper_1810_10197_b200.diagnostics import diag_from_sums, reduce_sums
    from paper_1810_10197_b200.slab import SlabFlowRHS, dist_sum_in_rank_order, hit_slab, slab_geometry

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    n = args.n
    g = srk.Grid((n, n, n))
    params = srk.PhysParams(reynolds=2000.0)
    energy, k_f = 0.5, 2.0
    red = dist_sum_in_rank_order()
    chunks = args.chunks if args.chunks is not None else (4 if world > 1 else 1)
    rhs = SlabFlowRHS(g, params, rank, world, chunks=chunks, peer=args.exchange == "peer")
    plan = rhs.backend.h
    y0 = hit_slab(g, rank, world, a=4.0, energy=energy, seed=42, allreduce=red)
    pair = srk.make_bs5()
    cfg = srk.ControllerConfig(tol_abs=1e-6, tol_rel=1e-6)

    def new_state():
        y = y0.clone()
        return dict(y=y, t=0.0, f=rhs(0.0, y), ctrl=srk.ControllerState(h=1e-3))

    def step(s):
        out = srk.adaptive_advance(s["y"], s["t"], pair, s["ctrl"], cfg, rhs, first_stage=s["f"], grid=g,
                                   allreduce=red, plan=plan)
        y = out.y_new
        srk.apply_forcing(y, g, energy, k_f, plan=plan, allreduce=red, slab=(rank, world),
                          energy_sum=out.diag_sums[4])
        f = rhs(out.t_new, y)
        q = red(reduce_sums(g, y, fl=f, flags=2, ncomp=3, plan=plan))
        s.update(y=y, t=out.t_new, f=f)
        return out.rhs_evals + 1, diag_from_sums(q, g)

    s = new_state()
    for _ in range(args.warmup):
        step(s)
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    evals = 0
    l0 = _native.LAUNCHES
    with ClockSampler(local_rank) as clk:
        e0.record(st)
        for _ in range(args.steps):
            ev, _ = step(s)
            evals += ev
        e1.record(st)
        torch.cuda.synchronize()
    launches = _native.LAUNCHES - l0
    dist.barrier()
    t_sec = torch.tensor([e0.elapsed_time(e1) / 1e3], dtype=torch.float64, device=dev)
    dist.all_reduce(t_sec, op=dist.ReduceOp.MAX)
    T = t_sec.item()
    value = evals / T  # every rank works on the same global stages

    # phase timing of one RHS: 3 kernel groups + 2 exchanges (max over ranks)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(7)]
    yk = s["y"]
    fk = torch.empty_like(yk)
    b = rhs.backend
    def xchg(r, sd):
        w = rhs.exchange(r, sd)
        if w is not None:
            w.wait()

    K = g.kshape[2]
    ev[0].record(st)
    if rhs.peer:  # K1 with its peer stores | barrier | K2-K4 (K4 with peer stores) | barrier | K5-K6
        b.forward_kz_peer(yk, 0, K)
        ev[1].record(st)
        rhs.barrier()
        ev[2].record(st)
        b.inverse_y_kz(rhs.recv1, 0, K)
        b.zpass()
        b.forward_y_kz_peer(0, K)
        ev[3].record(st)
        rhs.barrier()
        ev[4].record(st)
        b.forward_x_kz(rhs.recv2, 0, K)
        b.project(yk, fk)
    else:
        b.forward(yk, rhs.send1)
        ev[1].record(st)
        xchg(rhs.recv1, rhs.send1)
        ev[2].record(st)
        b.middle(rhs.recv1, rhs.send2)
        ev[3].record(st)
        xchg(rhs.recv2, rhs.send2)
        ev[4].record(st)
        b.finish(rhs.recv2, yk, fk)
    ev[5].record(st)
    # the pipelined RHS as the steps run it (exchanges overlapped with kernels)
    rhs(0.0, yk, out=fk)
    ev[6].record(st)
    torch.cuda.synchronize()
    ph = torch.tensor([ev[i].elapsed_time(ev[i + 1]) for i in range(6)], dtype=torch.float64, device=dev)
    dist.all_reduce(ph, op=dist.ReduceOp.MAX)
    ph = ph.cpu().numpy()
    geo = slab_geometry(g, world)
    mb = model_bytes(n)["per_kernel"]
    kb = list(mb.values())
    grp_bytes = [kb[0] / world, (kb[1] + kb[2] + kb[3]) / world, (kb[4] + kb[5]) / world]
    grp_ms = [ph[0], ph[2], ph[4]]
    dom = int(np.argmax(grp_ms))
    peak, peak_src = peaks()
    achieved = grp_bytes[dom] / (grp_ms[dom] * 1e-3) / 1e9
    a2a_bytes = (geo["send1"] + geo["send2"]) * 16 * (world - 1) / world
    a2a_ms = ph[1] + ph[3]
    # ---- e2e: each rank's slab resident on its host, as in run_native ----
    e2e = None
    if not args.no_e2e:
        s2 = new_state()
        mirror = srk.HostMirror(s2["y"])
        mirror.load_host(s2["y"].cpu())
        fplanes = srk.forcing_planes(g, k_f)
        spec = {}

        def on_y_new(v):
            mirror.push(v)
            spec["next"] = mirror.pull(wait=False)

        torch.cuda.synchronize()
        dist.barrier()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev2, t2_ = 0, s2["t"]
        n_e2e = max(2, args.steps // 2)
        def e2e_step(yd, t):
            fd = rhs(t, yd)
            red(reduce_sums(g, yd, fl=fd, flags=2, ncomp=3, plan=plan))
            out = srk.adaptive_advance(yd, t, pair, s2["ctrl"], cfg, rhs, first_stage=fd, grid=g,
                                       allreduce=red, plan=plan, on_y_new=on_y_new)
            srk.apply_forcing(out.y_new, g, energy, k_f, plan=plan, allreduce=red, slab=(rank, world),
                              energy_sum=out.diag_sums[4])
            mirror.push(out.y_new, planes=fplanes)
            ev, t = out.rhs_evals + 1, out.t_new
            del yd, fd, out
            return mirror.pull(into=spec.pop("next"), planes=fplanes), t, ev

        yd = mirror.pull()
        yd, t2_, _ = e2e_step(yd, t2_)  # untimed: first-use costs of the host path
        mirror.wait()
        torch.cuda.synchronize()
        dist.barrier()
        del yd
        b_in0, b_out0 = mirror.h2d_bytes, mirror.d2h_bytes
        a0.record(st)
        yd = mirror.pull()
        for _ in range(n_e2e):
            yd, t2_, ev = e2e_step(yd, t2_)
            ev2 += ev
        mirror.wait()
        a1.record(st)
        torch.cuda.synchronize()
        t2 = torch.tensor([a0.elapsed_time(a1) / 1e3], dtype=torch.float64, device=dev)
        dist.all_reduce(t2, op=dist.ReduceOp.MAX)
        e2e = {"value": ev2 / t2.item(), "unit": "stages/s",
               "h2d_bytes_per_step": (mirror.h2d_bytes - b_in0) // n_e2e,
               "d2h_bytes_per_step": (mirror.d2h_bytes - b_out0) // n_e2e + 9 * 8,
               "path": "per rank: y-slab host->device (pinned HostMirror), cached tendency + diagnostics, "
                       "adaptive_advance (BS5, rank-order sums) + forcing, y_new slab device->host overlapped "
                       "with the FSAL stage; bytes are per rank"}

    big = None
    rhs_peer, rhs_chunks = rhs.peer, len(rhs.chunks)
    ep_test = args.ep_test is not None
    if (world >= 4 and n == 512 and not args.no_1024) or ep_test:
        rhs.close()
        del s, rhs, b, yk, fk
        if not args.no_e2e:
            del s2, mirror, yd
        try:
            big = leg_1024(args, rank, world, *(args.ep_test if ep_test else ()))
        except Exception as exc:  # evidence leg: never lose the main line
            big = {"workload": "forced_hit_bs5_1024^3", "error": repr(exc)[:300]}
    if rank != 0:
        return
    names = ["K1 (forward)", "K2-K4 (middle)", "K5-K6 (finish)"]
    line = {
        "metric": METRIC, "value": value, "unit": "stages/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": T * 1e3 / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (device-side seeded HIT-spectrum slabs, E=0.5)",
        "config": {"workload": f"forced_hit_bs5_{n}^3", "n": n, "nu": 5e-4, "tol": 1e-6, "k_f": 2.0,
                   "parallelism": (f"y-slab x{world}, exchange fused into K1/K4 (peer stores over CUDA IPC)"
                                   if rhs_peer else
                                   f"y-slab x{world}, NCCL all-to-all, {rhs_chunks} kz chunks pipelined"),
                   "l2": "inputs larger than L2"},
        "gpts_stage_per_s": value * n ** 3 / 1e9,
        "rhs_evals": evals,
        "stage_hbm_frac": model_bytes(n)["b_stage_bs5"] * value / world / (peak * 1e9),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": None, "kernel": names[dom], "peak_source": peak_src,
                     "phase_ms": {"forward": ph[0], "a2a1": ph[1], "middle": ph[2], "a2a2": ph[3],
                                  "finish": ph[4], "serial_rhs": float(sum(ph[:5])),
                                  "pipelined_rhs": ph[5], "kz_chunks": rhs_chunks}},
        "nvlink": {"bytes_per_rhs_per_gpu": a2a_bytes, "achieved_GBps": a2a_bytes / (a2a_ms * 1e-3) / 1e9
                   if world > 1 else None, "peak_GBps": 770.0, "peak_source": "B200_PROFILING.md peer copy"},
        "cpu_baseline": None, "e2e": e2e, "gpu_launches": launches, "clocks": clk.summary(),
    }
    if big is not None:
        line["strong_1024"] = big
    assert line["n_gpus"] == args.gpus
    print(json.dumps(line), flush=True)


def single_gpu_ms_per_stage(n, steps, warmup):
    """ms per RHS evaluation of the single-GPU forced-HIT BS5 loop (run_native's step)."""
    import torch

    import paper_1810_10197_b200 as srk

    g = srk.Grid((n, n, n))
    params = srk.PhysParams(reynolds=2000.0)
    rhs = srk.FlowRHS(g, params)
    pair, cfg = srk.make_bs5(), srk.ControllerConfig(tol_abs=1e-6, tol_rel=1e-6)
    y = srk.hit_init(g, srk.ProblemSpec("hit", a=4.0, energy=0.5, seed=42)).fields
    s = dict(y=y, t=0.0, f=rhs(0.0, y), ctrl=srk.ControllerState(h=1e-3))
    a21 = float(pair.A[1, 0])

    def step():
        out = srk.adaptive_advance(s["y"], s["t"], pair, s["ctrl"], cfg, rhs, first_stage=s["f"], grid=g,
                                   second_input=s.get("y2"))
        srk.apply_forcing(out.y_new, g, 0.5, 2.0, energy_sum=out.diag_sums[4])
        h = s["ctrl"].h
        f, y2, _ = rhs.refresh(out.t_new, out.y_new, h * a21)
        s.update(y=out.y_new, t=out.t_new, f=f, y2=(h, y2))
        return out.rhs_evals + 1

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ev = sum(step() for _ in range(steps))
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / ev


def slab_ms_per_stage(args, n, steps, warmup, rank, world):
    """ms per RHS evaluation (max over ranks) of the y-slab BS5 loop at N = n."""
    import torch
    import torch.distributed as dist

    import paper_1810_10197_b200 as srk
    from paper_1810_10197_b200.diagnostics import reduce_sums
    from paper_1810_10197_b200.slab import SlabFlowRHS, dist_sum_in_rank_order, hit_slab

    g = srk.Grid((n, n, n))
    red = dist_sum_in_rank_order()
    rhs = SlabFlowRHS(g, srk.PhysParams(reynolds=2000.0), rank, world, chunks=4, peer=args.exchange == "peer")
    plan = rhs.backend.h
    pair, cfg = srk.make_bs5(), srk.ControllerConfig(tol_abs=1e-6, tol_rel=1e-6)
    y = hit_slab(g, rank, world, a=4.0, energy=0.5, seed=42, allreduce=red)
    s = dict(y=y, t=0.0, f=rhs(0.0, y), ctrl=srk.ControllerState(h=1e-3))

    def step():
        out = srk.adaptive_advance(s["y"], s["t"], pair, s["ctrl"], cfg, rhs, first_stage=s["f"], grid=g,
                                   allreduce=red, plan=plan)
        srk.apply_forcing(out.y_new, g, 0.5, 2.0, plan=plan, allreduce=red, slab=(rank, world),
                          energy_sum=out.diag_sums[4])
        f = rhs(out.t_new, out.y_new)
        red(reduce_sums(g, out.y_new, fl=f, flags=2, ncomp=3, plan=plan))
        s.update(y=out.y_new, t=out.t_new, f=f)
        return out.rhs_evals + 1

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ev = sum(step() for _ in range(steps))
    e1.record()
    e1.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / ev], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    rhs.close()
    return t.item()


def leg_1024(args, rank, world, n_big=1024, n_base=512, mem_per_point=725e9 / 1024 ** 3):
    """SURVEY M4 at 1024^3 (does not fit one GPU): E_P = (B_stage(1024) / (P T_P)) /
    (B_stage(512) / T_1(512)), T = time per RHS evaluation, T_1 measured here on
    rank 0 with the single-GPU path, T_P with the y-slab path on all P ranks.
    n_big / n_base: smaller grids exercise the same code path on one GPU (--ep-test)."""
    import gc

    import torch
    import torch.distributed as dist

    gc.collect()
    torch.cuda.empty_cache()
    t1 = torch.zeros(1, dtype=torch.float64, device="cuda")
    if rank == 0:
        t1[0] = single_gpu_ms_per_stage(n_base, steps=3, warmup=2)
        gc.collect()
        torch.cuda.empty_cache()
    dist.broadcast(t1, 0)
    need = mem_per_point * n_big ** 3 / world  # 1024^3 y-slab BS5 run: ~725 GB in all
    free = float(torch.cuda.mem_get_info()[0])
    fits = torch.tensor([1.0 if free > 1.05 * need else 0.0], device="cuda")
    dist.all_reduce(fits, op=dist.ReduceOp.MIN)
    out = {"workload": f"forced_hit_bs5_{n_big}^3", "T1_ms_per_stage": t1.item(), "T1_workload": f"{n_base}^3 on 1 GPU",
           "need_GB_per_gpu": need / 1e9, "free_GB_per_gpu": free / 1e9}
    if fits.item() < 1.0:
        out["skipped"] = f"{n_big}^3 y-slab state does not fit this GPU count"
        return out
    tp = slab_ms_per_stage(args, n_big, steps=2, warmup=1, rank=rank, world=world)
    b1024, b512 = model_bytes(n_big)["b_stage_bs5"], model_bytes(n_base)["b_stage_bs5"]
    out.update({"TP_ms_per_stage": tp, "stages_per_s": 1e3 / tp, "gpts_stage_per_s": n_big ** 3 / (tp * 1e-3) / 1e9,
                "E_P": (b1024 / (world * tp)) / (b512 / t1.item()), "P": world,
                "E_P_definition": "SURVEY M4: per-GPU achieved model bandwidth at P GPUs (1024^3) / 1-GPU (512^3)"})
    return out


def free_port():
    import socket

    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def self_launch(args):
    """`bench.py --gpus N` without a torchrun environment: re-run this command under
    torch.distributed.run with N ranks (one per GPU) on 127.0.0.1; rank 0's JSON
    line reaches our stdout."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ)
    env.setdefault("OMP_NUM_THREADS", "4")
    return subprocess.call(cmd, env=env)


def run_dry(args, rank, world):
    """Launcher / rank plumbing check on the CPU (gloo): barrier, max-over-ranks
    timing of a token host step, rank 0 prints the line shape the GPU run prints."""
    import torch
    import torch.distributed as dist

    dist.init_process_group("gloo")
    x = torch.ones(1 << 16, dtype=torch.float64)
    for _ in range(args.warmup):
        x = x * 1.0000001
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        x = x * 1.0000001
    dt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64)
    dist.all_reduce(dt, op=dist.ReduceOp.MAX)
    ranks = torch.tensor([1.0])
    dist.all_reduce(ranks)
    if rank == 0:
        print(json.dumps({"metric": METRIC, "value": None, "unit": "stages/s", "n_gpus": world,
                          "ranks_seen": int(ranks.item()), "steps": args.steps, "warmup": args.warmup,
                          "dry_run": True, "backend": "gloo", "max_rank_s": dt.item(),
                          "config": {"workload": f"forced_hit_bs5_{args.n}^3"}}), flush=True)
    dist.destroy_process_group()


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl != "reference" and world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world} ranks")
    if args.dry_run:
        run_dry(args, rank, world)
        return
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    mode = args.mode
    if mode == "auto":
        mode = "single" if world == 1 else "slab"
    if world > 1 or mode == "slab":
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", str(free_port()))
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl")
    if mode == "slab":
        run_slab(args, rank, world, local_rank)
    else:
        run_native(args, rank, world, local_rank)
    if world > 1 or mode == "slab":
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
