"""ncu capture of one srk_rhs (6 launches, K1..K6 in order) -> profiles/ncu_kernels.json.

    python tools/ncu_kernels.py <report.ncu-rep> --n 512 [--lib paper_1810_10197_b200/_lib/libsrk.so]

The JSON records srk_source_hash() of the libsrk.so the capture was taken from
(kernel sources + compile flags); bench.py reports these counters
(roofline.traffic, the z-pass's shared-memory wavefronts and fp64 flops) only
when the loaded library was built from the same sources.
Capture command (GPU box, one GPU):
    ncu --set full --metrics smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,\
smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum \
        --clock-control none -k regex:"k_colpass|k_zpass|k_project" -s 6 -c 6 -o <report> \
        python tools/rhs_timing.py --n 512 --reps 2
and then, on the same box (the hash must be of the library that ran):
    python tools/ncu_kernels.py <report> --n 512
"""
import argparse
import csv
import hashlib
import io
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NAMES = ["K1_xinv_curl", "K2_yinv", "K3_z_c2r_cross_r2c", "K4_yfwd", "K5_xfwd", "K6_project"]


def sha256(path):
    h = hashlib.sha256()
    with open(path, "rb") as fh:
        for blk in iter(lambda: fh.read(1 << 22), b""):
            h.update(blk)
    return h.hexdigest()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--n", type=int, default=512)
    ap.add_argument("--lib", default=os.path.join(ROOT, "paper_1810_10197_b200", "_lib", "libsrk.so"))
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "ncu_kernels.json"))
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.report, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h = rows[0]
    ix = {n: i for i, n in enumerate(h)}

    def g(r, n):
        try:
            return float(r[ix[n]].replace(",", ""))
        except (KeyError, ValueError):
            return None

    launches = [r for r in rows[2:] if r and len(r) == len(h)]
    if len(launches) != 6:
        raise SystemExit(f"expected the 6 launches of one srk_rhs, found {len(launches)}")
    # the capture may start anywhere in the RHS chain: rotate so the z-pass is K3
    z = [i for i, r in enumerate(launches) if "k_zpass" in r[ix["Kernel Name"]]]
    if len(z) != 1:
        raise SystemExit("expected exactly one z-pass launch")
    launches = [launches[(z[0] - 2 + i) % 6] for i in range(6)]
    per = {}
    for name, r in zip(NAMES, launches):
        unit_scale = 1e9 if "Gbyte" in (rows[1][ix["dram__bytes_read.sum"]] or "") else 1.0
        rd, wr = g(r, "dram__bytes_read.sum"), g(r, "dram__bytes_write.sum")
        dfma = g(r, "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum")
        dadd = g(r, "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum")
        dmul = g(r, "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum")
        per[name] = {
            "kernel": r[ix["Kernel Name"]][:160],
            "ncu_ms": g(r, "gpu__time_duration.sum"),
            "dram_bytes": (rd + wr) * unit_scale if rd is not None else None,
            "fp64_pipe": (g(r, "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active") or 0) / 100,
            "smem_wavefronts": g(r, "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
            "smem_pipe_frac": (g(r, "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed")
                               or 0) / 100,
            "fp64_flops": (2 * dfma + dadd + dmul) if None not in (dfma, dadd, dmul) else None,
            "registers": g(r, "launch__registers_per_thread"),
            "warps_active": (g(r, "sm__warps_active.avg.pct_of_peak_sustained_active") or 0) / 100,
        }
    try:
        d = json.load(open(a.out))
    except Exception:
        d = {}
    import ctypes

    h = ctypes.CDLL(a.lib).srk_source_hash
    h.restype = ctypes.c_char_p
    src = h().decode()
    if d.get("source_hash") != src:
        d = {}
    d.update({"source_hash": src, "lib_sha256": sha256(a.lib), "report": os.path.basename(a.report),
              "source": "ncu --set full + sass per-opcode fp64 counters, one srk_rhs (tools/ncu_kernels.py)"})
    d[str(a.n)] = per
    with open(a.out, "w") as fh:
        json.dump(d, fh, indent=1)
    print(json.dumps({k: {kk: v[kk] for kk in ("ncu_ms", "dram_bytes", "smem_wavefronts", "fp64_flops")}
                      for k, v in per.items()}, indent=1))


if __name__ == "__main__":
    main()
