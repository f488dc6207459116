"""bench.py contract on the GPU at a small grid: the single-GPU line (roofline,
e2e through HostMirror, clocks, launches) and the slab path over NCCL (world of
one; the N > 1 orchestration is covered by tests/test_slab_gloo.py)."""

import json
import os
import random
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(*args, env=None):
    e = dict(os.environ)
    e.update(env or {})
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, env=e,
                       capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_single_gpu_line():
    d = run_bench("--grid", "64", "--steps", "3", "--warmup", "3", "--no-cpu")
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3
    assert d["value"] > 0 and d["unit"] == "stages/s" and d["higher_is_better"] is True
    assert d["rhs_evals"] >= 8 * 3  # 7 stages + the refresh per accepted step (+7 per rejection)
    r = d["roofline"]
    assert r["bound"] == "hbm" and 0 < r["frac"] < 1.5 and r["kernel"] in r["kernel_ms"]
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] >= 3 * 64 * 64 * 33 * 16
    assert e["d2h_bytes_per_step"] >= 3 * 64 * 64 * 33 * 16
    assert d["gpu_launches"] > 0 and "sm_mhz" in d["clocks"]


def test_bench_slab_over_nccl():
    d = run_bench("--mode", "slab", "--grid", "64", "--steps", "2", "--warmup", "3",
                  env={"MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(random.randint(20000, 40000))})
    assert d["n_gpus"] == 1 and d["scaling"] == "strong" and d["value"] > 0
    assert d["roofline"]["phase_ms"]["serial_rhs"] > 0 and d["gpu_launches"] > 0
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] >= 3 * 64 * 64 * 33 * 16


def test_bench_slab_peer_exchange():
    d = run_bench("--mode", "slab", "--exchange", "peer", "--grid", "64", "--steps", "2", "--warmup", "3", "--no-e2e",
                  env={"MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(random.randint(20000, 40000))})
    assert d["value"] > 0 and "peer stores" in d["config"]["parallelism"]


def test_bench_strong_scaling_leg_code_path():
    """The 1024^3 E_P leg (run at N >= 4) on small grids with one rank: rank 0's
    single-GPU baseline, the fit check, the slab loop and E_P."""
    d = run_bench("--mode", "slab", "--grid", "64", "--steps", "2", "--warmup", "3", "--no-e2e",
                  "--ep-test", "128", "64",
                  env={"MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(random.randint(20000, 40000))})
    big = d["strong_1024"]
    assert big["workload"] == "forced_hit_bs5_128^3", big
    assert big["T1_ms_per_stage"] > 0 and big["TP_ms_per_stage"] > 0 and big["P"] == 1
    assert 0.05 < big["E_P"] < 5.0


def test_bench_single_gpu_line_on_chip_ceilings():
    d = run_bench("--grid", "64", "--steps", "3", "--warmup", "3", "--no-cpu", "--no-e2e")
    c = d["roofline"]["on_chip_ceilings"]
    assert c["probe"]["fp64_tflops"] > 5 and c["probe"]["smem_GBps"] > 5000
