"""Generate golden vectors by running the REFERENCE itself (build container only).

    PYTHONDONTWRITEBYTECODE=1 python oracle/make_golden.py [--round2]

Imports ``spectralrk`` read-only from /root/reference/pkg/src and writes small
fixtures to tests/golden/.  /root/reference does not exist on the GPU box; the
fixtures travel instead.  The manifest records numpy/scipy versions because the
reference's FFT bits come from those un-vendored libraries.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")


def _ref():
    sys.dont_write_bytecode = True
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import spectralrk as srk  # noqa: E402

    return srk


def rhs_cases(srk):
    """Single FlowRHS evaluations (physics.py:188-206) on seeded inputs."""
    rng = np.random.default_rng(20260814)
    cases = {}

    def add(name, shape, y, re, density=False, ri=1.0, pr=1.0, lengths=None):
        g = srk.Grid(shape, lengths)
        p = srk.PhysParams(reynolds=re, richardson=ri, prandtl=pr)
        f = srk.FlowRHS(g, p, density=density)(0.0, y)
        cases[name] = dict(y=y, f=f, shape=np.array(shape), re=re, ri=ri, pr=pr,
                           density=int(density), lengths=np.array(g.lengths))

    g = srk.Grid((16, 16, 16))
    add("tg16", (16, 16, 16), srk.taylor_green_init(g).fields, 1600.0)
    g = srk.Grid((16, 16, 16))
    add("hit16_s1", (16, 16, 16),
        srk.hit_init(g, srk.ProblemSpec(kind="hit", a=4.0, energy=0.5, seed=1)).fields, 1000.0)
    g = srk.Grid((32, 32, 32))
    add("hit32_s42", (32, 32, 32),
        srk.hit_init(g, srk.ProblemSpec(kind="hit", a=4.0, energy=0.5, seed=42)).fields, 1000.0)
    # fully populated, non-Hermitian input incl. all Nyquist planes (exercises
    # the exact axis-order / C2R imaginary-part semantics)
    g = srk.Grid((8, 12, 16))
    y = rng.standard_normal((3,) + g.kshape) + 1j * rng.standard_normal((3,) + g.kshape)
    add("rand_8x12x16", (8, 12, 16), y, 37.0)
    g = srk.Grid((32, 32))
    add("tg2d_32", (32, 32), srk.taylor_green_init(g).fields, 100.0)
    g = srk.Grid((16, 24))
    y = rng.standard_normal((2,) + g.kshape) + 1j * rng.standard_normal((2,) + g.kshape)
    add("rand2d_16x24", (16, 24), y, 50.0)
    # Rayleigh-Taylor Boussinesq: erf interface -> z-Nyquist content
    shape = (16, 64)
    lengths = srk.default_lengths("rayleigh_taylor", shape)
    g = srk.Grid(shape, lengths)
    y = srk.rayleigh_taylor_init(g, srk.ProblemSpec(kind="rayleigh_taylor", amplitude=0.05)).fields
    y = y + 0.0
    y[:2] = 0.01 * (rng.standard_normal((2,) + g.kshape) + 1j * rng.standard_normal((2,) + g.kshape))
    add("rt2d_16x64", shape, y, 1600.0, density=True, ri=1.0, pr=0.7, lengths=lengths)
    g = srk.Grid((8, 8, 12))
    y = rng.standard_normal((4,) + g.kshape) + 1j * rng.standard_normal((4,) + g.kshape)
    add("bq3d_8x8x12", (8, 8, 12), y, 20.0, density=True, ri=2.0, pr=0.7)
    return cases


def dealias_cases(srk):
    """widen / narrow (spectral.py:215-304) on random stacks, incl. odd padded sizes."""
    rng = np.random.default_rng(7)
    out = {}
    for shape, c in [((8, 6, 4), 2), ((12, 12), 3), ((8, 10, 6), 1), ((16, 8, 8), 2)]:
        g = srk.Grid(shape)
        ws = srk.DealiasWorkspace(g, c)
        spec = rng.standard_normal((c,) + g.kshape) + 1j * rng.standard_normal((c,) + g.kshape)
        phys = ws.widen(spec).copy()
        pin = rng.standard_normal((c,) + g.padded_shape)
        narrow = ws.narrow(pin)
        key = "x".join(map(str, shape))
        out[key] = dict(shape=np.array(shape), spec=spec, phys=phys, pin=pin, narrow=narrow)
    return out


def _records(res):
    return np.array([[r.t, r.h, r.e_kin, r.eps, r.rhs_evals, r.rejections] for r in res.records])


def trajectories(srk):
    """Config-1 style runs through the reference driver (simulation.py:350-368)."""
    out = {}

    def cfg(shape, kind, re, integ, mode, t_end, h=None, tol=None, seed=None, a=9.5, energy=1.0):
        spec = srk.ProblemSpec(kind=kind, params=srk.PhysParams(reynolds=re), seed=seed,
                               a=a, energy=energy)
        c = srk.RunConfig(grid_shape=shape, problem=spec, integrator=integ, mode=mode,
                          t_end=t_end, h=h)
        if tol is not None:
            c.tol_abs = c.tol_rel = tol
        return c

    # C1: TG 32^3 nu=1/1600, RK4 dt=0.01 (100 steps) and BS5 tol 1e-6 to t=1
    r = srk.run_simulation(cfg((32, 32, 32), "taylor_green", 1600.0, "rk4", "fixed", 1.0, h=0.01))
    out["c1_rk4"] = dict(y=r.state.fields, rec=_records(r))
    r = srk.run_simulation(cfg((32, 32, 32), "taylor_green", 1600.0, "bs5", "adaptive", 1.0, tol=1e-6))
    out["c1_bs5"] = dict(y=r.state.fields, rec=_records(r))
    # HIT 16^3 BS5 with an oversized h0 -> rejections exercised
    c = cfg((16, 16, 16), "hit", 1000.0, "bs5", "adaptive", 0.2, tol=1e-6, seed=3, a=4.0, energy=0.5)
    c.h0 = 0.5
    r = srk.run_simulation(c)
    out["hit16_bs5_rej"] = dict(y=r.state.fields, rec=_records(r))
    # forced HIT 16^3 (config-5 scheme, physics.py:209-239)
    c = cfg((16, 16, 16), "hit", 2000.0, "bs5", "adaptive", 0.05, tol=1e-6, seed=5, a=4.0, energy=0.5)
    c.forcing = True
    c.k_f = 2.0
    r = srk.run_simulation(c)
    out["hit16_forced"] = dict(y=r.state.fields, rec=_records(r))
    # 2D RT Boussinesq 16x64, RK4 fixed, 20 steps
    spec = srk.ProblemSpec(kind="rayleigh_taylor", params=srk.PhysParams(reynolds=1600.0))
    c = srk.RunConfig(grid_shape=(16, 64), problem=spec, integrator="rk4", mode="fixed",
                      t_end=0.2, h=0.01, lengths=srk.default_lengths("rayleigh_taylor", (16, 64)))
    r = srk.run_simulation(c)
    out["rt2d_rk4"] = dict(y=r.state.fields, rec=_records(r))
    return out


def round2_cases(srk):
    """Round-2 pins: AB2 trajectories (simulation.py:274-310, integrators.py:361-363)
    incl. the uneven-tail RK4 restart, and 3D Boussinesq at fast-plan sizes --
    a Rayleigh-Taylor RHS (problems.py:65-82, z-Nyquist content) and RK4 / BS5
    windows through the reference driver."""
    out = {}

    def run(shape, kind, re, integ, mode, t_end, h=None, tol=None, lengths=None, **kw):
        spec = srk.ProblemSpec(kind=kind, params=srk.PhysParams(reynolds=re), **kw)
        c = srk.RunConfig(grid_shape=shape, problem=spec, integrator=integ, mode=mode, t_end=t_end, h=h,
                          lengths=lengths)
        if tol is not None:
            c.tol_abs = c.tol_rel = tol
        return srk.run_simulation(c)

    # AB2: TG 32^3, 10 full steps + a 0.005 tail (RK4 restart)
    r = run((32, 32, 32), "taylor_green", 1600.0, "ab2", "fixed", 0.105, h=0.01)
    out["ab2_tg32"] = dict(y=r.state.fields, rec=_records(r))
    # AB2: 2D RT Boussinesq 16x64 (density in the multistep update)
    L = srk.default_lengths("rayleigh_taylor", (16, 64))
    r = run((16, 64), "rayleigh_taylor", 1600.0, "ab2", "fixed", 0.2, h=0.01, lengths=L)
    out["ab2_rt2d"] = dict(y=r.state.fields, rec=_records(r))
    # 3D RT Boussinesq 32x32x64 (padded lengths 48, 48, 96: fast plans)
    shape = (32, 32, 64)
    L = srk.default_lengths("rayleigh_taylor", shape)
    g = srk.Grid(shape, L)
    y = srk.rayleigh_taylor_init(g, srk.ProblemSpec(kind="rayleigh_taylor", amplitude=0.05)).fields + 0.0
    rng = np.random.default_rng(33)
    y[:3] = 0.01 * (rng.standard_normal((3,) + g.kshape) + 1j * rng.standard_normal((3,) + g.kshape))
    p = srk.PhysParams(reynolds=800.0, richardson=1.0, prandtl=0.7)
    out["rt3d_rhs"] = dict(y=y, f=srk.FlowRHS(g, p, density=True)(0.0, y), shape=np.array(shape),
                           lengths=np.array(L))
    r = run(shape, "rayleigh_taylor", 1600.0, "rk4", "fixed", 0.05, h=0.01, lengths=L)
    out["rt3d_rk4"] = dict(y=r.state.fields, rec=_records(r))
    r = run(shape, "rayleigh_taylor", 1600.0, "bs5", "adaptive", 0.3, tol=1e-6, lengths=L)
    out["rt3d_bs5"] = dict(y=r.state.fields, rec=_records(r))
    # the reference's `spectrum` command (cli.py:90-103) on a checkpoint it wrote
    import tempfile

    with tempfile.TemporaryDirectory() as td:
        spec = srk.ProblemSpec(kind="hit", params=srk.PhysParams(reynolds=500.0), seed=9, a=4.0, energy=0.5)
        c = srk.RunConfig(grid_shape=(16, 16, 16), problem=spec, integrator="bs5", mode="adaptive", t_end=0.02,
                          output_dir=td)
        srk.run_simulation(c)
        ck = os.path.join(td, "final.srkl")
        from spectralrk.cli import build_parser, main as cli_main  # noqa: F401
        import io
        import contextlib

        buf = io.StringIO()
        with contextlib.redirect_stdout(buf):
            cli_main(["spectrum", ck])
        with open(ck, "rb") as fh:
            out["spectrum_cli"] = dict(srkl=np.frombuffer(fh.read(), dtype=np.uint8),
                                       text=np.frombuffer(buf.getvalue().encode(), dtype=np.uint8))
    return out


def ics(srk):
    out = {}
    g = srk.Grid((16, 16, 16))
    out["hit16_a4_s42"] = srk.hit_init(g, srk.ProblemSpec(kind="hit", a=4.0, energy=0.5, seed=42)).fields
    out["tg16"] = srk.taylor_green_init(g).fields
    g = srk.Grid((16, 64), srk.default_lengths("rayleigh_taylor", (16, 64)))
    out["rt16x64"] = srk.rayleigh_taylor_init(g, srk.ProblemSpec(kind="rayleigh_taylor")).fields
    return out


def io_cases(srk):
    """SRKL checkpoint + diagnostics CSV written by the reference driver, and an
    energy spectrum (simulation.py:371-516, diagnostics.py:73-91)."""
    import tempfile

    out = {}
    with tempfile.TemporaryDirectory() as td:
        spec = srk.ProblemSpec(kind="taylor_green", params=srk.PhysParams(reynolds=100.0), seed=7)
        c = srk.RunConfig(grid_shape=(16, 16), problem=spec, integrator="dp5", mode="fixed", t_end=0.5, h=0.1,
                          output_dir=td, checkpoint_interval=0.2)
        srk.run_simulation(c)
        for name in ("final.srkl", "checkpoint_t0.200000.srkl", "diagnostics.csv"):
            with open(os.path.join(td, name), "rb") as fh:
                out[name.replace(".", "_")] = np.frombuffer(fh.read(), dtype=np.uint8)
    g = srk.Grid((16, 16, 16))
    u = srk.hit_init(g, srk.ProblemSpec(kind="hit", a=4.0, energy=0.5, seed=42)).fields
    sp = srk.energy_spectrum(u, g)
    out["spectrum_hit16_E"] = sp.E
    return out


def _save(name, dct):
    flat = {}
    for case, vals in dct.items():
        if isinstance(vals, dict):
            for k, v in vals.items():
                flat[f"{case}__{k}"] = v
        else:
            flat[case] = vals
    np.savez_compressed(os.path.join(OUT, name), **flat)


def main():
    import scipy

    srk = _ref()
    os.makedirs(OUT, exist_ok=True)
    if "--round2" in sys.argv:  # only the round-2 file (the earlier fixtures stay as committed)
        _save("r2_cases.npz", round2_cases(srk))
        print("wrote r2_cases.npz")
        return
    _save("rhs_cases.npz", rhs_cases(srk))
    _save("dealias_cases.npz", dealias_cases(srk))
    _save("ics.npz", ics(srk))
    _save("trajectories.npz", trajectories(srk))
    _save("io_cases.npz", io_cases(srk))
    _save("r2_cases.npz", round2_cases(srk))
    man = dict(reference="spectralrk " + srk.__version__, numpy=np.__version__,
               scipy=scipy.__version__, generator="oracle/make_golden.py")
    with open(os.path.join(OUT, "MANIFEST.json"), "w") as fh:
        json.dump(man, fh, indent=1)
    print("wrote", sorted(os.listdir(OUT)))


if __name__ == "__main__":
    main()
