"""SRKL checkpoint + diagnostics CSV format (CPU): byte compatibility with files
written by the reference driver (tests/golden/io_cases.npz, oracle/make_golden.py)."""
import numpy as np
import pytest

from conftest import load_golden
from paper_1810_10197_b200.checkpoint import (CheckpointError, read_checkpoint, read_diagnostics_csv,
                                              write_checkpoint, write_diagnostics_csv)

IO = load_golden("io_cases")


@pytest.mark.parametrize("name", ["final_srkl", "checkpoint_t0_200000_srkl"])
def test_reference_checkpoint_round_trips_byte_exact(name, tmp_path):
    src = tmp_path / "ref.srkl"
    src.write_bytes(IO[name].tobytes())
    data = read_checkpoint(src)
    assert data.grid.shape == (16, 16) and not data.has_density
    assert data.f_now is not None and data.fields.shape == (2, 16, 9)
    assert data.rng_state is not None
    out = tmp_path / "mine.srkl"
    write_checkpoint(out, data)
    assert out.read_bytes() == src.read_bytes()


def test_reference_checkpoint_header_values(tmp_path):
    src = tmp_path / "ref.srkl"
    src.write_bytes(IO["final_srkl"].tobytes())
    d = read_checkpoint(src)
    assert d.time == 0.5 and d.h == 0.1 and d.steps == 5
    assert d.rhs_evals == 5 * 6 + 1  # dp5 fixed: 6 evals/step + 1 (test_simulation.py:68-76)


def test_reference_csv_round_trip(tmp_path):
    src = tmp_path / "ref.csv"
    src.write_bytes(IO["diagnostics_csv"].tobytes())
    recs = read_diagnostics_csv(src)
    assert len(recs) == 6 and recs[-1].t == 0.5
    out = tmp_path / "mine.csv"
    write_diagnostics_csv(recs, out)
    assert out.read_bytes() == src.read_bytes()


def test_corrupt_checkpoints_rejected(tmp_path):
    raw = IO["final_srkl"].tobytes()
    bad = tmp_path / "bad.srkl"
    bad.write_bytes(b"XXXX" + raw[4:])
    with pytest.raises(CheckpointError, match="magic"):
        read_checkpoint(bad)
    bad.write_bytes(raw[:-16])
    with pytest.raises(CheckpointError, match="truncated"):
        read_checkpoint(bad)


def test_wrong_csv_header(tmp_path):
    p = tmp_path / "x.csv"
    p.write_text("time,step\n0,1\n")
    with pytest.raises(ValueError, match="header"):
        read_diagnostics_csv(p)
