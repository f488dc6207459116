"""`spectrum` entry point (reference cli.py:90-103): the shell-binned energy
spectrum of an SRKL checkpoint, computed on the device, written in the
reference's text format ("k,E" header, %.16e pairs).

    python -m paper_1810_10197_b200.spectrum CHECKPOINT [--out PATH]

The rest of the reference CLI (run / bench / INI configs) is out of scope
(SURVEY §2); this is the one command whose arithmetic sits on the device path.
"""

from __future__ import annotations

import argparse
import sys
from pathlib import Path

__all__ = ["spectrum_text", "main"]


def spectrum_text(checkpoint_path) -> str:
    from .checkpoint import read_checkpoint
    from .diagnostics import energy_spectrum

    data = read_checkpoint(checkpoint_path)
    sp = energy_spectrum(data.fields[: data.grid.dims], data.grid)
    lines = ["k,E"] + [f"{k:.16e},{e:.16e}" for k, e in zip(sp.k, sp.E)]
    return "\n".join(lines) + "\n"


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="spectrum", description="energy spectrum of an SRKL checkpoint")
    ap.add_argument("checkpoint")
    ap.add_argument("--out", default=None)
    args = ap.parse_args(argv)
    text = spectrum_text(args.checkpoint)
    if args.out:
        Path(args.out).write_text(text)
        print(f"spectrum written to {args.out}")
    else:
        sys.stdout.write(text)
    return 0


if __name__ == "__main__":
    sys.exit(main())
