#!/bin/bash
# Access-pattern ceilings of the strided RHS passes at 512^3 (run on a GPU box from the repo root):
# SRK_PROBE_INV / SRK_PROBE_FWD make K1, K2 / K4, K5 stage their TMA tile and return (1), also
# store in the output pattern without transforming (2), or (K2 only) store without loading (5);
# SRK_PROBE_Z: the z-pass stages its rows (1) and stores zeros in its output pattern (2);
# SRK_YB=0 / SRK_KPAD=0 switch the y-blocked / padded-pitch layouts of the intermediates off.
# Prints one line per setting: per-kernel ms [K1 K2 K3 K4 K5 K6], their sum, back-to-back ms per RHS.
OUT=${1:-gpurun_out/ab/pass_probe.jsonl}
bash tools/ab_env.sh "$OUT" paper_1810_10197_b200/_lib \
  "SRK_PROBE_INV=0" \
  "SRK_PROBE_INV=1 SRK_PROBE_FWD=1" \
  "SRK_PROBE_INV=2 SRK_PROBE_FWD=2" \
  "SRK_PROBE_INV=5" \
  "SRK_PROBE_Z=1" "SRK_PROBE_Z=2" \
  "SRK_YB=0 SRK_KPAD=0" \
  "SRK_YB=0 SRK_KPAD=0 SRK_PROBE_INV=1 SRK_PROBE_FWD=1" \
  "SRK_YB=0 SRK_KPAD=0 SRK_PROBE_INV=2 SRK_PROBE_FWD=2" \
  "SRK_YB=0 SRK_KPAD=0 SRK_PROBE_INV=5"
