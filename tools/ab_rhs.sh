#!/bin/bash
# A/B of library builds on one GPU box: tools/ab_rhs.sh <out.jsonl> <lib dir> [<lib dir> ...]
# Alternates `tools/rhs_timing.py --n 512 --reps 6 --chain 20` over the builds (3 rounds).
OUT=$1; shift
mkdir -p "$(dirname "$OUT")"; : > "$OUT"
for round in 1 2 3; do
  for L in "$@"; do
    echo -n "{\"lib\": \"$L\", \"round\": $round, \"r\": " >> "$OUT"
    SRK_LIB_PATH=$PWD/$L/libsrk.so timeout 300 python tools/rhs_timing.py --n 512 --reps 6 --chain 20 | tr -d '\n' >> "$OUT"
    echo "}" >> "$OUT"
  done
done
