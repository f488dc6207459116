#!/bin/bash
# tools/ab_env.sh <out.jsonl> <lib dir> "<ENV=.. ENV=..>" ["<env set 2>" ...]: rhs_timing at 512^3 under
# different environment settings of one build (3 alternating rounds)
OUT=$1; L=$2; shift 2
mkdir -p "$(dirname "$OUT")"; : > "$OUT"
for round in 1 2 3; do
  for E in "$@"; do
    echo -n "{\"env\": \"$E\", \"round\": $round, \"r\": " >> "$OUT"
    env $E SRK_LIB_PATH=$PWD/$L/libsrk.so timeout 300 python tools/rhs_timing.py --n 512 --reps 6 --chain 20 | tr -d '\n' >> "$OUT"
    echo "}" >> "$OUT"
  done
done
python - "$OUT" <<'PY'
import json, sys
for l in open(sys.argv[1]):
    d = json.loads(l)
    print(f'{d["env"]:40s}', d["r"]["ms"], d["r"]["total_ms"], d["r"].get("chain_ms_per_rhs"))
PY
