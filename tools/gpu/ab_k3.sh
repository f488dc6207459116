# K3 (z-pass) time of experiment libs: python tools/rhs_timing per lib, 2 rounds
for r in 1 2; do
for L in "$@"; do SRK_LIB=$L timeout 300 python tools/rhs_timing.py --n 512 --reps 5 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$L', d['ms'][2], d['total_ms'])"; done
done
