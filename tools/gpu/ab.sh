# A/B: per-kernel RHS timing of the default lib vs experiment libs given as args
for r in 1 2; do
timeout 300 python tools/rhs_timing.py --n 512 --reps 5 | sed 's/^/default /'
for L in "$@"; do SRK_LIB=$L timeout 300 python tools/rhs_timing.py --n 512 --reps 5 | sed "s|^|$L |"; done
done
