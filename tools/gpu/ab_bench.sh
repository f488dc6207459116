# A/B of whole-step throughput (bench.py, no e2e / cpu legs) between libs, alternating
for r in 1 2; do
for L in "$@"; do SRK_LIB=$L timeout 600 python bench.py --no-e2e --no-cpu --steps 8 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$L', round(d['value'],3), d['clocks']['sm_mhz'], d['roofline']['kernel_ms'])"; done
done
