for i in 1 2 3; do
timeout 600 python bench.py --no-e2e --no-cpu --grid 256 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('sampler', round(d['value'],1), round(d['ms_per_step'],2))"
SRK_BENCH_NO_CLOCKS=1 timeout 600 python bench.py --no-e2e --no-cpu --grid 256 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('nosampler', round(d['value'],1), round(d['ms_per_step'],2))"
done
