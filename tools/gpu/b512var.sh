for i in 1 2 3; do
SRK_BENCH_STEPS=1 timeout 600 python bench.py --no-e2e --no-cpu 2>gpurun_out/b512_steps_$i.log | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('b512', round(d['value'],2), round(d['ms_per_step'],2), d['clocks']['sm_mhz'])"
grep per-step gpurun_out/b512_steps_$i.log
done
