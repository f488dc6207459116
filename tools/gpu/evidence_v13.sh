# round evidence v13: tests, smoke, benches, launch list
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/bench512.log 2>&1; echo "bench rc=$?"
timeout 600 python bench.py --grid 256 --no-cpu > gpurun_out/bench256.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 6 -c 16 --csv --log-file gpurun_out/launches512.csv python tools/rhs_timing.py --n 512 --reps 2 > gpurun_out/ncu_l.log 2>&1
echo done
