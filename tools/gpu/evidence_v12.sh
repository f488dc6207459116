# round evidence v12 (host-resident e2e, 2D one-pencil z-pass): tests, smoke, benches, launch lists, 2D ncu
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/bench512.log 2>&1; echo "bench rc=$?"
timeout 600 python bench.py --grid 256 --no-cpu > gpurun_out/bench256.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1
timeout 300 python tools/rhs_timing.py --n 512 --reps 5 > gpurun_out/t512.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 6 -c 16 --csv --log-file gpurun_out/launches512.csv python tools/rhs_timing.py --n 512 --reps 2 > gpurun_out/ncu_l.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -s 8 -c 4 -o gpurun_out/prof2d_full python tools/rhs_timing.py --n 1024 --dims 2 --density --reps 2 > gpurun_out/ncu_2d.log 2>&1
echo done
