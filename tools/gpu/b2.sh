timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x -k "boussinesq or c4 or rt" > gpurun_out/pytest_b2.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_b2.log
timeout 300 python tools/rhs_timing.py --n 1024 --dims 2 --density --reps 20 > gpurun_out/t2d.log 2>&1
timeout 600 python tools/c4_timing.py >> gpurun_out/t2d.log 2>&1
cat gpurun_out/t2d.log
