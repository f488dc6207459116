mkdir -p gpurun_out/r02b
timeout 300 python tools/probe_peaks.py > gpurun_out/r02b/probe.json 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02b/pytest_gpu.log 2>&1
echo pytest rc=$?
timeout 300 python tools/rhs_timing.py --n 512 --reps 6 > gpurun_out/r02b/rhs512.json 2>&1
