timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 600 python tools/e2e_timeline.py 512 4 > gpurun_out/e2e_tl.log 2>&1
timeout 600 python bench.py --no-cpu > gpurun_out/bench512_mirror.log 2>&1; echo "bench rc=$?"
