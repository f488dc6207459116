timeout 600 python -m pytest tests/test_gpu_behaviour.py -q -x -k "mirror" > gpurun_out/pytest_mirror.log 2>&1; echo "pytest rc=$?"
timeout 600 python bench.py --no-cpu > gpurun_out/bench512_mirror.log 2>&1; echo "bench rc=$?"
