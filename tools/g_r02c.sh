mkdir -p gpurun_out/r02c
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/r02c/pytest_gpu.log 2>&1
echo pytest rc=$?
tail -3 gpurun_out/r02c/pytest_gpu.log
