python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_gpu.log 2>&1
python tools/rhs_timing.py --n 512 > gpurun_out/rhs_timing.log 2>&1
python bench.py > gpurun_out/bench512.log 2>&1
python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1
echo done
