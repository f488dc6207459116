python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/pytest_gpu.log 2>&1
for n in 256 512; do python tools/rhs_timing.py --n $n; done > gpurun_out/rhs_timing.log 2>&1
python tools/cufft_ref.py > gpurun_out/cufft_ref.log 2>&1
echo done
