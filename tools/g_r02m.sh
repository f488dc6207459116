mkdir -p gpurun_out/r02m
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r02m/pytest_gpu.log 2>&1
echo pytest rc=$? >> gpurun_out/r02m/pytest_gpu.log
for i in 1 2 3; do
  SRK_LIB_PATH=$PWD/_lib_base/libsrk.so timeout 300 python tools/rhs_timing.py --n 512 --reps 4 >> gpurun_out/r02m/ab_base.jsonl 2>&1
  timeout 300 python tools/rhs_timing.py --n 512 --reps 4 >> gpurun_out/r02m/ab_new.jsonl 2>&1
done
timeout 900 python tools/graph_timing.py c4 c1 > gpurun_out/r02m/graph_timing.jsonl 2>&1
timeout 900 python bench.py > gpurun_out/r02m/bench512.json 2> gpurun_out/r02m/bench512.err
