set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_gpu.log 2>&1
python bench.py --grid 128 --steps 5 --warmup 3 > gpurun_out/bench128.log 2>&1
python bench.py > gpurun_out/bench512.log 2>&1
python bench.py --grid 256 --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/bench256_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches256.csv python bench.py --grid 256 --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_zpass -s 2 -c 1 -o gpurun_out/prof_zpass256 python bench.py --grid 256 --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_full.log 2>&1
echo done
