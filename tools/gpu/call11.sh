python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_gpu.log 2>&1
python bench.py --mode slab --grid 256 --steps 3 --warmup 2 > gpurun_out/bench_slab256.log 2>&1
torchrun --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --mode slab --grid 256 --steps 3 --warmup 2 > gpurun_out/bench_slab256_torchrun.log 2>&1
echo done
