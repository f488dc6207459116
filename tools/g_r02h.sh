mkdir -p gpurun_out/r02h
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_graphs.py tests/test_gpu_round2.py tests/test_gpu_fused_stage.py tests/test_gpu_behaviour.py -q -x > gpurun_out/r02h/pytest.log 2>&1
echo pytest rc=$? >> gpurun_out/r02h/pytest.log
for i in 1 2; do
 for n in 512 256 64 32; do
  SRK_LIB_PATH=$PWD/_lib_base/libsrk.so timeout 300 python tools/rhs_timing.py --n $n --reps 3 --chain 20 >> gpurun_out/r02h/ab_base.jsonl 2>&1
  timeout 300 python tools/rhs_timing.py --n $n --reps 3 --chain 20 >> gpurun_out/r02h/ab_new.jsonl 2>&1
 done
 SRK_LIB_PATH=$PWD/_lib_base/libsrk.so timeout 300 python tools/rhs_timing.py --n 1024 --dims 2 --density --reps 3 --chain 50 >> gpurun_out/r02h/ab_base.jsonl 2>&1
 timeout 300 python tools/rhs_timing.py --n 1024 --dims 2 --density --reps 3 --chain 50 >> gpurun_out/r02h/ab_new.jsonl 2>&1
done
SRK_LIB_PATH=$PWD/_lib_base/libsrk.so timeout 900 python tools/graph_timing.py all > gpurun_out/r02h/graph_base.jsonl 2>&1
timeout 900 python tools/graph_timing.py all > gpurun_out/r02h/graph_new.jsonl 2>&1
