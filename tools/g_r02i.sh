mkdir -p gpurun_out/r02i
for c in c4 c1; do
  SRK_LIB_PATH=$PWD/_lib_base/libsrk.so timeout 300 python tools/graph_probe.py $c >> gpurun_out/r02i/probe_base.jsonl 2>&1
  timeout 300 python tools/graph_probe.py $c >> gpurun_out/r02i/probe_new.jsonl 2>&1
done
for x in 1 2 3; do
  SRK_LIB_PATH=$PWD/_lib_x$x/libsrk.so timeout 300 python tools/rhs_timing.py --n 512 --reps 4 --chain 10 >> gpurun_out/r02i/x$x.jsonl 2>&1
done
timeout 300 python tools/rhs_timing.py --n 512 --reps 4 --chain 10 >> gpurun_out/r02i/x0.jsonl 2>&1
for x in 1 2 3; do
  SRK_LIB_PATH=$PWD/_lib_x$x/libsrk.so timeout 300 python tools/rhs_timing.py --n 512 --reps 4 --chain 10 >> gpurun_out/r02i/x$x.jsonl 2>&1
done
timeout 300 python tools/rhs_timing.py --n 512 --reps 4 --chain 10 >> gpurun_out/r02i/x0.jsonl 2>&1
SRK_LIB_PATH=$PWD/_lib_x3/libsrk.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "fast_plans or fullsize or 256" > gpurun_out/r02i/x3_parity.log 2>&1
