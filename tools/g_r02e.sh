mkdir -p gpurun_out/r02e
timeout 900 python bench.py > gpurun_out/r02e/bench512.json 2> gpurun_out/r02e/bench512.err
echo bench rc=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02e/bench_ref.json 2> gpurun_out/r02e/bench_ref.err
echo ref rc=$?
M=smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum
timeout 300 python tools/rhs_timing.py --n 512 --reps 2 > gpurun_out/r02e/plain.log 2>&1 && \
timeout 1200 ncu --set full --metrics $M --clock-control none --import-source on -s 6 -c 6 -o gpurun_out/r02e/rhs512 python tools/rhs_timing.py --n 512 --reps 2 > gpurun_out/r02e/ncu.log 2>&1
echo ncu rc=$?
