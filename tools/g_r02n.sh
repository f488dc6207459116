mkdir -p gpurun_out/r02n
M=smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum
timeout 300 python tools/rhs_timing.py --n 512 --reps 2 > gpurun_out/r02n/plain.log 2>&1 && \
timeout 1500 ncu --set full --metrics $M --clock-control none --import-source on -k regex:"k_colpass|k_zpass|k_project" -s 6 -c 6 -o /tmp/rhs512 python tools/rhs_timing.py --n 512 --reps 2 > gpurun_out/r02n/ncu.log 2>&1
echo ncu rc=$? >> gpurun_out/r02n/ncu.log
python tools/ncu_kernels.py /tmp/rhs512.ncu-rep --n 512 > gpurun_out/r02n/ncu_kernels.out 2>&1
cp profiles/ncu_kernels.json gpurun_out/r02n/ncu_kernels.json
python tools/ncu_summary.py /tmp/rhs512.ncu-rep > gpurun_out/r02n/ncu_summary.txt 2>&1
timeout 600 python bench.py --steps 6 --warmup 3 --no-e2e --no-cpu > gpurun_out/r02n/bench_check.json 2>&1
