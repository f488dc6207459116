OUT=gpurun_out/evidence2; mkdir -p $OUT
M=smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum
timeout 300 python tools/rhs_timing.py --n 512 --reps 2 > $OUT/rhs_plain.log 2>&1 && \
timeout 1500 ncu --set full --metrics $M --clock-control none --import-source on -k regex:"k_colpass|k_zpass|k_project" \
    -s 6 -c 6 -f -o /tmp/rhs512 python tools/rhs_timing.py --n 512 --reps 2 > $OUT/ncu.log 2>&1 && \
python tools/ncu_kernels.py /tmp/rhs512.ncu-rep --n 512 > $OUT/ncu_kernels.out 2>&1 && \
cp profiles/ncu_kernels.json $OUT/ncu_kernels.json && python tools/ncu_summary.py /tmp/rhs512.ncu-rep > $OUT/ncu_summary.txt 2>&1
cp profiles/ncu_kernels.json $OUT/ 2>/dev/null
timeout 900 python bench.py --steps 6 --warmup 3 --no-cpu > $OUT/bench512.json 2> $OUT/bench512.err
