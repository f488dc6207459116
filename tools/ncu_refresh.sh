#!/bin/bash
# Re-capture the ncu counters bench.py reports (profiles/ncu_kernels.json, tied to the
# build by srk_source_hash) after a source change: one 512^3 RHS under ncu --set full.
# Run on a GPU box from the repo root; outputs also in gpurun_out/evidence/.
set -u
OUT=gpurun_out/evidence
mkdir -p $OUT
M=smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum
timeout 300 python tools/rhs_timing.py --n 512 --reps 2 > $OUT/rhs_plain.log 2>&1 && \
timeout 1500 ncu --set full --metrics $M --clock-control none --import-source on -k regex:"k_colpass|k_zpass|k_project" \
    -s 6 -c 6 -f -o /tmp/rhs512 python tools/rhs_timing.py --n 512 --reps 2 > $OUT/ncu.log 2>&1 && \
python tools/ncu_kernels.py /tmp/rhs512.ncu-rep --n 512 > $OUT/ncu_kernels.out 2>&1 && \
cp profiles/ncu_kernels.json $OUT/ncu_kernels.json && python tools/ncu_summary.py /tmp/rhs512.ncu-rep > $OUT/ncu_summary.txt 2>&1
timeout 900 python bench.py --no-cpu > $OUT/bench512_with_counters.json 2> $OUT/bench512_with_counters.err
