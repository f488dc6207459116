#!/bin/bash
# Round-2 evidence on one B200 (run from the repo root under gpurun; outputs in gpurun_out/evidence/):
#   GPU tests, smoke, the bench line (512^3), the reference arm, graph vs eager loops (C1, C4),
#   the per-pass cuFFT comparison, the ncu capture of one 512^3 RHS -> profiles/ncu_kernels.json
#   (tied to this build by srk_source_hash), and the hazard-probe build check.
set -u
OUT=gpurun_out/evidence
mkdir -p $OUT
timeout 2400 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
timeout 900 python bench.py > $OUT/bench512.json 2> $OUT/bench512.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
timeout 900 python bench.py --grid 256 --no-cpu > $OUT/bench256.json 2> $OUT/bench256.err
timeout 1500 python tools/graph_timing.py c1 c1rk4 c4 c4rk4 c2 c2rk4 > $OUT/graph_timing.jsonl 2>&1
timeout 600 python tools/cufft_passes.py > $OUT/cufft_passes.json 2> $OUT/cufft_passes.err
M=smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum
timeout 300 python tools/rhs_timing.py --n 512 --reps 2 > $OUT/rhs_plain.log 2>&1 && \
timeout 1500 ncu --set full --metrics $M --clock-control none --import-source on -k regex:"k_colpass|k_zpass|k_project" \
    -s 6 -c 6 -f -o /tmp/rhs512 python tools/rhs_timing.py --n 512 --reps 2 > $OUT/ncu.log 2>&1 && \
python tools/ncu_kernels.py /tmp/rhs512.ncu-rep --n 512 > $OUT/ncu_kernels.out 2>&1 && \
cp profiles/ncu_kernels.json $OUT/ncu_kernels.json && python tools/ncu_summary.py /tmp/rhs512.ncu-rep > $OUT/ncu_summary.txt 2>&1
for k in k_zpass k_colpass; do
  ncu -i /tmp/rhs512.ncu-rep --page source --csv --print-source sass -k regex:$k --launch-count 2 > $OUT/source_$k.csv 2>/dev/null
done
# launch list of the bench command itself (shares of the step; times under ncu are serialised / cold-cache)
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $OUT/launches_bench512.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu > $OUT/ncu_launches.log 2>&1
bash tools/check_build.sh > $OUT/checks.out 2>&1
