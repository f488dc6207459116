mkdir -p gpurun_out/r02l
bash tools/check_build.sh > gpurun_out/r02l/checks.out 2>&1
head -1 gpurun_out/checks/chk.log > gpurun_out/r02l/chk_head.txt
for i in 1 2 3; do
  SRK_LIB_PATH=$PWD/_lib_base/libsrk.so timeout 300 python tools/rhs_timing.py --n 512 --reps 4 >> gpurun_out/r02l/ab_base.jsonl 2>&1
  timeout 300 python tools/rhs_timing.py --n 512 --reps 4 >> gpurun_out/r02l/ab_new.jsonl 2>&1
done
timeout 600 python tools/cufft_passes.py > gpurun_out/r02l/cufft_passes.json 2> gpurun_out/r02l/cufft_passes.err
timeout 300 python tools/graph_probe.py c4 > gpurun_out/r02l/gp_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02l/c4_launches.csv python tools/graph_probe.py c4 > gpurun_out/r02l/gp_ncu.log 2>&1
