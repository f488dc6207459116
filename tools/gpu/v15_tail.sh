# B2 forward suffix 16 24 vs default 24 16 (alternating), then the ncu launch list of the bench command
mkdir -p gpurun_out
for r in 1 2; do for L in "" paper_1810_10197_b200/_lib_b2f3/libsrk.so; do
  SRK_LIB=$L timeout 300 python tools/c4_timing.py >> gpurun_out/b2f3_ab.jsonl 2>&1; echo "lib=$L" >> gpurun_out/b2f3_ab.jsonl
done; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench512.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_l.log 2>&1
echo done
