python bench.py > gpurun_out/bench512.log 2>&1
python bench.py --grid 256 --no-cpu > gpurun_out/bench256.log 2>&1
python tools/rhs_timing.py --n 512 --reps 2 > gpurun_out/t512.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 20 -c 60 --csv --log-file gpurun_out/launches512.csv python tools/rhs_timing.py --n 512 --reps 2 > gpurun_out/ncu_l.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_(zpass|colpass|project)" -c 7 -o gpurun_out/prof512_full python tools/rhs_timing.py --n 512 --reps 2 > gpurun_out/ncu_f.log 2>&1
echo done
