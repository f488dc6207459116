python tools/rhs_timing.py --n 512 --reps 2 > gpurun_out/t512.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_colpass" -c 3 -o gpurun_out/prof512_col python tools/rhs_timing.py --n 512 --reps 2 > gpurun_out/ncu512.log 2>&1
echo done
