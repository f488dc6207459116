SRK_NOPERSIST=1 python tools/rhs_timing.py --n 512 --reps 2 > gpurun_out/t512.log 2>&1 && \
SRK_NOPERSIST=1 ncu --set full --clock-control none -k regex:"k_zpass" -c 1 -o gpurun_out/prof512_k3b python tools/rhs_timing.py --n 512 --reps 2 > gpurun_out/ncu512.log 2>&1
echo done
