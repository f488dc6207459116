mkdir -p gpurun_out/r02a
nvidia-smi > gpurun_out/r02a/smi.txt 2>&1
timeout 300 python tools/rhs_timing.py --n 512 --reps 6 > gpurun_out/r02a/rhs512.json 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_zpass_ns3p -s 1 -c 1 -o gpurun_out/r02a/k3 python tools/rhs_timing.py --n 512 --reps 2 > gpurun_out/r02a/ncu.log 2>&1
echo rc=$?
