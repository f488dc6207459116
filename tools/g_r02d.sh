mkdir -p gpurun_out/r02d
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_round2.py tests/test_gpu_fullsize.py -q -x > gpurun_out/r02d/pytest.log 2>&1
echo pytest rc=$? >> gpurun_out/r02d/pytest.log
for i in 1 2 3; do
  SRK_LIB_PATH=$PWD/_lib_base/libsrk.so timeout 300 python tools/rhs_timing.py --n 512 --reps 6 >> gpurun_out/r02d/ab_base.jsonl 2>&1
  timeout 300 python tools/rhs_timing.py --n 512 --reps 6 >> gpurun_out/r02d/ab_new.jsonl 2>&1
done
timeout 300 python tools/rhs_timing.py --n 512 --reps 2 > gpurun_out/r02d/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_zpass_ns3p -s 1 -c 1 -o gpurun_out/r02d/k3 python tools/rhs_timing.py --n 512 --reps 2 > gpurun_out/r02d/ncu.log 2>&1
