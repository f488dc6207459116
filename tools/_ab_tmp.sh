mkdir -p gpurun_out/r02u
timeout 900 python -m pytest tests/test_gpu_round2.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_fused_stage.py -q -x > gpurun_out/r02u/pytest.log 2>&1; echo rc=$? >> gpurun_out/r02u/pytest.log
for i in 1 2 3; do
  SRK_LIB_PATH=$PWD/_lib_base/libsrk.so timeout 300 python tools/rhs_timing.py --n 512 --reps 4 >> gpurun_out/r02u/ab_base.jsonl 2>&1
  timeout 300 python tools/rhs_timing.py --n 512 --reps 4 >> gpurun_out/r02u/ab_new.jsonl 2>&1
done
bash tools/check_build.sh > gpurun_out/r02u/checks.out 2>&1
timeout 300 python tools/rhs_timing.py --n 512 --reps 2 > gpurun_out/r02u/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_zpass -s 1 -c 1 -f -o gpurun_out/r02u/k3q python tools/rhs_timing.py --n 512 --reps 2 > gpurun_out/r02u/ncu.log 2>&1
