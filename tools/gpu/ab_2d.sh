for i in 1 2; do
timeout 300 python tools/rhs_timing.py --n 1024 --dims 2 --density --reps 30 > gpurun_out/t2d_base$i.log 2>&1
SRK_LIB=$PWD/paper_1810_10197_b200/_lib_e12/libsrk.so timeout 300 python tools/rhs_timing.py --n 1024 --dims 2 --density --reps 30 > gpurun_out/t2d_e12_$i.log 2>&1
done
SRK_LIB=$PWD/paper_1810_10197_b200/_lib_e12/libsrk.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "boussinesq" > gpurun_out/pytest_e12.log 2>&1; tail -1 gpurun_out/pytest_e12.log
for f in gpurun_out/t2d_*.log; do echo $f $(cat $f); done
