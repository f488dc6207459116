# round evidence: tests, bench (512^3 and 256^3), slab bench, launch list, full ncu of the RHS kernels
# (each guarded by timeout; ncu runs only after the same command exited 0 without it)
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
timeout 600 python bench.py > gpurun_out/bench512.log 2>&1
timeout 600 python bench.py --grid 256 --no-e2e --no-cpu > gpurun_out/bench256.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1
timeout 900 python bench.py --mode slab --steps 3 --warmup 3 > gpurun_out/bench_slab.log 2>&1
timeout 300 python tools/rhs_timing.py --n 512 --reps 5 > gpurun_out/t512.log 2>&1
timeout 300 python tools/phase_timing.py 512 > gpurun_out/phase512.log 2>&1
timeout 300 python tools/rhs_timing.py --n 512 --reps 2 > gpurun_out/t512b.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 6 -c 12 --csv --log-file gpurun_out/launches512.csv python tools/rhs_timing.py --n 512 --reps 2 > gpurun_out/ncu_l.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_(zpass|colpass|project)" -c 6 -o gpurun_out/prof512_full python tools/rhs_timing.py --n 512 --reps 2 > gpurun_out/ncu_f.log 2>&1
echo done
