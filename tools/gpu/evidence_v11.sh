# round evidence v11 (one-pencil K3, fused stage combination): tests, benches, per-kernel timing, launch list, full ncu
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
timeout 600 python bench.py > gpurun_out/bench512.log 2>&1
timeout 600 python bench.py --grid 256 --no-e2e --no-cpu > gpurun_out/bench256.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1
timeout 300 python tools/rhs_timing.py --n 512 --reps 5 > gpurun_out/t512.log 2>&1
timeout 600 python tools/advance_timeline.py 512 > gpurun_out/atl512.log 2>&1
timeout 300 python tools/rhs_timing.py --n 512 --reps 2 > gpurun_out/t512b.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 6 -c 16 --csv --log-file gpurun_out/launches512.csv python tools/rhs_timing.py --n 512 --reps 2 > gpurun_out/ncu_l.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_(zpass|colpass|project)" -c 6 -o gpurun_out/prof512_full python tools/rhs_timing.py --n 512 --reps 2 > gpurun_out/ncu_f.log 2>&1
echo done
