# v15 re-check after container restore: tests, smoke, bench (512^3, 256^3), reference arm, bench launch list
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/bench512.log 2>&1
timeout 600 python bench.py --grid 256 --no-e2e --no-cpu > gpurun_out/bench256.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1
echo done
