# session-3 re-entry check: tests, smoke, bench at 512^3
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/bench512.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench512.log
