timeout 900 python -m pytest tests/test_gpu_fused_stage.py -q -x > gpurun_out/fused_pytest.log 2>&1; tail -5 gpurun_out/fused_pytest.log
timeout 600 python tools/advance_timeline.py 512 > gpurun_out/atl512_fused.log 2>&1; cat gpurun_out/atl512_fused.log
timeout 600 python bench.py --no-e2e --no-cpu > gpurun_out/bench512_fused.log 2>&1; tail -1 gpurun_out/bench512_fused.log
