mkdir -p gpurun_out/r02f
timeout 900 python -m pytest tests/test_gpu_graphs.py tests/test_gpu_parity.py tests/test_gpu_fused_stage.py tests/test_gpu_bench.py -q -x > gpurun_out/r02f/pytest.log 2>&1
echo pytest rc=$? >> gpurun_out/r02f/pytest.log
timeout 900 python tools/graph_timing.py all > gpurun_out/r02f/graph_timing.jsonl 2> gpurun_out/r02f/graph_timing.err
echo timing rc=$?
