mkdir -p gpurun_out/r02g
timeout 900 python -m pytest tests/test_gpu_graphs.py tests/test_gpu_behaviour.py tests/test_gpu_configs.py -q -x > gpurun_out/r02g/pytest.log 2>&1
echo pytest rc=$? >> gpurun_out/r02g/pytest.log
timeout 900 python tools/graph_timing.py all > gpurun_out/r02g/graph_timing.jsonl 2> gpurun_out/r02g/graph_timing.err
echo timing rc=$?
