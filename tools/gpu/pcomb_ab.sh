# density fused stage sum: parity tests, then alternating A/B (fused vs SRK_NO_PCOMB=1)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fused_stage.py tests/test_gpu_configs.py -q > gpurun_out/pytest_fused.log 2>&1
for c in 2d 3d; do for r in 1 2; do
  timeout 300 python tools/pcomb_ab.py $c >> gpurun_out/pcomb_ab.jsonl 2>>gpurun_out/pcomb_ab.err
  SRK_NO_PCOMB=1 timeout 300 python tools/pcomb_ab.py $c >> gpurun_out/pcomb_ab.jsonl 2>>gpurun_out/pcomb_ab.err
done; done
echo done
