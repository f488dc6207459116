# final v15 check of the committed tree: smoke, 512^3 bench line, reference arm, C4 2D timing
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/bench512.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1
timeout 300 python tools/c4_timing.py > gpurun_out/c4.log 2>&1
echo done
