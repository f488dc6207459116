for v in base pre hit re2k hit_pre base; do timeout 300 python tools/rhs_bisect.py $v >> gpurun_out/bisect.log 2>&1; done
nvidia-smi --query-gpu=clocks.sm,clocks.mem,power.draw,temperature.gpu --format=csv >> gpurun_out/bisect.log
cat gpurun_out/bisect.log
