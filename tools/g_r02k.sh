mkdir -p gpurun_out/r02k
timeout 600 python tools/sanitize_cases.py > gpurun_out/r02k/plain.log 2>&1 && \
timeout 2400 compute-sanitizer --tool memcheck --print-limit 100 python tools/sanitize_cases.py > gpurun_out/r02k/memcheck.log 2>&1
echo memcheck rc=$? >> gpurun_out/r02k/memcheck.log
