for i in 1 2; do
timeout 600 python bench.py --grid 256 --no-cpu --no-e2e > gpurun_out/b256_a$i.log 2>&1
SRK_NO_HOST_RESULT=1 timeout 600 python bench.py --grid 256 --no-cpu --no-e2e > gpurun_out/b256_b$i.log 2>&1
done
for f in gpurun_out/b256_*.log; do echo $f $(tail -1 $f | cut -c1-140); done
