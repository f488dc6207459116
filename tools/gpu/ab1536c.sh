for v in base r1 r2; do
  if [ $v = base ]; then L=""; else L="SRK_LIB=$PWD/paper_1810_10197_b200/_lib_$v/libsrk.so"; fi
  env $L timeout 600 python -m pytest tests/test_gpu_fullsize.py -q -x -k "1536" > gpurun_out/p1536_$v.log 2>&1
  env $L timeout 900 python tools/slab_rank_probe.py 1024 8 1 > gpurun_out/srp_$v.log 2>&1
  echo "$v $(tail -1 gpurun_out/p1536_$v.log) $(tail -1 gpurun_out/srp_$v.log | cut -c1-200)"
done
