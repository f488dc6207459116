for r in 1 2; do for v in base e3 g1 g3; do
  if [ $v = base ]; then L=""; else L="SRK_LIB=$PWD/paper_1810_10197_b200/_lib_$v/libsrk.so"; fi
  echo "$v $(env $L timeout 300 python tools/rhs_timing.py --n 512 --reps 4 | cut -c1-90)"
done; done
SRK_LIB=$PWD/paper_1810_10197_b200/_lib_g3/libsrk.so timeout 600 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -q -x -k "512 or golden or hit" 2>&1 | tail -1
