for r in 1 2; do for v in base b1 b2; do
  if [ $v = base ]; then L=""; else L="SRK_LIB=$PWD/paper_1810_10197_b200/_lib_$v/libsrk.so"; fi
  echo "$v $(env $L timeout 300 python tools/rhs_timing.py --n 1024 --dims 2 --density --reps 30)"
done; done
SRK_LIB=$PWD/paper_1810_10197_b200/_lib_b1/libsrk.so timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "boussinesq_2d" 2>&1 | tail -1
SRK_LIB=$PWD/paper_1810_10197_b200/_lib_b2/libsrk.so timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "boussinesq_2d" 2>&1 | tail -1
