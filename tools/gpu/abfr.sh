for r in 1 2; do for v in base f1 f2 f3; do
  if [ $v = base ]; then L=""; else L="SRK_LIB=$PWD/paper_1810_10197_b200/_lib_$v/libsrk.so"; fi
  echo "$v $(env $L timeout 300 python tools/rhs_timing.py --n 512 --reps 4 | cut -c1-90)"
done; done
