X=paper_1810_10197_b200/_lib_x/libsrk.so
SRK_LIB=$X timeout 600 python -m pytest tests/test_gpu_fullsize.py -q -s 2>&1 | grep -E "512|passed|failed|Error"
bash tools/gpu/ab.sh $X
SRK_LIB=$X SRK_ZPF1=0 timeout 300 python tools/rhs_timing.py --n 512 --reps 5 | sed 's/^/x-nopf /'
