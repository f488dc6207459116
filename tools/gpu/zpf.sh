for d in 370 740 1480 2960; do SRK_ZPF1=$d timeout 300 python tools/rhs_timing.py --n 512 --reps 5 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('zpf=$d', d['ms'][2])"; done
bash tools/gpu/ab_k3.sh paper_1810_10197_b200/_lib/libsrk.so paper_1810_10197_b200/_lib_x1/libsrk.so
