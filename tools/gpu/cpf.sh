for d in 0 444 888 1776; do SRK_CPF=$d timeout 300 python tools/rhs_timing.py --n 512 --reps 5 | sed "s/^/cpf=$d /" | cut -c1-150; done
for d in 0 444; do SRK_CPF=$d timeout 300 python tools/rhs_timing.py --n 512 --reps 5 | sed "s/^/cpf=$d /" | cut -c1-150; done
