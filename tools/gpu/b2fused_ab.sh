# 2D Boussinesq fused z-pass (k_zpass_ns3p<..., ZOP_B2>): parity tests, then A/B
# default (FR 24,16) vs SRK_B2GEN (previous k_zpass PPC=1) vs FR 12,32
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_b2.log 2>&1
for r in 1 2; do
  for L in "" paper_1810_10197_b200/_lib_b2gen/libsrk.so paper_1810_10197_b200/_lib_b2fr/libsrk.so; do
    SRK_LIB=$L timeout 300 python tools/c4_timing.py >> gpurun_out/b2_ab.jsonl 2>>gpurun_out/b2_ab.err; echo "lib=$L" >> gpurun_out/b2_ab.jsonl
  done
done
timeout 300 python tools/c4_timing.py > /dev/null 2>&1 && timeout 300 ncu --set full --clock-control none -k regex:"k_zpass" -c 2 -o gpurun_out/b2_zpass python tools/c4_timing.py > gpurun_out/ncu_b2.log 2>&1
echo done
