// Fast compile-time FFT plan instantiations (see registry.cuh).
#include "registry.cuh"
SRK_DEFINE_SIZE_F(srk_reg_96_base, 96, 24, 32, 12, (4, 4, 6), 8, 4, 3)
void srk_reg_96(KEntry* t) {
  srk_reg_96_base(t);
  SRK_NS3F(96, (24), 12, (2, 12))
}
