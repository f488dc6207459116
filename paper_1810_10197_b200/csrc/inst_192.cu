// Fast compile-time FFT plan instantiations (see registry.cuh).
#include "registry.cuh"
SRK_DEFINE_SIZE_F(srk_reg_192_base, 192, 24, 16, 12, (4, 4, 12), 8, 8, 3)
void srk_reg_192(KEntry* t) {
  srk_reg_192_base(t);
  SRK_NS3F(192, (24, 2), 12, (4, 12))
}
