// Fast compile-time FFT plan instantiations (see registry.cuh).
#include "registry.cuh"
SRK_DEFINE_SIZE_F(srk_reg_384_base, 384, 24, 8, 12, (4, 4, 4, 6), 8, 8, 6)
void srk_reg_384(KEntry* t) {
  srk_reg_384_base(t);
  SRK_NS3F(384, (24, 4), 12, (2, 4, 12))
}
