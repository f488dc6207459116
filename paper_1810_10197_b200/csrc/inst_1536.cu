// Fast compile-time FFT plan instantiations (see registry.cuh).
#include "registry.cuh"
SRK_DEFINE_SIZE_F(srk_reg_1536_base, 1536, 24, 4, 12, (4, 4, 4, 4, 6), 8, 8, 24)
void srk_reg_1536(KEntry* t) {
  srk_reg_1536_base(t);
  SRK_NS3F(1536, (8, 8, 6), 12, (4, 4, 2, 12))
}
