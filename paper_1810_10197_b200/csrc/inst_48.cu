// Fast compile-time FFT plan instantiations (see registry.cuh).
#include "registry.cuh"
SRK_DEFINE_SIZE(srk_reg_48_base, 48, 12, 32, 4, 4, 3)
void srk_reg_48(KEntry* t) {
  srk_reg_48_base(t);
  SRK_NS3F(48, (12), 12, (12))
}
