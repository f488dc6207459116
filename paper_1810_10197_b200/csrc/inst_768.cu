// Fast compile-time FFT plan instantiations (see registry.cuh).
#include "registry.cuh"
SRK_DEFINE_SIZE(srk_reg_768_base, 768, 24, 4, 8, 8, 12)
void srk_reg_768(KEntry* t) {
  srk_reg_768_base(t);
  SRK_NS3F(768, (24, 8), 24, (8, 24))
}
