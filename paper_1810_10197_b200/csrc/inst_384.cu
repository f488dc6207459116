// Fast compile-time FFT plan instantiations (see registry.cuh).
#include "registry.cuh"
#ifndef SRK_P384
#define SRK_P384 0  // measured at 256^3: 0 (3-stage, C=8) 2.85 ms, 1: 3.45, 2: 3.10, 3: 3.03
#endif
#if SRK_P384 == 0
SRK_DEFINE_SIZE_F(srk_reg_384_base, 384, 24, 8, 12, (4, 4, 4, 6), 8, 8, 6)
#elif SRK_P384 == 1
SRK_DEFINE_SIZE_1(srk_reg_384_base, 384, 4, (12, 32), 24, 12, (4, 4, 4, 6), 8, 8, 6)
#elif SRK_P384 == 2
SRK_DEFINE_SIZE_1(srk_reg_384_base, 384, 8, (16, 24), 24, 12, (4, 4, 4, 6), 8, 8, 6)
#else
SRK_DEFINE_SIZE_1(srk_reg_384_base, 384, 4, (16, 24), 24, 12, (4, 4, 4, 6), 8, 8, 6)
#endif
void srk_reg_384(KEntry* t) {
  srk_reg_384_base(t);
  SRK_NS3F(384, (24, 4), 12, (2, 4, 12))
}
