// Fast compile-time FFT plan instantiations (see registry.cuh).
#include "registry.cuh"
SRK_DEFINE_SIZE_F(srk_reg_1536, 1536, 24, 4, 12, (4, 4, 4, 4, 6), 8, 8, 24)
