// Fast compile-time FFT plan instantiations (see registry.cuh).
#include "registry.cuh"
SRK_DEFINE_SIZE_F(srk_reg_192, 192, 24, 16, 12, (4, 4, 12), 8, 8, 3)
