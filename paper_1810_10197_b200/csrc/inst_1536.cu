// Fast compile-time FFT plan instantiations (see registry.cuh).
#include "registry.cuh"
SRK_DEFINE_SIZE(srk_reg_1536, 1536, 24, 4, 8, 8, 24)
