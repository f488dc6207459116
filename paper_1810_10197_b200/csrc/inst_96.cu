// Fast compile-time FFT plan instantiations (see registry.cuh).
#include "registry.cuh"
SRK_DEFINE_SIZE(srk_reg_96, 96, 24, 32, 8, 4, 3)
