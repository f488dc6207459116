// Fast compile-time FFT plan instantiations (see registry.cuh).
#include "registry.cuh"
SRK_DEFINE_SIZE(srk_reg_192, 192, 24, 16, 8, 8, 3)
