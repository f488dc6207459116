// Fast compile-time FFT plan instantiations (see registry.cuh).
#include "registry.cuh"
SRK_DEFINE_SIZE(srk_reg_768, 768, 24, 4, 8, 8, 12)
