// Fast compile-time FFT plan instantiations (see registry.cuh).
#include "registry.cuh"
SRK_DEFINE_SIZE_PLAIN(srk_reg_32, 32, 8, 32, 8, 4)
SRK_DEFINE_SIZE_PLAIN(srk_reg_64, 64, 8, 16, 8, 8)
SRK_DEFINE_SIZE_PLAIN(srk_reg_128, 128, 8, 8, 8, 4, 4)
SRK_DEFINE_SIZE_PLAIN(srk_reg_256, 256, 8, 8, 8, 8, 4)
SRK_DEFINE_SIZE_PLAIN(srk_reg_512, 512, 8, 8, 8, 8, 8)
SRK_DEFINE_SIZE_PLAIN(srk_reg_1024, 1024, 8, 8, 8, 8, 4, 4)
