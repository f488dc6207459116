// Fast compile-time FFT plan instantiations (see registry.cuh).
#include "registry.cuh"
// 768 = 24 * 32 on the one-butterfly engine: 23.9 vs 25.0 ms per 512^3 RHS for 8 * 8 * 12
#ifdef SRK_OLD768
SRK_DEFINE_SIZE(srk_reg_768_base, 768, 24, 4, 8, 8, 12)
#else
#ifndef SRK_C768
#define SRK_C768 4  // strided-pass tile columns
#endif
SRK_DEFINE_SIZE_1(srk_reg_768_base, 768, SRK_C768, (24, 32), 24, 24, (8, 8, 12), 8, 8, 12)
#endif
void srk_reg_768(KEntry* t) {
  srk_reg_768_base(t);
#ifndef SRK_Z768F
#define SRK_Z768F 2  // forward suffix: 0 (8,24) on 96 threads 9.10 ms, 1 (12,16) 9.50, 2 (16,12) 8.97
#endif
#if SRK_Z768F == 0
  SRK_NS3F(768, (24, 8), 24, (8, 24))
#elif SRK_Z768F == 1
  SRK_NS3F(768, (24, 8), 0, (12, 16))
#else
  SRK_NS3F(768, (24, 8), 0, (16, 12))
#endif
#ifndef SRK_ZPAIR
  // one pencil per CTA, forward suffix (8, 24): K3 9.02 -> 8.53 ms at 512^3
  // (forward (16, 12) 8.67, (12, 16) 8.84, (24, 8) 8.64; inverse (8, 24) 8.69)
#if defined(SRK_K3E12) && SRK_K3E12 == 1
  SRK_NS3P12(768, (12, 4, 4), (8, 24))
#elif defined(SRK_K3E12) && SRK_K3E12 == 2
  SRK_NS3P12(768, (4, 4, 12), (8, 24))
#elif defined(SRK_K3E12) && SRK_K3E12 == 3
  SRK_NS3P12(768, (12, 4, 4), (16, 12))
#else
  SRK_NS3P(768, (24, 8), (8, 24))
#endif
#endif
}
