// Fast compile-time FFT plan instantiations (see registry.cuh).
#include "registry.cuh"
// 384 (256^3): three-stage plan on 8-column strided tiles (2.85 ms per pass
// at 256^3; one-butterfly plans 3.0-3.45 ms)
SRK_DEFINE_SIZE_F(srk_reg_384_base, 384, 24, 8, 12, (4, 4, 4, 6), 8, 8, 6)
void srk_reg_384(KEntry* t) {
  srk_reg_384_base(t);
  // the pencil-pair z-pass already runs 5 CTAs per SM at 384 (one-pencil: 1.25 vs 1.02 ms)
  SRK_NS3F(384, (24, 4), 12, (2, 4, 12))
}
