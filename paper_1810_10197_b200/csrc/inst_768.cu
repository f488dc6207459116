// Fast compile-time FFT plan instantiations (see registry.cuh).
#include "registry.cuh"
// Strided passes: 768 = 24 * 32 on the one-butterfly engine, 4-column tiles
// (23.9 vs 25.0 ms per 512^3 RHS for 8 * 8 * 12; DESIGN §3 lists the other
// plans measured).
SRK_DEFINE_SIZE_1(srk_reg_768_base, 768, 4, (24, 32), 24, 24, (8, 8, 12), 8, 8, 12)
void srk_reg_768(KEntry* t) {
  srk_reg_768_base(t);
  // K3: one pencil per CTA, inverse prefix (24, 8), forward suffix (8, 24):
  // 9.02 -> 8.53 ms at 512^3 vs the pencil-pair kernel
  SRK_NS3P(768, (24, 8), (8, 24))
}
