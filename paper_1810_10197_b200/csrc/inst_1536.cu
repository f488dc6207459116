// Fast compile-time FFT plan instantiations (see registry.cuh).
#include "registry.cuh"
SRK_DEFINE_SIZE_F(srk_reg_1536_base, 1536, 24, 4, 12, (4, 4, 4, 4, 6), 8, 8, 24)
void srk_reg_1536(KEntry* t) {
  srk_reg_1536_base(t);
  SRK_NS3F(1536, (8, 8, 6), 12, (4, 4, 2, 12))
#ifndef SRK_B2PAIR
  // 2D Boussinesq z-pass, one pencil per CTA (2 columns, 128 threads, 3 CTAs/SM)
  {
    using Z2 = ColTile<1536, 2>;
#ifdef SRK_B2E12
    using E2 = FastFFT<1536, 12, Z2, 4, 4, 4, 4, 6>;
#else
    using E2 = FastFFT<1536, 24, Z2, 8, 8, 24>;
#endif
    t[KK_Z_B2] = KEntry{(const void*)(k_zpass<E2, Z2, ZOP_B2, E2, 1>), E2::NT, 2, (int)(Z2::SIZE * 16) + E2::TWN * 16, 0, 1};
  }
#endif
#ifndef SRK_2D4COL
  // 2D x passes (K1 with the curl on load, K5) on two-column tiles: 128 threads,
  // up to 3 CTAs per SM (the 2D working set is L2-resident, so 32 B row pieces cost
  // little; 3D keeps the four-column tiles of the base plan)
  {
    using SL2 = RowTile<1536, 2>;
#ifdef SRK_X2E12
    using SE2 = FastFFT<1536, 12, SL2, 4, 4, 4, 4, 6>;
#else
    using SE2 = FastFFT<1536, 24, SL2, 8, 8, 24>;
#endif
    constexpr int rhs_smem = (SL2::SIZE > 2 * 1024 * 2 ? SL2::SIZE : 2 * 1024 * 2) * 16;
    t[KK_INV_RHS] = SRK_ENTRY((k_colpass<SE2, PK_INV_RHS, +1, PF_CTN>), SE2, rhs_smem);
    t[KK_FWD_P2D] = SRK_ENTRY((k_colpass<SE2, PK_FWD, -1, PF_CTN>), SE2, SL2::SIZE * 16);
  }
#endif
}
