// Runtime-plan (GenericFFT) instantiations for small lengths with factors in
// {2,3,4,5,7,8} that have no compile-time plan -- the odd grids of the
// reference's own test suite, e.g. (8, 6, 4) and (8, 10, 6).
#include "registry.cuh"

void srk_reg_generic(KEntry* t) {
  using SE = GenericFFT<GenCols<32>>;
  t[KK_INV] = SRK_ENTRY((k_colpass<SE, PK_INV, +1, 0>), SE, 0);
  t[KK_FWD] = SRK_ENTRY((k_colpass<SE, PK_FWD, -1, 0>), SE, 0);
  t[KK_INV_P] = t[KK_INV];
  t[KK_FWD_P] = t[KK_FWD];
  t[KK_INV_RHS] = SRK_ENTRY((k_colpass<SE, PK_INV_RHS, +1, 0>), SE, 0);
  t[KK_INV_RHS_SLAB] = SRK_ENTRY((k_colpass<SE, PK_INV_RHS, +1, PF_BOUT>), SE, 0);
  t[KK_INV_P_SLAB] = SRK_ENTRY((k_colpass<SE, PK_INV, +1, PF_BIN>), SE, 0);
  t[KK_FWD_P_SLABO] = SRK_ENTRY((k_colpass<SE, PK_FWD, -1, PF_BOUT>), SE, 0);
  t[KK_FWD_P_SLABI] = SRK_ENTRY((k_colpass<SE, PK_FWD, -1, PF_BIN>), SE, 0);
  t[KK_INV_KX] = SRK_ENTRY((k_colpass<SE, PK_INV_KX, +1, 0>), SE, 0);
  t[KK_INV_KX_SLAB] = SRK_ENTRY((k_colpass<SE, PK_INV_KX, +1, PF_BOUT>), SE, 0);
  t[KK_INV_KX_PEER] = SRK_ENTRY((k_colpass<SE, PK_INV_KX, +1, PF_BOUT | PF_PEER>), SE, 0);
  t[KK_FWD_P_PEER] = SRK_ENTRY((k_colpass<SE, PK_FWD, -1, PF_BOUT | PF_PEER>), SE, 0);
  t[KK_INV_CURLY] = SRK_ENTRY((k_colpass<SE, PK_INV_CURLY, +1, 0>), SE, 0);
  t[KK_INV_CURLY_SLAB] = SRK_ENTRY((k_colpass<SE, PK_INV_CURLY, +1, PF_BIN>), SE, 0);
  using Z4 = ColTile<SRK_GEN_MAXM, 4>;
  using Z3 = ColTile<SRK_GEN_MAXM, 3>;
  using Z6 = ColTile<SRK_GEN_MAXM, 6>;
  using Z7 = ColTile<SRK_GEN_MAXM, 7>;
  using E4 = GenericFFT<Z4>;
  using E3 = GenericFFT<Z3>;
  using E6 = GenericFFT<Z6>;
  using E7 = GenericFFT<Z7>;
  t[KK_Z_C2R] = SRK_ENTRY((k_zpass<E4, Z4, ZOP_C2R>), E4, Z4::SIZE * 16 + SRK_GEN_STG(4));
  t[KK_Z_R2C] = SRK_ENTRY((k_zpass<E4, Z4, ZOP_R2C>), E4, Z4::SIZE * 16);
  t[KK_Z_NS3] = SRK_ENTRY((k_zpass<E6, Z6, ZOP_NS3>), E6, Z6::SIZE * 16 + SRK_GEN_STG(6));
  t[KK_Z_NS2] = SRK_ENTRY((k_zpass<E3, Z3, ZOP_NS2>), E3, Z3::SIZE * 16 + SRK_GEN_STG(3));
  t[KK_Z_B3] = SRK_ENTRY((k_zpass<E7, Z7, ZOP_B3>), E7, Z7::SIZE * 16 + SRK_GEN_STG(7));
  t[KK_Z_B2] = SRK_ENTRY((k_zpass<E4, Z4, ZOP_B2>), E4, Z4::SIZE * 16 + SRK_GEN_STG(4));
}
