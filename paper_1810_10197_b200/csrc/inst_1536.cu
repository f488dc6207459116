// Fast compile-time FFT plan instantiations (see registry.cuh).
#include "registry.cuh"
// Strided-pass tiles at 1536 (3D 1024^3 slabs): two columns, 128 threads, 3 CTAs
// per SM instead of one 256-thread CTA (140+ registers): one 1024^3/8 rank, K1
// 4.69 -> 3.58, K2 10.77 -> 6.43, K4 4.64 -> 3.06 ms (tools/slab_rank_probe.py)
SRK_DEFINE_SIZE_F(srk_reg_1536_base, 1536, 24, 2, 12, (4, 4, 4, 4, 6), 8, 8, 24)
void srk_reg_1536(KEntry* t) {
  srk_reg_1536_base(t);
  // one z-pencil per CTA (192 threads, 89 KB, 2 CTAs per SM) instead of the pencil
  // pair (384 threads, 166 KB, 1 CTA per SM): K3 of one 1024^3/8 rank 13.75 ->
  // 10.66 ms with the forward suffix (24, 16); (16, 24) 11.55, (8, 8, 6) 11.72
  SRK_NS3P(1536, (8, 8, 6), (24, 16))
  // 2D Boussinesq z-pass with the fused middle stage (v15): one pencil per CTA,
  // inverse prefix 8 8 6 on 2 columns (E = 24, 128 threads), last inverse
  // radix-4 | u x w, rho u | first forward radix-4 in registers, forward suffix
  // (24, 16) on the 2 packed product columns
  {
    using Z2 = ColTile<1536, 2>;
    using E2 = FastFFT<1536, 24, Z2, 8, 8, 6>;
    t[KK_Z_B2] = KEntry{(const void*)(k_zpass_ns3p<1536, Z2, E2, ZOP_B2, 24, 16>), E2::NT, 2,
                        (int)(Z2::SIZE * 16) + E2::TWN * 16, 1};
  }
  // 2D x passes (K1 with the curl on load, K5) on two-column tiles: 128 threads,
  // up to 3 CTAs per SM (the 2D working set is L2-resident, so 32 B row pieces cost
  // little; 3D keeps the four-column tiles of the base plan)
  {
    using SL2 = RowTile<1536, 2>;
    using SE2 = FastFFT<1536, 24, SL2, 8, 8, 24>;
    constexpr int rhs_smem = (SL2::SIZE > 2 * 1024 * 2 ? SL2::SIZE : 2 * 1024 * 2) * 16;
    t[KK_INV_RHS] = SRK_ENTRY((k_colpass<SE2, PK_INV_RHS, +1, PF_CTN>), SE2, rhs_smem);
    t[KK_FWD_P2D] = SRK_ENTRY((k_colpass<SE2, PK_FWD, -1, PF_CTN>), SE2, SL2::SIZE * 16);
  }
}
