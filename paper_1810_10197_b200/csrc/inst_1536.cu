// Fast compile-time FFT plan instantiations (see registry.cuh).
#include "registry.cuh"
#ifndef SRK_C1536
// strided-pass tile columns at 1536 (3D 1024^3 slabs): two columns, 128 threads,
// 3 CTAs per SM instead of one 256-thread CTA (140+ registers): one 1024^3/8 rank,
// K1 4.69 -> 3.58, K2 10.77 -> 6.43, K4 4.64 -> 3.06 ms (tools/slab_rank_probe.py)
#define SRK_C1536 2
#endif
#if defined(SRK_R1536) && SRK_R1536 == 1
SRK_DEFINE_SIZE_F(srk_reg_1536_base, 1536, 24, SRK_C1536, 12, (4, 4, 4, 4, 6), 24, 8, 8)
#elif defined(SRK_R1536) && SRK_R1536 == 2
SRK_DEFINE_SIZE_F(srk_reg_1536_base, 1536, 24, SRK_C1536, 12, (4, 4, 4, 4, 6), 8, 24, 8)
#else
SRK_DEFINE_SIZE_F(srk_reg_1536_base, 1536, 24, SRK_C1536, 12, (4, 4, 4, 4, 6), 8, 8, 24)
#endif
void srk_reg_1536(KEntry* t) {
  srk_reg_1536_base(t);
  SRK_NS3F(1536, (8, 8, 6), 12, (4, 4, 2, 12))
#ifndef SRK_NS3P1536
#define SRK_NS3P1536 3
#endif
  // one z-pencil per CTA (192 threads, 89 KB, 2 CTAs per SM) instead of the pencil
  // pair (384 threads, 166 KB, 1 CTA per SM): K3 of one 1024^3/8 rank 13.75 ->
  // 10.66 ms with the forward suffix (24, 16); (16, 24) 11.55, (8, 8, 6) 11.72
#if SRK_NS3P1536 == 1
  SRK_NS3P(1536, (8, 8, 6), (16, 24))
#elif SRK_NS3P1536 == 2
  SRK_NS3P(1536, (8, 8, 6), (8, 8, 6))
#elif SRK_NS3P1536 == 3
  SRK_NS3P(1536, (8, 8, 6), (24, 16))
#elif SRK_NS3P1536 == 4
  SRK_NS3P(1536, (24, 8, 2), (24, 16))
#elif SRK_NS3P1536 == 5
  SRK_NS3P(1536, (12, 8, 4), (24, 16))
#elif SRK_NS3P1536 == 6
  SRK_NS3P(1536, (6, 8, 8), (24, 16))
#elif SRK_NS3P1536 == 7
  SRK_NS3P(1536, (8, 8, 6), (32, 12))
#elif SRK_NS3P1536 == 8
  SRK_NS3P(1536, (8, 8, 6), (12, 32))
#endif
#if !defined(SRK_B2PAIR) && !defined(SRK_B2GEN)
  // 2D Boussinesq z-pass with the fused middle stage (v15): one pencil per CTA,
  // inverse prefix 8 8 6 on 2 columns (E = 24, 128 threads), last inverse
  // radix-4 | u x w, rho u | first forward radix-4 in registers, forward suffix
  // FR on the 2 packed product columns
#if defined(SRK_B2FRSEL) && SRK_B2FRSEL == 2
#define SRK_B2FR 12, 32
#elif defined(SRK_B2FRSEL) && SRK_B2FRSEL == 3
#define SRK_B2FR 16, 24
#else
#define SRK_B2FR 24, 16
#endif
  {
    using Z2 = ColTile<1536, 2>;
    using E2 = FastFFT<1536, 24, Z2, 8, 8, 6>;
    t[KK_Z_B2] = KEntry{(const void*)(k_zpass_ns3p<1536, Z2, E2, ZOP_B2, SRK_B2FR>), E2::NT, 2,
                        (int)(Z2::SIZE * 16) + E2::TWN * 16, 0, 1};
  }
#elif !defined(SRK_B2PAIR)
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
