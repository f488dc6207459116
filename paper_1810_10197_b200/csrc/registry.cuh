// Kernel registry: one entry per (FFT length, kernel kind).  Fast sizes are
// compile-time plans instantiated in inst_<M>.cu; anything else small falls back
// to the runtime GenericFFT entries in inst_generic.cu.
#pragma once

#include "pass_kernels.cuh"

enum KernelKind {
  KK_INV = 0,      // strided inverse C2C, runtime n (unpadded transforms)
  KK_INV_RHS = 1,  // strided inverse C2C with curl on load, padded      K1
  KK_FWD = 2,      // strided forward C2C, runtime n
  KK_Z_C2R = 3,
  KK_Z_R2C = 4,
  KK_Z_NS3 = 5,
  KK_Z_NS2 = 6,
  KK_Z_B3 = 7,
  KK_Z_B2 = 8,
  KK_INV_P = 9,          // padded inverse (n = 2M/3 compile time)        K2
  KK_FWD_P = 10,         // padded forward + truncation                   K4, K5
  KK_INV_RHS_SLAB = 11,  // K1, blocked output rows (all-to-all #1 send)
  KK_INV_P_SLAB = 12,    // K2, blocked input rows (all-to-all #1 receive)
  KK_FWD_P_SLABO = 13,   // K4, blocked output rows (all-to-all #2 send)
  KK_FWD_P_SLABI = 14,   // K5, blocked input rows (all-to-all #2 receive)
  KK_INV_KX = 15,        // 3D K1 (u, kx u signals)
  KK_INV_KX_SLAB = 16,   // 3D K1, all-to-all #1 send layout
  KK_INV_CURLY = 17,     // 3D K2 (curl completed on load)
  KK_INV_CURLY_SLAB = 18,  // 3D K2 from the all-to-all #1 receive layout
  KK_FWD_P2D = 19,         // 2D x-forward + truncation (K5) when a narrower tile is registered
  KK_INV_KX_PEER = 20,     // 3D K1, rows stored straight into the peers' all-to-all #1 receive buffers
  KK_FWD_P_PEER = 21,      // K4, rows stored straight into the peers' all-to-all #2 receive buffers
  KK_COUNT = 22
};

struct KEntry {
  const void* fn;
  int nt;    // threads per block
  int cols;  // columns per block (strided) / complex columns capacity (z)
  int smem;  // dynamic shared memory bytes
  int ppc = 2;         // z pass: pencils per CTA (k_zpass_ns3p: 1)
};

// plain z ops process up to this many real signals per pencil per launch
#define SRK_Z_PLAIN_C 4
// generic z kernels stage their inputs after the tile: 2 * C * (MAXM/2+1) complex
#define SRK_GEN_STG(C) (2 * (C) * (SRK_GEN_MAXM / 2 + 1) * 16)

typedef void (*srk_reg_fn)(KEntry* tab);

// Layout used only for the column count of the generic strided engine.
template <int C_>
struct GenCols {
  static constexpr int C = C_;
};

#define SRK_ENTRY(KFN, ENG, SMB) KEntry{(const void*)(KFN), ENG::NT, ENG::C, (int)(SMB) + ENG::TWN * 16}

// Strided kinds of one fast length (SE / SL in scope).
#define SRK_RHS_SMEM(M, CS) ((SL::SIZE > 2 * (2 * M / 3) * CS ? SL::SIZE : 2 * (2 * M / 3) * CS) * 16)
#define SRK_STRIDED_KINDS(M, CS)                                                                   \
    t[KK_INV] = SRK_ENTRY((k_colpass<SE, PK_INV, +1, 0>), SE, SL::SIZE * 16);                      \
    t[KK_FWD] = SRK_ENTRY((k_colpass<SE, PK_FWD, -1, 0>), SE, SL::SIZE * 16);                      \
    t[KK_INV_P] = SRK_ENTRY((k_colpass<SE, PK_INV, +1, PF_CTN>), SE, SL::SIZE * 16);               \
    t[KK_FWD_P] = SRK_ENTRY((k_colpass<SE, PK_FWD, -1, PF_CTN>), SE, SL::SIZE * 16);               \
    t[KK_INV_RHS] = SRK_ENTRY((k_colpass<SE, PK_INV_RHS, +1, PF_CTN>), SE, SRK_RHS_SMEM(M, CS));   \
    t[KK_INV_RHS_SLAB] = SRK_ENTRY((k_colpass<SE, PK_INV_RHS, +1, PF_CTN | PF_BOUT>), SE,          \
                                   SRK_RHS_SMEM(M, CS));                                           \
    t[KK_INV_P_SLAB] = SRK_ENTRY((k_colpass<SE, PK_INV, +1, PF_CTN | PF_BIN>), SE, SL::SIZE * 16); \
    t[KK_FWD_P_SLABO] = SRK_ENTRY((k_colpass<SE, PK_FWD, -1, PF_CTN | PF_BOUT>), SE, SL::SIZE * 16); \
    t[KK_FWD_P_SLABI] = SRK_ENTRY((k_colpass<SE, PK_FWD, -1, PF_CTN | PF_BIN>), SE, SL::SIZE * 16); \
    t[KK_INV_KX] = SRK_ENTRY((k_colpass<SE, PK_INV_KX, +1, PF_CTN>), SE, SL::SIZE * 16);           \
    t[KK_INV_KX_SLAB] = SRK_ENTRY((k_colpass<SE, PK_INV_KX, +1, PF_CTN | PF_BOUT>), SE, SL::SIZE * 16); \
    t[KK_INV_KX_PEER] = SRK_ENTRY((k_colpass<SE, PK_INV_KX, +1, PF_CTN | PF_BOUT | PF_PEER>), SE, SL::SIZE * 16); \
    t[KK_FWD_P_PEER] = SRK_ENTRY((k_colpass<SE, PK_FWD, -1, PF_CTN | PF_BOUT | PF_PEER>), SE, SL::SIZE * 16); \
    t[KK_INV_CURLY] = SRK_ENTRY((k_colpass<SE, PK_INV_CURLY, +1, PF_CTN>), SE, SRK_RHS_SMEM(M, CS)); \
    t[KK_INV_CURLY_SLAB] = SRK_ENTRY((k_colpass<SE, PK_INV_CURLY, +1, PF_CTN | PF_BIN>), SE,       \
                                     SRK_RHS_SMEM(M, CS));

// Instantiate every kernel kind for one fast FFT length.
#define SRK_DEFINE_SIZE(NAME, M, E, CS, ...) SRK_DEFINE_SIZE_F(NAME, M, E, CS, E, (__VA_ARGS__), __VA_ARGS__)
#define SRK_UNPAREN(...) __VA_ARGS__
// EF / FR: elements-per-thread and radices of the forward transform of the NS3
// z-pass (3 forward columns vs 6 inverse ones: E = 12 keeps every thread busy).
#define SRK_DEFINE_SIZE_F(NAME, M, E, CS, EF, FR, ...)                                             \
  void NAME(KEntry* t) {                                                                           \
    using SL = RowTile<M, CS>;                                                                     \
    using SE = FastFFT<M, E, SL, __VA_ARGS__>;                                                     \
    SRK_STRIDED_KINDS(M, CS)                                                                       \
    using Z4 = ColTile<M, 4>;                                                                      \
    using Z3 = ColTile<M, 3>;                                                                      \
    using Z6 = ColTile<M, 6>;                                                                      \
    using Z7 = ColTile<M, 7>;                                                                      \
    using E4 = FastFFT<M, E, Z4, __VA_ARGS__>;                                                     \
    using E3 = FastFFT<M, E, Z3, __VA_ARGS__>;                                                     \
    using E6 = FastFFT<M, E, Z6, __VA_ARGS__>;                                                     \
    using E7 = FastFFT<M, E, Z7, __VA_ARGS__>;                                                     \
    using E6F = FastFFT<M, EF, Z6, SRK_UNPAREN FR>;                                                \
    t[KK_Z_C2R] = SRK_ENTRY((k_zpass<E4, Z4, ZOP_C2R>), E4, Z4::SIZE * 16);                        \
    t[KK_Z_R2C] = SRK_ENTRY((k_zpass<E4, Z4, ZOP_R2C>), E4, Z4::SIZE * 16);                        \
    t[KK_Z_NS3] = SRK_ENTRY((k_zpass<E6, Z6, ZOP_NS3, E6F>), E6, Z6::SIZE * 16);                   \
    t[KK_Z_NS2] = SRK_ENTRY((k_zpass<E3, Z3, ZOP_NS2>), E3, Z3::SIZE * 16);                        \
    t[KK_Z_B3] = SRK_ENTRY((k_zpass<E7, Z7, ZOP_B3>), E7, Z7::SIZE * 16);                          \
    t[KK_Z_B2] = SRK_ENTRY((k_zpass<E4, Z4, ZOP_B2>), E4, Z4::SIZE * 16);                          \
  }

// Strided passes on the one-butterfly-per-thread engine (radices SR, CS
// columns); z passes on FastFFT<M, E, ...> as in SRK_DEFINE_SIZE_F.
#define SRK_DEFINE_SIZE_1(NAME, M, CS, SR, E, EF, FR, ...)                                         \
  void NAME(KEntry* t) {                                                                           \
    using SL = RowTile<M, CS>;                                                                     \
    using SE = FastFFT1<M, SL, SRK_UNPAREN SR>;                                                    \
    SRK_STRIDED_KINDS(M, CS)                                                                       \
    using Z4 = ColTile<M, 4>;                                                                      \
    using Z3 = ColTile<M, 3>;                                                                      \
    using Z6 = ColTile<M, 6>;                                                                      \
    using Z7 = ColTile<M, 7>;                                                                      \
    using E4 = FastFFT<M, E, Z4, __VA_ARGS__>;                                                     \
    using E3 = FastFFT<M, E, Z3, __VA_ARGS__>;                                                     \
    using E6 = FastFFT<M, E, Z6, __VA_ARGS__>;                                                     \
    using E7 = FastFFT<M, E, Z7, __VA_ARGS__>;                                                     \
    using E6F = FastFFT<M, EF, Z6, SRK_UNPAREN FR>;                                                \
    t[KK_Z_C2R] = SRK_ENTRY((k_zpass<E4, Z4, ZOP_C2R>), E4, Z4::SIZE * 16);                        \
    t[KK_Z_R2C] = SRK_ENTRY((k_zpass<E4, Z4, ZOP_R2C>), E4, Z4::SIZE * 16);                        \
    t[KK_Z_NS3] = SRK_ENTRY((k_zpass<E6, Z6, ZOP_NS3, E6F>), E6, Z6::SIZE * 16);                   \
    t[KK_Z_NS2] = SRK_ENTRY((k_zpass<E3, Z3, ZOP_NS2>), E3, Z3::SIZE * 16);                        \
    t[KK_Z_B3] = SRK_ENTRY((k_zpass<E7, Z7, ZOP_B3>), E7, Z7::SIZE * 16);                          \
    t[KK_Z_B2] = SRK_ENTRY((k_zpass<E4, Z4, ZOP_B2>), E4, Z4::SIZE * 16);                          \
  }

// Separate strided-pass plan (ES elements/thread, CSS columns, radices SR) and
// z-pass plan (E, CS, radices ...).
#define SRK_DEFINE_SIZE_S(NAME, M, ES, CSS, SR, E, ...)                                             \
  void NAME(KEntry* t) {                                                                           \
    using SL = RowTile<M, CSS>;                                                                    \
    using SE = FastFFT<M, ES, SL, SRK_UNPAREN SR>;                                                 \
    SRK_STRIDED_KINDS(M, CSS)                                                                      \
    using Z4 = ColTile<M, 4>;                                                                      \
    using Z3 = ColTile<M, 3>;                                                                      \
    using Z6 = ColTile<M, 6>;                                                                      \
    using Z7 = ColTile<M, 7>;                                                                      \
    using E4 = FastFFT<M, E, Z4, __VA_ARGS__>;                                                     \
    using E3 = FastFFT<M, E, Z3, __VA_ARGS__>;                                                     \
    using E6 = FastFFT<M, E, Z6, __VA_ARGS__>;                                                     \
    using E7 = FastFFT<M, E, Z7, __VA_ARGS__>;                                                     \
    t[KK_Z_C2R] = SRK_ENTRY((k_zpass<E4, Z4, ZOP_C2R>), E4, Z4::SIZE * 16);                        \
    t[KK_Z_R2C] = SRK_ENTRY((k_zpass<E4, Z4, ZOP_R2C>), E4, Z4::SIZE * 16);                        \
    t[KK_Z_NS3] = SRK_ENTRY((k_zpass<E6, Z6, ZOP_NS3>), E6, Z6::SIZE * 16);                        \
    t[KK_Z_NS2] = SRK_ENTRY((k_zpass<E3, Z3, ZOP_NS2>), E3, Z3::SIZE * 16);                        \
    t[KK_Z_B3] = SRK_ENTRY((k_zpass<E7, Z7, ZOP_B3>), E7, Z7::SIZE * 16);                          \
    t[KK_Z_B2] = SRK_ENTRY((k_zpass<E4, Z4, ZOP_B2>), E4, Z4::SIZE * 16);                          \
  }

// Unpadded power-of-two lengths only need the plain kinds.
#define SRK_DEFINE_SIZE_PLAIN(NAME, M, E, CS, ...)                                                 \
  void NAME(KEntry* t) {                                                                           \
    using SL = RowTile<M, CS>;                                                                     \
    using SE = FastFFT<M, E, SL, __VA_ARGS__>;                                                     \
    t[KK_INV] = SRK_ENTRY((k_colpass<SE, PK_INV, +1>), SE, SL::SIZE * 16);                         \
    t[KK_FWD] = SRK_ENTRY((k_colpass<SE, PK_FWD, -1>), SE, SL::SIZE * 16);                         \
    using Z4 = ColTile<M, 4>;                                                                      \
    using E4 = FastFFT<M, E, Z4, __VA_ARGS__>;                                                     \
    t[KK_Z_C2R] = SRK_ENTRY((k_zpass<E4, Z4, ZOP_C2R>), E4, Z4::SIZE * 16);                        \
    t[KK_Z_R2C] = SRK_ENTRY((k_zpass<E4, Z4, ZOP_R2C>), E4, Z4::SIZE * 16);                        \
  }

// NS3 z-pass with the fused middle stage: inverse prefix (IR..., product M/4),
// forward suffix (FR..., product M/4), E = 24.
// Pitch >= 4K so that tile columns 3..5 hold the 12 staged rows of K modes.
// NS3 z-pass, one pencil per CTA (k_zpass_ns3p): inverse prefix (IR..., product
// M/4) on 3 columns with E = 24 (M/8 threads), forward suffix FR... looped.
#define SRK_NS3P(M, IR, FR)                                                                        \
  {                                                                                                \
    using ZL = ColTile<M, 3>;                                                                      \
    using EI = FastFFT<M, 24, ZL, SRK_UNPAREN IR>;                                                 \
    t[KK_Z_NS3] = KEntry{(const void*)(k_zpass_ns3p<M, ZL, EI, ZOP_NS3, SRK_UNPAREN FR>), M / 8, 3,          \
                         (int)(ZL::SIZE * 16) + EI::TWN * 16, 1};                                  \
  }
#define SRK_NS3F(M, IR, EF, FR)                                                                     \
  {                                                                                                \
    using ZL = ColTile<M, 6>;                                                                           \
    using EI = FastFFT<M, 24, ZL, SRK_UNPAREN IR>;                                                 \
    t[KK_Z_NS3] = KEntry{(const void*)(k_zpass_ns3f<M, ZL, EI, EF, SRK_UNPAREN FR>), M / 4, 6,      \
                         (int)(ZL::SIZE * 16) + EI::TWN * 16, 2};                                  \
  }
