// FFT engines for the strided-axis (x, y) and contiguous-axis (z) passes.
//
// A CTA owns a tile of C independent length-M FFT "columns".  Both engines use
// the self-sorting Stockham formulation: at a stage with radix R after a
// cumulative length Ls,
//     j in [0, M/R):  k = j mod Ls
//     v[t] = x[j + t*M/R] * W^{t*k*M/(Ls*R)}            (t = 0..R-1)
//     x'[(j-k)*R + k + q*Ls] = DFT_R(v)[q]              (q = 0..R-1)
// The first stage pulls its inputs straight from the caller's loader (global
// memory, with the 3/2-rule pad applied on the fly) and the last stage pushes
// its outputs straight to the caller's storer (global memory with truncation /
// epilogue), so intermediate data crosses shared memory only between stages.
//
// FastFFT: compile-time plan (radices, E = elements per thread, TPC = M/E
// threads per column); every stage keeps E values per thread in registers and
// works in place on one shared-memory tile (load all -> barrier -> store all).
// GenericFFT: runtime radix list for small odd-factor sizes used by the
// reference's own tests; one thread per column, local-memory ping-pong.
#pragma once

#include <type_traits>

#include "srk_common.cuh"

// ---------------------------------------------------------------------------
// Shared-memory tile layouts.
// RowTile:  [row][col], col fastest.  For C >= 8 any warp access pattern of the
//           engines is bank-conflict free (8 lanes x 16 B cover all 32 banks).
//           Thread map: col = tid % C, tj = tid / C  (global accesses coalesce
//           along the C consecutive columns).
// ColTile:  [col][row] with one 16 B pad every 8 rows.  Thread map:
//           tj = tid % TPC, col = tid / TPC (lanes run along the FFT axis, which
//           is the contiguous z axis in global memory).
// ---------------------------------------------------------------------------
template <int M_, int C_>
struct RowTile {
  static constexpr int M = M_, C = C_;
  // C >= 8: a row spans all 32 banks -> conflict free as is.
  // C == 4: a row is half a bank cycle; one pad row after every 8 rows puts
  // rows 8j+q and 8(j+1)+q in opposite halves, so the stride-R stores of the
  // first Stockham stage and the consecutive-row accesses of later stages
  // both split 4/4 over the halves (conflict free).
  // C == 2 (one 32 B row per 16 B bank pair): the same pad row every 8 rows
  // makes the stride-24 stores of the first Stockham stage (rows 24j + q) and
  // the consecutive-row accesses of later stages conflict free per 8-lane
  // wavefront (tj 0..3 land in slots 0, 6, 4, 2 of 8).
  static constexpr int SIZE = (C_ >= 8) ? M_ * C_ : (M_ + M_ / 8 + 1) * C_;  // in cplx
  // idx(row + 8m) = idx(row) + m*STEP8; within an aligned group of 8 rows
  // idx(row + 1) = idx(row) + ROWSTEP  (lets the stages hoist index math)
  static constexpr int STEP8 = (C_ >= 8) ? 8 * C_ : 9 * C_;
  static constexpr int ROWSTEP = C_;
  __device__ __forceinline__ static int idx(int row, int col) {
    SRK_ASSERT(row >= 0 && row < M_ && col >= 0 && col < C_);
    if constexpr (C_ >= 8) {
      return row * C_ + col;
    } else {
      static_assert(C_ == 4 || C_ == 2, "RowTile supports C = 2, 4 or C >= 8");
      return (row + (row >> 3)) * C_ + col;
    }
  }
  SRK_DEV static int col_of(int tid, int) { return tid % C_; }
  SRK_DEV static int tj_of(int tid, int) { return tid / C_; }
  // idx(base + q, c) - idx(base, c) for base a multiple of 8
  static constexpr int roff(int q) { return C_ >= 8 ? q * C_ : (q + (q >> 3)) * C_; }
};

template <int M_, int C_, int MINPITCH = 0>
struct ColTile {
  static constexpr int M = M_, C = C_;
  static constexpr int PITCH0 = M_ + (M_ + 7) / 8 + 1;
  static constexpr int PITCH = PITCH0 > MINPITCH ? PITCH0 : MINPITCH;
  static constexpr int SIZE = PITCH * C_;
  static constexpr int STEP8 = 9;
  static constexpr int ROWSTEP = 1;
  __device__ __forceinline__ static int idx(int row, int col) {
    SRK_ASSERT(row >= 0 && row < M_ && col >= 0 && col < C_);
    return col * PITCH + row + (row >> 3);
  }
  SRK_DEV static int col_of(int tid, int tpc) { return tid / tpc; }
  SRK_DEV static int tj_of(int tid, int tpc) { return tid % tpc; }
  static constexpr int roff(int q) { return q + (q >> 3); }
};

struct GenPlan {
  int M;
  int nr;
  int r[10];
};

// ---------------------------------------------------------------------------
// Compile-time engine
// ---------------------------------------------------------------------------
// WS: column-private stages (a warp owns whole columns, TPC <= 32): the
// barriers between stages only need to order the warp itself, except the
// first stage's load->store barrier when its input (staging) aliases other
// columns' tile space.
// Shared-memory twiddle table: the first quarter wave exp(-2 pi i r / M),
// r < M/4, stored XOR-swizzled (conflict-free for the power-of-two strides of
// the stage lookups).  w^m = (-i)^(m / (M/4)) * tab[m mod M/4] is exact (the
// quarter-turn rotations only swap / negate), so every twiddle equals the
// correctly rounded full-table value.  Filled once per CTA from the global
// table (twiddles read through L1 missed ~60% under the FFT tiles' smem
// carve-out and were the largest single stall source).
template <int M>
struct TwTab {
  static constexpr int Q = M / 4;
  static constexpr int N = (M % 4 == 0) ? ((Q + 7) / 8) * 8 : 0;
};
SRK_DEV int tw_swz(int r) { return r ^ ((r >> 3) & 7); }
// cp.async (no register round trip): completes with the caller's next
// cp_async_wait_all(), which every fast kernel issues before its first barrier.
template <int M>
__device__ __forceinline__ void tw_fill(cplx* tws, const cplx* __restrict__ tw) {
  for (int i = threadIdx.x; i < TwTab<M>::Q; i += blockDim.x) cp_async16(&tws[tw_swz(i)], &tw[i]);
}
template <int M>
__device__ __forceinline__ cplx tw_get(const cplx* tws, unsigned m) {
  static_assert(M % 4 == 0, "quarter-wave table needs 4 | M");
  constexpr unsigned Q = M / 4;
  const unsigned q = m / Q, r = m - q * Q;
  const cplx w = tws[tw_swz((int)r)];
  const double a = (q & 1u) ? w.y : w.x;
  const double b = (q & 1u) ? -w.x : w.y;
  return (q & 2u) ? make_double2(-a, -b) : make_double2(a, b);
}

// v[t] *= w^t, w = exp(SIGN 2 pi i kts / M), t = 1..R-1: only w^1, w^2, w^4
// (and w^8, w^16) come from the table; w^(8a+b) = w^(8a) * w^b is formed on
// the fly, so at most 10 powers are live (a few extra roundings, ~5e-16
// relative).  Products instead of per-exponent table lookups measured 0.8 ms
// faster per 512^3 RHS.
template <int M, int SIGN>
__device__ __forceinline__ cplx tw_pow(const cplx* tw, unsigned e) {
  cplx w = tw_get<M>(tw, e);
  if (SIGN > 0) w.y = -w.y;
  return w;
}
template <int M, int R, int SIGN>
__device__ __forceinline__ void stage_twiddle(cplx* v, const cplx* tw, unsigned kts) {
  constexpr int B = R < 8 ? R : 8;
  cplx wb[8];
#pragma unroll
  for (int b = 1; b < B; ++b) {
    if ((b & (b - 1)) == 0)
      wb[b] = tw_pow<M, SIGN>(tw, (unsigned)b * kts);
    else
      wb[b] = cmul(wb[b & (b - 1)], wb[b & -b]);
    v[b] = cmul(v[b], wb[b]);
  }
  if constexpr (R > 8) {
    cplx w8 = tw_pow<M, SIGN>(tw, 8u * kts);
    cplx w16 = (R > 16) ? tw_pow<M, SIGN>(tw, 16u * kts) : w8;
#pragma unroll
    for (int a = 1; 8 * a < R; ++a) {
      const cplx wa = a == 1 ? w8 : (a == 2 ? w16 : cmul(w8, w16));
      v[8 * a] = cmul(v[8 * a], wa);
#pragma unroll
      for (int b = 1; b < 8 && 8 * a + b < R; ++b) v[8 * a + b] = cmul(v[8 * a + b], cmul(wa, wb[b]));
    }
  }
  static_assert(R <= 32, "stage_twiddle covers radices up to 32");
}

// Shared-memory-lean twiddles for the z passes, which are bound by the SM's
// shared-memory datapath (128 B/clk, shuffles included -- tools/probe_peaks.py),
// not by the fp64 pipe: one table read (w^1) per butterfly, every other power
// formed in registers (w^2 = (w^1)^2, w^4 = (w^2)^2, w^8, w^16 likewise;
// w^(a+b) = w^a w^b).  A few roundings more than stage_twiddle (~1e-16
// relative per product); the table reads they replace were ~9% of the z-pass's
// shared-memory wavefronts (ncu, v15).
SRK_DEV cplx csq(cplx a) { return make_double2(fma(a.x, a.x, -a.y * a.y), fma(a.x, a.y, a.x * a.y)); }
template <int M, int R, int SIGN>
__device__ __forceinline__ void stage_twiddle_sq(cplx* v, const cplx* tw, unsigned kts) {
  static_assert(R <= 32, "stage_twiddle_sq covers radices up to 32");
  constexpr int B = R < 8 ? R : 8;
  cplx wb[8];
  wb[1] = tw_pow<M, SIGN>(tw, kts);
#pragma unroll
  for (int b = 2; b < B; ++b) wb[b] = ((b & (b - 1)) == 0) ? csq(wb[b / 2]) : cmul(wb[b & (b - 1)], wb[b & -b]);
#pragma unroll
  for (int b = 1; b < B; ++b) v[b] = cmul(v[b], wb[b]);
  if constexpr (R > 8) {
    const cplx w8 = csq(wb[4]);
    const cplx w16 = (R > 16) ? csq(w8) : w8;
#pragma unroll
    for (int a = 1; 8 * a < R; ++a) {
      const cplx wa = a == 1 ? w8 : (a == 2 ? w16 : cmul(w8, w16));
      v[8 * a] = cmul(v[8 * a], wa);
#pragma unroll
      for (int b = 1; b < 8 && 8 * a + b < R; ++b) v[8 * a + b] = cmul(v[8 * a + b], cmul(wa, wb[b]));
    }
  }
}

// First-stage loaders may take the compile-time row range of the 32-lane group
// (rlo, rhi: the rows j + t*STRIDE can reach for any lane): a loader that knows
// which rows are structurally zero (the 3/2-rule zero band of a padded inverse)
// then skips their shared-memory reads at compile time.
template <class T, class = void>
struct ld_has_range : std::false_type {};
template <class T>
struct ld_has_range<T, decltype(void(T::kRange))> : std::true_type {};

// A first-stage loader with a member kColPrivate reads staged inputs that lie inside the
// tile column it transforms: the load -> store hazard of the first stage is then private
// to the warp(s) that own the column, like every later stage.
template <class T, class = void>
struct ld_col_private : std::false_type {};
template <class T>
struct ld_col_private<T, decltype(void(T::kColPrivate))> : std::true_type {};

template <bool WS, int TPC>
__device__ __forceinline__ void stage_sync() {
  if constexpr (WS && TPC <= 32)
    SRK_WBAR();
  else
    SRK_BAR();
}

template <int M, int E, class L, int SIGN, bool LD_SMEM, bool ST_SMEM, int Ls, int R, int... Rest>
struct FastStageW;

template <int M, int E, class L, int SIGN, bool LD_SMEM, bool ST_SMEM, int Ls, int R, int... Rest>
struct FastStage {
  template <class LD, class ST>
  __device__ __forceinline__ static void go(cplx* sm, const cplx* __restrict__ tw, int col, int tj,
                                            bool act, LD& ld, ST& st) {
    constexpr int TPC = M / E;
    constexpr int NB = E / R;
    constexpr int STRIDE = M / R;
    constexpr bool FIRST = (Ls == 1);
    constexpr bool LAST = (sizeof...(Rest) == 0);
    static_assert(E % R == 0, "radix must divide elements-per-thread");
    cplx v[NB][R];
    if (act) {
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        const int j = tj + b * TPC;
        if constexpr (FIRST) {
#pragma unroll
          for (int t = 0; t < R; ++t) v[b][t] = ld(j + t * STRIDE, col);
        } else if constexpr (STRIDE % 8 == 0) {
          const int a0 = L::idx(j, col);
#pragma unroll
          for (int t = 0; t < R; ++t) v[b][t] = sm[a0 + t * (STRIDE / 8) * L::STEP8];
        } else {
#pragma unroll
          for (int t = 0; t < R; ++t) v[b][t] = sm[L::idx(j + t * STRIDE, col)];
        }
      }
    }
    // twiddles + butterflies before the load->store barrier: only the
    // transformed values are live across it
    if (act) {
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        const unsigned j = (unsigned)tj + (unsigned)(b * TPC);
        const unsigned k = j % (unsigned)Ls;
        if constexpr (Ls > 1) {
          constexpr int TS = M / (Ls * R);
          const unsigned kts = k * (unsigned)TS;
          stage_twiddle<M, R, SIGN>(v[b], tw, kts);
        }
        DFT<R, SIGN>::run(v[b]);
      }
    }
    if constexpr ((!FIRST || LD_SMEM) && (!LAST || ST_SMEM)) SRK_BAR();
    if (act) {
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        const unsigned j = (unsigned)tj + (unsigned)(b * TPC);
        const unsigned k = j % (unsigned)Ls;
        const int base = (int)((j - k) * (unsigned)R + k);
        if constexpr (LAST) {
#pragma unroll
          for (int q = 0; q < R; ++q) st(base + q * Ls, col, v[b][q]);
        } else if constexpr (Ls % 8 == 0) {
          const int a0 = L::idx(base, col);
#pragma unroll
          for (int q = 0; q < R; ++q) sm[a0 + q * (Ls / 8) * L::STEP8] = v[b][q];
        } else if constexpr (Ls == 1 && (8 % R == 0)) {
          const int a0 = L::idx(base, col);  // base = j*R: the R rows share one 8-row group
#pragma unroll
          for (int q = 0; q < R; ++q) sm[a0 + q * L::ROWSTEP] = v[b][q];
        } else {
#pragma unroll
          for (int q = 0; q < R; ++q) sm[L::idx(base + q * Ls, col)] = v[b][q];
        }
      }
    }
    if constexpr (!LAST) {
      SRK_BAR();
      FastStage<M, E, L, SIGN, LD_SMEM, ST_SMEM, Ls * R, Rest...>::go(sm, tw, col, tj, act, ld, st);
    }
  }
};

template <int M, int E, class L, int SIGN, bool LD_SMEM, bool ST_SMEM, int Ls, int R, int... Rest>
struct FastStageW {
  template <class LD, class ST>
  __device__ __forceinline__ static void go(cplx* sm, const cplx* __restrict__ tw, int col, int tj,
                                            bool act, LD& ld, ST& st) {
    constexpr int TPC = M / E;
    constexpr int NB = E / R;
    constexpr int STRIDE = M / R;
    constexpr bool FIRST = (Ls == 1);
    constexpr bool LAST = (sizeof...(Rest) == 0);
    static_assert(E % R == 0, "radix must divide elements-per-thread");
    cplx v[NB][R];
    if (act) {
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        const int j = tj + b * TPC;
        if constexpr (FIRST && ld_has_range<LD>::value) {
#pragma unroll
          for (int t = 0; t < R; ++t) v[b][t] = ld(j + t * STRIDE, col, t * STRIDE + b * TPC, t * STRIDE + b * TPC + TPC - 1);
        } else if constexpr (FIRST) {
#pragma unroll
          for (int t = 0; t < R; ++t) v[b][t] = ld(j + t * STRIDE, col);
        } else if constexpr (STRIDE % 8 == 0) {
          const int a0 = L::idx(j, col);
#pragma unroll
          for (int t = 0; t < R; ++t) v[b][t] = sm[a0 + t * (STRIDE / 8) * L::STEP8];
        } else {
#pragma unroll
          for (int t = 0; t < R; ++t) v[b][t] = sm[L::idx(j + t * STRIDE, col)];
        }
      }
    }
    // twiddles + butterflies before the load->store barrier: only the
    // transformed values are live across it
    if (act) {
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        const unsigned j = (unsigned)tj + (unsigned)(b * TPC);
        const unsigned k = j % (unsigned)Ls;
        if constexpr (Ls > 1) {
          constexpr int TS = M / (Ls * R);
          const unsigned kts = k * (unsigned)TS;
          stage_twiddle_sq<M, R, SIGN>(v[b], tw, kts);
        }
        DFT<R, SIGN>::run(v[b]);
      }
    }
    if constexpr ((!FIRST || LD_SMEM) && (!LAST || ST_SMEM)) {
      if constexpr (FIRST && !ld_col_private<LD>::value)
        SRK_BAR();  // staging may alias other columns
      else
        stage_sync<true, TPC>();  // (a loader whose staged inputs lie inside its own tile column)
    }
    if (act) {
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        const unsigned j = (unsigned)tj + (unsigned)(b * TPC);
        const unsigned k = j % (unsigned)Ls;
        const int base = (int)((j - k) * (unsigned)R + k);
        if constexpr (LAST) {
#pragma unroll
          for (int q = 0; q < R; ++q) st(base + q * Ls, col, v[b][q]);
        } else if constexpr (Ls % 8 == 0) {
          const int a0 = L::idx(base, col);
#pragma unroll
          for (int q = 0; q < R; ++q) sm[a0 + q * (Ls / 8) * L::STEP8] = v[b][q];
        } else if constexpr (Ls == 1 && (8 % R == 0)) {
          const int a0 = L::idx(base, col);  // base = j*R: the R rows share one 8-row group
#pragma unroll
          for (int q = 0; q < R; ++q) sm[a0 + q * L::ROWSTEP] = v[b][q];
        } else {
#pragma unroll
          for (int q = 0; q < R; ++q) sm[L::idx(base + q * Ls, col)] = v[b][q];
        }
      }
    }
    if constexpr (!LAST) {
      stage_sync<true, TPC>();
      FastStageW<M, E, L, SIGN, LD_SMEM, ST_SMEM, Ls * R, Rest...>::go(sm, tw, col, tj, act, ld, st);
    }
  }
};

template <int M_, int E_, class L, int... Rs>
struct FastFFT {
  static constexpr int M = M_, E = E_, TPC = M_ / E_;
  static constexpr int C = L::C;
  static constexpr int NT = C * TPC;
  static constexpr bool kFast = true;
  static constexpr int RPROD = (1 * ... * Rs);
  static constexpr int TWN = TwTab<M_>::N;  // shared twiddle table entries (before the tile)
  // RPROD < M: a prefix of a longer plan (the remaining stages are run by the
  // caller, e.g. the fused middle stage of the NS3 z-pass)
  static_assert(M_ % RPROD == 0, "radices must divide M");
  SRK_DEV static int col_of(int tid) { return L::col_of(tid, TPC); }
  // ncols: columns of the tile that carry data (<= C); idle threads still hit barriers.
  template <int SIGN, bool LD_SMEM, bool ST_SMEM, class LD, class ST>
  __device__ __forceinline__ static void run(const GenPlan&, cplx* sm, const cplx* __restrict__ tw,
                                             int ncols, LD& ld, ST& st) {
    const int tid = threadIdx.x;
    const int col = L::col_of(tid, TPC);
    const int tj = L::tj_of(tid, TPC);
    const bool act = (tid < NT) && (col < ncols);
    __builtin_assume(tj >= 0 && tj < TPC);
    FastStage<M_, E_, L, SIGN, LD_SMEM, ST_SMEM, 1, Rs...>::go(sm, tw, col, tj, act, ld, st);
  }
  // column-private variant (ColTile: a warp owns whole columns when TPC <= 32)
  template <int SIGN, bool LD_SMEM, bool ST_SMEM, class LD, class ST>
  __device__ __forceinline__ static void run_ws(const GenPlan&, cplx* sm, const cplx* __restrict__ tw,
                                                int ncols, LD& ld, ST& st) {
    const int tid = threadIdx.x;
    const int col = L::col_of(tid, TPC);
    const int tj = L::tj_of(tid, TPC);
    const bool act = (tid < NT) && (col < ncols);
    __builtin_assume(tj >= 0 && tj < TPC);
    FastStageW<M_, E_, L, SIGN, LD_SMEM, ST_SMEM, 1, Rs...>::go(sm, tw, col, tj, act, ld, st);
  }
};

// ---------------------------------------------------------------------------
// One butterfly per thread per stage: the stage with radix R runs on M/R
// threads per column (the rest idle), so a plan may mix radices that do not
// divide a common per-thread element count -- e.g. 768 = 24 * 32 in two
// stages: one shared-memory round trip instead of two for 8 * 8 * 12.
// ---------------------------------------------------------------------------
template <int M, class L, int SIGN, bool LD_SMEM, bool ST_SMEM, int Ls, int R, int... Rest>
struct OneStage {
  template <class LD, class ST>
  __device__ __forceinline__ static void go(cplx* sm, const cplx* tw, int col, int tj, bool act_col, LD& ld,
                                            ST& st) {
    constexpr int STRIDE = M / R;  // butterflies per column
    constexpr bool FIRST = (Ls == 1);
    constexpr bool LAST = (sizeof...(Rest) == 0);
    const bool act = act_col && tj < STRIDE;
    const int j = tj;
    cplx v[R];
    if (act) {
      if constexpr (FIRST) {
#pragma unroll
        for (int t = 0; t < R; ++t) v[t] = ld(j + t * STRIDE, col);
      } else if constexpr (STRIDE % 8 == 0) {
        const int a0 = L::idx(j, col);
#pragma unroll
        for (int t = 0; t < R; ++t) v[t] = sm[a0 + t * (STRIDE / 8) * L::STEP8];
      } else {
#pragma unroll
        for (int t = 0; t < R; ++t) v[t] = sm[L::idx(j + t * STRIDE, col)];
      }
    }
    const unsigned k = (unsigned)j % (unsigned)Ls;
    if (act) {  // twiddles + butterfly before the load->store barrier
      if constexpr (Ls > 1) stage_twiddle<M, R, SIGN>(v, tw, k * (unsigned)(M / (Ls * R)));
      DFT<R, SIGN>::run(v);
    }
    if constexpr ((!FIRST || LD_SMEM) && (!LAST || ST_SMEM)) SRK_BAR();
    if (act) {
      const int base = (int)(((unsigned)j - k) * (unsigned)R + k);
      if constexpr (LAST) {
#pragma unroll
        for (int q = 0; q < R; ++q) st(base + q * Ls, col, v[q]);
      } else if constexpr (Ls % 8 == 0) {
        const int a0 = L::idx(base, col);
#pragma unroll
        for (int q = 0; q < R; ++q) sm[a0 + q * (Ls / 8) * L::STEP8] = v[q];
      } else if constexpr (Ls == 1 && R % 8 == 0) {
        const int a0 = L::idx(base, col);  // base = j*R, a multiple of 8
#pragma unroll
        for (int q = 0; q < R; ++q) sm[a0 + L::roff(q)] = v[q];
      } else {
#pragma unroll
        for (int q = 0; q < R; ++q) sm[L::idx(base + q * Ls, col)] = v[q];
      }
    }
    if constexpr (!LAST) {
      SRK_BAR();
      OneStage<M, L, SIGN, LD_SMEM, ST_SMEM, Ls * R, Rest...>::go(sm, tw, col, tj, act_col, ld, st);
    }
  }
};

// Stages after a caller-run prefix (Ls > 1), one butterfly per thread with the
// thread -> (column, butterfly) map redone per stage, so every stage spreads
// its ncols * M/R butterflies over the whole CTA (NS3 z-pass forward suffix:
// 3 columns on M/4 threads).  Requires ncols * M/R <= blockDim.x.
template <int M, class L, int SIGN, int Ls, int R, int... Rest>
struct OneStageZ {
  template <class ST>
  __device__ __forceinline__ static void go(cplx* sm, const cplx* tw, int ncols, ST& st) {
    constexpr int STRIDE = M / R;
    constexpr bool LAST = (sizeof...(Rest) == 0);
    const int tid = threadIdx.x;
    const int col = tid / STRIDE, j = tid - col * STRIDE;
    const bool act = col < ncols;
    cplx v[R];
    if (act) {
      if constexpr (STRIDE % 8 == 0) {
        const int a0 = L::idx(j, col);
#pragma unroll
        for (int t = 0; t < R; ++t) v[t] = sm[a0 + t * (STRIDE / 8) * L::STEP8];
      } else {
#pragma unroll
        for (int t = 0; t < R; ++t) v[t] = sm[L::idx(j + t * STRIDE, col)];
      }
    }
    const unsigned k = (unsigned)j % (unsigned)Ls;
    if (act) {
      stage_twiddle_sq<M, R, SIGN>(v, tw, k * (unsigned)(M / (Ls * R)));
      DFT<R, SIGN>::run(v);
    }
    SRK_BAR();
    if (act) {
      const int base = (int)(((unsigned)j - k) * (unsigned)R + k);
      if constexpr (LAST) {
#pragma unroll
        for (int q = 0; q < R; ++q) st(base + q * Ls, col, v[q]);
      } else if constexpr (Ls % 8 == 0) {
        const int a0 = L::idx(base, col);
#pragma unroll
        for (int q = 0; q < R; ++q) sm[a0 + q * (Ls / 8) * L::STEP8] = v[q];
      } else {
#pragma unroll
        for (int q = 0; q < R; ++q) sm[L::idx(base + q * Ls, col)] = v[q];
      }
    }
    if constexpr (!LAST) {
      SRK_BAR();
      OneStageZ<M, L, SIGN, Ls * R, Rest...>::go(sm, tw, ncols, st);
    }
  }
};

template <int A, int... Bs>
constexpr int cmin() {
  if constexpr (sizeof...(Bs) == 0)
    return A;
  else
    return A < cmin<Bs...>() ? A : cmin<Bs...>();
}

template <int M_, class L, int... Rs>
struct FastFFT1 {
  static constexpr int M = M_;
  static constexpr int TPC = M_ / cmin<Rs...>();
  static constexpr int C = L::C;
  static constexpr int NT = C * TPC;
  static constexpr bool kFast = true;
  static constexpr int TWN = TwTab<M_>::N;
  static_assert((1 * ... * Rs) == M_, "radices must multiply to M");
  SRK_DEV static int col_of(int tid) { return L::col_of(tid, TPC); }
  template <int SIGN, bool LD_SMEM, bool ST_SMEM, class LD, class ST>
  __device__ __forceinline__ static void run(const GenPlan&, cplx* sm, const cplx* __restrict__ tw, int ncols,
                                             LD& ld, ST& st) {
    const int tid = threadIdx.x;
    const int col = L::col_of(tid, TPC);
    const int tj = L::tj_of(tid, TPC);
    const bool act = (tid < NT) && (col < ncols);
    __builtin_assume(tj >= 0 && tj < TPC);
    OneStage<M_, L, SIGN, LD_SMEM, ST_SMEM, 1, Rs...>::go(sm, tw, col, tj, act, ld, st);
  }
};

// ---------------------------------------------------------------------------
// Runtime engine (one thread per column, radices in {2,3,4,5,7,8})
// ---------------------------------------------------------------------------
#define SRK_GEN_MAXM 96
#define SRK_GEN_MAXR 8


template <int SIGN>
__device__ __forceinline__ void gen_dft(int R, cplx* v) {
  switch (R) {
    case 2: DFT<2, SIGN>::run(v); break;
    case 3: DFT<3, SIGN>::run(v); break;
    case 4: DFT<4, SIGN>::run(v); break;
    case 5: DFT<5, SIGN>::run(v); break;
    case 7: DFT<7, SIGN>::run(v); break;
    case 8: DFT<8, SIGN>::run(v); break;
    default: break;
  }
}

template <class L>
struct GenericFFT {
  static constexpr bool kFast = false;
  static constexpr int TWN = 0;
  static constexpr int M = 0;  // runtime
  static constexpr int C = L::C;
  static constexpr int NT = L::C;
  SRK_DEV static int col_of(int tid) { return tid; }
  template <int SIGN, bool LD_SMEM, bool ST_SMEM, class LD, class ST>
  __device__ static void run(const GenPlan& p, cplx*, const cplx* __restrict__ tw, int ncols, LD& ld, ST& st) {
    const int col = threadIdx.x;
    if (col >= ncols || col >= C) return;
    const int M = p.M;
    cplx a[SRK_GEN_MAXM], b[SRK_GEN_MAXM];
    for (int r = 0; r < M; ++r) a[r] = ld(r, col);
    cplx* x = a;
    cplx* y = b;
    int Ls = 1;
    for (int s = 0; s < p.nr; ++s) {
      const int R = p.r[s];
      const int stride = M / R;
      const int ts = M / (Ls * R);
      for (int j = 0; j < stride; ++j) {
        const int k = j % Ls;
        cplx v[SRK_GEN_MAXR];
        for (int t = 0; t < R; ++t) {
          cplx z = x[j + t * stride];
          if (t > 0 && k > 0) {
            cplx w = tw[t * k * ts];
            if (SIGN > 0) w.y = -w.y;
            z = cmul(z, w);
          }
          v[t] = z;
        }
        gen_dft<SIGN>(R, v);
        const int base = (j - k) * R + k;
        for (int q = 0; q < R; ++q) y[base + q * Ls] = v[q];
      }
      cplx* tmp = x;
      x = y;
      y = tmp;
      Ls *= R;
    }
    for (int r = 0; r < M; ++r) st(r, col, x[r]);
  }
};
