// Axis-pass kernels of the dealiased pseudo-spectral RHS (templates; instantiated
// per FFT length in inst_*.cu).  Data layout in HBM everywhere: component-major,
// C-order, complex128, last (z) axis contiguous -- the reference's rfftn layout
// (grid.py:11-18).  Kernel map:
//
//   K1 k_colpass<INV_RHS>  : curl on load + x zero-pad + inverse C2C along x
//                            (spectral.py:47-65 curl, :229-258 widen x-pass)
//   K2 k_colpass<INV>      : y zero-pad + inverse C2C along y (:249-258)
//   K3 k_zpass<NS*/B*>     : per z-pencil C2R (:259-261), u x w / rho u in
//                            registers (physics.py:62-82,151-158), R2C (:275)
//   K4 k_colpass<FWD>      : forward C2C along y + truncation (:276-291)
//   K5 k_colpass<FWD>      : forward C2C along x + truncation + 1/1.5^d,
//                            Nyquist / self-conjugate zeroing (:292-303)
//   K6 k_project           : Leray projection + viscous term, Boussinesq
//                            buoyancy / density tendency (physics.py:119-129,
//                            :163-184)   [rhs_kernels.cu]
#pragma once

#include "fft_engine.cuh"

#define SRK_MAX_PEERS 8

enum PassKind {
  PK_INV = 0,      // plain padded / unpadded inverse
  PK_INV_RHS = 1,  // x inverse with the full curl on load (2D K1)
  PK_FWD = 2,      // forward + truncation
  PK_INV_KX = 3,   // 3D K1: x inverse of [u0, u1, u2, kx u1, kx u2, (rho)]
  PK_INV_CURLY = 4 // 3D K2: y inverse of [u, w, (rho)], w = i k x u formed on load from the K1 signals
};
enum ZOp { ZOP_C2R = 0, ZOP_R2C = 1, ZOP_NS3 = 2, ZOP_NS2 = 3, ZOP_B3 = 4, ZOP_B2 = 5 };

// Strided-axis pass.  Global column g within a plane (plane = signal for the
// x pass, (signal, x) for the y pass); element (plane, row, w) lives at
//   plane * plane_stride + row * row_stride + w.
struct PassArgs {
  const cplx* in;
  cplx* out;
  const cplx* tw;
  GenPlan gp;
  int M;          // FFT length on this axis
  int n;          // coarse length on this axis (pad / truncate maps)
  int planes;     // number of planes
  int Qp;         // columns per plane
  int tpp;        // column tiles per plane
  int sig_minor;  // 1: plane index varies fastest over blocks (L2 reuse of curl reads)
  long long row_stride;
  long long in_plane_stride;
  long long out_plane_stride;
  double scale;
  int zero_nyq;      // FWD: zero the Nyquist row (narrow)
  int zero_dc_imag;  // FWD (x pass of narrow): Im of (0,0,0) -> 0
  // INV_RHS (x pass with curl): planes = signals [u(d), w(wc), rho?]
  int dims;
  int n1;  // 3D: coarse y extent (columns are w = y*K + kz); 2D: 1
  int K;   // r2c extent n_last/2+1
  double ck0, ck1, ck2;  // 2*pi/L per axis (x, y, z) -- 2D uses ck0, ck2
  long long comp_stride;  // between state components
  // slab decomposition: rows are grouped in blocks of *_rpb rows
  // that sit *_bstride elements apart (all-to-all send / receive layouts);
  // rpb == 0 means plain rows.  y0 / n1g: global y of the slab's first row and
  // the global y extent (wavenumber labels in the curl).
  int in_rpb, out_rpb;
  unsigned in_magic, out_magic;  // ceil(2^32 / rpb) of the row blocks (row_blk; set by launch_col)
  long long in_bstride, out_bstride;
  int y0, n1g;
  int xplanes;  // PK_INV_CURLY: x planes per signal (m0, or m0/P on a slab)
  int xblk;     // PK_INV_CURLY: x planes per block (divides xplanes)
  // fused K5+K6 (k_xfwd_proj)
  const cplx* y;   // state (velocity, density) of this (slab)
  cplx* f;         // tendency out
  int density;
  double nu, ri, re_pr;
  int nsig;     // PK_INV_CURLY: output signals; block planes run signal-fastest
                // (p = x*nsig + s) so the 6 signals of one x share L2-resident inputs
  unsigned long long* dbg;  // optional phase timestamps (tools/phase_timing.py)
  int tma;       // 1: stage the input tile with 3D TMA copies (tensor map = kernel parameter)
  int tma_rows;  // rows per TMA box (divides the staged row count)
  int tma_out;   // 1: inverse passes write their output tile with 3D TMA stores
  int tmo_rows;  // rows per output box (divides M)
  int probe;     // measurement only (SRK_PROBE_INV / SRK_PROBE_FWD, tools/pass_probe.sh): the pass stages
                 // its tile and returns (1), also stores in the output pattern (2), or (K2) only stores (5)
  // Column groups (kz chunks of the pipelined slab RHS): the Qp columns of a
  // plane are ngrp groups of kc columns; group g, local column c sits at
  // memory column g*in_kst + in_k0 + c of the input (out_* for the output),
  // global kz = kz0 + c.  Unchunked passes: ngrp = 1, kc = Qp, offsets 0
  // (normalised by the host).  tpg = tiles per group, tpp = ngrp * tpg.
  int kc, ngrp, tpg, in_k0, out_k0, kz0;
  long long in_kst, out_kst;
  // kc_out > kc (y passes over pitch-padded rows): the pass also stores the pad columns
  // up to kc_out (zeros: their input is the TMA's out-of-bounds fill), so that a row's
  // last 32 B sector is written whole.
  int kc_out;
  long long in_rs, out_rs;  // row strides of input / output (0 -> row_stride)
  // PF_PEER (slab all-to-all fused into the pass): output row block b goes to
  // peer[b] (rank b's receive buffer at this rank's source block, UVA / CUDA IPC
  // pointer) instead of out + b * out_bstride
  cplx* peer[SRK_MAX_PEERS];
};

// Phase timestamps of every 97th CTA (diagnostics only; dbg == nullptr in
// production launches, so the branch is uniform and never taken).
#define SRK_TS_INIT(ptr, nts)                                                          \
  unsigned long long* dbg_ =                                                           \
      ((ptr) && (blockIdx.x % 97 == 0) && threadIdx.x == 0) ? (ptr) + (blockIdx.x / 97) * (nts) : nullptr;
#define SRK_TS(i)          \
  if (dbg_) {              \
    dbg_[i] = clock64();   \
  }

// magic = ceil(2^32 / rpb) (0 for rpb == 1): row / rpb = (row * magic) >> 32, exact for
// row * rpb < 2^32 -- one multiply instead of a division per access (launch_col sets it)
SRK_DEV int row_blk(int row, unsigned magic) {
  return magic ? (int)(((unsigned long long)(unsigned)row * magic) >> 32) : row;
}
SRK_DEV unsigned row_off(int row, unsigned rs, int rpb, long long bstride, unsigned magic) {
  if (rpb <= 0) return (unsigned)row * rs;
  const int blk = row_blk(row, magic);
  return (unsigned)blk * (unsigned)bstride + (unsigned)(row - blk * rpb) * rs;
}

// Fast path: the input rows of the tile are first copied to shared memory with
// cp.async (16 B per request, no register staging, all requests in flight at
// once); the engine's first stage then reads them from smem.  The staging
// area aliases the FFT tile (the first stage loads everything before its
// first barrier-protected store).  Loaders are branch-free (selects, clamped
// addresses).  Generic path: loaders read global memory directly.
template <int C>
__device__ __forceinline__ void stage_rows(cplx* dst, const cplx* __restrict__ src, int rows, unsigned rs,
                                           int ncols, int rpb, long long bstride, unsigned magic) {
  const int tot = rows * C;
  for (int i = threadIdx.x; i < tot; i += blockDim.x) {
    const int r = i / C, c = i - (i / C) * C;
    if (c < ncols) cp_async16(dst + i, src + row_off(r, rs, rpb, bstride, magic) + (unsigned)c);
    else dst[i] = cmk(0.0, 0.0);  // pad / out-of-range columns (the TMA path zero-fills them too)
  }
}

// FL bits: PF_CTN -- padded pass with n = 2M/3 known at compile time (lets the
// pad / truncate maps resolve statically); PF_BIN / PF_BOUT -- blocked input /
// output rows (slab all-to-all layouts).
// PF_PEER -- with PF_BOUT: output row blocks go straight to the peers' receive
// buffers (PassArgs::peer), the exchange rides on the pass's own stores.
enum PassFlags { PF_CTN = 1, PF_BIN = 2, PF_BOUT = 4, PF_PEER = 8 };

// Block -> (plane, column group, first local column) of a strided pass.
template <int KIND, int C>
SRK_DEV void tile_of(const PassArgs& a, int bid, int& plane, int& g, int& wl) {
  int wt;
  if (a.sig_minor) {
    plane = bid % a.planes;
    wt = bid / a.planes;
  } else {
    plane = bid / a.tpp;
    wt = bid % a.tpp;
  }
  g = wt / a.tpg;
  wl = (wt - g * a.tpg) * C;
  if constexpr (KIND == PK_INV_CURLY) {
    // blocks of XB x-planes, signal-major inside a block: the 5 input planes of
    // XB x values stay L2-resident while the 6 signals read them
    const int XB = a.xblk;
    const int span = a.nsig * XB;
    const int xb = plane / span, r = plane - xb * span;
    const int s_ = r / XB, x_ = xb * XB + (r - (r / XB) * XB);
    plane = s_ * a.xplanes + x_;
  }
}

// TMA staging of a strided tile: rows [0, rows) x local columns [wl, wl + C) of one or
// two source planes into the dense [row][C] staging layout (second plane at
// +n*C), by one elected thread in rows/box 3D tensor copies.  Columns past the
// plane end are zero-filled by the TMA bounds check.
template <int C>
__device__ __forceinline__ void tma_stage(cplx* sm, const CUtensorMap* tm, int wl, int g, int rows, int box,
                                          int rpb, int plA, int plB, int boff, unsigned long long* bar) {
  if (threadIdx.x == 0) {
    const int nb = rows / box;
    const unsigned bytes = (unsigned)(nb * box * C * 16) * (plB >= 0 ? 2u : 1u);
    mbar_expect_tx(bar, bytes);
    // rows are (row in block, block) -- blocked slab receive layouts; plain rows
    // are one block of `rows`
    // a box is part of one row block or a run of whole blocks
    if (rpb < 0) {  // blocked rows of an unchunked pass: 4D map {columns, row in block, block, plane}
      const int rb = -rpb;
      for (int b = 0; b < nb; ++b) {
        const int r0 = b * box, blk = r0 / rb;
        tma_load_4d(sm + b * box * C, tm, 2 * wl, r0 - blk * rb, blk, plA, bar);
        if (plB >= 0) tma_load_4d(sm + boff + b * box * C, tm, 2 * wl, r0 - blk * rb, blk, plB, bar);
      }
    } else if (rpb > 0) {  // 5D map {columns, column group, row in block, block, plane}
      for (int b = 0; b < nb; ++b) {
        const int r0 = b * box, blk = r0 / rpb;
        tma_load_5d(sm + b * box * C, tm, 2 * wl, g, r0 - blk * rpb, blk, plA, bar);
        if (plB >= 0) tma_load_5d(sm + boff + b * box * C, tm, 2 * wl, g, r0 - blk * rpb, blk, plB, bar);
      }
    } else {  // 4D map
      for (int b = 0; b < nb; ++b) {
        tma_load_4d(sm + b * box * C, tm, 2 * wl, g, b * box, plA, bar);
        if (plB >= 0) tma_load_4d(sm + boff + b * box * C, tm, 2 * wl, g, b * box, plB, bar);
      }
    }
  }
  cp_async_wait_all();  // this thread's twiddle-table copies
  mbar_wait(bar, 0);
  SRK_BAR();
}

template <class Eng, int KIND, int SIGN, int FL = 0>
__global__ void __launch_bounds__(Eng::NT, (Eng::NT <= 64 ? 6 : (Eng::NT <= 128 ? 3 : (Eng::NT <= 384 ? 2 : 1)))) k_colpass(const PassArgs a, const __grid_constant__ CUtensorMap tm,
                                                                  const __grid_constant__ CUtensorMap tmo) {
  extern __shared__ __align__(128) cplx smraw[];
  pdl_launch_dependents();
  srk_poison_smem(smraw);
  cplx* const sm = smraw + Eng::TWN;
  const cplx* const twp = Eng::kFast ? smraw : a.tw;
  if constexpr (Eng::kFast) tw_fill<Eng::M>(smraw, a.tw);  // ordered by the staging barrier
  constexpr int C = Eng::C;
  constexpr bool CTN = (FL & PF_CTN) && Eng::kFast;
  SRK_TS_INIT(a.dbg, 3)
  SRK_TS(0)
  const int bid = blockIdx.x;
  int plane, g, wl;
  tile_of<KIND, C>(a, bid, plane, g, wl);
  const int ncols_in = min(C, a.kc - wl);  // data columns of the tile
  const int ncols = a.kc_out > a.kc ? min(C, a.kc_out - wl) : ncols_in;  // + pad columns stored
  const long long w_in = (long long)g * a.in_kst + a.in_k0 + wl;    // memory column of the tile
  const long long w_out = (long long)g * a.out_kst + a.out_k0 + wl;
  const unsigned rs = (unsigned)a.in_rs;    // intra-plane offsets fit in 32 bits
  const unsigned rso = (unsigned)a.out_rs;
  const cplx* __restrict__ inp = a.in + plane * a.in_plane_stride + w_in;
  cplx* __restrict__ outp = a.out + plane * a.out_plane_stride + w_out;
  // output element (row, col): rows in blocks of out_rpb; PF_PEER sends block b to
  // peer b (one shared-memory table lookup per store instead of a dynamically
  // indexed kernel parameter)
  __shared__ cplx* s_peer[(FL & PF_PEER) ? SRK_MAX_PEERS : 1];
  if constexpr ((FL & PF_PEER) != 0) {
    if (threadIdx.x < SRK_MAX_PEERS) {
      cplx* q = a.peer[0];
#pragma unroll
      for (int i = 1; i < SRK_MAX_PEERS; ++i)
        if ((int)threadIdx.x == i) q = a.peer[i];
      s_peer[threadIdx.x] = q ? q + plane * a.out_plane_stride + w_out : nullptr;
    }
    SRK_BAR();
  }
  const unsigned rso_ = (unsigned)a.out_rs;
  const int orpb_ = (FL & PF_BOUT) ? a.out_rpb : 0;
  auto oel = [&](int row, int col) -> cplx& {
    if constexpr ((FL & PF_PEER) != 0) {
      const int blk = row_blk(row, a.out_magic);
      return s_peer[blk][(unsigned)(row - blk * orpb_) * rso_ + (unsigned)col];
    } else {
      return outp[row_off(row, rso_, orpb_, a.out_bstride, a.out_magic) + (unsigned)col];
    }
  };
  const int M = CTN ? Eng::M : a.M;
  const int n = CTN ? 2 * Eng::M / 3 : a.n;
  const int in_rpb = (FL & PF_BIN) ? a.in_rpb : 0;
  const int out_rpb = (FL & PF_BOUT) ? a.out_rpb : 0;
  // TMA staging: plain (unblocked) input rows of the fast engines
  constexpr bool kTMA = Eng::kFast && KIND != PK_INV_RHS;
  // > 0: blocked input rows (5D TMA map); < 0: blocked rows, one column group (4D map)
  const int trpb = (in_rpb > 0 && a.tma == 2) ? -in_rpb : in_rpb;
  __shared__ __align__(8) unsigned long long tbar;
  const bool use_tma = kTMA && a.tma;
  // TMA output: the last stage writes a dense [M][C] tile in smem (over the
  // FFT tile, after the stage's load barrier), then one thread stores it
  // (K2 only: measured 5.48 -> 5.30 ms at 512^3; the x-pass K1, whose output
  // rows are 2 MB apart, was slower with TMA stores, 2.98 -> 3.43 ms)
  constexpr bool kTMAO = Eng::kFast && !(FL & PF_BOUT) && KIND == PK_INV_CURLY;
  const bool use_tmo = kTMAO && a.tma_out;
  auto flush_out = [&]() {
    if (use_tmo) {
      fence_proxy_async_smem();
      SRK_BAR();
      if (threadIdx.x == 0) {
        for (int b = 0; b < M / a.tmo_rows; ++b)
          tma_store_4d(&tmo, sm + b * a.tmo_rows * C, 2 * wl, g, b * a.tmo_rows, plane);
        bulk_commit_and_wait_read();
      }
    }
  };
  if (use_tma) {
    if (threadIdx.x == 0) {
      mbar_init(&tbar, 1);
      fence_mbar_init();
    }
    SRK_BAR();
  }
  pdl_wait();  // the previous kernel's output is complete and visible from here on

  if constexpr (KIND == PK_INV) {
    const double sc = a.scale;
    if (use_tma) {
      tma_stage<C>(sm, &tm, wl, g, n, a.tma_rows, trpb, plane, -1, 0, &tbar);
      SRK_TS(1)
    } else if constexpr (Eng::kFast) {
      stage_rows<C>(sm, inp, n, rs, ncols_in, in_rpb, a.in_bstride, a.in_magic);
      cp_async_wait_all();
      SRK_BAR();
      SRK_TS(1)
    }
    auto ld = [&](int row, int col) -> cplx {
      const int cr = pad_src(row, n, M);
      const bool ok = cr >= 0;
      const int r = ok ? cr : 0;
      cplx v = Eng::kFast ? sm[r * C + col] : inp[row_off(r, rs, in_rpb, a.in_bstride, a.in_magic) + (unsigned)col];
      const double f = ok ? sc : 0.0;
      return cmk(v.x * f, v.y * f);
    };
    auto st = [&](int row, int col, cplx v) {
      if (use_tmo)
        sm[row * C + col] = v;
      else
        oel(row, col) = v;
    };
    Eng::template run<SIGN, Eng::kFast, kTMAO>(a.gp, sm, twp, ncols, ld, st);
    flush_out();
  } else if constexpr (KIND == PK_INV_RHS) {
    // plane = signal s: [u_0..u_{d-1}, w (3 comps in 3D, 1 in 2D), rho]
    const int d = a.dims;
    const int wc = (d == 3) ? 3 : 1;
    const int s = plane;
    const cplx* __restrict__ base = a.in + w_in;  // component 0 (2D: unchunked)
    // per-thread column constants (the column of a thread never changes)
    const int mycol = Eng::col_of(threadIdx.x);
    const int q = wl + mycol;
    double ky = 0.0, kz = 0.0;
    if (d == 3) {
      const int y = q / a.K, kzi = q - y * a.K;
      ky = mode_full(a.y0 + y, a.n1g) * a.ck1;
      kz = (double)kzi * a.ck2;
    } else {
      kz = (double)q * a.ck2;
    }
    // w = i (fa * u_ca - fb * u_cb), fa/fb = kx (row dependent) where flagged.
    int ca = s, cb = s;
    double sa = 1.0, sb = 0.0;
    int kxa = 0, kxb = 0;
    const bool is_curl = (s >= d && s < d + wc);
    if (is_curl) {
      if (d == 3) {
        if (s == 3) { ca = 2; sa = ky; cb = 1; sb = kz; }
        else if (s == 4) { ca = 0; sa = kz; cb = 2; kxb = 1; }
        else { ca = 1; kxa = 1; cb = 0; sb = ky; }
      } else {
        ca = 1; kxa = 1; cb = 0; sb = kz;
      }
    } else if (s == d + wc) {
      ca = cb = d;  // density
    }
    const cplx* __restrict__ pa = base + ca * a.comp_stride;
    const cplx* __restrict__ pb = base + cb * a.comp_stride;
    const double sc = a.scale;
    cplx* sb_ = sm + (is_curl ? n * C : 0);
    if constexpr (Eng::kFast) {
      stage_rows<C>(sm, pa, n, rs, ncols_in, in_rpb, a.in_bstride, a.in_magic);
      if (is_curl) stage_rows<C>(sm + n * C, pb, n, rs, ncols_in, in_rpb, a.in_bstride, a.in_magic);
      cp_async_wait_all();
      SRK_BAR();
      SRK_TS(1)
    }
    auto ld = [&](int row, int col) -> cplx {
      const int cr = pad_src(row, n, M);
      const bool ok = cr >= 0;
      const int r = ok ? cr : 0;
      const unsigned off = row_off(r, rs, in_rpb, a.in_bstride, a.in_magic) + (unsigned)col;
      const cplx ua = Eng::kFast ? sm[r * C + col] : pa[off];
      const cplx ub = Eng::kFast ? sb_[r * C + col] : pb[off];
      // spectral.py:47-65: w = i k x u (k_a = mode_a * 2pi/L_a, grid.py:75-93)
      const double kx = mode_full(r, n) * a.ck0;
      const double fa = kxa ? kx : sa, fb = kxb ? kx : sb;
      const cplx df = csub(cscale(ua, fa), cscale(ub, fb));
      cplx v = is_curl ? cmk(-df.y, df.x) : ua;
      const double f = ok ? sc : 0.0;
      return cmk(v.x * f, v.y * f);
    };
    auto st = [&](int row, int col, cplx v) { oel(row, col) = v; };
    Eng::template run<SIGN, Eng::kFast, false>(a.gp, sm, twp, ncols, ld, st);
  } else if constexpr (KIND == PK_INV_KX) {
    // 3D K1.  k_y and k_z are constant along x, so the x inverse commutes with
    // them: only k_x u1 and k_x u2 need their own transforms; the curl is
    // completed in K2 (PK_INV_CURLY).  plane = signal s of
    // [u0, u1, u2, kx*u1, kx*u2, rho]; one component staged per CTA.
    const int s = plane;
    const int comp = (s < 3) ? s : (s == 3 ? 1 : (s == 4 ? 2 : 3));
    const bool use_kx = (s == 3 || s == 4);
    const cplx* __restrict__ pa = a.in + w_in + comp * a.comp_stride;
    const double sc = a.scale;
    if (use_tma) {  // host guarantees comp_stride == in_plane_stride
      tma_stage<C>(sm, &tm, wl, g, n, a.tma_rows, trpb, comp, -1, 0, &tbar);
      SRK_TS(1)
      if (a.probe) {  // access-pattern ceiling (see PK_FWD)
        if (a.probe == 2)
          for (int r = threadIdx.x / C; r < M; r += Eng::NT / C)
            if ((int)(threadIdx.x % C) < ncols) oel(r, threadIdx.x % C) = cmk(0.0, 0.0);
        return;
      }
    } else if constexpr (Eng::kFast) {
      stage_rows<C>(sm, pa, n, rs, ncols_in, in_rpb, a.in_bstride, a.in_magic);
      cp_async_wait_all();
      SRK_BAR();
      SRK_TS(1)
    }
    auto ld = [&](int row, int col) -> cplx {
      const int cr = pad_src(row, n, M);
      const bool ok = cr >= 0;
      const int r = ok ? cr : 0;
      const cplx u = Eng::kFast ? sm[r * C + col] : pa[row_off(r, rs, in_rpb, a.in_bstride, a.in_magic) + (unsigned)col];
      const double kx = mode_full(r, n) * a.ck0;
      const double f = ok ? (use_kx ? kx * sc : sc) : 0.0;
      return cmk(u.x * f, u.y * f);
    };
    auto st = [&](int row, int col, cplx v) {
      if (use_tmo)
        sm[row * C + col] = v;
      else
        oel(row, col) = v;
    };
    Eng::template run<SIGN, Eng::kFast, kTMAO>(a.gp, sm, twp, ncols, ld, st);
    flush_out();
  } else if constexpr (KIND == PK_INV_CURLY) {
    // 3D K2.  plane = (s, x), s over [u0, u1, u2, w0, w1, w2, (rho)]; the input
    // planes are the K1 signals [U0, U1, U2, X1 = F(kx u1), X2 = F(kx u2), R]:
    //   w0 = i (ky U2 - kz U1),  w1 = i (kz U0 - X2),  w2 = i (X1 - ky U0)
    // (spectral.py:47-65 after the x transform; ky varies along this pass's
    // rows, kz along its columns).
    const int X = a.xplanes;
    const int s = plane / X, x = plane - (plane / X) * X;
    int ca = s, cb = s, fa_ky = 0, fa_kz = 0, fb_ky = 0, fb_kz = 0;
    bool is_curl = false;
    if (s == 3) { ca = 2; fa_ky = 1; cb = 1; fb_kz = 1; is_curl = true; }
    else if (s == 4) { ca = 0; fa_kz = 1; cb = 4; is_curl = true; }
    else if (s == 5) { ca = 3; cb = 0; fb_ky = 1; is_curl = true; }
    else if (s == 6) { ca = cb = 5; }
    const cplx* __restrict__ pa = a.in + (long long)(ca * X + x) * a.in_plane_stride + w_in;
    const cplx* __restrict__ pb = a.in + (long long)(cb * X + x) * a.in_plane_stride + w_in;
    const int mycol = Eng::col_of(threadIdx.x);
    const double kz = (double)(a.kz0 + wl + mycol) * a.ck2;  // global kz of the column
    cplx* sb_ = sm + (is_curl ? n * C : 0);
    if (use_tma) {
      if (a.probe == 5)  // probe: stores only
        SRK_BAR();
      else
        tma_stage<C>(sm, &tm, wl, g, n, a.tma_rows, trpb, ca * X + x, is_curl ? cb * X + x : -1, n * C, &tbar);
      SRK_TS(1)
      if (a.probe) {  // access-pattern ceiling (see PK_FWD): the staged rows go out as they are
        if (a.probe == 2 || a.probe == 5) {
          if (use_tmo) flush_out();
          else
            for (int r = threadIdx.x / C; r < M; r += Eng::NT / C)
              if ((int)(threadIdx.x % C) < ncols) oel(r, threadIdx.x % C) = cmk(0.0, 0.0);
        }
        return;
      }
    } else if constexpr (Eng::kFast) {
      stage_rows<C>(sm, pa, n, rs, ncols_in, in_rpb, a.in_bstride, a.in_magic);
      if (is_curl) stage_rows<C>(sm + n * C, pb, n, rs, ncols_in, in_rpb, a.in_bstride, a.in_magic);
      cp_async_wait_all();
      SRK_BAR();
      SRK_TS(1)
    }
    auto ld = [&](int row, int col) -> cplx {
      const int cr = pad_src(row, n, M);
      const bool ok = cr >= 0;
      const int r = ok ? cr : 0;
      const unsigned off = row_off(r, rs, in_rpb, a.in_bstride, a.in_magic) + (unsigned)col;
      const cplx A = Eng::kFast ? sm[r * C + col] : pa[off];
      const cplx B = Eng::kFast ? sb_[r * C + col] : pb[off];
      const double ky = mode_full(r, n) * a.ck1;
      const double fa = fa_ky ? ky : (fa_kz ? kz : 1.0);
      const double fb = fb_ky ? ky : (fb_kz ? kz : 1.0);
      const cplx df = csub(cscale(A, fa), cscale(B, fb));
      cplx v = is_curl ? cmk(-df.y, df.x) : A;
      return ok ? v : cmk(0.0, 0.0);
    };
    auto st = [&](int row, int col, cplx v) {
      if (use_tmo)
        sm[row * C + col] = v;
      else
        oel(row, col) = v;
    };
    Eng::template run<SIGN, Eng::kFast, kTMAO>(a.gp, sm, twp, ncols, ld, st);
    flush_out();
  } else {  // PK_FWD: forward C2C + truncation (+ scale, Nyquist / DC-imag zeroing)
    const bool zn = a.zero_nyq != 0;
    const bool zdc = (a.zero_dc_imag != 0) && (g == 0) && (a.kz0 + wl == 0) && (a.y0 == 0);
    const double sc = a.scale;
    if (use_tma) {
      tma_stage<C>(sm, &tm, wl, g, M, a.tma_rows, trpb, plane, -1, 0, &tbar);
      SRK_TS(1)
      if (a.probe) {  // access-pattern ceiling of the pass (no transform): not a compute path
        if (a.probe == 2)
          for (int r = threadIdx.x / C; r < n; r += Eng::NT / C)
            if ((int)(threadIdx.x % C) < ncols) oel(r, threadIdx.x % C) = cmk(0.0, 0.0);
        return;
      }
    } else if constexpr (Eng::kFast) {
      stage_rows<C>(sm, inp, M, rs, ncols_in, in_rpb, a.in_bstride, a.in_magic);
      cp_async_wait_all();
      SRK_BAR();
      SRK_TS(1)
    }
    auto ld = [&](int row, int col) -> cplx {
      return Eng::kFast ? sm[row * C + col] : inp[row_off(row, rs, in_rpb, a.in_bstride, a.in_magic) + (unsigned)col];
    };
    auto st = [&](int row, int col, cplx v) {
      const int c = trunc_dst(row, n, M, zn);
      if (c == -1) return;
      cplx o = cmk(v.x * sc, v.y * sc);
      if (c == -2) o = cmk(0.0, 0.0);
      if (zdc && c == 0 && col == 0) o.y = 0.0;
      oel(c == -2 ? (n >> 1) : c, col) = o;
    };
    Eng::template run<SIGN, Eng::kFast, false>(a.gp, sm, twp, ncols, ld, st);
  }
  if (a.dbg) {
    SRK_BAR();
    SRK_TS(2)
  }
}

// ---------------------------------------------------------------------------
// z-pencil pass.  Pencil p (= x*m1 + y; m1 = 1 in 2D) of signal s lives at
// s * sig_stride + p * K in the spectral buffers, at s * rsig_stride + p * M in
// the real physical buffers.  One CTA = two pencils; the 2*S real signals are
// packed pairwise into S complex FFTs (two-for-one real transforms).
// ---------------------------------------------------------------------------
struct ZArgs {
  const cplx* in;
  cplx* out;
  const double* in_real;
  double* out_real;
  const cplx* tw;
  GenPlan gp;
  int M;  // padded z length (real)
  int n;  // coarse z length
  int K;  // stored modes n/2+1
  int Kp; // pencil pitch of the spectral buffers in complex elements (0: K); the RHS pads it so
          // that every pencil row starts on a 32 B sector (rhs_impl)
  int P;  // pencils
  int S;  // input real signals per pencil
  int So; // output real signals per pencil
  long long in_sig_stride, out_sig_stride;  // complex elements (P*K) or real (P*M)
  int zero_nyq;  // R2C: zero the kz = n/2 plane (narrow)
  int mode;      // measurement only (SRK_PROBE_Z, one-pencil NS3 pass): 1 = stage the rows and return,
                 // 2 = also store zeros in the output pattern (no transforms)
  int pf_dist;   // NS3 z-pass: > 0 prefetch the inputs of block bid + pf_dist into L2
  unsigned long long* dbg;  // optional phase timestamps (tools/phase_timing.py)
};

template <int OP>
struct ZSig {
  static constexpr int S = (OP == ZOP_NS3) ? 6 : (OP == ZOP_NS2) ? 3 : (OP == ZOP_B3) ? 7 : (OP == ZOP_B2) ? 4 : 0;
  static constexpr int So = (OP == ZOP_NS3) ? 3 : (OP == ZOP_NS2) ? 2 : (OP == ZOP_B3) ? 6 : (OP == ZOP_B2) ? 4 : 0;
};

// physics.py:62-82 (u x w) and :151-158 (rho u) on one padded grid point
template <int OP>
SRK_DEV void zphys(const double* r, double* o) {
  if constexpr (OP == ZOP_NS3 || OP == ZOP_B3) {
    o[0] = r[1] * r[5] - r[2] * r[4];
    o[1] = r[2] * r[3] - r[0] * r[5];
    o[2] = r[0] * r[4] - r[1] * r[3];
    if constexpr (OP == ZOP_B3) {
      o[3] = r[6] * r[0];
      o[4] = r[6] * r[1];
      o[5] = r[6] * r[2];
    }
  } else if constexpr (OP == ZOP_NS2 || OP == ZOP_B2) {
    o[0] = r[1] * r[2];
    o[1] = -(r[0] * r[2]);
    if constexpr (OP == ZOP_B2) {
      o[2] = r[3] * r[0];
      o[3] = r[3] * r[1];
    }
  }
}

// Eng runs the inverse transforms (PPC*S/2 complex columns); EngF the forward
// ones (PPC*So/2 columns) -- a different plan when So < S so all threads stay
// busy.  PPC = pencils per CTA: 2 (real signals paired across the two pencils)
// or 1 (S and So even: paired within the pencil; half the tile, twice the CTAs
// per SM -- the 2D Boussinesq pass at 1024^2, where one CTA per SM left each
// SM waiting on one tile at a time).
template <class Eng, class L, int OP, class EngF = Eng, int PPC = 2>
__global__ void __launch_bounds__(Eng::NT, (PPC == 1 && Eng::NT <= 128 ? 3 : (Eng::NT <= 192 ? 2 : 1))) k_zpass(const ZArgs a, int S_rt, int So_rt) {
  extern __shared__ __align__(16) cplx smraw[];
  pdl_launch_dependents();
  srk_poison_smem(smraw);
  cplx* const sm = smraw + Eng::TWN;  // [twiddle table][tile]
  const cplx* const twp = Eng::kFast ? smraw : a.tw;
  if constexpr (Eng::kFast) {
    tw_fill<Eng::M>(smraw, a.tw);  // first use is after a CTA barrier
    cp_async_wait_all();
  }
  pdl_wait();
  const int p0 = PPC * blockIdx.x;
  const int S = (OP >= ZOP_NS3) ? ZSig<OP>::S : S_rt;
  const int So = (OP >= ZOP_NS3) ? ZSig<OP>::So : So_rt;
  // physics ops always run on the 3/2-padded axis: M = 3n/2, K = n/2 + 1 = M/3 + 1,
  // known at compile time for the fast plans (lets the compiler resolve the
  // Hermitian / zero-band selects and prune dead outputs statically)
  constexpr bool kCT = Eng::kFast && OP >= ZOP_NS3;
  const int M = kCT ? Eng::M : a.M;
  const int K = kCT ? Eng::M / 3 + 1 : a.K;
  const int KP = a.Kp ? a.Kp : K;  // pencil pitch in the spectral buffers
  if constexpr (OP != ZOP_R2C) {
    // ---- stage the 2*S input rows (K contiguous modes each) in smem.  Fast
    // path: one elected thread issues 1D TMA bulk copies (cp.async.bulk) that
    // complete on an mbarrier; the engine's tile aliases the staging area (its
    // first stage loads everything before its first barrier-protected store).
    cplx* stg = Eng::kFast ? sm : sm + L::SIZE;
    __shared__ __align__(8) unsigned long long mbar;
    const bool bulk = Eng::kFast && ((K * 16) % 16 == 0);
    if (bulk) {
      if (threadIdx.x == 0) {
        mbar_init(&mbar, 1);
        fence_mbar_init();
      }
      SRK_BAR();
      if (threadIdx.x == 0) {
        unsigned bytes = 0;
        for (int g = 0; g < PPC * S; ++g) bytes += (p0 + g / S < a.P) ? (unsigned)(K * 16) : 0u;
        mbar_expect_tx(&mbar, bytes);
        for (int g = 0; g < PPC * S; ++g) {
          const int pp = g / S, s = g - pp * S, pen = p0 + pp;
          if (pen < a.P)
            bulk_g2s(stg + g * K, a.in + s * a.in_sig_stride + (long long)pen * KP, (unsigned)(K * 16), &mbar);
        }
      }
      // rows of a missing second pencil (odd P) are zero
      if (PPC == 2 && p0 + 1 >= a.P)
        for (int i = threadIdx.x; i < S * K; i += blockDim.x) stg[S * K + i] = cmk(0.0, 0.0);
      mbar_wait(&mbar, 0);
      SRK_BAR();
    } else {
      for (int g = 0; g < PPC * S; ++g) {
        const int pp = g / S, s = g - pp * S, pen = p0 + pp;
        const cplx* __restrict__ src = a.in + s * a.in_sig_stride + (long long)pen * KP;
        for (int k = threadIdx.x; k < K; k += blockDim.x) stg[g * K + k] = (pen < a.P) ? src[k] : cmk(0.0, 0.0);
      }
      SRK_BAR();
    }
    // Hermitian extension of stored modes onto the padded z axis (branch free)
    auto hs = [&](int g, int k) -> cplx {
      const bool head = k < K;
      const bool tail = k >= M - (K - 1);
      const int kk = head ? k : (tail ? M - k : 0);
      cplx X = stg[g * K + kk];
      X.y = tail ? -X.y : X.y;
      if (k == 0 || 2 * k == M) X.y = 0.0;  // irfft ignores Im of DC / Nyquist
      return (head || tail) ? X : cmk(0.0, 0.0);
    };
    // ---- inverse: PPC*S/2 complex columns, column c carries real signals 2c, 2c+1 ----
    const int NCI = PPC * S / 2 + (PPC * S) % 2;
    auto ld = [&](int k, int c) -> cplx {
      cplx A = hs(2 * c, k), B = hs(2 * c + 1, k);
      return cmk(A.x - B.y, A.y + B.x);
    };
    if constexpr (OP == ZOP_C2R) {
      auto st = [&](int n, int c, cplx v) {
        const int g0 = 2 * c, g1 = 2 * c + 1;
        {
          const int pp = g0 / S, s = g0 - pp * S, pen = p0 + pp;
          if (pen < a.P) a.out_real[s * a.out_sig_stride + (long long)pen * M + n] = v.x;
        }
        if (g1 < PPC * S) {
          const int pp = g1 / S, s = g1 - pp * S, pen = p0 + pp;
          if (pen < a.P) a.out_real[s * a.out_sig_stride + (long long)pen * M + n] = v.y;
        }
      };
      Eng::template run<+1, true, false>(a.gp, sm, twp, NCI, ld, st);
      return;
    } else {
      auto st = [&](int n, int c, cplx v) { sm[L::idx(n, c)] = v; };
      Eng::template run<+1, true, true>(a.gp, sm, twp, NCI, ld, st);
      SRK_BAR();
      // ---- physical space: per row n, both pencils ----
      for (int n = threadIdx.x; n < M; n += blockDim.x) {
        double r[2 * 7];
#pragma unroll
        for (int c = 0; c < PPC * ZSig<OP>::S / 2; ++c) {
          cplx z = sm[L::idx(n, c)];
          r[2 * c] = z.x;
          r[2 * c + 1] = z.y;
        }
        double o[2 * 6];
        zphys<OP>(r, o);
        if constexpr (PPC == 2) zphys<OP>(r + ZSig<OP>::S, o + ZSig<OP>::So);
#pragma unroll
        for (int c = 0; c < PPC * ZSig<OP>::So / 2; ++c) sm[L::idx(n, c)] = cmk(o[2 * c], o[2 * c + 1]);
      }
      SRK_BAR();
    }
  }
  // ---- forward: PPC*So/2 complex columns ----
  const int NCO = PPC * So / 2 + (PPC * So) % 2;
  if constexpr (OP == ZOP_R2C) {
    auto ld = [&](int n, int c) -> cplx {
      double v[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int g = 2 * c + h;
        const int pp = g / So, s = g - pp * So, pen = p0 + pp;
        v[h] = (g < PPC * So && pen < a.P) ? a.in_real[s * a.in_sig_stride + (long long)pen * M + n] : 0.0;
      }
      return cmk(v[0], v[1]);
    };
    auto st = [&](int n, int c, cplx v) { sm[L::idx(n, c)] = v; };
    Eng::template run<-1, false, true>(a.gp, sm, twp, NCO, ld, st);
  } else {
    auto ld = [&](int n, int c) -> cplx { return sm[L::idx(n, c)]; };
    // only rows [0, K-1) and (M-K+1, M) feed the kept modes (kz = n/2 is zeroed)
    auto st = [&](int n, int c, cplx v) {
      if (n < K - 1 || n > M - K + 1) sm[L::idx(n, c)] = v;
    };
    EngF::template run<-1, true, true>(a.gp, sm, twp, NCO, ld, st);
  }
  SRK_BAR();
  // ---- extraction: two real spectra from each complex column, keep K modes ----
  const bool zn = a.zero_nyq != 0;
  for (int i = threadIdx.x; i < NCO * K; i += blockDim.x) {
    const int c = i / K, k = i - (i / K) * K;
    const bool live = !(zn && k == K - 1);
    const cplx Zk = live ? sm[L::idx(k, c)] : cmk(0.0, 0.0);
    const cplx Zm = live ? sm[L::idx(k == 0 ? 0 : M - k, c)] : cmk(0.0, 0.0);
    cplx A = cmk(0.5 * (Zk.x + Zm.x), 0.5 * (Zk.y - Zm.y));
    cplx B = cmk(0.5 * (Zk.y + Zm.y), -0.5 * (Zk.x - Zm.x));
    if (zn && k == K - 1) {
      A = cmk(0.0, 0.0);
      B = A;
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int g = 2 * c + h;
      if (g >= PPC * So) break;
      const int pp = g / So, s = g - pp * So, pen = p0 + pp;
      if (pen < a.P) a.out[s * a.out_sig_stride + (long long)pen * KP + k] = h ? B : A;
    }
  }
}


// ---------------------------------------------------------------------------
// First-stage loader of the fused z-passes: Hermitian extension of the staged
// rows (K stored modes each) onto the padded axis and two-for-one packing of
// real signals 2c, 2c+1 into complex column c.  With the row range of the lane
// group known at compile time (ld_has_range), rows in the 3/2-rule zero band
// [K, M-K+1) are never read and pure head / tail groups drop the selects (the
// inverse's staged-row reads were ~19% of the z-pass's shared-memory traffic).
// irfft ignores Im of the DC mode (2k == M cannot occur inside the padded band).
// ---------------------------------------------------------------------------
// CP > 0: the two staged rows of complex column c lie at stg + c * CP (+ K for the second),
// i.e. inside tile column c itself (CP = the tile's column pitch): the first stage then
// needs no CTA barrier (ld_col_private).  CP = 0: dense rows, 2c and 2c + 1.
template <int M, int CP = 0>
struct ZHermLoadT {
  static constexpr int kRange = 1;
  static constexpr int K = M / 3 + 1;
  const cplx* stg;
  __device__ __forceinline__ static int rowA(int c) { return CP > 0 ? c * CP : (2 * c) * K; }
  __device__ __forceinline__ static int rowB(int c) { return rowA(c) + K; }
  __device__ __forceinline__ static cplx pack(cplx A, cplx B) { return cmk(A.x - B.y, A.y + B.x); }
  __device__ __forceinline__ cplx head(int k, int c) const {
    cplx A = stg[rowA(c) + k], B = stg[rowB(c) + k];
    if (k == 0) A.y = B.y = 0.0;
    return pack(A, B);
  }
  __device__ __forceinline__ cplx tail(int k, int c) const {
    const cplx A = stg[rowA(c) + (M - k)], B = stg[rowB(c) + (M - k)];
    return pack(cmk(A.x, -A.y), cmk(B.x, -B.y));
  }
  __device__ __forceinline__ cplx operator()(int k, int c) const {
    const bool hd = k < K, tl = k >= M - (K - 1);
    const int kk = hd ? k : (tl ? M - k : 0);
    cplx A = stg[rowA(c) + kk], B = stg[rowB(c) + kk];
    if (tl) {
      A.y = -A.y;
      B.y = -B.y;
    }
    if (k == 0) A.y = B.y = 0.0;
    return (hd || tl) ? pack(A, B) : cmk(0.0, 0.0);
  }
  __device__ __forceinline__ cplx operator()(int k, int c, int rlo, int rhi) const {
    if (rlo >= K && rhi < M - (K - 1)) return cmk(0.0, 0.0);  // zero band: no read
    if (rhi < K) return head(k, c);
    if (rlo >= M - (K - 1)) return tail(k, c);
    return (*this)(k, c);
  }
};
template <int M>
using ZHermLoad = ZHermLoadT<M, 0>;
template <int M, int CP>
struct ZHermLoadCol : ZHermLoadT<M, CP> {
  static constexpr int kColPrivate = 1;
};

// ---------------------------------------------------------------------------
// NS3 z-pass with a fused middle stage (fast plans only).  Inverse plan
// (IR..., 4), forward plan (4, FR...), E = 24, M/4 threads (= 6 columns x
// M/24).  Thread j runs the last inverse radix-4 butterfly of all 6 complex
// columns (both pencils) on rows j + M/4*q, forms u x w for both pencils on
// those 4 rows in registers, packs the 6 real products into the 3 forward
// columns and runs the first forward radix-4 butterfly (same rows) before
// writing back -- no physical-space pass through shared memory.  The final
// forward stage only stores the rows the extraction reads (dead outputs of the
// last butterfly are removed at compile time).
// ---------------------------------------------------------------------------
template <int M, class L, class EngI, int EF, int... FR>
__global__ void __launch_bounds__(M / 4, (M / 4 <= 224 ? 2 : 1)) k_zpass_ns3f(const ZArgs a, int, int) {
  extern __shared__ __align__(16) cplx smraw[];
  cplx* const sm = smraw + EngI::TWN;  // [twiddle table][tile]
  const cplx* const twp = smraw;
  pdl_launch_dependents();
  srk_poison_smem(smraw);
  tw_fill<M>(smraw, a.tw);  // cp.async; waited for before the staging barrier
  constexpr int S = 6, So = 3, NT = M / 4, K = M / 3 + 1, Q = M / 4;
  const int KP = a.Kp ? a.Kp : K;  // pencil pitch in the spectral buffers
  static_assert(EngI::NT == NT, "inverse prefix must use M/4 threads");
  const int p0 = 2 * blockIdx.x;
  const int tid = threadIdx.x;
  SRK_TS_INIT(a.dbg, 6)
  SRK_TS(0)
  // ---- staging: 12 real-signal rows of K modes via 1D TMA bulk copies ----
  cplx* stg = sm;
  __shared__ __align__(8) unsigned long long mbar;
  if (tid == 0) {
    mbar_init(&mbar, 1);
    fence_mbar_init();
  }
  SRK_BAR();
  pdl_wait();
  if (tid == 0) {
    unsigned bytes = 0;
    for (int g = 0; g < 2 * S; ++g) bytes += (p0 + g / S < a.P) ? (unsigned)(K * 16) : 0u;
    mbar_expect_tx(&mbar, bytes);
    for (int g = 0; g < 2 * S; ++g) {
      const int pp = g / S, s = g - pp * S, pen = p0 + pp;
      if (pen < a.P) bulk_g2s(stg + g * K, a.in + s * a.in_sig_stride + (long long)pen * KP, (unsigned)(K * 16), &mbar);
    }
    // warm L2 with the rows of the pencil pair about one wave of CTAs ahead
    if (a.pf_dist) {
      const int q0 = p0 + 2 * a.pf_dist;
      for (int g = 0; g < 2 * S; ++g) {
        const int pp = g / S, s = g - pp * S, pen = q0 + pp;
        if (pen < a.P) bulk_prefetch_l2(a.in + s * a.in_sig_stride + (long long)pen * KP, (unsigned)(K * 16));
      }
    }
  }
  if (p0 + 1 >= a.P)
    for (int i = tid; i < S * K; i += NT) stg[S * K + i] = cmk(0.0, 0.0);
  mbar_wait(&mbar, 0);
  cp_async_wait_all();
  SRK_BAR();
  SRK_TS(1)
  // ---- inverse prefix stages (Stockham, in place) ----
  {
    ZHermLoad<M> ld{stg};
    auto st = [&](int n, int c, cplx v) { sm[L::idx(n, c)] = v; };
    EngI::template run_ws<+1, true, true>(a.gp, sm, twp, S, ld, st);
  }
  SRK_BAR();
  SRK_TS(2)
  // ---- fused: last inverse radix-4 (Ls = M/4) | u x w | first forward radix-4 ----
  {
    const int j = tid;
    cplx v[S][4];
#pragma unroll
    for (int c = 0; c < S; ++c) {
      if constexpr (Q % 8 == 0) {
        const int a0 = L::idx(j, c);
#pragma unroll
        for (int t = 0; t < 4; ++t) v[c][t] = sm[a0 + t * (Q / 8) * L::STEP8];
      } else {
#pragma unroll
        for (int t = 0; t < 4; ++t) v[c][t] = sm[L::idx(j + t * Q, c)];
      }
    }
    cplx w[4];
    w[1] = tw_get<M>(twp, (unsigned)j);
    w[1].y = -w[1].y;  // inverse sign
    w[2] = csq(w[1]);
    w[3] = cmul(w[2], w[1]);
    SRK_BAR();
    double o[4][6];
#pragma unroll
    for (int c = 0; c < S; ++c) {
#pragma unroll
      for (int t = 1; t < 4; ++t) v[c][t] = cmul(v[c][t], w[t]);
      DFT<4, +1>::run(v[c]);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
#pragma unroll
      for (int pp = 0; pp < 2; ++pp) {
        double r[6] = {v[3 * pp][q].x, v[3 * pp][q].y, v[3 * pp + 1][q].x,
                       v[3 * pp + 1][q].y, v[3 * pp + 2][q].x, v[3 * pp + 2][q].y};
        zphys<ZOP_NS3>(r, &o[q][3 * pp]);
      }
    }
#pragma unroll
    for (int c = 0; c < So; ++c) {
      cplx F[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) F[q] = cmk(o[q][2 * c], o[q][2 * c + 1]);
      DFT<4, -1>::run(F);
      const int a0 = L::idx(4 * j, c);  // Stockham stage-1 outputs: rows 4j + q
#pragma unroll
      for (int q = 0; q < 4; ++q) sm[a0 + q * L::ROWSTEP] = F[q];
    }
  }
  SRK_BAR();
  SRK_TS(3)
  // ---- forward suffix stages (Ls = 4 ...) on the 3 packed columns ----
  {
    // EF elements per thread: 12 puts all M/4 threads on the 3 forward columns
    constexpr int TPC = M / (EF > 0 ? EF : 24);
    const int col = tid / TPC, tj = tid - (tid / TPC) * TPC;
    const bool act = col < So;
    __builtin_assume(tj >= 0 && tj < TPC);
    auto ld = [&](int, int) -> cplx { return cmk(0.0, 0.0); };
    auto st = [&](int n, int c, cplx v) {
      if (n < K - 1 || n > M - K + 1) sm[L::idx(n, c)] = v;
    };
    if constexpr (EF == 0)  // one butterfly per thread, all threads on the 3 columns
      OneStageZ<M, L, -1, 4, FR...>::go(sm, twp, So, st);
    else
      FastStageW<M, (EF > 0 ? EF : 24), L, -1, true, true, 4, FR...>::go(sm, twp, col, tj, act, ld, st);
  }
  SRK_BAR();
  SRK_TS(4)
  // ---- extraction: two real spectra per complex column, K modes, kz = n/2 zeroed.
  // The 6 output rows are assembled in the idle tile columns So..S-1 and
  // written by 1D TMA bulk stores (one elected thread), so the CTA retires
  // without waiting on per-thread global stores.
  static_assert(2 * So * K <= (S - So) * L::PITCH, "output rows must fit the idle tile columns");
  cplx* const ost = sm + So * L::PITCH;  // [g][K], g = 2c + h
  for (int i = tid; i < So * K; i += NT) {
    const int c = i / K, k = i - (i / K) * K;
    const bool live = k != K - 1;
    const cplx Zk = live ? sm[L::idx(k, c)] : cmk(0.0, 0.0);
    const cplx Zm = live ? sm[L::idx(k == 0 ? 0 : M - k, c)] : cmk(0.0, 0.0);
    ost[(2 * c) * K + k] = cmk(0.5 * (Zk.x + Zm.x), 0.5 * (Zk.y - Zm.y));
    ost[(2 * c + 1) * K + k] = cmk(0.5 * (Zk.y + Zm.y), -0.5 * (Zk.x - Zm.x));
  }
  fence_proxy_async_smem();
  SRK_BAR();
  if (tid == 0) {
    for (int g = 0; g < 2 * So; ++g) {
      const int pp = g / So, s = g - pp * So, pen = p0 + pp;
      if (pen < a.P) bulk_s2g(a.out + s * a.out_sig_stride + (long long)pen * KP, ost + g * K, (unsigned)(K * 16));
    }
    bulk_commit_and_wait_read();
  }
  if (a.dbg) {
    SRK_BAR();
    SRK_TS(5)
  }
}



// ---------------------------------------------------------------------------
// Stages after a caller-run prefix with the thread -> (column, butterfly) map
// redone per stage and NCOL * M/R butterflies looped over the CTA (each
// thread keeps ceil(NCOL*M/R / NT) butterflies live across the barrier).
// ---------------------------------------------------------------------------
// A storer with a member kFin consumes the last stage's butterflies whole
// (fin(v, col, j): outputs v[q] = row j + q*Ls, still in registers) instead of
// row by row through shared memory -- no store barrier, no extraction pass.
template <class T, class = void>
struct st_has_fin : std::false_type {};
template <class T>
struct st_has_fin<T, decltype(void(T::kFin))> : std::true_type {};

template <int M, class L, int SIGN, int NCOL, int NT, int Ls, int R, int... Rest>
struct LoopStageZ {
  template <class ST>
  __device__ __forceinline__ static void go(cplx* sm, const cplx* tw, ST& st) {
    constexpr int STRIDE = M / R;
    constexpr int TOT = NCOL * STRIDE;
    constexpr int NB = (TOT + NT - 1) / NT;
    constexpr bool LAST = (sizeof...(Rest) == 0);
    if constexpr (LAST && st_has_fin<ST>::value) {
      static_assert(NB == 1 && Ls == STRIDE && STRIDE == 32, "fused last stage: one warp per column");
      const int u = threadIdx.x;
      if (u < TOT) {  // warp-uniform (TOT is a multiple of 32)
        const int col = u / STRIDE, j = u - col * STRIDE;
        cplx v[R];
        const int a0 = L::idx(j, col);
#pragma unroll
        for (int t = 0; t < R; ++t) v[t] = sm[a0 + t * (STRIDE / 8) * L::STEP8];
        stage_twiddle_sq<M, R, SIGN>(v, tw, (unsigned)j * (unsigned)(M / (Ls * R)));
        DFT<R, SIGN>::run(v);
        st.template fin<R>(v, col, j);
      }
    } else {
      go_rows(sm, tw, st);
    }
  }
  template <class ST>
  __device__ __forceinline__ static void go_rows(cplx* sm, const cplx* tw, ST& st) {
    constexpr int STRIDE = M / R;
    constexpr int TOT = NCOL * STRIDE;
    constexpr int NB = (TOT + NT - 1) / NT;
    constexpr bool LAST = (sizeof...(Rest) == 0);
    const int tid = threadIdx.x;
    cplx v[NB][R];
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const int u = tid + b * NT;
      if (TOT % NT == 0 || u < TOT) {
        const int col = u / STRIDE, j = u - col * STRIDE;
        if constexpr (STRIDE % 8 == 0) {
          const int a0 = L::idx(j, col);
#pragma unroll
          for (int t = 0; t < R; ++t) v[b][t] = sm[a0 + t * (STRIDE / 8) * L::STEP8];
        } else {
#pragma unroll
          for (int t = 0; t < R; ++t) v[b][t] = sm[L::idx(j + t * STRIDE, col)];
        }
        const unsigned k = (unsigned)j % (unsigned)Ls;
        stage_twiddle_sq<M, R, SIGN>(v[b], tw, k * (unsigned)(M / (Ls * R)));
        DFT<R, SIGN>::run(v[b]);
      }
    }
    SRK_BAR();
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const int u = tid + b * NT;
      if (TOT % NT == 0 || u < TOT) {
        const int col = u / STRIDE, j = u - col * STRIDE;
        const unsigned k = (unsigned)j % (unsigned)Ls;
        const int base = (int)(((unsigned)j - k) * (unsigned)R + k);
        if constexpr (LAST) {
#pragma unroll
          for (int q = 0; q < R; ++q) st(base + q * Ls, col, v[b][q]);
        } else if constexpr (Ls % 8 == 0) {
          const int a0 = L::idx(base, col);
#pragma unroll
          for (int q = 0; q < R; ++q) sm[a0 + q * (Ls / 8) * L::STEP8] = v[b][q];
        } else {
#pragma unroll
          for (int q = 0; q < R; ++q) sm[L::idx(base + q * Ls, col)] = v[b][q];
        }
      }
    }
    if constexpr (!LAST) {
      SRK_BAR();
      LoopStageZ<M, L, SIGN, NCOL, NT, Ls * R, Rest...>::go(sm, tw, st);
    }
  }
};

// ---------------------------------------------------------------------------
// NS3 z-pass, one pencil per CTA (SRK_ZP1): 3 inverse complex columns
// (two-for-one: [u0 u1][u2 w0][w1 w2]), fused middle stage (last inverse
// radix-4 | u x w | first forward radix-4, two butterfly rows per thread),
// forward suffix on 2 columns [P0 + i P1][P2] looped over the CTA, extraction
// (two-for-one for P0/P1, P2 read directly).  A third of the pencil-pair
// kernel's shared memory and half its threads per CTA: 5 CTAs (15 warps) per
// SM with independent phases instead of 2 CTAs (12 warps) -- at the price of
// one extra 768-point forward transform per two pencils (P2 rides alone).
// ---------------------------------------------------------------------------
// Last-stage consumer of the one-pencil NS3 z-pass (see LoopStageZ / st_has_fin).
// Column 0 = FFT(P0 + i P1): P0[k] = (Z[k] + conj Z[M-k]) / 2, P1[k] = (Z[k] -
// conj Z[M-k]) / (2i); column 1 = FFT(P2) stored directly.  Butterfly j of the
// last stage (radix R = M/32, Ls = 32) holds rows j + 32 q; rows k < K - 1 are
// q < R/3, and row M - k = (32 - j) + 32 (R - 1 - q) is output R - 1 - q of
// lane 32 - j (j = 0: output R - q of lane 0 itself).
template <int M>
struct ZFinNS3 {
  static constexpr int kFin = 1;
  cplx* o;  // out + pen * pitch
  long long ss;
  bool pad;  // pitch > K
  template <int R>
  __device__ __forceinline__ void fin(cplx (&v)[R], int col, int j) const {
    constexpr int K = M / 3 + 1, QK = R / 3;
    static_assert(M == 32 * R && R % 3 == 0, "one warp per column, K - 1 = 32 R / 3 rows kept");
    if (col == 0) {
      const int src = (32 - j) & 31;
#pragma unroll
      for (int q = 0; q < QK; ++q) {
        const cplx Zk = v[q];
        cplx Zm;
        Zm.x = __shfl_sync(0xffffffffu, v[R - 1 - q].x, src);
        Zm.y = __shfl_sync(0xffffffffu, v[R - 1 - q].y, src);
        if (j == 0) Zm = v[(R - q) % R];
        const int k = j + 32 * q;
        o[k] = cmk(0.5 * (Zk.x + Zm.x), 0.5 * (Zk.y - Zm.y));
        o[ss + k] = cmk(0.5 * (Zk.y + Zm.y), -0.5 * (Zk.x - Zm.x));
      }
      if (j == 0) {
        o[K - 1] = o[ss + K - 1] = cmk(0.0, 0.0);  // kz = n/2 zeroed (narrow)
        if (pad) o[K] = o[ss + K] = cmk(0.0, 0.0);   // pad column: the row's last 32 B sector is written whole
      }
    } else {
#pragma unroll
      for (int q = 0; q < QK; ++q) {
        const int k = j + 32 * q;
        o[2 * ss + k] = (k == 0) ? cmk(v[q].x, 0.0) : v[q];
      }
      if (j == 0) {
        o[2 * ss + K - 1] = cmk(0.0, 0.0);
        if (pad) o[2 * ss + K] = cmk(0.0, 0.0);
      }
    }
  }
};
template <int M, int... FR>
struct ns3p_fused_last {
  static constexpr int RL = (FR, ...);  // last radix
  static constexpr bool value = (M == 32 * RL) && (RL % 3 == 0);
};

#define SRK_ZP1_MINB 5   // CTAs per SM the register budget targets (shared memory allows 5)
#define SRK_ZB2P_MINB 3  // CTAs per SM of the 2D Boussinesq variant (M = 1536, 128 threads)
// OP = ZOP_B2 (2D Boussinesq, v15): 2 inverse columns [u0 + i u1][w + i rho],
// the four products [w u1 + i(-w u0)][rho u0 + i rho u1] packed in the 2
// forward columns, both extracted two-for-one; NT = M/12 (E = 24 on 2 columns,
// three fused-middle rows per thread).
template <int M, class L, class EngI, int OP, int... FR>
__global__ void __launch_bounds__(EngI::NT, (OP == ZOP_B2 ? SRK_ZB2P_MINB : (M <= 768 ? SRK_ZP1_MINB : 2)))
    k_zpass_ns3p(const ZArgs a, int, int) {
  extern __shared__ __align__(16) cplx smraw[];
  cplx* const sm = smraw + EngI::TWN;  // [twiddle table][tile]
  const cplx* const twp = smraw;
  pdl_launch_dependents();
  srk_poison_smem(smraw);
  tw_fill<M>(smraw, a.tw);
  static_assert(OP == ZOP_NS3 || OP == ZOP_B2, "NS3 or 2D Boussinesq");
  // NT = M/8 (E = 24: two fused-middle rows per thread); B2: M/12 (three rows)
  constexpr int S = OP == ZOP_B2 ? 2 : 3, NT = EngI::NT, K = M / 3 + 1, Q = M / 4, RPT = Q / NT;
  const int KP = a.Kp ? a.Kp : K;  // pencil pitch in the spectral buffers
  static_assert(OP == ZOP_B2 ? NT == M / 12 : NT == M / 8, "inverse prefix thread count");
  static_assert(L::C == S, "one tile column per inverse complex signal");
  static_assert(Q % NT == 0, "whole fused-middle rows per thread");
  const int pen = blockIdx.x;
  const int tid = threadIdx.x;
  SRK_TS_INIT(a.dbg, 6)
  SRK_TS(0)
  // ---- staging: 6 real-signal rows of K modes via 1D TMA bulk copies ----
  // When a warp owns a whole tile column (M / 24 = 32 threads per column), the two rows of
  // complex column c are staged inside tile column c: the first inverse stage then needs
  // no CTA barrier and the three warps run the whole prefix independently.
  constexpr bool kColStg = (EngI::TPC <= 32) && (2 * K <= L::PITCH);
  cplx* stg = sm;
  __shared__ __align__(8) unsigned long long mbar;
  if (tid == 0) {
    mbar_init(&mbar, 1);
    fence_mbar_init();
  }
  SRK_BAR();
  pdl_wait();
  if (tid == 0) {
    mbar_expect_tx(&mbar, (unsigned)(2 * S * K * 16));
    for (int s = 0; s < 2 * S; ++s)
      bulk_g2s(stg + (kColStg ? (s >> 1) * L::PITCH + (s & 1) * K : s * K),
               a.in + s * a.in_sig_stride + (long long)pen * KP, (unsigned)(K * 16), &mbar);
    if (a.pf_dist) {
      const int q0 = pen + a.pf_dist;
      if (q0 < a.P)
        for (int s = 0; s < 2 * S; ++s)
          bulk_prefetch_l2(a.in + s * a.in_sig_stride + (long long)q0 * KP, (unsigned)(K * 16));
    }
  }
  // every thread waits on the mbarrier itself (the TMA rows are then visible to
  // it); the twiddle table (cp.async by all threads) is first read in the second
  // inverse stage, after the first stage's CTA barrier (or the one below)
  mbar_wait(&mbar, 0);
  cp_async_wait_all();
  // column-private staging: the first stage has no CTA barrier to publish the twiddle
  // table (filled by all threads) before the second stage reads it -- sync here, where the
  // warps arrive together anyway (they all just left the same mbarrier)
  if constexpr (kColStg) SRK_BAR();
  SRK_TS(1)
  if (a.mode) {  // measurement only (SRK_PROBE_Z): the pencil's access pattern without the transforms
    if (a.mode == 2)
      for (int k = tid; k < (KP > K ? K + 1 : K); k += NT)
        for (int s = 0; s < ZSig<OP>::So; ++s) a.out[s * a.out_sig_stride + (long long)pen * KP + k] = cmk(0.0, 0.0);
    return;
  }
  {
    auto st = [&](int n, int c, cplx v) { sm[L::idx(n, c)] = v; };
    if constexpr (kColStg) {
      ZHermLoadCol<M, L::PITCH> ld{stg};
      EngI::template run_ws<+1, true, true>(a.gp, sm, twp, S, ld, st);
    } else {
      ZHermLoad<M> ld{stg};
      EngI::template run_ws<+1, true, true>(a.gp, sm, twp, S, ld, st);
    }
  }
  SRK_BAR();
  SRK_TS(2)
  // ---- fused: last inverse radix-4 | u x w | first forward radix-4; rows j, j + NT ----
  {
    cplx v[RPT][S][4];
#pragma unroll
    for (int h = 0; h < RPT; ++h) {
      const int j = tid + h * NT;
#pragma unroll
      for (int c = 0; c < S; ++c) {
        if constexpr (Q % 8 == 0) {
          const int a0 = L::idx(j, c);
#pragma unroll
          for (int t = 0; t < 4; ++t) v[h][c][t] = sm[a0 + t * (Q / 8) * L::STEP8];
        } else {
#pragma unroll
          for (int t = 0; t < 4; ++t) v[h][c][t] = sm[L::idx(j + t * Q, c)];
        }
      }
    }
    SRK_BAR();
#pragma unroll
    for (int h = 0; h < RPT; ++h) {
      const int j = tid + h * NT;
      cplx w[4];
      w[1] = tw_get<M>(twp, (unsigned)j);
      w[1].y = -w[1].y;  // inverse sign
      w[2] = csq(w[1]);  // one table read per row (stage_twiddle_sq)
      w[3] = cmul(w[2], w[1]);
#pragma unroll
      for (int c = 0; c < S; ++c) {
#pragma unroll
        for (int t = 1; t < 4; ++t) v[h][c][t] = cmul(v[h][c][t], w[t]);
        DFT<4, +1>::run(v[h][c]);
      }
      cplx F0[4], F1[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        double r[2 * S];
#pragma unroll
        for (int c = 0; c < S; ++c) {
          r[2 * c] = v[h][c][q].x;
          r[2 * c + 1] = v[h][c][q].y;
        }
        double o[4];
        zphys<OP>(r, o);
        F0[q] = cmk(o[0], o[1]);
        F1[q] = cmk(o[2], OP == ZOP_B2 ? o[3] : 0.0);
      }
      DFT<4, -1>::run(F0);
      DFT<4, -1>::run(F1);
      const int a0 = L::idx(4 * j, 0), a1 = L::idx(4 * j, 1);  // Stockham stage-1 outputs: rows 4j + q
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        sm[a0 + q * L::ROWSTEP] = F0[q];
        sm[a1 + q * L::ROWSTEP] = F1[q];
      }
    }
  }
  SRK_BAR();
  SRK_TS(3)
  // ---- NS3, last forward stage on one warp per column (M/R = 32): the stage's
  // outputs stay in registers; the mirror rows M - k of the two-for-one
  // separation sit in lane 32 - j of the same warp (lane 0: in its own
  // butterfly) and come over by shuffle, P2 is stored as computed -- the f2 ->
  // extraction exchange (~8% of the pass's shared-memory wavefronts), its
  // barrier and the extraction loop are gone (same arithmetic, bitwise).
  if constexpr (OP == ZOP_NS3 && ns3p_fused_last<M, FR...>::value) {
    ZFinNS3<M> fin{a.out + (long long)pen * KP, a.out_sig_stride, KP > K};
    LoopStageZ<M, L, -1, 2, NT, 4, FR...>::go(sm, twp, fin);
    if (a.dbg) {  // phase stamps (tools/phase_timing.py): the suffix now includes the extraction
      SRK_BAR();
      SRK_TS(4)
      SRK_TS(5)
    }
    return;
  }
  // ---- forward suffix (Ls = 4 ...) on the 2 packed columns ----
  {
    // only rows the extraction reads: column 0 (two-for-one) needs k < K-1 and its
    // mirror M-k; NS3's column 1 is the real P2 alone and needs k < K-1 only
    auto st = [&](int n, int c, cplx v) {
      const bool keep = (OP == ZOP_NS3 && c == 1) ? (n < K - 1) : (n < K - 1 || n > M - K + 1);
      if (keep) sm[L::idx(n, c)] = v;
    };
    LoopStageZ<M, L, -1, 2, NT, 4, FR...>::go(sm, twp, st);
  }
  SRK_BAR();
  SRK_TS(4)
  // ---- extraction: P0, P1 from column 0 (two-for-one), P2 = column 1; kz = n/2 zeroed ----
  for (int k = tid; k < K; k += NT) {
    const bool live = k != K - 1;
    const cplx Zk = live ? sm[L::idx(k, 0)] : cmk(0.0, 0.0);
    const cplx Zm = live ? sm[L::idx(k == 0 ? 0 : M - k, 0)] : cmk(0.0, 0.0);
    const cplx P2 = live ? sm[L::idx(k, 1)] : cmk(0.0, 0.0);
    cplx* o = a.out + (long long)pen * KP + k;
    o[0] = cmk(0.5 * (Zk.x + Zm.x), 0.5 * (Zk.y - Zm.y));
    o[a.out_sig_stride] = cmk(0.5 * (Zk.y + Zm.y), -0.5 * (Zk.x - Zm.x));
    if constexpr (OP == ZOP_B2) {  // column 1 = [P2 + i P3]: two-for-one as well
      const cplx Wm = live ? sm[L::idx(k == 0 ? 0 : M - k, 1)] : cmk(0.0, 0.0);
      o[2 * a.out_sig_stride] = cmk(0.5 * (P2.x + Wm.x), 0.5 * (P2.y - Wm.y));
      o[3 * a.out_sig_stride] = cmk(0.5 * (P2.y + Wm.y), -0.5 * (P2.x - Wm.x));
    } else {
      o[2 * a.out_sig_stride] = (k == 0) ? cmk(P2.x, 0.0) : P2;
    }
  }
  if (a.dbg) {
    SRK_BAR();
    SRK_TS(5)
  }
}
