// Argument structs / launchers for pointwise.cu (internal to libsrk).
#pragma once

#include "host_util.cuh"
#include "srk_common.cuh"

#define SRK_NQ 9
#define SRK_RED_BLOCKS 592  // 4 x 148 SMs; fixed so reductions are run-to-run deterministic
#define SRK_MAX_TERMS 8

struct GeomArgs {
  int dims;
  int n0, n1, K;  // 2D: n1 = 1, K = n_last/2+1; slab: n1 = local y rows
  double ck0, ck1, ck2;  // 2*pi/L per axis; 2D uses ck0 (x) and ck2 (last)
  int y0, n1g;    // slab: global y of local row 0, global y extent (n1g = n1, y0 = 0 unsplit)
};

struct ProjArgs {
  GeomArgs g;
  const cplx* G;  // narrow output: [u x w (d), (rho u)(d) if density]
  int Gp;         // pitch of G's kz rows in complex elements (0: g.K, the state's): the RHS pads
                  // its intermediates to whole 32 B sectors per row (rhs_pitch)
  const cplx* y;  // state [u (d), rho]
  cplx* f;
  long long modes;  // n0*n1*K
  int density;
  double nu, ri, re_pr;
  // fused next-stage combination (k_project_tma<DIMS, DENS, NT>, every state component):
  //   ynext = yb + sum_{t < nt} c[t] F[t] + cself * f
  const cplx* yb;
  const cplx* F[SRK_MAX_TERMS];
  double c[SRK_MAX_TERMS];
  int nt;
  double cself;
  cplx* ynext;
  // non-null: the coefficients are multiples of a step size held in device memory:
  // every c[t] and cself is used as (*hs) * c (one rounding: exactly the host
  // product h * a the reference forms) -- a CUDA graph replays with a new h
  const double* hs;
  // k_project_tma<3, false, 0, true> (srk_rhs_refresh): ybase is the state itself
  // (not streamed) and the block partials of E, eps, Z over the velocity
  // components go to partial[q * gridDim.x + block] (q = 4, 5, 8; others 0)
  double* partial;
};

struct CombArgs {
  const cplx* y;  // may be null (start from zero)
  const cplx* F[SRK_MAX_TERMS];
  double c[SRK_MAX_TERMS];
  const double* hs;  // non-null: c[j] scaled by *hs in the kernel (ProjArgs::hs)
  int nt;
  cplx* out;
  long long n;
};

struct RedArgs {
  GeomArgs g;
  const cplx* y0;  // pre-step state (norm)
  const cplx* y1;  // new state
  const cplx* F[SRK_MAX_TERMS];
  double c[SRK_MAX_TERMS];  // h*(b - b_hat) for the error vector
  const double* hs;         // non-null: c[j] = (b - b_hat)_j scaled by *hs in the kernel
  int nt;
  const cplx* fl;  // tendency at y1 (diag)
  int fl_term;     // >= 0: fl is F[fl_term] (the FSAL stage): streamed once, read from that slot
  int ncomp;
  int dvel;
  long long modes;
  int K;
  double atol, rtol;
  int do_norm, do_diag;
  double* partial;  // SRK_NQ * SRK_RED_BLOCKS
};

void srk_launch_project(const ProjArgs& a, cudaStream_t st);
#define SRK_PC_MAXT 6
bool srk_launch_project_comb(const ProjArgs& a, cudaStream_t st);
void srk_launch_curl(const GeomArgs& g, const cplx* u, cplx* w, long long n, cudaStream_t st);
void srk_launch_leray(const GeomArgs& g, const cplx* u, cplx* o, long long n, cudaStream_t st);
void srk_launch_combine(const CombArgs& a, cudaStream_t st);
void srk_launch_reduce(const RedArgs& a, double* out, cudaStream_t st);
void srk_launch_band_energy(const cplx* u, const long long* idx, const double* w, int nb, int ncomp,
                            long long modes, double* out, cudaStream_t st);
// srk_rhs_refresh: K6 + ynext = y + cself f + the (E, eps, Z) sums of (y, f);
// returns false when the fused kernel does not apply (2D, Boussinesq, >= 2^32 modes)
bool srk_launch_project_refresh(const ProjArgs& a, double* out, cudaStream_t st);
void srk_launch_store_mapped(const double* src, double* dst, int n, cudaStream_t st);
void srk_launch_band_scale(cplx* u, const long long* idx, int nb, int ncomp, long long modes, double gamma,
                           cudaStream_t st);
