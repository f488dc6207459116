// Pointwise and reduction kernels: projection/viscous epilogue (K6), curl and
// Leray projection (API helpers), RK stage combination (K6b), the fused
// embedded-error-norm + diagnostics reduction (K7) and the forcing band ops (K9).
//
// Where the reference's numpy op order is cheap to mirror (projection, stage
// sums, norms) the kernels use explicit _rn intrinsics so no FMA contraction
// changes the rounding relative to physics.py / integrators.py.
#include "pointwise.cuh"

#include <algorithm>
#include <cstdlib>

#define DMUL __dmul_rn
#define DADD __dadd_rn
#define DSUB __dsub_rn

__device__ __forceinline__ cplx rmul(double s, cplx a) { return make_double2(DMUL(s, a.x), DMUL(s, a.y)); }
__device__ __forceinline__ cplx radd(cplx a, cplx b) { return make_double2(DADD(a.x, b.x), DADD(a.y, b.y)); }
__device__ __forceinline__ cplx rsub(cplx a, cplx b) { return make_double2(DSUB(a.x, b.x), DSUB(a.y, b.y)); }

// coefficient j of a combination: c[j], or (*hs) * c[j] when the step size lives
// in device memory (graph replays); one rounding either way
__device__ __forceinline__ double coef(const double* c, const double* hs, int j) {
  return hs ? DMUL(__ldg(hs), c[j]) : c[j];
}

struct KVec {
  double k[3];
  double k2, inv_k2;
};

// grid.py:75-100: k_a = mode_a * (2 pi / L_a); k2 accumulated 0 + k0^2 + k1^2 (+ k2^2)
__device__ __forceinline__ KVec kvec(long long idx, const GeomArgs& g) {
  KVec r;
  const int kz = (int)(idx % g.K);
  const long long xy = idx / g.K;
  if (g.dims == 3) {
    const int y = (int)(xy % g.n1), x = (int)(xy / g.n1);
    r.k[0] = DMUL(mode_full(x, g.n0), g.ck0);
    r.k[1] = DMUL(mode_full(g.y0 + y, g.n1g), g.ck1);
    r.k[2] = DMUL((double)kz, g.ck2);
    r.k2 = DADD(DADD(DMUL(r.k[0], r.k[0]), DMUL(r.k[1], r.k[1])), DMUL(r.k[2], r.k[2]));
  } else {
    const int x = (int)xy;
    r.k[0] = DMUL(mode_full(x, g.n0), g.ck0);
    r.k[1] = DMUL((double)kz, g.ck2);
    r.k[2] = 0.0;
    r.k2 = DADD(DMUL(r.k[0], r.k[0]), DMUL(r.k[1], r.k[1]));
  }
  r.inv_k2 = (r.k2 == 0.0) ? 0.0 : __ddiv_rn(1.0, r.k2);
  return r;
}

// |k|^2 only (reductions): 32-bit index arithmetic when the mode count allows,
// no 1/k^2 division
__device__ __forceinline__ double k2_at(long long idx, const GeomArgs& g, bool small) {
  int kz, y, x;
  if (small) {
    const unsigned u = (unsigned)idx, K = (unsigned)g.K;
    const unsigned xy = u / K;
    kz = (int)(u - xy * K);
    if (g.dims == 3) {
      const unsigned n1 = (unsigned)g.n1, xq = xy / n1;
      y = (int)(xy - xq * n1);
      x = (int)xq;
    } else {
      y = 0;
      x = (int)xy;
    }
  } else {
    kz = (int)(idx % g.K);
    const long long xy = idx / g.K;
    y = g.dims == 3 ? (int)(xy % g.n1) : 0;
    x = g.dims == 3 ? (int)(xy / g.n1) : (int)xy;
  }
  if (g.dims == 3) {
    const double k0 = DMUL(mode_full(x, g.n0), g.ck0);
    const double k1 = DMUL(mode_full(g.y0 + y, g.n1g), g.ck1);
    const double k2 = DMUL((double)kz, g.ck2);
    return DADD(DADD(DMUL(k0, k0), DMUL(k1, k1)), DMUL(k2, k2));
  }
  const double k0 = DMUL(mode_full(x, g.n0), g.ck0);
  const double k1 = DMUL((double)kz, g.ck2);
  return DADD(DMUL(k0, k0), DMUL(k1, k1));
}

// kvec() with 32-bit index arithmetic (mode counts < 2^32)
__device__ __forceinline__ KVec kvec32(unsigned idx, const GeomArgs& g) {
  KVec r;
  const unsigned K = (unsigned)g.K;
  const unsigned xy = idx / K;
  const int kz = (int)(idx - xy * K);
  if (g.dims == 3) {
    const unsigned n1 = (unsigned)g.n1, xq = xy / n1;
    const int y = (int)(xy - xq * n1), x = (int)xq;
    r.k[0] = DMUL(mode_full(x, g.n0), g.ck0);
    r.k[1] = DMUL(mode_full(g.y0 + y, g.n1g), g.ck1);
    r.k[2] = DMUL((double)kz, g.ck2);
    r.k2 = DADD(DADD(DMUL(r.k[0], r.k[0]), DMUL(r.k[1], r.k[1])), DMUL(r.k[2], r.k[2]));
  } else {
    r.k[0] = DMUL(mode_full((int)xy, g.n0), g.ck0);
    r.k[1] = DMUL((double)kz, g.ck2);
    r.k[2] = 0.0;
    r.k2 = DADD(DMUL(r.k[0], r.k[0]), DMUL(r.k[1], r.k[1]));
  }
  r.inv_k2 = (r.k2 == 0.0) ? 0.0 : __ddiv_rn(1.0, r.k2);
  return r;
}

// K6, TMA-streamed (default): the G and state components of a chunk of
// CH modes arrive by 1D bulk copies in a two-stage shared-memory ring (one
// elected thread, mbarrier completion); f is stored straight from registers.
// Same arithmetic as k_project.
//
// NTC >= 0 (2D / 3D, NS or Boussinesq): the next RK stage input is formed in the same pass
// (integrators.py:327-339 / :336-339):
//   ynext = ybase + sum_{t < NTC} c_t F_t + cself * f
// ascending in the stage index with f = the tendency just computed (the last,
// highest-index term), one rounding per multiply and add -- bitwise what
// k_combine produces from the stored f, without reading f back.  ybase and the
// F_t ride in the same ring (256-mode chunks: one CTA per SM from 4 earlier
// stages on, still faster than 128-mode chunks at two CTAs per SM).
#define SRK_PT_CH 256
#define SRK_PC_CH 256  // modes per chunk (and threads) of the fused K6 + stage-sum kernel; ncu: 128 -> 256 is 1-7% faster
// shared-memory components streamed per mode: G, state, and (fused stage sum)
// ybase + the NTC earlier stages, each with the state's component count
template <int DIMS, bool DENS, int NTC, bool DIAG>
constexpr int proj_streams() {
  return (DENS ? 2 * DIMS : DIMS) + (DENS ? DIMS + 1 : DIMS) +
         (NTC < 0 ? 0 : ((DIAG ? 0 : 1) + NTC) * (DENS ? DIMS + 1 : DIMS));
}
// modes per chunk: 256, or 128 when a 256-mode two-stage ring would not fit
// the 227 KB opt-in shared memory (3D Boussinesq with 5-6 earlier stages)
template <int DIMS, bool DENS, int NTC, bool DIAG>
constexpr int proj_chunk() {
  return NTC < 0 ? SRK_PT_CH
                 : (2 * proj_streams<DIMS, DENS, NTC, DIAG>() * SRK_PC_CH * 16 <= 227 * 1024 - 64 ? SRK_PC_CH : 128);
}
template <int DIMS, bool DENS, int NTC = -1, bool DIAG = false>
__global__ void __launch_bounds__(proj_chunk<DIMS, DENS, NTC, DIAG>()) k_project_tma(const ProjArgs a) {
  extern __shared__ __align__(128) cplx psm[];
  srk_poison_smem(psm);
  constexpr int CH = proj_chunk<DIMS, DENS, NTC, DIAG>();
  constexpr int d = DIMS;
  constexpr int NG = DENS ? 2 * d : d;  // G components
  constexpr int NY = DENS ? d + 1 : d;  // state components
  // ybase + F_t components, NY each (DIAG: ybase is the state, already in the ring)
  constexpr int NC = NTC < 0 ? 0 : ((DIAG ? 0 : 1) + NTC) * NY;
  constexpr int NS = NG + NY + NC;
  static_assert(NS == proj_streams<DIMS, DENS, NTC, DIAG>(), "stream count");
  static_assert(!DIAG || NTC == 0, "refresh: the state's own next-stage input only");
  double e_acc = 0.0, ep_acc = 0.0, z_acc = 0.0;  // DIAG: E, eps, Z partial sums of this thread
  double cf[NTC > 0 ? NTC : 1];
#pragma unroll
  for (int t = 0; t < (NTC > 0 ? NTC : 0); ++t) cf[t] = coef(a.c, a.hs, t);
  const double cself = a.hs ? DMUL(__ldg(a.hs), a.cself) : a.cself;
  __shared__ __align__(8) unsigned long long mb[2];
  const int tid = threadIdx.x;
  const long long n = a.modes;
  const long long nch = (n + CH - 1) / CH;
  const int G = gridDim.x;
  if (tid == 0) {
    mbar_init(&mb[0], 1);
    mbar_init(&mb[1], 1);
    fence_mbar_init();
  }
  pdl_launch_dependents();
  pdl_wait();
  SRK_BAR();
  auto issue = [&](long long k, int b) {
    if (tid != 0 || k >= nch) return;
    const long long i0 = k * CH;
    const unsigned cnt = (unsigned)min((long long)CH, n - i0);
    cplx* st = psm + b * NS * CH;
    mbar_expect_tx(&mb[b], cnt * 16u * NS);
    if (a.Gp > a.g.K) {
      // G rows have a padded pitch: the chunk's modes [i0, i0 + cnt) are row segments of G
      const unsigned K = (unsigned)a.g.K, Kp = (unsigned)a.Gp;
      const long long nG = n / K * Kp;  // modes per component at the padded pitch
      unsigned done = 0;
      while (done < cnt) {
        const unsigned i = (unsigned)i0 + done, r = i / K, c = i - r * K;
        const unsigned len = min(cnt - done, K - c);
#pragma unroll
        for (int j = 0; j < NG; ++j)
          bulk_g2s(st + j * CH + done, a.G + j * nG + (long long)r * Kp + c, len * 16u, &mb[b]);
        done += len;
      }
    } else {
#pragma unroll
      for (int j = 0; j < NG; ++j) bulk_g2s(st + j * CH, a.G + j * n + i0, cnt * 16u, &mb[b]);
    }
#pragma unroll
    for (int j = 0; j < NY; ++j) bulk_g2s(st + (NG + j) * CH, a.y + j * n + i0, cnt * 16u, &mb[b]);
    if constexpr (NTC >= 0 && !DIAG) {
#pragma unroll
      for (int j = 0; j < NY; ++j) bulk_g2s(st + (NG + NY + j) * CH, a.yb + j * n + i0, cnt * 16u, &mb[b]);
#pragma unroll
      for (int t = 0; t < (NTC < 0 ? 0 : NTC); ++t)
#pragma unroll
        for (int j = 0; j < NY; ++j)
          bulk_g2s(st + (NG + 2 * NY + t * NY + j) * CH, a.F[t] + j * n + i0, cnt * 16u, &mb[b]);
    }
  };
  issue(blockIdx.x, 0);
  issue(blockIdx.x + G, 1);
  unsigned phase = 0;
  for (int it = 0; (long long)blockIdx.x + (long long)it * G < nch; ++it) {
    const long long k = blockIdx.x + (long long)it * G;
    const int b = it & 1;
    const long long i0 = k * CH;
    const int cnt = (int)min((long long)CH, n - i0);
    mbar_wait(&mb[b], (phase >> b) & 1u);
    phase ^= 1u << b;
    const cplx* st = psm + b * NS * CH;
    if (tid < cnt) {
      const long long i = i0 + tid;
      const KVec kv = kvec32((unsigned)i, a.g);
      cplx Gv[3];
#pragma unroll
      for (int j = 0; j < d; ++j) Gv[j] = st[j * CH + tid];
      cplx rho = make_double2(0.0, 0.0);
      if constexpr (DENS) {
        rho = st[(NG + d) * CH + tid];
        Gv[d - 1] = rsub(Gv[d - 1], rmul(a.ri, rho));
      }
      cplx kd = rmul(kv.k[0], Gv[0]);
#pragma unroll
      for (int j = 1; j < d; ++j) kd = radd(kd, rmul(kv.k[j], Gv[j]));
      kd = rmul(kv.inv_k2, kd);
      const double nuk2 = DMUL(a.nu, kv.k2);
      double wgt = 0.0;
      if constexpr (DIAG) {  // Hermitian weight of the mode (diagnostics.py:39-45)
        const int kz = (int)((unsigned)i % (unsigned)a.g.K);
        wgt = (kz == 0 || kz == a.g.K - 1) ? 1.0 : 2.0;
      }
#pragma unroll
      for (int j = 0; j < d; ++j) {
        const cplx u = st[(NG + j) * CH + tid];
        cplx o = rsub(Gv[j], rmul(kv.k[j], kd));
        o = rsub(o, rmul(nuk2, u));
        a.f[j * n + i] = o;
        if constexpr (DIAG) {  // same op order as k_reduce_tma's diagnostics
          const double m2 = DADD(DMUL(u.x, u.x), DMUL(u.y, u.y));
          e_acc = DADD(e_acc, DMUL(wgt, m2));
          ep_acc = DADD(ep_acc, DMUL(wgt, DADD(DMUL(u.x, o.x), DMUL(u.y, o.y))));
          z_acc = DADD(z_acc, DMUL(DMUL(wgt, kv.k2), m2));
        }
        if constexpr (NTC >= 0) {
          cplx acc = DIAG ? u : st[(NG + NY + j) * CH + tid];
#pragma unroll
          for (int t = 0; t < (NTC < 0 ? 0 : NTC); ++t)
            acc = radd(acc, rmul(cf[t], st[(NG + NY + (DIAG ? 0 : NY) + t * NY + j) * CH + tid]));
          a.ynext[j * n + i] = radd(acc, rmul(cself, o));
        }
      }
      if constexpr (DENS) {
        cplx div = rmul(kv.k[0], st[d * CH + tid]);
#pragma unroll
        for (int j = 1; j < d; ++j) div = radd(div, rmul(kv.k[j], st[(d + j) * CH + tid]));
        cplx o = make_double2(div.y, -div.x);  // -1j * div
        o = rsub(o, rmul(__ddiv_rn(kv.k2, a.re_pr), rho));
        a.f[d * n + i] = o;
        if constexpr (NTC >= 0) {  // the density component of the next stage input
          cplx acc = DIAG ? rho : st[(NG + NY + d) * CH + tid];
#pragma unroll
          for (int t = 0; t < (NTC < 0 ? 0 : NTC); ++t)
            acc = radd(acc, rmul(cf[t], st[(NG + 2 * NY + t * NY + d) * CH + tid]));
          a.ynext[d * n + i] = radd(acc, rmul(cself, o));
        }
      }
    }
    SRK_BAR();  // stage b consumed
    issue(k + 2LL * G, b);
  }
  if constexpr (DIAG) {  // fixed-order block reduction -> partials (deterministic)
    __shared__ double red[3][CH / 32];
    const int lane = tid & 31, warp = tid >> 5;
    double v[3] = {e_acc, ep_acc, z_acc};
#pragma unroll
    for (int q = 0; q < 3; ++q) {
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) v[q] += __shfl_down_sync(0xffffffffu, v[q], off);
      if (lane == 0) red[q][warp] = v[q];
    }
    SRK_BAR();
    if (tid < SRK_NQ) {
      double s = 0.0;
      const int q = tid == 4 ? 0 : (tid == 5 ? 1 : (tid == 8 ? 2 : -1));
      if (q >= 0)
        for (int w = 0; w < CH / 32; ++w) s += red[q][w];
      a.partial[tid * gridDim.x + blockIdx.x] = s;
    }
  }
}

// K6: f = P[G] - nu k^2 u (physics.py:119-129); Boussinesq adds the buoyancy
// before the projection and the density tendency (physics.py:163-184).
__global__ void k_project(const ProjArgs a) {
  pdl_launch_dependents();
  pdl_wait();
  const GeomArgs& g = a.g;
  const long long n = a.modes;
  const int d = g.dims;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const KVec kv = kvec(i, g);
    cplx G[3];
    for (int j = 0; j < d; ++j) G[j] = a.G[j * n + i];
    cplx rho = make_double2(0.0, 0.0);
    if (a.density) {
      rho = a.y[d * n + i];
      G[d - 1] = rsub(G[d - 1], rmul(a.ri, rho));
    }
    cplx kd = rmul(kv.k[0], G[0]);
    for (int j = 1; j < d; ++j) kd = radd(kd, rmul(kv.k[j], G[j]));
    kd = rmul(kv.inv_k2, kd);
    const double nuk2 = DMUL(a.nu, kv.k2);
    for (int j = 0; j < d; ++j) {
      cplx o = rsub(G[j], rmul(kv.k[j], kd));
      o = rsub(o, rmul(nuk2, a.y[j * n + i]));
      a.f[j * n + i] = o;
    }
    if (a.density) {
      cplx div = rmul(kv.k[0], a.G[d * n + i]);
      for (int j = 1; j < d; ++j) div = radd(div, rmul(kv.k[j], a.G[(d + j) * n + i]));
      cplx o = make_double2(div.y, -div.x);  // -1j * div
      o = rsub(o, rmul(__ddiv_rn(kv.k2, a.re_pr), rho));
      a.f[d * n + i] = o;
    }
  }
}

// spectral.py:47-65
__global__ void k_curl(const GeomArgs g, const cplx* __restrict__ u, cplx* __restrict__ w, long long n) {
  pdl_launch_dependents();
  pdl_wait();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const KVec kv = kvec(i, g);
    auto im = [](cplx z) { return make_double2(-z.y, z.x); };
    if (g.dims == 3) {
      cplx u0 = u[i], u1 = u[n + i], u2 = u[2 * n + i];
      w[i] = im(rsub(rmul(kv.k[1], u2), rmul(kv.k[2], u1)));
      w[n + i] = im(rsub(rmul(kv.k[2], u0), rmul(kv.k[0], u2)));
      w[2 * n + i] = im(rsub(rmul(kv.k[0], u1), rmul(kv.k[1], u0)));
    } else {
      cplx u0 = u[i], u1 = u[n + i];
      w[i] = im(rsub(rmul(kv.k[0], u1), rmul(kv.k[1], u0)));
    }
  }
}

// physics.py:89-102
__global__ void k_leray(const GeomArgs g, const cplx* __restrict__ u, cplx* __restrict__ out, long long n) {
  pdl_launch_dependents();
  pdl_wait();
  const int d = g.dims;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const KVec kv = kvec(i, g);
    cplx kd = make_double2(0.0, 0.0);
    for (int j = 0; j < d; ++j) kd = radd(kd, rmul(kv.k[j], u[j * n + i]));
    kd = rmul(kv.inv_k2, kd);
    for (int j = 0; j < d; ++j) out[j * n + i] = rsub(u[j * n + i], rmul(kv.k[j], kd));
  }
}

// integrators.py:327-339: out = y + sum_j (h a_ij) F_j, ascending j, one rounding
// per multiply and per add (y == nullptr starts from zeros, :343-347).
template <int NT>
__global__ void k_combine(const CombArgs a) {
  pdl_launch_dependents();
  pdl_wait();
  double cf[NT > 0 ? NT : 1];
#pragma unroll
  for (int j = 0; j < NT; ++j) cf[j] = coef(a.c, a.hs, j);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < a.n;
       i += (long long)gridDim.x * blockDim.x) {
    cplx acc = a.y ? a.y[i] : make_double2(0.0, 0.0);
#pragma unroll
    for (int j = 0; j < NT; ++j) acc = radd(acc, rmul(cf[j], a.F[j][i]));
    a.out[i] = acc;
  }
}

void srk_launch_combine(const CombArgs& a, cudaStream_t st) {
  const int threads = 256;
  long long blocks = (a.n + threads - 1) / threads;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  switch (a.nt) {
#define CASE(N) \
  case N: srk_launch_k(k_combine<N>, dim3((int)blocks), dim3(threads), 0, st, a); break;
    CASE(0) CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8)
#undef CASE
    default: break;
  }
}

// ---------------------------------------------------------------------------
// K7: fused step reduction.  Deterministic: fixed grid, per-thread sequential
// sums, fixed shuffle tree, per-block partials summed in fixed order.
//   q[c]   (c < 4) : sum |Delta_c|^2 / sc_c^2      (control.py:51-79)
//   q[4]           : sum_w |y1|^2 over velocity     (diagnostics.py:48-50)
//   q[5]           : sum_w Re(y1 conj fl) velocity  (diagnostics.py:53-70)
//   q[6]           : non-finite entries of Delta / y1 (integrators.py:341-351)
//   q[7]           : count of sc <= 0 (control.py:74-75)
//   q[8]           : sum_w |k|^2 |y1|^2 velocity    (enstrophy)
// ---------------------------------------------------------------------------
// TMA-streamed K7 (default): the up to NT + 3 input streams of a chunk of
// SRK_RT_CH modes are fetched by 1D bulk copies into a two-stage shared-memory
// ring (one elected thread, mbarrier completion), so the memory parallelism no
// longer depends on registers: k_reduce ran at ~40% of the DRAM peak, bound by
// load latency at 24 warps per SM.  Persistent fixed grid + fixed chunk order
// per block + fixed per-thread order -> run-to-run deterministic.
#define SRK_RT_CH 256
#define SRK_RT_BLOCKS 296
static_assert(SRK_RT_BLOCKS <= SRK_RED_BLOCKS, "partials buffer sized by SRK_RED_BLOCKS");

template <int NT>
__global__ void __launch_bounds__(SRK_RT_CH) k_reduce_tma(const RedArgs a) {
  extern __shared__ __align__(128) cplx rsm[];
  srk_poison_smem(rsm);
  constexpr int CH = SRK_RT_CH;
  constexpr int NS = 3 + NT;  // y1, y0, F[0..NT), fl
  __shared__ __align__(8) unsigned long long mb[2];
  const int tid = threadIdx.x;
  const long long n = a.modes;
  const long long cpc = (n + CH - 1) / CH;
  const long long nch = cpc * a.ncomp;
  const int G = gridDim.x;
  double acc[SRK_NQ];
#pragma unroll
  for (int q = 0; q < SRK_NQ; ++q) acc[q] = 0.0;
  double cf[NT > 0 ? NT : 1];
#pragma unroll
  for (int j = 0; j < NT; ++j) cf[j] = coef(a.c, a.hs, j);
  if (tid == 0) {
    mbar_init(&mb[0], 1);
    mbar_init(&mb[1], 1);
    fence_mbar_init();
  }
  pdl_launch_dependents();
  pdl_wait();
  SRK_BAR();
  auto issue = [&](long long k, int b) {
    if (tid != 0 || k >= nch) return;
    const int c = (int)(k / cpc);
    const long long i0 = (k - c * cpc) * CH;
    const unsigned cnt = (unsigned)min((long long)CH, n - i0);
    const long long off = c * n + i0;
    cplx* st = rsm + b * NS * CH;
    const bool vel = c < a.dvel;
    unsigned bytes = cnt * 16u;
    if (a.do_norm) bytes += cnt * 16u * (1u + NT);
    const bool fl_own = a.do_diag && vel && !(a.do_norm && a.fl_term >= 0);  // fl needs its own stream
    if (fl_own) bytes += cnt * 16u;
    mbar_expect_tx(&mb[b], bytes);
    bulk_g2s(st, a.y1 + off, cnt * 16u, &mb[b]);
    if (a.do_norm) {
      bulk_g2s(st + CH, a.y0 + off, cnt * 16u, &mb[b]);
#pragma unroll
      for (int j = 0; j < NT; ++j) bulk_g2s(st + (2 + j) * CH, a.F[j] + off, cnt * 16u, &mb[b]);
    }
    if (fl_own) bulk_g2s(st + (2 + NT) * CH, a.fl + off, cnt * 16u, &mb[b]);
  };
  issue(blockIdx.x, 0);
  issue(blockIdx.x + G, 1);
  unsigned phase = 0;
  for (int it = 0; (long long)blockIdx.x + (long long)it * G < nch; ++it) {
    const long long k = blockIdx.x + (long long)it * G;
    const int b = it & 1;
    const int c = (int)(k / cpc);
    const long long i0 = (k - c * cpc) * CH;
    const int cnt = (int)min((long long)CH, n - i0);
    const bool vel = c < a.dvel;
    mbar_wait(&mb[b], (phase >> b) & 1u);
    phase ^= 1u << b;
    const cplx* st = rsm + b * NS * CH;
    if (tid < cnt) {
      const long long i = i0 + tid;
      const cplx y1 = st[tid];
      double r2 = 0.0;
      if (a.do_norm) {
        cplx dl = make_double2(0.0, 0.0);
#pragma unroll
        for (int j = 0; j < NT; ++j) dl = radd(dl, rmul(cf[j], st[(2 + j) * CH + tid]));
        const cplx y0 = st[CH + tid];
        const double sc = DADD(a.atol, DMUL(fmax(hypot(y0.x, y0.y), hypot(y1.x, y1.y)), a.rtol));
        const double rt = __ddiv_rn(hypot(dl.x, dl.y), sc);
        r2 = DMUL(rt, rt);
        if (!(isfinite(dl.x) && isfinite(dl.y))) acc[6] += 1.0;
        if (sc <= 0.0) acc[7] += 1.0;
      }
      if (!(isfinite(y1.x) && isfinite(y1.y))) acc[6] += 1.0;
#pragma unroll
      for (int cc = 0; cc < 4; ++cc)
        if (cc == c) acc[cc] = DADD(acc[cc], r2);  // static indices only
      if (a.do_diag && vel) {
        const bool small = n < (1LL << 32);
        const int kz = small ? (int)((unsigned)i % (unsigned)a.K) : (int)(i % a.K);
        const double w = (kz == 0 || kz == a.K - 1) ? 1.0 : 2.0;
        const double m2 = DADD(DMUL(y1.x, y1.x), DMUL(y1.y, y1.y));
        acc[4] = DADD(acc[4], DMUL(w, m2));
        const int fslot = (a.do_norm && a.fl_term >= 0) ? 2 + a.fl_term : 2 + NT;
        const cplx fl = st[fslot * CH + tid];
        acc[5] = DADD(acc[5], DMUL(w, DADD(DMUL(y1.x, fl.x), DMUL(y1.y, fl.y))));
        const double k2 = k2_at(i, a.g, small);
        acc[8] = DADD(acc[8], DMUL(DMUL(w, k2), m2));
      }
    }
    SRK_BAR();  // stage b consumed (bulk copies only write it: no proxy fence needed)
    issue(k + 2LL * G, b);
  }
  __shared__ double red[SRK_NQ][CH / 32];
  const int lane = tid & 31, warp = tid >> 5;
#pragma unroll
  for (int q = 0; q < SRK_NQ; ++q) {
    double v = acc[q];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
    if (lane == 0) red[q][warp] = v;
  }
  SRK_BAR();
  if (tid < SRK_NQ) {
    double v = 0.0;
    for (int w = 0; w < CH / 32; ++w) v += red[tid][w];
    a.partial[tid * gridDim.x + blockIdx.x] = v;
  }
}

// One warp per reduced quantity (blockDim = 32 * SRK_NQ): lane l sums partials
// l, l + 32, ... in order, then a fixed xor-shuffle tree -- deterministic, and
// all nine sums proceed at once (the earlier one-block, nine-pass shared-memory
// tree took ~15 us, a visible share of a 2D 1024^2 BS5 attempt).
__global__ void k_finalize(const double* __restrict__ partial, int nblk, double* __restrict__ out) {
  pdl_launch_dependents();
  pdl_wait();
  const int q = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (q >= SRK_NQ) return;
  double v = 0.0;
  for (int i = lane; i < nblk; i += 32) v += partial[q * nblk + i];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  if (lane == 0) out[q] = v;
}

void srk_launch_reduce(const RedArgs& a, double* out, cudaStream_t st) {
  switch (a.nt) {
#define CASE(N)                                                                                      \
  case N: {                                                                                          \
    const int smem = 2 * (3 + N) * SRK_RT_CH * 16;                                                   \
    srk_ensure_smem((const void*)k_reduce_tma<N>, smem);                                             \
    srk_launch_k(k_reduce_tma<N>, dim3(SRK_RT_BLOCKS), dim3(SRK_RT_CH), smem, st, a);                 \
  } break;
    CASE(0) CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8)
#undef CASE
    default: break;
  }
  srk_launch_k(k_finalize, dim3(1), dim3(32 * SRK_NQ), 0, st, (const double*)a.partial, (int)SRK_RT_BLOCKS, out);
}

// ---------------------------------------------------------------------------
// K9 forcing helpers (physics.py:209-239): weighted |u|^2 over a small list of
// band modes (one block, fixed order) and the in-place band rescale.
// ---------------------------------------------------------------------------
__global__ void k_band_energy(const cplx* __restrict__ u, const long long* __restrict__ idx,
                              const double* __restrict__ w, int nb, int ncomp, long long modes,
                              double* __restrict__ out) {
  pdl_launch_dependents();
  pdl_wait();
  __shared__ double sh[256];
  double v = 0.0;
  for (int c = 0; c < ncomp; ++c)
    for (int b = threadIdx.x; b < nb; b += blockDim.x) {
      const cplx z = u[c * modes + idx[b]];
      v = DADD(v, DMUL(w[b], DADD(DMUL(z.x, z.x), DMUL(z.y, z.y))));
    }
  sh[threadIdx.x] = v;
  SRK_BAR();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
    SRK_BAR();
  }
  if (threadIdx.x == 0) out[0] = sh[0];
}

__global__ void k_band_scale(cplx* __restrict__ u, const long long* __restrict__ idx, int nb, int ncomp,
                             long long modes, double gamma) {
  pdl_launch_dependents();
  pdl_wait();
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nb * ncomp) return;
  const int c = t / nb, b = t - (t / nb) * nb;
  cplx* p = u + c * modes + idx[b];
  *p = rmul(gamma, *p);
}

template <int DIMS, bool DENS, int NTC = -1, bool DIAG = false>
static int launch_project_tma(const ProjArgs& a, cudaStream_t st) {
  constexpr int CH = proj_chunk<DIMS, DENS, NTC, DIAG>();
  constexpr int NS = proj_streams<DIMS, DENS, NTC, DIAG>();
  const int smem = 2 * NS * CH * 16;
  const void* fn = (const void*)k_project_tma<DIMS, DENS, NTC, DIAG>;
  srk_ensure_smem(fn, smem);  // per (device, kernel)
  int blocks = srk_blocks_per_sm(fn, CH, smem) * srk_sm_count();
  if (DIAG) blocks = std::min(blocks, SRK_RED_BLOCKS);  // partials buffer
  const long long nch = (a.modes + CH - 1) / CH;
  const int grid = (int)std::min<long long>(blocks, nch);
  srk_launch_k(k_project_tma<DIMS, DENS, NTC, DIAG>, dim3(grid), dim3(CH), smem, st, a);
  return grid;
}

bool srk_launch_project_refresh(const ProjArgs& a, double* out, cudaStream_t st) {
  if (a.modes >= (1LL << 32) || !a.partial) return false;
  int grid;
  if (a.g.dims == 3)
    grid = a.density ? launch_project_tma<3, true, 0, true>(a, st) : launch_project_tma<3, false, 0, true>(a, st);
  else
    grid = a.density ? launch_project_tma<2, true, 0, true>(a, st) : launch_project_tma<2, false, 0, true>(a, st);
  srk_launch_k(k_finalize, dim3(1), dim3(32 * SRK_NQ), 0, st, (const double*)a.partial, grid, out);
  return true;
}

// K6 with the next stage input formed in the same pass (3D / 2D, NS or
// Boussinesq, modes < 2^32, at most SRK_PC_MAXT earlier stages); returns false
// when the shape does not qualify
template <int DIMS, bool DENS>
static void launch_project_comb(const ProjArgs& a, cudaStream_t st) {
  switch (a.nt) {
#define CASE(N) \
  case N: launch_project_tma<DIMS, DENS, N>(a, st); break;
    CASE(0) CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6)
#undef CASE
    default: break;
  }
}
bool srk_launch_project_comb(const ProjArgs& a, cudaStream_t st) {
  if (a.modes >= (1LL << 32) || a.nt < 0 || a.nt > SRK_PC_MAXT) return false;
  if (a.g.dims == 3)
    a.density ? launch_project_comb<3, true>(a, st) : launch_project_comb<3, false>(a, st);
  else
    a.density ? launch_project_comb<2, true>(a, st) : launch_project_comb<2, false>(a, st);
  return true;
}

void srk_launch_project(const ProjArgs& a, cudaStream_t st) {
  if (a.modes < (1LL << 32)) {  // TMA-streamed kernel (32-bit mode indices)
    if (a.g.dims == 3)
      a.density ? launch_project_tma<3, true>(a, st) : launch_project_tma<3, false>(a, st);
    else
      a.density ? launch_project_tma<2, true>(a, st) : launch_project_tma<2, false>(a, st);
    return;
  }
  long long blocks = (a.modes + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  srk_launch_k(k_project, dim3((int)blocks), dim3(256), 0, st, a);
}
void srk_launch_curl(const GeomArgs& g, const cplx* u, cplx* w, long long n, cudaStream_t st) {
  long long blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  srk_launch_k(k_curl, dim3((int)blocks), dim3(256), 0, st, g, u, w, n);
}
void srk_launch_leray(const GeomArgs& g, const cplx* u, cplx* o, long long n, cudaStream_t st) {
  long long blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  srk_launch_k(k_leray, dim3((int)blocks), dim3(256), 0, st, g, u, o, n);
}
void srk_launch_band_energy(const cplx* u, const long long* idx, const double* w, int nb, int ncomp,
                            long long modes, double* out, cudaStream_t st) {
  srk_launch_k(k_band_energy, dim3(1), dim3(256), 0, st, u, idx, w, nb, ncomp, modes, out);
}
__global__ void k_store_mapped(const double* __restrict__ src, double* dst, int n) {
  pdl_launch_dependents();
  pdl_wait();
  for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
}
void srk_launch_store_mapped(const double* src, double* dst, int n, cudaStream_t st) {
  if (n > 0) srk_launch_k(k_store_mapped, dim3(1), dim3(32), 0, st, src, dst, n);
}
void srk_launch_band_scale(cplx* u, const long long* idx, int nb, int ncomp, long long modes, double gamma,
                           cudaStream_t st) {
  const int tot = nb * ncomp;
  if (tot <= 0) return;
  srk_launch_k(k_band_scale, dim3((tot + 127) / 128), dim3(128), 0, st, u, idx, nb, ncomp, modes, gamma);
}
