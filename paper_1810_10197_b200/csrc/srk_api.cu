// libsrk C ABI (include/srk.h): plans, kernel dispatch, RHS / widen / narrow
// pipelines.  See DESIGN.md for the pass structure and the HBM layout.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/srk.h"
#include "pointwise.cuh"
#include "registry.cuh"

// ---------------------------------------------------------------------------
// registry
// ---------------------------------------------------------------------------
void srk_reg_48(KEntry*);
void srk_reg_96(KEntry*);
void srk_reg_192(KEntry*);
void srk_reg_384(KEntry*);
void srk_reg_768(KEntry*);
void srk_reg_1536(KEntry*);
void srk_reg_32(KEntry*);
void srk_reg_64(KEntry*);
void srk_reg_128(KEntry*);
void srk_reg_256(KEntry*);
void srk_reg_512(KEntry*);
void srk_reg_1024(KEntry*);
void srk_reg_generic(KEntry*);

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

struct Table {
  KEntry e[KK_COUNT];
};

std::mutex g_mu;
std::map<int, Table>* g_fast = nullptr;
Table* g_generic = nullptr;

void init_registry() {
  std::lock_guard<std::mutex> lk(g_mu);
  if (g_fast) return;
  auto* m = new std::map<int, Table>();
  struct {
    int M;
    srk_reg_fn f;
  } fs[] = {{48, srk_reg_48},   {96, srk_reg_96},   {192, srk_reg_192}, {384, srk_reg_384},
            {768, srk_reg_768}, {1536, srk_reg_1536}, {32, srk_reg_32}, {64, srk_reg_64},
            {128, srk_reg_128}, {256, srk_reg_256}, {512, srk_reg_512}, {1024, srk_reg_1024}};
  for (auto& x : fs) {
    Table t;
    memset(&t, 0, sizeof(t));
    x.f(t.e);
    (*m)[x.M] = t;
  }
  g_generic = new Table();
  memset(g_generic, 0, sizeof(Table));
  srk_reg_generic(g_generic->e);
  g_fast = m;
}

bool gen_factor(int M, GenPlan& gp) {
  gp.M = M;
  gp.nr = 0;
  int m = M;
  const int rs[] = {8, 4, 2, 3, 5, 7};
  for (int r : rs) {
    while (m % r == 0) {
      if (gp.nr >= 10) return false;
      gp.r[gp.nr++] = r;
      m /= r;
    }
  }
  return m == 1;
}

// Find the kernel for (kind, M): a compile-time plan if one exists, else the
// runtime engine for M <= SRK_GEN_MAXM with factors in {2,3,5,7}.
int get_entry(int kind, int M, KEntry& e, GenPlan& gp) {
  init_registry();
  memset(&gp, 0, sizeof(gp));
  auto it = g_fast->find(M);
  if (it != g_fast->end() && it->second.e[kind].fn) {
    e = it->second.e[kind];
    gp.M = M;
    return SRK_OK;
  }
  if (M <= SRK_GEN_MAXM && gen_factor(M, gp) && g_generic->e[kind].fn) {
    e = g_generic->e[kind];
    return SRK_OK;
  }
  return fail(SRK_ERR_UNSUPPORTED, "FFT length " + std::to_string(M) +
                                       " has no sm_100a plan (supported: 3*2^k and 2^k up to 1536, or "
                                       "<= 96 with factors 2,3,5,7)");
}

int ensure_smem(const KEntry& e) {
  cudaError_t err = srk_ensure_smem(e.fn, e.smem);  // per (device, kernel)
  if (err != cudaSuccess) return fail(SRK_ERR_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(err));
  return SRK_OK;
}

int check_launch(const char* what) {
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) return fail(SRK_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(err));
  return SRK_OK;
}

}  // namespace

// ---------------------------------------------------------------------------
// plan
// ---------------------------------------------------------------------------
struct srk_plan {
  int dims, density, max_comps;
  int n0, n1, n2, K, m0, m1, m2;  // 2D: n1 = m1 = 1 and n2 = last axis
  double ck0, ck1, ck2;
  long long modes;  // n0*n1*K per component
  int S, So;        // rhs signal counts (widened, products)
  int S1;           // 3D: K1 output signals [u0,u1,u2,kx u1,kx u2,(rho)]; 2D: S
  int nranks = 1, rank = 0;  // slab decomposition over y (3D only)
  int n1g = 0, y0 = 0, Mx = 0;
  std::map<int, cplx*> tw;
  long long A_elems = 0, B_elems = 0;
  char* ws = nullptr;
  long long ws_bytes = 0, need_bytes = 0;
  cplx* A = nullptr;
  cplx* B = nullptr;
  double* partial = nullptr;
  int last_launches = 0;
  // optional per-kernel timing of srk_rhs (srk_rhs_timed)
  bool timing = false;
  unsigned long long* dbg = nullptr;  // phase timestamps (srk_debug_phase_buffer)
  int dbg_launch = -1;                // ... recorded by this launch of the chain
  cudaEvent_t ev[16];
  int nev = 0;
  cudaStream_t tstream = nullptr;
  // slab exchange fused into K1 / K4 (srk_slab_set_peers): every rank's
  // all-to-all #1 / #2 receive buffer, indexed by rank (UVA / CUDA IPC pointers)
  cplx* peer1[SRK_MAX_PEERS] = {};
  cplx* peer2[SRK_MAX_PEERS] = {};
  bool peers_set = false;
};

namespace {

long long align256(long long b) { return (b + 255) / 256 * 256; }

int get_tw(srk_plan* p, int M, const cplx** out) {
  auto it = p->tw.find(M);
  if (it != p->tw.end()) {
    *out = it->second;
    return SRK_OK;
  }
  std::vector<double2> h(M);
  for (int e = 0; e < M; ++e) {
    // exp(-2 pi i e / M) with the angle reduced exactly in integers, long double math
    const long double ang = 2.0L * 3.14159265358979323846264338327950288L * (long double)e / (long double)M;
    h[e] = make_double2((double)cosl(ang), (double)-sinl(ang));
  }
  cplx* d = nullptr;
  cudaError_t err = cudaMalloc(&d, sizeof(cplx) * M);
  if (err != cudaSuccess) return fail(SRK_ERR_CUDA, std::string("cudaMalloc(twiddles): ") + cudaGetErrorString(err));
  err = cudaMemcpy(d, h.data(), sizeof(cplx) * M, cudaMemcpyHostToDevice);
  if (err != cudaSuccess) return fail(SRK_ERR_CUDA, std::string("cudaMemcpy(twiddles): ") + cudaGetErrorString(err));
  p->tw[M] = d;
  *out = d;
  return SRK_OK;
}

int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return (v && *v) ? atoi(v) : dflt;
}

// Layout of the RHS intermediates of unsplit fast plans (rhs_impl):
//  * pencil pitch Kp = K rounded up to 4 complex: K = n2/2 + 1 is odd, so with pitch K
//    every other row of a y pass starts 16 B into a 32 B sector and its 64 B tile pieces
//    are partial-sector writes (K2's stores ran at 3.1 TB/s; 7.7 TB/s with an even pitch);
//  * the x-padded buffers (K1 -> K2, K4 -> K5) y-blocked, [yb][signal][x][y in block][kz],
//    when a plain x row reaches 1 MB: an x-pass tile then spans ~100 instead of m0 2 MB
//    pages per signal (the plain order thrashes the TLB).
// SRK_KPAD=0 / SRK_YB=0 switch them off (A/B timing); both 0 for every other plan.
bool rhs_fast(const srk_plan* p) {  // unsplit plan on the compile-time FFT plans, 32-bit mode indices
  init_registry();
  return p->nranks == 1 && p->modes < (1LL << 32) && g_fast->count(p->m0) && g_fast->count(p->m2) &&
         (p->dims == 2 || g_fast->count(p->m1));
}
// (K >= 128, i.e. n2 >= 256: below that the rows are short, K6 needs several row
// segments per 256-mode chunk and the padding costs more than it gains -- 32^3 ... 128^3
// measured 0.5-5 % slower padded, 256^3 0.8 %, 512^3 1.7 % faster)
int pitch_of(int K) { return K >= 128 ? ((K + 3) & ~3) : K; }
int rhs_pitch(const srk_plan* p) {
  static const int env_kpad = env_int("SRK_KPAD", 1);
  return (env_kpad && rhs_fast(p)) ? pitch_of(p->K) : p->K;
}
// Slab plans: the rank-local K2 -> K3 -> K4 buffers get the padded pitch too (the
// exchange buffers keep the all-to-all layouts at pitch K).
int slab_pitch(const srk_plan* p) {
  static const int env_kpad = env_int("SRK_KPAD", 1);
  init_registry();
  const bool fast = g_fast->count(p->m0) && g_fast->count(p->m1) && g_fast->count(p->m2);
  return (env_kpad && p->dims == 3 && fast) ? pitch_of(p->K) : p->K;
}
int rhs_yblock(const srk_plan* p) {
  static const int env_yb = env_int("SRK_YB", -1);
  if (p->dims != 3 || !rhs_fast(p)) return 0;
  int yb = env_yb >= 0 ? env_yb : ((long long)p->n1 * p->K * 16 >= (1 << 20) ? 64 : 0);
  if (yb <= 0 || yb >= p->n1 || p->n1 % yb) return 0;
  return yb;
}

int need_ws(srk_plan* p) {
  if (!p->A) return fail(SRK_ERR_WORKSPACE, "plan has no workspace bound (srk_plan_set_workspace)");
  return SRK_OK;
}

// ---- strided pass launch -------------------------------------------------
int curly_xblk(int X) { return X % 2 == 0 ? 2 : 1; }

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link).
typedef CUresult (*srk_encode_tiled_fn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                         const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                         CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                         CUtensorMapFloatOOBfill);
srk_encode_tiled_fn encode_tiled() {
  static srk_encode_tiled_fn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return (srk_encode_tiled_fn) nullptr;
    return (srk_encode_tiled_fn)f;
  }();
  return fn;
}

CUtensorMapL2promotion promo() { return CU_TENSOR_MAP_L2_PROMOTION_L2_256B; }

// Tensor map of a strided pass's input: 4D {2*kc doubles, ngrp column groups,
// rows, planes} based at the chunk's first column, box {2*C, 1, rows/nb <= 256,
// 1}.  Leaves a.tma = 0 when TMA does not apply (generic lengths, blocked slab
// rows, 2D curl kinds, box constraints).
// wcols: columns the map covers per group (a.kc, or the padded store width).
bool encode_pass_map(CUtensorMap* tm, const cplx* base, const PassArgs& a, long long kst, long long rs,
                     long long pst, int rows, int box, int cols, CUtensorMapL2promotion pr, int rpb = 0,
                     long long bstride = 0, int wcols = 0) {
  srk_encode_tiled_fn enc = encode_tiled();
  if (!enc) return false;
  if (wcols <= 0) wcols = a.kc;
  const cuuint64_t ks = (cuuint64_t)(a.ngrp > 1 ? kst : a.kc) * 16;
  if (rpb > 0 && a.ngrp == 1) {  // rank 4: {columns, row in block, block, plane} (a.tma = 2)
    cuuint64_t dims[4] = {(cuuint64_t)(2 * wcols), (cuuint64_t)rpb, (cuuint64_t)(rows / rpb), (cuuint64_t)a.planes};
    cuuint64_t strides[3] = {(cuuint64_t)rs * 16, (cuuint64_t)bstride * 16, (cuuint64_t)pst * 16};
    cuuint32_t boxd[4] = {(cuuint32_t)(2 * cols), (cuuint32_t)(box < rpb ? box : rpb),
                          (cuuint32_t)(box < rpb ? 1 : box / rpb), 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    return enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, (void*)base, dims, strides, boxd, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, pr,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  }
  if (rpb > 0) {  // rank 5: {columns, column groups, row in block, block, plane}
    cuuint64_t dims[5] = {(cuuint64_t)(2 * wcols), (cuuint64_t)a.ngrp, (cuuint64_t)rpb, (cuuint64_t)(rows / rpb),
                          (cuuint64_t)a.planes};
    cuuint64_t strides[4] = {ks, (cuuint64_t)rs * 16, (cuuint64_t)bstride * 16, (cuuint64_t)pst * 16};
    // a box covers `box` rows: part of one block, or whole blocks (box a multiple of rpb)
    cuuint32_t boxd[5] = {(cuuint32_t)(2 * cols), 1, (cuuint32_t)(box < rpb ? box : rpb),
                          (cuuint32_t)(box < rpb ? 1 : box / rpb), 1};
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    return enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, (void*)base, dims, strides, boxd, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, pr,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  }
  // rank 4: {columns, column groups, rows, plane}
  cuuint64_t dims[4] = {(cuuint64_t)(2 * wcols), (cuuint64_t)a.ngrp, (cuuint64_t)rows, (cuuint64_t)a.planes};
  cuuint64_t strides[3] = {ks, (cuuint64_t)rs * 16, (cuuint64_t)pst * 16};
  cuuint32_t boxd[4] = {(cuuint32_t)(2 * cols), 1, (cuuint32_t)box, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, (void*)base, dims, strides, boxd, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, pr,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

void setup_tma(int kind, int cols, PassArgs& a, CUtensorMap* tm) {
  a.tma = 0;
  const bool inv = kind == KK_INV || kind == KK_INV_P || kind == KK_INV_KX || kind == KK_INV_KX_SLAB ||
                   kind == KK_INV_KX_PEER ||
                   kind == KK_INV_CURLY;
  const bool fwd = kind == KK_FWD || kind == KK_FWD_P || kind == KK_FWD_P_SLABO || kind == KK_FWD_P_SLABI ||
                   kind == KK_FWD_P_PEER ||
                   kind == KK_FWD_P2D;
  const bool slab_in = kind == KK_INV_CURLY_SLAB || kind == KK_INV_P_SLAB;  // blocked input rows
  if (!(inv || fwd || slab_in) || !g_fast->count(a.M)) return;
  if ((kind == KK_INV_KX || kind == KK_INV_KX_SLAB || kind == KK_INV_KX_PEER) && a.comp_stride != a.in_plane_stride)
    return;
  const int rows = fwd ? a.M : a.n;
  const int rb = a.in_rpb > 0 ? a.in_rpb : rows;
  if (rows % rb) return;
  // rows per box (<= 256): a divisor of a row block, or -- small blocks (the
  // y-blocked RHS intermediates) -- as many whole blocks as fit
  int box;
  if (a.in_rpb > 0 && rb <= 128) {
    int k = 256 / rb;
    while (k > 1 && (rows / rb) % k) --k;
    box = k * rb;
  } else {
    const int nb = (rb + 255) / 256;
    if (rb % nb) return;
    box = rb / nb;
  }
  if (!encode_pass_map(tm, a.in + a.in_k0, a, a.in_kst, a.in_rs, a.in_plane_stride, rows, box, cols, promo(),
                       a.in_rpb, a.in_bstride))
    return;
  a.tma = (a.in_rpb > 0 && a.ngrp == 1) ? 2 : 1;  // 2: blocked rows through the rank-4 map
  a.tma_rows = box;
}

// Output tensor map of the 3D K2 pass (y inverse): {2*Qp doubles, M rows,
// planes}, box {2*C, M/nb <= 256, 1} (plain output rows only).
void setup_tma_out(int kind, int cols, PassArgs& a, CUtensorMap* tm) {
  a.tma_out = 0;
  const bool inv = kind == KK_INV_CURLY || kind == KK_INV_CURLY_SLAB;  // see kTMAO in k_colpass
  if (!inv || a.out_rpb != 0 || !g_fast->count(a.M)) return;
  const int nb = (a.M + 255) / 256;
  if (a.M % nb) return;
  const int box = a.M / nb;
  // the map ends at the chunk's last column: partial tiles are clipped, so a
  // chunk never writes its neighbour's columns
  if (!encode_pass_map(tm, a.out + a.out_k0, a, a.out_kst, a.out_rs, a.out_plane_stride, a.M, box, cols,
                       CU_TENSOR_MAP_L2_PROMOTION_NONE, 0, 0, a.kc_out > a.kc ? a.kc_out : 0))
    return;
  a.tma_out = 1;
  a.tmo_rows = box;
}

// Column-group defaults (unchunked passes) and tile counts.
void normalise_cols(PassArgs& a, int cols) {
  if (a.kc == 0) {
    a.kc = a.Qp;
    a.ngrp = 1;
    a.in_kst = a.out_kst = 0;
    a.in_k0 = a.out_k0 = a.kz0 = 0;
  }
  if (a.in_rs == 0) a.in_rs = a.row_stride;
  if (a.out_rs == 0) a.out_rs = a.row_stride;
  a.tpg = (a.kc + cols - 1) / cols;
  a.tpp = a.ngrp * a.tpg;
}

// NS3 z-pass L2 warm-up distance: one wave of resident CTAs (2 per SM); measured
// 9.48 -> 9.24 ms at 512^3.  One-pencil kernels recompute it from their own
// occupancy in launch_z.
int zpass_prefetch_distance() { return 2 * srk_sm_count(); }

int launch_col(srk_plan* p, int kind, PassArgs a, cudaStream_t st) {
  const bool padded_kind = kind == KK_INV_P || kind == KK_FWD_P || kind == KK_INV_RHS || kind >= KK_INV_RHS_SLAB;
  if (padded_kind && 3 * a.n != 2 * a.M) return fail(SRK_ERR_INVALID, "padded pass needs M = 3n/2");
  KEntry e;
  int rc = get_entry(kind, a.M, e, a.gp);
  if (rc) return rc;
  a.dbg = (p->dbg && p->last_launches == p->dbg_launch) ? p->dbg : nullptr;
  if ((rc = get_tw(p, a.M, &a.tw))) return rc;
  normalise_cols(a, e.cols);
  auto magic = [](int rpb) { return rpb > 1 ? 0xFFFFFFFFu / (unsigned)rpb + 1u : 0u; };
  a.in_magic = magic(a.in_rpb);
  a.out_magic = magic(a.out_rpb);
  const long long ntiles = (long long)a.planes * a.tpp;
  if (ntiles <= 0) return SRK_OK;
  if (ntiles > 0x7fffffffLL) return fail(SRK_ERR_INVALID, "strided pass: too many tiles");
  alignas(64) CUtensorMap tm;
  memset(&tm, 0, sizeof(tm));
  setup_tma(kind, e.cols, a, &tm);
  const long long grid = ntiles;
  alignas(64) CUtensorMap tmo;
  memset(&tmo, 0, sizeof(tmo));
  setup_tma_out(kind, e.cols, a, &tmo);
  if ((rc = ensure_smem(e))) return rc;
  // access-pattern probes (measurement only, tools/pass_probe.sh): 1 = stage the tile and
  // return, 2 = also store in the output pattern, no transform
  static const int probe_fwd = env_int("SRK_PROBE_FWD", 0), probe_inv = env_int("SRK_PROBE_INV", 0);
  a.probe = 0;
  if (a.tma && (kind == KK_FWD_P || kind == KK_FWD_P_SLABO)) a.probe = probe_fwd;
  if (a.tma && (kind == KK_INV_KX || kind == KK_INV_CURLY || kind == KK_INV_CURLY_SLAB)) a.probe = probe_inv;
  void* args[] = {&a, &tm, &tmo};
  cudaError_t err = srk_launch(e.fn, dim3((unsigned)grid), dim3(e.nt), args, e.smem, st);
  if (err != cudaSuccess) return fail(SRK_ERR_CUDA, std::string("colpass launch: ") + cudaGetErrorString(err));
  p->last_launches++;
  if (p->timing && p->nev < 16) cudaEventRecord(p->ev[p->nev++], st);
  return SRK_OK;
}

// ---- z pass launch (pairs of pencils) ---------------------------------------
int launch_z(srk_plan* p, int kind, ZArgs a, int S_rt, int So_rt, cudaStream_t st) {
  KEntry e;
  int rc = get_entry(kind, a.M, e, a.gp);
  if (rc) return rc;
  if ((rc = get_tw(p, a.M, &a.tw))) return rc;
  if ((rc = ensure_smem(e))) return rc;
  int grid = e.ppc == 1 ? a.P : (a.P + 1) / 2;
  static const int probe_z = env_int("SRK_PROBE_Z", 0);
  a.mode = (e.ppc == 1 && kind == KK_Z_NS3) ? probe_z : 0;
  if (e.ppc == 1 && a.pf_dist)  // L2 warm-up one wave of resident CTAs ahead (in pencils)
    a.pf_dist = srk_blocks_per_sm(e.fn, e.nt, e.smem) * srk_sm_count();
  void* args[] = {&a, &S_rt, &So_rt};
  cudaError_t err = srk_launch(e.fn, dim3(grid), dim3(e.nt), args, e.smem, st);
  if (err != cudaSuccess) return fail(SRK_ERR_CUDA, std::string("zpass launch: ") + cudaGetErrorString(err));
  p->last_launches++;
  if (p->timing && p->nev < 16) cudaEventRecord(p->ev[p->nev++], st);
  return SRK_OK;
}

GeomArgs geom(const srk_plan* p) {
  GeomArgs g;
  g.dims = p->dims;
  g.n0 = p->n0;
  g.n1 = p->n1;
  g.K = p->K;
  g.ck0 = p->ck0;
  g.ck1 = p->ck1;
  g.ck2 = p->ck2;
  g.y0 = p->y0;
  g.n1g = p->n1g;
  return g;
}

PassArgs base_pass() {
  PassArgs a;
  memset(&a, 0, sizeof(a));
  a.scale = 1.0;
  return a;
}

// x pass: planes = signals, columns = (y, kz) flattened
PassArgs x_pass(const srk_plan* p, const cplx* in, cplx* out, int nsig, int n_in_rows, int n_out_rows, int M,
                int n) {
  PassArgs a = base_pass();
  a.in = in;
  a.out = out;
  a.M = M;
  a.n = n;
  a.planes = nsig;
  a.Qp = p->n1 * p->K;
  a.sig_minor = 1;
  a.row_stride = (long long)p->n1 * p->K;
  a.in_plane_stride = (long long)n_in_rows * a.row_stride;
  a.out_plane_stride = (long long)n_out_rows * a.row_stride;
  return a;
}

// y pass (3D): planes = (signal, x), columns = kz
PassArgs y_pass(const srk_plan* p, const cplx* in, cplx* out, int nsig, int xrows, int n_in_rows,
                int n_out_rows, int M, int n) {
  PassArgs a = base_pass();
  a.in = in;
  a.out = out;
  a.M = M;
  a.n = n;
  a.planes = nsig * xrows;
  a.Qp = p->K;
  a.sig_minor = 0;
  a.row_stride = p->K;
  a.in_plane_stride = (long long)n_in_rows * p->K;
  a.out_plane_stride = (long long)n_out_rows * p->K;
  return a;
}

ZArgs z_args(const srk_plan* p, int M, int n, int P) {
  ZArgs z;
  memset(&z, 0, sizeof(z));
  z.M = M;
  z.n = n;
  z.K = p->K;
  z.P = P;
  return z;
}

// inverse 3/2-padded (pad=true) or plain (pad=false) transform of c signals:
// spec (c, n0, n1, K) -> phys (c, M0, M1, M2)
int inverse_chain(srk_plan* p, const cplx* spec, int c, double* phys, bool pad, cudaStream_t st) {
  const int M0 = pad ? p->m0 : p->n0, M1 = pad ? p->m1 : p->n1, M2 = pad ? p->m2 : p->n2;
  const double scale = (pad ? std::pow(1.5, p->dims) : 1.0) / ((double)M0 * M1 * M2);
  PassArgs a = x_pass(p, spec, p->A, c, p->n0, M0, M0, p->n0);
  a.scale = scale;
  int rc = launch_col(p, pad ? KK_INV_P : KK_INV, a, st);
  if (rc) return rc;
  const cplx* zin = p->A;
  if (p->dims == 3) {
    PassArgs b = y_pass(p, p->A, p->B, c, M0, p->n1, M1, M1, p->n1);
    if ((rc = launch_col(p, pad ? KK_INV_P : KK_INV, b, st))) return rc;
    zin = p->B;
  }
  const int P = M0 * M1;
  for (int s0 = 0; s0 < c; s0 += SRK_Z_PLAIN_C) {
    const int sc = std::min(SRK_Z_PLAIN_C, c - s0);
    ZArgs z = z_args(p, M2, p->n2, P);
    z.in_sig_stride = (long long)P * p->K;
    z.out_sig_stride = (long long)P * M2;
    z.in = zin + s0 * z.in_sig_stride;
    z.out_real = phys + s0 * z.out_sig_stride;
    if ((rc = launch_z(p, KK_Z_C2R, z, sc, 0, st))) return rc;
  }
  return SRK_OK;
}

// forward (narrow when trunc=true, plain rfftn otherwise): phys -> spec
int forward_chain(srk_plan* p, const double* phys, int c, cplx* spec, bool trunc, cudaStream_t st) {
  const int M0 = trunc ? p->m0 : p->n0, M1 = trunc ? p->m1 : p->n1, M2 = trunc ? p->m2 : p->n2;
  const int P = M0 * M1;
  int rc;
  for (int s0 = 0; s0 < c; s0 += SRK_Z_PLAIN_C) {
    const int sc = std::min(SRK_Z_PLAIN_C, c - s0);
    ZArgs z = z_args(p, M2, p->n2, P);
    z.in_sig_stride = (long long)P * M2;
    z.out_sig_stride = (long long)P * p->K;
    z.in_real = phys + s0 * z.in_sig_stride;
    z.out = p->A + s0 * z.out_sig_stride;
    z.zero_nyq = trunc ? 1 : 0;
    if ((rc = launch_z(p, KK_Z_R2C, z, 0, sc, st))) return rc;
  }
  const cplx* xin = p->A;
  if (p->dims == 3) {
    PassArgs b = y_pass(p, p->A, p->B, c, M0, M1, p->n1, M1, p->n1);
    b.zero_nyq = trunc ? 1 : 0;
    if ((rc = launch_col(p, trunc ? KK_FWD_P : KK_FWD, b, st))) return rc;
    xin = p->B;
  }
  PassArgs a = x_pass(p, xin, spec, c, M0, p->n0, M0, p->n0);
  a.scale = trunc ? std::pow(1.0 / 1.5, p->dims) : 1.0;
  a.zero_nyq = trunc ? 1 : 0;
  a.zero_dc_imag = trunc ? 1 : 0;
  return launch_col(p, trunc ? KK_FWD_P : KK_FWD, a, st);
}

}  // namespace

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
extern "C" {

int srk_abi_version(void) { return 1; }

#ifndef SRK_SRC_HASH
#define SRK_SRC_HASH "unknown"
#endif
const char* srk_source_hash(void) { return SRK_SRC_HASH; }

int srk_plan_layout(const srk_plan* p, int* pitch, int* yblock) {
  if (!p || !pitch || !yblock) return fail(SRK_ERR_INVALID, "null argument");
  *pitch = p->nranks == 1 ? rhs_pitch(p) : slab_pitch(p);
  *yblock = rhs_yblock(p);
  return SRK_OK;
}

int srk_build_info(void) {
#ifdef SRK_DEBUG_CHECKS
  return 1;  // hazard-probe build (schedule fuzzing, NaN-poisoned shared memory, asserts)
#else
  return 0;
#endif
}

const char* srk_last_error(void) { return g_err.c_str(); }

int srk_plan_create(srk_plan** out, int dims, const int64_t* shape, const double* lengths, int density,
                    int max_comps) {
  if (!out) return fail(SRK_ERR_INVALID, "null plan pointer");
  *out = nullptr;
  if (dims != 2 && dims != 3) return fail(SRK_ERR_INVALID, "grid must be 2D or 3D, got " + std::to_string(dims) + " axes");
  for (int i = 0; i < dims; ++i) {
    if (shape[i] < 4 || shape[i] % 2)
      return fail(SRK_ERR_INVALID, "grid extent " + std::to_string(shape[i]) + " must be even and >= 4");
    if (!(lengths[i] > 0)) return fail(SRK_ERR_INVALID, "domain lengths must be positive");
  }
  srk_plan* p = new srk_plan();
  p->dims = dims;
  p->density = density ? 1 : 0;
  const double two_pi = 2.0 * 3.141592653589793;
  if (dims == 3) {
    p->n0 = (int)shape[0];
    p->n1 = (int)shape[1];
    p->n2 = (int)shape[2];
    p->ck0 = two_pi / lengths[0];
    p->ck1 = two_pi / lengths[1];
    p->ck2 = two_pi / lengths[2];
  } else {
    p->n0 = (int)shape[0];
    p->n1 = 1;
    p->n2 = (int)shape[1];
    p->ck0 = two_pi / lengths[0];
    p->ck1 = 0.0;
    p->ck2 = two_pi / lengths[1];
  }
  p->K = p->n2 / 2 + 1;
  p->n1g = p->n1;
  p->m0 = 3 * p->n0 / 2;
  p->m1 = dims == 3 ? 3 * p->n1 / 2 : 1;
  p->m2 = 3 * p->n2 / 2;
  p->modes = (long long)p->n0 * p->n1 * p->K;
  const int d = dims, wc = dims == 3 ? 3 : 1;
  p->S = d + wc + p->density;
  p->So = p->density ? 2 * d : d;
  p->S1 = dims == 3 ? 5 + p->density : p->S;
  const int nstate = d + p->density;
  p->max_comps = std::max(max_comps, nstate);
  // every padded length must have a kernel
  {
    KEntry e;
    GenPlan gp;
    int lens[3] = {p->m0, p->m1, p->m2};
    for (int i = 0; i < 3; ++i) {
      if (lens[i] == 1) continue;
      int rc = get_entry(i == 2 ? KK_Z_C2R : KK_INV, lens[i], e, gp);
      if (rc) {
        delete p;
        return rc;
      }
    }
  }
  // workspace regions (complex elements)
  const long long K = p->K, n0 = p->n0, n1 = p->n1, m0 = p->m0, m1 = p->m1;
  const long long c = std::max<long long>(p->max_comps, 1);
  long long A = 0, B = 0;
  auto upA = [&](long long v) { A = std::max(A, v); };
  auto upB = [&](long long v) { B = std::max(B, v); };
  if (dims == 3) {
    const long long Kp = rhs_pitch(p);  // padded pencil pitch of the RHS intermediates
    upA(p->S1 * m0 * n1 * K);   // K1 out
    upB(p->S * m0 * m1 * Kp);   // K2 out
    upA(p->So * m0 * m1 * Kp);  // K3 out
    upB(p->So * m0 * n1 * Kp);  // K4 out
    upA(p->So * n0 * n1 * Kp);  // K5 out (G)
    upA(c * m0 * n1 * K);
    upB(c * m0 * m1 * K);
    upA(c * m0 * m1 * K);
    upB(c * m0 * n1 * K);
  } else {
    const long long Kp = rhs_pitch(p);
    upA(p->S * m0 * Kp);
    upB(p->So * m0 * Kp);
    upA(p->So * n0 * Kp);
    upA(c * m0 * K);
  }
  p->A_elems = A;
  p->B_elems = B;
  p->need_bytes = align256(A * 16) + align256(std::max<long long>(B, 1) * 16);
  {
    cudaError_t err = cudaMalloc(&p->partial, sizeof(double) * SRK_NQ * SRK_RED_BLOCKS);
    if (err != cudaSuccess) {
      delete p;
      return fail(SRK_ERR_CUDA, std::string("cudaMalloc(partials): ") + cudaGetErrorString(err));
    }
  }
  *out = p;
  return SRK_OK;
}

void srk_plan_destroy(srk_plan* p) {
  if (!p) return;
  for (auto& kv : p->tw) cudaFree(kv.second);
  if (p->partial) cudaFree(p->partial);
  delete p;
}

int srk_plan_workspace_bytes(const srk_plan* p, int64_t* bytes) {
  if (!p || !bytes) return fail(SRK_ERR_INVALID, "null argument");
  *bytes = p->need_bytes;
  return SRK_OK;
}

int srk_plan_set_workspace(srk_plan* p, void* ptr, int64_t bytes) {
  if (!p) return fail(SRK_ERR_INVALID, "null plan");
  if (bytes < p->need_bytes)
    return fail(SRK_ERR_WORKSPACE, "workspace too small: " + std::to_string(bytes) + " < " + std::to_string(p->need_bytes));
  if (((uintptr_t)ptr) % 256) return fail(SRK_ERR_WORKSPACE, "workspace must be 256-byte aligned");
  char* b = (char*)ptr;
  p->ws = b;
  p->ws_bytes = bytes;
  p->A = (cplx*)b;
  b += align256(p->A_elems * 16);
  p->B = (cplx*)b;
  return SRK_OK;
}

namespace {
// next-stage accumulation carried by one RHS call (srk_rhs_combine)
struct CombSpec {
  const cplx* yb;
  int nt;
  const cplx* F[SRK_MAX_TERMS];
  double c[SRK_MAX_TERMS];
  double cself;
  cplx* ynext;
  double* diag_out;  // srk_rhs_refresh: (E, eps, Z) sums of (y, f) -> out[4], [5], [8]
  const double* hs;  // non-null: coefficients are multiples of the device step size *hs
};
int rhs_impl(srk_plan* p, const void* y_, void* f_, double nu, double ri, double re_pr, void* stream,
             const CombSpec* cs);
}  // namespace

int srk_rhs(srk_plan* p, const void* y_, void* f_, double nu, double ri, double re_pr, void* stream) {
  return rhs_impl(p, y_, f_, nu, ri, re_pr, stream, nullptr);
}

namespace {
int rhs_combine_impl(srk_plan* p, const void* y, void* f, double nu, double ri, double re_pr, const void* ybase,
                     int nterms, const void* const* F, const double* coef, double coef_self, const double* hs,
                     void* ynext, void* stream);
}

int srk_rhs_combine(srk_plan* p, const void* y, void* f, double nu, double ri, double re_pr, const void* ybase,
                    int nterms, const void* const* F, const double* coef, double coef_self, void* ynext,
                    void* stream) {
  return rhs_combine_impl(p, y, f, nu, ri, re_pr, ybase, nterms, F, coef, coef_self, nullptr, ynext, stream);
}

int srk_rhs_combine_scaled(srk_plan* p, const void* y, void* f, double nu, double ri, double re_pr,
                           const void* ybase, int nterms, const void* const* F, const double* a, double a_self,
                           const double* h_dev, void* ynext, void* stream) {
  if (!h_dev) return fail(SRK_ERR_INVALID, "srk_rhs_combine_scaled: null step-size pointer");
  return rhs_combine_impl(p, y, f, nu, ri, re_pr, ybase, nterms, F, a, a_self, h_dev, ynext, stream);
}

namespace {
int rhs_combine_impl(srk_plan* p, const void* y, void* f, double nu, double ri, double re_pr, const void* ybase,
                     int nterms, const void* const* F, const double* coef, double coef_self, const double* hs,
                     void* ynext, void* stream) {
  if (nterms < 0 || nterms + 1 > SRK_MAX_TERMS) return fail(SRK_ERR_INVALID, "srk_rhs_combine: at most 7 terms");
  if (!ynext || ynext == y || ynext == f) return fail(SRK_ERR_INVALID, "srk_rhs_combine: ynext must not alias y or f");
  CombSpec cs;
  memset(&cs, 0, sizeof(cs));
  cs.yb = (const cplx*)ybase;
  cs.nt = nterms;
  for (int j = 0; j < nterms; ++j) {
    if (F[j] == ynext) return fail(SRK_ERR_INVALID, "srk_rhs_combine: ynext must not alias a term");
    cs.F[j] = (const cplx*)F[j];
    cs.c[j] = coef[j];
  }
  cs.cself = coef_self;
  cs.ynext = (cplx*)ynext;
  cs.hs = hs;
  return rhs_impl(p, y, f, nu, ri, re_pr, stream, &cs);
}
}  // namespace

int srk_rhs_refresh(srk_plan* p, const void* y, void* f, double nu, double ri, double re_pr, double coef_self,
                    void* ynext, double* diag_out, void* stream) {
  if (!p) return fail(SRK_ERR_INVALID, "null plan");
  if (p->nranks != 1) return fail(SRK_ERR_UNSUPPORTED, "srk_rhs_refresh: unsplit plans only");
  if (!ynext || !diag_out || ynext == y || ynext == f) return fail(SRK_ERR_INVALID, "srk_rhs_refresh: bad outputs");
  if (!p->partial) {
    cudaError_t err = cudaMalloc(&p->partial, sizeof(double) * SRK_NQ * SRK_RED_BLOCKS);
    if (err != cudaSuccess) return fail(SRK_ERR_CUDA, std::string("cudaMalloc(partials): ") + cudaGetErrorString(err));
  }
  CombSpec cs;
  memset(&cs, 0, sizeof(cs));
  cs.yb = (const cplx*)y;
  cs.cself = coef_self;
  cs.ynext = (cplx*)ynext;
  cs.diag_out = diag_out;
  return rhs_impl(p, y, f, nu, ri, re_pr, stream, &cs);
}

namespace {
// unfused tail of srk_rhs_combine: ynext = yb + sum c F + cself f (k_combine)
int comb_after(srk_plan* p, const CombSpec* cs, const cplx* f, cudaStream_t st) {
  CombArgs a;
  memset(&a, 0, sizeof(a));
  a.y = cs->yb;
  for (int j = 0; j < cs->nt; ++j) {
    a.F[j] = cs->F[j];
    a.c[j] = cs->c[j];
  }
  a.F[cs->nt] = f;
  a.c[cs->nt] = cs->cself;
  a.hs = cs->hs;
  a.nt = cs->nt + 1;
  a.out = cs->ynext;
  a.n = (long long)(p->dims + (p->density ? 1 : 0)) * p->modes;
  srk_launch_combine(a, st);
  p->last_launches++;
  return check_launch("k_combine");
}

int rhs_impl(srk_plan* p, const void* y_, void* f_, double nu, double ri, double re_pr, void* stream,
             const CombSpec* cs) {
  if (!p) return fail(SRK_ERR_INVALID, "null plan");
  int rc = need_ws(p);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  const cplx* y = (const cplx*)y_;
  cplx* f = (cplx*)f_;
  p->last_launches = 0;
  const int d = p->dims;
  // K1: x pad + inverse x (3D: [u, kx u1, kx u2] -- the curl is completed in K2;
  // 2D: curl on load)
  PassArgs a = x_pass(p, y, p->A, p->S1, p->n0, p->m0, p->m0, p->n0);
  a.scale = std::pow(1.5, d) / ((double)p->m0 * p->m1 * p->m2);
  a.dims = d;
  a.n1 = p->n1;
  a.K = p->K;
  a.ck0 = p->ck0;
  a.ck1 = p->ck1;
  a.ck2 = p->ck2;
  a.comp_stride = p->modes;
  a.y0 = p->y0;
  a.n1g = p->n1g;
  // layout of the intermediates (rhs_pitch / rhs_yblock):
  //   X1 (K1 -> K2)           [yb][s][x][yi][kz]   pitch K (K1's flattened (y, kz) tiles stay
  //                                                64 B-aligned on the state and on X1)
  //   K2 -> K3 -> K4          [s][x][y][kz]        pitch Kp
  //   X2 (K4 -> K5)           [yb][s][x][yi][kz]   pitch Kp
  //   G  (K5 -> K6)           [s][x][y][kz]        pitch Kp
  const int Kp = rhs_pitch(p), YB = rhs_yblock(p);
  const bool lay = Kp != p->K || YB > 0;
  const int YBe = YB ? YB : p->n1;
  const long long yb1 = (long long)YBe * p->K;  // x-row stride of X1
  const long long yb2 = (long long)YBe * Kp;    // x-row stride of X2
  if (YB) {  // K1: column groups = y blocks of flattened (y, kz) columns
    a.kc = (int)yb1;
    a.ngrp = p->n1 / YB;
    a.in_kst = yb1;  // the state keeps its plain order
    a.in_rs = a.row_stride;
    a.out_kst = (long long)p->S1 * p->m0 * yb1;
    a.out_rs = yb1;
    a.out_plane_stride = (long long)p->m0 * yb1;
  }
  if (d == 2 && lay) {  // 2D: x-pass rows at pitch Kp (the state's rows keep pitch K)
    a.out_rs = Kp;
    a.kc_out = Kp;
    a.out_plane_stride = (long long)p->m0 * Kp;
  }
  if ((rc = launch_col(p, d == 3 ? KK_INV_KX : KK_INV_RHS, a, st))) return rc;
  const cplx* zin = p->A;
  cplx* zout = p->B;
  if (d == 3) {
    // K2: curl completion + y pad + inverse y
    PassArgs b = y_pass(p, p->A, p->B, p->S, p->m0, p->n1, p->m1, p->m1, p->n1);
    b.xplanes = p->m0;
    b.xblk = curly_xblk(p->m0);
    b.nsig = p->S;
    b.ck1 = p->ck1;
    b.ck2 = p->ck2;
    int k2 = KK_INV_CURLY;
    if (lay) {
      b.out_rs = Kp;
      b.kc_out = Kp;
      b.out_plane_stride = (long long)p->m1 * Kp;
      if (YB) {  // y-blocked rows in
        b.in_plane_stride = yb1;
        b.in_rpb = YB;
        b.in_bstride = (long long)p->S1 * p->m0 * yb1;
        k2 = KK_INV_CURLY_SLAB;
      }
    }
    if ((rc = launch_col(p, k2, b, st))) return rc;
    zin = p->B;
    zout = p->A;
  }
  // K3: z C2R -> products -> z R2C
  const int P = p->m0 * p->m1;
  ZArgs z = z_args(p, p->m2, p->n2, P);
  z.in = zin;
  z.out = zout;
  z.Kp = lay ? Kp : 0;
  z.in_sig_stride = (long long)P * (lay ? Kp : p->K);
  z.out_sig_stride = (long long)P * (lay ? Kp : p->K);
  z.zero_nyq = 1;
  z.dbg = (p->dbg && p->last_launches == p->dbg_launch) ? p->dbg : nullptr;
  z.pf_dist = zpass_prefetch_distance();
  int kind = d == 3 ? (p->density ? KK_Z_B3 : KK_Z_NS3) : (p->density ? KK_Z_B2 : KK_Z_NS2);
  if ((rc = launch_z(p, kind, z, 0, 0, st))) return rc;
  const cplx* xin = zout;
  cplx* gbuf = p->A;
  if (d == 3) {
    // K4: forward y + truncate
    PassArgs b = y_pass(p, p->A, p->B, p->So, p->m0, p->m1, p->n1, p->m1, p->n1);
    b.zero_nyq = 1;
    int k4 = KK_FWD_P;
    if (lay) {
      b.in_rs = b.out_rs = Kp;
      b.kc_out = Kp;
      b.in_plane_stride = (long long)p->m1 * Kp;
      b.out_plane_stride = yb2;
      if (YB) {  // y-blocked rows out
        b.out_rpb = YB;
        b.out_bstride = (long long)p->So * p->m0 * yb2;
        k4 = KK_FWD_P_SLABO;
      }
    }
    if ((rc = launch_col(p, k4, b, st))) return rc;
    xin = p->B;
  }
  // K5: forward x + truncate + 1/1.5^d + Nyquist / DC-imag zeroing -> G
  PassArgs c5 = x_pass(p, xin, gbuf, p->So, p->m0, p->n0, p->m0, p->n0);
  c5.scale = std::pow(1.0 / 1.5, d);
  c5.zero_nyq = 1;
  c5.zero_dc_imag = 1;
  int k5 = KK_FWD_P;
  if (d == 2) {  // 2D: a narrower x-forward tile where one is registered (more CTAs per SM)
    init_registry();
    auto it = g_fast->find(p->m0);
    if (it != g_fast->end() && it->second.e[KK_FWD_P2D].fn) k5 = KK_FWD_P2D;
  }
  if (lay) {  // K5: flattened (y, kz) columns at pitch Kp on both sides (pad columns transformed too)
    c5.Qp = p->n1 * Kp;
    c5.row_stride = (long long)p->n1 * Kp;
    c5.in_plane_stride = (long long)p->m0 * yb2;
    c5.out_plane_stride = (long long)p->n0 * p->n1 * Kp;
    if (YB) {
      c5.kc = (int)yb2;
      c5.ngrp = p->n1 / YB;
      c5.in_kst = (long long)p->So * p->m0 * yb2;
      c5.in_rs = yb2;
      c5.out_kst = yb2;
      c5.out_rs = c5.row_stride;
    }
  }
  if ((rc = launch_col(p, k5, c5, st))) return rc;
  // K6: projection + viscous (+ Boussinesq terms)
  ProjArgs pa{};
  pa.g = geom(p);
  pa.G = gbuf;
  pa.Gp = lay ? Kp : 0;
  pa.y = y;
  pa.f = f;
  pa.modes = p->modes;
  pa.density = p->density;
  pa.nu = nu;
  pa.ri = ri;
  pa.re_pr = re_pr;
  bool fused = false;
  if (cs && cs->diag_out) {  // srk_rhs_refresh (ybase == y, no earlier terms)
    pa.partial = p->partial;
    pa.cself = cs->cself;
    pa.ynext = cs->ynext;
    if (!srk_launch_project_refresh(pa, cs->diag_out, st)) return fail(SRK_ERR_UNSUPPORTED, "srk_rhs_refresh: mode count >= 2^32");
    p->last_launches += 2;
    if (p->timing && p->nev < 16) cudaEventRecord(p->ev[p->nev++], st);
    return check_launch("k_project_tma (refresh)");
  }
  if (cs) {
    pa.yb = cs->yb;
    pa.nt = cs->nt;
    for (int j = 0; j < cs->nt; ++j) {
      pa.F[j] = cs->F[j];
      pa.c[j] = cs->c[j];
    }
    pa.cself = cs->cself;
    pa.ynext = cs->ynext;
    pa.hs = cs->hs;
    fused = srk_launch_project_comb(pa, st);
  }
  if (!fused) srk_launch_project(pa, st);
  p->last_launches++;
  if (p->timing && p->nev < 16) cudaEventRecord(p->ev[p->nev++], st);
  if ((rc = check_launch("k_project"))) return rc;
  return (cs && !fused) ? comb_after(p, cs, f, st) : SRK_OK;
}
}  // namespace

int srk_rhs_timed(srk_plan* p, const void* y, void* f, double nu, double ri, double re_pr, void* stream,
                  float* ms_out, int max_kernels) {
  if (!p) return fail(SRK_ERR_INVALID, "null plan");
  cudaStream_t st = (cudaStream_t)stream;
  for (int i = 0; i < 16; ++i) cudaEventCreate(&p->ev[i]);
  p->timing = true;
  p->nev = 0;
  cudaEventRecord(p->ev[p->nev++], st);
  int rc = srk_rhs(p, y, f, nu, ri, re_pr, stream);
  p->timing = false;
  if (rc == SRK_OK) {
    cudaError_t err = cudaEventSynchronize(p->ev[p->nev - 1]);
    if (err != cudaSuccess) rc = fail(SRK_ERR_CUDA, std::string("srk_rhs_timed: ") + cudaGetErrorString(err));
  }
  int n = p->nev - 1;
  if (rc == SRK_OK)
    for (int i = 0; i < n && i < max_kernels; ++i) cudaEventElapsedTime(&ms_out[i], p->ev[i], p->ev[i + 1]);
  for (int i = 0; i < 16; ++i) cudaEventDestroy(p->ev[i]);
  return rc == SRK_OK ? -n : rc;  // negative = kernel count on success
}

int srk_rhs_launch_count(const srk_plan* p) { return p ? p->last_launches : 0; }

int srk_debug_phase_buffer(srk_plan* p, void* dev_buf, int launch_index) {
  if (!p) return fail(SRK_ERR_INVALID, "null plan");
  p->dbg = (unsigned long long*)dev_buf;
  p->dbg_launch = launch_index;
  return SRK_OK;
}

int srk_widen(srk_plan* p, const void* spec, int ncomp, void* phys, void* stream) {
  if (!p) return fail(SRK_ERR_INVALID, "null plan");
  int rc = need_ws(p);
  if (rc) return rc;
  if (ncomp < 1 || ncomp > p->max_comps)
    return fail(SRK_ERR_INVALID, std::to_string(ncomp) + " components exceed workspace size " + std::to_string(p->max_comps));
  return inverse_chain(p, (const cplx*)spec, ncomp, (double*)phys, true, (cudaStream_t)stream);
}

int srk_narrow(srk_plan* p, const void* phys, int ncomp, void* spec, void* stream) {
  if (!p) return fail(SRK_ERR_INVALID, "null plan");
  int rc = need_ws(p);
  if (rc) return rc;
  if (ncomp < 1 || ncomp > p->max_comps)
    return fail(SRK_ERR_INVALID, std::to_string(ncomp) + " components exceed workspace size " + std::to_string(p->max_comps));
  return forward_chain(p, (const double*)phys, ncomp, (cplx*)spec, true, (cudaStream_t)stream);
}

int srk_forward_transform(srk_plan* p, const void* phys, int ncomp, void* spec, void* stream) {
  if (!p) return fail(SRK_ERR_INVALID, "null plan");
  int rc = need_ws(p);
  if (rc) return rc;
  if (ncomp < 1 || ncomp > p->max_comps) return fail(SRK_ERR_INVALID, "component count exceeds the plan's workspace");
  return forward_chain(p, (const double*)phys, ncomp, (cplx*)spec, false, (cudaStream_t)stream);
}

int srk_inverse_transform(srk_plan* p, const void* spec, int ncomp, void* phys, void* stream) {
  if (!p) return fail(SRK_ERR_INVALID, "null plan");
  int rc = need_ws(p);
  if (rc) return rc;
  if (ncomp < 1 || ncomp > p->max_comps) return fail(SRK_ERR_INVALID, "component count exceeds the plan's workspace");
  return inverse_chain(p, (const cplx*)spec, ncomp, (double*)phys, false, (cudaStream_t)stream);
}

int srk_curl(srk_plan* p, const void* u, void* w, void* stream) {
  if (!p) return fail(SRK_ERR_INVALID, "null plan");
  srk_launch_curl(geom(p), (const cplx*)u, (cplx*)w, p->modes, (cudaStream_t)stream);
  return check_launch("k_curl");
}

int srk_leray_project(srk_plan* p, const void* u, void* out, void* stream) {
  if (!p) return fail(SRK_ERR_INVALID, "null plan");
  srk_launch_leray(geom(p), (const cplx*)u, (cplx*)out, p->modes, (cudaStream_t)stream);
  return check_launch("k_leray");
}

int srk_combine_scaled(int64_t n, const void* y, int nterms, const void* const* F, const double* a_coef,
                       const double* h_dev, void* out, void* stream);

int srk_combine(int64_t n, const void* y, int nterms, const void* const* F, const double* coef, void* out,
                void* stream) {
  return srk_combine_scaled(n, y, nterms, F, coef, nullptr, out, stream);
}

int srk_combine_scaled(int64_t n, const void* y, int nterms, const void* const* F, const double* coef,
                       const double* h_dev, void* out, void* stream) {
  if (nterms < 0 || nterms > SRK_MAX_TERMS) return fail(SRK_ERR_INVALID, "srk_combine: at most 8 terms");
  CombArgs a;
  memset(&a, 0, sizeof(a));
  a.hs = h_dev;
  a.y = (const cplx*)y;
  for (int j = 0; j < nterms; ++j) {
    a.F[j] = (const cplx*)F[j];
    a.c[j] = coef[j];
  }
  a.nt = nterms;
  a.out = (cplx*)out;
  a.n = n;
  srk_launch_combine(a, (cudaStream_t)stream);
  return check_launch("k_combine");
}

int srk_step_reduce_scaled(srk_plan* p, const void* y0, const void* y1, int nterms, const void* const* F,
                           const double* coef, const double* h_dev, const void* fl, int ncomp, double tol_abs,
                           double tol_rel, int flags, double* out_dev, void* stream);

int srk_step_reduce(srk_plan* p, const void* y0, const void* y1, int nterms, const void* const* F,
                    const double* coef, const void* fl, int ncomp, double tol_abs, double tol_rel, int flags,
                    double* out_dev, void* stream) {
  return srk_step_reduce_scaled(p, y0, y1, nterms, F, coef, nullptr, fl, ncomp, tol_abs, tol_rel, flags, out_dev,
                                stream);
}

int srk_step_reduce_scaled(srk_plan* p, const void* y0, const void* y1, int nterms, const void* const* F,
                           const double* coef, const double* h_dev, const void* fl, int ncomp, double tol_abs,
                           double tol_rel, int flags, double* out_dev, void* stream) {
  if (!p) return fail(SRK_ERR_INVALID, "null plan");
  if (nterms < 0 || nterms > SRK_MAX_TERMS) return fail(SRK_ERR_INVALID, "srk_step_reduce: at most 8 terms");
  if (ncomp < 1 || ncomp > 4) return fail(SRK_ERR_INVALID, "srk_step_reduce: 1..4 components");
  RedArgs a;
  memset(&a, 0, sizeof(a));
  a.g = geom(p);
  a.y0 = (const cplx*)y0;
  a.y1 = (const cplx*)y1;
  a.do_norm = (flags & 1) ? 1 : 0;
  a.do_diag = (flags & 2) ? 1 : 0;
  a.nt = a.do_norm ? nterms : 0;
  for (int j = 0; j < a.nt; ++j) {
    a.F[j] = (const cplx*)F[j];
    a.c[j] = coef[j];
  }
  a.hs = h_dev;
  a.fl = (const cplx*)fl;
  a.fl_term = -1;
  for (int j = 0; j < a.nt; ++j)
    if (a.F[j] == a.fl) a.fl_term = j;  // the FSAL stage is also an error term: stream it once
  a.ncomp = ncomp;
  a.dvel = std::min(p->dims, ncomp);
  a.modes = p->modes;
  a.K = p->K;
  a.atol = tol_abs;
  a.rtol = tol_rel;
  a.partial = p->partial;
  srk_launch_reduce(a, out_dev, (cudaStream_t)stream);
  return check_launch("k_reduce");
}

int srk_band_energy(srk_plan* p, const void* u, int ncomp, const int64_t* idx, const double* w, int nb,
                    double* out_dev, void* stream) {
  if (!p) return fail(SRK_ERR_INVALID, "null plan");
  srk_launch_band_energy((const cplx*)u, (const long long*)idx, w, nb, ncomp, p->modes, out_dev,
                         (cudaStream_t)stream);
  return check_launch("k_band_energy");
}

int srk_band_scale(srk_plan* p, void* u, int ncomp, const int64_t* idx, int nb, double gamma, void* stream) {
  if (!p) return fail(SRK_ERR_INVALID, "null plan");
  srk_launch_band_scale((cplx*)u, (const long long*)idx, nb, ncomp, p->modes, gamma, (cudaStream_t)stream);
  return check_launch("k_band_scale");
}

int srk_store_mapped(const double* src, double* dst, int n, void* stream) {
  if ((!src || !dst) && n > 0) return fail(SRK_ERR_INVALID, "null pointer");
  if (n < 0) return fail(SRK_ERR_INVALID, "negative count");
  srk_launch_store_mapped(src, dst, n, (cudaStream_t)stream);
  return check_launch("k_store_mapped");
}

// ---------------------------------------------------------------------------
// Slab decomposition over y: rank r owns y-slab [r*Ny, (r+1)*Ny)
// of the spectral state.  srk_slab_forward (K1) writes the x-padded signals
// straight into the all-to-all #1 send layout [dest][s][x_loc][y_loc][kz];
// srk_slab_middle (K2-K4) reads the receive layout [src][s][x_loc][y_loc][kz]
// of its x-slab and writes the all-to-all #2 send layout
// [dest][o][x_loc][y_loc][kz]; srk_slab_finish (K5-K6) reads the receive
// layout [src][o][x_loc][y_loc][kz] and writes the tendency y-slab.
// ---------------------------------------------------------------------------
int srk_plan_create_slab(srk_plan** out, const int64_t* shape, const double* lengths, int density, int nranks,
                         int rank) {
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(SRK_ERR_INVALID, "bad rank / nranks");
  if (shape[1] % nranks || (3 * shape[0] / 2) % nranks)
    return fail(SRK_ERR_INVALID, "slab decomposition needs nranks | n1 and nranks | 3*n0/2");
  int64_t loc[3] = {shape[0], shape[1] / nranks, shape[2]};  // local y extent
  if (loc[1] < 1) return fail(SRK_ERR_INVALID, "too many ranks for n1");
  // create with the local y extent (workspace sizing is redone below)
  int64_t tmp[3] = {shape[0], shape[1], shape[2]};
  int rc = srk_plan_create(out, 3, tmp, lengths, density, 0);
  if (rc) return rc;
  srk_plan* p = *out;
  p->nranks = nranks;
  p->rank = rank;
  p->n1g = (int)shape[1];
  p->n1 = (int)loc[1];
  p->y0 = rank * p->n1;
  p->Mx = p->m0 / nranks;
  p->modes = (long long)p->n0 * p->n1 * p->K;
  const long long K = p->K, Ny = p->n1, Mx = p->Mx, m1 = p->m1, n0 = p->n0;
  const long long Kp = slab_pitch(p);
  long long A = std::max<long long>(p->So * Mx * m1 * Kp, p->So * n0 * Ny * K);
  long long B = p->S * Mx * m1 * Kp;
  (void)loc;
  p->A_elems = A;
  p->B_elems = B;
  p->need_bytes = align256(A * 16) + align256(std::max<long long>(B, 1) * 16);
  return SRK_OK;
}

int srk_slab_sizes(const srk_plan* p, int64_t* send1, int64_t* send2) {
  if (!p) return fail(SRK_ERR_INVALID, "null plan");
  *send1 = (int64_t)p->S1 * p->m0 * p->n1 * p->K;
  *send2 = (int64_t)p->So * p->Mx * p->n1g * p->K;
  return SRK_OK;
}

int srk_slab_forward(srk_plan* p, const void* y, void* send1, void* stream) {
  if (!p || !p->Mx) return fail(SRK_ERR_INVALID, "not a slab plan");
  cudaStream_t st = (cudaStream_t)stream;
  const int d = p->dims;
  const long long blk = (long long)p->S1 * p->Mx * p->n1 * p->K;
  PassArgs a = x_pass(p, (const cplx*)y, (cplx*)send1, p->S1, p->n0, p->m0, p->m0, p->n0);
  a.out_plane_stride = (long long)p->Mx * p->n1 * p->K;
  a.out_rpb = p->Mx;
  a.out_bstride = blk;
  a.scale = std::pow(1.5, d) / ((double)p->m0 * p->m1 * p->m2);
  a.dims = d;
  a.n1 = p->n1;
  a.K = p->K;
  a.ck0 = p->ck0;
  a.ck1 = p->ck1;
  a.ck2 = p->ck2;
  a.comp_stride = p->modes;
  a.y0 = p->y0;
  a.n1g = p->n1g;
  return launch_col(p, KK_INV_KX_SLAB, a, st);
}

int srk_slab_middle(srk_plan* p, const void* recv1, void* send2, void* stream) {
  if (!p || !p->Mx) return fail(SRK_ERR_INVALID, "not a slab plan");
  int rc = need_ws(p);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  const long long K = p->K, Ny = p->n1, Mx = p->Mx, m1 = p->m1;
  // K2: y pad + inverse y from the receive layout
  PassArgs b = base_pass();
  b.in = (const cplx*)recv1;
  b.out = p->B;
  b.M = p->m1;
  b.n = p->n1g;
  b.planes = p->S * p->Mx;
  b.Qp = p->K;
  b.row_stride = K;
  const long long Kp = slab_pitch(p);  // pitch of the rank-local B / A buffers
  b.in_plane_stride = Ny * K;
  b.out_plane_stride = m1 * Kp;
  b.out_rs = Kp;
  b.kc_out = (int)Kp;
  b.in_rpb = (int)Ny;
  b.in_bstride = (long long)p->S1 * Mx * Ny * K;
  b.xplanes = p->Mx;
  b.xblk = curly_xblk(p->Mx);
  b.nsig = p->S;
  b.ck1 = p->ck1;
  b.ck2 = p->ck2;
  if ((rc = launch_col(p, KK_INV_CURLY_SLAB, b, st))) return rc;
  // K3: z pencils of the x-slab
  const int P = (int)(Mx * m1);
  ZArgs z = z_args(p, p->m2, p->n2, P);
  z.in = p->B;
  z.out = p->A;
  z.Kp = (int)Kp;
  z.in_sig_stride = (long long)P * Kp;
  z.out_sig_stride = (long long)P * Kp;
  z.zero_nyq = 1;
  if ((rc = launch_z(p, p->density ? KK_Z_B3 : KK_Z_NS3, z, 0, 0, st))) return rc;
  // K4: forward y + truncation into the all-to-all #2 send layout
  PassArgs c = base_pass();
  c.in = p->A;
  c.out = (cplx*)send2;
  c.M = p->m1;
  c.n = p->n1g;
  c.planes = p->So * p->Mx;
  c.Qp = p->K;
  c.row_stride = K;
  c.in_rs = Kp;
  c.in_plane_stride = m1 * Kp;
  c.out_plane_stride = Ny * K;
  c.out_rpb = (int)Ny;
  c.out_bstride = (long long)p->So * Mx * Ny * K;
  c.zero_nyq = 1;
  return launch_col(p, KK_FWD_P_SLABO, c, st);
}

int srk_slab_finish(srk_plan* p, const void* recv2, const void* y, void* f, double nu, double ri, double re_pr,
                    void* stream) {
  if (!p || !p->Mx) return fail(SRK_ERR_INVALID, "not a slab plan");
  int rc = need_ws(p);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  const long long K = p->K, Ny = p->n1, Mx = p->Mx;
  PassArgs c5 = x_pass(p, (const cplx*)recv2, p->A, p->So, p->m0, p->n0, p->m0, p->n0);
  c5.in_plane_stride = Mx * Ny * K;
  c5.in_rpb = p->Mx;
  c5.in_bstride = (long long)p->So * Mx * Ny * K;
  c5.scale = std::pow(1.0 / 1.5, p->dims);
  c5.zero_nyq = 1;
  c5.zero_dc_imag = 1;
  c5.y0 = p->y0;
  if ((rc = launch_col(p, KK_FWD_P_SLABI, c5, st))) return rc;
  ProjArgs pa{};
  pa.g = geom(p);
  pa.G = p->A;
  pa.y = (const cplx*)y;
  pa.f = (cplx*)f;
  pa.modes = p->modes;
  pa.density = p->density;
  pa.nu = nu;
  pa.ri = ri;
  pa.re_pr = re_pr;
  srk_launch_project(pa, st);
  return check_launch("k_project");
}


// ---- pipelined slab RHS: kz-chunked kernel groups (see srk.h) -----------------
static int bad_chunk(const srk_plan* p, int k0, int kc) {
  return !p || !p->Mx || k0 < 0 || kc < 1 || k0 + kc > p->K;
}

int srk_slab_forward_kz(srk_plan* p, const void* y, void* send1, int k0, int kc, void* stream) {
  if (bad_chunk(p, k0, kc)) return fail(SRK_ERR_INVALID, "not a slab plan / bad kz chunk");
  const int d = p->dims;
  const long long Ny = p->n1, Mx = p->Mx;
  PassArgs a = x_pass(p, (const cplx*)y, (cplx*)send1, p->S1, p->n0, p->m0, p->m0, p->n0);
  // columns: groups y_loc of kc kz values; input rows of n1*K, output rows of n1*kc
  a.kc = kc;
  a.ngrp = (int)Ny;
  a.in_kst = p->K;
  a.in_k0 = k0;
  a.out_kst = kc;
  a.out_k0 = 0;
  a.kz0 = k0;
  a.in_rs = Ny * p->K;
  a.out_rs = Ny * kc;
  a.out_plane_stride = Mx * Ny * kc;
  a.out_rpb = (int)Mx;
  a.out_bstride = (long long)p->S1 * Mx * Ny * kc;
  a.scale = std::pow(1.5, d) / ((double)p->m0 * p->m1 * p->m2);
  a.dims = d;
  a.n1 = p->n1;
  a.K = p->K;
  a.ck0 = p->ck0;
  a.ck1 = p->ck1;
  a.ck2 = p->ck2;
  a.comp_stride = p->modes;
  a.y0 = p->y0;
  a.n1g = p->n1g;
  return launch_col(p, KK_INV_KX_SLAB, a, (cudaStream_t)stream);
}

int srk_slab_inverse_y_kz(srk_plan* p, const void* recv1, int k0, int kc, void* stream) {
  if (bad_chunk(p, k0, kc)) return fail(SRK_ERR_INVALID, "not a slab plan / bad kz chunk");
  int rc = need_ws(p);
  if (rc) return rc;
  const long long K = p->K, Ny = p->n1, Mx = p->Mx, m1 = p->m1;
  PassArgs b = base_pass();
  b.in = (const cplx*)recv1;
  b.out = p->B;
  b.M = p->m1;
  b.n = p->n1g;
  b.planes = p->S * p->Mx;
  b.Qp = kc;
  b.kc = kc;
  b.ngrp = 1;
  b.in_k0 = 0;
  b.out_k0 = k0;
  b.kz0 = k0;
  b.in_rs = kc;
  b.out_rs = slab_pitch(p);
  if (k0 + kc == p->K) b.kc_out = kc + (slab_pitch(p) - p->K);  // the last chunk stores the pad columns
  b.in_plane_stride = Ny * kc;
  b.out_plane_stride = m1 * slab_pitch(p);
  b.in_rpb = (int)Ny;
  b.in_bstride = (long long)p->S1 * Mx * Ny * kc;
  b.xplanes = p->Mx;
  b.xblk = curly_xblk(p->Mx);
  b.nsig = p->S;
  b.ck1 = p->ck1;
  b.ck2 = p->ck2;
  return launch_col(p, KK_INV_CURLY_SLAB, b, (cudaStream_t)stream);
}

int srk_slab_zpass(srk_plan* p, void* stream) {
  if (!p || !p->Mx) return fail(SRK_ERR_INVALID, "not a slab plan");
  int rc = need_ws(p);
  if (rc) return rc;
  const long long K = p->K;
  const int P = (int)(p->Mx * p->m1);
  ZArgs z = z_args(p, p->m2, p->n2, P);
  z.in = p->B;
  z.out = p->A;
  z.Kp = slab_pitch(p);
  z.in_sig_stride = (long long)P * z.Kp;
  z.out_sig_stride = (long long)P * z.Kp;
  z.zero_nyq = 1;
  z.pf_dist = zpass_prefetch_distance();
  return launch_z(p, p->density ? KK_Z_B3 : KK_Z_NS3, z, 0, 0, (cudaStream_t)stream);
}

int srk_slab_forward_y_kz(srk_plan* p, void* send2, int k0, int kc, void* stream) {
  if (bad_chunk(p, k0, kc)) return fail(SRK_ERR_INVALID, "not a slab plan / bad kz chunk");
  int rc = need_ws(p);
  if (rc) return rc;
  const long long K = p->K, Ny = p->n1, Mx = p->Mx, m1 = p->m1;
  PassArgs c = base_pass();
  c.in = p->A;
  c.out = (cplx*)send2;
  c.M = p->m1;
  c.n = p->n1g;
  c.planes = p->So * p->Mx;
  c.Qp = kc;
  c.kc = kc;
  c.ngrp = 1;
  c.in_k0 = k0;
  c.out_k0 = 0;
  c.kz0 = k0;
  c.in_rs = slab_pitch(p);
  c.out_rs = kc;
  c.in_plane_stride = m1 * slab_pitch(p);
  c.out_plane_stride = Ny * kc;
  c.out_rpb = (int)Ny;
  c.out_bstride = (long long)p->So * Mx * Ny * kc;
  c.zero_nyq = 1;
  return launch_col(p, KK_FWD_P_SLABO, c, (cudaStream_t)stream);
}

int srk_slab_set_peers(srk_plan* p, const void* const* recv1, const void* const* recv2, int n) {
  if (!p || !p->Mx) return fail(SRK_ERR_INVALID, "not a slab plan");
  if (n != p->nranks || n > SRK_MAX_PEERS)
    return fail(SRK_ERR_INVALID, "peer tables need one entry per rank (at most " +
                                     std::to_string(SRK_MAX_PEERS) + ")");
  for (int r = 0; r < n; ++r) {
    if (!recv1[r] || !recv2[r]) return fail(SRK_ERR_INVALID, "null peer receive buffer");
    p->peer1[r] = (cplx*)recv1[r];
    p->peer2[r] = (cplx*)recv2[r];
  }
  p->peers_set = true;
  return SRK_OK;
}

// K1 of kz chunk (k0, kc) with its output row blocks stored straight into the
// peers' receive buffers: block d -> rank d's recv1 chunk region at this rank's
// source block (the layout srk_slab_inverse_y_kz reads), so all-to-all #1 is the
// pass's own NVLink stores.  Ordering: every rank's K1 must complete before any
// rank's K2 reads its recv1 (a stream-ordered barrier between the two).
int srk_slab_forward_kz_peer(srk_plan* p, const void* y, int k0, int kc, void* stream) {
  if (bad_chunk(p, k0, kc)) return fail(SRK_ERR_INVALID, "not a slab plan / bad kz chunk");
  if (!p->peers_set) return fail(SRK_ERR_INVALID, "srk_slab_set_peers not called");
  const long long Ny = p->n1, Mx = p->Mx;
  const long long per_kz = (long long)p->S1 * p->m0 * Ny;  // recv1 elements per kz
  const long long bs = (long long)p->S1 * Mx * Ny * kc;     // source-block stride of the chunk
  PassArgs a = x_pass(p, (const cplx*)y, p->peer1[p->rank], p->S1, p->n0, p->m0, p->m0, p->n0);
  a.kc = kc;
  a.ngrp = (int)Ny;
  a.in_kst = p->K;
  a.in_k0 = k0;
  a.out_kst = kc;
  a.out_k0 = 0;
  a.kz0 = k0;
  a.in_rs = Ny * p->K;
  a.out_rs = Ny * kc;
  a.out_plane_stride = Mx * Ny * kc;
  a.out_rpb = (int)Mx;
  a.out_bstride = bs;
  for (int r = 0; r < p->nranks; ++r) a.peer[r] = p->peer1[r] + per_kz * k0 + (long long)p->rank * bs;
  a.scale = std::pow(1.5, p->dims) / ((double)p->m0 * p->m1 * p->m2);
  a.dims = p->dims;
  a.n1 = p->n1;
  a.K = p->K;
  a.ck0 = p->ck0;
  a.ck1 = p->ck1;
  a.ck2 = p->ck2;
  a.comp_stride = p->modes;
  a.y0 = p->y0;
  a.n1g = p->n1g;
  return launch_col(p, KK_INV_KX_PEER, a, (cudaStream_t)stream);
}

// K4 of kz chunk (k0, kc) storing into the peers' recv2 chunk regions (all-to-all #2).
int srk_slab_forward_y_kz_peer(srk_plan* p, int k0, int kc, void* stream) {
  if (bad_chunk(p, k0, kc)) return fail(SRK_ERR_INVALID, "not a slab plan / bad kz chunk");
  if (!p->peers_set) return fail(SRK_ERR_INVALID, "srk_slab_set_peers not called");
  int rc = need_ws(p);
  if (rc) return rc;
  const long long K = p->K, Ny = p->n1, Mx = p->Mx, m1 = p->m1;
  const long long per_kz = (long long)p->So * Mx * p->n1g;  // recv2 elements per kz
  const long long bs = (long long)p->So * Mx * Ny * kc;
  PassArgs c = base_pass();
  c.in = p->A;
  c.out = p->peer2[p->rank];
  c.M = p->m1;
  c.n = p->n1g;
  c.planes = p->So * p->Mx;
  c.Qp = kc;
  c.kc = kc;
  c.ngrp = 1;
  c.in_k0 = k0;
  c.out_k0 = 0;
  c.kz0 = k0;
  c.in_rs = slab_pitch(p);
  c.out_rs = kc;
  c.in_plane_stride = m1 * slab_pitch(p);
  c.out_plane_stride = Ny * kc;
  c.out_rpb = (int)Ny;
  c.out_bstride = bs;
  for (int r = 0; r < p->nranks; ++r) c.peer[r] = p->peer2[r] + per_kz * k0 + (long long)p->rank * bs;
  c.zero_nyq = 1;
  return launch_col(p, KK_FWD_P_PEER, c, (cudaStream_t)stream);
}

// ---- CUDA IPC of receive buffers between the ranks' processes ---------------
typedef CUresult (*srk_get_range_fn)(CUdeviceptr*, size_t*, CUdeviceptr);

int srk_ipc_export(const void* dev_ptr, void* handle_out, int64_t* offset_out) {
  if (!dev_ptr || !handle_out || !offset_out) return fail(SRK_ERR_INVALID, "null argument");
  static srk_get_range_fn range = nullptr;
  if (!range) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
      return fail(SRK_ERR_CUDA, "cuMemGetAddressRange entry point unavailable");
    range = (srk_get_range_fn)fn;
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  if (range(&base, &size, (CUdeviceptr)dev_ptr) != CUDA_SUCCESS) return fail(SRK_ERR_CUDA, "cuMemGetAddressRange failed");
  cudaIpcMemHandle_t h;
  cudaError_t err = cudaIpcGetMemHandle(&h, (void*)base);
  if (err != cudaSuccess) return fail(SRK_ERR_CUDA, std::string("cudaIpcGetMemHandle: ") + cudaGetErrorString(err));
  memcpy(handle_out, &h, sizeof(h));
  *offset_out = (int64_t)((const char*)dev_ptr - (const char*)base);
  return SRK_OK;
}

int srk_ipc_import(const void* handle, int64_t offset, void** dev_ptr_out) {
  if (!handle || !dev_ptr_out) return fail(SRK_ERR_INVALID, "null argument");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  void* base = nullptr;
  cudaError_t err = cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess);
  if (err != cudaSuccess) return fail(SRK_ERR_CUDA, std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(err));
  *dev_ptr_out = (char*)base + offset;
  return SRK_OK;
}

int srk_ipc_close(void* dev_ptr, int64_t offset) {
  if (!dev_ptr) return SRK_OK;
  cudaError_t err = cudaIpcCloseMemHandle((char*)dev_ptr - offset);
  if (err != cudaSuccess) return fail(SRK_ERR_CUDA, std::string("cudaIpcCloseMemHandle: ") + cudaGetErrorString(err));
  return SRK_OK;
}

int srk_slab_forward_x_kz(srk_plan* p, const void* recv2, int k0, int kc, void* stream) {
  if (bad_chunk(p, k0, kc)) return fail(SRK_ERR_INVALID, "not a slab plan / bad kz chunk");
  int rc = need_ws(p);
  if (rc) return rc;
  const long long K = p->K, Ny = p->n1, Mx = p->Mx;
  // G (So, n0, ny, K) goes to workspace B (free after the z-pass): K4 of later
  // chunks still reads the z-pass output in A
  PassArgs c5 = x_pass(p, (const cplx*)recv2, p->B, p->So, p->m0, p->n0, p->m0, p->n0);
  c5.kc = kc;
  c5.ngrp = (int)Ny;
  c5.in_kst = kc;
  c5.in_k0 = 0;
  c5.out_kst = K;
  c5.out_k0 = k0;
  c5.kz0 = k0;
  c5.in_rs = Ny * kc;
  c5.out_rs = Ny * K;
  c5.in_plane_stride = Mx * Ny * kc;
  c5.in_rpb = (int)Mx;
  c5.in_bstride = (long long)p->So * Mx * Ny * kc;
  c5.scale = std::pow(1.0 / 1.5, p->dims);
  c5.zero_nyq = 1;
  c5.zero_dc_imag = 1;
  c5.y0 = p->y0;
  return launch_col(p, KK_FWD_P_SLABI, c5, (cudaStream_t)stream);
}

int srk_slab_project(srk_plan* p, const void* y, void* f, double nu, double ri, double re_pr, void* stream) {
  if (!p || !p->Mx) return fail(SRK_ERR_INVALID, "not a slab plan");
  int rc = need_ws(p);
  if (rc) return rc;
  ProjArgs pa{};
  pa.g = geom(p);
  pa.G = p->B;
  pa.y = (const cplx*)y;
  pa.f = (cplx*)f;
  pa.modes = p->modes;
  pa.density = p->density;
  pa.nu = nu;
  pa.ri = ri;
  pa.re_pr = re_pr;
  srk_launch_project(pa, (cudaStream_t)stream);
  return check_launch("k_project");
}

}  // extern "C"
