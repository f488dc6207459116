/*
 * srk.h -- C ABI of libsrk, the sm_100a (B200) implementation of the hot path of
 * the `spectralrk` reference (arxiv/paper_1810_10197): the 3/2-rule dealiased
 * pseudo-spectral incompressible Navier-Stokes / Boussinesq right-hand side and
 * the Runge-Kutta stage / error-norm arithmetic around it.
 *
 * The reference is pure Python; its "operator API" for this path is duck
 * typing.  Each entry point below names the reference callable
 * it replaces (paths relative to /root/reference/pkg/src/spectralrk/).  The
 * ctypes binding that a reference maintainer would add is in INTEGRATION.md;
 * the one this repo uses is paper_1810_10197_b200/_native.py.
 *
 * Conventions
 *  - All arrays are DEVICE pointers to caller-owned memory (torch tensors),
 *    C-order, complex128 spectra in the numpy rfftn layout
 *    (ncomp, n0, n1, n2/2+1) [2D: (ncomp, n0, n1/2+1)], float64 physical fields
 *    (ncomp, *shape).  The r2c axis is the LAST axis (grid.py:71).
 *  - `stream` is a cudaStream_t (may be NULL = legacy default stream); every
 *    call is asynchronous and stream-ordered.
 *  - Return value 0 = success; non-zero = error, text in srk_last_error().
 *    SRK_ERR_INVALID maps to the reference's ValueError (grid.py:55-66,
 *    spectral.py:25-28,40-43, :212-214, :269-271).
 *  - A plan is single-owner and not re-entrant, like FlowRHS's shared
 *    DealiasWorkspace (physics.py:195-201).
 */
#ifndef SRK_H
#define SRK_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SRK_OK 0
#define SRK_ERR_INVALID 1
#define SRK_ERR_UNSUPPORTED 2
#define SRK_ERR_CUDA 3
#define SRK_ERR_WORKSPACE 4

typedef struct srk_plan srk_plan;

/* ABI version of this header (bumped on any signature change). */
int srk_abi_version(void);

/* Thread-local description of the last error. */
const char* srk_last_error(void);

/* Grid + dealiasing workspace geometry.
 * Replaces Grid(shape, lengths) (grid.py:53-110) together with
 * DealiasWorkspace(grid, ncomp) (spectral.py:187-207) and the workspace that
 * FlowRHS(grid, params, density) owns (physics.py:195-201).
 * dims = 2 or 3; shape[dims] even and >= 4; lengths[dims] > 0;
 * density = 0|1 (Boussinesq); max_comps = largest component count passed to
 * srk_widen / srk_narrow / the transforms (0 -> the RHS's own need). */
int srk_plan_create(srk_plan** out, int dims, const int64_t* shape, const double* lengths,
                    int density, int max_comps);
void srk_plan_destroy(srk_plan* plan);

/* Device workspace the caller must allocate (bytes) and bind before any
 * compute call.  Replaces the numpy buffers of spectral.py:187-207.  The layout
 * inside is the library's own: plans on the compile-time FFT lengths keep the RHS
 * intermediates at a sector-aligned pencil pitch (ceil4(n_last/2 + 1) for n_last >=
 * 256) and the x-padded buffers y-blocked, so the size is slightly larger than the
 * reference's buffers (+1.2 % at 512^3); always query it here. */
int srk_plan_workspace_bytes(const srk_plan* plan, int64_t* bytes);
int srk_plan_set_workspace(srk_plan* plan, void* ptr, int64_t bytes);

/* FlowRHS.__call__(t, fields) (physics.py:203-206):
 *   density == 0: ns_rhs         (physics.py:105-129), nu = 1/Re
 *   density == 1: boussinesq_rhs (physics.py:132-185), ri = Ri, re_pr = Re*Pr
 * y, f: (d [+1], ...kshape) complex128; f must not alias y. */
int srk_rhs(srk_plan* plan, const void* y, void* f, double nu, double ri, double re_pr, void* stream);

/* srk_rhs fused with the next rk_step accumulation (integrators.py:327-339 for
 * the next stage input, :336-339 for y_new of a non-FSAL pair):
 *   f     = FlowRHS(y)
 *   ynext = ybase + sum_{j < nterms} coef[j] * F[j] + coef_self * f
 * summed in that order (ascending stage index, f being the highest), one
 * rounding per multiply and add: bitwise equal to srk_rhs followed by
 * srk_combine(ybase, [F..., f], [coef..., coef_self]).  On the 3D NS path the
 * projection kernel forms ynext while f is still in registers (f is not read
 * back); other shapes run the two calls.  nterms <= 6 on the fused path
 * (<= 7 otherwise); F / coef are HOST arrays; ynext must not alias y, f, F. */
int srk_rhs_combine(srk_plan* plan, const void* y, void* f, double nu, double ri, double re_pr,
                    const void* ybase, int nterms, const void* const* F, const double* coef, double coef_self,
                    void* ynext, void* stream);

/* The refresh after a step's forcing (simulation.py:165-182 after_accept: the
 * cached tendency and the diagnostics record of the new state) fused with the
 * next step's first stage sum (integrators.py:327-333, row 2 of A):
 *   f     = FlowRHS(y)
 *   ynext = y + coef_self * f              (bitwise srk_rhs_combine(ybase = y))
 *   diag_out[4] = sum_k w_k sum_j |y_jk|^2, diag_out[5] = sum w Re(y conj f),
 *   diag_out[8] = sum w |k|^2 |y|^2, other entries 0 -- the srk_step_reduce
 *   (flags = 2) layout, fixed-order (deterministic) sums; diag_out may be
 *   mapped pinned host memory.
 * One pass of the projection kernel (y is read once); 2D / 3D, NS or
 * Boussinesq (E, eps, Z over the velocity components), unsplit plans. */
int srk_rhs_refresh(srk_plan* plan, const void* y, void* f, double nu, double ri, double re_pr, double coef_self,
                    void* ynext, double* diag_out, void* stream);

/* DealiasWorkspace.widen (spectral.py:215-261): spec (ncomp, kshape) ->
 * phys (ncomp, 3n0/2, 3n1/2[, 3n2/2]) float64. */
int srk_widen(srk_plan* plan, const void* spec, int ncomp, void* phys, void* stream);

/* DealiasWorkspace.narrow (spectral.py:263-304): phys (ncomp, padded shape)
 * float64 -> spec (ncomp, kshape) complex128 with Nyquist / self-conjugate
 * zeroing. */
int srk_narrow(srk_plan* plan, const void* phys, int ncomp, void* spec, void* stream);

/* forward_transform (spectral.py:17-30), unnormalised rfftn over the grid axes. */
int srk_forward_transform(srk_plan* plan, const void* phys, int ncomp, void* spec, void* stream);

/* inverse_transform (spectral.py:33-44), irfftn with 1/points normalisation. */
int srk_inverse_transform(srk_plan* plan, const void* spec, int ncomp, void* phys, void* stream);

/* curl (spectral.py:47-65): 3D (3,kshape)->(3,kshape); 2D (2,kshape)->(1,kshape). */
int srk_curl(srk_plan* plan, const void* u, void* w, void* stream);

/* leray_project (physics.py:89-102): (d,kshape) -> (d,kshape). */
int srk_leray_project(srk_plan* plan, const void* u, void* out, void* stream);

/* rk_step stage input / update (integrators.py:327-339, 341-347):
 *   out[i] = y[i] + sum_j coef[j] * F[j][i]   (ascending j; y may be NULL -> 0)
 * n = number of complex128 elements; nterms <= 8; F is a HOST array of device
 * pointers; coef is a HOST array. */
int srk_combine(int64_t n, const void* y, int nterms, const void* const* F, const double* coef, void* out,
                void* stream);

/* Step-size-scaled variants for CUDA-graph replay of an RK attempt
 * (integrators.py:322-347 with h read on the device): every coefficient is
 * passed as the tableau value a (host array, baked into the graph) and used as
 * (*h_dev) * a -- one rounding, bitwise the host product h * a of the unscaled
 * calls.  h_dev: one double in device memory, updated before each replay. */
int srk_combine_scaled(int64_t n, const void* y, int nterms, const void* const* F, const double* a,
                       const double* h_dev, void* out, void* stream);
int srk_rhs_combine_scaled(srk_plan* plan, const void* y, void* f, double nu, double ri, double re_pr,
                           const void* ybase, int nterms, const void* const* F, const double* a, double a_self,
                           const double* h_dev, void* ynext, void* stream);
int srk_step_reduce_scaled(srk_plan* plan, const void* y0, const void* y1, int nterms, const void* const* F,
                           const double* d, const double* h_dev, const void* fl, int ncomp, double tol_abs,
                           double tol_rel, int flags, double* out_dev, void* stream);

/* Fused embedded-error norm + diagnostics reduction (deterministic):
 *   flags & 1: error vector Delta = sum_j coef[j] F[j] (integrators.py:341-347),
 *              sc = tol_abs + max(|y0|,|y1|) tol_rel (control.py:51-57),
 *              out[c] = sum_modes (|Delta_c|/sc_c)^2 for c < 4 (control.py:72-79)
 *   flags & 2: out[4] = sum_k w_k sum_{j<d} |y1_kj|^2    (diagnostics.py:39-50)
 *              out[5] = sum_k w_k sum_{j<d} Re(y1 conj fl) (diagnostics.py:53-70)
 *              out[8] = sum_k w_k |k|^2 sum_{j<d} |y1_kj|^2  (enstrophy)
 *   always:    out[6] = number of non-finite entries in Delta and y1
 *              (integrators.py:348-351), out[7] = count(sc <= 0).
 * out_dev: 9 doubles in device memory or in pinned (UVA-mapped) host memory,
 *          stored by the last kernel.  Needs no bound workspace. */
int srk_step_reduce(srk_plan* plan, const void* y0, const void* y1, int nterms, const void* const* F,
                    const double* coef, const void* fl, int ncomp, double tol_abs, double tol_rel, int flags,
                    double* out_dev, void* stream);

/* apply_forcing band helpers (physics.py:209-239):
 * srk_band_energy: out_dev[0] = sum_{j<ncomp} sum_b w[b] |u_j[idx[b]]|^2
 * srk_band_scale:  u_j[idx[b]] *= gamma for j < ncomp
 * idx_dev: flat mode indices within one component; w_dev: Hermitian weights. */
int srk_band_energy(srk_plan* plan, const void* u, int ncomp, const int64_t* idx_dev, const double* w_dev,
                    int nb, double* out_dev, void* stream);
int srk_band_scale(srk_plan* plan, void* u, int ncomp, const int64_t* idx_dev, int nb, double gamma,
                   void* stream);

/* Small-result store: dst[i] = src[i], i < n, by a kernel on ``stream``; dst is
 * pinned (UVA-mapped) host memory, so the host reads the values after a stream
 * sync without a cudaMemcpy that could queue behind bulk host copies on the
 * copy engines (the reference reads its sums as numpy scalars,
 * control.py:72-79; the slab path's rank-order sums come back through this). */
int srk_store_mapped(const double* src_dev, double* dst_mapped, int n, void* stream);

/* srk_rhs with a CUDA event after every kernel (synchronises): writes the
 * per-kernel device times [ms] in launch order to ms_out and returns
 * -(number of kernels) on success, a positive error code otherwise.
 * Used by bench.py for the live roofline figure. */
int srk_rhs_timed(srk_plan* plan, const void* y, void* f, double nu, double ri, double re_pr, void* stream,
                  float* ms_out, int max_kernels);

/* ---- slab decomposition over y (multi-GPU, one plan per rank) ----
 * The state on rank r is the y-slab (ncomp, n0, n1/nranks, n2/2+1) holding
 * global rows y in [r*n1/nranks, (r+1)*n1/nranks).  One RHS is
 *   srk_slab_forward (K1)  -> all-to-all(send1 -> recv1, equal splits)
 *   srk_slab_middle (K2-K4) -> all-to-all(send2 -> recv2, equal splits)
 *   srk_slab_finish (K5-K6)
 * with the exchanges done by the caller (NCCL).  The kernels write the send
 * layouts and read the receive layouts directly (no pack / unpack passes).
 * Requires dims = 3, nranks | n1 and nranks | 3*n0/2. */
int srk_plan_create_slab(srk_plan** out, const int64_t* shape, const double* lengths, int density, int nranks,
                         int rank);
/* complex128 element counts of the send (== receive) buffers */
int srk_slab_sizes(const srk_plan* plan, int64_t* send1, int64_t* send2);
int srk_slab_forward(srk_plan* plan, const void* y, void* send1, void* stream);
int srk_slab_middle(srk_plan* plan, const void* recv1, void* send2, void* stream);
int srk_slab_finish(srk_plan* plan, const void* recv2, const void* y, void* f, double nu, double ri, double re_pr,
                    void* stream);

/* Pipelined slab RHS (SURVEY §8e "pipeline over kz-chunks"): the same kernel
 * groups split over kz chunks [k0, k0+kc) so that the caller's exchange of
 * chunk c overlaps the kernels of chunk c+1.  Chunk c of send1 / recv1 occupies
 * elements [S1*m0*ny*k0, S1*m0*ny*(k0+kc)) laid out [rank][s][x_loc][y_loc][kc]
 * (send2 / recv2 likewise with So*Mx*n1, [rank][o][x_loc][y_loc][kc]); the
 * pointers passed are the chunk starts.  Order per RHS:
 *   for c: srk_slab_forward_kz (K1)     -> exchange(send1_c -> recv1_c)
 *   for c: srk_slab_inverse_y_kz (K2)   (after recv1_c landed)
 *   srk_slab_zpass (K3)
 *   for c: srk_slab_forward_y_kz (K4)   -> exchange(send2_c -> recv2_c)
 *   for c: srk_slab_forward_x_kz (K5)   (after recv2_c landed)
 *   srk_slab_project (K6)
 * kc = K, k0 = 0 is the unchunked RHS.  Replaces the same reference call
 * chain as srk_rhs (physics.py:188-206 -> spectral.py:215-337). */
int srk_slab_forward_kz(srk_plan* plan, const void* y, void* send1_chunk, int k0, int kc, void* stream);
int srk_slab_inverse_y_kz(srk_plan* plan, const void* recv1_chunk, int k0, int kc, void* stream);
int srk_slab_zpass(srk_plan* plan, void* stream);
int srk_slab_forward_y_kz(srk_plan* plan, void* send2_chunk, int k0, int kc, void* stream);
int srk_slab_forward_x_kz(srk_plan* plan, const void* recv2_chunk, int k0, int kc, void* stream);
int srk_slab_project(srk_plan* plan, const void* y, void* f, double nu, double ri, double re_pr, void* stream);

/* Exchange fused into the passes (P <= 8 ranks): K1 and K4 store
 * their output row blocks straight into the peers' receive buffers over NVLink
 * (peer pointers from CUDA IPC, srk_ipc_*), so the two all-to-alls ride on the
 * passes' own stores, tile by tile, instead of separate NCCL collectives.
 * srk_slab_set_peers: recv1[r] / recv2[r] = rank r's all-to-all #1 / #2
 * receive buffer (sizes from srk_slab_sizes), n = nranks, r = this rank included.
 * srk_slab_forward_kz_peer / srk_slab_forward_y_kz_peer: srk_slab_forward_kz /
 * srk_slab_forward_y_kz writing rank d's block into rank d's receive chunk
 * region at this rank's source block -- the layout srk_slab_inverse_y_kz /
 * srk_slab_forward_x_kz read.  Ordering is the caller's: every rank's K1 (K4)
 * must complete before any rank reads its recv1 (recv2), e.g. a one-element
 * NCCL all-reduce on the compute streams between them.
 * Replaces the all_to_all_single exchanges of slab.py (the reference has no
 * multi-GPU path). */
int srk_slab_set_peers(srk_plan* plan, const void* const recv1[], const void* const recv2[], int n);
int srk_slab_forward_kz_peer(srk_plan* plan, const void* y, int k0, int kc, void* stream);
int srk_slab_forward_y_kz_peer(srk_plan* plan, int k0, int kc, void* stream);

/* CUDA IPC of a device buffer between the ranks' processes: export writes the
 * 64-byte cudaIpcMemHandle of the allocation holding dev_ptr and dev_ptr's
 * offset in it; import opens a peer's handle (lazy peer access) and returns the
 * peer's buffer address in this process; close releases an imported mapping. */
int srk_ipc_export(const void* dev_ptr, void* handle64_out, int64_t* offset_out);
int srk_ipc_import(const void* handle64, int64_t offset, void** dev_ptr_out);
int srk_ipc_close(void* dev_ptr, int64_t offset);

/* Diagnostics: when dev_buf (u64) is non-NULL, launch number launch_index of
 * the next srk_rhs chain (0 = K1) records clock64() phase timestamps of every
 * 97th CTA into it (3 per CTA for the axis passes, 6 for the NS3 z-pass;
 * tools/phase_timing.py).  Not a compute entry point. */
int srk_debug_phase_buffer(srk_plan* plan, void* dev_buf, int launch_index);

/* Throughput probe (not a compute entry point): one launch of blocks_per_sm
 * x SMs CTAs of 256 threads, each thread running `iters` trips of 8 ops:
 * mode 0 fp64 FMA, 1 fp64 add, 2 16-byte shared-memory loads, 3 warp
 * shuffles, 4 two shared loads + eight shuffles interleaved, 5 16-byte global
 * loads hitting L1, 6 two global (L1-hit) + two shared loads interleaved.
 * scratch: a device buffer of >= max(blocks_per_sm * SMs doubles, 64 KB).  *ops_out = thread-level
 * operations issued (time the launch with events on `stream`).  Used by
 * bench.py for the measured fp64 ceiling of the z-pass. */
int srk_probe(int mode, int iters, int blocks_per_sm, void* scratch, void* stream, double* ops_out);

/* Layout of the RHS intermediates inside the workspace (introspection, tests, docs):
 * *pitch = pencil pitch in complex elements (n_last/2 + 1, or that rounded up to 4 for
 * the sector-aligned layout), *yblock = rows per y block of the x-padded buffers
 * (0: plain [signal][x][y][kz] order).  No reference counterpart: numpy owns the
 * reference's buffers (spectral.py:187-207). */
int srk_plan_layout(const srk_plan* plan, int* pitch, int* yblock);

/* Build flags: bit 0 = hazard-probe build (make checks: schedule fuzzing at every
 * barrier, NaN-poisoned shared memory, tile bounds asserts; tools/check_build.sh). */
int srk_build_info(void);
/* Hash of the kernel sources + compile flags of this build (evidence provenance:
 * bench.py reports ncu counters only from a capture of the same sources). */
const char* srk_source_hash(void);

/* Number of kernel launches the last srk_rhs issued (launch accounting for
 * the bench's gpu_launches claim). */
int srk_rhs_launch_count(const srk_plan* plan);

#ifdef __cplusplus
}
#endif

#endif /* SRK_H */
