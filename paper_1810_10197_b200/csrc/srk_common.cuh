// Common device helpers for the sm_100a spectral NS path: complex fp64 arithmetic
// and the in-register DFT butterflies used by the FFT engines (fft_engine.cuh).
#pragma once

#include <cuda.h>  // CUtensorMap
#include <cuda_runtime.h>
#include <stdint.h>

#include "twiddle_consts.h"

typedef double2 cplx;

#define SRK_DEV __host__ __device__ __forceinline__

SRK_DEV cplx cmk(double r, double i) { return make_double2(r, i); }
SRK_DEV cplx cadd(cplx a, cplx b) { return make_double2(a.x + b.x, a.y + b.y); }
SRK_DEV cplx csub(cplx a, cplx b) { return make_double2(a.x - b.x, a.y - b.y); }
SRK_DEV cplx cscale(cplx a, double s) { return make_double2(a.x * s, a.y * s); }
SRK_DEV cplx cconj(cplx a) { return make_double2(a.x, -a.y); }
SRK_DEV cplx cmul(cplx a, cplx b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// multiply by SIGN*i
template <int SIGN>
SRK_DEV cplx cmul_si(cplx a) {
  return SIGN > 0 ? make_double2(-a.y, a.x) : make_double2(a.y, -a.x);
}

// ---------------------------------------------------------------------------
// Multiply by the compile-time constant exp(SIGN * 2*pi*i * m / 96) (96 =
// lcm of the composite radices 6, 8, 12, 16, 24, 32).  Cheap paths for
// multiples of pi/4; generic complex multiply otherwise.
// ---------------------------------------------------------------------------
template <int M96, int SIGN>
SRK_DEV cplx twc(cplx a) {
  constexpr int m = ((M96 % 96) + 96) % 96;
  if constexpr (m == 0) {
    return a;
  } else if constexpr (m == 24) {
    return cmul_si<SIGN>(a);
  } else if constexpr (m == 48) {
    return make_double2(-a.x, -a.y);
  } else if constexpr (m == 72) {
    return cmul_si<-SIGN>(a);
  } else if constexpr (m == 12 || m == 36 || m == 60 || m == 84) {
    constexpr double r = 0.7071067811865476;  // sqrt(2)/2
    constexpr double c = kcos96(m) > 0 ? 1.0 : -1.0;
    constexpr double s = (ksin96(m) > 0 ? 1.0 : -1.0) * (SIGN > 0 ? 1.0 : -1.0);
    // (a.x + i a.y)(c + i s) r
    return make_double2((c * a.x - s * a.y) * r, (s * a.x + c * a.y) * r);
  } else {
    constexpr double c = kcos96(m);
    constexpr double s = (SIGN > 0 ? 1.0 : -1.0) * ksin96(m);
    return make_double2(fma(a.x, c, -a.y * s), fma(a.x, s, a.y * c));
  }
}

// ---------------------------------------------------------------------------
// DFT_R in registers: v'[q] = sum_t v[t] exp(SIGN*2*pi*i*t*q/R), in place.
// ---------------------------------------------------------------------------
template <int R, int SIGN>
struct DFT;

template <int SIGN>
struct DFT<1, SIGN> {
  SRK_DEV static void run(cplx*) {}
};

template <int SIGN>
struct DFT<2, SIGN> {
  SRK_DEV static void run(cplx* v) {
    cplx a = v[0], b = v[1];
    v[0] = cadd(a, b);
    v[1] = csub(a, b);
  }
};

template <int SIGN>
struct DFT<3, SIGN> {
  SRK_DEV static void run(cplx* v) {
    constexpr double h = 0.8660254037844386;  // sqrt(3)/2
    cplx s = cadd(v[1], v[2]);
    cplx d = csub(v[1], v[2]);
    cplx m = make_double2(fma(-0.5, s.x, v[0].x), fma(-0.5, s.y, v[0].y));
    cplx r = cmul_si<SIGN>(cscale(d, h));
    v[0] = cadd(v[0], s);
    v[1] = cadd(m, r);
    v[2] = csub(m, r);
  }
};

template <int SIGN>
struct DFT<4, SIGN> {
  SRK_DEV static void run(cplx* v) {
    cplx a = cadd(v[0], v[2]), b = csub(v[0], v[2]);
    cplx c = cadd(v[1], v[3]), d = cmul_si<SIGN>(csub(v[1], v[3]));
    v[0] = cadd(a, c);
    v[2] = csub(a, c);
    v[1] = cadd(b, d);
    v[3] = csub(b, d);
  }
};

// odd prime radix via symmetric pairs (generic engine only)
template <int R, int SIGN>
struct DFTPrime {
  SRK_DEV static double co(int m) { return R == 5 ? kcos5(m) : kcos7(m); }
  SRK_DEV static double si(int m) { return R == 5 ? ksin5(m) : ksin7(m); }
  SRK_DEV static void run(cplx* v) {
    cplx out[R];
    cplx sum = v[0];
#pragma unroll
    for (int t = 1; t < R; ++t) sum = cadd(sum, v[t]);
    out[0] = sum;
#pragma unroll
    for (int q = 1; q < R; ++q) {
      cplx acc = v[0];
#pragma unroll
      for (int t = 1; t <= (R - 1) / 2; ++t) {
        double c = co(t * q), s = (SIGN > 0 ? 1.0 : -1.0) * si(t * q);
        cplx p = cadd(v[t], v[R - t]);
        cplx m = csub(v[t], v[R - t]);
        acc.x += p.x * c - m.y * s;
        acc.y += p.y * c + m.x * s;
      }
      out[q] = acc;
    }
#pragma unroll
    for (int q = 0; q < R; ++q) v[q] = out[q];
  }
};
template <int SIGN>
struct DFT<5, SIGN> : DFTPrime<5, SIGN> {};
template <int SIGN>
struct DFT<7, SIGN> : DFTPrime<7, SIGN> {};

// Composite radix R = A*B: t = B*a + b, q = q1 + A*q2.
template <int A, int B, int SIGN>
struct DFTComposite {
  static constexpr int R = A * B;
  static_assert(96 % R == 0, "composite radix must divide 96");
  template <int b, int q1>
  SRK_DEV static void tw(cplx (&u)[B][A]) {
    u[b][q1] = twc<(b * q1 * (96 / R)), SIGN>(u[b][q1]);
  }
  template <int b, int q1>
  SRK_DEV static void tw_row(cplx (&u)[B][A]) {
    if constexpr (q1 < A) {
      tw<b, q1>(u);
      tw_row<b, q1 + 1>(u);
    }
  }
  template <int b>
  SRK_DEV static void tw_all(cplx (&u)[B][A]) {
    if constexpr (b < B) {
      tw_row<b, 0>(u);
      tw_all<b + 1>(u);
    }
  }
  SRK_DEV static void run(cplx* v) {
    cplx u[B][A];
#pragma unroll
    for (int b = 0; b < B; ++b) {
#pragma unroll
      for (int a = 0; a < A; ++a) u[b][a] = v[B * a + b];
      DFT<A, SIGN>::run(u[b]);
    }
    tw_all<0>(u);
#pragma unroll
    for (int q1 = 0; q1 < A; ++q1) {
      cplx z[B];
#pragma unroll
      for (int b = 0; b < B; ++b) z[b] = u[b][q1];
      DFT<B, SIGN>::run(z);
#pragma unroll
      for (int q2 = 0; q2 < B; ++q2) v[q1 + A * q2] = z[q2];
    }
  }
};
template <int SIGN>
struct DFT<6, SIGN> : DFTComposite<2, 3, SIGN> {};
template <int SIGN>
struct DFT<8, SIGN> : DFTComposite<2, 4, SIGN> {};
template <int SIGN>
struct DFT<12, SIGN> : DFTComposite<4, 3, SIGN> {};
template <int SIGN>
struct DFT<16, SIGN> : DFTComposite<4, 4, SIGN> {};
template <int SIGN>
struct DFT<24, SIGN> : DFTComposite<8, 3, SIGN> {};
template <int SIGN>
struct DFT<32, SIGN> : DFTComposite<4, 8, SIGN> {};

// ---------------------------------------------------------------------------
// Row maps for the 3/2-rule padding (spectral.py:229-258 widen, :276-301 narrow).
// pad_src: padded row r -> coarse row, or -1 inside the zero band.
// trunc_dst: padded row r -> coarse row, -1 = discard, -2 = write zero at n/2.
// With m == n both are the identity (unpadded transforms).
// ---------------------------------------------------------------------------
SRK_DEV int pad_src(int r, int n, int m) {
  const int h = n >> 1;
  if (r <= h) return r;
  if (r >= m - (h - 1)) return r - (m - n);
  return -1;
}
SRK_DEV int trunc_dst(int r, int n, int m, bool zero_nyq) {
  const int h = n >> 1;
  if (r < h) return r;
  if (r == h) return zero_nyq ? -2 : (m == n ? r : -1);
  if (r >= m - (h - 1)) return r - (m - n);
  return -1;
}

// full-axis mode label (grid.py:75-82): Nyquist relabelled +n/2
SRK_DEV double mode_full(int i, int n) { return (double)(i <= (n >> 1) ? i : i - n); }


// ---------------------------------------------------------------------------
// Debug-check builds (make CHECKS=1 -> _lib_chk/libsrk.so, tools/check_build.sh):
// compute-sanitizer is closed on this GPU pool, so the library carries its own
// hazard probes, compiled out of the production build:
//  * SRK_BAR / SRK_WBAR: every CTA / warp barrier is followed by a pseudo-random
//    per-warp delay (up to ~2k cycles, keyed by block, warp, site, launch) --
//    schedule fuzzing: a missing barrier between a shared-memory write and a
//    read by another warp turns into a wrong (or NaN) result under the checks;
//  * srk_poison_smem(): dynamic shared memory is filled with NaN at kernel
//    entry, so a read of a slot no thread wrote propagates into the output
//    (initcheck for shared memory);
//  * SRK_ASSERT: tile index bounds; mbarrier waits trap instead of hanging.
// ---------------------------------------------------------------------------
#ifdef SRK_DEBUG_CHECKS
#include <cstdio>
__device__ __forceinline__ unsigned srk_hash(unsigned a) {
  a ^= a >> 16;
  a *= 0x7feb352dU;
  a ^= a >> 15;
  a *= 0x846ca68bU;
  a ^= a >> 16;
  return a;
}
__device__ __forceinline__ void srk_fuzz(unsigned site) {
  const unsigned h = srk_hash(blockIdx.x * 0x9E3779B9U ^ (threadIdx.x >> 5) * 0x85EBCA6BU ^ site * 0xC2B2AE35U ^
                              (unsigned)(clock64() >> 20));
  const long long t0 = clock64();
  const long long d = (h & 7u) == 0 ? 0 : (long long)(h >> 21);  // 0 .. 2047 cycles
  while (clock64() - t0 < d) {
  }
}
#define SRK_BAR()        \
  do {                   \
    __syncthreads();     \
    srk_fuzz(__LINE__);  \
  } while (0)
#define SRK_WBAR()       \
  do {                   \
    __syncwarp();        \
    srk_fuzz(__LINE__);  \
  } while (0)
#define SRK_ASSERT(c)                                                                              \
  do {                                                                                             \
    if (!(c)) {                                                                                    \
      printf("srk check failed: %s (%s:%d) block %d thread %d\n", #c, __FILE__, __LINE__, blockIdx.x, \
             threadIdx.x);                                                                         \
      __trap();                                                                                    \
    }                                                                                              \
  } while (0)
__device__ __forceinline__ void srk_poison_smem(void* base) {
  unsigned n;
  asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(n));
  unsigned long long* p = (unsigned long long*)base;
  for (unsigned i = threadIdx.x; i < n / 8; i += blockDim.x) p[i] = 0x7FF8DEADBEEF0000ULL;  // quiet NaN
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // before TMA / bulk copies overwrite it
  __syncthreads();
}
#else
#define SRK_BAR() __syncthreads()
#define SRK_WBAR() __syncwarp()
#define SRK_ASSERT(c) \
  do {                \
  } while (0)
__device__ __forceinline__ void srk_poison_smem(void*) {}
#endif

// ---------------------------------------------------------------------------
// Programmatic dependent launch (PDL).  Every libsrk kernel is launched with
// cudaLaunchAttributeProgrammaticStreamSerialization (host_util.cuh
// srk_launch), so the next kernel of a stream is scheduled while this one's
// last wave drains and runs its prologue (shared twiddle table, mbarriers)
// early.  Rules that keep it exact: each kernel signals launch_dependents at its
// start (all its CTAs are then resident or done, so a waiting dependent can
// never block it), and calls pdl_wait() -- which returns once the previous grid
// of the stream has completed and its memory is visible -- before it touches
// any global data another kernel produces or consumes.  Without the attribute
// (or after a non-kernel stream operation) both are no-ops.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" :::); }

// ---------------------------------------------------------------------------
// mbarrier + 1D TMA bulk copy (sm_90+ PTX; used on sm_100a)
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
#ifdef SRK_DEBUG_CHECKS
  {
    const long long t0 = clock64();
    unsigned done = 0;
    while (!done) {
      asm volatile(
          "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
          : "=r"(done)
          : "r"(smem_u32(bar)), "r"(phase)
          : "memory");
      SRK_ASSERT(clock64() - t0 < (1LL << 34));  // ~8 s: a lost transaction, not a slow copy
    }
    return;
  }
#endif
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// 4D TMA tile load / store (columns, column group, rows, planes)
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* tm, int c0, int c1, int c2, int c3,
                                            unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
      "%5}], [%6];" ::"r"(smem_u32(dst)),
      "l"((unsigned long long)tm), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load_5d(void* dst, const CUtensorMap* tm, int c0, int c1, int c2, int c3,
                                            int c4, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
      "%5, %6}], [%7];" ::"r"(smem_u32(dst)),
      "l"((unsigned long long)tm), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store_4d(const CUtensorMap* tm, const void* src, int c0, int c1, int c2, int c3) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
                   (unsigned long long)tm),
               "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
               : "memory");
}

// 3D TMA tile load (cp.async.bulk.tensor) completing on an mbarrier; the tensor
// map is a __grid_constant__ kernel parameter.
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* tm, int c0, int c1, int c2,
                                            unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(smem_u32(dst)),
      "l"((unsigned long long)tm), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

// L2 prefetch of a contiguous global range (16 B aligned, multiple of 16 B)
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

// 1D bulk copy shared -> global (bulk-group completion) and the proxy fence
// that orders generic-proxy smem writes before it.
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit_and_wait_read() {
  asm volatile("cp.async.bulk.commit_group;\ncp.async.bulk.wait_group.read 0;" ::: "memory");
}

// 3D TMA tile store (bulk-group completion)
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* tm, const void* src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                   (unsigned long long)tm),
               "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}

// cp.async (16 B, L2-only caching) global -> shared
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
}
