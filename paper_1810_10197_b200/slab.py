"""Slab-decomposed multi-GPU RHS: one process per GPU, NCCL all-to-all.

Rank r of P owns the y-slab ``(ncomp, n0, n1/P, n2/2+1)`` of the spectral
state (global rows y in [r*n1/P, (r+1)*n1/P)).  One RHS evaluation:

    K1 (x-inverse of u, kx u1, kx u2)   -> send1 [dest][s][x_loc][y_loc][kz]  (5 signals)
    all-to-all #1 (equal splits)         -> recv1 [src][s][x_loc][y_loc][kz]  (x-slab)
    K2 (curl completed on load) + K3 + K4 -> send2 [dest][o][x_loc][y_loc][kz]
    all-to-all #2                        -> recv2 [src][o][x_loc][y_loc][kz]  (y-slab)
    K5 + K6 (x-forward + projection)     -> f (y-slab)

The exchange happens after the x padding and before the y padding, so it moves
8*S_x complex values per RHS (5 K1 signals + 3 products; SURVEY §8e counts 9
with the curl finished before the exchange) instead of 9*S_xy.  The kernels write
the send layouts and read the receive layouts directly; there is no pack or
unpack pass.  Reductions (error norm, E_kin, eps, Z, forcing band energy) are
per-slab device sums, all-gathered and added in rank order so every rank takes
the same accept/reject decision bit for bit.

With ``chunks > 1`` (SURVEY §8e "pipeline over kz-chunks") the same kernel
groups run per kz chunk and each chunk's exchange is issued asynchronously, so
K1 of chunk c+1 and K2 of chunk c-1 overlap the all-to-all of chunk c (and K4 /
K5 likewise for the second exchange); only the z-pass (K3, needs every kz of a
pencil) separates the two halves.

The stage functions are pluggable (``backend``) so the CPU test-suite can run
the same orchestration on gloo with a numpy restatement of the three kernel
groups (tests/slab_numpy_backend.py).
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _native
from .grid import Grid
from .physics import PhysParams


def slab_geometry(grid: Grid, nranks: int, density=False):
    """Buffer sizes (complex elements) and local extents of the decomposition."""
    if grid.dims != 3:
        raise ValueError("slab decomposition is 3D only (2D configs run as replicas)")
    n0, n1, n2 = grid.shape
    m0 = 3 * n0 // 2
    if n1 % nranks or m0 % nranks:
        raise ValueError(f"need nranks | n1 ({n1}) and nranks | 3*n0/2 ({m0})")
    K = n2 // 2 + 1
    S = 3 + 3 + (1 if density else 0)
    S1 = 5 + (1 if density else 0)  # K1 signals [u0, u1, u2, kx u1, kx u2, (rho)]
    So = 6 if density else 3
    ny, mx = n1 // nranks, m0 // nranks
    return dict(n0=n0, n1=n1, n2=n2, K=K, m0=m0, m1=3 * n1 // 2, m2=3 * n2 // 2, ny=ny, mx=mx, S=S, S1=S1,
                So=So, send1=S1 * m0 * ny * K, send2=So * mx * n1 * K)


def scatter_slab(y_full, rank, nranks):
    """(c, n0, n1, K) -> this rank's y-slab (contiguous copy)."""
    ny = y_full.shape[2] // nranks
    return y_full[:, :, rank * ny:(rank + 1) * ny].contiguous() if isinstance(y_full, torch.Tensor) else \
        np.ascontiguousarray(y_full[:, :, rank * ny:(rank + 1) * ny])


class CudaSlabBackend:
    """The three libsrk kernel groups of one rank (srk_slab_forward / _middle / _finish)."""

    def __init__(self, grid: Grid, params: PhysParams, rank: int, nranks: int, density=False):
        self.lib = _native.load()
        self.params = params
        shape = (ctypes.c_int64 * 3)(*grid.shape)
        lengths = (ctypes.c_double * 3)(*grid.lengths)
        h = ctypes.c_void_p()
        _native.check(self.lib.srk_plan_create_slab(ctypes.byref(h), shape, lengths, int(density), nranks, rank),
                      "srk_plan_create_slab")
        self.h = h
        nb = ctypes.c_int64()
        _native.check(self.lib.srk_plan_workspace_bytes(h, ctypes.byref(nb)))
        self.ws = torch.empty(max(nb.value, 256), dtype=torch.uint8, device="cuda")
        _native.check(self.lib.srk_plan_set_workspace(h, ctypes.c_void_p(self.ws.data_ptr()), self.ws.numel()))
        self.device = torch.device("cuda", torch.cuda.current_device())

    def empty(self, n):
        return torch.empty(n, dtype=torch.complex128, device=self.device)

    def forward(self, y, send1):
        _native.check(self.lib.srk_slab_forward(self.h, _native.ptr(y), _native.ptr(send1), _native.stream_ptr()))
        _native.count(1)

    def middle(self, recv1, send2):
        _native.check(self.lib.srk_slab_middle(self.h, _native.ptr(recv1), _native.ptr(send2),
                                               _native.stream_ptr()))
        _native.count(3)

    def finish(self, recv2, y, f):
        p = self.params
        _native.check(self.lib.srk_slab_finish(self.h, _native.ptr(recv2), _native.ptr(y), _native.ptr(f),
                                               1.0 / p.reynolds, float(p.richardson),
                                               float(p.reynolds) * float(p.prandtl), _native.stream_ptr()))
        _native.count(2)

    # ---- kz-chunked kernel groups (pipelined RHS) ----
    def forward_kz(self, y, send1_c, k0, kc):
        _native.check(self.lib.srk_slab_forward_kz(self.h, _native.ptr(y), _native.ptr(send1_c), k0, kc,
                                                   _native.stream_ptr()))
        _native.count(1)

    def inverse_y_kz(self, recv1_c, k0, kc):
        _native.check(self.lib.srk_slab_inverse_y_kz(self.h, _native.ptr(recv1_c), k0, kc, _native.stream_ptr()))
        _native.count(1)

    def zpass(self):
        _native.check(self.lib.srk_slab_zpass(self.h, _native.stream_ptr()))
        _native.count(1)

    def forward_y_kz(self, send2_c, k0, kc):
        _native.check(self.lib.srk_slab_forward_y_kz(self.h, _native.ptr(send2_c), k0, kc, _native.stream_ptr()))
        _native.count(1)

    def forward_x_kz(self, recv2_c, k0, kc):
        _native.check(self.lib.srk_slab_forward_x_kz(self.h, _native.ptr(recv2_c), k0, kc, _native.stream_ptr()))
        _native.count(1)

    def project(self, y, f):
        p = self.params
        _native.check(self.lib.srk_slab_project(self.h, _native.ptr(y), _native.ptr(f), 1.0 / p.reynolds,
                                                float(p.richardson), float(p.reynolds) * float(p.prandtl),
                                                _native.stream_ptr()))
        _native.count(1)

    # ---- exchange fused into K1 / K4 (peer stores, srk_slab_*_peer) ----
    def set_peers(self, recv1_ptrs, recv2_ptrs):
        n = len(recv1_ptrs)
        a1 = (ctypes.c_void_p * n)(*[ctypes.c_void_p(int(q)) for q in recv1_ptrs])
        a2 = (ctypes.c_void_p * n)(*[ctypes.c_void_p(int(q)) for q in recv2_ptrs])
        _native.check(self.lib.srk_slab_set_peers(self.h, a1, a2, n), "srk_slab_set_peers")

    def forward_kz_peer(self, y, k0, kc):
        _native.check(self.lib.srk_slab_forward_kz_peer(self.h, _native.ptr(y), k0, kc, _native.stream_ptr()))
        _native.count(1)

    def forward_y_kz_peer(self, k0, kc):
        _native.check(self.lib.srk_slab_forward_y_kz_peer(self.h, k0, kc, _native.stream_ptr()))
        _native.count(1)

    def __del__(self):
        try:
            self.lib.srk_plan_destroy(self.h)
        except Exception:
            pass


def ipc_export(t):
    """(64-byte CUDA IPC handle, offset) of a CUDA tensor's storage (srk_ipc_export)."""
    lib = _native.load()
    h = (ctypes.c_char * 64)()
    off = ctypes.c_int64()
    _native.check(lib.srk_ipc_export(_native.ptr(t), h, ctypes.byref(off)), "srk_ipc_export")
    return bytes(h), off.value


def ipc_import(handle, offset):
    """Address of a peer process's buffer in this process (srk_ipc_import)."""
    lib = _native.load()
    buf = ctypes.create_string_buffer(bytes(handle), 64)
    out = ctypes.c_void_p()
    _native.check(lib.srk_ipc_import(buf, int(offset), ctypes.byref(out)), "srk_ipc_import")
    return out.value


def ipc_close(ptr, offset):
    _native.check(_native.load().srk_ipc_close(ctypes.c_void_p(int(ptr)), int(offset)), "srk_ipc_close")


def exchange_peer_tables(recv1, recv2, group=None):
    """All ranks' recv1 / recv2 addresses in this process: own buffers directly,
    the others through CUDA IPC (handles all-gathered over torch.distributed).
    Returns (recv1_ptrs, recv2_ptrs, imported) -- ``imported`` lists the (ptr,
    offset) mappings to close."""
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    mine = (ipc_export(recv1), ipc_export(recv2))
    allh = [None] * world
    dist.all_gather_object(allh, mine, group=group)
    p1, p2, imported = [], [], []
    for r in range(world):
        if r == rank:
            p1.append(recv1.data_ptr())
            p2.append(recv2.data_ptr())
            continue
        (h1, o1), (h2, o2) = allh[r]
        a, b = ipc_import(h1, o1), ipc_import(h2, o2)
        p1.append(a)
        p2.append(b)
        imported += [(a, o1), (b, o2)]
    return p1, p2, imported


def dist_stream_barrier(group=None):
    """Stream-ordered barrier for the peer-store exchange: a one-element NCCL
    all-reduce on the compute stream completes on a rank only after every rank
    has reached it, i.e. after every rank's preceding K1 / K4 (and its NVLink
    stores) finished."""
    import torch.distributed as dist

    flag = {}

    def barrier():
        t = flag.get("t")
        if t is None:
            t = flag["t"] = torch.zeros(1, dtype=torch.float32, device=torch.device("cuda", torch.cuda.current_device()))
        dist.all_reduce(t, group=group)

    return barrier


def dist_all_to_all(group=None, async_op=False):
    """Equal-split all-to-all over torch.distributed (NCCL on GPUs, gloo on CPU).

    ``async_op=True`` returns the work handle: ``wait()`` orders the caller's
    current CUDA stream after the exchange without blocking the host, so the
    kernels queued meanwhile overlap it (the kz-chunk pipeline)."""
    import torch.distributed as dist

    def exchange(recv, send):
        if recv.is_complex():  # NCCL / gloo move the (re, im) float64 pairs
            recv, send = torch.view_as_real(recv), torch.view_as_real(send)
        return dist.all_to_all_single(recv, send, group=group, async_op=async_op)

    return exchange


def kz_chunks(K, n):
    """Split [0, K) into n chunks whose widths are multiples of 4 (the strided
    tile width), the remainder going to the last one."""
    n = max(1, min(n, K // 4 if K >= 4 else 1))
    base = (K // n) // 4 * 4 or K
    out, k0 = [], 0
    for c in range(n):
        kc = base if c < n - 1 else K - k0
        if kc <= 0:
            break
        out.append((k0, kc))
        k0 += kc
    return out


def dist_sum_in_rank_order(group=None):
    """Deterministic all-reduce of a small vector: all-gather, then add in rank order."""
    import torch.distributed as dist

    def reduce(q):
        q = torch.as_tensor(q, dtype=torch.float64)
        t = q.to(dist_device(group))
        parts = [torch.empty_like(t) for _ in range(dist.get_world_size(group))]
        dist.all_gather(parts, t, group=group)
        acc = parts[0].clone()
        for p in parts[1:]:
            acc += p
        # kernel store into mapped host memory (no cudaMemcpy behind HostMirror copies)
        return (_native.fetch_small(acc) if acc.is_cuda else acc).tolist()

    return reduce


def dist_device(group=None):
    import torch.distributed as dist

    return torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else \
        torch.device("cpu")


class SlabFlowRHS:
    """``f(t, y_slab)`` for one rank of a slab-decomposed grid (drop-in for FlowRHS)."""

    def __init__(self, grid: Grid, params: PhysParams, rank: int, nranks: int, density=False, backend=None,
                 exchange=None, chunks=1, peer=False, barrier=None):
        """``chunks`` > 1 pipelines the RHS over kz chunks: the exchange of
        chunk c (asynchronous, ``exchange`` must then return a handle with
        ``wait()``) overlaps the kernels of the neighbouring chunks.

        ``peer=True`` fuses the two all-to-alls into K1 / K4: their row blocks
        are stored straight into the ranks' receive buffers (CUDA IPC peer
        pointers over NVLink, srk_slab_*_peer) and a stream-ordered ``barrier``
        (default: one-element NCCL all-reduce) separates them from the readers;
        no NCCL data movement, the transfer rides on the passes' stores tile by
        tile.  ``peer_tables`` may be given instead of torch.distributed (one
        process driving several emulated ranks)."""
        self.grid, self.params, self.rank, self.nranks = grid, params, rank, nranks
        self.density = bool(density)
        self.geo = slab_geometry(grid, nranks, density)
        self.backend = backend if backend is not None else CudaSlabBackend(grid, params, rank, nranks, density)
        self.chunks = kz_chunks(self.geo["K"], chunks)
        self.pipelined = len(self.chunks) > 1
        if exchange is None:
            exchange = dist_all_to_all(async_op=self.pipelined)
        self.exchange = exchange
        g = self.geo
        self.peer = bool(peer)
        self._imported = []
        if self.peer:
            self.send1 = self.send2 = None
            self.recv1, self.recv2 = self.backend.empty(g["send1"]), self.backend.empty(g["send2"])
            if nranks == 1:
                p1, p2 = [self.recv1.data_ptr()], [self.recv2.data_ptr()]
            else:
                p1, p2, self._imported = exchange_peer_tables(self.recv1, self.recv2)
            self.backend.set_peers(p1, p2)
            self.barrier = barrier if barrier is not None else \
                (dist_stream_barrier() if nranks > 1 else (lambda: None))
            self.chunks = [(0, g["K"])]
            self.pipelined = False
        else:
            self.send1, self.recv1 = self.backend.empty(g["send1"]), self.backend.empty(g["send1"])
            self.send2, self.recv2 = self.backend.empty(g["send2"]), self.backend.empty(g["send2"])
        self.calls = 0

    def close(self):
        """Release the CUDA IPC mappings of the other ranks' receive buffers (peer mode)."""
        for ptr, off in self._imported:
            ipc_close(ptr, off)
        self._imported = []

    @property
    def local_kshape(self):
        g = self.geo
        return (g["n0"], g["ny"], g["K"])

    def _views(self, buf, per_kz, k0, kc):
        return buf[per_kz * k0:per_kz * (k0 + kc)]

    def __call__(self, t, y, out=None):
        f = out if out is not None else (torch.empty_like(y) if isinstance(y, torch.Tensor) else np.empty_like(y))
        if self.peer:
            be, K = self.backend, self.geo["K"]
            be.forward_kz_peer(y, 0, K)        # K1 + all-to-all #1 (peer stores)
            self.barrier()
            be.inverse_y_kz(self.recv1, 0, K)  # K2
            be.zpass()                         # K3
            be.forward_y_kz_peer(0, K)         # K4 + all-to-all #2 (peer stores)
            self.barrier()
            be.forward_x_kz(self.recv2, 0, K)  # K5
            be.project(y, f)                   # K6
            self.calls += 1
            return f
        if not self.pipelined:
            self.backend.forward(y, self.send1)
            self.exchange(self.recv1, self.send1)
            self.backend.middle(self.recv1, self.send2)
            self.exchange(self.recv2, self.send2)
            self.backend.finish(self.recv2, y, f)
            self.calls += 1
            return f
        g, be = self.geo, self.backend
        p1 = g["send1"] // g["K"]  # elements per kz of a send1 chunk (S1 * m0 * ny)
        p2 = g["send2"] // g["K"]
        work = []
        for k0, kc in self.chunks:  # K1 of chunk c+1 overlaps the exchange of chunk c
            s1 = self._views(self.send1, p1, k0, kc)
            be.forward_kz(y, s1, k0, kc)
            work.append(self.exchange(self._views(self.recv1, p1, k0, kc), s1))
        for (k0, kc), w in zip(self.chunks, work):  # K2 of chunk c overlaps the later exchanges
            if w is not None:
                w.wait()
            be.inverse_y_kz(self._views(self.recv1, p1, k0, kc), k0, kc)
        be.zpass()
        work = []
        for k0, kc in self.chunks:
            s2 = self._views(self.send2, p2, k0, kc)
            be.forward_y_kz(s2, k0, kc)
            work.append(self.exchange(self._views(self.recv2, p2, k0, kc), s2))
        for (k0, kc), w in zip(self.chunks, work):
            if w is not None:
                w.wait()
            be.forward_x_kz(self._views(self.recv2, p2, k0, kc), k0, kc)
        be.project(y, f)
        self.calls += 1
        return f


def hit_slab(grid: Grid, rank: int, nranks: int, a=4.0, energy=0.5, seed=42, allreduce=None):
    """Device-side synthetic HIT y-slab for throughput runs (FFT cost is
    data independent): modulus |k| exp(-|k|^2/a^2), uniform random phases from a
    per-rank torch generator, Leray projection, energy scaled to ``energy``.
    Unlike hit_init the kz=0 / n/2 planes are not symmetrised (that couples
    slabs); parity runs use hit_init instead."""
    from .physics import leray_project  # noqa: F401  (slab-local projection below)

    n0, n1, n2 = grid.shape
    ny, K = n1 // nranks, n2 // 2 + 1
    dev = torch.device("cuda", torch.cuda.current_device())
    L = grid.lengths

    def modes(n):
        m = torch.arange(n, dtype=torch.float64, device=dev)
        return torch.where(m > n // 2, m - n, m)

    kx = (modes(n0) * (2 * np.pi / L[0]))[:, None, None]
    ky = (modes(n1)[rank * ny:(rank + 1) * ny] * (2 * np.pi / L[1]))[None, :, None]
    kz = (torch.arange(K, dtype=torch.float64, device=dev) * (2 * np.pi / L[2]))[None, None, :]
    k2 = kx * kx + ky * ky + kz * kz
    gen = torch.Generator(device=dev)
    gen.manual_seed(int(seed) * 7919 + rank)
    u = torch.empty((3, n0, ny, K), dtype=torch.complex128, device=dev)
    for j in range(3):
        ph = torch.rand((n0, ny, K), dtype=torch.float64, device=dev, generator=gen) * (2 * np.pi)
        u[j] = torch.polar(torch.sqrt(k2) * torch.exp(-k2 / a ** 2), ph)
    inv = torch.where(k2 == 0, torch.zeros_like(k2), 1.0 / torch.where(k2 == 0, torch.ones_like(k2), k2))
    kd = (kx * u[0] + ky * u[1] + kz * u[2]) * inv
    u[0] -= kx * kd
    u[1] -= ky * kd
    u[2] -= kz * kd
    u[:, n0 // 2] = 0
    u[..., K - 1] = 0
    w = torch.full((K,), 2.0, dtype=torch.float64, device=dev)
    w[0] = w[-1] = 1.0
    e = float((w * (u.real ** 2 + u.imag ** 2)).sum()) / (2.0 * float(grid.points) ** 2)
    if allreduce is not None:
        e = allreduce([e])[0]
    u *= float(np.sqrt(energy / e))
    return u
