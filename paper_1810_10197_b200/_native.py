"""ctypes binding of libsrk (include/srk.h).

The product's compute path is this library; there is no CPU fallback.  Loading
fails loudly when the shared object is missing, and every compute entry point
raises when no CUDA device is present.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# SRK_LIB_PATH: load another build of the same sources (A/B timing of a change, tools/ab_lib.sh)
LIB_PATH = os.environ.get("SRK_LIB_PATH") or os.path.join(_HERE, "_lib", "libsrk.so")

SRK_OK = 0
SRK_ERR_INVALID = 1
SRK_ERR_UNSUPPORTED = 2
SRK_ERR_CUDA = 3
SRK_ERR_WORKSPACE = 4

# Every symbol include/srk.h declares (checked by tests/test_native_abi.py).
EXPORTS = (
    "srk_abi_version", "srk_last_error", "srk_plan_create", "srk_plan_destroy",
    "srk_plan_workspace_bytes", "srk_plan_set_workspace", "srk_rhs", "srk_rhs_combine", "srk_widen",
    "srk_narrow", "srk_forward_transform", "srk_inverse_transform", "srk_curl",
    "srk_leray_project", "srk_combine", "srk_step_reduce", "srk_band_energy",
    "srk_band_scale", "srk_rhs_launch_count", "srk_rhs_timed", "srk_plan_create_slab", "srk_slab_sizes",
    "srk_slab_forward", "srk_slab_middle", "srk_slab_finish", "srk_debug_phase_buffer",
    "srk_slab_forward_kz", "srk_slab_inverse_y_kz", "srk_slab_zpass", "srk_slab_forward_y_kz",
    "srk_slab_forward_x_kz", "srk_slab_project", "srk_store_mapped", "srk_slab_set_peers",
    "srk_slab_forward_kz_peer", "srk_slab_forward_y_kz_peer", "srk_ipc_export", "srk_ipc_import", "srk_ipc_close",
    "srk_rhs_refresh", "srk_probe", "srk_combine_scaled", "srk_rhs_combine_scaled", "srk_step_reduce_scaled",
    "srk_build_info", "srk_source_hash", "srk_plan_layout",
)

_lib = None

# Number of libsrk kernels launched through the Python API (bench.py's
# gpu_launches claim reads the difference around its timed region).
LAUNCHES = 0


def count(n):
    global LAUNCHES
    LAUNCHES += int(n)


class SrkError(RuntimeError):
    """A libsrk call failed (CUDA error, workspace, unsupported size)."""


def load():
    """Load libsrk.so (once) and declare its signatures."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"libsrk.so not built at {LIB_PATH}; run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback for the B200 path)")
    lib = ctypes.CDLL(LIB_PATH)
    c_int, c_dbl, vp, i64 = ctypes.c_int, ctypes.c_double, ctypes.c_void_p, ctypes.c_int64
    P = ctypes.POINTER
    sig = {
        "srk_abi_version": (c_int, []),
        "srk_last_error": (ctypes.c_char_p, []),
        "srk_plan_create": (c_int, [P(vp), c_int, P(i64), P(c_dbl), c_int, c_int]),
        "srk_plan_destroy": (None, [vp]),
        "srk_plan_workspace_bytes": (c_int, [vp, P(i64)]),
        "srk_plan_set_workspace": (c_int, [vp, vp, i64]),
        "srk_rhs": (c_int, [vp, vp, vp, c_dbl, c_dbl, c_dbl, vp]),
        "srk_rhs_combine": (c_int, [vp, vp, vp, c_dbl, c_dbl, c_dbl, vp, c_int, P(vp), P(c_dbl), c_dbl, vp, vp]),
        "srk_widen": (c_int, [vp, vp, c_int, vp, vp]),
        "srk_narrow": (c_int, [vp, vp, c_int, vp, vp]),
        "srk_forward_transform": (c_int, [vp, vp, c_int, vp, vp]),
        "srk_inverse_transform": (c_int, [vp, vp, c_int, vp, vp]),
        "srk_curl": (c_int, [vp, vp, vp, vp]),
        "srk_leray_project": (c_int, [vp, vp, vp, vp]),
        "srk_combine": (c_int, [i64, vp, c_int, P(vp), P(c_dbl), vp, vp]),
        "srk_step_reduce": (c_int, [vp, vp, vp, c_int, P(vp), P(c_dbl), vp, c_int, c_dbl, c_dbl, c_int, vp, vp]),
        "srk_band_energy": (c_int, [vp, vp, c_int, vp, vp, c_int, vp, vp]),
        "srk_band_scale": (c_int, [vp, vp, c_int, vp, c_int, c_dbl, vp]),
        "srk_store_mapped": (c_int, [vp, vp, c_int, vp]),
        "srk_probe": (c_int, [c_int, c_int, c_int, vp, vp, P(c_dbl)]),
        "srk_build_info": (c_int, []),
        "srk_plan_layout": (c_int, [vp, P(c_int), P(c_int)]),
        "srk_source_hash": (ctypes.c_char_p, []),
        "srk_combine_scaled": (c_int, [i64, vp, c_int, P(vp), P(c_dbl), vp, vp, vp]),
        "srk_rhs_combine_scaled": (c_int, [vp, vp, vp, c_dbl, c_dbl, c_dbl, vp, c_int, P(vp), P(c_dbl), c_dbl, vp,
                                           vp, vp]),
        "srk_step_reduce_scaled": (c_int, [vp, vp, vp, c_int, P(vp), P(c_dbl), vp, vp, c_int, c_dbl, c_dbl, c_int,
                                           vp, vp]),
        "srk_rhs_refresh": (c_int, [vp, vp, vp, c_dbl, c_dbl, c_dbl, c_dbl, vp, vp, vp]),
        "srk_slab_set_peers": (c_int, [vp, P(vp), P(vp), c_int]),
        "srk_slab_forward_kz_peer": (c_int, [vp, vp, c_int, c_int, vp]),
        "srk_slab_forward_y_kz_peer": (c_int, [vp, c_int, c_int, vp]),
        "srk_ipc_export": (c_int, [vp, vp, P(i64)]),
        "srk_ipc_import": (c_int, [vp, i64, P(vp)]),
        "srk_ipc_close": (c_int, [vp, i64]),
        "srk_rhs_launch_count": (c_int, [vp]),
        "srk_rhs_timed": (c_int, [vp, vp, vp, c_dbl, c_dbl, c_dbl, vp, P(ctypes.c_float), c_int]),
        "srk_plan_create_slab": (c_int, [P(vp), P(i64), P(c_dbl), c_int, c_int, c_int]),
        "srk_slab_sizes": (c_int, [vp, P(i64), P(i64)]),
        "srk_slab_forward": (c_int, [vp, vp, vp, vp]),
        "srk_slab_middle": (c_int, [vp, vp, vp, vp]),
        "srk_slab_finish": (c_int, [vp, vp, vp, vp, c_dbl, c_dbl, c_dbl, vp]),
        "srk_debug_phase_buffer": (c_int, [vp, vp, c_int]),
        "srk_slab_forward_kz": (c_int, [vp, vp, vp, c_int, c_int, vp]),
        "srk_slab_inverse_y_kz": (c_int, [vp, vp, c_int, c_int, vp]),
        "srk_slab_zpass": (c_int, [vp, vp]),
        "srk_slab_forward_y_kz": (c_int, [vp, vp, c_int, c_int, vp]),
        "srk_slab_forward_x_kz": (c_int, [vp, vp, c_int, c_int, vp]),
        "srk_slab_project": (c_int, [vp, vp, vp, c_dbl, c_dbl, c_dbl, vp]),
    }
    for name, (res, args) in sig.items():
        try:
            fn = getattr(lib, name)
        except AttributeError:
            if os.environ.get("SRK_LIB_PATH"):  # an older build under A/B timing: bind what it has
                continue
            raise
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc, what=""):
    """Map a non-zero libsrk status to the reference's exception classes."""
    if rc == SRK_OK:
        return
    msg = load().srk_last_error().decode(errors="replace")
    if rc == SRK_ERR_INVALID:
        raise ValueError(msg)
    raise SrkError(f"{what}: {msg}" if what else msg)


def ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def stream_ptr(stream=None):
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


_HOST_RESULT = {}


def host_result(n):
    """Pinned host float64[n] a kernel can store into directly (UVA-mapped), for
    small results read by the host: no cudaMemcpy, so nothing queues behind bulk
    copies on the copy engines.  One cached buffer per (thread, size): callers
    wait for the stream (``wait_stream_point``) and copy the values out before the
    next call reuses it (a fresh pinned allocation per call cost ~1 ms)."""
    import threading

    import torch

    key = (threading.get_ident(), int(n))
    buf = _HOST_RESULT.get(key)
    if buf is None:
        buf = _HOST_RESULT[key] = torch.empty(int(n), dtype=torch.float64, pin_memory=True)
    return buf


def fetch_small(t, stream=None):
    """Small CUDA float64 tensor -> CPU tensor through a kernel store into mapped
    pinned memory (srk_store_mapped) instead of a cudaMemcpy (which would queue
    behind a large HostMirror copy on the copy engine)."""
    import torch

    t = t.to(torch.float64).contiguous()
    buf = host_result(t.numel())
    check(load().srk_store_mapped(ptr(t), ctypes.c_void_p(buf.data_ptr()), t.numel(), stream_ptr(stream)),
          "srk_store_mapped")
    count(1)
    wait_stream_point(stream)
    return buf.clone()


def wait_stream_point(stream=None):
    """Block the host until the work queued so far on ``stream`` (default: current) is done."""
    import torch

    ev = torch.cuda.Event()
    ev.record(stream if stream is not None else torch.cuda.current_stream())
    ev.synchronize()


def ptr_array(tensors):
    arr = (ctypes.c_void_p * max(1, len(tensors)))()
    for i, t in enumerate(tensors):
        arr[i] = t.data_ptr()
    return arr


def dbl_array(vals):
    arr = (ctypes.c_double * max(1, len(vals)))()
    for i, v in enumerate(vals):
        arr[i] = float(v)
    return arr


# ---------------------------------------------------------------------------
# NVTX ranges (SURVEY §5 tracing): SRK_NVTX=1 wraps every RHS evaluation, adaptive
# attempt and step reduction in a named range for nsys / ncu --nvtx timelines.
# Off by default: a no-op context manager, nothing on the hot path.
# ---------------------------------------------------------------------------
NVTX = os.environ.get("SRK_NVTX", "0") not in ("", "0")


class _NoRange:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


_NO_RANGE = _NoRange()


class _Range:
    __slots__ = ("name",)

    def __init__(self, name):
        self.name = name

    def __enter__(self):
        import torch
        torch.cuda.nvtx.range_push(self.name)
        return self

    def __exit__(self, *a):
        import torch
        torch.cuda.nvtx.range_pop()
        return False


def nvtx(name):
    """``with nvtx("srk_rhs"):`` -- an NVTX range when SRK_NVTX=1, else a no-op."""
    return _Range(name) if NVTX else _NO_RANGE
