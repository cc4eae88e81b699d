"""ctypes binding of libpdz.so (include/pdz.h) plus device-buffer plumbing.

The CUDA library is the only compute path: if it is missing or no CUDA device
is visible, every call raises -- there is no CPU fallback.  PyTorch is used
only to own device memory and to provide the current CUDA stream.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

__all__ = [
    "LIB_PATH",
    "EXPORTED_SYMBOLS",
    "SolveParams",
    "lib",
    "check",
    "device",
    "stream_ptr",
    "workspace",
    "LAMBDA_MODES_C",
]

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)),
                        os.environ.get("PDZ_LIB_NAME", "libpdz.so"))  # libpdz_prof.so: profiling

PDZ_OK, PDZ_EINVAL, PDZ_ENONFINITE, PDZ_ECUDA, PDZ_EWORKSPACE = 0, 1, 2, 3, 4

LAMBDA_MODES_C = {"as-printed": 0, "prose": 1, "zero": 2, "const": 3}


class SolveParams(ctypes.Structure):
    """pdz_solve_params (include/pdz.h)."""

    _fields_ = [
        ("height", ctypes.c_int32),
        ("width", ctypes.c_int32),
        ("planes", ctypes.c_int32),
        ("channels", ctypes.c_int32),
        ("kernel_size", ctypes.c_int32),
        ("edge_preserving", ctypes.c_int32),
        ("max_iters", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
        ("sigma", ctypes.c_double),
        ("epsilon", ctypes.c_double),
        ("tau", ctypes.c_double),
        ("rel_tol", ctypes.c_double),
    ]


_vp = ctypes.c_void_p
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_f64 = ctypes.c_double
_sz = ctypes.c_size_t
_pp = ctypes.POINTER(SolveParams)

# name -> (restype, argtypes); every symbol include/pdz.h declares.
_SIGNATURES = {
    "pdz_version": (_i32, []),
    "pdz_last_error": (ctypes.c_char_p, []),
    "pdz_gaussian_taps": (_i32, [_f64, _i32, _vp]),
    "pdz_dark_channel_workspace_bytes": (_sz, [_i32, _i32]),
    "pdz_dark_channel": (_i32, [_vp, _i32, _i32, _i32, _i32, _vp, _i32, _vp, _vp, _sz, _vp]),
    "pdz_multiscale_dark_channel": (
        _i32, [_vp, _i32, _i32, _i32, _i32, _vp, _vp, _vp, _i32, _vp, _vp, _sz, _vp]),
    "pdz_airlight_count": (_i64, [_i32, _i32, _f64]),
    "pdz_airlight_workspace_bytes": (_sz, [_i32, _i32, _f64]),
    "pdz_atmospheric_light": (
        _i32, [_vp, _i32, _i32, _i32, _i32, _vp, _f64, _vp, _vp, _vp, _sz, _vp]),
    "pdz_transmission": (_i32, [_vp, _i32, _i32, _f64, _vp, _vp]),
    "pdz_solver_fields": (
        _i32, [_vp, _i32, _i32, _i32, _i32, _vp, _vp, _f64, _i32, _f64, _f64, _vp, _vp, _vp,
               _vp]),
    "pdz_adaptive_lambda": (_i32, [_vp, _i64, _i32, _f64, _f64, _vp, _vp]),
    "pdz_diffusion_coefficient": (_i32, [_vp, _i64, _f64, _vp, _vp]),
    "pdz_tau_bound_workspace_bytes": (_sz, [_pp]),
    "pdz_tau_bound": (_i32, [_pp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "pdz_tau_bound_f64": (_i32, [_pp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "pdz_tau_bound_hwc": (_i32, [_pp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "pdz_divergence": (_i32, [_pp, _vp, _vp, _vp]),
    "pdz_divergence_f64": (_i32, [_pp, _vp, _vp, _vp]),
    "pdz_gaussian_workspace_bytes": (_sz, [_pp, _i32]),
    "pdz_gaussian": (_i32, [_pp, _vp, _vp, _vp, _sz, _vp]),
    "pdz_gaussian_f64": (_i32, [_pp, _vp, _vp, _vp, _sz, _vp]),
    "pdz_step_workspace_bytes": (_sz, [_pp]),
    "pdz_fixed_point_step": (_i32, [_pp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "pdz_solve_state_bytes": (_sz, [_pp]),
    "pdz_fixed_point_solve_async": (_i32, [_pp, _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "pdz_fixed_point_sweeps_from": (
        _i32, [_pp, _vp, _vp, _vp, _i32, _i32, _vp, _vp, _vp, _vp, _sz, _vp]),
    "pdz_front_end_batch_workspace_bytes": (_sz, [_i32, _i32, _i32, _i32, _f64]),
    "pdz_front_end_batch": (
        _i32, [_vp, _i32, _i32, _i32, _i32, _i32, _vp, _vp, _i32, _f64, _f64, _f64, _i32, _f64,
               _f64, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "pdz_slab_layout": (_i32, [_pp, _vp, _i32]),
    "pdz_fixed_point_sweeps_resident": (
        _i32, [_pp, _vp, _vp, _vp, _i32, _i32, _i32, _vp, _vp, _vp, _sz, _vp]),
    "pdz_fixed_point_step_rows": (_i32, [_pp, _vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _vp,
                                         _vp, _vp, _sz, _vp]),
    "pdz_solve_workspace_bytes": (_sz, [_pp]),
    "pdz_fixed_point_solve": (
        _i32, [_pp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "pdz_fixed_point_sweeps_async": (_i32, [_pp, _vp, _vp, _vp, _sz, _vp]),
    "pdz_solve_result_plane": (_vp, [_pp, _vp, _i32, _i32]),
    "pdz_time_sweep_kernels": (None, [_i32]),
    "pdz_last_sweep_kernel_ms": (ctypes.c_float, []),
    "pdz_solve_kernel_launches": (_i64, [_pp]),
    "pdz_sweep_kernel_kind": (_i32, [_pp]),
    "pdz_solve_plan_info": (_i32, [_pp, _vp, _i32]),
    "pdz_solve_kernel_name": (_i32, [_pp, ctypes.c_char_p, _i32]),
    "pdz_clamp_interleave": (_i32, [_vp, _i32, _i32, _i32, _vp, _i32, _vp]),
    "pdz_quantize_u8": (_i32, [_vp, ctypes.c_int64, _vp, _vp, _vp]),
    "pdz_synthesize_haze": (_i32, [_vp, _vp, _vp, ctypes.c_int64, _i32, _vp, _vp]),
    "pdz_compare_workspace_bytes": (_sz, []),
    "pdz_compare": (_i32, [_vp, _vp, ctypes.c_int64, _vp, _vp, _vp, _sz, _vp]),
    "pdz_guided_workspace_bytes": (_sz, [_i32, _i32]),
    "pdz_box_mean": (_i32, [_vp, _i32, _i32, _i32, _vp, _vp, _sz, _vp]),
    "pdz_guided_filter": (_i32, [_vp, _vp, _i32, _i32, _i32, _f64, _vp, _vp, _sz, _vp]),
    "pdz_refine_transmission": (
        _i32, [_vp, _i32, _i32, _i32, _i32, _vp, _i32, _f64, _vp, _vp, _sz, _vp]),
}

EXPORTED_SYMBOLS = tuple(_SIGNATURES)

_lock = threading.Lock()
_lib = None


def lib():
    """Load libpdz.so (once).  Raises if the CUDA library was never built."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise RuntimeError(
                        f"CUDA library {LIB_PATH} is missing; build it with "
                        "`python -c 'import __graft_entry__ as g; g.build()'` -- there is no "
                        "CPU fallback")
                handle = ctypes.CDLL(LIB_PATH)
                for name, (res, args) in _SIGNATURES.items():
                    fn = getattr(handle, name)
                    fn.restype = res
                    fn.argtypes = args
                _lib = handle
    return _lib


def check(rc: int) -> None:
    """Map a pdz status code onto the reference's exception types."""
    if rc == PDZ_OK:
        return
    msg = (lib().pdz_last_error() or b"").decode(errors="replace")
    if rc == PDZ_ENONFINITE:
        raise FloatingPointError(msg)
    if rc in (PDZ_EINVAL, PDZ_EWORKSPACE):
        raise ValueError(msg)
    raise RuntimeError(msg or f"pdz error {rc}")


PLAN_FIELDS = ("kind", "ctas", "ctas_per_strip", "bonus", "geometry", "radius",
               "partials_per_plane", "strips", "block_rows", "threads", "stop_rule",
               "channel_inner")


class trace_range:
    """NVTX range around a pipeline stage (front end, solve, result copies,
    slab blocks, halo exchange) for nsys / ncu timelines; off unless PDZ_NVTX=1
    (tracing)."""

    enabled = os.environ.get("PDZ_NVTX", "") == "1"

    def __init__(self, name: str):
        self.name = name

    def __enter__(self):
        if self.enabled:
            import torch

            torch.cuda.nvtx.range_push(self.name)
        return self

    def __exit__(self, *exc):
        if self.enabled:
            import torch

            torch.cuda.nvtx.range_pop()
        return False


def plan_info(params) -> dict:
    """The launch plan of a solve (pdz_solve_plan_info; host only)."""
    buf = (ctypes.c_int32 * len(PLAN_FIELDS))()
    check(lib().pdz_solve_plan_info(ctypes.byref(params), buf, len(PLAN_FIELDS)))
    return dict(zip(PLAN_FIELDS, list(buf)))


def kernel_name(params) -> str:
    """Name of the sweep kernel template a solve launches (pdz_solve_kernel_name)."""
    buf = ctypes.create_string_buffer(128)
    check(lib().pdz_solve_kernel_name(ctypes.byref(params), buf, 128))
    return buf.value.decode()


def device():
    """The CUDA device computations run on (torch's current device)."""
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("paper_2506_08793_b200 needs a CUDA device (B200, sm_100a); "
                           "no CUDA device is visible and there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr():
    import torch

    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


_ws_cache: dict = {}
_ws_lock = threading.Lock()


def workspace(nbytes: int, tag: str = "default"):
    """A cached device scratch tensor of at least nbytes (per device, tag, thread).

    Reusing the same buffer keeps the library's CUDA-graph cache warm."""
    import torch

    dev = device()
    key = (dev.index, tag, threading.get_ident())
    nbytes = max(int(nbytes), 256)
    with _ws_lock:
        buf = _ws_cache.get(key)
        if buf is None or buf.numel() < nbytes:
            buf = torch.empty(nbytes, dtype=torch.uint8, device=dev)
            _ws_cache[key] = buf
    return buf


def ptr(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def as_f64_array(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.float64))
