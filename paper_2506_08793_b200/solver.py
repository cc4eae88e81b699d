"""Relaxed fixed-point dehazing solve on B200 (drop-in for pdehaze.solver).

Public functions keep the reference names, signatures, defaults and error
behaviour (pdehaze/solver.py:152-446).  The work runs in libpdz.so:

* `fixed_point_step` / `fixed_point_solve` / `dehaze` -> the fused float32
  sweep kernel (csrc/pdz_sweep.cu), all channels (and, for `dehaze_batch`,
  all images) of a solve in one launch per iteration, iterations replayed
  from a captured CUDA graph, stop rule evaluated on the device;
* the operator probes `divergence_term`, `gaussian_convolve`,
  `tau_stability_bound`, `adaptive_lambda`, `diffusion_coefficient` ->
  float64 kernels (csrc/pdz_ops.cu, pdz_frontend.cu);
* the front end -> csrc/pdz_frontend.cu, pdz_guided.cu (bit-exact).

numpy inputs return float64 numpy outputs like the reference; torch.cuda
tensors stay on the device.  Precision: the solve iterates in float32 (the
north-star contract: max-abs 1e-4 against the float64 reference at the
stable step); see DESIGN.md for the documented deviations.
"""

from __future__ import annotations

import csv
import logging

import threading

import numpy as np

from . import _native as nat
from .config import (ABLATIONS, LAMBDA_MODES, DehazeResult, SolverConfig, SolverTrace,
                     normalize_ablation)
from .image import (clamp01, is_device_array, to_device, to_host, to_host_async,
                    validate_field, validate_image, validate_unit_image)
from .refine import refine_dev
from .scattering import _airlight_dev, _blend_weights, _dark_dev, _device_vec, _unit_range

__all__ = [
    "ABLATIONS",
    "DehazeResult",
    "SolverConfig",
    "SolverTrace",
    "adaptive_lambda",
    "dehaze",
    "dehaze_batch",
    "diffusion_coefficient",
    "divergence_term",
    "fixed_point_solve",
    "fixed_point_step",
    "gaussian_convolve",
    "gaussian_kernel",
    "tau_stability_bound",
    "write_trace_csv",
    "DeviceProblem",
    "prepare_problem",
    "solve_problem",
]

# Same logger name as the reference module so existing log filters keep working
# (the stability warning is asserted on "pdehaze.solver", tests/test_solver.py:126-131).
logger = logging.getLogger("pdehaze.solver")


def _params(h, w, planes, channels, cfg, *, edge_preserving=True, tau=None, max_iters=None,
            rel_tol=None, kernel_size=None, sigma=None, epsilon=None) -> nat.SolveParams:
    p = nat.SolveParams()
    p.height, p.width, p.planes, p.channels = int(h), int(w), int(planes), int(channels)
    p.kernel_size = int(cfg.kernel_size if kernel_size is None else kernel_size)
    p.edge_preserving = 1 if edge_preserving else 0
    p.max_iters = int(cfg.max_iters if max_iters is None else max_iters)
    p.sigma = float(cfg.sigma if sigma is None else sigma)
    p.epsilon = float(cfg.epsilon if epsilon is None else epsilon)
    p.tau = float(cfg.tau if tau is None else tau)
    p.rel_tol = float(cfg.rel_tol if rel_tol is None else rel_tol)
    return p


# --------------------------------------------------------------------------
# operator probes (float64 kernels)
# --------------------------------------------------------------------------

def diffusion_coefficient(grad_magnitude, epsilon: float):
    """D = 1 / (|grad| + epsilon), range (0, 1/eps] (solver.py:152-164)."""
    import torch

    scalar = np.isscalar(grad_magnitude)
    g = grad_magnitude if is_device_array(grad_magnitude) else np.asarray(grad_magnitude,
                                                                          dtype=np.float64)
    if bool((g < 0.0).any()):
        raise ValueError("gradient magnitude must be >= 0")
    if epsilon <= 0.0:
        raise ValueError("epsilon must be > 0")
    g_dev = to_device(np.atleast_1d(g) if not is_device_array(g) else g, torch.float64)
    out = torch.empty_like(g_dev)
    nat.check(nat.lib().pdz_diffusion_coefficient(nat.ptr(g_dev), g_dev.numel(),
                                                  float(epsilon), nat.ptr(out),
                                                  nat.stream_ptr()))
    if scalar:
        return float(out.reshape(-1)[0].item())
    res = to_host(out, grad_magnitude)
    return res.reshape(np.shape(g)) if not is_device_array(grad_magnitude) else res


def divergence_term(u, epsilon: float, edge_preserving: bool = True):
    """div(D(grad u) grad u) with zero flux through the border (solver.py:190-210)."""
    import torch

    f = validate_field(u)
    if f.shape[0] < 2 or f.shape[1] < 2:
        raise ValueError(f"field must be at least 2x2, got {tuple(f.shape)}")
    if epsilon <= 0.0:
        raise ValueError("epsilon must be > 0")
    f_dev = to_device(f, torch.float64)
    out = torch.empty_like(f_dev)
    prm = _params(f_dev.shape[0], f_dev.shape[1], 1, 1, SolverConfig(),
                  edge_preserving=edge_preserving, epsilon=epsilon)
    nat.check(nat.lib().pdz_divergence_f64(prm, nat.ptr(f_dev), nat.ptr(out), nat.stream_ptr()))
    return to_host(out, u)


def gaussian_kernel(sigma: float, kernel_size: int) -> np.ndarray:
    """Sampled 2-D Gaussian normalised to sum 1 (solver.py:213-222): the outer
    product of the library's normalised 1-D factor."""
    if sigma <= 0.0:
        raise ValueError("sigma must be > 0")
    if kernel_size < 1 or kernel_size % 2 == 0:
        raise ValueError(f"kernel_size must be odd and >= 1, got {kernel_size}")
    taps = np.empty(kernel_size, dtype=np.float64)
    nat.check(nat.lib().pdz_gaussian_taps(float(sigma), int(kernel_size), taps.ctypes.data))
    return np.outer(taps, taps)


def gaussian_convolve(field, sigma: float, kernel_size: int):
    """Normalised Gaussian blur with symmetric (edge-inclusive) borders
    (solver.py:225-241), evaluated separably."""
    import torch

    f = validate_field(field)
    if sigma <= 0.0:
        raise ValueError("sigma must be > 0")
    if kernel_size < 1 or kernel_size % 2 == 0:
        raise ValueError(f"kernel_size must be odd and >= 1, got {kernel_size}")
    f_dev = to_device(f, torch.float64)
    out = torch.empty_like(f_dev)
    prm = _params(f_dev.shape[0], f_dev.shape[1], 1, 1, SolverConfig(), sigma=sigma,
                  kernel_size=kernel_size)
    lib = nat.lib()
    ws = nat.workspace(lib.pdz_gaussian_workspace_bytes(prm, 1), "gauss")
    nat.check(lib.pdz_gaussian_f64(prm, nat.ptr(f_dev), nat.ptr(out), nat.ptr(ws), ws.numel(),
                                   nat.stream_ptr()))
    return to_host(out, field)


def adaptive_lambda(transmission, lambda0: float = 0.5, beta: float = 3.0,
                    monotonicity: str = "as-printed"):
    """lambda0 exp(-beta (1 - t)) ("as-printed") or lambda0 exp(-beta t)
    ("prose") (solver.py:244-263)."""
    import torch

    t = validate_field(transmission)
    if float(t.min()) < 0.0 or float(t.max()) > 1.0:
        raise ValueError("transmission values must lie in [0, 1]")
    if lambda0 <= 0.0:
        raise ValueError("lambda0 must be > 0")
    if beta < 0.0:
        raise ValueError("beta must be >= 0")
    if monotonicity not in LAMBDA_MODES:
        raise ValueError(f"monotonicity must be one of {LAMBDA_MODES}")
    t_dev = to_device(t, torch.float64)
    out = torch.empty_like(t_dev)
    nat.check(nat.lib().pdz_adaptive_lambda(nat.ptr(t_dev), t_dev.numel(),
                                            nat.LAMBDA_MODES_C[monotonicity], float(lambda0),
                                            float(beta), nat.ptr(out), nat.stream_ptr()))
    return to_host(out, transmission)


def tau_stability_bound(u, lambda_map, epsilon: float) -> float:
    """2 / (8 max D + max(max lambda, 0)), D edge-preserving (solver.py:266-277)."""
    import torch

    f = validate_field(u)
    lam = validate_field(lambda_map)
    f_dev = to_device(f, torch.float64)
    if tuple(lam.shape) == tuple(f.shape):
        lam_dev = to_device(lam, torch.float64)
        lam_extra = None
    else:  # the reference reduces the two fields independently
        lam_dev = torch.zeros_like(f_dev)
        lam_extra = float(lam.max())
    prm = _params(f_dev.shape[0], f_dev.shape[1], 1, 1, SolverConfig(), epsilon=epsilon)
    lib = nat.lib()
    ws = nat.workspace(lib.pdz_tau_bound_workspace_bytes(prm), "tau")
    bound = torch.empty(1, dtype=torch.float64, device=f_dev.device)
    nat.check(lib.pdz_tau_bound_f64(prm, nat.ptr(f_dev), nat.ptr(lam_dev), nat.ptr(bound),
                                    nat.ptr(ws), ws.numel(), nat.stream_ptr()))
    b = float(bound.item())
    if lam_extra is not None:
        max_d = (2.0 / b) / 8.0
        b = 2.0 / (8.0 * max_d + max(lam_extra, 0.0))
    return b


# --------------------------------------------------------------------------
# the sweep
# --------------------------------------------------------------------------

def fixed_point_step(u, source, lambda_map, cfg: SolverConfig, *, edge_preserving: bool = True,
                     tau: float | None = None):
    """One relaxed update (u + tau r, ||r||_2), r = div(D grad u) - lambda G(u) +
    source (solver.py:280-302), on the fused float32 sweep kernel."""
    import torch

    uu = validate_field(u)
    src = validate_field(source)
    lam = validate_field(lambda_map)
    if tuple(uu.shape) != tuple(src.shape) or tuple(uu.shape) != tuple(lam.shape):
        raise ValueError(f"shape mismatch: u {tuple(uu.shape)}, source {tuple(src.shape)}, "
                         f"lambda {tuple(lam.shape)}")
    step = cfg.tau if tau is None else float(tau)
    h, w = uu.shape
    u_dev = to_device(uu, torch.float32)
    s_dev = to_device(src, torch.float32)
    l_dev = to_device(lam, torch.float32)
    out = torch.empty_like(u_dev)
    prm = _params(h, w, 1, 1, cfg, edge_preserving=edge_preserving, tau=step, max_iters=1)
    lib = nat.lib()
    ws = nat.workspace(lib.pdz_step_workspace_bytes(prm), "step")
    norms = torch.empty(1, dtype=torch.float64, device=u_dev.device)
    nat.check(lib.pdz_fixed_point_step(prm, nat.ptr(u_dev), nat.ptr(out), nat.ptr(s_dev),
                                       nat.ptr(l_dev), nat.ptr(norms), None, nat.ptr(ws),
                                       ws.numel(), nat.stream_ptr()))
    norm = float(norms.item())
    if step == 0.0:
        # u + 0 * r is u itself; keep the caller's values bit-for-bit
        # (the float32 iterate would round them).
        return (uu.clone() if is_device_array(uu) else np.array(uu, dtype=np.float64)), norm
    return to_host(out.to(torch.float64) if not is_device_array(u) else out, u), norm


class DeviceProblem:
    """Device-resident solver inputs for P = batch * C planes of H x W."""

    def __init__(self, phi, lam, height, width, planes, channels, bounds=None):
        self.phi = phi          # float32 [P][H][W]
        self.lam = lam          # float32 [P/C][H][W]
        self.height = height
        self.width = width
        self.planes = planes
        self.channels = channels
        # tau_stability_bound per plane at u0 = Phi, from the float64 Phi when
        # the front end produced it (float32 Phi shifts the minimum face
        # gradient of near-flat regions by ~1e-6 relative)
        self.bounds = bounds


def _tau_bounds(problem: DeviceProblem, cfg, epsilon) -> np.ndarray:
    import torch

    prm = _params(problem.height, problem.width, problem.planes, problem.channels, cfg,
                  epsilon=epsilon)
    lib = nat.lib()
    ws = nat.workspace(lib.pdz_tau_bound_workspace_bytes(prm), "tau")
    out = torch.empty(problem.planes, dtype=torch.float64, device=problem.phi.device)
    nat.check(lib.pdz_tau_bound(prm, nat.ptr(problem.phi), nat.ptr(problem.lam), nat.ptr(out),
                                nat.ptr(ws), ws.numel(), nat.stream_ptr()))
    return out.to("cpu").numpy()


def solve_problem(problem: DeviceProblem, cfg: SolverConfig, *, edge_preserving=True,
                  tau=None, warn=True):
    """fixed_point_solve for every plane at once.  Returns (u [P][H][W] float32
    device tensor, [SolverTrace] * P)."""
    u, finish = queue_solve_problem(problem, cfg, edge_preserving=edge_preserving, tau=tau,
                                    warn=warn)
    return u, finish()


_solve_pinned = threading.local()


def queue_solve_problem(problem: DeviceProblem, cfg: SolverConfig, *, edge_preserving=True,
                        tau=None, warn=True):
    """Queue the solve of every plane (pdz_fixed_point_solve_async) and the
    copy of its outcome (norms, iterations, flags, tau bounds) to pinned host
    memory.  Returns (u, finish): u is the device result, valid for work
    queued after this call on the current stream; finish() waits for the
    outcome only, raises the reference's errors and warning (solver.py:335-350)
    and returns the [SolverTrace] * P."""
    import torch

    step = cfg.tau if tau is None else float(tau)
    P = problem.planes
    bounds = problem.bounds if problem.bounds is not None else _tau_bounds(problem, cfg,
                                                                          cfg.epsilon)
    prm = _params(problem.height, problem.width, P, problem.channels, cfg,
                  edge_preserving=edge_preserving, tau=step)
    lib = nat.lib()
    ws = nat.workspace(lib.pdz_solve_workspace_bytes(prm), "solve")
    nbytes = int(lib.pdz_solve_state_bytes(prm))
    state = nat.workspace(nbytes, "solve-state")
    u = torch.empty_like(problem.phi)
    nat.check(lib.pdz_fixed_point_solve_async(prm, nat.ptr(problem.phi), nat.ptr(problem.lam),
                                              nat.ptr(u), nat.ptr(state), nat.ptr(ws),
                                              ws.numel(), nat.stream_ptr()))
    # one pinned landing buffer per thread: the outcome, then the bounds
    nb_host = nbytes + 8 * P
    # keyed by device too: a CUDA event belongs to the device it was recorded on
    slots = getattr(_solve_pinned, "slots", None)
    if slots is None:
        slots = _solve_pinned.slots = {}
    dev_idx = problem.phi.device.index
    buf, ev = slots.get(dev_idx, (None, None))
    if buf is None or buf.numel() < nb_host:
        buf = torch.empty(max(nb_host, 4096), dtype=torch.uint8, pin_memory=True)
        ev = torch.cuda.Event()
        slots[dev_idx] = (buf, ev)
    buf[:nbytes].copy_(state[:nbytes], non_blocking=True)
    dev_bounds = hasattr(bounds, "is_cuda")
    if dev_bounds:
        buf[nbytes:nb_host].copy_(bounds.contiguous().view(torch.uint8), non_blocking=True)
    ev.record()

    def finish():
        ev.synchronize()
        raw = buf[:nb_host].numpy()
        norms = raw[:8 * cfg.max_iters * P].view(np.float64).reshape(cfg.max_iters, P)
        ints = raw[8 * cfg.max_iters * P:nbytes].view(np.int32)
        iters, conv, failed, abort = ints[:P], ints[P:2 * P], ints[2 * P:3 * P], ints[3 * P]
        hb = (raw[nbytes:nb_host].view(np.float64).copy() if dev_bounds
              else np.asarray(bounds, dtype=np.float64))
        if warn:  # solver.py:335-339
            for b in hb:
                if step > b:
                    logger.warning(
                        "relaxation step %.3g exceeds the stability bound %.3g at the "
                        "initial iterate; convergence is not guaranteed", step, b)
        if abort:
            raise RuntimeError("persistent sweep aborted: a CTA dependency wait timed out")
        bad = np.flatnonzero(failed)
        if bad.size:
            raise FloatingPointError(
                f"solver produced non-finite values at iteration {int(failed[bad[0]])}")
        traces = []
        for p in range(P):
            n = int(iters[p])
            traces.append(SolverTrace(residual_norms=[float(v) for v in norms[:n, p]],
                                      iterations_run=n, converged=bool(conv[p]), tau_used=step,
                                      tau_bound=float(hb[p])))
        return traces

    return u, finish


def _lambda_mode(flags, cfg) -> int:
    if "no-nonlocal" in flags:
        return nat.LAMBDA_MODES_C["zero"]
    if "no-adaptive" in flags:
        return nat.LAMBDA_MODES_C["const"]
    return nat.LAMBDA_MODES_C[cfg.lambda_monotonicity]


def prepare_problem(img_dev, is_f64, t_dev, a_dev, cfg, lambda_mode, phi=None, lam=None,
                    with_bounds=False, lam_override=None):
    """Phi planes and lambda for one image straight from the device front end.
    With `with_bounds`, also returns the per-channel tau_stability_bound at
    u0 = Phi evaluated on the float64 Phi (solver.py:334)."""
    import torch

    h, w, c = img_dev.shape
    if phi is None:
        phi = torch.empty((c, h, w), dtype=torch.float32, device=img_dev.device)
    if lam is None:
        lam = torch.empty((h, w), dtype=torch.float32, device=img_dev.device)
    phi64 = (torch.empty((h, w, c), dtype=torch.float64, device=img_dev.device)
             if with_bounds else None)
    lib = nat.lib()
    nat.check(lib.pdz_solver_fields(nat.ptr(img_dev), is_f64, h, w, c, nat.ptr(t_dev),
                                    nat.ptr(a_dev), float(cfg.t_floor), int(lambda_mode),
                                    float(cfg.lambda0), float(cfg.beta), nat.ptr(phi),
                                    nat.ptr(lam), nat.ptr(phi64), nat.stream_ptr()))
    if lam_override is not None:
        lam.copy_(lam_override)
    if not with_bounds:
        return phi, lam
    if h < 2 or w < 2:
        raise ValueError(f"field must be at least 2x2, got {(h, w)}")
    prm = _params(h, w, c, c, cfg)
    ws = nat.workspace(lib.pdz_tau_bound_workspace_bytes(prm), "tau")
    bounds = torch.empty(c, dtype=torch.float64, device=img_dev.device)
    nat.check(lib.pdz_tau_bound_hwc(prm, nat.ptr(phi64), nat.ptr(lam), nat.ptr(bounds),
                                    nat.ptr(ws), ws.numel(), nat.stream_ptr()))
    return phi, lam, bounds  # device tensor: read after the solve (one sync less)


def fixed_point_solve(channel, transmission, airlight_c: float, cfg: SolverConfig, *,
                      lambda_map=None, edge_preserving: bool = True, tau: float | None = None):
    """Relaxed fixed-point solve of one channel from u0 = Phi with the
    relative residual-change stop rule (solver.py:305-359).  Returns
    (u unclamped, SolverTrace)."""
    import torch

    ch = validate_field(channel)
    t = validate_field(transmission)
    if tuple(t.shape) != tuple(ch.shape):
        raise ValueError(f"transmission shape {tuple(t.shape)} != channel shape "
                         f"{tuple(ch.shape)}")
    if not 0.0 < airlight_c <= 1.0:
        raise ValueError("per-channel airlight must lie in (0, 1]")
    if float(t.min()) < 0.0 or float(t.max()) > 1.0:
        raise ValueError("transmission values must lie in [0, 1]")
    lam_given = None
    if lambda_map is not None:
        lam_given = validate_field(lambda_map)
        if tuple(lam_given.shape) != tuple(ch.shape):
            raise ValueError(f"lambda map shape {tuple(lam_given.shape)} != channel shape "
                             f"{tuple(ch.shape)}")
    h, w = ch.shape
    img_dev = to_device(ch, torch.float64).reshape(h, w, 1)
    t_dev = to_device(t, torch.float64)
    a_dev = _device_vec(np.array([float(airlight_c)]))
    override = None if lam_given is None else to_device(lam_given, torch.float32).reshape(h, w)
    phi, lam, bounds = prepare_problem(img_dev, 1, t_dev, a_dev, cfg,
                                       nat.LAMBDA_MODES_C[cfg.lambda_monotonicity],
                                       with_bounds=True, lam_override=override)
    problem = DeviceProblem(phi, lam, h, w, 1, 1, bounds)
    u, traces = solve_problem(problem, cfg, edge_preserving=edge_preserving, tau=tau)
    out = u[0]
    if not is_device_array(channel):
        out = out.to(torch.float64).to("cpu").numpy()
    return out, traces[0]


# --------------------------------------------------------------------------
# the pipeline
# --------------------------------------------------------------------------

def _front_end(img_dev, is_f64, cfg, flags):
    """dark (A = 1) -> airlight -> normalised dark -> t -> guided refinement
    (solver.py:393-408), all on the device.  Returns (t_dev, a_dev)."""
    import torch

    h, w, c = img_dev.shape
    if "no-multiscale" in flags:
        radii, weights = (cfg.patch_radius,), (1.0,)
    else:
        radii, weights = _blend_weights(cfg.multiscale_radii, cfg.multiscale_weights)
    if any(r < 0 for r in radii):
        raise ValueError("patch_radius must be >= 0")
    ones = torch.ones(c, dtype=torch.float64, device=img_dev.device)
    dark = torch.empty((h, w), dtype=torch.float64, device=img_dev.device)
    _dark_dev(img_dev, is_f64, ones, radii, weights, dark)
    a_dev, _ = _airlight_dev(img_dev, is_f64, dark, cfg.airlight_fraction)
    _dark_dev(img_dev, is_f64, a_dev, radii, weights, dark)
    t_dev = torch.empty_like(dark)
    nat.check(nat.lib().pdz_transmission(nat.ptr(dark), h, w, float(cfg.omega), nat.ptr(t_dev),
                                         nat.stream_ptr()))
    if "no-guided" not in flags:
        t_dev = refine_dev(img_dev, is_f64, t_dev, cfg.guided_radius, cfg.guided_reg)
    return t_dev, a_dev


_stage_pinned = threading.local()


def _pinned_like(array):
    """A page-locked torch copy of a numpy array (one cached buffer per thread
    and size; the upload that follows is asynchronous and runs at full rate)."""
    import torch

    buf = getattr(_stage_pinned, "buf", None)
    nbytes = array.nbytes
    if buf is None or buf.numel() < nbytes:
        buf = _stage_pinned.buf = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8,
                                              pin_memory=True)
    t = buf[:nbytes].view(torch.float32 if array.dtype == np.float32 else torch.float64)
    t = t.view(array.shape)
    t.copy_(torch.from_numpy(np.ascontiguousarray(array)))
    return t


def _front_end_fused(img_dev, is_f64, cfg, flags):
    """(t, A, Phi, lambda, tau bounds) of one image without the guided
    refinement: pdz_front_end_batch on a batch of one, then the float64 tau
    bound.  Bitwise the values of _front_end + prepare_problem."""
    import torch

    h, w, c = img_dev.shape
    lib = nat.lib()
    if "no-multiscale" in flags:
        radii, weights = (cfg.patch_radius,), (1.0,)
    else:
        radii, weights = _blend_weights(cfg.multiscale_radii, cfg.multiscale_weights)
    if any(r < 0 for r in radii):
        raise ValueError("patch_radius must be >= 0")
    dev = img_dev.device
    r_np = np.ascontiguousarray(radii, dtype=np.int32)
    w_np = np.ascontiguousarray(weights, dtype=np.float64)
    a_dev = torch.empty(c, dtype=torch.float64, device=dev)
    t_dev = torch.empty((h, w), dtype=torch.float64, device=dev)
    phi = torch.empty((c, h, w), dtype=torch.float32, device=dev)
    lam = torch.empty((h, w), dtype=torch.float32, device=dev)
    phi64 = torch.empty((h, w, c), dtype=torch.float64, device=dev)
    ws = nat.workspace(lib.pdz_front_end_batch_workspace_bytes(
        1, h, w, len(radii), float(cfg.airlight_fraction)), "front-batch")
    nat.check(lib.pdz_front_end_batch(
        nat.ptr(img_dev), is_f64, 1, h, w, c, r_np.ctypes.data, w_np.ctypes.data, len(radii),
        float(cfg.airlight_fraction), float(cfg.omega), float(cfg.t_floor),
        int(_lambda_mode(flags, cfg)), float(cfg.lambda0), float(cfg.beta), nat.ptr(a_dev),
        nat.ptr(t_dev), nat.ptr(phi), nat.ptr(lam), nat.ptr(phi64), nat.ptr(ws), ws.numel(),
        nat.stream_ptr()))
    prm = _params(h, w, c, c, cfg)
    tws = nat.workspace(lib.pdz_tau_bound_workspace_bytes(prm), "tau")
    bounds = torch.empty(c, dtype=torch.float64, device=dev)
    nat.check(lib.pdz_tau_bound_hwc(prm, nat.ptr(phi64), nat.ptr(lam), nat.ptr(bounds),
                                    nat.ptr(tws), tws.numel(), nat.stream_ptr()))
    return t_dev, a_dev, phi, lam, bounds


def _image_dev(img):
    import torch

    t = to_device(img)
    return t, 1 if t.dtype == torch.float64 else 0


def dehaze(image, cfg: SolverConfig | None = None, ablation=(), workers: int = 1):
    """Full pipeline (solver.py:375-436): front end -> per-channel relaxed
    solve (all channels in one fused sweep per iteration) -> clamp.  `workers`
    is accepted for compatibility; the output does not depend on it."""
    import torch

    cfg = cfg or SolverConfig()
    flags = normalize_ablation(ablation)
    # torch inputs (pinned host or device) are moved first and validated on the
    # GPU with one combined reduction (finite, min, max); its host read is
    # deferred until the front end is queued, so the GPU never waits for the
    # host in between (the errors are the same and come before any result)
    dev_in = is_device_array(image)
    staged = image
    if (not dev_in and isinstance(image, np.ndarray) and image.ndim == 3
            and image.dtype in (np.float32, np.float64)):
        # numpy float images take the same road: staged through a page-locked
        # buffer, uploaded as they are (float32 stays float32 -- its float64
        # value is the same) and validated on the GPU, instead of a float64
        # copy and three passes over it on the host
        staged = _pinned_like(image)
        dev_in = True
    img, unit_check = validate_unit_image(to_device(staged) if dev_in else image, defer=dev_in)
    if workers < 1:
        if dev_in:
            unit_check()  # the finiteness error comes first, as in the reference
        raise ValueError("workers must be >= 1")
    if not dev_in:
        unit_check()
    img_dev, is_f64 = _image_dev(img)
    h, w, c = img_dev.shape
    lib = nat.lib()
    if "no-guided" in flags and "no-pde" not in flags and h >= 2 and w >= 2:
        # no guided refinement: the whole front end and the solver inputs are
        # one library call (pdz_front_end_batch with a batch of one)
        with nat.trace_range("pdz.front_end"):
            t_dev, a_dev, phi, lam, bounds = _front_end_fused(img_dev, is_f64, cfg, flags)
        if dev_in:
            unit_check()
        t_host, a_host = to_host_async(t_dev, image), to_host_async(a_dev, image)
        with nat.trace_range("pdz.solve"):
            u, finish = queue_solve_problem(DeviceProblem(phi, lam, h, w, c, c, bounds), cfg,
                                            edge_preserving="no-edge" not in flags)
        out = torch.empty((h, w, c), dtype=torch.float64, device=img_dev.device)
        nat.check(lib.pdz_clamp_interleave(nat.ptr(u), h, w, c, nat.ptr(out), 1,
                                           nat.stream_ptr()))
        out_host = to_host_async(out, image)
        traces = finish()
        return (out_host(), DehazeResult(a_host(), t_host(), traces, flags))
    with nat.trace_range("pdz.front_end"):
        t_dev, a_dev = _front_end(img_dev, is_f64, cfg, flags)
    if dev_in:
        unit_check()
    if "no-pde" in flags:
        phi64 = torch.empty((h, w, c), dtype=torch.float64, device=img_dev.device)
        nat.check(lib.pdz_solver_fields(nat.ptr(img_dev), is_f64, h, w, c, nat.ptr(t_dev),
                                        nat.ptr(a_dev), float(cfg.t_floor), 0, 0.5, 3.0, None,
                                        None, nat.ptr(phi64), nat.stream_ptr()))
        out = clamp01(phi64)
        return (to_host(out, image),
                DehazeResult(to_host(a_dev, image), to_host(t_dev, image), [], flags))
    if h < 2 or w < 2:
        raise ValueError(f"field must be at least 2x2, got {(h, w)}")
    phi, lam, bounds = prepare_problem(img_dev, is_f64, t_dev, a_dev, cfg,
                                       _lambda_mode(flags, cfg), with_bounds=True)
    # the transmission map and airlight are final: copy them out while the
    # solve runs
    t_host, a_host = to_host_async(t_dev, image), to_host_async(a_dev, image)
    problem = DeviceProblem(phi, lam, h, w, c, c, bounds)
    # clamp + interleave and the result copy are queued behind the solve
    # before the host reads the solve's outcome: the GPU never waits for it
    with nat.trace_range("pdz.solve"):
        u, finish = queue_solve_problem(problem, cfg, edge_preserving="no-edge" not in flags)
    out = torch.empty((h, w, c), dtype=torch.float64, device=img_dev.device)
    nat.check(lib.pdz_clamp_interleave(nat.ptr(u), h, w, c, nat.ptr(out), 1, nat.stream_ptr()))
    out_host = to_host_async(out, image)
    traces = finish()
    return (out_host(), DehazeResult(a_host(), t_host(), traces, flags))


def dehaze_batch(images, cfg: SolverConfig | None = None, ablation=()):
    """Extension for batched serving (BASELINE config 3): same results as
    calling `dehaze` on each image, but every image's planes are swept by one
    persistent launch.  `images`: (B, H, W, C) array or sequence of equal-
    shaped images.  Returns (restored (B, H, W, C), [DehazeResult] * B).

    The batch is uploaded into one device tensor and validated there with one
    deferred reduction (finite, min, max over the whole batch); the per-image
    front ends, the solve, the clamp and the result copies are all queued
    before the host reads anything back, and the transmission maps and
    airlights travel to the host as two stacked copies while the solve runs."""
    import torch

    cfg = cfg or SolverConfig()
    flags = normalize_ablation(ablation)
    if "no-pde" in flags:
        outs = [dehaze(im, cfg, ablation) for im in images]
        return np.stack([o for o, _ in outs]), [r for _, r in outs]
    items = list(images)
    if not items:
        raise ValueError("images must be nonempty")
    shape = tuple(items[0].shape)
    if len(shape) != 3 or shape[2] not in (1, 3):
        raise ValueError(f"expected (H, W, C) image with C in {{1, 3}}, got shape {shape}")
    if any(tuple(im.shape) != shape for im in items):
        raise ValueError("all images of a batch must share one shape")
    h, w, c = shape
    if h < 2 or w < 2:
        raise ValueError(f"field must be at least 2x2, got {(h, w)}")
    B = len(items)
    dev = nat.device()
    like = items[0]
    # float32 inputs stay float32 on the device (like dehaze); anything else
    # is carried in float64
    def kind(im):
        return str(im.dtype).replace("torch.", "")

    dtype = torch.float32 if all(kind(im) == "float32" for im in items) else torch.float64
    stack = torch.empty((B, h, w, c), dtype=dtype, device=dev)
    # uploads run on a side stream in groups of 16 images; the front ends of
    # a group start as soon as its copies landed (copy engine || SMs)
    main = torch.cuda.current_stream(dev)
    side = torch.cuda.Stream(device=dev)
    side.wait_stream(main)
    landed = []
    with torch.cuda.stream(side):
        for i, im in enumerate(items):
            src = im if is_device_array(im) else torch.from_numpy(np.ascontiguousarray(im))
            stack[i].copy_(src, non_blocking=True)
            if i % 16 == 15 or i == B - 1:
                ev = torch.cuda.Event()
                ev.record(side)
                landed.append(ev)
    stack.record_stream(side)
    is_f64 = 1 if dtype == torch.float64 else 0
    phi = torch.empty((B * c, h, w), dtype=torch.float32, device=dev)
    lam = torch.empty((B, h, w), dtype=torch.float32, device=dev)
    lib = nat.lib()
    if "no-guided" in flags:
        # every front-end stage is one launch sequence for the whole batch
        # (pdz_front_end_batch; the guided refinement is per image)
        main.wait_event(landed[-1])
        if "no-multiscale" in flags:
            radii, weights = (cfg.patch_radius,), (1.0,)
        else:
            radii, weights = _blend_weights(cfg.multiscale_radii, cfg.multiscale_weights)
        if any(r < 0 for r in radii):
            raise ValueError("patch_radius must be >= 0")
        r_np = np.ascontiguousarray(radii, dtype=np.int32)
        w_np = np.ascontiguousarray(weights, dtype=np.float64)
        a_all = torch.empty((B, c), dtype=torch.float64, device=dev)
        t_all = torch.empty((B, h, w), dtype=torch.float64, device=dev)
        phi64 = torch.empty((B, h, w, c), dtype=torch.float64, device=dev)
        ws = nat.workspace(lib.pdz_front_end_batch_workspace_bytes(
            B, h, w, len(radii), float(cfg.airlight_fraction)), "front-batch")
        nat.check(lib.pdz_front_end_batch(
            nat.ptr(stack), is_f64, B, h, w, c, r_np.ctypes.data, w_np.ctypes.data, len(radii),
            float(cfg.airlight_fraction), float(cfg.omega), float(cfg.t_floor),
            int(_lambda_mode(flags, cfg)), float(cfg.lambda0), float(cfg.beta), nat.ptr(a_all),
            nat.ptr(t_all), nat.ptr(phi), nat.ptr(lam), nat.ptr(phi64), nat.ptr(ws), ws.numel(),
            nat.stream_ptr()))
        # tau_stability_bound at u0 = Phi from the float64 Phi, image by image
        prm = _params(h, w, c, c, cfg)
        tws = nat.workspace(lib.pdz_tau_bound_workspace_bytes(prm), "tau")
        bound_all = torch.empty((B, c), dtype=torch.float64, device=dev)
        for i in range(B):
            nat.check(lib.pdz_tau_bound_hwc(prm, nat.ptr(phi64[i]), nat.ptr(lam[i]),
                                            nat.ptr(bound_all[i]), nat.ptr(tws), tws.numel(),
                                            nat.stream_ptr()))
        del phi64
        bounds_cat = bound_all.reshape(-1)
    else:
        ts, airs, bounds = [], [], []
        for i in range(B):
            if i % 16 == 0:
                main.wait_event(landed[i // 16])
            t_dev, a_dev = _front_end(stack[i], is_f64, cfg, flags)
            _, _, b = prepare_problem(stack[i], is_f64, t_dev, a_dev, cfg,
                                      _lambda_mode(flags, cfg), phi=phi[i * c:(i + 1) * c],
                                      lam=lam[i], with_bounds=True)
            ts.append(t_dev)
            airs.append(a_dev)
            bounds.append(b)
        t_all, a_all = torch.stack(ts), torch.stack(airs)
        bounds_cat = torch.cat(bounds)
        del ts, airs, bounds
    _, unit_check = validate_unit_image(stack.view(B * h, w, c), defer=True)
    t_host, a_host = to_host_async(t_all, like), to_host_async(a_all, like)
    problem = DeviceProblem(phi, lam, h, w, B * c, c, bounds_cat)
    with nat.trace_range("pdz.solve_batch"):
        u, finish = queue_solve_problem(problem, cfg, edge_preserving="no-edge" not in flags)
    out = torch.empty((B, h, w, c), dtype=torch.float64, device=dev)
    for i in range(B):
        nat.check(lib.pdz_clamp_interleave(nat.ptr(u[i * c:(i + 1) * c]), h, w, c,
                                           nat.ptr(out[i]), 1, nat.stream_ptr()))
    out_host = to_host_async(out, like)
    unit_check()  # the errors of a bad batch come before any result
    traces = finish()
    t_res, a_res = t_host(), a_host()
    results = [DehazeResult(a_res[i], t_res[i], traces[i * c:(i + 1) * c], flags)
               for i in range(B)]
    return out_host(), results


def write_trace_csv(traces, path) -> None:
    """CSV rows (channel, iteration, residual_norm) with repr() norms
    (solver.py:439-446)."""
    with open(path, "w", newline="") as fh:
        writer = csv.writer(fh)
        writer.writerow(["channel", "iteration", "residual_norm"])
        for channel, trace in enumerate(traces):
            for iteration, norm in enumerate(trace.residual_norms, start=1):
                writer.writerow([channel, iteration, repr(norm)])

