"""CPU oracle for the pdehaze hot path -- TEST INFRASTRUCTURE ONLY.

This module is a from-scratch numpy restatement of the reference algorithm
(`/root/reference/pkg/src/pdehaze`, version 0.1.0).  It exists so that the
parity tests, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` have a checker that travels to the
GPU box (the reference tree does not).  Nothing in
``paper_2506_08793_b200`` may import it: the product path is the CUDA
library and fails loudly when that library is missing.

Pinning: ``tests/golden/make_golden.py`` runs the real reference (imported
from ``/root/reference/pkg/src`` in the build container) on seeded inputs and
stores its outputs under ``tests/golden/``; ``tests/test_oracle_golden.py``
checks this module against those fixtures -- bit-for-bit wherever the
reference's floating-point operation order is reproduced here (all of the
front end, the operators and short solves), and to 1e-12 otherwise.

Every function cites the reference lines it restates.  Arithmetic is float64
throughout, exactly like the reference; operation order follows the
reference so that results are bitwise identical:

* np.gradient (edge_order=1, unit spacing) -- centred (f[i+1]-f[i-1])/2,
  one-sided f[1]-f[0] / f[n-1]-f[n-2] at the ends    (solver.py:178-179)
* np.pad(mode="symmetric") -- edge-inclusive repeated reflection (solver.py:235)
* scipy.ndimage.minimum_filter(mode="nearest") with a scalar size -- the
  border-truncated window minimum (scattering.py:61-64); min is exact so any
  correct window minimum is bitwise equal
* stable argsort of -dark -- (value desc, flat index asc) (scattering.py:105)
* picked.mean(axis=0) on an (n, C) array -- sequential sum in selection order
  for C = 3, numpy's pairwise summation for C = 1, then division by n
  (scattering.py:106-107)
"""

from __future__ import annotations

import math
import os

import numpy as np

__all__ = [
    "TAU_STABLE",
    "SolverSettings",
    "reflect_index",
    "gaussian_taps_2d",
    "gaussian_taps_1d",
    "gaussian_blur_direct",
    "gaussian_blur_separable",
    "face_coefficients",
    "flux_divergence",
    "relaxed_step",
    "relaxed_solve",
    "per_pixel_channel_min",
    "window_min",
    "dark_channel",
    "blend_dark_channels",
    "airlight_selection",
    "airlight_from_selection",
    "pairwise_sum",
    "transmission_from_dark",
    "haze_weight",
    "scattering_inverse",
    "stability_bound",
    "box_average",
    "guided_smooth",
    "luminance_refine",
    "run_pipeline",
    "native_lib",
    "solve_planes_native",
    "relaxed_solve_native",
]

# tests/conftest.py:12 of the reference -- the step every parity run pins.
TAU_STABLE = 0.9 * 2.0 / (8.0 / 1e-3 + 0.5)


class SolverSettings:
    """Plain record of the solver tunables (mirrors SolverConfig, solver.py:78-94)."""

    def __init__(self, epsilon=1e-3, sigma=2.0, kernel_size=5, lambda0=0.5, beta=3.0,
                 tau=0.2, t_floor=0.1, omega=0.95, patch_radius=7, max_iters=200,
                 rel_tol=1e-4, lambda_monotonicity="as-printed", guided_radius=30,
                 guided_reg=1e-3, multiscale_radii=(3, 7, 15), multiscale_weights=None,
                 airlight_fraction=0.001):
        self.epsilon = float(epsilon)
        self.sigma = float(sigma)
        self.kernel_size = int(kernel_size)
        self.lambda0 = float(lambda0)
        self.beta = float(beta)
        self.tau = float(tau)
        self.t_floor = float(t_floor)
        self.omega = float(omega)
        self.patch_radius = int(patch_radius)
        self.max_iters = int(max_iters)
        self.rel_tol = float(rel_tol)
        self.lambda_monotonicity = lambda_monotonicity
        self.guided_radius = int(guided_radius)
        self.guided_reg = float(guided_reg)
        self.multiscale_radii = tuple(int(r) for r in multiscale_radii)
        self.multiscale_weights = multiscale_weights
        self.airlight_fraction = float(airlight_fraction)

    @classmethod
    def from_config(cls, cfg):
        names = ("epsilon", "sigma", "kernel_size", "lambda0", "beta", "tau", "t_floor",
                 "omega", "patch_radius", "max_iters", "rel_tol", "lambda_monotonicity",
                 "guided_radius", "guided_reg", "multiscale_radii", "multiscale_weights",
                 "airlight_fraction")
        return cls(**{n: getattr(cfg, n) for n in names})


# --------------------------------------------------------------------------
# Gaussian nonlocal operator  (solver.py:213-241)
# --------------------------------------------------------------------------

def reflect_index(idx, n):
    """np.pad(mode="symmetric") source index for (possibly far) out-of-range idx.

    Period-2n fold: -1 -> 0, -2 -> 1, n -> n-1, and repeats for pads >= n
    (solver.py:235; pinned by the reference test helper mirror_index,
    tests/test_pde_operators.py:63-70).
    """
    m = np.mod(np.asarray(idx, dtype=np.int64), 2 * n)
    return np.where(m >= n, 2 * n - 1 - m, m)


def gaussian_taps_2d(sigma, size):
    """outer(g, g) / sum with g = exp(-d^2 / 2 sigma^2)   (solver.py:219-222)."""
    d = np.arange(size) - size // 2
    g = np.exp(-(d * d) / (2.0 * sigma * sigma))
    k2 = np.outer(g, g)
    return k2 / k2.sum()


def gaussian_taps_1d(sigma, size):
    """Normalised 1-D factor g / sum(g); outer(w, w) equals gaussian_taps_2d to ~1e-17."""
    d = np.arange(size) - size // 2
    g = np.exp(-(d * d) / (2.0 * sigma * sigma))
    return g / g.sum()


def gaussian_blur_direct(u, sigma, size):
    """Direct K x K accumulation in the reference's (row, col) tap order
    (solver.py:233-241): bitwise identical to gaussian_convolve."""
    u = np.asarray(u, dtype=np.float64)
    h, w = u.shape
    r = size // 2
    taps = gaussian_taps_2d(sigma, size)
    rows = reflect_index(np.arange(-r, h + r), h)
    cols = reflect_index(np.arange(-r, w + r), w)
    ext = u[np.ix_(rows, cols)]
    acc = np.zeros_like(u)
    for a in range(size):
        band = ext[a:a + h]
        for b in range(size):
            acc += taps[a, b] * band[:, b:b + w]
    return acc


def gaussian_blur_separable(u, sigma, size):
    """Row pass then column pass with the 1-D factor (SPEC.md:236 allows the
    separable form); agrees with gaussian_blur_direct to ~1e-15."""
    u = np.asarray(u, dtype=np.float64)
    h, w = u.shape
    r = size // 2
    g = gaussian_taps_1d(sigma, size)
    cols = reflect_index(np.arange(-r, w + r), w)
    ext = u[:, cols]
    tmp = np.zeros_like(u)
    for b in range(size):
        tmp += g[b] * ext[:, b:b + w]
    rows = reflect_index(np.arange(-r, h + r), h)
    ext = tmp[rows, :]
    out = np.zeros_like(u)
    for a in range(size):
        out += g[a] * ext[a:a + h, :]
    return out


# --------------------------------------------------------------------------
# Edge-preserving diffusion  (solver.py:167-210)
# --------------------------------------------------------------------------

def _centred(u, axis):
    """np.gradient(u, axis) with unit spacing, edge_order=1 (solver.py:178-179)."""
    g = np.empty_like(u)
    if axis == 0:
        g[1:-1] = (u[2:] - u[:-2]) / 2.0
        g[0] = u[1] - u[0]
        g[-1] = u[-1] - u[-2]
    else:
        g[:, 1:-1] = (u[:, 2:] - u[:, :-2]) / 2.0
        g[:, 0] = u[:, 1] - u[:, 0]
        g[:, -1] = u[:, -1] - u[:, -2]
    return g


def face_coefficients(u, epsilon, edge_preserving=True):
    """(jump_e, jump_s, D_e, D_s) on the east (H, W-1) and south (H-1, W) faces.

    Across-face forward difference, along-face mean of the two adjacent
    centred differences, D = 1 / (|grad| + eps)  (solver.py:175-187).
    """
    jump_e = u[:, 1:] - u[:, :-1]
    jump_s = u[1:, :] - u[:-1, :]
    if not edge_preserving:
        return jump_e, jump_s, np.ones_like(jump_e), np.ones_like(jump_s)
    gy = _centred(u, 0)
    gx = _centred(u, 1)
    tang_e = 0.5 * (gy[:, 1:] + gy[:, :-1])
    tang_s = 0.5 * (gx[1:, :] + gx[:-1, :])
    d_e = 1.0 / (np.sqrt(jump_e * jump_e + tang_e * tang_e) + epsilon)
    d_s = 1.0 / (np.sqrt(jump_s * jump_s + tang_s * tang_s) + epsilon)
    return jump_e, jump_s, d_e, d_s


def flux_divergence(u, epsilon, edge_preserving=True):
    """Conservative div(D grad u), zero flux through the outer boundary
    (solver.py:190-210); accumulation order east+, east-, south+, south-."""
    u = np.asarray(u, dtype=np.float64)
    if u.ndim != 2 or u.shape[0] < 2 or u.shape[1] < 2:
        raise ValueError(f"field must be at least 2x2, got {u.shape}")
    je, js, de, ds = face_coefficients(u, epsilon, edge_preserving)
    fe = de * je
    fs = ds * js
    acc = np.zeros_like(u)
    acc[:, :-1] = acc[:, :-1] + fe
    acc[:, 1:] = acc[:, 1:] - fe
    acc[:-1, :] = acc[:-1, :] + fs
    acc[1:, :] = acc[1:, :] - fs
    return acc


def stability_bound(u, lam, epsilon):
    """2 / (8 max D + max(max lambda, 0)), D always edge-preserving (solver.py:266-277)."""
    _, _, de, ds = face_coefficients(np.asarray(u, dtype=np.float64), epsilon, True)
    dmax = max(de.max(), ds.max())
    return 2.0 / (8.0 * dmax + max(np.asarray(lam).max(), 0.0))


# --------------------------------------------------------------------------
# Relaxed fixed-point iteration  (solver.py:244-263, 280-359)
# --------------------------------------------------------------------------

def haze_weight(t, lambda0=0.5, beta=3.0, mode="as-printed"):
    """lambda0 exp(-beta (1-t)) ("as-printed") or lambda0 exp(-beta t) ("prose")
    (solver.py:262-263)."""
    t = np.asarray(t, dtype=np.float64)
    e = (1.0 - t) if mode == "as-printed" else t
    return lambda0 * np.exp(-beta * e)


def relaxed_step(u, src, lam, settings, edge_preserving=True, tau=None, separable=False):
    """(u + tau r, ||r||_2) with r = div - lam G(u) + src   (solver.py:295-302)."""
    step = settings.tau if tau is None else float(tau)
    blur = gaussian_blur_separable if separable else gaussian_blur_direct
    r = (flux_divergence(u, settings.epsilon, edge_preserving)
         - lam * blur(u, settings.sigma, settings.kernel_size) + src)
    return u + step * r, float(np.sqrt(np.sum(r * r)))


class OracleTrace:
    def __init__(self, tau_used, tau_bound):
        self.residual_norms = []
        self.iterations_run = 0
        self.converged = False
        self.tau_used = tau_used
        self.tau_bound = tau_bound


def relaxed_solve(channel, t, a_c, settings, lambda_map=None, edge_preserving=True,
                  tau=None, separable=False):
    """Per-channel solve from u0 = Phi with the relative-change stop rule
    (solver.py:324-359).  Returns (u unclamped, OracleTrace)."""
    chan = np.asarray(channel, dtype=np.float64)
    t = np.asarray(t, dtype=np.float64)
    src = (chan - a_c * (1.0 - t)) / np.maximum(t, settings.t_floor)
    if lambda_map is None:
        lam = haze_weight(t, settings.lambda0, settings.beta, settings.lambda_monotonicity)
    else:
        lam = np.asarray(lambda_map, dtype=np.float64)
    step = settings.tau if tau is None else float(tau)
    u = src.copy()
    trace = OracleTrace(step, stability_bound(u, lam, settings.epsilon))
    prev = None
    for it in range(1, settings.max_iters + 1):
        u, nrm = relaxed_step(u, src, lam, settings, edge_preserving, step, separable)
        if not (np.isfinite(nrm) and np.all(np.isfinite(u))):
            raise FloatingPointError(f"solver produced non-finite values at iteration {it}")
        trace.residual_norms.append(nrm)
        trace.iterations_run = it
        if prev is not None and abs(nrm - prev) / max(prev, 1e-30) <= settings.rel_tol:
            trace.converged = True
            break
        prev = nrm
    return u, trace


# --------------------------------------------------------------------------
# Dark-channel-prior front end  (scattering.py:48-139)
# --------------------------------------------------------------------------

def per_pixel_channel_min(img, airlight):
    """min_c I_c / A_c in float64 (scattering.py:60)."""
    img = np.asarray(img, dtype=np.float64)
    return np.min(img / np.asarray(airlight, dtype=np.float64), axis=2)


def window_min(p, radius):
    """Border-truncated (2r+1)^2 window minimum, separable (scattering.py:61-64)."""
    out = np.array(p, dtype=np.float64, copy=True)
    for axis in (1, 0):
        src = out.copy()
        n = src.shape[axis]
        for d in range(1, min(radius, n - 1) + 1):
            if axis == 1:
                np.minimum(out[:, d:], src[:, :-d], out=out[:, d:])
                np.minimum(out[:, :-d], src[:, d:], out=out[:, :-d])
            else:
                np.minimum(out[d:], src[:-d], out=out[d:])
                np.minimum(out[:-d], src[d:], out=out[:-d])
    return out


def dark_channel(img, airlight, radius):
    """Airlight-normalised dark channel capped at 1 (scattering.py:48-65)."""
    return np.minimum(window_min(per_pixel_channel_min(img, airlight), radius), 1.0)


def blend_dark_channels(img, airlight, radii, weights=None):
    """w0 d0 + w1 d1 + ... accumulated in radius order (scattering.py:68-85)."""
    radii = [int(r) for r in radii]
    if weights is None:
        weights = [1.0 / len(radii)] * len(radii)
    weights = [float(w) for w in weights]
    acc = weights[0] * dark_channel(img, airlight, radii[0])
    for r, w in zip(radii[1:], weights[1:]):
        acc += w * dark_channel(img, airlight, r)
    return acc


def airlight_selection(dark, fraction=0.001):
    """Flat indices of the ceil(f HW) largest dark values, ordered by
    (value desc, index asc)  (scattering.py:102-105)."""
    flat = np.asarray(dark, dtype=np.float64).ravel()
    count = math.ceil(fraction * flat.size)
    order = np.lexsort((np.arange(flat.size), -flat))
    return order[:count]


def pairwise_sum(v):
    """numpy's pairwise summation (numpy 2.3.5, _core/src/umath/loops_utils.h.src
    `pairwise_sum`): sequential below 8 items, 8 running partials up to 128,
    otherwise split at n/2 rounded down to a multiple of 8."""
    n = len(v)
    if n < 8:
        res = 0.0
        for x in v:
            res = res + x
        return res
    if n <= 128:
        r = [v[j] for j in range(8)]
        top = n - n % 8
        for i in range(8, top, 8):
            for j in range(8):
                r[j] = r[j] + v[i + j]
        res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
        for i in range(top, n):
            res = res + v[i]
        return res
    half = n // 2
    half -= half % 8
    return pairwise_sum(v[:half]) + pairwise_sum(v[half:])


def airlight_from_selection(img, picked):
    """Mean of I over the picked pixels in selection order, clipped to
    [0.05, 1]  (scattering.py:106-107).  numpy's picked.mean(axis=0) on the
    (n, C) gather sums sequentially over rows for C = 3, but for C = 1 the
    reduced axis is the contiguous one and numpy switches to its pairwise
    summation -- both orders are reproduced here (pinned by the golden tests)."""
    img = np.asarray(img, dtype=np.float64)
    rows = img.reshape(-1, img.shape[2])[picked]
    if rows.shape[1] == 1:
        total = np.array([0.0 + pairwise_sum(list(rows[:, 0]))])
    else:
        total = np.cumsum(rows, axis=0)[-1]
    return np.clip(total / rows.shape[0], 0.05, 1.0)


def transmission_from_dark(dark, omega=0.95):
    """t = 1 - omega dark  (scattering.py:121)."""
    return 1.0 - omega * np.asarray(dark, dtype=np.float64)


def scattering_inverse(img, t, airlight, t_floor=0.1):
    """Phi = (I - A (1-t)) / max(t, t0), unclamped  (scattering.py:138-139)."""
    img = np.asarray(img, dtype=np.float64)
    t = np.asarray(t, dtype=np.float64)
    a = np.asarray(airlight, dtype=np.float64)
    return (img - a * (1.0 - t)[:, :, None]) / np.maximum(t, t_floor)[:, :, None]


# --------------------------------------------------------------------------
# Guided-filter refinement  (refine.py:21-80) -- "next" row of SURVEY 8(f)
# --------------------------------------------------------------------------

def box_average(f, radius):
    """Border-truncated box mean from an integral image (refine.py:21-40)."""
    f = np.asarray(f, dtype=np.float64)
    h, w = f.shape
    sat = np.zeros((h + 1, w + 1))
    sat[1:, 1:] = f.cumsum(axis=0).cumsum(axis=1)
    r0 = np.maximum(np.arange(h) - radius, 0)
    r1 = np.minimum(np.arange(h) + radius, h - 1) + 1
    c0 = np.maximum(np.arange(w) - radius, 0)
    c1 = np.minimum(np.arange(w) + radius, w - 1) + 1
    total = (sat[np.ix_(r1, c1)] - sat[np.ix_(r0, c1)] - sat[np.ix_(r1, c0)]
             + sat[np.ix_(r0, c0)])
    return total / ((r1 - r0)[:, None] * (c1 - c0)[None, :])


def guided_smooth(guide, target, radius, reg):
    """Classic guided filter (refine.py:43-62)."""
    mg = box_average(guide, radius)
    mt = box_average(target, radius)
    vg = box_average(guide * guide, radius) - mg * mg
    cgt = box_average(guide * target, radius) - mg * mt
    a = cgt / (vg + reg)
    b = mt - a * mg
    return box_average(a, radius) * guide + box_average(b, radius)


def luminance_refine(img, t_raw, radius=30, reg=1e-3):
    """Guided refinement against luminance, clipped to [0, 1] (refine.py:65-80)."""
    img = np.asarray(img, dtype=np.float64)
    if img.shape[2] == 1:
        guide = img[:, :, 0]
    else:
        guide = 0.299 * img[:, :, 0] + 0.587 * img[:, :, 1] + 0.114 * img[:, :, 2]
    return np.clip(guided_smooth(guide, t_raw, radius, reg), 0.0, 1.0)


# --------------------------------------------------------------------------
# Whole pipeline  (solver.py:375-436)
# --------------------------------------------------------------------------

def run_pipeline(image, settings, ablation=(), separable=False, channel_workers=1,
                 native=False):
    """Front end -> per-channel relaxed solve -> clamp.  Returns
    (restored, airlight, transmission, traces).  native=True runs the solve
    loop in the C restatement (relaxed_solve_native)."""
    flags = frozenset((ablation,) if isinstance(ablation, str) else ablation)
    img = np.asarray(image, dtype=np.float64)
    channels = img.shape[2]
    if "no-multiscale" in flags:
        radii, weights = (settings.patch_radius,), (1.0,)
    else:
        radii, weights = settings.multiscale_radii, settings.multiscale_weights
    dark_unit = blend_dark_channels(img, np.ones(channels), radii, weights)
    picked = airlight_selection(dark_unit, settings.airlight_fraction)
    airlight = airlight_from_selection(img, picked)
    dark = blend_dark_channels(img, airlight, radii, weights)
    t = transmission_from_dark(dark, settings.omega)
    if "no-guided" not in flags:
        t = luminance_refine(img, t, settings.guided_radius, settings.guided_reg)
    if "no-pde" in flags:
        return np.clip(scattering_inverse(img, t, airlight, settings.t_floor), 0.0, 1.0), \
            airlight, t, []
    if "no-nonlocal" in flags:
        lam = np.zeros_like(t)
    elif "no-adaptive" in flags:
        lam = np.full_like(t, settings.lambda0)
    else:
        lam = None
    edge = "no-edge" not in flags

    def one(c):
        if native:
            return relaxed_solve_native(img[:, :, c], t, float(airlight[c]), settings, lam,
                                        edge)
        return relaxed_solve(img[:, :, c], t, float(airlight[c]), settings, lam, edge,
                             None, separable)

    if channel_workers > 1 and channels > 1:
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(max_workers=channel_workers) as pool:
            solved = list(pool.map(one, range(channels)))
    else:
        solved = [one(c) for c in range(channels)]
    out = np.clip(np.stack([u for u, _ in solved], axis=2), 0.0, 1.0)
    return out, airlight, t, [tr for _, tr in solved]


# --------------------------------------------------------------------------
# C restatement of the solve loop (oracle/pdz_oracle_solve.c)
# --------------------------------------------------------------------------

_NATIVE = None
NATIVE_LIB = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_build",
                          "liboracle_solve.so")


def native_lib():
    """ctypes handle of oracle/_build/liboracle_solve.so (built by
    __graft_entry__.build(); test infrastructure like the rest of oracle/)."""
    global _NATIVE
    if _NATIVE is None:
        import ctypes

        lib = ctypes.CDLL(NATIVE_LIB)
        d, i = ctypes.c_double, ctypes.c_int
        vp = ctypes.c_void_p
        lib.oracle_relaxed_solve.argtypes = [vp, vp, i, i, i, i, i, d, d, d, i, i, d, vp, vp, vp,
                                             vp, i]
        lib.oracle_relaxed_solve.restype = i
        lib.oracle_max_threads.restype = i
        _NATIVE = lib
    return _NATIVE


def solve_planes_native(src, lam, settings, edge_preserving=True, tau=None, max_iters=None,
                        rel_tol=None, threads=None):
    """Relaxed solve of P planes from u0 = src (solver.py:324-359) in C.
    src: (P, H, W) float64; lam: (H, W) shared by every plane or (P / k, H, W)
    with k planes per map.  Returns (u (P, H, W), norms (iters, P) list per
    plane, iterations_run [P], converged [P])."""
    src = np.ascontiguousarray(src, dtype=np.float64)
    if src.ndim == 2:
        src = src[None]
    P, H, W = src.shape
    lam = np.ascontiguousarray(lam, dtype=np.float64)
    if lam.ndim == 2:
        lam = lam[None]
    lam_div = P // lam.shape[0]
    iters_max = settings.max_iters if max_iters is None else int(max_iters)
    tol = settings.rel_tol if rel_tol is None else float(rel_tol)
    step = settings.tau if tau is None else float(tau)
    lib = native_lib()
    u = np.empty_like(src)
    norms = np.zeros((iters_max, P), dtype=np.float64)
    iters = np.zeros(P, dtype=np.int32)
    conv = np.zeros(P, dtype=np.int32)
    nt = lib.oracle_max_threads() if threads is None else int(threads)
    rc = lib.oracle_relaxed_solve(src.ctypes.data, lam.ctypes.data, P, lam_div, H, W,
                                  settings.kernel_size, settings.sigma, settings.epsilon, step,
                                  1 if edge_preserving else 0, iters_max, tol, u.ctypes.data,
                                  norms.ctypes.data, iters.ctypes.data, conv.ctypes.data, nt)
    if rc < 0:
        raise ValueError("invalid solve arguments")
    if rc > 0:
        raise FloatingPointError(f"solver produced non-finite values at iteration {rc}")
    return u, [norms[:iters[p], p].tolist() for p in range(P)], iters.tolist(), \
        [bool(c) for c in conv]


def relaxed_solve_native(channel, t, a_c, settings, lambda_map=None, edge_preserving=True,
                         tau=None, threads=None):
    """relaxed_solve with the sweep loop in C (same inputs, same OracleTrace)."""
    chan = np.asarray(channel, dtype=np.float64)
    t = np.asarray(t, dtype=np.float64)
    src = (chan - a_c * (1.0 - t)) / np.maximum(t, settings.t_floor)
    if lambda_map is None:
        lam = haze_weight(t, settings.lambda0, settings.beta, settings.lambda_monotonicity)
    else:
        lam = np.asarray(lambda_map, dtype=np.float64)
    step = settings.tau if tau is None else float(tau)
    trace = OracleTrace(step, stability_bound(src, lam, settings.epsilon))
    u, norms, iters, conv = solve_planes_native(src, lam, settings, edge_preserving, step,
                                                threads=threads)
    trace.residual_norms = norms[0]
    trace.iterations_run = iters[0]
    trace.converged = conv[0]
    return u[0], trace
