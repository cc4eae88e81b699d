"""Dark-channel-prior front end on the GPU (drop-in for pdehaze.scattering).

Each function keeps the reference signature and error behaviour
(pdehaze/scattering.py:30-139) and runs the CUDA kernels of
csrc/pdz_frontend.cu.  Outputs are bit-exact with the reference: the dark
channel, the airlight pixel selection/order and A, and t.  numpy inputs give
float64 numpy outputs; torch.cuda tensors give device tensors.
"""

from __future__ import annotations

import math

import numpy as np

from . import _native as nat
from .image import is_device_array, to_device, to_host, validate_field, validate_image

__all__ = [
    "dark_channel",
    "multiscale_dark_channel",
    "estimate_atmospheric_light",
    "estimate_atmospheric_light_indices",
    "estimate_transmission",
    "reconstruct",
    "synthesize_haze",
]


def _airlight_vector(airlight, channels: int) -> np.ndarray:
    """(C,) float64 in (0, 1] (scattering.py:30-38 semantics)."""
    if is_device_array(airlight):
        airlight = airlight.detach().to("cpu").numpy()
    a = np.asarray(airlight, dtype=np.float64)
    if a.shape != (channels,):
        raise ValueError(f"airlight must have shape ({channels},), got {a.shape}")
    if np.any(a <= 0.0):
        raise ValueError("airlight components must be strictly positive")
    if np.any(a > 1.0) or not np.all(np.isfinite(a)):
        raise ValueError("airlight components must lie in (0, 1]")
    return a


def _unit_range(img) -> None:
    lo, hi = (float(img.min()), float(img.max()))
    if lo < 0.0 or hi > 1.0:
        raise ValueError("image values must lie in [0, 1]")


def _image_on_device(img):
    """Device copy of a validated image; keeps float32 device tensors as-is."""
    import torch

    t = to_device(img)
    return t, 1 if t.dtype == torch.float64 else 0


def _dark_dev(img_dev, is_f64, a_dev, radii, weights, out):
    h, w, c = img_dev.shape
    lib = nat.lib()
    ws = nat.workspace(lib.pdz_dark_channel_workspace_bytes(h, w), "dark")
    if len(radii) == 1 and weights[0] == 1.0:
        nat.check(lib.pdz_dark_channel(nat.ptr(img_dev), is_f64, h, w, c, nat.ptr(a_dev),
                                       int(radii[0]), nat.ptr(out), nat.ptr(ws), ws.numel(),
                                       nat.stream_ptr()))
        return out
    w_arr = np.ascontiguousarray(weights, dtype=np.float64)
    r_np = np.ascontiguousarray(radii, dtype=np.int32)
    nat.check(lib.pdz_multiscale_dark_channel(
        nat.ptr(img_dev), is_f64, h, w, c, nat.ptr(a_dev), r_np.ctypes.data,
        w_arr.ctypes.data, len(radii), nat.ptr(out), nat.ptr(ws), ws.numel(),
        nat.stream_ptr()))
    return out


def _device_vec(a: np.ndarray):
    import torch

    return torch.tensor(a, dtype=torch.float64, device=nat.device())


def dark_channel(image, airlight, patch_radius: int):
    """min over the border-truncated (2r+1)^2 patch and channels of I_c / A_c,
    capped at 1 (scattering.py:48-65)."""
    import torch

    img = validate_image(image)
    _unit_range(img)
    a = _airlight_vector(airlight, img.shape[2])
    if patch_radius < 0:
        raise ValueError("patch_radius must be >= 0")
    img_dev, is_f64 = _image_on_device(img)
    out = torch.empty(img_dev.shape[:2], dtype=torch.float64, device=img_dev.device)
    _dark_dev(img_dev, is_f64, _device_vec(a), (int(patch_radius),), (1.0,), out)
    return to_host(out, image)


def _blend_weights(radii, weights):
    radii = [int(r) for r in radii]
    if not radii:
        raise ValueError("radii must be nonempty")
    if weights is None:
        weights = [1.0 / len(radii)] * len(radii)
    weights = [float(w) for w in weights]
    if len(weights) != len(radii):
        raise ValueError(f"{len(radii)} radii but {len(weights)} weights")
    if any(w < 0.0 for w in weights):
        raise ValueError("weights must be nonnegative")
    if abs(sum(weights) - 1.0) > 1e-9:
        raise ValueError(f"weights must sum to 1, got {sum(weights)}")
    return radii, weights


def multiscale_dark_channel(image, airlight, radii, weights=None):
    """w0 d0 + w1 d1 + ... over patch radii, float64 without contraction
    (scattering.py:68-85)."""
    import torch

    radii, weights = _blend_weights(radii, weights)
    img = validate_image(image)
    _unit_range(img)
    a = _airlight_vector(airlight, img.shape[2])
    if any(r < 0 for r in radii):
        raise ValueError("patch_radius must be >= 0")
    img_dev, is_f64 = _image_on_device(img)
    out = torch.empty(img_dev.shape[:2], dtype=torch.float64, device=img_dev.device)
    if len(radii) == 1:
        # weight * dark for a single radius: multiply explicitly like the reference
        _dark_dev(img_dev, is_f64, _device_vec(a), radii, [weights[0]], out)
    else:
        _dark_dev(img_dev, is_f64, _device_vec(a), radii, weights, out)
    return to_host(out, image)


def _airlight_dev(img_dev, is_f64, dark_dev, fraction, want_indices=False):
    import torch

    h, w, c = img_dev.shape
    lib = nat.lib()
    ws = nat.workspace(lib.pdz_airlight_workspace_bytes(h, w, fraction), "airlight")
    a = torch.empty(c, dtype=torch.float64, device=img_dev.device)
    picked = None
    if want_indices:
        picked = torch.empty(int(lib.pdz_airlight_count(h, w, fraction)), dtype=torch.int64,
                             device=img_dev.device)
    nat.check(lib.pdz_atmospheric_light(nat.ptr(img_dev), is_f64, h, w, c, nat.ptr(dark_dev),
                                        float(fraction), nat.ptr(a), nat.ptr(picked),
                                        nat.ptr(ws), ws.numel(), nat.stream_ptr()))
    return a, picked


def _airlight_args(image, dark, fraction):
    img = validate_image(image)
    _unit_range(img)
    d = validate_field(dark)
    if tuple(d.shape) != tuple(img.shape[:2]):
        raise ValueError(f"dark channel shape {tuple(d.shape)} != image shape "
                         f"{tuple(img.shape[:2])}")
    if not 0.0 < fraction <= 1.0:
        raise ValueError("fraction must lie in (0, 1]")
    img_dev, is_f64 = _image_on_device(img)
    import torch

    return img_dev, is_f64, to_device(d, torch.float64)


def estimate_atmospheric_light(image, dark, fraction: float = 0.001):
    """Mean colour of the ceil(fraction*H*W) largest dark-channel pixels,
    clipped to [0.05, 1] (scattering.py:88-107)."""
    img_dev, is_f64, d_dev = _airlight_args(image, dark, fraction)
    a, _ = _airlight_dev(img_dev, is_f64, d_dev, fraction)
    return to_host(a, image)


def estimate_atmospheric_light_indices(image, dark, fraction: float = 0.001):
    """Extension: (A, flat indices in selection order) -- the indices the
    reference's stable argsort picks (scattering.py:105), for parity checks."""
    img_dev, is_f64, d_dev = _airlight_args(image, dark, fraction)
    a, picked = _airlight_dev(img_dev, is_f64, d_dev, fraction, want_indices=True)
    if is_device_array(image):
        return a, picked
    return to_host(a, image), picked.to("cpu").numpy()


def estimate_transmission(dark, omega: float = 0.95):
    """t = 1 - omega * dark, values in [1 - omega, 1] (scattering.py:110-121)."""
    import torch

    d = validate_field(dark)
    if not 0.0 < omega <= 1.0:
        raise ValueError("omega must lie in (0, 1]")
    if float(d.min()) < 0.0 or float(d.max()) > 1.0:
        raise ValueError("dark channel values must lie in [0, 1]")
    d_dev = to_device(d, torch.float64)
    t = torch.empty_like(d_dev)
    h, w = d_dev.shape
    nat.check(nat.lib().pdz_transmission(nat.ptr(d_dev), h, w, float(omega), nat.ptr(t),
                                         nat.stream_ptr()))
    return to_host(t, dark)


def reconstruct(image, transmission, airlight, t_floor: float = 0.1):
    """(I - A (1 - t)) / max(t, t_floor), unclamped (scattering.py:124-139)."""
    import torch

    img = validate_image(image)
    t = validate_field(transmission)
    if tuple(t.shape) != tuple(img.shape[:2]):
        raise ValueError(f"transmission shape {tuple(t.shape)} != image shape "
                         f"{tuple(img.shape[:2])}")
    a = _airlight_vector(airlight, img.shape[2])
    if t_floor <= 0.0:
        raise ValueError("t_floor must be > 0")
    img_dev, is_f64 = _image_on_device(img)
    t_dev = to_device(t, torch.float64)
    h, w, c = img_dev.shape
    out = torch.empty((h, w, c), dtype=torch.float64, device=img_dev.device)
    nat.check(nat.lib().pdz_solver_fields(nat.ptr(img_dev), is_f64, h, w, c, nat.ptr(t_dev),
                                          nat.ptr(_device_vec(a)), float(t_floor), 0, 0.5, 3.0,
                                          None, None, nat.ptr(out), nat.stream_ptr()))
    return to_host(out, image)


def _count(h: int, w: int, fraction: float) -> int:
    return math.ceil(fraction * h * w)


def synthesize_haze(clean, transmission, airlight):
    """Forward haze model J * t + A * (1 - t) (scattering.py:142-158), in
    float64 on the device with the reference's operation order (bitwise)."""
    import torch

    img = validate_image(clean)
    _unit_range(img)
    t = validate_field(transmission)
    if tuple(t.shape) != tuple(img.shape[:2]):
        raise ValueError(f"transmission shape {tuple(t.shape)} != image shape "
                         f"{tuple(img.shape[:2])}")
    if float(t.min()) < 0.0 or float(t.max()) > 1.0:
        raise ValueError("transmission values must lie in [0, 1]")
    h, w, c = img.shape
    a = _airlight_vector(airlight, c)
    img_dev = to_device(img, torch.float64)
    t_dev = to_device(t, torch.float64)
    a_dev = _device_vec(a)
    out = torch.empty_like(img_dev)
    nat.check(nat.lib().pdz_synthesize_haze(nat.ptr(img_dev), nat.ptr(t_dev), nat.ptr(a_dev),
                                            h * w, c, nat.ptr(out), nat.stream_ptr()))
    return to_host(out, clean)
