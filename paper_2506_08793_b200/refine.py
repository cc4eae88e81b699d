"""Guided-filter refinement on the GPU (drop-in for pdehaze.refine, refine.py:21-80).

SURVEY 8(f) "next #1": on the reference's default dehaze path.  The integral
image is built with the reference's sequential cumsum order, so results are
bit-exact (csrc/pdz_guided.cu).
"""

from __future__ import annotations

from . import _native as nat
from .image import to_device, to_host, validate_field, validate_image

__all__ = ["box_mean", "guided_filter", "refine_transmission"]

LUMA_WEIGHTS = (0.299, 0.587, 0.114)


def box_mean(field, radius: int):
    """Mean over border-truncated (2r+1)-sided windows (refine.py:21-40)."""
    import torch

    f = validate_field(field)
    if radius < 1:
        raise ValueError("radius must be >= 1")
    f_dev = to_device(f, torch.float64)
    h, w = f_dev.shape
    lib = nat.lib()
    ws = nat.workspace(lib.pdz_guided_workspace_bytes(h, w), "guided")
    out = torch.empty_like(f_dev)
    nat.check(lib.pdz_box_mean(nat.ptr(f_dev), h, w, int(radius), nat.ptr(out), nat.ptr(ws),
                               ws.numel(), nat.stream_ptr()))
    return to_host(out, field)


def guided_filter(guide, target, radius: int, reg: float):
    """Classic guided filter (refine.py:43-62)."""
    import torch

    g = validate_field(guide)
    p = validate_field(target)
    if tuple(g.shape) != tuple(p.shape):
        raise ValueError(f"guide shape {tuple(g.shape)} != target shape {tuple(p.shape)}")
    if reg <= 0.0:
        raise ValueError("reg must be > 0")
    if radius < 1:
        raise ValueError("radius must be >= 1")
    g_dev = to_device(g, torch.float64)
    p_dev = to_device(p, torch.float64)
    h, w = g_dev.shape
    lib = nat.lib()
    ws = nat.workspace(lib.pdz_guided_workspace_bytes(h, w), "guided")
    out = torch.empty_like(g_dev)
    nat.check(lib.pdz_guided_filter(nat.ptr(g_dev), nat.ptr(p_dev), h, w, int(radius),
                                    float(reg), nat.ptr(out), nat.ptr(ws), ws.numel(),
                                    nat.stream_ptr()))
    return to_host(out, guide)


def refine_dev(img_dev, is_f64, t_dev, radius, reg):
    """Device-resident refinement used by dehaze."""
    import torch

    h, w, c = img_dev.shape
    lib = nat.lib()
    ws = nat.workspace(lib.pdz_guided_workspace_bytes(h, w), "guided")
    out = torch.empty_like(t_dev)
    nat.check(lib.pdz_refine_transmission(nat.ptr(img_dev), is_f64, h, w, c, nat.ptr(t_dev),
                                          int(radius), float(reg), nat.ptr(out), nat.ptr(ws),
                                          ws.numel(), nat.stream_ptr()))
    return out


def refine_transmission(image, t_raw, radius: int = 30, reg: float = 1e-3):
    """Guided refinement against luminance, clipped to [0, 1] (refine.py:65-80)."""
    import torch

    img = validate_image(image)
    t = validate_field(t_raw)
    if tuple(t.shape) != tuple(img.shape[:2]):
        raise ValueError(f"transmission shape {tuple(t.shape)} != image shape "
                         f"{tuple(img.shape[:2])}")
    if reg <= 0.0:
        raise ValueError("reg must be > 0")
    if radius < 1:
        raise ValueError("radius must be >= 1")
    img_dev = to_device(img)
    t_dev = to_device(t, torch.float64)
    out = refine_dev(img_dev, 1 if img_dev.dtype == torch.float64 else 0, t_dev, radius, reg)
    return to_host(out, t_raw)
