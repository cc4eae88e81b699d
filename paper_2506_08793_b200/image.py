"""Array conventions at the API boundary (pdehaze/image.py:34-61).

Host (numpy) inputs are validated here exactly like the reference (float64
coercion, layout, finiteness); device (torch.cuda) inputs are validated with
device reductions and stay on the GPU.  `to_device` / `to_host` move data
between the two worlds; the compute itself is always the CUDA library.
"""

from __future__ import annotations

import threading

import numpy as np

__all__ = ["validate_image", "validate_unit_image", "validate_field", "clamp01",
           "is_device_array", "to_device", "to_host"]


def is_device_array(x) -> bool:
    try:
        import torch
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, torch.Tensor)


def _finite(x) -> bool:
    if is_device_array(x):
        import torch

        return bool(torch.isfinite(x).all().item())
    return bool(np.all(np.isfinite(x)))


def validate_image(image):
    """(H, W, C) with C in {1, 3}, H, W >= 1, all finite."""
    arr = image if is_device_array(image) else np.asarray(image, dtype=np.float64)
    shape = tuple(arr.shape)
    if len(shape) != 3 or shape[2] not in (1, 3):
        raise ValueError(f"expected (H, W, C) image with C in {{1, 3}}, got shape {shape}")
    if shape[0] < 1 or shape[1] < 1:
        raise ValueError(f"image dimensions must be >= 1, got shape {shape}")
    if not _finite(arr):
        raise ValueError("image contains non-finite values")
    return arr


_stats_pinned = threading.local()


def validate_unit_image(image, defer: bool = False):
    """validate_image followed by the [0, 1] range check (scattering.py:41-45).
    Returns (image, range_check): the finiteness error is raised here, the
    range error by range_check() so callers keep the reference's check order.
    Device tensors need ONE host read for both (finite, min, max).  With
    `defer` (device tensors) that read is queued asynchronously and BOTH
    errors are raised by range_check(), in the same order: the caller keeps
    queueing device work meanwhile instead of stalling the GPU on the read."""
    if not is_device_array(image):
        arr = validate_image(image)

        def check():
            if float(arr.min()) < 0.0 or float(arr.max()) > 1.0:
                raise ValueError("image values must lie in [0, 1]")
        return arr, check
    import torch

    shape = tuple(image.shape)
    if len(shape) != 3 or shape[2] not in (1, 3):
        raise ValueError(f"expected (H, W, C) image with C in {{1, 3}}, got shape {shape}")
    if shape[0] < 1 or shape[1] < 1:
        raise ValueError(f"image dimensions must be >= 1, got shape {shape}")
    lo, hi = torch.aminmax(image)
    stats_dev = torch.stack((torch.isfinite(image).all().to(torch.float64),
                             lo.to(torch.float64), hi.to(torch.float64)))
    if not defer:
        stats = stats_dev.to("cpu").tolist()
        if stats[0] != 1.0:
            raise ValueError("image contains non-finite values")

        def check():
            if stats[1] < 0.0 or stats[2] > 1.0:
                raise ValueError("image values must lie in [0, 1]")
        return image, check
    # one pinned 3-double slot per thread, read behind an event
    # (per thread and device: a CUDA event belongs to the device it records on)
    slots = getattr(_stats_pinned, "slots", None)
    if slots is None:
        slots = _stats_pinned.slots = {}
    buf, ev = slots.get(stats_dev.device.index, (None, None))
    if buf is None:
        buf = torch.empty(3, dtype=torch.float64, pin_memory=True)
        ev = torch.cuda.Event()
        slots[stats_dev.device.index] = (buf, ev)
    buf.copy_(stats_dev, non_blocking=True)
    ev.record()

    def deferred_check():
        ev.synchronize()
        stats = buf.tolist()
        if stats[0] != 1.0:
            raise ValueError("image contains non-finite values")
        if stats[1] < 0.0 or stats[2] > 1.0:
            raise ValueError("image values must lie in [0, 1]")
    return image, deferred_check


def validate_field(field):
    """(H, W) with all samples finite."""
    arr = field if is_device_array(field) else np.asarray(field, dtype=np.float64)
    if len(arr.shape) != 2:
        raise ValueError(f"expected (H, W) scalar field, got shape {tuple(arr.shape)}")
    if not _finite(arr):
        raise ValueError("field contains non-finite values")
    return arr


def clamp01(values):
    """Clip to [0, 1]; rejects non-finite input (image.py:56-61)."""
    if is_device_array(values):
        if not _finite(values):
            raise ValueError("cannot clamp non-finite values")
        return values.clamp(0.0, 1.0)
    arr = np.asarray(values, dtype=np.float64)
    if not np.all(np.isfinite(arr)):
        raise ValueError("cannot clamp non-finite values")
    return np.clip(arr, 0.0, 1.0)


def to_device(x, dtype=None):
    """numpy / torch -> contiguous CUDA tensor (float64 unless dtype given or
    the tensor is already float32/float64 on the device)."""
    import torch

    from ._native import device

    dev = device()
    if is_device_array(x):
        t = x
        if dtype is not None and t.dtype != dtype:
            t = t.to(dtype)
        elif t.dtype not in (torch.float32, torch.float64):
            t = t.to(torch.float64)
        return t.to(dev, non_blocking=True).contiguous()
    arr = np.ascontiguousarray(np.asarray(x, dtype=np.float64 if dtype is None else
                                          {torch.float32: np.float32,
                                           torch.float64: np.float64}[dtype]))
    return torch.from_numpy(arr).to(dev)


def to_host(t, like) -> object:
    """Return `t` as the caller's kind: numpy float64 for numpy (host)
    callers, like the reference; a tensor on the caller's device for torch
    callers (CPU tensors get the device -> host copy, CUDA tensors none)."""
    if is_device_array(like):
        if like.is_cuda:
            return t
        import torch

        # page-locked result (torch's caching host allocator): full-speed copy
        out = torch.empty(tuple(t.shape), dtype=t.dtype, pin_memory=True)
        out.copy_(t, non_blocking=True)
        torch.cuda.current_stream(t.device).synchronize()
        return out
    return t.detach().to("cpu").numpy().astype(np.float64, copy=False)


_SIDE_STREAMS: dict = {}


def to_host_async(t, like):
    """Start `to_host(t, like)` now, on a side stream after the work queued so
    far, so the copy overlaps later GPU work (dehaze: the transmission map and
    airlight while the solve runs).  Returns a callable that waits and gives
    the same value `to_host` would."""
    if is_device_array(like) and like.is_cuda:
        return lambda: t
    import torch

    dev = t.device
    side = _SIDE_STREAMS.get(dev)
    if side is None:
        side = _SIDE_STREAMS[dev] = torch.cuda.Stream(device=dev)
    ready = torch.cuda.Event()
    ready.record(torch.cuda.current_stream(dev))
    out = torch.empty(tuple(t.shape), dtype=t.dtype, pin_memory=True)
    with torch.cuda.stream(side):
        side.wait_event(ready)
        out.copy_(t, non_blocking=True)
        t.record_stream(side)  # keep the device buffer alive until the copy ran
        done = torch.cuda.Event()
        done.record(side)

    def finish():
        done.synchronize()
        if is_device_array(like):
            return out
        return out.numpy()  # float64 view of the page-locked copy

    return finish
