"""Binary Netpbm I/O (pdehaze/image.py:30-145): P5 grayscale / P6 colour,
maxval 255.

Parsing is host byte work.  Saving quantises on the device
(pdz_quantize_u8: clamp, then floor(v * 255 + 0.5) in float64 without FMA
contraction), so the written bytes equal the reference's; device images
(torch.cuda tensors) never leave the GPU as float64 -- only the uint8
samples are copied back.
"""

from __future__ import annotations

import numpy as np

from . import _native as nat
from .image import is_device_array, to_device, validate_image

__all__ = ["NetpbmError", "load_image", "save_image"]

_WHITESPACE = (b" ", b"\t", b"\n", b"\r", b"\x0b", b"\x0c")


class NetpbmError(ValueError):
    """Malformed or unsupported Netpbm file (image.py:30-31)."""


def _token(raw: bytes, pos: int):
    """Next header token after whitespace and `#` comments (to end of line)."""
    n = len(raw)
    while pos < n:
        ch = raw[pos:pos + 1]
        if ch == b"#":
            nl = raw.find(b"\n", pos)
            pos = n if nl < 0 else nl
        elif ch in _WHITESPACE:
            pos += 1
        else:
            break
    start = pos
    while pos < n and raw[pos:pos + 1] not in _WHITESPACE and raw[pos:pos + 1] != b"#":
        pos += 1
    if pos == start:
        raise NetpbmError("malformed header: unexpected end of header")
    return raw[start:pos], pos


def _int_field(raw: bytes, pos: int, what: str):
    tok, pos = _token(raw, pos)
    if not tok.isdigit():
        raise NetpbmError(f"malformed header: expected integer {what}, got {tok!r}")
    return int(tok), pos


def load_image(path) -> np.ndarray:
    """(H, W, 1) or (H, W, 3) float64 in [0, 1] (v / 255) from a P5 / P6 file;
    header comments tolerated (image.py:91-125)."""
    with open(path, "rb") as fh:
        raw = fh.read()
    magic = raw[:2]
    if magic not in (b"P5", b"P6"):
        raise NetpbmError(
            f"malformed header: not a binary Netpbm (P5/P6) file, magic {magic!r}")
    channels = 1 if magic == b"P5" else 3
    width, pos = _int_field(raw, 2, "width")
    height, pos = _int_field(raw, pos, "height")
    maxval, pos = _int_field(raw, pos, "maxval")
    if width < 1 or height < 1:
        raise NetpbmError(f"malformed header: non-positive dimensions {width}x{height}")
    if maxval != 255:
        raise NetpbmError(f"unsupported maxval {maxval}: only 255 is supported")
    if pos >= len(raw) or raw[pos:pos + 1] not in _WHITESPACE:
        raise NetpbmError("malformed header: missing whitespace after maxval")
    pos += 1  # one whitespace byte ends the header
    count = width * height * channels
    payload = raw[pos:pos + count]
    if len(payload) < count:
        raise NetpbmError(f"truncated payload: expected {count} bytes, found {len(payload)}")
    samples = np.frombuffer(payload, dtype=np.uint8).astype(np.float64) / 255.0
    return samples.reshape(height, width, channels)


def quantize(image):
    """uint8 samples of `image` (any shape, float) on the device, as numpy."""
    import torch

    dev = to_device(image, torch.float64).reshape(-1)
    out = torch.empty(dev.numel(), dtype=torch.uint8, device=dev.device)
    flag = torch.empty(1, dtype=torch.int32, device=dev.device)
    nat.check(nat.lib().pdz_quantize_u8(nat.ptr(dev), dev.numel(), nat.ptr(out), nat.ptr(flag),
                                        nat.stream_ptr()))
    if int(flag.item()):
        raise ValueError("cannot clamp non-finite values")
    return out.to("cpu").numpy()


def save_image(image, path) -> None:
    """P5 (1 channel) / P6 (3 channels) with a comment-free header; samples
    clamped to [0, 1] and rounded half away from zero on v * 255
    (image.py:128-145).  A 2-D array is saved as P5."""
    shape = tuple(image.shape) if is_device_array(image) else np.shape(image)
    if len(shape) == 2:
        image = image[:, :, None] if is_device_array(image) else \
            np.asarray(image, dtype=np.float64)[:, :, np.newaxis]
    arr = validate_image(image)
    height, width, channels = tuple(arr.shape)
    samples = quantize(arr)
    header = (b"P5" if channels == 1 else b"P6") + b"\n%d %d\n255\n" % (width, height)
    with open(path, "wb") as fh:
        fh.write(header)
        fh.write(samples.tobytes())
