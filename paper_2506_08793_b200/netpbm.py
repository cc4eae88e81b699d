"""Binary Netpbm I/O (pdehaze/image.py:30-145): P5 grayscale / P6 colour,
maxval 255.

Parsing is host byte work.  Saving quantises on the device
(pdz_quantize_u8: clamp, then floor(v * 255 + 0.5) in float64 without FMA
contraction), so the written bytes equal the reference's; device images
(torch.cuda tensors) never leave the GPU as float64 -- only the uint8
samples are copied back.
"""

from __future__ import annotations

import re

import numpy as np

from . import _native as nat
from .image import is_device_array, to_device, validate_image

__all__ = ["NetpbmError", "load_image", "save_image"]

_GAP = re.compile(rb"(?:[ \t\n\r\x0b\x0c]|#[^\n]*)*")   # whitespace and `#` comments
_WORD = re.compile(rb"[^ \t\n\r\x0b\x0c#]+")
_SPACE = b" \t\n\r\x0b\x0c"
_FORMATS = {b"P5": 1, b"P6": 3}  # magic -> channels


class NetpbmError(ValueError):
    """Malformed or unsupported Netpbm file (image.py:30-31)."""


class _Header:
    """Cursor over the header bytes: words separated by whitespace / comments."""

    def __init__(self, raw: bytes, start: int):
        self.raw = raw
        self.pos = start

    def word(self) -> bytes:
        self.pos = _GAP.match(self.raw, self.pos).end()
        found = _WORD.match(self.raw, self.pos)
        if found is None:
            raise NetpbmError("malformed header: unexpected end of header")
        self.pos = found.end()
        return found.group()

    def number(self, what: str) -> int:
        text = self.word()
        if not text.isdigit():
            raise NetpbmError(f"malformed header: expected integer {what}, got {text!r}")
        return int(text)

    def end(self) -> int:
        """Offset of the payload: exactly one whitespace byte closes the header."""
        if self.pos >= len(self.raw) or self.raw[self.pos] not in _SPACE:
            raise NetpbmError("malformed header: missing whitespace after maxval")
        return self.pos + 1


def load_image(path) -> np.ndarray:
    """(H, W, 1) or (H, W, 3) float64 in [0, 1] (v / 255) from a P5 / P6 file;
    header comments tolerated (image.py:91-125)."""
    with open(path, "rb") as fh:
        raw = fh.read()
    channels = _FORMATS.get(raw[:2])
    if channels is None:
        raise NetpbmError(
            f"malformed header: not a binary Netpbm (P5/P6) file, magic {raw[:2]!r}")
    header = _Header(raw, 2)
    width, height, maxval = (header.number(n) for n in ("width", "height", "maxval"))
    if min(width, height) < 1:
        raise NetpbmError(f"malformed header: non-positive dimensions {width}x{height}")
    if maxval != 255:
        raise NetpbmError(f"unsupported maxval {maxval}: only 255 is supported")
    start = header.end()
    want = width * height * channels
    samples = np.frombuffer(raw, dtype=np.uint8, count=min(want, len(raw) - start), offset=start)
    if samples.size < want:
        raise NetpbmError(f"truncated payload: expected {want} bytes, found {samples.size}")
    return (samples.astype(np.float64) / 255.0).reshape(height, width, channels)


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
