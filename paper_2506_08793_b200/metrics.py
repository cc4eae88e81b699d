"""Full-reference fidelity metrics (pdehaze/metrics.py:13-37) on the device."""

from __future__ import annotations

import math
from dataclasses import dataclass

from . import _native as nat
from .image import is_device_array, to_device

__all__ = ["MetricReport", "compare"]


@dataclass(frozen=True)
class MetricReport:
    mse: float
    psnr: float  # dB; math.inf for identical images
    mae: float


def compare(a, b) -> MetricReport:
    """MSE / PSNR / MAE between two same-shaped images in [0, 1]
    (metrics.py:20-37); PSNR = 10 log10(1 / mse), infinite exactly when
    mse == 0.  The sums are a fixed-order float64 reduction on the GPU."""
    import numpy as np
    import torch

    xs = tuple(a.shape) if is_device_array(a) else np.shape(np.asarray(a, dtype=np.float64))
    ys = tuple(b.shape) if is_device_array(b) else np.shape(np.asarray(b, dtype=np.float64))
    if tuple(xs) != tuple(ys):
        raise ValueError(f"shape mismatch: {tuple(xs)} vs {tuple(ys)}")
    x = to_device(a, torch.float64).reshape(-1)
    y = to_device(b, torch.float64).reshape(-1)
    n = x.numel()
    if n == 0:
        raise ValueError("first image must have finite values in [0, 1]")
    lib = nat.lib()
    ws = nat.workspace(lib.pdz_compare_workspace_bytes(), "compare")
    sums = torch.empty(2, dtype=torch.float64, device=x.device)
    flag = torch.empty(1, dtype=torch.int32, device=x.device)
    nat.check(lib.pdz_compare(nat.ptr(x), nat.ptr(y), n, nat.ptr(sums), nat.ptr(flag),
                              nat.ptr(ws), ws.numel(), nat.stream_ptr()))
    f = int(flag.item())
    if f & 1:
        raise ValueError("first image must have finite values in [0, 1]")
    if f & 2:
        raise ValueError("second image must have finite values in [0, 1]")
    s2, s1 = (float(v) for v in sums.to("cpu"))
    mse = s2 / n
    mae = s1 / n
    psnr = math.inf if mse == 0.0 else 10.0 * math.log10(1.0 / mse)
    return MetricReport(mse=mse, psnr=psnr, mae=mae)
