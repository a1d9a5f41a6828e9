"""PSNR and mean SSIM scoring on the device (reference metrics.py:30-102).

Same convention as the reference: the clean image is peak-scaled, both images are mapped to
[0, 255] by 255 / peak and data_range is 255; SSIM uses an 11 x 11 Gaussian window (sigma 1.5)
with valid-mode local statistics.  fp64 kernels with fixed-order sums (``foe_score``).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

SSIM_WINDOW = 11
SSIM_SIGMA = 1.5
SSIM_K1 = 0.01
SSIM_K2 = 0.03


@dataclass(frozen=True)
class ScoreReport:
    """Quality of one denoised image against its ground truth (metrics.py:75-88)."""

    psnr_db: float
    mssim: float
    image_id: str
    method_id: str
    peak: float

    def __post_init__(self):
        if not (-1e-12 <= self.mssim <= 1.0 + 1e-12):
            raise ValueError(f"mssim out of range: {self.mssim}")
        if not (np.isfinite(self.psnr_db) or self.psnr_db == float("inf")):
            raise ValueError(f"psnr must be finite or +inf, got {self.psnr_db}")


def _as_device(a):
    import torch

    from ._host import upload
    if isinstance(a, torch.Tensor):
        return a.to(device="cuda", dtype=torch.float64).contiguous()
    return upload(np.asarray(a, dtype=np.float64))


def score_batch(x_hat, g, peak: float):
    """(psnr[B], mssim[B]) of (B,H,W) or (H,W) estimates against ground truths (numpy or CUDA),
    after the [0, 255] convention with the given peak."""
    import torch

    from . import _lib
    xd, gd = _as_device(x_hat), _as_device(g)
    if xd.shape != gd.shape:
        raise ValueError(f"shape mismatch {tuple(xd.shape)} vs {tuple(gd.shape)}")
    if xd.dim() == 2:
        xd, gd = xd[None], gd[None]
    B, H, W = xd.shape
    if min(H, W) < SSIM_WINDOW:
        raise ValueError(f"images must be at least {SSIM_WINDOW} pixels per side, got {(H, W)}")
    if not peak > 0:
        raise ValueError(f"peak must be positive, got {peak}")
    L = _lib.lib()
    nbytes = L.foe_score_workspace_size(B, H, W)
    ws = torch.empty(nbytes, dtype=torch.uint8, device=xd.device)
    out = torch.empty((2, B), dtype=torch.float64, device=xd.device)
    _lib.check(L.foe_score(xd.data_ptr(), gd.data_ptr(), B, H, W, float(peak), out[0].data_ptr(),
                           out[1].data_ptr(), ws.data_ptr(), nbytes, torch.cuda.current_stream().cuda_stream),
               "score")
    res = out.cpu().numpy()
    return res[0], res[1]


def score_denoised(x_hat, g, peak: float, image_id: str = "", method_id: str = "") -> ScoreReport:
    """Apply the [0, 255] scoring convention and produce a report (metrics.py:91-102)."""
    p, m = score_batch(x_hat, g, peak)
    return ScoreReport(psnr_db=float(p[0]), mssim=float(m[0]), image_id=image_id, method_id=method_id, peak=peak)
