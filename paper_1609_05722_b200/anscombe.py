"""Anscombe transform kernels (reference: anscombe.py) with numpy-facing wrappers."""

from __future__ import annotations

import numpy as np

from . import _lib

ANSCOMBE_ZERO = float(np.sqrt(1.5))  # anscombe.py:13


def forward_device(y64, out=None):
    """v = 2 sqrt(y + 3/8) for a float64 CUDA tensor of counts -> float32 (anscombe.py:19-24)."""
    import torch
    v = out if out is not None else torch.empty(y64.shape, dtype=torch.float32, device=y64.device)
    _lib.check(_lib.lib().foe_anscombe_forward(y64.data_ptr(), v.data_ptr(), y64.numel(),
                                               torch.cuda.current_stream().cuda_stream), "anscombe_forward")
    return v


def forward_device_f32(y32):
    """The same from counts staged as exact float32 values (a CUDA tensor) -> float32."""
    import torch
    v = torch.empty(y32.shape, dtype=torch.float32, device=y32.device)
    _lib.check(_lib.lib().foe_anscombe_forward_f32(y32.data_ptr(), v.data_ptr(), y32.numel(),
                                                   torch.cuda.current_stream().cuda_stream), "anscombe_forward_f32")
    return v


def inverse_exact_unbiased_device(z32, counts=None):
    """Closed-form exact unbiased inverse (anscombe.py:33-51) -> float64 CUDA tensor."""
    import torch
    x = torch.empty(z32.shape, dtype=torch.float64, device=z32.device)
    _lib.check(_lib.lib().foe_anscombe_inverse_exact_unbiased(
        z32.data_ptr(), x.data_ptr(), z32.numel(), counts.data_ptr() if counts is not None else None,
        torch.cuda.current_stream().cuda_stream), "anscombe_inverse_exact_unbiased")
    return x


def anscombe_forward(y):
    """anscombe.py:19-24 (rejects negative counts)."""
    import torch
    y = np.asarray(y, dtype=np.float64)
    if y.size and y.min() < 0:
        raise ValueError("counts must be nonnegative")
    yd = torch.from_numpy(np.ascontiguousarray(y)).cuda()
    return forward_device(yd).double().cpu().numpy()


def anscombe_inverse_exact_unbiased(z, diagnostics: dict | None = None):
    """anscombe.py:33-51; ``diagnostics`` receives the two clamp counts."""
    import torch
    z = np.asarray(z, dtype=np.float64)
    zd = torch.from_numpy(np.ascontiguousarray(z)).to("cuda", torch.float32)
    cnt = torch.zeros(2, dtype=torch.int64, device="cuda")
    x = inverse_exact_unbiased_device(zd, cnt).cpu().numpy()
    if diagnostics is not None:
        c = cnt.cpu().tolist()
        diagnostics["n_clamped_input"] = int(c[0])
        diagnostics["n_clamped_output"] = int(c[1])
    return x
