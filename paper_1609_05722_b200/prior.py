"""Fields-of-Experts prior (reference: prior.py) on the GPU.

E(u) = sum_i w_i sum_p rho((k_i * u)_p),  rho(z) = log(1 + z^2)   (prior.py:1-10)

``FoEModel`` keeps the reference's model type (prior.py:38-84).  Energy and
gradient are one fused kernel pass (``foe_energy_grad`` in the C ABI), which
replaces the reference's per-filter convolve_same / potential /
convolve_adjoint loop (prior.py:95-110).
"""

from __future__ import annotations

import threading
from dataclasses import dataclass, replace

import numpy as np

from .image import BOUNDARY_CODES, FilterBasis

DOMAIN_TAGS = ("original", "anscombe")


def potential(z, order: int = 0):
    """rho and its derivatives (prior.py:23-35); host numpy helper for tests/tools."""
    z = np.asarray(z, dtype=np.float64)
    if order == 0:
        return np.log1p(z ** 2)
    if order == 1:
        return 2.0 * z / (1.0 + z ** 2)
    if order == 2:
        return 2.0 * (1.0 - z ** 2) / (1.0 + z ** 2) ** 2
    raise ValueError(f"order must be 0, 1 or 2, got {order}")


@dataclass(frozen=True)
class FoEModel:
    """Filter bank prior (prior.py:38-84)."""

    basis: FilterBasis
    betas: np.ndarray
    weights: np.ndarray
    domain_tag: str
    boundary: str = "symmetric"

    def __post_init__(self):
        betas = np.atleast_2d(np.asarray(self.betas, dtype=np.float64))
        weights = np.atleast_1d(np.asarray(self.weights, dtype=np.float64))
        object.__setattr__(self, "betas", betas)
        object.__setattr__(self, "weights", weights)
        if betas.shape[1] != self.basis.n_atoms:
            raise ValueError(f"betas have {betas.shape[1]} coefficients, basis has {self.basis.n_atoms} atoms")
        if weights.shape != (betas.shape[0],):
            raise ValueError(f"need one weight per filter, got {weights.shape} for {betas.shape[0]}")
        if not np.all(weights > 0):
            raise ValueError("expert weights must be strictly positive")
        if self.domain_tag not in DOMAIN_TAGS:
            raise ValueError(f"domain_tag must be one of {DOMAIN_TAGS}, got {self.domain_tag!r}")
        if self.boundary not in BOUNDARY_CODES:
            raise ValueError(f"boundary must be one of {tuple(BOUNDARY_CODES)}, got {self.boundary!r}")

    @property
    def n_filters(self) -> int:
        return self.betas.shape[0]

    @property
    def filters(self) -> np.ndarray:
        """(n_filters, m, m) composed filter stack (prior.py:75-78)."""
        return np.tensordot(self.betas, self.basis.atoms, axes=1)

    def with_weights(self, weights) -> "FoEModel":
        return replace(self, weights=np.asarray(weights, dtype=np.float64))

    def scaled(self, factor: float) -> "FoEModel":
        return self.with_weights(self.weights * factor)


class DeviceBank:
    """Device-resident filter bank (foe_bank_create) for one CUDA device."""

    def __init__(self, filters, weights, boundary: str = "symmetric"):
        from . import _lib
        import ctypes
        import torch

        filters = np.ascontiguousarray(filters, dtype=np.float64)
        weights = np.ascontiguousarray(weights, dtype=np.float64)
        if filters.ndim != 3 or filters.shape[1] != filters.shape[2]:
            raise ValueError(f"filters must be (n, m, m), got {filters.shape}")
        if boundary not in BOUNDARY_CODES:
            raise ValueError(f"boundary must be one of {tuple(BOUNDARY_CODES)}, got {boundary!r}")
        self.n, self.m = filters.shape[0], filters.shape[1]
        self.boundary = boundary
        self.device = torch.cuda.current_device()
        h = ctypes.c_void_p()
        _lib.check(_lib.lib().foe_bank_create(filters.ctypes.data, weights.ctypes.data, self.n, self.m,
                                              BOUNDARY_CODES[boundary], ctypes.byref(h)), "foe_bank_create")
        self.handle = h

    def __del__(self):
        try:
            from . import _lib
            if getattr(self, "handle", None):
                _lib.lib().foe_bank_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


_BANKS: dict = {}
_BANK_LOCK = threading.Lock()


def device_bank(model: FoEModel) -> DeviceBank:
    """Cached DeviceBank for ``model`` on the current device (keyed by content)."""
    import torch

    filters = np.ascontiguousarray(model.filters)
    key = (filters.tobytes(), model.weights.tobytes(), filters.shape, model.boundary, torch.cuda.current_device())
    with _BANK_LOCK:
        bank = _BANKS.get(key)
        if bank is None:
            if len(_BANKS) > 64:
                _BANKS.clear()
            bank = _BANKS[key] = DeviceBank(filters, model.weights, model.boundary)
    return bank


def _check_dims(shape, model: FoEModel):
    m = model.basis.size
    if len(shape) < 2 or shape[-2] < m or shape[-1] < m:
        raise ValueError(f"image shape {tuple(shape)} smaller than filter size {m}")


def energy_grad_device(u, model: FoEModel):
    """Fused F(u) and grad F(u) for a (B,H,W) or (H,W) fp32 CUDA tensor -> (energy fp64 (B,), grad)."""
    import torch

    from . import _lib

    _check_dims(u.shape, model)
    squeeze = u.dim() == 2
    u3 = (u[None] if squeeze else u).to(torch.float32).contiguous()
    B, H, W = u3.shape
    bank = device_bank(model)
    grad = torch.empty_like(u3)
    energy = torch.empty(B, dtype=torch.float64, device=u3.device)
    ws_bytes = _lib.lib().foe_eval_workspace_size(bank.handle, B, H, W)
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=u3.device)
    st = torch.cuda.current_stream().cuda_stream
    _lib.check(_lib.lib().foe_energy_grad(bank.handle, u3.data_ptr(), grad.data_ptr(), energy.data_ptr(), B, H, W,
                                          ws.data_ptr(), ws_bytes, st), "foe_energy_grad")
    return (energy, grad[0] if squeeze else grad)


def _to_device(u):
    import torch
    if isinstance(u, torch.Tensor):
        return u.cuda() if not u.is_cuda else u, True
    u = np.asarray(u, dtype=np.float64)
    return torch.from_numpy(u).to("cuda", torch.float32), False


def foe_energy(u, model: FoEModel) -> float:
    """sum_i w_i sum_p rho((k_i * u)_p) (prior.py:95-101)."""
    ud, _ = _to_device(u)
    e, _ = energy_grad_device(ud, model)
    return float(e[0].item()) if ud.dim() == 2 else e


def foe_gradient(u, model: FoEModel):
    """sum_i w_i K_i^T rho'(K_i u) (prior.py:104-110)."""
    ud, is_t = _to_device(u)
    _, g = energy_grad_device(ud, model)
    return g if is_t else g.double().cpu().numpy()
