"""Filter bases and the convolution operators (reference: image.py).

``FilterBasis`` / ``dct_basis`` / ``basis_by_name`` decode model files on the
host (image.py:86-141).  ``convolve_same`` / ``convolve_adjoint`` keep the
reference's operator surface (image.py:37-83) but run on the GPU through
``foe_convolve_same`` / ``foe_convolve_adjoint``; the solver itself never calls
them -- it uses the fused pass kernel.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

BOUNDARY_RULES = ("symmetric", "periodic")
BOUNDARY_CODES = {"symmetric": 0, "periodic": 1}


def _check_kernel(kernel: np.ndarray) -> int:
    """image.py:23-29: square, odd side; returns the radius."""
    kernel = np.asarray(kernel)
    if kernel.ndim != 2 or kernel.shape[0] != kernel.shape[1]:
        raise ValueError(f"kernel must be square 2D, got shape {kernel.shape}")
    if kernel.shape[0] % 2 != 1:
        raise ValueError(f"kernel side must be odd, got {kernel.shape[0]}")
    return kernel.shape[0] // 2


def _check_boundary(boundary: str) -> None:
    if boundary not in BOUNDARY_RULES:
        raise ValueError(f"boundary must be one of {BOUNDARY_RULES}, got {boundary!r}")


def _single_filter_op(x, kernel, boundary, adjoint):
    import torch

    from . import _lib
    from .prior import DeviceBank

    _check_kernel(kernel)
    _check_boundary(boundary)
    x = np.asarray(x, dtype=np.float64)
    if x.ndim != 2:
        raise ValueError("expected a 2d array")
    kernel = np.asarray(kernel, dtype=np.float64)
    bank = DeviceBank(kernel[None], np.ones(1), boundary)
    dev = torch.device("cuda", torch.cuda.current_device())
    xd = torch.from_numpy(x).to(dev, torch.float32).contiguous()
    out = torch.empty_like(xd)
    st = torch.cuda.current_stream().cuda_stream
    fn = _lib.lib().foe_convolve_adjoint if adjoint else _lib.lib().foe_convolve_same
    _lib.check(fn(bank.handle, 0, xd.data_ptr(), out.data_ptr(), 1, x.shape[0], x.shape[1], st),
               "convolve_adjoint" if adjoint else "convolve_same")
    return out.double().cpu().numpy()


def convolve_same(x: np.ndarray, kernel: np.ndarray, boundary: str = "symmetric") -> np.ndarray:
    """True 2-D convolution, 'same' output (image.py:37-58), fp32 on the GPU."""
    return _single_filter_op(x, kernel, boundary, adjoint=False)


def convolve_adjoint(y: np.ndarray, kernel: np.ndarray, boundary: str = "symmetric") -> np.ndarray:
    """Exact adjoint of convolve_same (image.py:68-83), fp32 on the GPU."""
    return _single_filter_op(y, kernel, boundary, adjoint=True)


@dataclass(frozen=True)
class FilterBasis:
    """Orthonormal zero-mean filter basis (image.py:86-114)."""

    atoms: np.ndarray
    name: str

    @property
    def n_atoms(self) -> int:
        return self.atoms.shape[0]

    @property
    def size(self) -> int:
        return self.atoms.shape[1]

    def compose(self, beta: np.ndarray) -> np.ndarray:
        beta = np.asarray(beta, dtype=np.float64)
        if beta.shape != (self.n_atoms,):
            raise ValueError(f"beta must have shape ({self.n_atoms},), got {beta.shape}")
        return np.tensordot(beta, self.atoms, axes=1)

    def coefficients(self, kernel: np.ndarray) -> np.ndarray:
        return np.tensordot(self.atoms, kernel, axes=2)


def dct_basis(m: int) -> FilterBasis:
    """2-D orthonormal DCT-II basis minus the constant atom (image.py:117-130)."""
    if m < 2:
        raise ValueError("basis needs m >= 2")
    i = np.arange(m)
    d = np.cos(np.pi * (2 * i[None, :] + 1) * i[:, None] / (2 * m))
    d[0] *= np.sqrt(1.0 / m)
    d[1:] *= np.sqrt(2.0 / m)
    atoms = np.einsum("pi,qj->pqij", d, d).reshape(m * m, m, m)[1:]
    return FilterBasis(atoms=np.ascontiguousarray(atoms), name=f"dct{m}")


_BASIS_BUILDERS = {"dct": dct_basis}


def basis_by_name(name: str) -> FilterBasis:
    """'dct7' -> dct_basis(7) (image.py:136-141)."""
    for prefix, builder in _BASIS_BUILDERS.items():
        if name.startswith(prefix) and name[len(prefix):].isdigit():
            return builder(int(name[len(prefix):]))
    raise ValueError(f"unknown filter basis {name!r}")
