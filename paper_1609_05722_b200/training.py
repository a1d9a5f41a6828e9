"""Training-side operators on the device, fp64 (reference training.py).

The bilevel trainer differentiates the loss through the lower-level minimiser by implicit
differentiation, which needs the Hessian of the lower energy applied matrix-free, a CG solve with
it, and the parameter-gradient reductions:

    H p = sum_i wgt_i K_i^T diag(rho''(K_i w)) K_i p + d2D p            (training.py:158-174)
    dL/dbeta_ij = -wgt_i ( <rho'(K_i w), B_j q> + <rho''(K_i w) K_i q, B_j w> ),
    dL/dlog w_i = -wgt_i <rho'(K_i w), K_i q>,   q = H^-1 dL/dw           (training.py:317-356)

The Hessian-vector product is one fused fp64 kernel per call (``foe_hessian_apply64``: K w and K p,
the rho'' weighting and the exact adjoint per tile, no N x H x W intermediate); the conjugate-gradient
solve runs on the device (``foe_cg_solve64``: dot products, step lengths, the residual test and the
breakdown test in kernels, the iteration loop a CUDA graph) with one host synchronise per CG attempt;
the reference's restart rule (H + eps I, eps escalating tenfold) stays on the host.  The gradient and
the parameter-gradient reductions use the fp64 bank kernels (``foe_conv_bank64`` /
``foe_adjoint_bank64``) and fp64 GEMMs.  fp64 throughout because the reference trains with 1e-9 CG and
stationarity tolerances.  The L-BFGS driver, lower solve and checkpointing are out of scope.
"""
from __future__ import annotations

import warnings
from dataclasses import dataclass

import numpy as np

from .prior import FoEModel

OBJECTIVES = ("original_domain", "anscombe_domain")
_OBJECTIVE_TAG = {"original_domain": "original", "anscombe_domain": "anscombe"}
ANSCOMBE_ZERO = float(np.sqrt(1.5))
_S = float(np.sqrt(1.5))


@dataclass(frozen=True)
class TrainingSample:
    """One clean/noisy pair with the cached Anscombe transform (training.py:43-70)."""

    clean: np.ndarray
    noisy: np.ndarray
    transformed: np.ndarray

    def __post_init__(self):
        if self.clean.shape != self.noisy.shape or self.clean.shape != self.transformed.shape:
            raise ValueError("sample images must share one shape")
        if not np.array_equal(self.noisy, np.round(self.noisy)) or self.noisy.min() < 0:
            raise ValueError("noisy image must hold nonnegative integer counts")
        if not np.allclose(self.transformed, 2.0 * np.sqrt(self.noisy + 0.375), atol=1e-12):
            raise ValueError("cached transform inconsistent with noisy image")

    @classmethod
    def create(cls, clean: np.ndarray, noisy: np.ndarray) -> "TrainingSample":
        noisy = np.asarray(noisy, dtype=np.float64)
        return cls(clean=np.asarray(clean, dtype=np.float64), noisy=noisy, transformed=2.0 * np.sqrt(noisy + 0.375))


@dataclass(frozen=True)
class TrainConfig:
    """The knobs the operators read (training.py:78-104 defaults)."""

    objective: str = "anscombe_domain"
    hessian_cg_tol: float = 1e-9
    hessian_cg_max_iters: int = 600
    data_weight: float = 1.0

    def __post_init__(self):
        if self.objective not in OBJECTIVES:
            raise ValueError(f"objective must be one of {OBJECTIVES}, got {self.objective!r}")
        if self.hessian_cg_tol <= 0:
            raise ValueError("tolerances must be positive")


def _check_domain(model: FoEModel, objective: str) -> None:
    if objective not in OBJECTIVES:
        raise ValueError(f"objective must be one of {OBJECTIVES}, got {objective!r}")
    if model.domain_tag != _OBJECTIVE_TAG[objective]:
        raise ValueError(f"model domain_tag {model.domain_tag!r} inconsistent with objective {objective!r}")


# ---- device helpers ---------------------------------------------------------------------------------

def _dev(a):
    import torch
    if isinstance(a, torch.Tensor):
        return a.to(device="cuda", dtype=torch.float64).contiguous()
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float64))).cuda()


class _Bank64:
    """Device copy of a model's filters / weights / atoms (fp64, reference orientation)."""

    def __init__(self, model: FoEModel):
        from .image import BOUNDARY_CODES
        self.filters = _dev(model.filters)
        self.weights = _dev(model.weights)
        self.atoms = _dev(model.basis.atoms)
        self.m = int(self.filters.shape[-1])
        self.boundary = BOUNDARY_CODES[model.boundary]

    def conv(self, x, filt=None):
        """(B,H,W) -> (B,n,H,W): convolve_same with every filter (image.py:37-58)."""
        import torch

        from . import _lib
        filt = self.filters if filt is None else filt
        x3 = x[None] if x.dim() == 2 else x
        B, H, W = x3.shape
        out = torch.empty((B, filt.shape[0], H, W), dtype=torch.float64, device=x.device)
        _lib.check(_lib.lib().foe_conv_bank64(filt.data_ptr(), filt.shape[0], self.m, self.boundary, x3.data_ptr(),
                                              out.data_ptr(), B, H, W, torch.cuda.current_stream().cuda_stream),
                   "conv_bank64")
        return out

    def adjoint(self, y, filt=None):
        """(B,n,H,W) -> (B,H,W): sum_i convolve_adjoint(y_i, k_i) (image.py:68-83)."""
        import torch

        from . import _lib
        filt = self.filters if filt is None else filt
        B, n, H, W = y.shape
        out = torch.empty((B, H, W), dtype=torch.float64, device=y.device)
        _lib.check(_lib.lib().foe_adjoint_bank64(filt.data_ptr(), n, self.m, self.boundary, y.contiguous().data_ptr(),
                                                 out.data_ptr(), B, H, W, torch.cuda.current_stream().cuda_stream),
                   "adjoint_bank64")
        return out


def _rho1(z):  # prior.py:31-32
    return 2.0 * z / (1.0 + z * z)


def _rho2(z):  # prior.py:33-34
    q = 1.0 + z * z
    return 2.0 * (1.0 - z * z) / (q * q)


# ---- operators (numpy in / numpy out, as the reference) ---------------------------------------------

def foe_gradient64(w, model: FoEModel) -> np.ndarray:
    """sum_i wgt_i K_i^T rho'(K_i w) in fp64 on the device (prior.py:104-110)."""
    bank = _Bank64(model)
    wd = _dev(w)
    z = bank.conv(wd)
    return bank.adjoint(bank.weights[None, :, None, None] * _rho1(z))[0].cpu().numpy()


def _data_gradient_dev(wd, sample, objective, lam):
    import torch
    if objective == "anscombe_domain":
        return wd - _dev(sample.transformed)
    f = _dev(sample.noisy)
    ratio = torch.where(f > 0, f / torch.clamp(wd, min=1e-150), torch.zeros_like(wd))
    return lam * (1.0 - ratio)


def _total_gradient_dev(bank, wd, sample, objective, lam):
    z = bank.conv(wd)
    return bank.adjoint(bank.weights[None, :, None, None] * _rho1(z))[0] + _data_gradient_dev(wd, sample, objective, lam)


def total_gradient(w, model, sample, objective, lam=1.0) -> np.ndarray:
    """Gradient of the full lower objective at w (training.py:132-134)."""
    _check_domain(model, objective)
    return _total_gradient_dev(_Bank64(model), _dev(w), sample, objective, lam).cpu().numpy()


def _pinned_mask_dev(wd, gd, sample, objective):
    """Pixels on the x = 0 constraint with the gradient pushing into it (training.py:137-146)."""
    if objective != "original_domain":
        return None
    return (_dev(sample.noisy) == 0) & (wd <= 1e-12) & (gd > 0)


def stationarity_residual(w, model, sample, objective, lam=1.0) -> float:
    """Sup-norm of the lower gradient, KKT-consistent zeros masked out (training.py:149-155)."""
    import torch
    _check_domain(model, objective)
    wd = _dev(w)
    g = _total_gradient_dev(_Bank64(model), wd, sample, objective, lam)
    pinned = _pinned_mask_dev(wd, g, sample, objective)
    if pinned is not None:
        g = torch.where(pinned, torch.zeros_like(g), g)
    return float(g.abs().max().item())


_OBJECTIVE_CODE = {"anscombe_domain": 0, "original_domain": 1}
CG_CONVERGED, CG_BREAKDOWN, CG_MAXITER = 1, 2, 3


def _hvp_fused(bank, wd, p, objective, lam, fd=None, free=None, eps=0.0):
    """(H + eps I) p through foe_hessian_apply64 (one fused kernel); free: uint8 device mask or None."""
    import torch

    from . import _lib
    H, W = p.shape
    out = torch.empty_like(p)
    _lib.check(_lib.lib().foe_hessian_apply64(
        bank.filters.data_ptr(), bank.weights.data_ptr(), bank.filters.shape[0], bank.m, bank.boundary,
        _OBJECTIVE_CODE[objective], float(lam), wd.data_ptr(), fd.data_ptr() if fd is not None else None,
        free.data_ptr() if free is not None else None, p.contiguous().data_ptr(), float(eps), out.data_ptr(), H, W,
        torch.cuda.current_stream().cuda_stream), "hessian_apply64")
    return out


def hessian_apply(w, model, objective, p, sample, lam=1.0) -> np.ndarray:
    """H p with H = sum_i wgt_i K_i^T diag(rho''(K_i w)) K_i + d2D, matrix-free (training.py:158-174)."""
    bank = _Bank64(model)
    fd = _dev(sample.noisy) if objective == "original_domain" else None
    return _hvp_fused(bank, _dev(w), _dev(p), objective, lam, fd).cpu().numpy()


def solve_hessian_system(w, model, objective, rhs, sample, lam=1.0, tol=1e-9, max_iters=600, free=None):
    """Conjugate gradient for H q = rhs on the device; returns (q, info) (training.py:183-237).

    Same algorithm as the reference: restarts with H + eps I when a search direction has
    non-positive curvature (eps from the same Philox trace estimate, escalating tenfold), ``free``
    restricting the system to unpinned pixels.  Each attempt is one device-resident CG
    (``foe_cg_solve64``); the host reads its status and residual history once per attempt."""
    import ctypes

    import torch

    from . import _lib
    bank = _Bank64(model)
    wd = _dev(w)
    fd = _dev(sample.noisy) if objective == "original_domain" else None
    rhs_d = _dev(rhs)
    H, W = rhs_d.shape
    fr = None
    if free is not None:
        fr = torch.as_tensor(np.ascontiguousarray(np.asarray(free, dtype=np.uint8)), device="cuda")
        rhs_d = torch.where(fr.bool(), rhs_d, torch.zeros_like(rhs_d))
    rhs_norm = float(torch.linalg.vector_norm(rhs_d).item())
    info = {"iterations": 0, "residuals": [], "regularization": 0.0}
    if rhs_norm == 0:
        return np.zeros(rhs_d.shape), info
    # stochastic trace estimate with the reference's Rademacher probe (training.py:177-180)
    zt = np.where(np.random.Generator(np.random.Philox(key=0xC0FFEE)).random(tuple(rhs_d.shape)) < 0.5, -1.0, 1.0)
    zt = _dev(zt)
    tr_est = float(torch.dot(zt.reshape(-1), _hvp_fused(bank, wd, zt, objective, lam, fd, fr).reshape(-1)).item())
    eps = 0.0
    eps_unit = 1e-6 * max(tr_est, 0.0) / rhs_d.numel() + 1e-300
    L = _lib.lib()
    ws = torch.empty(L.foe_cg_workspace_size(H, W, max_iters), dtype=torch.uint8, device="cuda")
    q = torch.empty_like(rhs_d)
    residuals = []
    for _ in range(6):
        status, iters = ctypes.c_int(), ctypes.c_int()
        res = np.zeros(max_iters + 1)
        _lib.check(L.foe_cg_solve64(
            bank.filters.data_ptr(), bank.weights.data_ptr(), bank.filters.shape[0], bank.m, bank.boundary,
            _OBJECTIVE_CODE[objective], float(lam), wd.data_ptr(), fd.data_ptr() if fd is not None else None,
            fr.data_ptr() if fr is not None else None, rhs_d.data_ptr(), float(eps), float(tol), int(max_iters),
            q.data_ptr(), ctypes.byref(status), ctypes.byref(iters), res.ctypes.data, H, W, ws.data_ptr(),
            ws.numel(), torch.cuda.current_stream().cuda_stream), "cg_solve64")
        residuals = res[:iters.value + 1].tolist()
        if status.value in (CG_CONVERGED, CG_MAXITER):
            info.update(iterations=iters.value, residuals=residuals, regularization=eps)
            return q.cpu().numpy(), info
        eps = eps_unit if eps == 0.0 else eps * 10.0  # CG_BREAKDOWN: training.py:233-235
        warnings.warn(f"non-positive curvature in Hessian solve; regularizing with eps={eps:.3e}")
    info.update(iterations=max_iters, residuals=residuals, regularization=eps)
    return q.cpu().numpy(), info


def _loss_gradient_wrt_w_dev(wd, sample, objective):
    """dL/dw of the upper loss (training.py:308-314)."""
    import torch
    g = _dev(sample.clean)
    if objective == "original_domain":
        return wd - g
    zc = torch.clamp(wd, min=ANSCOMBE_ZERO)
    x = zc ** 2 / 4.0 + _S / (4.0 * zc) - 11.0 / (8.0 * zc ** 2) + 5.0 * _S / (8.0 * zc ** 3) - 0.125  # anscombe.py:46
    x = torch.where(x < 0, torch.zeros_like(x), x)
    deriv = zc / 2.0 - _S / (4.0 * zc ** 2) + 11.0 / (4.0 * zc ** 3) - 15.0 * _S / (8.0 * zc ** 4)  # anscombe.py:59
    deriv = torch.where(wd > ANSCOMBE_ZERO, deriv, torch.zeros_like(deriv))
    return deriv * (x - g)


def param_gradients(w_star, model, sample, objective, cfg: TrainConfig):
    """Implicit-differentiation gradients (dL/dbeta, dL/dlogweight) (training.py:317-356)."""
    import torch
    _check_domain(model, objective)
    lam = cfg.data_weight
    res = stationarity_residual(w_star, model, sample, objective, lam)
    if res > 1e-4:
        raise ValueError(f"w_star is not stationary (gradient sup-norm {res:.3e})")
    bank = _Bank64(model)
    wd = _dev(w_star)
    g = _total_gradient_dev(bank, wd, sample, objective, lam)
    pinned = _pinned_mask_dev(wd, g, sample, objective)
    rhs = _loss_gradient_wrt_w_dev(wd, sample, objective)
    q, _ = solve_hessian_system(w_star, model, objective, rhs, sample, lam, tol=cfg.hessian_cg_tol,
                                max_iters=cfg.hessian_cg_max_iters,
                                free=None if pinned is None else (~pinned).cpu().numpy())
    qd = _dev(q)
    bq = bank.conv(qd, bank.atoms)[0].reshape(bank.atoms.shape[0], -1)   # B_j q
    bw = bank.conv(wd, bank.atoms)[0].reshape(bank.atoms.shape[0], -1)   # B_j w
    z = bank.conv(wd)[0].reshape(bank.filters.shape[0], -1)              # K_i w
    kq = bank.conv(qd)[0].reshape(bank.filters.shape[0], -1)             # K_i q
    rho1 = _rho1(z)
    gkq = _rho2(z) * kq
    t1 = rho1 @ bq.T                                                     # einsum("ihw,jhw->ij")
    t2 = gkq @ bw.T
    d_beta = -bank.weights[:, None] * (t1 + t2)
    d_logw = -bank.weights * torch.sum(rho1 * kq, dim=1)
    return d_beta.cpu().numpy(), d_logw.cpu().numpy()
