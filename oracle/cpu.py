"""CPU oracle for the FoE denoise hot path -- TEST INFRASTRUCTURE ONLY.

Python face of ``oracle/foe_oracle.c`` (float64 restatement of the reference
``foepoisson`` hot path) plus the host-side rules of ``pipeline.py`` restated in
plain Python/numpy.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (cpu_baseline leg and ``--impl reference`` arm) may import this
module; the product package never does.

Pinned against golden vectors produced by the reference itself
(``tests/golden/make_golden.py`` -> ``tests/golden/*.npz``), see
``tests/test_oracle.py``.
"""

from __future__ import annotations

import ctypes
import json
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

_dp = ctypes.POINTER(ctypes.c_double)
_lp = ctypes.POINTER(ctypes.c_long)
_ip = ctypes.POINTER(ctypes.c_int)

BOUNDARY_CODES = {"symmetric": 0, "periodic": 1}


def build(force: bool = False) -> str:
    """Compile liboracle.so with oracle/Makefile (gcc, no GPU needed)."""
    src = os.path.join(_HERE, "foe_oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.orc_convolve_same.argtypes = [_dp, ctypes.c_int, ctypes.c_int, _dp, ctypes.c_int, ctypes.c_int, _dp]
        L.orc_convolve_adjoint.argtypes = L.orc_convolve_same.argtypes
        L.orc_foe_energy.argtypes = [_dp, ctypes.c_int, ctypes.c_int, _dp, _dp, ctypes.c_int, ctypes.c_int, ctypes.c_int]
        L.orc_foe_energy.restype = ctypes.c_double
        L.orc_foe_gradient.argtypes = [_dp, ctypes.c_int, ctypes.c_int, _dp, _dp, ctypes.c_int, ctypes.c_int,
                                       ctypes.c_int, _dp]
        L.orc_prox_quadratic.argtypes = [_dp, _dp, ctypes.c_double, ctypes.c_long, _dp]
        L.orc_prox_idiv.argtypes = [_dp, _dp, ctypes.c_double, ctypes.c_long, _dp]
        L.orc_anscombe_forward.argtypes = [_dp, ctypes.c_long, _dp]
        L.orc_anscombe_inverse_exact_unbiased.argtypes = [_dp, ctypes.c_long, _dp, _lp]
        L.orc_ipiano_foe.argtypes = [_dp, _dp, ctypes.c_int, ctypes.c_int, _dp, _dp, ctypes.c_int, ctypes.c_int,
                                     ctypes.c_int, ctypes.c_double, ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                     ctypes.c_double, ctypes.c_double, ctypes.c_int, ctypes.c_double,
                                     ctypes.c_double, _dp, _dp, _ip, _ip]
        L.orc_ipiano_foe.restype = ctypes.c_int
        L.orc_ipiano_foe_ex.argtypes = L.orc_ipiano_foe.argtypes + [ctypes.c_void_p]
        L.orc_ipiano_foe_ex.restype = ctypes.c_int
        L.orc_num_threads.restype = ctypes.c_int
        L.orc_set_num_threads.argtypes = [ctypes.c_int]
        _lib = L
    return _lib


def num_threads() -> int:
    return lib().orc_num_threads()


def set_num_threads(n: int) -> None:
    lib().orc_set_num_threads(int(n))


def _c(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _p(a):
    return a.ctypes.data_as(_dp)


# --------------------------------------------------------------------------
# filter basis / model decode: image.py:117-130 (dct_basis), prior.py:75-78


def dct_atoms(m: int) -> np.ndarray:
    """Zero-mean orthonormal 2-D DCT-II atoms (m*m - 1, m, m); image.py:117-130."""
    i = np.arange(m)
    d = np.cos(np.pi * (2 * i[None, :] + 1) * i[:, None] / (2 * m))
    d[0] *= np.sqrt(1.0 / m)
    d[1:] *= np.sqrt(2.0 / m)
    return np.einsum("pi,qj->pqij", d, d).reshape(m * m, m, m)[1:].copy()


@dataclass
class OracleModel:
    """Filter bank in the reference's terms: filters (N, m, m), weights (N,)."""

    filters: np.ndarray
    weights: np.ndarray
    boundary: str = "symmetric"
    domain_tag: str = "anscombe"

    @property
    def m(self) -> int:
        return self.filters.shape[1]

    @property
    def n(self) -> int:
        return self.filters.shape[0]


def read_foe(path) -> OracleModel:
    """Minimal FOE 1 reader (fileio.py:51-79) for the oracle side."""
    with open(path) as fh:
        lines = [ln.strip() for ln in fh if ln.strip()]
    assert lines[0] == "FOE 1"
    tag, nf, m, basis, boundary = lines[1].split()
    nf, m = int(nf), int(m)
    assert basis == f"dct{m}"
    rows = np.array([[float(t) for t in ln.split()] for ln in lines[2:2 + nf]])
    atoms = dct_atoms(m)
    filters = np.tensordot(rows[:, 1:], atoms, axes=1)
    return OracleModel(filters=filters, weights=rows[:, 0].copy(), boundary=boundary, domain_tag=tag)


# --------------------------------------------------------------------------
# numerics core (foe_oracle.c)


def convolve_same(x, k, boundary="symmetric"):
    """image.py:37-58."""
    x = _c(x)
    k = _c(k)
    out = np.empty_like(x)
    lib().orc_convolve_same(_p(x), x.shape[0], x.shape[1], _p(k), k.shape[0], BOUNDARY_CODES[boundary], _p(out))
    return out


def convolve_adjoint(y, k, boundary="symmetric"):
    """image.py:68-83."""
    y = _c(y)
    k = _c(k)
    out = np.empty_like(y)
    lib().orc_convolve_adjoint(_p(y), y.shape[0], y.shape[1], _p(k), k.shape[0], BOUNDARY_CODES[boundary], _p(out))
    return out


def foe_energy(u, model: OracleModel) -> float:
    """prior.py:95-101."""
    u = _c(u)
    f = _c(model.filters)
    w = _c(model.weights)
    return float(lib().orc_foe_energy(_p(u), u.shape[0], u.shape[1], _p(f), _p(w), model.n, model.m,
                                      BOUNDARY_CODES[model.boundary]))


def foe_gradient(u, model: OracleModel) -> np.ndarray:
    """prior.py:104-110."""
    u = _c(u)
    f = _c(model.filters)
    w = _c(model.weights)
    g = np.empty_like(u)
    lib().orc_foe_gradient(_p(u), u.shape[0], u.shape[1], _p(f), _p(w), model.n, model.m,
                           BOUNDARY_CODES[model.boundary], _p(g))
    return g


def prox_quadratic(ut, t, v):
    """solver.py:92-100."""
    ut = _c(ut)
    v = _c(v)
    out = np.empty_like(ut)
    lib().orc_prox_quadratic(_p(ut), _p(v), float(t), ut.size, _p(out))
    return out


def prox_idiv(ut, t, obs):
    """solver.py:103-125."""
    ut = _c(ut)
    obs = _c(obs)
    out = np.empty_like(ut)
    lib().orc_prox_idiv(_p(ut), _p(obs), float(t), ut.size, _p(out))
    return out


def anscombe_forward(y):
    """anscombe.py:19-24."""
    y = _c(y)
    if y.min() < 0:
        raise ValueError("counts must be nonnegative")
    v = np.empty_like(y)
    lib().orc_anscombe_forward(_p(y), y.size, _p(v))
    return v


def anscombe_inverse_exact_unbiased(z, diagnostics=None):
    """anscombe.py:33-51."""
    z = _c(z)
    x = np.empty_like(z)
    cnt = (ctypes.c_long * 2)()
    lib().orc_anscombe_inverse_exact_unbiased(_p(z), z.size, _p(x), cnt)
    if diagnostics is not None:
        diagnostics["n_clamped_input"] = int(cnt[0])
        diagnostics["n_clamped_output"] = int(cnt[1])
    return x


@dataclass
class OracleTrace:
    F: list = field(default_factory=list)
    G: list = field(default_factory=list)
    L: list = field(default_factory=list)
    step_norm: list = field(default_factory=list)
    descent_slack: list = field(default_factory=list)
    slack_tol: list = field(default_factory=list)
    n_trials: int = 0
    status: int = 0


def ipiano_foe(u0, obs, model: OracleModel, lam, branch, *, gamma=0.8, lipschitz_init=1.0,
               backtrack_factor=1.2, relax_factor=1.05, max_iters=150, rel_tol=1e-6,
               max_lipschitz=1e15, return_iterates=False):
    """ipiano_minimize (solver.py:128-175) with FoE callbacks (pipeline.py:167-172, 205-208).

    branch: "quadratic" or "idiv" (prox and energy_G, pipeline.py:197-204).
    Returns (u, OracleTrace), plus (n_iters, H, W) fp32 accepted iterates if return_iterates."""
    u0 = _c(u0)
    obs = _c(obs)
    f = _c(model.filters)
    w = _c(model.weights)
    H, W = u0.shape
    u = np.empty_like(u0)
    trace = np.zeros((max_iters, 6))
    it = ctypes.c_int(0)
    tr = ctypes.c_int(0)
    iters = np.empty((int(max_iters), H, W), dtype=np.float32) if return_iterates else None
    status = lib().orc_ipiano_foe_ex(_p(u0), _p(obs), H, W, _p(f), _p(w), model.n, model.m,
                                     BOUNDARY_CODES[model.boundary], float(lam),
                                     0 if branch == "quadratic" else 1, gamma, lipschitz_init,
                                     backtrack_factor, relax_factor, int(max_iters), rel_tol,
                                     max_lipschitz, _p(u), _p(trace), ctypes.byref(it), ctypes.byref(tr),
                                     iters.ctypes.data if return_iterates else None)
    n = it.value
    t = OracleTrace(F=list(trace[:n, 0]), G=list(trace[:n, 1]), L=list(trace[:n, 2]),
                    step_norm=list(trace[:n, 3]), descent_slack=list(trace[:n, 4]),
                    slack_tol=list(trace[:n, 5]), n_trials=tr.value, status=status)
    if return_iterates:
        return u, t, iters[:n]
    return u, t


# --------------------------------------------------------------------------
# pipeline rules (pipeline.py:83-131) restated


QUADRATIC_PEAK_THRESHOLD = 5.0  # pipeline.py:25
BIN_FACTOR = 3  # noise.py:9


def load_lambda_table(path):
    with open(path) as fh:
        return json.load(fh)


def solver_budget(peak: float) -> int:
    """pipeline.py:83-87: 150 iterations below peak 5, else 60."""
    return 150 if peak < QUADRATIC_PEAK_THRESHOLD else 60


def select_lambda(peak, variant, table, force_branch=None) -> float:
    """pipeline.py:98-131: log-log interpolation, clamped at the ends."""
    if variant == "direct":
        name, p = "direct", peak
    else:
        p = peak * BIN_FACTOR ** 2 if variant == "transform_binned" else peak
        if force_branch is not None:
            name = f"transform_{force_branch}"
        elif p >= QUADRATIC_PEAK_THRESHOLD:
            name = "transform_quadratic"
        else:
            name = "transform_idiv"
    rows = sorted(table["tables"][name])
    peaks = np.array([r[0] for r in rows])
    lams = np.array([r[1] for r in rows])
    return float(np.exp(np.interp(np.log(p), np.log(peaks), np.log(lams))))


def bin3(img, factor=BIN_FACTOR):
    """noise.py:55-71: factor x factor block sums, bottom/right edge-replicate padding."""
    img = np.asarray(img, dtype=np.float64)
    if factor == 1:
        return img.copy()
    h, w = img.shape
    img = np.pad(img, ((0, (-h) % factor), (0, (-w) % factor)), mode="edge")
    return img.reshape(img.shape[0] // factor, factor, img.shape[1] // factor, factor).sum(axis=(1, 3))


def unbin_bilinear(img, target_shape, factor=BIN_FACTOR):
    """noise.py:74-113: divide by factor^2, corner-aligned bilinear upsampling, crop."""
    img = np.asarray(img, dtype=np.float64)
    H, W = target_shape
    if factor == 1 and img.shape == (H, W):
        return img.copy()
    Hp, Wp = -(-H // factor) * factor, -(-W // factor) * factor
    src = img / float(factor ** 2)
    h, w = src.shape
    out = np.empty((Hp, Wp))
    for Y in range(Hp):
        row = Y * (h - 1.0) / (Hp - 1.0) if (h > 1 and Hp > 1) else 0.0
        i0 = min(int(row), h - 2) if h > 1 else 0
        di = row - i0 if h > 1 else 0.0
        i1 = min(i0 + 1, h - 1)
        for X in range(Wp):
            col = X * (w - 1.0) / (Wp - 1.0) if (w > 1 and Wp > 1) else 0.0
            j0 = min(int(col), w - 2) if w > 1 else 0
            dj = col - j0 if w > 1 else 0.0
            j1 = min(j0 + 1, w - 1)
            top = src[i0, j0] + (src[i0, j1] - src[i0, j0]) * dj
            bot = src[i1, j0] + (src[i1, j1] - src[i1, j0]) * dj
            out[Y, X] = top + (bot - top) * di
    return out[:H, :W]


def denoise(noisy, peak, model: OracleModel, variant, table, lam="auto", zero_offset_c=0.1,
            force_branch=None, rel_tol=1e-6, max_iters=None, bin_factor=BIN_FACTOR):
    """denoise_transform / denoise_direct (pipeline.py:152-211) on the C oracle.

    max_iters=None applies solver_budget (pipeline.py:83-87); an explicit value
    bypasses it (the truncated-oracle mode of SURVEY.md Appendix B)."""
    noisy = _c(noisy)
    if variant == "transform_binned":  # pipeline.py:214-235
        f = int(bin_factor)
        inner = denoise(bin3(noisy, f), float(f ** 2) * peak, model, "transform", table, lam, zero_offset_c,
                        force_branch, rel_tol, max_iters)
        inner["image"] = unbin_bilinear(inner["image"], noisy.shape, f)
        inner["peak_used"] = float(f ** 2) * peak
        return inner
    lam_v = select_lambda(peak, variant, table, force_branch) if lam == "auto" else float(lam)
    iters = solver_budget(peak) if max_iters is None else int(max_iters)
    if variant == "direct":
        obs = np.where(noisy == 0, zero_offset_c, noisy)
        u, tr = ipiano_foe(obs, obs, model, lam_v, "idiv", max_iters=iters, rel_tol=rel_tol)
        return {"image": u, "branch": "direct_idiv", "lam": lam_v, "trace": tr, "transformed": None}
    v = anscombe_forward(noisy)
    quadratic = (force_branch == "quadratic") if force_branch is not None else peak >= QUADRATIC_PEAK_THRESHOLD
    branch = "quadratic" if quadratic else "idiv"
    u, tr = ipiano_foe(v, v, model, lam_v, branch, max_iters=iters, rel_tol=rel_tol)
    return {"image": anscombe_inverse_exact_unbiased(u), "branch": f"transform_{branch}", "lam": lam_v,
            "trace": tr, "transformed": u}


# --- scoring (metrics.py:30-102) ---------------------------------------------------------------------

SSIM_WINDOW, SSIM_SIGMA, SSIM_K1, SSIM_K2 = 11, 1.5, 0.01, 0.03


def _ssim_window():
    """metrics.py:41-45: normalised 1-D Gaussian (sigma 1.5), 2-D window = outer product."""
    d = np.arange(SSIM_WINDOW) - (SSIM_WINDOW - 1) / 2
    g = np.exp(-0.5 * (d / SSIM_SIGMA) ** 2)
    g /= g.sum()
    return np.outer(g, g)


def _valid_filter(a, w):
    """Valid-mode correlation with the (symmetric) window: sum_{a,b} w[a,b] x[i+a, j+b]."""
    win = np.lib.stride_tricks.sliding_window_view(a, w.shape)
    return np.einsum("ijab,ab->ij", win, w)


def psnr(x_hat, g, data_range):
    """metrics.py:30-38."""
    mse = float(np.mean((np.asarray(x_hat, float) - np.asarray(g, float)) ** 2))
    return float("inf") if mse == 0.0 else float(10.0 * np.log10(data_range ** 2 / mse))


def mssim(x_hat, g, data_range):
    """metrics.py:51-72: valid-mode local statistics, K1 = 0.01, K2 = 0.03."""
    x, y = np.asarray(x_hat, float), np.asarray(g, float)
    w = _ssim_window()
    ux, uy = _valid_filter(x, w), _valid_filter(y, w)
    vx = _valid_filter(x * x, w) - ux * ux
    vy = _valid_filter(y * y, w) - uy * uy
    vxy = _valid_filter(x * y, w) - ux * uy
    c1, c2 = (SSIM_K1 * data_range) ** 2, (SSIM_K2 * data_range) ** 2
    s = ((2 * ux * uy + c1) * (2 * vxy + c2)) / ((ux ** 2 + uy ** 2 + c1) * (vx + vy + c2))
    return float(s.mean())


def score_denoised(x_hat, g, peak):
    """metrics.py:91-102: both mapped to [0, 255] by 255 / peak, data_range 255 -> (psnr, mssim)."""
    scale = 255.0 / peak
    return psnr(x_hat * scale, g * scale, 255.0), mssim(x_hat * scale, g * scale, 255.0)
