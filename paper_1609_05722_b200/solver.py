"""iPiano with backtracking (reference: solver.py), executed entirely on the device.

The reference runs the loop on the host with numpy callbacks
(``ipiano_minimize(grad_F, energy_F, prox_G, energy_G, u0, cfg)``,
solver.py:128-175).  Here the FoE instance of that loop -- the only one the
denoise path uses (pipeline.py:167-172, 205-208) -- runs on the GPU: one fused
pass kernel per trial step, accept/reject decisions taken by the device, and the
host only polls a live-image counter every few passes.  ``SolverConfig``,
``SolverTrace`` and ``NumericalFailure`` keep the reference's fields and
semantics.
"""

from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass, field

import numpy as np

from . import _lib

_SLACK_RTOL = 1e-12  # solver.py:23 (applied on the device)

BRANCH_CODES = {"quadratic": 0, "idiv": 1}


class NumericalFailure(RuntimeError):
    """Solver abort (non-finite energy or hopeless backtracking); carries the trace (solver.py:26-31)."""

    def __init__(self, message, trace=None):
        super().__init__(message)
        self.trace = trace


@dataclass
class SolverConfig:
    """Step-size and stopping constants (solver.py:34-65)."""

    gamma: float = 0.8
    lipschitz_init: float = 1.0
    backtrack_factor: float = 1.2
    relax_factor: float = 1.05
    max_iters: int = 150
    rel_tol: float = 1e-6
    max_lipschitz: float = 1e15

    def __post_init__(self):
        if not 0.0 <= self.gamma < 1.0:
            raise ValueError(f"gamma must be in [0, 1), got {self.gamma}")
        if not self.lipschitz_init > 0:
            raise ValueError(f"lipschitz_init must be positive, got {self.lipschitz_init}")
        if not self.backtrack_factor > 1:
            raise ValueError(f"backtrack_factor must exceed 1, got {self.backtrack_factor}")
        if self.max_iters < 1:
            raise ValueError("max_iters must be at least 1")

    def step_size(self, lipschitz: float) -> float:
        return 1.99 * (1.0 - self.gamma) / lipschitz

    def to_c(self) -> _lib.SolverCfgC:
        return _lib.SolverCfgC(self.gamma, self.lipschitz_init, self.backtrack_factor, self.relax_factor,
                               self.rel_tol, self.max_lipschitz)


@dataclass
class SolverTrace:
    """Per accepted iteration: energies, curvature estimate, step norm, slack (solver.py:68-89)."""

    iteration: list = field(default_factory=list)
    F: list = field(default_factory=list)
    G: list = field(default_factory=list)
    L: list = field(default_factory=list)
    step_norm: list = field(default_factory=list)
    descent_slack: list = field(default_factory=list)
    slack_tol: list = field(default_factory=list)
    n_trials: int = 0  # energy evaluations of trial points (device counter; not in the reference)

    def __len__(self):
        return len(self.iteration)

    def save_csv(self, path) -> None:
        with open(path, "w") as fh:
            fh.write("iteration,F,G,L,step_norm\n")
            for row in zip(self.iteration, self.F, self.G, self.L, self.step_norm):
                fh.write("%d,%.17g,%.17g,%.17g,%.17g\n" % row)

    @classmethod
    def from_rows(cls, rows: np.ndarray, n_trials: int = 0) -> "SolverTrace":
        n = rows.shape[0]
        return cls(iteration=list(range(n)), F=rows[:, 0].tolist(), G=rows[:, 1].tolist(),
                   L=rows[:, 2].tolist(), step_norm=rows[:, 3].tolist(), descent_slack=rows[:, 4].tolist(),
                   slack_tol=rows[:, 5].tolist(), n_trials=n_trials)


def _stream():
    import torch
    return torch.cuda.current_stream().cuda_stream


def prox_quadratic(u_tilde, t: float, v):
    """argmin_u 1/2|u - u~|^2 + t/2 |u - v|^2 = (u~ + t v)/(1 + t)  (solver.py:92-100), fp32 GPU."""
    import torch
    if t < 0:
        raise ValueError(f"t must be >= 0, got {t}")
    a = np.asarray(u_tilde, dtype=np.float64)
    b = np.asarray(v, dtype=np.float64)
    if a.shape != b.shape:
        raise ValueError(f"shape mismatch {a.shape} vs {b.shape}")
    ad = torch.from_numpy(np.ascontiguousarray(a)).to("cuda", torch.float32)
    bd = torch.from_numpy(np.ascontiguousarray(b)).to("cuda", torch.float32)
    out = torch.empty_like(ad)
    _lib.check(_lib.lib().foe_prox_quadratic(ad.data_ptr(), bd.data_ptr(), out.data_ptr(), float(t), ad.numel(),
                                             _stream()), "prox_quadratic")
    return out.double().cpu().numpy()


def prox_idiv(u_tilde, t: float, obs):
    """argmin_u 1/2|u - u~|^2 + t (u - obs log u)  (solver.py:103-125), fp32 GPU."""
    import torch
    if t < 0:
        raise ValueError(f"t must be >= 0, got {t}")
    a = np.asarray(u_tilde, dtype=np.float64)
    b = np.asarray(obs, dtype=np.float64)
    if a.shape != b.shape:
        raise ValueError(f"shape mismatch {a.shape} vs {b.shape}")
    if b.size and b.min() < 0:
        raise ValueError("observed counts must be >= 0")
    ad = torch.from_numpy(np.ascontiguousarray(a)).to("cuda", torch.float32)
    bd = torch.from_numpy(np.ascontiguousarray(b)).to("cuda", torch.float32)
    out = torch.empty_like(ad)
    _lib.check(_lib.lib().foe_prox_idiv(ad.data_ptr(), bd.data_ptr(), out.data_ptr(), float(t), ad.numel(),
                                        _stream()), "prox_idiv")
    return out.double().cpu().numpy()


@dataclass
class DeviceSolveResult:
    u: object                # (B,H,W) fp32 CUDA tensor
    traces: list             # SolverTrace per image
    status: list             # foe_solve_status per image (0 ok, 1 non-finite, 2 stalled)
    failed_at: list


_tls = threading.local()


def _workspace(nbytes: int, device):
    """Per-thread cached solve workspace: stable device pointers keep the captured solve-loop graph
    (keyed by the pass arguments, hence by the workspace address) valid across calls."""
    import torch
    cache = getattr(_tls, "ws", None)
    if cache is None:
        cache = _tls.ws = {}
    key = (str(device), nbytes)
    ws = cache.get(key)
    if ws is None:
        if len(cache) >= 4:
            cache.clear()
        ws = cache[key] = torch.empty(nbytes, dtype=torch.uint8, device=device)
    return ws


def solve_device(model, u0, obs, lam, branch, max_iters, cfg: SolverConfig | None = None,
                 raise_on_failure: bool = True) -> DeviceSolveResult:
    """Device-resident iPiano over the FoE energy for a batch (B,H,W) of fp32 CUDA tensors.

    lam, branch ("quadratic"/"idiv" or 0/1) and max_iters are scalars or length-B sequences.
    Replaces ipiano_minimize with the FoE callbacks (solver.py:128-175, pipeline.py:167-172, 205-208).
    """
    import torch

    from .prior import device_bank

    cfg = cfg or SolverConfig()
    squeeze = u0.dim() == 2
    u0 = (u0[None] if squeeze else u0).to(torch.float32).contiguous()
    obs = (obs[None] if obs.dim() == 2 else obs).to(torch.float32).contiguous()
    B, H, W = u0.shape
    if obs.shape != u0.shape:
        raise ValueError(f"shape mismatch {tuple(obs.shape)} vs {tuple(u0.shape)}")

    def per_image(x, dtype):
        arr = np.broadcast_to(np.asarray(x, dtype=dtype), (B,))
        return np.ascontiguousarray(arr)

    if isinstance(branch, str) or (np.ndim(branch) and isinstance(np.asarray(branch).flat[0], str)):
        branch = [BRANCH_CODES[b] for b in np.broadcast_to(np.asarray(branch), (B,))]
    lam_a = per_image(lam, np.float64)
    br_a = per_image(branch, np.int32)
    it_a = per_image(max_iters, np.int32)
    cap = int(it_a.max())
    bank = device_bank(model)
    L = _lib.lib()
    ws_bytes = L.foe_solve_workspace_size(bank.handle, B, H, W, cap)
    ws = _workspace(ws_bytes, u0.device)
    u_out = torch.empty_like(u0)
    status = (_lib.ImageStatusC * B)()
    trace = np.zeros((B, cap, 6))
    c = cfg.to_c()
    rc = L.foe_solve(bank.handle, ctypes.byref(c), B, H, W, u0.data_ptr(), obs.data_ptr(),
                     lam_a.ctypes.data, br_a.ctypes.data, it_a.ctypes.data, u_out.data_ptr(),
                     ctypes.cast(status, ctypes.c_void_p), trace.ctypes.data, cap, ws.data_ptr(), ws_bytes,
                     _stream())
    if rc not in (_lib.FOE_OK, _lib.FOE_E_NUMERICAL) or (rc == _lib.FOE_E_NUMERICAL and not any(
            status[b].status for b in range(B))):
        _lib.check(rc, "foe_solve")
    traces = [SolverTrace.from_rows(trace[b, :status[b].n_iters], status[b].n_trials) for b in range(B)]
    st = [status[b].status for b in range(B)]
    fa = [status[b].failed_at for b in range(B)]
    if raise_on_failure:
        for b in range(B):
            if st[b] == 1:
                raise NumericalFailure(f"non-finite smooth energy at iteration {fa[b]}", traces[b])
            if st[b] == 2:
                raise NumericalFailure(f"backtracking stalled at iteration {fa[b]}", traces[b])
    res = DeviceSolveResult(u=u_out[0] if squeeze else u_out, traces=traces, status=st, failed_at=fa)
    res._workspace = ws  # keep for foe_bench_trial_pass
    res._bank = bank
    res._cap = cap
    return res
