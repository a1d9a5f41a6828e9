"""Build and load ``libfoe_b200.so`` (the sm_100a CUDA library behind ``include/foe_b200.h``).

There is no CPU fallback: every operator of this package runs through this
library, and loading it fails loudly when it has not been built.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(PKG)
SRC = os.path.join(PKG, "csrc", "foe_b200.cu")
INCLUDE = os.path.join(REPO, "include")
LIB_PATH = os.path.join(PKG, "libfoe_b200.so")
# diagnostic builds (e.g. -DFOE_STAMPS=1, built by tools/build_diag.py) load through FOE_LIB
LOAD_PATH = os.environ.get("FOE_LIB", LIB_PATH)

# host code (count validation, band geometry, descriptor setup) for x86-64-v3 (AVX2), as the oracle: the GPU
# boxes' hosts support it
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC,-march=x86-64-v3", "-shared"]

FOE_OK, FOE_E_INVALID, FOE_E_CUDA, FOE_E_NUMERICAL, FOE_E_UNSUPPORTED = 0, -1, -2, -3, -4


def _sources():
    d = os.path.join(PKG, "csrc")
    return [os.path.join(d, f) for f in sorted(os.listdir(d)) if f.endswith((".cu", ".cuh", ".h"))] + \
        [os.path.join(INCLUDE, f) for f in sorted(os.listdir(INCLUDE))]


def needs_build() -> bool:
    if not os.path.exists(LIB_PATH):
        return True
    t = os.path.getmtime(LIB_PATH)
    return any(os.path.getmtime(s) > t for s in _sources())


def build(force: bool = False, verbose: bool = False, out: str = LIB_PATH, defines: tuple = ()) -> str:
    """nvcc -gencode arch=compute_100a,code=sm_100a ... -> libfoe_b200.so (no GPU needed)."""
    if out == LIB_PATH and not force and not needs_build():
        return LIB_PATH
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    cmd = [nvcc, *NVCC_FLAGS, *("-D" + d for d in defines), "-I" + INCLUDE, "-o", out + ".tmp", SRC]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + res.stderr[-4000:])
    os.replace(out + ".tmp", out)
    if verbose:
        print(res.stderr)
    return out


class FoeError(RuntimeError):
    pass


_lib = None

_vp = ctypes.c_void_p
_i64 = ctypes.c_int64


class SolverCfgC(ctypes.Structure):
    _fields_ = [("gamma", ctypes.c_double), ("lipschitz_init", ctypes.c_double),
                ("backtrack_factor", ctypes.c_double), ("relax_factor", ctypes.c_double),
                ("rel_tol", ctypes.c_double), ("max_lipschitz", ctypes.c_double)]


class ImageStatusC(ctypes.Structure):
    _fields_ = [("status", ctypes.c_int), ("n_iters", ctypes.c_int), ("n_trials", ctypes.c_int),
                ("failed_at", ctypes.c_int)]


def lib():
    """The loaded CUDA library; raises if it is missing (no fallback path exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LOAD_PATH):
        raise FoeError(f"{LOAD_PATH} is not built; run paper_1609_05722_b200._lib.build() "
                       "(or __graft_entry__.build()) -- there is no CPU fallback")
    L = ctypes.CDLL(LOAD_PATH)
    L.foe_last_error.restype = ctypes.c_char_p
    L.foe_abi_version.restype = ctypes.c_int
    L.foe_device_sm_count.argtypes = [ctypes.c_int]
    L.foe_counts_check.argtypes = [_vp, ctypes.c_size_t]
    L.foe_counts_check_stage.argtypes = [_vp, ctypes.c_size_t, _vp]
    L.foe_kernel_launch_count.restype = ctypes.c_longlong
    L.foe_bank_create.argtypes = [_vp, _vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(_vp)]
    L.foe_bank_destroy.argtypes = [_vp]
    L.foe_bank_info.argtypes = [_vp, _vp, _vp, _vp]
    L.foe_anscombe_forward.argtypes = [_vp, _vp, _i64, _vp]
    L.foe_anscombe_forward_f32.argtypes = [_vp, _vp, _i64, _vp]
    L.foe_direct_obs.argtypes = [_vp, _vp, ctypes.c_double, _i64, _vp]
    L.foe_anscombe_inverse_exact_unbiased.argtypes = [_vp, _vp, _i64, _vp, _vp]
    L.foe_prox_quadratic.argtypes = [_vp, _vp, _vp, ctypes.c_double, _i64, _vp]
    L.foe_prox_idiv.argtypes = [_vp, _vp, _vp, ctypes.c_double, _i64, _vp]
    L.foe_bin.argtypes = [_vp, _vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, _vp]
    L.foe_unbin_bilinear.argtypes = [_vp, _vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                     _vp]
    L.foe_estimate_peak.argtypes = [_vp, ctypes.c_int, ctypes.c_int, _vp, _vp, _vp]
    L.foe_convolve_same.argtypes = [_vp, ctypes.c_int, _vp, _vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, _vp]
    L.foe_convolve_adjoint.argtypes = L.foe_convolve_same.argtypes
    L.foe_eval_workspace_size.argtypes = [_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int]
    L.foe_eval_workspace_size.restype = ctypes.c_size_t
    L.foe_energy_grad.argtypes = [_vp, _vp, _vp, _vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, _vp,
                                  ctypes.c_size_t, _vp]
    L.foe_solve_workspace_size.argtypes = [_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int]
    L.foe_solve_workspace_size.restype = ctypes.c_size_t
    L.foe_solve.argtypes = [_vp, ctypes.POINTER(SolverCfgC), ctypes.c_int, ctypes.c_int, ctypes.c_int, _vp, _vp,
                            _vp, _vp, _vp, _vp, _vp, _vp, ctypes.c_int, _vp, ctypes.c_size_t, _vp]
    L.foe_bench_trial_pass.argtypes = [_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                       _vp, ctypes.c_size_t, _vp]
    L.foe_tc_selftest.argtypes = [_vp, _vp, _vp, _vp]
    L.foe_pass_uses_tensor_cores.argtypes = [ctypes.c_int, ctypes.c_int]
    L.foe_measure_ffma_peak.argtypes = [ctypes.c_int, _vp, ctypes.POINTER(ctypes.c_double), _vp]
    for fn in (L.foe_conv_bank64, L.foe_adjoint_bank64):
        fn.argtypes = [_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, _vp, _vp, ctypes.c_int, ctypes.c_int,
                       ctypes.c_int, _vp]
    L.foe_hessian_apply64.argtypes = [_vp, _vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                      _vp, _vp, _vp, _vp, ctypes.c_double, _vp, ctypes.c_int, ctypes.c_int, _vp]
    L.foe_cg_workspace_size.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int]
    L.foe_cg_workspace_size.restype = ctypes.c_size_t
    L.foe_cg_solve64.argtypes = [_vp, _vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                 _vp, _vp, _vp, _vp, ctypes.c_double, ctypes.c_double, ctypes.c_int, _vp,
                                 ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int), _vp, ctypes.c_int,
                                 ctypes.c_int, _vp, ctypes.c_size_t, _vp]
    L.foe_score_workspace_size.argtypes = [ctypes.c_int] * 3
    L.foe_score_workspace_size.restype = ctypes.c_size_t
    L.foe_score.argtypes = [_vp, _vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double, _vp, _vp, _vp,
                            ctypes.c_size_t, _vp]
    L.foe_debug_tc_rate.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, _vp, _vp]
    L.foe_debug_tmem_rate.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, _vp, _vp]
    L.foe_debug_pass_times.argtypes = [_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, _vp,
                                       ctypes.c_size_t, _vp, _vp]
    _lib = L
    return L


def check(rc: int, what: str = "") -> int:
    if rc == FOE_OK:
        return rc
    msg = lib().foe_last_error().decode(errors="replace")
    if rc == FOE_E_INVALID:
        raise ValueError(f"{what}: {msg}" if what else msg)
    raise FoeError(f"{what} failed ({rc}): {msg}")


EXPORTED_SYMBOLS = [
    "foe_abi_version", "foe_last_error", "foe_device_sm_count", "foe_counts_check", "foe_counts_check_stage", "foe_kernel_launch_count", "foe_bank_create", "foe_bank_destroy",
    "foe_bank_info", "foe_anscombe_forward", "foe_anscombe_forward_f32", "foe_direct_obs", "foe_anscombe_inverse_exact_unbiased",
    "foe_prox_quadratic", "foe_prox_idiv", "foe_bin", "foe_unbin_bilinear", "foe_estimate_peak", "foe_convolve_same", "foe_convolve_adjoint",
    "foe_eval_workspace_size", "foe_energy_grad", "foe_solve_workspace_size", "foe_solve",
    "foe_bench_trial_pass", "foe_debug_pass_times", "foe_tc_selftest", "foe_pass_uses_tensor_cores",
    "foe_debug_tc_rate", "foe_debug_tmem_rate", "foe_measure_ffma_peak", "foe_debug_pass_times_seq", "foe_score_workspace_size", "foe_score",
    "foe_conv_bank64", "foe_adjoint_bank64", "foe_hessian_apply64", "foe_cg_workspace_size", "foe_cg_solve64", "foe_tile_grid", "foe_band_geometry", "foe_band_describe", "foe_band_workspace_size",
    "foe_band_buffers_get", "foe_band_begin", "foe_band_trial", "foe_band_commit", "foe_band_final_pass", "foe_band_end",
]
