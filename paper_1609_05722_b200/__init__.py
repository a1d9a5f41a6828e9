"""B200-native FoE Poisson-denoise hot path (arXiv 1609.05722), drop-in for foepoisson.denoise.

Public surface mirrors the reference package (pkg/src/foepoisson): ``denoise``,
``DenoiseRequest``, ``DenoiseResult``, ``SolverConfig``, ``SolverTrace``,
``NumericalFailure``, ``FoEModel``, ``load_model`` / ``save_model`` /
``load_packaged_model``.  All numerics run in ``libfoe_b200.so`` (sm_100a).
"""

from .fileio import FileFormatError, load_model, load_packaged_model, save_model
from .image import FilterBasis, basis_by_name, dct_basis
from .pipeline import (DenoiseRequest, DenoiseResult, denoise, denoise_batch, denoise_direct, denoise_transform,
                       select_lambda, solver_budget)
from .prior import FoEModel, foe_energy, foe_gradient
from .solver import NumericalFailure, SolverConfig, SolverTrace, solve_device

__all__ = [
    "DenoiseRequest", "DenoiseResult", "FileFormatError", "FilterBasis", "FoEModel", "NumericalFailure",
    "SolverConfig", "SolverTrace", "basis_by_name", "dct_basis", "denoise", "denoise_batch", "denoise_direct",
    "denoise_transform", "foe_energy", "foe_gradient", "load_model", "load_packaged_model", "save_model",
    "select_lambda", "solve_device", "solver_budget",
]
