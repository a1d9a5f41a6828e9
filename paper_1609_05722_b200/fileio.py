"""``FOE 1`` model files -- the reference's filter-bank format (fileio.py:33-88).

Line 1 ``FOE 1``; line 2 ``<domain_tag> <n_filters> <m> <basis> <boundary>``;
then one line per filter: the positive weight followed by the m*m-1 basis
coefficients, printed with 17 significant digits so the round trip is
bit-exact (fileio.py:33-48).
"""

from __future__ import annotations

import os

import numpy as np

from .image import basis_by_name
from .prior import DOMAIN_TAGS, FoEModel

MODEL_MAGIC = "FOE 1"
ASSETS = os.path.join(os.path.dirname(os.path.abspath(__file__)), "assets")


class FileFormatError(ValueError):
    """A file does not match its declared format (fileio.py:25-26)."""


def save_model(path, model: FoEModel) -> None:
    nf = model.betas.shape[0]
    lines = [MODEL_MAGIC, f"{model.domain_tag} {nf} {model.basis.size} {model.basis.name} {model.boundary}"]
    for i in range(nf):
        row = [model.weights[i]] + list(model.betas[i])
        lines.append(" ".join(f"{float(v):.17g}" for v in row))
    with open(path, "w") as fh:
        fh.write("\n".join(lines) + "\n")


def load_model(path) -> FoEModel:
    with open(path) as fh:
        lines = [ln.strip() for ln in fh if ln.strip()]
    if not lines or lines[0] != MODEL_MAGIC:
        raise FileFormatError(f"{path}: missing '{MODEL_MAGIC}' header")
    if len(lines) < 2:
        raise FileFormatError(f"{path}: missing header line")
    header = lines[1].split()
    if len(header) != 5:
        raise FileFormatError(f"{path}: header needs 5 fields, got {len(header)}")
    domain_tag, nf_s, m_s, basis_id, boundary = header
    if domain_tag not in DOMAIN_TAGS:
        raise FileFormatError(f"{path}: unknown domain tag {domain_tag!r}")
    try:
        nf, m = int(nf_s), int(m_s)
    except ValueError as exc:
        raise FileFormatError(f"{path}: bad header counts") from exc
    basis = basis_by_name(basis_id)
    if basis.size != m:
        raise FileFormatError(f"{path}: basis {basis_id} has size {basis.size}, header says {m}")
    if len(lines) != 2 + nf:
        raise FileFormatError(f"{path}: expected {nf} filter lines, got {len(lines) - 2}")
    weights = np.empty(nf)
    betas = np.empty((nf, basis.n_atoms))
    for i, line in enumerate(lines[2:]):
        try:
            vals = [float(tok) for tok in line.split()]
        except ValueError as exc:
            raise FileFormatError(f"{path}: filter {i} has a non-numeric token") from exc
        if len(vals) != 1 + basis.n_atoms:
            raise FileFormatError(f"{path}: filter {i} has {len(vals) - 1} coefficients, need {basis.n_atoms}")
        weights[i] = vals[0]
        betas[i] = vals[1:]
    return FoEModel(basis=basis, betas=betas, weights=weights, domain_tag=domain_tag, boundary=boundary)


def load_packaged_model(name: str = "foe_a") -> FoEModel:
    """Packaged banks: foe_a (anscombe, 24x5x5), foe_s (original, 8x3x3), foe_fallback48x7."""
    path = os.path.join(ASSETS, f"{name}.foe")
    if not os.path.isfile(path):
        raise FileFormatError(f"no packaged model named {name!r}")
    return load_model(path)
