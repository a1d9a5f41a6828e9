"""Evaluation grid on the device: noise, denoise and score a grid of (image, peak, variant) jobs.

Mirrors the reference's benchmark runner (benchmark.py:32-122): the
same spec / row types, the same hash-derived per-job seeds (so results do not depend on order or
worker count) and the same row order and CSV format.  Instead of one ``denoise`` per job on a
thread pool, jobs that share a variant, image shape and peak are solved as ONE batched
device-resident solve (``denoise_batch``: per-image lambda / branch / budget / backtracking, results
equal to separate calls), scored on the device (``metrics.score_batch``), and the job list is
sharded over torch.distributed ranks when a process group is up (rows are all-gathered).
"""
from __future__ import annotations

import hashlib
import re
from collections import defaultdict
from dataclasses import dataclass

import numpy as np

from .pipeline import AUTO_LAMBDA, VARIANTS, DenoiseRequest, denoise, denoise_batch
from .prior import FoEModel
from .synth import sample_poisson, synthetic_clean


@dataclass(frozen=True)
class BenchmarkSpec:
    """A grid of evaluation jobs plus the models that serve them (benchmark.py:32-54)."""

    images: tuple
    peaks: tuple
    variants: tuple
    transform_model: FoEModel | None = None
    direct_model: FoEModel | None = None
    base_seed: int = 0
    lam: object = AUTO_LAMBDA

    def __post_init__(self):
        if not self.images or not self.peaks or not self.variants:
            raise ValueError("images, peaks, and variants must be non-empty")
        for v in self.variants:
            if v not in VARIANTS:
                raise ValueError(f"unknown variant {v!r}")
        if any(p <= 0 for p in self.peaks):
            raise ValueError("peaks must be positive")
        if self.direct_model is None and "direct" in self.variants:
            raise ValueError("direct variant listed but no direct_model given")
        if self.transform_model is None and set(self.variants) - {"direct"}:
            raise ValueError("transform variants listed but no transform_model given")


@dataclass(frozen=True)
class BenchmarkRow:
    image: str
    peak: float
    variant: str
    psnr_db: float
    mssim: float
    branch: str
    lam: float
    seed: int


def job_seed(image: str, peak: float, variant: str, base_seed: int) -> int:
    """Deterministic per-job seed from the job key; order-independent (benchmark.py:67-70)."""
    key = f"{image}|{peak!r}|{variant}|{base_seed}".encode()
    return int.from_bytes(hashlib.sha256(key).digest()[:8], "big")


def scale_to_peak(img: np.ndarray, peak: float) -> np.ndarray:
    """Rescale so the maximum pixel equals ``peak`` (noise.py:30-38)."""
    img = np.asarray(img, dtype=np.float64)
    top = img.max()
    if not peak > 0:
        raise ValueError(f"peak must be positive, got {peak}")
    if not top > 0:
        raise ValueError("image needs at least one strictly positive pixel")
    return img * (peak / top)


_SYN = re.compile(r"^syn(\d+)x(\d+)s(\d+)$")


def synthetic_eval_image(name: str) -> np.ndarray:
    """Clean image for a job name ``syn{H}x{W}s{seed}`` (the BASELINE.md synthetic generator).

    The reference's roster (``data.load_eval_image``: scikit-image samples) is not available here;
    synthetic images of the same kind stand in for it."""
    m = _SYN.match(name)
    if not m:
        raise ValueError(f"unknown evaluation image {name!r} (expected syn<H>x<W>s<seed>)")
    H, W, seed = (int(g) for g in m.groups())
    return synthetic_clean(H, W, seed)


def _model_for(spec: BenchmarkSpec, variant: str) -> FoEModel:
    return spec.direct_model if variant == "direct" else spec.transform_model


def _dist():
    try:
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            return dist
    except Exception:  # pragma: no cover - torch without distributed
        pass
    return None


def run_benchmark(spec: BenchmarkSpec, image_loader=synthetic_eval_image, workers: int | None = None,
                  progress=None, solver=None) -> list[BenchmarkRow]:
    """All jobs in the grid; the row order is fixed by sorting on the job key (benchmark.py:99-120).

    ``workers`` is accepted for signature compatibility; parallelism comes from batching on the
    device and from the torch.distributed ranks, not from host threads."""
    from .metrics import score_batch

    clean = {name: image_loader(name) for name in spec.images}
    jobs = [(name, peak, variant) for name in spec.images for peak in spec.peaks for variant in spec.variants]
    dist = _dist()
    rank, world = (dist.get_rank(), dist.get_world_size()) if dist else (0, 1)
    mine = jobs[rank::world]

    # group jobs that can share one batched solve and one scoring launch
    groups = defaultdict(list)
    for name, peak, variant in mine:
        groups[(variant, clean[name].shape, peak)].append(name)
    rows = []
    for (variant, shape, peak), names in groups.items():
        seeds = [job_seed(n, peak, variant, spec.base_seed) for n in names]
        scaled = [scale_to_peak(clean[n], peak) for n in names]
        noisy = np.stack([sample_poisson(s, sd) for s, sd in zip(scaled, seeds)])
        model = _model_for(spec, variant)
        if variant == "transform_binned":  # small binned solves, one call each
            outs = [denoise(DenoiseRequest(noisy=y, peak=peak, model=model, variant=variant, lam=spec.lam), solver)
                    for y in noisy]
            images = np.stack([o.image for o in outs])
            lams, branches = [o.lam for o in outs], [o.branch for o in outs]
        else:
            for y in noisy:  # the reference's request validation, per job
                DenoiseRequest(noisy=y, peak=peak, model=model, variant=variant, lam=spec.lam)
            images, _, lams, branches = denoise_batch(noisy, peak, model, variant, lam=spec.lam, solver=solver,
                                                      return_device=True)
            branches = ["direct_idiv" if variant == "direct" else f"transform_{b}" for b in branches]
        ps, ms = score_batch(images, np.stack(scaled), peak)
        for n, sd, p, m, br, lam in zip(names, seeds, ps, ms, branches, lams):
            row = BenchmarkRow(image=n, peak=peak, variant=variant, psnr_db=float(p), mssim=float(m), branch=br,
                               lam=float(lam), seed=sd)
            rows.append(row)
            if progress is not None:
                progress(row)
    if dist and world > 1:
        gathered = [None] * world
        dist.all_gather_object(gathered, rows)
        rows = [r for part in gathered for r in part]
    return sorted(rows, key=lambda r: (r.peak, r.image, r.variant))


def average_rows(rows: list[BenchmarkRow]) -> list[BenchmarkRow]:
    """Per (peak, variant) averages, reported under the image name 'average' (benchmark.py:125-137)."""
    groups: dict = {}
    for r in rows:
        groups.setdefault((r.peak, r.variant), []).append(r)
    out = []
    for (peak, variant), rs in sorted(groups.items()):
        out.append(BenchmarkRow(image="average", peak=peak, variant=variant,
                                psnr_db=float(np.mean([r.psnr_db for r in rs])),
                                mssim=float(np.mean([r.mssim for r in rs])), branch=rs[0].branch, lam=rs[0].lam,
                                seed=0))
    return out


def format_csv_report(rows: list[BenchmarkRow]) -> str:
    """Full-precision CSV, byte-stable for identical inputs (benchmark.py:150-156)."""
    out = ["image,peak,variant,psnr_db,mssim,branch,lambda,seed"]
    for r in rows:
        out.append(f"{r.image},{r.peak:.17g},{r.variant},{r.psnr_db:.17g},"
                   f"{r.mssim:.17g},{r.branch},{r.lam:.17g},{r.seed}")
    return "\n".join(out) + "\n"
