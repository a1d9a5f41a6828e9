"""Seeded synthetic inputs standing in for the reference's scikit-image eval set.

The reference benchmarks on images derived from scikit-image sample data
(data.py:17-26), which is absent here, so BASELINE.md section 4 freezes a
synthetic generator instead.  Parameters (all relative to the canvas):

* 20 axis-aligned rectangles: top-left uniform over the canvas, sides
  U[H/16, H/3] x U[W/16, W/3]; then 20 disks: centre uniform, radius
  U[min(H,W)/32, min(H,W)/8].  Each shape is painted over the previous ones with
  intensity U[0, 1].
* A low-frequency cosine ramp: amplitude 0.2, 0.5-1.5 cycles per image along
  each axis, random phase.
* 1/f noise: complex Gaussian spectrum divided by |f|, DC removed, real part,
  normalised to max-abs 1, times 0.05.
* Clip to [0, 1].

Noisy counts are ``sample_poisson(peak * x, seed)``: a Philox-keyed numpy
Poisson draw, restating the reference's noise.py:41-52 so both the GPU path
and the CPU oracle see identical counts.
"""

from __future__ import annotations

import numpy as np


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(key=int(seed)))


def synthetic_clean(H: int, W: int, seed: int) -> np.ndarray:
    """Clean image in [0, 1] of shape (H, W), deterministic in ``seed``."""
    rng = _rng(seed)
    x = np.zeros((H, W))
    for _ in range(20):
        y0 = rng.uniform(0, H)
        x0 = rng.uniform(0, W)
        h = rng.uniform(H / 16, H / 3)
        w = rng.uniform(W / 16, W / 3)
        val = rng.uniform(0.0, 1.0)
        r0, r1 = int(np.ceil(y0)), int(min(H, np.ceil(y0 + h)))
        c0, c1 = int(np.ceil(x0)), int(min(W, np.ceil(x0 + w)))
        x[r0:r1, c0:c1] = val
    lo, hi = min(H, W) / 32, min(H, W) / 8
    for _ in range(20):
        cy = rng.uniform(0, H)
        cx = rng.uniform(0, W)
        rad = rng.uniform(lo, hi)
        val = rng.uniform(0.0, 1.0)
        r0, r1 = max(0, int(cy - rad)), min(H, int(cy + rad) + 2)
        c0, c1 = max(0, int(cx - rad)), min(W, int(cx + rad) + 2)
        yy = np.arange(r0, r1)[:, None]
        xx = np.arange(c0, c1)[None, :]
        mask = (yy - cy) ** 2 + (xx - cx) ** 2 <= rad * rad
        x[r0:r1, c0:c1][mask] = val
    fy = rng.uniform(0.5, 1.5)
    fx = rng.uniform(0.5, 1.5)
    phase = rng.uniform(0.0, 2 * np.pi)
    ramp_y = 2 * np.pi * fy * np.arange(H)[:, None] / H
    ramp_x = 2 * np.pi * fx * np.arange(W)[None, :] / W
    x += 0.2 * np.cos(ramp_y + ramp_x + phase)
    spec = rng.standard_normal((H, W)) + 1j * rng.standard_normal((H, W))
    ky = np.fft.fftfreq(H)[:, None]
    kx = np.fft.fftfreq(W)[None, :]
    mag = np.sqrt(ky * ky + kx * kx)
    mag[0, 0] = 1.0
    spec /= mag
    spec[0, 0] = 0.0
    noise = np.real(np.fft.ifft2(spec))
    top = np.max(np.abs(noise))
    if top > 0:
        x += 0.05 * noise / top
    return np.clip(x, 0.0, 1.0)


def sample_poisson(img: np.ndarray, seed: int) -> np.ndarray:
    """y ~ Poisson(img) per pixel from a Philox(key=seed) stream (noise.py:41-52)."""
    img = np.asarray(img, dtype=np.float64)
    if img.min() < 0:
        raise ValueError("Poisson intensities must be nonnegative")
    return _rng(seed).poisson(img).astype(np.float64)


def make_counts(H: int, W: int, seed: int, peak: float):
    """(clean x, noisy counts y = Poisson(peak * x)) for one synthetic job."""
    x = synthetic_clean(H, W, seed)
    return x, sample_poisson(peak * x, seed)


def config_peak(cfg: int, seed: int = 0) -> float:
    """Peak of BASELINE.json config ``cfg`` (1-based); cfg 4 cycles {0.5,1,2,4}."""
    return {1: 4.0, 2: 1.0, 3: 8.0, 5: 2.0}.get(cfg, [0.5, 1.0, 2.0, 4.0][seed % 4])
