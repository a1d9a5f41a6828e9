"""Reference outputs for the device CG's restart and free-set paths (training.py:183-237).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_cg.py

Two small cases run through the REFERENCE's own solve_hessian_system / hessian_apply:
  * "brk": original-domain objective with a rough iterate -- every CG attempt meets non-positive
    curvature, so all six restarts with escalating eps run (the regularisation path);
  * "free": anscombe-domain objective with a random free set (the pinned-pixel identity).
"""
from __future__ import annotations

import os
import sys
import warnings

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)
from foepoisson import fileio, training  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    out = {}
    rng = np.random.default_rng(5)
    H = W = 40
    clean = rng.uniform(0.5, 3, (H, W))
    noisy = rng.poisson(clean).astype(float)
    smp = training.TrainingSample.create(clean, noisy)
    rhs = rng.standard_normal((H, W))
    w = np.abs(clean + 1.0 * rng.standard_normal((H, W))) + 0.05
    fs = fileio.load_packaged_model("foe_s")
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        q, info = training.solve_hessian_system(w, fs, "original_domain", rhs, smp, lam=0.1, tol=1e-9, max_iters=80)
    out.update(cg_clean=clean, cg_noisy=noisy, cg_rhs=rhs, brk_w=w, brk_q=q, brk_iters=info["iterations"],
               brk_reg=info["regularization"], brk_res=np.array(info["residuals"]),
               brk_hp=training.hessian_apply(w, fs, "original_domain", rhs, smp, lam=0.1))
    print("brk", info["iterations"], info["regularization"], len(info["residuals"]))
    fa = fileio.load_packaged_model("foe_a")
    wa = smp.transformed + 0.3 * rng.standard_normal((H, W))
    free = rng.random((H, W)) < 0.8
    q, info = training.solve_hessian_system(wa, fa, "anscombe_domain", rhs, smp, lam=1.0, tol=1e-9, max_iters=600,
                                            free=free)
    out.update(free_w=wa, free_mask=free, free_q=q, free_iters=info["iterations"], free_reg=info["regularization"],
               free_res=np.array(info["residuals"]))
    print("free", info["iterations"], info["regularization"])
    np.savez_compressed(os.path.join(HERE, "cg.npz"), **out)


if __name__ == "__main__":
    main()
