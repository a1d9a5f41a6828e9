"""Training-side operators on the device (training.py:158-237), foe_a at 256^2 and 512^2:
the fused fp64 Hessian-vector product (foe_hessian_apply64, CUDA events over 20 back-to-back calls),
the same product composed from the bank kernels (conv -> rho'' weighting -> adjoint, the round-1 path),
and one device-resident CG solve (foe_cg_solve64) with its iteration count and time per iteration."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1609_05722_b200 as fp  # noqa: E402
from paper_1609_05722_b200 import training as tr  # noqa: E402
from paper_1609_05722_b200.synth import make_counts  # noqa: E402


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


model = fp.load_packaged_model("foe_a")
bank = tr._Bank64(model)
out = {}
for n in (256, 512):
    x, y = make_counts(n, n, 0, 4.0)
    smp = tr.TrainingSample.create(4.0 * x, y)
    w = tr._dev(smp.transformed)
    p = tr._dev(np.random.default_rng(0).normal(size=(n, n)))
    fused = timed(lambda: tr._hvp_fused(bank, w, p, "anscombe_domain", 1.0))
    zw = bank.conv(w)
    composed = timed(lambda: bank.adjoint(bank.weights[None, :, None, None] * tr._rho2(zw) * bank.conv(p))[0] + p)
    rhs = np.random.default_rng(1).normal(size=(n, n))
    yy, xx = np.mgrid[0:n, 0:n]
    wn = 3.0 + 0.5 * np.sin(xx / 40.0) * np.cos(yy / 50.0)  # smooth iterate: rho'' > 0, a positive definite system
    tr.solve_hessian_system(wn, model, "anscombe_domain", rhs, smp, 1.0, tol=1e-9, max_iters=600)  # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    q, info = tr.solve_hessian_system(wn, model, "anscombe_domain", rhs, smp, 1.0, tol=1e-9, max_iters=600)
    cg_s = time.perf_counter() - t0
    out[f"{n}x{n}"] = {"hvp_fused_ms": fused, "hvp_composed_ms": composed, "cg_iterations": info["iterations"],
                       "cg_wall_ms": cg_s * 1e3, "cg_ms_per_iteration": cg_s * 1e3 / max(info["iterations"], 1),
                       "cg_final_residual": info["residuals"][-1]}
    print(n, out[f"{n}x{n}"], flush=True)
print(json.dumps(out))
