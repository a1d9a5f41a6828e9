"""Host-side phases of one end-to-end fp.denoise call (512^2 cfg2): request validation, upload, solve,
inverse + download -- where the e2e time beyond the device solve goes."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1609_05722_b200 as fp  # noqa: E402
from paper_1609_05722_b200 import pipeline  # noqa: E402
from paper_1609_05722_b200._host import download, upload  # noqa: E402
from paper_1609_05722_b200.anscombe import forward_device, inverse_exact_unbiased_device  # noqa: E402
from paper_1609_05722_b200.synth import make_counts  # noqa: E402

model = fp.load_packaged_model("foe_a")
_, y = make_counts(512, 512, 0, 1.0)
cfg = fp.SolverConfig(rel_tol=0.0)
T = {}
for rep in range(6):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    req = fp.DenoiseRequest(noisy=y, peak=1.0, model=model, variant="transform", force_branch="quadratic")
    t1 = time.perf_counter()
    v = forward_device(upload(req.noisy))
    t2 = time.perf_counter()
    res = fp.solve_device(model, v, v, 0.6075, "quadratic", 150, cfg)
    t3 = time.perf_counter()
    x = inverse_exact_unbiased_device(res.u)
    image, u = download(x, res.u.to(torch.float64))
    t4 = time.perf_counter()
    r = fp.denoise(req, cfg)
    t5 = time.perf_counter()
    if rep >= 2:
        for k, d in (("request", t1 - t0), ("upload+anscombe", t2 - t1), ("solve_device", t3 - t2),
                     ("inverse+download", t4 - t3), ("fp.denoise total", t5 - t4)):
            T.setdefault(k, []).append(d * 1e3)
for k, v in T.items():
    print(f"{k:20s} {np.median(v):7.3f} ms")
