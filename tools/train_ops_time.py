"""Device fp64 Hessian-vector product (training.py:158-174) at 256^2 and 512^2 (foe_a)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1609_05722_b200 as fp  # noqa: E402
from paper_1609_05722_b200 import training as tr  # noqa: E402
from paper_1609_05722_b200.synth import make_counts  # noqa: E402

model = fp.load_packaged_model("foe_a")
bank = tr._Bank64(model)
for n in (256, 512):
    x, y = make_counts(n, n, 0, 4.0)
    smp = tr.TrainingSample.create(4.0 * x, y)
    w = tr._dev(smp.transformed)
    p = tr._dev(np.random.default_rng(0).normal(size=(n, n)))
    zw = bank.conv(w)
    for _ in range(3):
        tr._hvp_dev(bank, w, zw, p, smp, "anscombe_domain", 1.0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        tr._hvp_dev(bank, w, zw, p, smp, "anscombe_domain", 1.0)
    e1.record()
    e1.synchronize()
    hvp_ms = e0.elapsed_time(e1) / 20
    print(f"{n}^2: hessian_apply {hvp_ms:.3f} ms/matvec (device, fp64)")
