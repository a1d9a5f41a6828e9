"""Device-timed config-3 solves (512^2, peak 8, direct variant, 60 iterations) with foe_s (3x3, FFMA pass)
and foe_a re-tagged (5x5, tensor-core pass): median of 10 after 3 warm-ups, for A/B of library builds."""
import dataclasses
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1609_05722_b200 as fp  # noqa: E402
from paper_1609_05722_b200.synth import make_counts  # noqa: E402

_, y = make_counts(512, 512, 0, 8.0)
fa = fp.load_packaged_model("foe_a")
for name, model in (("foe_s", fp.load_packaged_model("foe_s")),
                    ("foe_a_original", dataclasses.replace(fa, domain_tag="original"))):
    req = fp.DenoiseRequest(noisy=y, peak=8.0, model=model, variant="direct")
    cfg = fp.SolverConfig(rel_tol=0.0)
    ts = []
    for i in range(13):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        r = fp.denoise(req, cfg)
        e1.record()
        e1.synchronize()
        if i >= 3:
            ts.append(e0.elapsed_time(e1))
    print(f"cfg3 {name}: {np.median(ts):.3f} ms, {len(r.trace)} iterations, {r.trace.n_trials} trials")
