"""Per-iteration gradient rel-L2 of both pass kernels vs the oracle (the north_star 1e-5 gate)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1609_05722_b200 as fp  # noqa: E402
from oracle import cpu as orc  # noqa: E402
from paper_1609_05722_b200.synth import make_counts  # noqa: E402

orc.build()
model = fp.load_packaged_model("foe_a")
om = orc.OracleModel(filters=model.filters, weights=model.weights, boundary=model.boundary,
                     domain_tag=model.domain_tag)
_, y = make_counts(256, 256, 0, 4.0)
v = orc.anscombe_forward(y)
TABLE = orc.load_lambda_table(os.path.join(os.path.dirname(fp.__file__), "assets", "lambda_table.json"))
lam = orc.select_lambda(4.0, "transform", TABLE, "quadratic")
for kernel in ("0", "1"):
    os.environ["FOE_TC"] = kernel
    worst = []
    for k in (1, 3, 10, 40, 150):
        uk, _ = orc.ipiano_foe(v, v, om, lam, "quadratic", max_iters=k, rel_tol=0.0)
        u32 = uk.astype(np.float32).astype(np.float64)
        g, ref = fp.foe_gradient(u32, model), orc.foe_gradient(u32, om)
        worst.append(np.linalg.norm(g - ref) / np.linalg.norm(ref))
    print(("tc  " if kernel == "1" else "ffma"), " ".join(f"{w:.2e}" for w in worst))
