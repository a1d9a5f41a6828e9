import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_1609_05722_b200 as fp
from oracle import cpu as orc
from paper_1609_05722_b200.synth import make_counts
model = fp.load_packaged_model("foe_fallback48x7")
om = orc.OracleModel(filters=model.filters, weights=model.weights, boundary=model.boundary)
x, y = make_counts(128, 128, 5, 1.0)
for k in ("0", "1"):
    os.environ["FOE_TC7"] = k
    r = fp.denoise(fp.DenoiseRequest(noisy=y, peak=1.0, model=model, variant="transform", force_branch="quadratic"), fp.SolverConfig(rel_tol=0.0))
    u = r.transformed.astype(np.float32).astype(np.float64)
    g_ref = orc.foe_gradient(u, om)
    for kk in ("0", "1"):
        os.environ["FOE_TC7"] = kk
        g = fp.foe_gradient(u, model)
        print("solve kernel", k, "grad kernel", kk, "rel-L2 vs oracle", np.linalg.norm(g - g_ref) / np.linalg.norm(g_ref))
    v = fp.anscombe_forward(y) if hasattr(fp, "anscombe_forward") else None
