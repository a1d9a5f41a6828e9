"""Small transform/quadratic denoise (64^2 or argv[1]) printing the first L-trace entries: quick check of the
solve path under different kernel / launch switches (FOE_TC, FOE_PDL, FOE_GRAPH)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1609_05722_b200 as fp  # noqa: E402
from paper_1609_05722_b200.synth import make_counts  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
m = fp.load_packaged_model("foe_a")
x, y = make_counts(n, n, 0, 4.0)
req = fp.DenoiseRequest(noisy=y, peak=4.0, model=m, variant="transform", force_branch="quadratic")
try:
    r = fp.denoise(req, fp.SolverConfig(rel_tol=0.0))
    print(os.environ.get("FOE_TC"), os.environ.get("FOE_PDL"), os.environ.get("FOE_GRAPH"), "trials",
          r.trace.n_trials, "L", [round(v, 4) for v in list(r.trace.L)[:6]], "max", float(np.abs(r.image).max()))
except Exception as e:  # noqa: BLE001
    print(os.environ.get("FOE_TC"), os.environ.get("FOE_PDL"), os.environ.get("FOE_GRAPH"), "FAILED", e)
