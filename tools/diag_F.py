"""Where does the trace's F column differ from the reference?  cfg1 (256^2, peak 4, quadratic):
per-iteration F_gpu - F_ref, and the device energy (EVAL pass) at v and at the final iterate against
the fp64 oracle at the same fp32 point."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1609_05722_b200 as fp  # noqa: E402
from oracle import cpu as orc  # noqa: E402
from paper_1609_05722_b200.synth import make_counts  # noqa: E402

g = dict(np.load("tests/golden/cfg1_256.npz"))
x, y = make_counts(256, 256, 0, 4.0)
model = fp.load_packaged_model("foe_a")
om = orc.OracleModel(filters=model.filters, weights=model.weights, boundary=model.boundary)
for kern in ("1", "0"):
    os.environ["FOE_TC"] = kern
    r = fp.denoise(fp.DenoiseRequest(noisy=y, peak=4.0, model=model, variant="transform", force_branch="quadratic"),
                   fp.SolverConfig(rel_tol=0.0))
    F = np.array(r.trace.F)
    Fr = g["trace"][:, 0]
    d = F - Fr
    print(f"FOE_TC={kern}: F_ref[0]={Fr[0]:.10g} F_ref[-1]={Fr[-1]:.10g}")
    for k in (0, 1, 2, 5, 10, 50, 100, 149):
        print(f"  it {k:3d} F_gpu-F_ref={d[k]:+.6e} rel={d[k] / Fr[k]:+.3e}")
    v = orc.anscombe_forward(y).astype(np.float32).astype(np.float64)
    for name, u in (("v", v), ("u_final", r.transformed.astype(np.float32).astype(np.float64))):
        e_dev = fp.foe_energy(u, model)
        e_orc = orc.foe_energy(u, om)
        print(f"  EVAL energy at {name}: dev={e_dev:.10g} oracle={e_orc:.10g} rel={(e_dev - e_orc) / e_orc:+.3e}")
