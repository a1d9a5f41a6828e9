"""Diagnostic: compare the device solve trace against the C oracle iteration by iteration."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1609_05722_b200 as fp  # noqa: E402
from oracle import cpu as orc  # noqa: E402
from paper_1609_05722_b200.synth import make_counts  # noqa: E402

H = int(sys.argv[1]) if len(sys.argv) > 1 else 64
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 10
model = fp.load_packaged_model("foe_a")
om = orc.OracleModel(filters=model.filters, weights=model.weights, boundary=model.boundary)
_, y = make_counts(H, H, 0, 4.0)
v = orc.anscombe_forward(y)
lam = 0.538107
import torch  # noqa: E402
vd = torch.from_numpy(v).to("cuda", torch.float32)
print("F(v) oracle", orc.foe_energy(v, om), "device", fp.foe_energy(v, model))
res = fp.solve_device(model, vd, vd, lam, "quadratic", iters, fp.SolverConfig(rel_tol=0.0), raise_on_failure=False)
u_ref, tr = orc.ipiano_foe(v, v, om, lam, "quadratic", max_iters=iters, rel_tol=0.0)
t = res.traces[0]
print("status", res.status, "n", len(t), "trials", t.n_trials, "oracle trials", tr.n_trials)
for k in range(min(len(t), len(tr.F))):
    print(k, "F", t.F[k], tr.F[k], "L", t.L[k], tr.L[k], "step", t.step_norm[k], tr.step_norm[k],
          "G", t.G[k], tr.G[k])
u = res.u.double().cpu().numpy()
print("max|du|", np.abs(u - u_ref).max())
