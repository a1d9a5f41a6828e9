"""Decision flips against the oracle on config-4 seeds (512^2, quadratic): first L-trace divergence and
max |dx|/peak for each pass kernel (FOE_TC=1 tensor cores, FOE_TC=0 FFMA), with the oracle's accepted
slack around the flip."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1609_05722_b200 as fp  # noqa: E402
from oracle import cpu as orc  # noqa: E402
from paper_1609_05722_b200.synth import make_counts  # noqa: E402

model = fp.load_packaged_model("foe_a")
om = orc.OracleModel(filters=model.filters, weights=model.weights, boundary=model.boundary)
tab = orc.load_lambda_table("paper_1609_05722_b200/assets/lambda_table.json")
seeds = [int(s) for s in sys.argv[1:]] or list(range(8))
for seed in seeds:
    peak = [0.5, 1.0, 2.0, 4.0][seed % 4]
    _, y = make_counts(512, 512, seed, peak)
    ref = orc.denoise(y, peak, om, "transform", tab, force_branch="quadratic", rel_tol=0.0)
    rt = ref["trace"]
    for kern in ("1", "0"):
        os.environ["FOE_TC"] = kern
        r = fp.denoise(fp.DenoiseRequest(noisy=y, peak=peak, model=model, variant="transform",
                                         force_branch="quadratic"), fp.SolverConfig(rel_tol=0.0))
        L, Lr = np.array(r.trace.L), np.array(rt.L)
        idx = np.nonzero(L != Lr)[0]
        div = int(idx[0]) if len(idx) else None
        err = np.abs(r.image - ref["image"]).max() / peak
        print(f"seed {seed} peak {peak} FOE_TC={kern}: first divergence {div} max|dx|/peak {err:.3e} trials {r.trace.n_trials} ref {rt.n_trials}")
        if div is not None:
            for k in range(max(0, div - 1), min(len(L), div + 2)):
                print(f"   it {k}: L {L[k]:.6g} ref {Lr[k]:.6g}  slack_ref {rt.descent_slack[k]:+.4e} tol {rt.slack_tol[k]:.2e}  slack_gpu {r.trace.descent_slack[k]:+.4e}")
