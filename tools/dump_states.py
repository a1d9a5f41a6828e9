"""Dump the device iterates u_k (fp32) of a cfg4 solve after k accepted iterations, for both pass kernels
(offline analysis of a decision flip: gpurun_out/states_seed{S}_tc{0,1}_k{K}.npy)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1609_05722_b200 as fp  # noqa: E402
from paper_1609_05722_b200.anscombe import forward_device  # noqa: E402
from paper_1609_05722_b200.synth import make_counts  # noqa: E402

seed, ks = int(sys.argv[1]), [int(k) for k in sys.argv[2:]]
peak = [0.5, 1.0, 2.0, 4.0][seed % 4]
_, y = make_counts(512, 512, seed, peak)
model = fp.load_packaged_model("foe_a")
lam = fp.select_lambda(peak, "transform", force_branch="quadratic")
os.makedirs("gpurun_out", exist_ok=True)
for kern in ("1", "0"):
    os.environ["FOE_TC"] = kern
    v = forward_device(torch.from_numpy(y).cuda())
    for k in ks:
        r = fp.solve_device(model, v, v, lam, "quadratic", k, fp.SolverConfig(rel_tol=0.0))
        np.save(f"gpurun_out/states_seed{seed}_tc{kern}_k{k}.npy", r.u.cpu().numpy())
        print(kern, k, r.traces[0].L[-1], r.traces[0].n_rechecks)
