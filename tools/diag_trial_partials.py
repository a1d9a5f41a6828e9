"""One band-mode init + trial pass on a 256^2 image (single band): per-tile partials of the trial pass, for
comparing the tensor-core and FFMA kernels (run twice: FOE_TC=1 / FOE_TC=0).  Output: .npy under gpurun_out/."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1609_05722_b200 as fp  # noqa: E402
from paper_1609_05722_b200 import bands  # noqa: E402
from paper_1609_05722_b200.anscombe import forward_device  # noqa: E402
from paper_1609_05722_b200.synth import make_counts  # noqa: E402

H = W = int(sys.argv[1]) if len(sys.argv) > 1 else 256
tag = sys.argv[2] if len(sys.argv) > 2 else "x"
model = fp.load_packaged_model("foe_a")
_, y = make_counts(H, W, 0, 1.0)
v = forward_device(torch.from_numpy(y).cuda()).view(1, H, W)
tx, ty = bands.tile_grid(5, H, W)
bs = bands.Band(model, 1, H, W, 0, ty, 8, fp.SolverConfig(rel_tol=0.0))
bs.begin(v, v, 0.6075, "quadratic", 5)
bs.commit(True)  # init pass decision (f_u)
NT = int(sys.argv[3]) if len(sys.argv) > 3 else 1
ps = []
for k in range(NT):
    bs.trial()
    torch.cuda.synchronize()
    ps.append(bs.partials.cpu().numpy().reshape(ty * tx, -1).copy())
    bs.commit(False)
p = np.stack(ps)
np.save(f"gpurun_out/trial_partials_{tag}.npy", p)
for k in range(NT):
    print(tag, k, "partials sum", p[k][:, :5].sum(axis=0))
