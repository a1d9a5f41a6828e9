"""One 512^2 cfg2 solve with max_iters from argv (for launch lists of a single solve under ncu)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1609_05722_b200 as fp  # noqa: E402
from paper_1609_05722_b200.anscombe import forward_device  # noqa: E402
from paper_1609_05722_b200.synth import make_counts  # noqa: E402

it = int(sys.argv[1]) if len(sys.argv) > 1 else 1
model = fp.load_packaged_model("foe_a")
_, y = make_counts(512, 512, 0, 1.0)
v = forward_device(torch.from_numpy(y).cuda())
cfg = fp.SolverConfig(rel_tol=0.0, max_iters=it)
fp.solve_device(model, v, v, 0.6075, "quadratic", it, cfg)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
res = fp.solve_device(model, v, v, 0.6075, "quadratic", it, cfg)
e1.record()
e1.synchronize()
print("solve ms", e0.elapsed_time(e1), "trials", res.traces[0].n_trials)
