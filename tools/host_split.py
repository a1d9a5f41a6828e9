"""Host-side cost of one solve_device call (512^2 foe_a): wall time of a 1-iteration solve (nearly all
fixed overhead) split into the Python preparation, the foe_solve C call and the result handling, plus
the device-timed fixed part (intercept of step time vs trials)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1609_05722_b200 as fp  # noqa: E402
from paper_1609_05722_b200 import _lib, solver  # noqa: E402
from paper_1609_05722_b200.anscombe import forward_device  # noqa: E402
from paper_1609_05722_b200.synth import make_counts  # noqa: E402

model = fp.load_packaged_model("foe_a")
_, y = make_counts(512, 512, 0, 1.0)
v = forward_device(torch.from_numpy(y).cuda())
L = _lib.lib()
t_c = []
orig = L.foe_solve


def timed(*args):
    t0 = time.perf_counter()
    r = orig(*args)
    t_c.append(time.perf_counter() - t0)
    return r


L.foe_solve = timed
for it in (150, 1):
    cfg = fp.SolverConfig(rel_tol=0.0, max_iters=it)
    for _ in range(3):
        solver.solve_device(model, v, v, 0.6075, "quadratic", it, cfg)
    torch.cuda.synchronize()
    t_c.clear()
    walls, devs, trials = [], [], 0
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0.record()
        res = solver.solve_device(model, v, v, 0.6075, "quadratic", it, cfg)
        e1.record()
        e1.synchronize()
        walls.append(time.perf_counter() - t0)
        devs.append(e0.elapsed_time(e1) * 1e-3)
        trials = res.traces[0].n_trials
    w, c, d = (float(np.median(x)) * 1e3 for x in (walls, t_c, devs))
    print(f"iters {it:4d} trials {trials:4d}: wall {w:.3f} ms, foe_solve call {c:.3f} ms, "
          f"python around it {w - c:.3f} ms, device events {d:.3f} ms")
