import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1609_05722_b200 as fp
from paper_1609_05722_b200.anscombe import forward_device
from paper_1609_05722_b200.synth import make_counts
model = fp.load_packaged_model("foe_a")
_, y = make_counts(512, 512, 0, 1.0)
v = forward_device(torch.from_numpy(y).cuda())
for it in (150, 100, 50, 10, 1):
    cfg = fp.SolverConfig(rel_tol=0.0, max_iters=it)
    for _ in range(2): fp.solve_device(model, v, v, 0.6075, "quadratic", it, cfg)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); res = fp.solve_device(model, v, v, 0.6075, "quadratic", it, cfg); e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    print("iters", it, "trials", res.traces[0].n_trials, "ms", round(float(np.median(ts)), 3))
