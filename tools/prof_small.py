import cProfile, pstats, os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1609_05722_b200 as fp
from paper_1609_05722_b200.anscombe import forward_device
from paper_1609_05722_b200.synth import make_counts
model = fp.load_packaged_model("foe_a")
_, y = make_counts(512, 512, 0, 1.0)
v = forward_device(torch.from_numpy(y).cuda())
cfg = fp.SolverConfig(rel_tol=0.0, max_iters=150)
for _ in range(3): fp.solve_device(model, v, v, 0.6075, "quadratic", 150, cfg)
torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable()
for _ in range(10): fp.solve_device(model, v, v, 0.6075, "quadratic", 150, cfg)
pr.disable()
st = pstats.Stats(pr); st.sort_stats("tottime").print_stats(12)
