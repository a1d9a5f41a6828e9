import cProfile, pstats, time, sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1609_05722_b200 as fp
from paper_1609_05722_b200.synth import make_counts
model = fp.load_packaged_model("foe_a")
_, y = make_counts(512, 512, 0, 1.0)
cfg = fp.SolverConfig(rel_tol=0.0)
req = fp.DenoiseRequest(noisy=y, peak=1.0, model=model, variant="transform", force_branch="quadratic")
for _ in range(3): fp.denoise(req, cfg)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5): fp.denoise(req, cfg)
print("mean ms", (time.perf_counter() - t0) / 5 * 1e3)
pr = cProfile.Profile(); pr.enable()
for _ in range(5): fp.denoise(req, cfg)
pr.disable()
st = pstats.Stats(pr); st.sort_stats("cumulative").print_stats(25)
