"""End-to-end fp.denoise wall times, call by call (host buffers in, image out)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1609_05722_b200 as fp  # noqa: E402
from paper_1609_05722_b200.synth import make_counts  # noqa: E402

model = fp.load_packaged_model("foe_a")
_, y = make_counts(512, 512, 0, 1.0)
cfg = fp.SolverConfig(rel_tol=0.0)
req = fp.DenoiseRequest(noisy=y, peak=1.0, model=model, variant="transform", force_branch="quadratic")
big = torch.empty(256 * 2 ** 20, dtype=torch.uint8, device="cuda") if "--flush" in sys.argv else None
ts = []
for i in range(int(os.environ.get("N", "15"))):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = fp.denoise(req, cfg)
    ts.append((time.perf_counter() - t0) * 1e3)
print("e2e ms:", [round(t, 2) for t in ts])
print("allocator: reserved %.1f MiB, num_alloc_retries %d" % (torch.cuda.memory_reserved() / 2 ** 20,
      torch.cuda.memory_stats().get("num_alloc_retries", 0)))
