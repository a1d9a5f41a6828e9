"""GPU idle gaps inside one bench step (512^2 cfg2): kernel timeline from torch.profiler (CUPTI activity
records, no replay), the step's span vs the summed kernel time, and the largest gaps with the kernels
either side -- where the device-timed step exceeds passes x pass time.

usage (GPU box): python tools/gap_profile.py [--e2e]
"""
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1609_05722_b200 as fp  # noqa: E402
from paper_1609_05722_b200.anscombe import forward_device, inverse_exact_unbiased_device  # noqa: E402
from paper_1609_05722_b200.synth import make_counts  # noqa: E402

model = fp.load_packaged_model("foe_a")
_, y = make_counts(512, 512, 0, 1.0)
y_dev = torch.from_numpy(y).cuda()
cfg = fp.solver_budget(1.0, fp.SolverConfig(rel_tol=0.0))
e2e = "--e2e" in sys.argv


def step():
    if e2e:
        return fp.denoise(fp.DenoiseRequest(noisy=y, peak=1.0, model=model, variant="transform",
                                            force_branch="quadratic"), cfg)
    v = forward_device(y_dev)
    res = fp.solve_device(model, v, v, 0.6075, "quadratic", cfg.max_iters, cfg)
    return res, inverse_exact_unbiased_device(res.u)


out = None
for _ in range(4):
    out = step()  # noqa: F841
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    out = step()
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ks = sorted(((e.time_range.start, e.time_range.end, e.name) for e in evs), key=lambda t: t[0])
span = ks[-1][1] - ks[0][0]
busy = 0.0
cur_s, cur_e = ks[0][0], ks[0][1]
for s, e, _ in ks[1:]:  # union of intervals (PDL overlaps successive passes)
    if s > cur_e:
        busy += cur_e - cur_s
        cur_s, cur_e = s, e
    else:
        cur_e = max(cur_e, e)
busy += cur_e - cur_s
gaps = []
last_e, last_n = ks[0][1], ks[0][2]
for s, e, n in ks[1:]:
    if s > last_e:
        gaps.append((s - last_e, last_n[:40], n[:40]))
    if e > last_e:
        last_e, last_n = e, n
gaps.sort(reverse=True)
print(f"{'e2e' if e2e else 'step'}: {len(ks)} device records, span {span:.1f} us, busy {busy:.1f} us, "
      f"idle {span - busy:.1f} us in {len(gaps)} gaps")
for g, a, b in gaps[:12]:
    print(f"  {g:8.1f} us  after {a!r} before {b!r}")
