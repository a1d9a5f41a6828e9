"""48 x 7 x 7 bank: fused energy / gradient and a 512^2 solve, tensor-core pass (FOE_TC7=1) vs the FFMA pass
(FOE_TC7=0).  Run twice (one process per switch); writes gpurun_out/tc7_<tag>.npz, compare with --cmp."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

if len(sys.argv) > 1 and sys.argv[1] == "--cmp":
    a, b = np.load("gpurun_out/tc7_tc.npz"), np.load("gpurun_out/tc7_ffma.npz")
    for k in a.files:
        x, y = a[k], b[k]
        if k.startswith("L"):
            n = min(len(x), len(y))
            print(k, "len", len(x), len(y), "first L diff at", int(np.argmax(np.abs(x[:n] - y[:n]) > 1e-9 * np.abs(y[:n]))) if np.any(np.abs(x[:n] - y[:n]) > 1e-9 * np.abs(y[:n])) else "none")
        else:
            err = np.max(np.abs(x - y)) / max(np.max(np.abs(y)), 1e-30)
            print(k, "shape", x.shape, "max rel (to max|ffma|)", float(err),
                  "rel-L2", float(np.linalg.norm(x - y) / max(np.linalg.norm(y), 1e-30)))
    sys.exit(0)

import torch  # noqa: E402

import paper_1609_05722_b200 as fp  # noqa: E402
from paper_1609_05722_b200.anscombe import forward_device  # noqa: E402
from paper_1609_05722_b200.synth import make_counts  # noqa: E402

tag = sys.argv[1]
model = fp.load_model(os.path.join(os.path.dirname(fp.__file__), "assets", "foe_fallback48x7.foe"))
out = {}
for (h, w) in ((512, 512), (97, 131), (48, 64)):
    _, y = make_counts(h, w, 1, 4.0)
    v = forward_device(torch.from_numpy(y).cuda())
    e, g = fp.prior.energy_grad_device(v, model)
    out[f"e_{h}x{w}"] = e.cpu().numpy()
    out[f"g_{h}x{w}"] = g.cpu().numpy()
_, y = make_counts(512, 512, 0, 1.0)
v = forward_device(torch.from_numpy(y).cuda())
res = fp.solve_device(model, v, v, 0.6075, "quadratic", 150, fp.SolverConfig(rel_tol=0.0))
out["u_solve"] = res.u.cpu().numpy()
out["L_solve"] = np.asarray(res.traces[0].L)
np.savez(f"gpurun_out/tc7_{tag}.npz", **out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
res = fp.solve_device(model, v, v, 0.6075, "quadratic", 150, fp.SolverConfig(rel_tol=0.0))
e1.record()
e1.synchronize()
print(tag, "solve ms", e0.elapsed_time(e1), "trials", res.traces[0].n_trials)
