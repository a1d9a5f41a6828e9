"""Per-block cycle stamps of the 7x7 tensor-core pass (FOE_STAMPS=1 build via FOE_LIB): 512^2, fallback bank."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1609_05722_b200 as fp  # noqa: E402
from paper_1609_05722_b200 import _lib  # noqa: E402
from paper_1609_05722_b200.anscombe import forward_device  # noqa: E402
from paper_1609_05722_b200.synth import make_counts  # noqa: E402

H = W = 512
model = fp.load_packaged_model("foe_fallback48x7")
_, y = make_counts(H, W, 0, 1.0)
v = forward_device(torch.from_numpy(y).cuda())
res = fp.solve_device(model, v, v, 0.6075, "quadratic", 150, fp.SolverConfig(rel_tol=0.0))
L = _lib.lib()
tx, ty = (-(-W // 58)), (-(-H // 34))
ncta = tx * ty
NB = 20
t = torch.zeros(ncta * 3 + NB * 16 + 16, dtype=torch.int64, device="cuda")
ws = res._workspace
for _ in range(3):
    _lib.check(L.foe_debug_pass_times(res._bank.handle, 1, H, W, res._cap, ws.data_ptr(), ws.numel(), t.data_ptr(),
                                      torch.cuda.current_stream().cuda_stream))
torch.cuda.synchronize()
full = t.cpu().numpy()
phs = full[ncta * 3:ncta * 3 + NB * 16].reshape(NB, 16).astype(np.float64)
loop0 = float(full[ncta * 3 + NB * 16])
cols = [5, 0, 1, 2, 3, 4, 6]
print("cycles from loop start: im2col-start, fwd-issued, fwd-seen, adj-issued, Y-drained, H-done, V-done(q)")
tab = phs[:, cols] - loop0
tab[phs[:, cols] == 0] = -1
np.set_printoptions(linewidth=200, suppress=True)
print(tab.astype(np.int64))
