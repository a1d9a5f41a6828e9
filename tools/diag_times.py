"""Per-CTA timing of one fused trial pass (512^2 cfg2 state after a solve): start skew, compute, tail."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1609_05722_b200 as fp  # noqa: E402
from paper_1609_05722_b200 import _lib  # noqa: E402
from paper_1609_05722_b200.anscombe import forward_device  # noqa: E402
from paper_1609_05722_b200.synth import make_counts  # noqa: E402

H = W = int(sys.argv[1]) if len(sys.argv) > 1 else 512
model = fp.load_packaged_model("foe_a")
_, y = make_counts(H, W, 0, 1.0)
v = forward_device(torch.from_numpy(y).cuda())
res = fp.solve_device(model, v, v, 0.6075, "quadratic", 150, fp.SolverConfig(rel_tol=0.0))
L = _lib.lib()
ws = res._workspace
ncta = (-(-H // 32)) * (-(-W // 60))
t = torch.zeros(ncta * 5 + 512, dtype=torch.int64, device="cuda")
for _ in range(3):
    _lib.check(L.foe_debug_pass_times(res._bank.handle, 1, H, W, res._cap, ws.data_ptr(), ws.numel(), t.data_ptr(),
                                      torch.cuda.current_stream().cuda_stream))
torch.cuda.synchronize()
full = t.cpu().numpy()
a = full[:ncta * 3].reshape(ncta, 3).astype(np.float64)
phs = full[ncta * 3:ncta * 3 + 18 * 16].reshape(18, 16).astype(np.float64)
loop0 = float(full[ncta * 3 + 18 * 16])
ext = full[ncta * 3 + 18 * 16: ncta * 3 + 18 * 16 + 15].astype(np.float64)
if ext[2]:
    names = ["loop start", "loop end", "kernel start", "griddep done", "fold done", "block reduce done", "ticket", "tmem released", "first fold value", "first fold store", "loads issued", "ctl read", "cells staged", "warp partials", "dF warp partial"]
    print("CTA (0,0) phase stamps, cycles from kernel start:",
          {n: int(ext[i] - ext[2]) for i, n in enumerate(names) if ext[i]})
if phs.any():
    np.set_printoptions(precision=0, suppress=True, linewidth=200)
    cols = [0, 1, 2, 3, 4, 5, 6, 7, 8, 9]
    print("block stamps (cycles from loop start): fwd issued (MMA), fwd seen (point), adj issued (MMA), Y in ring (mover), "
          "g summed (mover), im2col start (mover), Psi handed over (point), A built (mover), adj seen (mover), energy done (point)")
    tab = phs[:, cols] - loop0
    tab[phs[:, cols] == 0] = -1
    print(tab.astype(np.int64))
    print("MMA warp (cycles from loop start): z issue start, z issued, dz issue start, dz issued, adj issue start, adj issued")
    m = phs[:, [10, 11, 12, 0, 13, 2]] - loop0
    m[phs[:, [10, 11, 12, 0, 13, 2]] == 0] = -1
    print(m.astype(np.int64))
pw = full[ncta * 3 + 304: ncta * 3 + 304 + 200].reshape(25, 8)  # the first 25 warps.astype(np.float64)
if pw.any():
    t = pw - loop0
    t[pw == 0] = -1
    print("per-warp stamps, block 8 (movers, point set 0) / 9 (set 1): movers [im2col start, A built, sum start, sum done]; "
          "point [fwd seen, z/dz loaded, Psi handed, energy done, adj seen, Y in ring]")
    print(t[:, :6].astype(np.int64))
a -= a[:, 0].min()
start, comp, end = a[:, 0] / 1e3, a[:, 1] / 1e3, a[:, 2] / 1e3
dur = comp - start
print(f"CTAs {ncta}: start skew max {start.max():.2f} us; phase1 (t1-t0) min/med/max {dur.min():.2f}/"
      f"{np.median(dur):.2f}/{dur.max():.2f} us; phase2 (t2-t1) med {np.median(end - comp):.2f} max "
      f"{(end - comp).max():.2f}; last t1 {comp.max():.2f}; last t2 {end.max():.2f} us")
ty, tx = -(-H // 32), -(-W // 60)
grid = dur.reshape(ty, tx)
np.set_printoptions(precision=1, suppress=True, linewidth=200)
print(grid)
