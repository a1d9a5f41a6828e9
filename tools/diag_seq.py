"""Back-to-back fused passes (as in a solve): per-pass CTA start / loop-start / exit spans and the
gaps between passes, from %globaltimer stamps."""
import ctypes
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
NP = 6
model = fp.load_packaged_model("foe_a")
_, y = make_counts(H, W, 0, 1.0)
v = forward_device(torch.from_numpy(y).cuda())
res = fp.solve_device(model, v, v, 0.6075, "quadratic", 150, fp.SolverConfig(rel_tol=0.0))
L = _lib.lib()
L.foe_debug_pass_times_seq.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                       ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
ws = res._workspace
ncta = (-(-H // 32)) * (-(-W // 60))
stride = 5 * ncta + 512
t = torch.zeros(NP * stride, dtype=torch.int64, device="cuda")
for _ in range(3):
    _lib.check(L.foe_debug_pass_times_seq(res._bank.handle, 1, H, W, res._cap, ws.data_ptr(), ws.numel(), t.data_ptr(),
                                          NP, torch.cuda.current_stream().cuda_stream))
torch.cuda.synchronize()
full = t.cpu().numpy().astype(np.float64)
t0 = full[0:3 * ncta:3].min()
prev_exit = None
for k in range(NP):
    a = full[k * stride:k * stride + 3 * ncta].reshape(ncta, 3)
    start, loop, end = (a[:, 0] - t0) / 1e3, (a[:, 1] - t0) / 1e3, (a[:, 2] - t0) / 1e3
    line = (f"pass {k}: first start {start.min():8.2f}  last start {start.max():8.2f}  median loop-start "
            f"{np.median(loop):8.2f}  median exit {np.median(end):8.2f}  last exit {end.max():8.2f} us")
    rel = (full[k * stride + 3 * ncta + 512:k * stride + 4 * ncta + 512] - t0) / 1e3
    dec = full[k * stride + 4 * ncta + 512:k * stride + 5 * ncta + 512]
    dec = (dec[dec > 0].max() - t0) / 1e3 if (dec > 0).any() else float("nan")
    line += f"\n        released: first {rel.min():8.2f} median {np.median(rel):8.2f} last {rel.max():8.2f}  decider done {dec:8.2f}"
    if prev_exit is not None:
        line += f"  | gap last-exit(k-1) -> median loop-start(k) {np.median(loop) - prev_exit:6.2f}"
    print(line)
    prev_exit = end.max()
