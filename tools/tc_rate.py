"""tcgen05 kind::tf32 MMA throughput probe (M = 128, K = 8): cycles per MMA for A in TMEM / smem."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1609_05722_b200 import _lib  # noqa: E402

L = _lib.lib()
out = torch.zeros(1, dtype=torch.int64, device="cuda")
for ts in (1, 0):
    for n in (32, 64, 128):
        for nchain in (1, 2, 3, 4):
            if nchain * n > 256:
                continue
            res = []
            for nm in (1, 12, 36, 108):
                for _ in range(2):
                    _lib.check(L.foe_debug_tc_rate(n, ts, nm, nchain, 0, out.data_ptr(), torch.cuda.current_stream().cuda_stream))
                torch.cuda.synchronize()
                res.append((nm, int(out.item())))
            per = (res[-1][1] - res[1][1]) / (res[-1][0] - res[1][0])
            print(f"{'TS' if ts else 'SS'} N={n} chains={nchain}: " + ", ".join(f"{nm}->{c}" for nm, c in res) +
                  f"  => {per:.1f} cycles/MMA")

# a tcgen05.commit after every group of MMAs: does the commit stall the pipe?
for every in (0, 18, 9, 6, 3, 1):
    res = []
    for nm in (36, 108):
        for _ in range(2):
            _lib.check(L.foe_debug_tc_rate(64, 1, nm, 1, every, out.data_ptr(), torch.cuda.current_stream().cuda_stream))
        torch.cuda.synchronize()
        res.append((nm, int(out.item())))
    print(f"TS N=64 commit every {every}: " + ", ".join(f"{nm}->{c}" for nm, c in res) +
          f"  => {(res[1][1] - res[0][1]) / 72:.1f} cycles/MMA")
