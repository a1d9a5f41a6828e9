"""tcgen05.ld / tcgen05.st throughput probe: bytes per SM clock with 4..32 warps issuing .32x32b.x32 accesses."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1609_05722_b200 import _lib  # noqa: E402

L = _lib.lib()
out = torch.zeros(2, dtype=torch.int64, device="cuda")
for store in (0, 1):
    for nw in (4, 8, 16, 24):
        iters = 64
        for _ in range(2):
            _lib.check(L.foe_debug_tmem_rate(nw, store, iters, out.data_ptr(), torch.cuda.current_stream().cuda_stream))
        torch.cuda.synchronize()
        cyc = int(out[0].item())
        nbytes = nw * iters * 4 * 32 * 32 * 4
        print(f"{'st' if store else 'ld'} warps={nw}: {cyc} cycles, {nbytes / cyc:.1f} B/clk/SM")
