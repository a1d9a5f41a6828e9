"""Time the fused trial pass back to back (foe_bench_trial_pass) on a 512^2 cfg2 state, for the library named by
FOE_LIB (ablation / diagnostic builds); the state comes from a solve that may fail under an ablated kernel."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1609_05722_b200 as fp  # noqa: E402
from paper_1609_05722_b200 import _lib  # noqa: E402
from paper_1609_05722_b200.anscombe import forward_device  # noqa: E402
from paper_1609_05722_b200.synth import make_counts  # noqa: E402

H = W = 512
model = fp.load_packaged_model("foe_a")
_, y = make_counts(H, W, 0, 1.0)
v = forward_device(torch.from_numpy(y).cuda())
bank = fp.prior.device_bank(model)
L = _lib.lib()
cap = 150
ws = torch.zeros(L.foe_solve_workspace_size(bank.handle, 1, H, W, cap), dtype=torch.uint8, device="cuda")
state = "gpurun_out/pass_state.pt"
if "FOE_LIB" not in os.environ:  # the production library solves once and saves the state for the others
    res = fp.solve_device(model, v, v, 0.6075, "quadratic", 150, fp.SolverConfig(rel_tol=0.0))
    ws, cap = res._workspace, res._cap
    torch.save(ws.cpu(), state)
else:  # ablated kernels give wrong decisions: time them on the saved solved state only
    ws = torch.load(state).cuda()
st = torch.cuda.current_stream()
reps = 200
_lib.check(L.foe_bench_trial_pass(bank.handle, 1, H, W, cap, 10, ws.data_ptr(), ws.numel(), st.cuda_stream))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
_lib.check(L.foe_bench_trial_pass(bank.handle, 1, H, W, cap, reps, ws.data_ptr(), ws.numel(), st.cuda_stream))
e1.record(st)
e1.synchronize()
print(os.environ.get("FOE_LIB", "default"), "pass us", round(e0.elapsed_time(e1) / reps * 1e3, 2))
