"""The config-5 row-band path end to end across processes: one band per rank, torch.distributed, the
bands' decisions taken from all-gathered partials (bands.solve_bands with DistExchange).

Only one GPU is available per test box, so the ranks share cuda:0 over the gloo backend (NCCL refuses
two ranks on one device); DistExchange then stages the device partials and halo rows through host
memory.  No kernel of one rank waits on another rank's kernel: every exchange is a host-side
collective between passes.  The result must equal the single-device solve bit for bit."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _band_worker(rank, world, port, H, W, iters, bank, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist

    import paper_1609_05722_b200 as fp
    from paper_1609_05722_b200 import bands
    from paper_1609_05722_b200.anscombe import forward_device
    from paper_1609_05722_b200.synth import make_counts
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        model = fp.load_packaged_model(bank)
        _, y = make_counts(H, W, 7, 2.0)
        v = forward_device(torch.from_numpy(y).cuda())
        lam = fp.select_lambda(2.0, "transform", force_branch="quadratic")
        _, ty = bands.tile_grid(model.basis.size, H, W)
        t0, t1 = bands.partition_tile_rows(ty, world)[rank]
        band = bands.Band(model, 1, H, W, t0, t1, iters, fp.SolverConfig(rel_tol=0.0))
        l0, l1 = band.local_rows
        vl = v[None, l0:l1].contiguous()
        ex = bands.DistExchange()
        (u, traces, status, _), = bands.solve_bands([band], ex, [vl], [vl], lam, "quadratic", iters)
        q.put((rank, band.rows, u[0].cpu().numpy(), traces[0].L, traces[0].F, status, ex.backend))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,H,W,bank", [(2, 512, 384, "foe_a"), (3, 400, 260, "foe_a"),
                                            (2, 300, 200, "foe_fallback48x7")])
def test_solve_bands_over_processes_equals_single_device(world, H, W, bank):
    import torch
    import torch.multiprocessing as mp

    import paper_1609_05722_b200 as fp
    from paper_1609_05722_b200.anscombe import forward_device
    from paper_1609_05722_b200.synth import make_counts
    iters = 150
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29600 + (os.getpid() + world) % 2000
    procs = [ctx.Process(target=_band_worker, args=(r, world, port, H, W, iters, bank, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=600) for _ in procs), key=lambda t: t[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    model = fp.load_packaged_model(bank)
    _, y = make_counts(H, W, 7, 2.0)
    v = forward_device(torch.from_numpy(y).cuda())
    lam = fp.select_lambda(2.0, "transform", force_branch="quadratic")
    single = fp.solve_device(model, v, v, lam, "quadratic", iters, fp.SolverConfig(rel_tol=0.0))
    u_single = single.u.cpu().numpy()
    assert [r[1][0] for r in res] == sorted(r[1][0] for r in res) and res[-1][1][1] == H
    u_bands = np.concatenate([r[2] for r in res], axis=0)
    assert all(r[5] == [0] and r[6] == "gloo" for r in res)
    for r in res:
        assert r[3] == single.traces[0].L and r[4] == single.traces[0].F
    np.testing.assert_array_equal(u_bands, u_single)
