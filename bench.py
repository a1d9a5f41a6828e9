"""Benchmark of the FoE Poisson-denoise hot path on B200 (driver contract: one JSON line on rank 0).

Workload (BASELINE.json configs[1]): one 512x512 image from the frozen synthetic
generator, peak 1, Anscombe-domain model foe_a (24 filters 5x5), quadratic data
term, the reference's iPiano solver with its own 150-iteration budget
(pipeline.py:83-87).  A "step" = one full denoise: Anscombe forward -> device
iPiano solve (all backtracking on device) -> exact unbiased inverse, with the
counts already resident in HBM.  With N GPUs every rank denoises its own image
(seed = rank): weak scaling, no data-path collective.

Metric: Mpixel*iter/s = pixels x accepted iterations / time (whole job).
L2 handling: the 512^2 working set (~6 MB) lives in L2 by design; a 256 MiB
buffer is rewritten between timed steps so every step starts cold.

--impl reference times the CPU oracle port (oracle/foe_oracle.c, fp64, all host
threads) on the same config -- each step one full 150-iteration cfg2 solve, the
same workload and config dict as this arm.  The reference itself is pure Python
(cv2 + numpy) and has no compilable path; it is installed (pip --target) into
baseline/_ref and timed beside the port as ``cpu_baseline_reference``: its own
public denoise() on the same counts, with solver_budget patched to a truncated
iteration count (a bounded sample; the steady per-iteration rate is the
difference of a 13- and a 3-iteration run, so the iteration-0 backtracking climb
cancels).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

H = W = 512
PEAK = 1.0
N_FILT, K = 24, 5
ALG_FLOP_PER_PX_IT = 4 * N_FILT * K * K
_PEAKS_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "MEASURED_PEAKS.json")
PEAKS = json.load(open(_PEAKS_PATH)) if os.path.exists(_PEAKS_PATH) else {}  # forward + adjoint
METRIC = "Mpixel·iter/s of FoE solver (fp32, % FP32 peak); 512² denoise ms"
CONFIG = {"workload": "cfg2: 512x512 synthetic, peak 1, transform/quadratic, foe_a 24x5x5, 150 iters",
          "model": "foe_a (24 filters 5x5, dct5, symmetric)", "image": "512x512", "peak": PEAK,
          "iterations": 150, "l2": "flushed between steps (256 MiB rewrite); working set L2-resident within a step"}


def config_for(world: int) -> dict:
    """The config dict both arms print (identical, so the driver's same_config check holds)."""
    return dict(CONFIG, parallelism=f"replicas{world}" if world > 1 else "single")


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))


class ClockSampler:
    """Samples SM clock and throttle reasons with NVML during the timed region."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, index):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            # first queries outside the timed region: NVML initialises its per-device clock state lazily
            # (tens of ms, holding driver locks that stall the timed step's launches and copies)
            pynvml.nvmlDeviceGetClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            pynvml.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.05)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        if self.nv:
            self._stop.set()
            self.t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def bench_fallback_bank(fp, _lib, L, y_dev, lam, cfg, stream, fp32_peak_tflops, H, W, steps=3):
    """Config 2 with the 48 x 7 x 7 fallback bank: device-timed solves and the fused pass."""
    import torch
    from paper_1609_05722_b200.anscombe import forward_device
    model = fp.load_packaged_model("foe_fallback48x7")
    n, k = model.n_filters, model.basis.atoms.shape[-1]
    v = forward_device(y_dev)
    # warm-up (graph capture, allocator): the same calls as the timed loop, the previous result kept alive
    # while the next solve runs, so the caching allocator has reached its steady state before timing
    res = None
    for _ in range(3):
        res = fp.solve_device(model, forward_device(y_dev), v, lam, "quadratic", cfg.max_iters, cfg)  # noqa: F841
    torch.cuda.synchronize()
    ms, iters = 0.0, 0
    for _ in range(steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        res = fp.solve_device(model, forward_device(y_dev), v, lam, "quadratic", cfg.max_iters, cfg)
        e1.record(stream)
        e1.synchronize()
        ms += e0.elapsed_time(e1)
        iters += len(res.traces[0])
    ws = res._workspace
    reps = 20
    _lib.check(L.foe_bench_trial_pass(res._bank.handle, 1, H, W, res._cap, 3, ws.data_ptr(), ws.numel(),
                                      stream.cuda_stream))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    _lib.check(L.foe_bench_trial_pass(res._bank.handle, 1, H, W, res._cap, reps, ws.data_ptr(), ws.numel(),
                                      stream.cuda_stream))
    e1.record(stream)
    e1.synchronize()
    pass_ms = e0.elapsed_time(e1) / reps
    flop_px_it = 4 * n * k * k
    achieved = flop_px_it * H * W / (pass_ms * 1e-3) / 1e12
    tc = bool(L.foe_pass_uses_tensor_cores(k, n))
    return {"model": f"foe_fallback48x7 ({n} filters {k}x{k}, dct7, symmetric)", "ms_per_denoise": ms / steps,
            "value": H * W * iters / (ms * 1e-3) / 1e6, "unit": "Mpixel*iter/s", "iterations": iters / steps,
            "pass_ms": pass_ms, "alg_flop_per_px_it": flop_px_it,
            "kernel": (f"k_pass_tc7<TRIAL,SYM> (tcgen05 3xTF32, {k}x{k})" if k == 7 else "k_pass_tc") if tc
            else f"k_pass<{k},TRIAL,SYM> (FFMA)",
            "roofline_frac": achieved / fp32_peak_tflops, "achieved_tflops": achieved}


def pass_traffic(kernel):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the pass kernel, from the committed
    ncu --set full summary of the current kernel (profiles/roofline_traffic.json), else None."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "roofline_traffic.json")
    try:
        with open(path) as fh:
            rec = json.load(fh).get(kernel)
        return None if rec is None else rec["dram_bytes_per_launch"]
    except (OSError, ValueError, KeyError):
        return None


def measure_ffma_peak(L, dev, index):
    """FP32 FFMA TFLOP/s of this GPU from the library's probe kernel (best of 5, CUDA events), and
    the median SM clock NVML saw while it ran."""
    import ctypes

    import torch
    from paper_1609_05722_b200 import _lib
    scratch = torch.zeros(1, dtype=torch.float32, device=dev)
    flop = ctypes.c_double(0.0)
    stream = torch.cuda.current_stream()
    best = 0.0
    with ClockSampler(index) as clk:
        for rep in range(6):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            _lib.check(L.foe_measure_ffma_peak(4096, scratch.data_ptr(), ctypes.byref(flop), stream.cuda_stream))
            e1.record(stream)
            e1.synchronize()
            if rep:
                best = max(best, flop.value / (e0.elapsed_time(e1) * 1e-3) / 1e12)
    return best, clk.summary()["sm_mhz"]


def cpu_oracle_rate(y, iters, threads=None):
    """Oracle port (fp64 C, OpenMP) on a truncated 512^2 solve: Mpixel*iter/s, seconds, cores."""
    from oracle import cpu as orc
    orc.build()
    if threads:
        orc.set_num_threads(threads)
    m = orc.read_foe(os.path.join(REPO, "paper_1609_05722_b200", "assets", "foe_a.foe"))
    v = orc.anscombe_forward(y)
    lam = 0.6075  # select_lambda(1, transform, quadratic), lambda_table.json
    t0 = time.perf_counter()
    u, tr = orc.ipiano_foe(v, v, m, lam, "quadratic", max_iters=iters, rel_tol=0.0)
    orc.anscombe_inverse_exact_unbiased(u)
    dt = time.perf_counter() - t0
    return y.size * len(tr.F) / dt / 1e6, dt, orc.num_threads(), len(tr.F)


def reference_python_rate(y, k_lo=3, k_hi=13):
    """The reference itself (foepoisson from baseline/_ref, Python + cv2, all host threads) on the cfg2
    counts through its public denoise(), solver_budget patched to k iterations: steady Mpixel*iter/s
    from t(k_hi) - t(k_lo) (the iteration-0 backtracking climb cancels).  None if not installed."""
    ref_dir = os.path.join(REPO, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref_dir, "foepoisson")):
        return None
    if ref_dir not in sys.path:
        sys.path.insert(0, ref_dir)
    import cv2
    cv2.setNumThreads(os.cpu_count() or 1)
    from foepoisson import fileio, pipeline, solver
    model = fileio.load_packaged_model("foe_a")
    req = pipeline.DenoiseRequest(noisy=y, peak=PEAK, model=model, variant="transform", force_branch="quadratic")
    orig = pipeline.solver_budget
    times = {}
    try:
        for k in (k_lo, k_hi):
            pipeline.solver_budget = lambda peak, overrides=None, k=k: solver.SolverConfig(max_iters=k, rel_tol=0.0)
            t0 = time.perf_counter()
            r = pipeline.denoise(req)
            times[k] = time.perf_counter() - t0
            assert len(r.trace) == k
    finally:
        pipeline.solver_budget = orig
    rate = y.size * (k_hi - k_lo) / (times[k_hi] - times[k_lo]) / 1e6
    return {"value": rate, "unit": "Mpixel*iter/s", "cores": cv2.getNumThreads(), "kind": "reference",
            "sample": f"foepoisson (baseline/_ref, Python + cv2 {cv2.__version__}, cv2 threads "
                      f"{cv2.getNumThreads()}) public denoise() on the cfg2 counts, solver_budget patched: "
                      f"({k_hi} - {k_lo}) accepted iterations / (t({k_hi}) - t({k_lo})) = "
                      f"{times[k_hi]:.2f} s - {times[k_lo]:.2f} s; steady rate, iteration-0 climb excluded",
            "cpu_model": cpu_model(), "os_cpu_count": os.cpu_count()}


def run_reference(args, rank, world):
    """--impl reference: the CPU oracle port on the box's host cores (rank 0 only), one full 150-iteration
    cfg2 solve per timed step -- the same workload and config dict as the GPU arm."""
    if rank != 0:
        return
    from paper_1609_05722_b200.synth import make_counts
    _, y = make_counts(H, W, 0, PEAK)
    for _ in range(args.warmup):
        cpu_oracle_rate(y, 3)  # untimed warm-up: thread pool, page faults (a 3-iteration solve)
    iters, secs = 0, 0.0
    for _ in range(args.steps):
        _, dt, cores, n = cpu_oracle_rate(y, args.ref_iters)
        iters += n
        secs += dt
    value = y.size * iters / secs / 1e6
    sample = (f"512x512 cfg2 full solve, {args.ref_iters} accepted iterations per step (fp64 C oracle port of the "
              f"reference, OpenMP {cores} threads, {cpu_model()})")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "Mpixel*iter/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * secs / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_for(world),
            "cpu_baseline": {"value": value, "unit": "Mpixel*iter/s", "cores": cores, "kind": "port", "sample": sample},
            "e2e": {"value": value, "unit": "Mpixel*iter/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def scaling_roofline(args, fp, model, cfg0, world, seeds):
    """The trial pass of configs 4 / 5 on this rank's share (config 4: its images as one batch; config 5:
    the whole 8192^2 image on one device when N = 1, else this rank's band is not a solve workspace and
    the line carries the N = 1 figure only): CUDA-event time of back-to-back passes on a solved state,
    achieved = 2,400 algorithmic FLOP x pixels in the launch / pass time, against the FFMA probe."""
    import torch

    from paper_1609_05722_b200 import _lib
    from paper_1609_05722_b200.anscombe import forward_device
    from paper_1609_05722_b200.synth import make_counts
    if args.config == 5 and world > 1:
        return None
    L = _lib.lib()
    if args.config == 4:
        peaks = [[0.5, 1.0, 2.0, 4.0][s % 4] for s in seeds]
        y = torch.from_numpy(np.stack([make_counts(H, W, s, p)[1] for s, p in zip(seeds, peaks)])).cuda()
        B, HH, WW = len(seeds), H, W
        lams = [fp.select_lambda(p, "transform", force_branch="quadratic") for p in peaks]
    else:
        _, yy = make_counts(8192, 8192, 0, 2.0)
        y = torch.from_numpy(yy).cuda()[None]
        B, HH, WW = 1, 8192, 8192
        lams = [fp.select_lambda(2.0, "transform", force_branch="quadratic")]
    v = forward_device(y.double() if y.dtype != torch.float64 else y)
    res = fp.solve_device(model, v, v, lams, "quadratic", 3, cfg0, raise_on_failure=False)  # a state to time on
    ws, stream = res._workspace, torch.cuda.current_stream()
    reps = 10
    _lib.check(L.foe_bench_trial_pass(res._bank.handle, B, HH, WW, res._cap, 2, ws.data_ptr(), ws.numel(),
                                      stream.cuda_stream))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    _lib.check(L.foe_bench_trial_pass(res._bank.handle, B, HH, WW, res._cap, reps, ws.data_ptr(), ws.numel(),
                                      stream.cuda_stream))
    e1.record(stream)
    e1.synchronize()
    pass_ms = e0.elapsed_time(e1) / reps
    peak, clk = measure_ffma_peak(L, torch.device("cuda"), torch.cuda.current_device())
    flop = ALG_FLOP_PER_PX_IT * B * HH * WW
    achieved = flop / (pass_ms * 1e-3) / 1e12
    return {"bound": "fp32", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
            "traffic": None, "kernel": "k_pass_tc<24,TRIAL,SYM>", "pass_ms": pass_ms, "flop_per_launch": flop,
            "launch": f"{B} x {HH}x{WW} per launch",
            "peak_source": f"measured FFMA probe (SM clock {clk} MHz); achieved = 2400 FLOP x pixels / pass time"}


def run_scaling_config(args, rank, local_rank, world):
    """Configs 4 (batch sharding) and 5 (row bands): strong scaling, device-timed, max over ranks."""
    import torch
    import torch.distributed as dist

    import paper_1609_05722_b200 as fp
    from paper_1609_05722_b200 import bands
    from paper_1609_05722_b200.anscombe import forward_device, inverse_exact_unbiased_device
    from paper_1609_05722_b200.synth import make_counts

    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    model = fp.load_packaged_model("foe_a")
    cfg0 = fp.SolverConfig(rel_tol=0.0)
    stream = torch.cuda.current_stream()
    if args.config == 4:
        sl = bands.shard_batch(args.batch, rank, world)
        seeds = list(range(args.batch))[sl]
        peaks = [[0.5, 1.0, 2.0, 4.0][s % 4] for s in seeds]
        ys = torch.from_numpy(np.stack([make_counts(H, W, s, p)[1] for s, p in zip(seeds, peaks)])).cuda()

        def step():
            img, traces, _, _ = fp.denoise_batch(ys, peaks, model, "transform", force_branch="quadratic",
                                                 solver=cfg0, return_device=True)
            return sum(len(t) for t in traces) * H * W
        workload = f"cfg4: {args.batch} x 512x512, peaks cycling 0.5/1/2/4, quadratic, foe_a, 150 iters, " \
                   f"batch-sharded over {world} ranks (no collective)"
        dtag = "dp"
    else:
        HH = WW = 8192
        _, ty = bands.tile_grid(5, HH, WW)
        t0, t1 = bands.partition_tile_rows(ty, world)[rank]
        lam = fp.select_lambda(2.0, "transform", force_branch="quadratic")
        band = bands.Band(model, 1, HH, WW, t0, t1, 150, cfg0)
        l0, l1 = band.local_rows
        _, y = make_counts(HH, WW, 0, 2.0)
        v_local = forward_device(torch.from_numpy(np.ascontiguousarray(y[l0:l1])).cuda())[None]
        ex = bands.DistExchange() if world > 1 else bands.LocalExchange()

        def step():
            res = bands.solve_bands([band], ex, [v_local], [v_local], lam, "quadratic", 150)
            inverse_exact_unbiased_device(res[0][0])
            return len(res[0][1][0]) * HH * WW / world
        workload = f"cfg5: 8192x8192, peak 2, quadratic, foe_a, 150 iters, {world} row band(s), 4-row halo " \
                   f"+ per-pass partials all-gather"
        dtag = "bands"
    out = None
    for _ in range(args.warmup):
        # the previous step's outputs stay alive while the next one runs, as in the timed loop, so the
        # caching allocator has grown to its steady state before timing starts
        out = step()  # noqa: F841
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    total_ms, px_it = 0.0, 0.0
    with ClockSampler(local_rank) as clk:
        for _ in range(args.steps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            px_it += step()
            e1.record(stream)
            e1.synchronize()
            total_ms += e0.elapsed_time(e1)
            if os.environ.get("FOE_BENCH_VERBOSE"):
                print(f"step {e0.elapsed_time(e1):.3f} ms", file=sys.stderr)
    t = torch.tensor([total_ms, px_it], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.barrier()
        tmax = t.clone()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        total_ms, px_it = float(tmax[0]), float(t[1])
    value = px_it / (total_ms * 1e-3) / 1e6
    roof = None
    if rank == 0:
        roof = scaling_roofline(args, fp, model, cfg0, world, seeds if args.config == 4 else None)
    if rank == 0:
        print(json.dumps({"metric": METRIC, "value": value, "unit": "Mpixel*iter/s", "n_gpus": world,
                          "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
                          "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "fp32",
                          "data": "synthetic", "config": {"workload": workload, "parallelism": f"{dtag}{world}"},
                          "roofline": roof, "clocks": clk.summary()}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-iters", type=int, default=150, help="--impl reference: iterations per step (the full solve)")
    ap.add_argument("--cpu-iters", type=int, default=150, help="cpu_baseline sample: the full 150-iteration solve")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-fallback", action="store_true", help="skip the 48x7x7 fallback-bank line")
    ap.add_argument("--pass-reps", type=int, default=100)
    ap.add_argument("--config", type=int, default=2, choices=[2, 4, 5],
                    help="2: 512^2 single image (headline); 4: 256 x 512^2 batch sharded over ranks; "
                         "5: one 8192^2 image split into row bands over ranks")
    ap.add_argument("--batch", type=int, default=256, help="config 4: total images (strong scaling)")
    args = ap.parse_args()
    rank, local_rank, world = dist_env()
    args.warmup = max(args.warmup, 0)

    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if args.config in (4, 5):
        run_scaling_config(args, rank, local_rank, world)
        return

    import torch
    import torch.distributed as dist

    import paper_1609_05722_b200 as fp
    from paper_1609_05722_b200 import _lib
    from paper_1609_05722_b200.anscombe import forward_device, inverse_exact_unbiased_device
    from paper_1609_05722_b200.synth import make_counts

    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    dev = torch.device("cuda", local_rank)
    model = fp.load_packaged_model("foe_a")
    clean, y = make_counts(H, W, rank, PEAK)
    y_dev = torch.from_numpy(y).to(dev)
    lam = fp.select_lambda(PEAK, "transform", force_branch="quadratic")
    # the reference's own budget (150 iterations at peak < 5) as a fixed count: rel_tol = 0
    cfg = fp.solver_budget(PEAK, fp.SolverConfig(rel_tol=0.0))
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 * 2 ** 20, dtype=torch.uint8, device=dev)

    def step():
        v = forward_device(y_dev)
        res = fp.solve_device(model, v, v, lam, "quadratic", cfg.max_iters, cfg)
        x = inverse_exact_unbiased_device(res.u)
        return res, x

    L = _lib.lib()
    # the FFMA peak probe (~0.1 s of full-chip work) also brings an idle GPU up to its boost clock
    # before the warm-up steps
    fp32_peak_tflops, ffma_clk = measure_ffma_peak(L, dev, local_rank)
    out = None
    for _ in range(args.warmup):
        # the previous step's outputs stay alive while the next one runs, as in the timed loop, so the
        # caching allocator has grown to its steady state before timing starts
        out = step()  # noqa: F841
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = L.foe_kernel_launch_count()
    total_ms, iters, trials = 0.0, 0, 0
    with ClockSampler(local_rank) as clk:
        for _ in range(args.steps):
            flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            res, x = step()
            e1.record(stream)
            e1.synchronize()
            total_ms += e0.elapsed_time(e1)
            if os.environ.get("FOE_BENCH_VERBOSE"):
                print(f"step {e0.elapsed_time(e1):.3f} ms", file=sys.stderr)
            iters += len(res.traces[0])
            trials += res.traces[0].n_trials
    torch.cuda.synchronize()
    launches = L.foe_kernel_launch_count() - launches0
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.barrier()
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_per_step = float(t.item()) / args.steps
    px_it_per_step = H * W * iters / args.steps
    value = world * px_it_per_step / (ms_per_step * 1e-3) / 1e6

    # dominant kernel: the fused trial pass, timed back to back on the solved state
    ws = res._workspace
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    _lib.check(L.foe_bench_trial_pass(res._bank.handle, 1, H, W, res._cap, 5, ws.data_ptr(), ws.numel(),
                                      stream.cuda_stream))
    e0.record(stream)
    _lib.check(L.foe_bench_trial_pass(res._bank.handle, 1, H, W, res._cap, args.pass_reps, ws.data_ptr(),
                                      ws.numel(), stream.cuda_stream))
    e1.record(stream)
    e1.synchronize()
    pass_ms = e0.elapsed_time(e1) / args.pass_reps
    props = torch.cuda.get_device_properties(dev)
    sm_count = props.multi_processor_count
    peak_clock = clk.max_mhz or 1965.0
    fp32_nominal_tflops = sm_count * 128 * 2 * peak_clock * 1e6 / 1e12
    alg_flop_pass = ALG_FLOP_PER_PX_IT * H * W
    achieved = alg_flop_pass / (pass_ms * 1e-3) / 1e12
    use_tc = bool(L.foe_pass_uses_tensor_cores(K, N_FILT))
    traffic = pass_traffic("k_pass_tc<24, 1, 1>" if use_tc else "k_pass<5, 1, 1>")
    tensor = None
    if use_tc:
        # executed tcgen05 work of one trial pass: per 128-pixel block 2 x 7 forward (u, du) kind::tf32 MMAs of
        # 128 x 48 x 8 (both 3xTF32 sweeps merged along N) + 6 + 4 adjoint MMAs of 128 x 32 x 8, 18 blocks per tile
        ctas = -(-H // 32) * -(-W // 60)
        mma_flop = ctas * 18 * (14 * 48 + 10 * 32) * 2 * 128 * 8
        tf32_peak = PEAKS.get("bf16_tflops", 2 * 1125.0) / 2
        tensor = {"executed_tflops": mma_flop / (pass_ms * 1e-3) / 1e12, "mma_flop_per_launch": mma_flop,
                  "peak_tf32_tflops": tf32_peak, "frac": mma_flop / (pass_ms * 1e-3) / 1e12 / tf32_peak,
                  "peak_source": "dense tf32 = 1/2 of MEASURED_PEAKS.json bf16_tflops (burst)"}
    solve_frac = value * 1e6 * ALG_FLOP_PER_PX_IT / (world * fp32_peak_tflops * 1e12)

    # end to end through the public API with host buffers (H2D counts, D2H image + transformed)
    e2e_ms = []
    n_e2e_warm = 3  # first calls grow the allocator cache and the pinned staging buffers
    for i in range(max(1, min(args.steps, 5)) + n_e2e_warm):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = fp.denoise(fp.DenoiseRequest(noisy=y, peak=PEAK, model=model, variant="transform",
                                          force_branch="quadratic"), cfg)
        dt = time.perf_counter() - t0
        if i >= n_e2e_warm:
            e2e_ms.append(dt * 1e3)
    if os.environ.get("BENCH_DEBUG_E2E"):
        print("e2e samples (ms):", [round(t, 3) for t in e2e_ms], file=sys.stderr)
    e2e_iters = len(r.trace)
    e2e_t = torch.tensor([statistics.median(e2e_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_value = world * H * W * e2e_iters / (float(e2e_t.item()) * 1e-3) / 1e6

    # the same workload with the BASELINE 48 x 7 x 7 fallback bank ("all configs
    # repeat with the fallback bank"): 4 N k^2 = 9,408 algorithmic FLOP per pixel-iteration
    fallback = None
    if rank == 0 and not args.no_fallback:
        fallback = bench_fallback_bank(fp, _lib, L, y_dev, lam, cfg, stream, fp32_peak_tflops, H, W)

    cpu = cpu_ref = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rate, secs, cores, _ = cpu_oracle_rate(y, args.cpu_iters)
        cpu = {"value": rate, "unit": "Mpixel*iter/s", "cores": cores, "kind": "port",
               "sample": f"512x512 cfg2 full solve, {args.cpu_iters} iterations ({secs:.1f} s, fp64 C oracle port, "
                         f"{cpu_model()})"}
        try:
            cpu_ref = reference_python_rate(y)
        except Exception as exc:  # reported, not fatal: the reference's own deps live outside this repo
            cpu_ref = {"unavailable": f"{type(exc).__name__}: {exc}"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "Mpixel*iter/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "fp32", "data": "synthetic",
                "config": config_for(world),
                "denoise_ms_512": ms_per_step, "iterations_per_step": iters / args.steps,
                "trials_per_step": trials / args.steps,
                "algorithmic_fp32_frac": solve_frac,
                "roofline": {"bound": "fp32", "achieved": achieved, "peak": fp32_peak_tflops, "unit": "TFLOP/s",
                             "frac": achieved / fp32_peak_tflops, "traffic": traffic,
                             "kernel": ("k_pass_tc<24,TRIAL,SYM> (fused trial pass, tcgen05 3xTF32 implicit GEMMs)"
                                        if use_tc else "k_pass<5,TRIAL,SYM> (fused trial pass, FFMA)"),
                             "pass_ms": pass_ms, "tensor": tensor,
                             "flop_per_launch": alg_flop_pass,
                             "peak_source": "measured: FFMA probe k_ffma_peak (independent FMA chains on every SM, "
                                            f"CUDA events; SM clock {ffma_clk} MHz during the probe); nominal "
                                            f"{sm_count} SMs x 128 lanes x 2 x {peak_clock} MHz = "
                                            f"{fp32_nominal_tflops:.1f} TFLOP/s (MEASURED_PEAKS.json has no FP32 "
                                            "figure); achieved = algorithmic fp32 flops (forward + adjoint, 2400 "
                                            "per pixel) / pass time"},
                "e2e": {"value": e2e_value, "unit": "Mpixel*iter/s", "ms_per_denoise": float(e2e_t.item()),
                        # the request's validation pass stages the counts as exact floats in page-locked
                        # memory (_host.stage_counts): the H2D copy moves 4 bytes per pixel
                        "h2d_bytes_per_step": int(y.size * 4),
                        "d2h_bytes_per_step": int(H * W * (8 + 8))},  # image (f64) + transformed (f64, cast on the device)
                "gpu_launches": launches, "gpu_launches_per_step": launches / args.steps,
                "clocks": clk.summary(),
                "fallback_48x7": fallback,
                "cpu_baseline": cpu,
                "cpu_baseline_reference": cpu_ref}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
