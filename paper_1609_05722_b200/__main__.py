"""Command-line shim over the device path (reference cli.py:63-85 `denoise`, benchmark.py grid).

    python -m paper_1609_05722_b200 denoise INPUT.npy OUTPUT.npy [--peak P] [--variant transform]
                                            [--model FILE.foe] [--lam L] [--c C] [--trace TRACE.csv]
    python -m paper_1609_05722_b200 benchmark --images syn256x256s0 ... --peaks 1 2 4
                                              [--variants transform ...] [--csv OUT.csv]

Raster I/O of the reference CLI is out of scope; counts and images are
.npy arrays.  Exit codes follow cli.py:247-257: 0 ok, 1 invalid input, 2 numerical failure.
"""
from __future__ import annotations

import argparse
import sys

import numpy as np

EXIT_OK, EXIT_INVALID, EXIT_NUMERICAL = 0, 1, 2


def _estimate_peak(noisy: np.ndarray) -> float:
    return float(max(np.max(noisy), 1e-3))


def cmd_denoise(args) -> int:
    from . import DenoiseRequest, denoise, load_model, load_packaged_model
    model = load_model(args.model) if args.model else load_packaged_model(
        "foe_s" if args.variant == "direct" else "foe_a")
    noisy = np.load(args.input).astype(np.float64)
    peak = args.peak if args.peak is not None else _estimate_peak(noisy)
    req = DenoiseRequest(noisy=noisy, peak=peak, model=model, variant=args.variant,
                         lam=args.lam if args.lam is not None else "auto", zero_offset_c=args.c)
    out = denoise(req)
    np.save(args.output, out.image)
    print(f"branch: {out.branch}")
    print(f"lambda: {out.lam:.17g}")
    if args.trace:
        out.trace.save_csv(args.trace)
        print(f"trace: {args.trace}")
    print(f"wrote {args.output}")
    return EXIT_OK


def cmd_benchmark(args) -> int:
    from . import load_packaged_model
    from .evaluate import BenchmarkSpec, format_csv_report, run_benchmark
    spec = BenchmarkSpec(images=tuple(args.images), peaks=tuple(args.peaks), variants=tuple(args.variants),
                         transform_model=load_packaged_model("foe_a"), direct_model=load_packaged_model("foe_s"),
                         base_seed=args.seed)
    rows = run_benchmark(spec)
    text = format_csv_report(rows)
    if args.csv:
        with open(args.csv, "w") as fh:
            fh.write(text)
        print(f"wrote {args.csv} ({len(rows)} rows)")
    else:
        sys.stdout.write(text)
    return EXIT_OK


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_1609_05722_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    d = sub.add_parser("denoise", help="denoise one count image (.npy)")
    d.add_argument("input")
    d.add_argument("output")
    d.add_argument("--peak", type=float)
    d.add_argument("--variant", default="transform", choices=["transform", "transform_binned", "direct"])
    d.add_argument("--model")
    d.add_argument("--lam", type=float)
    d.add_argument("--c", type=float, default=0.1)
    d.add_argument("--trace")
    b = sub.add_parser("benchmark", help="evaluation grid on the device (CSV rows as benchmark.py)")
    b.add_argument("--images", nargs="+", default=["syn256x256s0", "syn256x256s1"])
    b.add_argument("--peaks", nargs="+", type=float, default=[0.5, 1.0, 2.0, 4.0])
    b.add_argument("--variants", nargs="+", default=["transform"])
    b.add_argument("--seed", type=int, default=0)
    b.add_argument("--csv")
    args = ap.parse_args(argv)
    from .solver import NumericalFailure
    try:
        return cmd_denoise(args) if args.cmd == "denoise" else cmd_benchmark(args)
    except NumericalFailure as e:
        print(f"numerical failure: {e}", file=sys.stderr)
        return EXIT_NUMERICAL
    except (ValueError, OSError) as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_INVALID


if __name__ == "__main__":
    sys.exit(main())
