"""Command-line shim over the device path (reference cli.py:63-85 `denoise`, benchmark.py grid).

    python -m paper_1609_05722_b200 denoise INPUT.npy OUTPUT.npy [--peak P] [--variant transform]
                                            [--model FILE.foe] [--lam L] [--c C] [--trace TRACE.csv]
    python -m paper_1609_05722_b200 benchmark --images syn256x256s0 ... --peaks 1 2 4
                                              [--variants transform ...] [--csv OUT.csv]

Raster I/O of the reference CLI is out of scope; counts and images are
.npy arrays.  Exit codes are the reference's (cli.py:1-5, 28-31, 244-257): 0 success, 1 usage error
(bad flags or invalid arguments), 2 data error (unreadable or malformed files), 3 numerical failure.
Without --peak the peak is estimated as the reference does (estimate_peak, pipeline.py:247-254:
max of the 3x3 median filter), on the device.
"""
from __future__ import annotations

import argparse
import sys

import numpy as np

EXIT_OK, EXIT_USAGE, EXIT_DATA, EXIT_NUMERIC = 0, 1, 2, 3


class _Parser(argparse.ArgumentParser):
    """argparse exits with 2 on bad flags; the contract reserves 2 for data errors (cli.py:37-43)."""

    def error(self, message):
        self.print_usage(sys.stderr)
        self.exit(EXIT_USAGE, f"{self.prog}: error: {message}\n")


def _read_counts(path: str) -> np.ndarray:
    from .fileio import FileFormatError
    try:
        arr = np.load(path, allow_pickle=False)
    except (FileNotFoundError, OSError):
        raise
    except ValueError as exc:  # not an .npy file / pickled payload
        raise FileFormatError(f"{path}: {exc}") from exc
    if not isinstance(arr, np.ndarray) or arr.ndim != 2:
        raise FileFormatError(f"{path}: expected a 2-d array")
    return arr.astype(np.float64)


def cmd_denoise(args) -> int:
    from . import DenoiseRequest, denoise, load_model, load_packaged_model
    from .pipeline import estimate_peak
    model = load_model(args.model) if args.model else load_packaged_model(
        "foe_s" if args.variant == "direct" else "foe_a")
    noisy = _read_counts(args.input)
    if args.peak is not None:
        peak = args.peak
    else:
        peak = estimate_peak(noisy)
        print(f"peak estimated from input: {peak:g}")
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


def build_parser() -> argparse.ArgumentParser:
    ap = _Parser(prog="python -m paper_1609_05722_b200")
    sub = ap.add_subparsers(dest="cmd", required=True, parser_class=_Parser)
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
    return ap


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    from .fileio import FileFormatError
    from .solver import NumericalFailure
    try:
        return cmd_denoise(args) if args.cmd == "denoise" else cmd_benchmark(args)
    except (FileFormatError, FileNotFoundError, OSError) as err:  # cli.py:247-249
        print(f"error: {err}", file=sys.stderr)
        return EXIT_DATA
    except NumericalFailure as err:  # cli.py:250-252
        print(f"numerical failure: {err}", file=sys.stderr)
        return EXIT_NUMERIC
    except ValueError as err:  # cli.py:253-255
        print(f"error: {err}", file=sys.stderr)
        return EXIT_USAGE


if __name__ == "__main__":
    sys.exit(main())
