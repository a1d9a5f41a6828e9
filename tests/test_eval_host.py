"""Evaluation-grid host logic and the scoring oracle vs the reference's golden vectors (CPU)."""
import numpy as np
import pytest

from oracle import cpu as orc
from paper_1609_05722_b200 import evaluate as ev


def test_oracle_metrics_vs_reference_golden(golden):
    """oracle psnr / mssim (metrics.py:30-102 restated) reproduce the reference's scores."""
    g = golden("metrics")
    for i in range(4):
        peak, ref_psnr, ref_mssim = g[f"m{i}_ref"]
        p, m = orc.score_denoised(g[f"m{i}_xhat"], g[f"m{i}_g"], peak)
        assert abs(p - ref_psnr) <= 1e-10 * abs(ref_psnr)
        assert abs(m - ref_mssim) <= 1e-12


def test_job_seed_matches_reference(golden):
    """benchmark.py:67-70: identical hash-derived seeds (order-independent jobs)."""
    g = golden("bench_grid")
    seeds = [ev.job_seed(n, p, v, 7) for n in ("a", "syn40x36s1") for p in (0.5, 40.0) for v in ("transform", "direct")]
    assert seeds == [int(s) for s in g["seeds"]]


def test_scale_to_peak_and_validation():
    x = np.array([[0.0, 0.5], [1.0, 0.25]])
    np.testing.assert_array_equal(ev.scale_to_peak(x, 4.0), x * 4.0)
    with pytest.raises(ValueError):
        ev.scale_to_peak(np.zeros((2, 2)), 1.0)
    with pytest.raises(ValueError):
        ev.scale_to_peak(x, 0.0)


def test_spec_validation_and_image_names():
    with pytest.raises(ValueError):
        ev.BenchmarkSpec(images=(), peaks=(1.0,), variants=("transform",))
    with pytest.raises(ValueError):
        ev.BenchmarkSpec(images=("syn8x8s0",), peaks=(1.0,), variants=("direct",))
    with pytest.raises(ValueError):
        ev.BenchmarkSpec(images=("syn8x8s0",), peaks=(-1.0,), variants=("transform",), transform_model=object())
    assert ev.synthetic_eval_image("syn12x20s3").shape == (12, 20)
    with pytest.raises(ValueError):
        ev.synthetic_eval_image("cameraman")


def test_csv_and_averages_format():
    rows = [ev.BenchmarkRow("a", 1.0, "transform", 20.5, 0.5, "transform_idiv", 0.65, 11),
            ev.BenchmarkRow("b", 1.0, "transform", 21.5, 0.7, "transform_idiv", 0.65, 12)]
    text = ev.format_csv_report(rows)
    assert text.splitlines()[0] == "image,peak,variant,psnr_db,mssim,branch,lambda,seed"
    assert text.splitlines()[1] == "a,1,transform,20.5,0.5,transform_idiv,0.65000000000000002,11"
    (avg,) = ev.average_rows(rows)
    assert avg.image == "average" and avg.psnr_db == 21.0 and abs(avg.mssim - 0.6) < 1e-15


def test_cli_parser_rejects_unknown_variant(capsys):
    from paper_1609_05722_b200.__main__ import main
    with pytest.raises(SystemExit):
        main(["denoise", "a.npy", "b.npy", "--variant", "nope"])
