"""GPU tests of the public API around the solve: the reference's own edge cases run through the
CUDA path (test_pipeline.py, test_solver.py), the CLI's peak estimate and exit codes, and concurrent
callers (benchmark.py:117-121 fans jobs out over a thread pool)."""

import threading

import numpy as np
import pytest

import paper_1609_05722_b200 as fp
from paper_1609_05722_b200.synth import make_counts

pytestmark = pytest.mark.gpu


def _model(rng, n_filters, m, domain_tag):
    """The reference tests' random_model (test_prior.py:18-23): DCT betas ~ N(0, 0.5), weights U[0.5, 2]."""
    basis = fp.dct_basis(m)
    return fp.FoEModel(basis=basis, betas=rng.normal(scale=0.5, size=(n_filters, basis.n_atoms)),
                       weights=rng.uniform(0.5, 2.0, size=n_filters), domain_tag=domain_tag)


def _noisy(rng, shape=(16, 16), peak=8.0):
    """The reference tests' make_noisy (test_pipeline.py:28-31)."""
    from paper_1609_05722_b200.evaluate import scale_to_peak
    from paper_1609_05722_b200.synth import sample_poisson
    clean = rng.random(shape) * 0.8 + 0.2
    return sample_poisson(scale_to_peak(clean, peak), seed=int(rng.integers(2 ** 31)))


# ---- test_pipeline.py:132-156 (direct variant) --------------------------------------------------------

def test_direct_huge_lambda_returns_observation():
    rng = np.random.default_rng(42)
    model = _model(rng, 3, 3, "original")
    y = np.full((16, 16), 7.0)
    out = fp.denoise_direct(fp.DenoiseRequest(noisy=y, peak=7.0, model=model, variant="direct", lam=1e8))
    np.testing.assert_allclose(out.image, y, rtol=1e-4)


def test_direct_zero_region_stays_zero_without_offset():
    rng = np.random.default_rng(42)
    model = _model(rng, 3, 3, "original")
    y = _noisy(rng, (64, 64), 10.0)
    y[12:52, 12:52] = 0.0
    out = fp.denoise_direct(fp.DenoiseRequest(noisy=y, peak=10.0, model=model, variant="direct", lam=0.5,
                                              zero_offset_c=0.0))
    assert np.all(out.image[27:37, 27:37] == 0.0)
    out = fp.denoise_direct(fp.DenoiseRequest(noisy=y, peak=10.0, model=model, variant="direct", lam=0.5,
                                              zero_offset_c=0.1))
    assert np.all(out.image[27:37, 27:37] > 0.0)


def test_direct_output_nonnegative_and_energy_not_increased():
    rng = np.random.default_rng(42)
    model = _model(rng, 3, 3, "original")
    y = _noisy(rng, (32, 32), 40.0)
    lam = 0.5
    out = fp.denoise_direct(fp.DenoiseRequest(noisy=y, peak=40.0, model=model, variant="direct", lam=lam))
    assert np.all(out.image >= 0.0)
    obs = np.where(y == 0, 0.1, y)

    def total(x):
        pos = obs > 0
        data = float(np.sum(x)) - float(np.sum(obs[pos] * np.log(x[pos])))
        return fp.foe_energy(x, model) + lam * data

    assert total(out.image) <= total(obs) + 1e-6 * abs(total(obs))  # fp32 state: relative slack


# ---- test_pipeline.py:192-226 (transform variant) ----------------------------------------------------

def test_transform_huge_lambda_inverts_untouched_transform():
    from oracle import cpu as orc
    rng = np.random.default_rng(7)
    model = _model(rng, 3, 3, "anscombe")
    y = _noisy(rng, peak=40.0)
    out = fp.denoise_transform(fp.DenoiseRequest(noisy=y, peak=40.0, model=model, variant="transform", lam=1e12))
    expect = orc.anscombe_inverse_exact_unbiased(orc.anscombe_forward(y))
    # the fp32 transform-domain state bounds the agreement (reference test: 1e-6 in fp64)
    np.testing.assert_allclose(out.image, expect, rtol=2e-6, atol=1e-5)


def test_transform_branch_threshold_and_transformed_exposed():
    rng = np.random.default_rng(7)
    model = _model(rng, 3, 3, "anscombe")
    y = _noisy(rng, peak=8.0)
    quad = fp.denoise_transform(fp.DenoiseRequest(noisy=y, peak=5.0, model=model, variant="transform", lam=1.0))
    idiv = fp.denoise_transform(fp.DenoiseRequest(noisy=y, peak=4.99, model=model, variant="transform", lam=1.0))
    assert quad.branch == "transform_quadratic" and idiv.branch == "transform_idiv"
    from paper_1609_05722_b200 import anscombe
    np.testing.assert_allclose(quad.image, anscombe.anscombe_inverse_exact_unbiased(quad.transformed), rtol=1e-12)


def test_transform_output_nonnegative_with_zero_counts():
    rng = np.random.default_rng(7)
    model = _model(rng, 3, 3, "anscombe")
    y = _noisy(rng, peak=0.5)
    assert np.any(y == 0)
    out = fp.denoise_transform(fp.DenoiseRequest(noisy=y, peak=0.5, model=model, variant="transform", lam=1.0))
    assert np.all(out.image >= 0.0) and np.all(np.isfinite(out.image))


# ---- test_pipeline.py:251-268 (binned variant) -------------------------------------------------------

def test_binned_factor_one_degenerates_to_transform():
    rng = np.random.default_rng(13)
    model = _model(rng, 3, 3, "anscombe")
    y = _noisy(rng, peak=8.0)
    binned = fp.denoise(fp.DenoiseRequest(noisy=y, peak=8.0, model=model, variant="transform_binned", lam=1.0,
                                          bin_factor=1))
    plain = fp.denoise(fp.DenoiseRequest(noisy=y, peak=8.0, model=model, variant="transform", lam=1.0))
    np.testing.assert_array_equal(binned.image, plain.image)


def test_binned_restores_input_shape_for_awkward_dims():
    rng = np.random.default_rng(13)
    model = _model(rng, 3, 3, "anscombe")
    y = _noisy(rng, (17, 13), 4.0)
    out = fp.denoise(fp.DenoiseRequest(noisy=y, peak=4.0, model=model, variant="transform_binned", lam=1.0))
    assert out.image.shape == (17, 13) and np.all(out.image >= 0.0)
    low = fp.denoise(fp.DenoiseRequest(noisy=_noisy(rng, (18, 18), 4.0), peak=0.5, model=model,
                                       variant="transform_binned", lam=1.0))
    assert low.branch == "transform_idiv" and low.peak_used == pytest.approx(4.5)


# ---- test_solver.py:231-248 -------------------------------------------------------------------------

def test_rel_tol_stops_early():
    model = fp.load_packaged_model("foe_a")
    _, y = make_counts(64, 64, 3, 4.0)
    r = fp.denoise(fp.DenoiseRequest(noisy=y, peak=4.0, model=model, variant="transform", force_branch="quadratic"),
                   fp.SolverConfig(rel_tol=1e-3))
    assert 0 < len(r.trace) < 150
    # the stop test of solver.py:173: the last accepted step is below rel_tol * |u_prev|
    assert r.trace.step_norm[-1] < 1e-3 * np.linalg.norm(r.transformed) * 1.01


def test_nonfinite_energy_aborts_with_trace():
    """A non-finite smooth energy at iteration 0 raises NumericalFailure carrying the (empty) trace
    (solver.py:142-144): an iterate whose responses overflow fp32 (K u ~ 1e30 -> z^2 = inf)."""
    import torch
    model = fp.load_packaged_model("foe_a")
    u0 = torch.zeros((32, 32), dtype=torch.float32, device="cuda")
    u0[::2] = 3e30
    with pytest.raises(fp.NumericalFailure) as err:
        fp.solve_device(model, u0, u0, 1.0, "quadratic", 5, fp.SolverConfig(rel_tol=0.0))
    assert isinstance(err.value.trace, fp.SolverTrace) and len(err.value.trace) == 0


# ---- CLI: estimate_peak (pipeline.py:247-254) and the numerical exit code (cli.py:250-252) ------------

@pytest.mark.parametrize("shape", [(1, 1), (1, 9), (2, 2), (3, 5), (37, 64), (256, 300)])
def test_estimate_peak_matches_scipy_median_filter(shape):
    from scipy.ndimage import median_filter
    rng = np.random.default_rng(shape[0] * 1000 + shape[1])
    y = rng.poisson(rng.uniform(0.5, 30.0, size=shape)).astype(np.float64)
    from paper_1609_05722_b200.pipeline import estimate_peak
    assert estimate_peak(y) == float(median_filter(y, size=3).max())
    z = rng.normal(size=shape)  # negative values too (the order-preserving max)
    assert estimate_peak(z) == float(median_filter(z, size=3).max())


def test_cli_estimates_peak_and_maps_numerical_failure(tmp_path, monkeypatch, capsys):
    from paper_1609_05722_b200 import pipeline
    from paper_1609_05722_b200.__main__ import EXIT_NUMERIC, EXIT_OK, main
    from scipy.ndimage import median_filter
    _, y = make_counts(40, 44, 5, 2.0)
    np.save(tmp_path / "in.npy", y)
    assert main(["denoise", str(tmp_path / "in.npy"), str(tmp_path / "out.npy")]) == EXIT_OK
    peak = float(median_filter(y, size=3).max())
    assert f"peak estimated from input: {peak:g}" in capsys.readouterr().out
    ref = fp.denoise(fp.DenoiseRequest(noisy=y, peak=peak, model=fp.load_packaged_model("foe_a"), variant="transform"))
    np.testing.assert_array_equal(np.load(tmp_path / "out.npy"), ref.image)
    stalled = fp.SolverConfig(lipschitz_init=1.0, max_lipschitz=1.5)
    monkeypatch.setattr(pipeline, "solver_budget", lambda p, o=None: stalled)
    assert main(["denoise", str(tmp_path / "in.npy"), str(tmp_path / "out.npy"), "--peak", "2"]) == EXIT_NUMERIC


# ---- concurrency ------------------------------------------------------------------------------------

def test_concurrent_denoise_calls_equal_serial_bitwise():
    """Four host threads calling denoise at once (each with its own staging buffers, workspace and loop
    graph) give exactly the serial results (benchmark.py:117-121 runs jobs concurrently)."""
    model = fp.load_packaged_model("foe_a")
    jobs = [(make_counts(96, 80, s, p)[1], p) for s, p in enumerate((0.5, 1.0, 2.0, 8.0))]
    reqs = [fp.DenoiseRequest(noisy=y, peak=p, model=model, variant="transform") for y, p in jobs]
    serial = [fp.denoise(r) for r in reqs]
    results, errors = [None] * len(reqs), []

    def run(k):
        try:
            for _ in range(3):
                results[k] = fp.denoise(reqs[k])
        except Exception as exc:  # surfaced below
            errors.append(exc)

    threads = [threading.Thread(target=run, args=(k,)) for k in range(len(reqs))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    for a, b in zip(serial, results):
        np.testing.assert_array_equal(a.image, b.image)
        assert a.trace.L == b.trace.L and a.trace.F == b.trace.F


def test_staged_upload_equals_plain_upload_bitwise():
    """The counts staged by the request's validation pass (float32 in page-locked memory) give exactly the result
    of the plain float64 upload, which a request falls back to once a later request has reused the staging buffer;
    counts too large for an exact float are never staged."""
    from paper_1609_05722_b200 import _host

    model = fp.load_packaged_model("foe_a")
    _, y = make_counts(96, 80, 3, 2.0)
    first = fp.DenoiseRequest(noisy=y, peak=2.0, model=model, variant="transform")
    assert first._staged is not None
    later = fp.DenoiseRequest(noisy=make_counts(96, 80, 4, 2.0)[1], peak=2.0, model=model, variant="transform")
    assert _host.upload_staged(first._staged, y.shape) is None  # superseded by `later`: plain upload
    plain = fp.denoise(first)
    fresh = fp.DenoiseRequest(noisy=y, peak=2.0, model=model, variant="transform")
    assert _host.upload_staged(fresh._staged, y.shape) is not None
    staged = fp.denoise(fresh)
    again = fp.denoise(fresh)  # the staged copy survives its own use
    np.testing.assert_array_equal(plain.image, staged.image)
    np.testing.assert_array_equal(plain.image, again.image)
    assert plain.trace.L == staged.trace.L and plain.trace.F == staged.trace.F
    assert later._staged is not None
    big = y.copy()
    big[0, 0] = 2.0 ** 24
    assert fp.DenoiseRequest(noisy=big, peak=2.0, model=model, variant="transform")._staged is None
