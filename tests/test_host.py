"""CPU-only tests: C-ABI exports, FOE 1 format, host-side pipeline rules (no GPU needed)."""

import ctypes
import os
import re

import numpy as np
import pytest

import paper_1609_05722_b200 as fp
from paper_1609_05722_b200 import _lib, pipeline
from oracle import cpu as orc
from tests.conftest import REPO


def test_library_builds_and_exports_every_header_symbol():
    _lib.build()
    header = open(os.path.join(REPO, "include", "foe_b200.h")).read()
    declared = set(re.findall(r"^(?:int|size_t|long long|const char \*)\s*(foe_[a-z0-9_]+)\(", header, re.M))
    assert declared == set(_lib.EXPORTED_SYMBOLS)
    so = ctypes.CDLL(_lib.LIB_PATH)
    for name in declared:
        assert hasattr(so, name), name
    assert _lib.lib().foe_abi_version() == 1


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_packaged_models():
    a = fp.load_packaged_model("foe_a")
    s = fp.load_packaged_model("foe_s")
    f = fp.load_packaged_model("foe_fallback48x7")
    assert (a.n_filters, a.basis.size, a.domain_tag, a.boundary) == (24, 5, "anscombe", "symmetric")
    assert (s.n_filters, s.basis.size, s.domain_tag) == (8, 3, "original")
    assert (f.n_filters, f.basis.size) == (48, 7)
    np.testing.assert_allclose(np.linalg.norm(f.betas, axis=1), 1.0, rtol=1e-12)


def test_model_round_trip_bit_exact(tmp_path):
    """fileio.py:33-48 promise (test_fileio.py:28-56)."""
    rng = np.random.default_rng(1)
    for m, bnd in ((3, "symmetric"), (5, "periodic"), (7, "symmetric")):
        basis = fp.dct_basis(m)
        model = fp.FoEModel(basis=basis, betas=rng.normal(size=(4, basis.n_atoms)),
                            weights=rng.uniform(0.1, 3, 4), domain_tag="anscombe", boundary=bnd)
        p = tmp_path / f"m{m}.foe"
        fp.save_model(p, model)
        back = fp.load_model(p)
        np.testing.assert_array_equal(back.betas, model.betas)
        np.testing.assert_array_equal(back.weights, model.weights)
        assert back.boundary == bnd and back.basis.name == f"dct{m}"


@pytest.mark.parametrize("text", ["FOE 2\n", "FOE 1\nanscombe 1 3 dct3\n", "FOE 1\nfoo 1 3 dct3 symmetric\n1 " +
                                  " ".join(["0"] * 8) + "\n", "FOE 1\nanscombe 1 3 dct5 symmetric\n1\n",
                                  "FOE 1\nanscombe 2 3 dct3 symmetric\n" + "1 " + " ".join(["0"] * 8) + "\n",
                                  "FOE 1\nanscombe 1 3 dct3 symmetric\n1 2 3\n"])
def test_malformed_model_files(tmp_path, text):
    p = tmp_path / "bad.foe"
    p.write_text(text)
    with pytest.raises(ValueError):
        fp.load_model(p)


def test_lambda_selection_matches_oracle_rules():
    table = orc.load_lambda_table(os.path.join(REPO, "paper_1609_05722_b200", "assets", "lambda_table.json"))
    for peak in (0.05, 0.1, 0.5, 1.0, 2.0, 3.0, 4.0, 4.99, 5.0, 8.0, 40.0, 100.0):
        for variant in ("direct", "transform", "transform_binned"):
            for fb in (None, "quadratic", "idiv"):
                if variant == "direct" and fb is not None:
                    continue
                assert fp.select_lambda(peak, variant, force_branch=fb) == orc.select_lambda(peak, variant, table, fb)
    # values quoted in SURVEY.md section 8(a) a3
    assert abs(fp.select_lambda(4.0, "transform", force_branch="quadratic") - 0.538107) < 1e-6
    assert abs(fp.select_lambda(4.0, "transform") - 2.100169) < 1e-6
    assert abs(fp.select_lambda(8.0, "direct") - 0.0963) < 1e-12


def test_budget_overrides_max_iters():
    """pipeline.py:83-87: the peak rule wins over a caller's max_iters."""
    assert fp.solver_budget(4.99, fp.SolverConfig(max_iters=7)).max_iters == 150
    assert fp.solver_budget(5.0, fp.SolverConfig(max_iters=7)).max_iters == 60


def test_request_validation():
    m = fp.load_packaged_model("foe_a")
    ok = np.zeros((8, 8))
    with pytest.raises(ValueError):
        fp.DenoiseRequest(noisy=np.zeros(8), peak=1.0, model=m, variant="transform")
    with pytest.raises(ValueError):
        fp.DenoiseRequest(noisy=ok + 0.5, peak=1.0, model=m, variant="transform")
    with pytest.raises(ValueError):
        fp.DenoiseRequest(noisy=ok - 1, peak=1.0, model=m, variant="transform")
    with pytest.raises(ValueError):
        fp.DenoiseRequest(noisy=ok, peak=0.0, model=m, variant="transform")
    with pytest.raises(ValueError):
        fp.DenoiseRequest(noisy=ok, peak=1.0, model=m, variant="nope")
    with pytest.raises(ValueError):
        fp.DenoiseRequest(noisy=ok, peak=1.0, model=m, variant="transform", force_branch="x")
    with pytest.raises(ValueError):
        fp.DenoiseRequest(noisy=ok, peak=1.0, model=m, variant="transform", lam=-1.0)
    with pytest.raises(ValueError):
        pipeline.denoise_direct(fp.DenoiseRequest(noisy=ok, peak=1.0, model=m, variant="direct"))
    with pytest.raises(ValueError):
        fp.SolverConfig(gamma=1.0)
    with pytest.raises(ValueError):
        fp.SolverConfig(backtrack_factor=1.0)


def test_counts_check_matches_reference_rule():
    """foe_counts_check == the reference's `np.any(x < 0) or not np.array_equal(x, np.rint(x))`
    (pipeline.py:54), element by element over the edge values, and at every position of a long array."""
    L = _lib.lib()
    edge = [0.0, -0.0, 1.0, 7.0, 0.5, 2.5, -1.0, 1e-300, 2.0 ** 52 - 0.5, 2.0 ** 52, 2.0 ** 52 + 2, 2.0 ** 53 + 2,
            1e300, np.inf, -np.inf, np.nan, 3.0000000000000004, 12345678.0]
    for v in edge:
        x = np.array([v])
        ref = bool(np.any(x < 0) or not np.array_equal(x, np.rint(x)))
        assert bool(L.foe_counts_check(x.ctypes.data, 1)) == ref, v
    rng = np.random.default_rng(3)
    base = rng.poisson(3.0, size=20000).astype(np.float64)
    assert L.foe_counts_check(base.ctypes.data, base.size) == 0
    for pos in (0, 8191, 8192, 19999):
        for bad in (-1.0, 0.25, np.nan):
            y = base.copy()
            y[pos] = bad
            assert L.foe_counts_check(y.ctypes.data, y.size) == 1, (pos, bad)
    assert L.foe_counts_check(None, 0) == 0


def test_synthetic_generator_is_deterministic():
    from paper_1609_05722_b200.synth import make_counts, synthetic_clean
    a = synthetic_clean(64, 48, 3)
    b = synthetic_clean(64, 48, 3)
    np.testing.assert_array_equal(a, b)
    assert a.min() >= 0 and a.max() <= 1 and a.std() > 0.05
    x, y = make_counts(64, 48, 3, 4.0)
    assert np.array_equal(y, np.rint(y)) and y.min() >= 0


def test_training_host_validation():
    """TrainingSample / TrainConfig / objective checks of the device training operators (host only)."""
    import numpy as np
    from paper_1609_05722_b200 import training as tr
    clean = np.ones((4, 4))
    s = tr.TrainingSample.create(clean, np.zeros((4, 4)))
    assert np.allclose(s.transformed, 2 * np.sqrt(0.375))
    with pytest.raises(ValueError):
        tr.TrainingSample.create(clean, np.full((4, 4), 0.5))
    with pytest.raises(ValueError):
        tr.TrainConfig(objective="nope")
    with pytest.raises(ValueError):
        tr._check_domain(fp.load_packaged_model("foe_a"), "original_domain")


def test_request_accepts_strided_views():
    """Non-contiguous inputs (flipped / transposed views, as the reference accepts) are validated on a
    buffer that outlives the native check -- no use-after-free of a temporary copy (large enough that a
    freed block would be returned to the OS)."""
    m = fp.load_packaged_model("foe_a")
    y = np.zeros((3000, 2000))
    y[5, 7] = 3.0
    for view in (y[::-1], y.T, y[:, ::2]):
        r = fp.DenoiseRequest(noisy=view, peak=1.0, model=m, variant="transform")
        assert r.noisy.flags.c_contiguous
        np.testing.assert_array_equal(r.noisy, view)
    bad = y.copy()
    bad[-1, -1] = 0.5
    with pytest.raises(ValueError):
        fp.DenoiseRequest(noisy=bad.T, peak=1.0, model=m, variant="transform")


def test_cli_exit_codes_without_a_gpu(tmp_path, capsys):
    """cli.py:28-31, 244-257: 1 usage (bad flags, invalid arguments), 2 data (missing / malformed
    files).  The numerical-failure code 3 needs a solve and is covered in the GPU suite."""
    from paper_1609_05722_b200.__main__ import EXIT_DATA, EXIT_USAGE, main
    with pytest.raises(SystemExit) as e:
        main(["denoise", "a.npy", "b.npy", "--bogus"])
    assert e.value.code == EXIT_USAGE
    with pytest.raises(SystemExit) as e:
        main(["nope"])
    assert e.value.code == EXIT_USAGE
    assert main(["denoise", str(tmp_path / "missing.npy"), str(tmp_path / "o.npy"), "--peak", "1"]) == EXIT_DATA
    (tmp_path / "junk.npy").write_bytes(b"not an npy file")
    assert main(["denoise", str(tmp_path / "junk.npy"), str(tmp_path / "o.npy"), "--peak", "1"]) == EXIT_DATA
    np.save(tmp_path / "vec.npy", np.zeros(5))
    assert main(["denoise", str(tmp_path / "vec.npy"), str(tmp_path / "o.npy"), "--peak", "1"]) == EXIT_DATA
    (tmp_path / "bad.foe").write_text("FOE 1\nanscombe 1 5\n")
    np.save(tmp_path / "y.npy", np.ones((8, 8)))
    assert main(["denoise", str(tmp_path / "y.npy"), str(tmp_path / "o.npy"), "--peak", "1",
                 "--model", str(tmp_path / "bad.foe")]) == EXIT_DATA
    np.save(tmp_path / "neg.npy", -np.ones((8, 8)))  # invalid counts: a usage-class ValueError
    assert main(["denoise", str(tmp_path / "neg.npy"), str(tmp_path / "o.npy"), "--peak", "1"]) == EXIT_USAGE
    assert main(["denoise", str(tmp_path / "y.npy"), str(tmp_path / "o.npy"), "--peak", "0"]) == EXIT_USAGE


def test_counts_check_stage_validates_and_stages():
    """foe_counts_check_stage: the same verdicts as foe_counts_check, every count written as an exact float,
    and code 2 (valid, not stageable) as soon as a count needs more than a float's 24 bits."""
    L = _lib.lib()
    rng = np.random.default_rng(5)
    base = rng.poisson(3.0, size=20000).astype(np.float64)
    dst = np.full(base.size, -1.0, dtype=np.float32)
    assert L.foe_counts_check_stage(base.ctypes.data, base.size, dst.ctypes.data) == 0
    np.testing.assert_array_equal(dst.astype(np.float64), base)
    for pos in (0, 8191, 8192, 19999):
        for bad in (-1.0, 0.25, np.nan):
            y = base.copy()
            y[pos] = bad
            assert L.foe_counts_check_stage(y.ctypes.data, y.size, dst.ctypes.data) == 1, (pos, bad)
    for big in (2.0 ** 24, 2.0 ** 24 + 1, 1e300, np.inf):
        y = base.copy()
        y[17] = big
        assert L.foe_counts_check_stage(y.ctypes.data, y.size, dst.ctypes.data) == 2, big
    y = base.copy()
    y[17] = 2.0 ** 24 - 1
    assert L.foe_counts_check_stage(y.ctypes.data, y.size, dst.ctypes.data) == 0
    assert dst[17] == 2.0 ** 24 - 1
    assert L.foe_counts_check_stage(None, 0, None) == 0
