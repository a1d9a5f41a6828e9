"""Pin the CPU oracle (oracle/foe_oracle.c) to golden vectors produced by the reference.

The golden .npz files come from tests/golden/make_golden.py, which runs the
reference foepoisson package itself (image.py, prior.py, solver.py,
anscombe.py, pipeline.py).  Tolerances follow the reference's own tests:
1e-12 for the convolution operators (test_image.py:17-39), rtol 1e-12 energy
(test_prior.py:96-108), 1e-12 prox (test_solver.py:35-59), 1e-14 Anscombe
(test_anscombe.py:50-60).
"""

import os

import numpy as np
import pytest

from oracle import cpu as orc
from tests.conftest import REPO

ASSETS = os.path.join(REPO, "paper_1609_05722_b200", "assets")


def _model(g, name):
    return orc.OracleModel(filters=g[f"filters_{name}"], weights=g[f"weights_{name}"],
                           boundary=str(g[f"boundary_{name}"]))


def test_convolutions_match_reference(golden):
    g = golden("conv")
    keys = [k[5:] for k in g if k.startswith("same_")]
    assert len(keys) == 16
    for key in keys:
        b = key.split("_")[-1]
        np.testing.assert_allclose(orc.convolve_same(g[f"x_{key}"], g[f"k_{key}"], b), g[f"same_{key}"],
                                   rtol=1e-12, atol=1e-12, err_msg=key)
        np.testing.assert_allclose(orc.convolve_adjoint(g[f"y_{key}"], g[f"k_{key}"], b), g[f"adj_{key}"],
                                   rtol=1e-12, atol=1e-12, err_msg=key)


def test_energy_gradient_match_reference(golden):
    g = golden("prior")
    names = [k[2:] for k in g if k.startswith("u_")]
    assert len(names) == 6
    for name in names:
        model = _model(g, name)
        u = g[f"u_{name}"]
        np.testing.assert_allclose(orc.foe_energy(u, model), float(g[f"energy_{name}"]), rtol=1e-12)
        np.testing.assert_allclose(orc.foe_gradient(u, model), g[f"grad_{name}"], rtol=1e-11, atol=1e-12)


def test_packaged_models_decode_like_reference(golden):
    g = golden("prior")
    m = orc.read_foe(os.path.join(ASSETS, "foe_a.foe"))
    np.testing.assert_allclose(m.filters, g["filters_foe_a"], rtol=0, atol=1e-15)
    np.testing.assert_array_equal(m.weights, g["weights_foe_a"])
    m = orc.read_foe(os.path.join(ASSETS, "foe_fallback48x7.foe"))
    np.testing.assert_allclose(m.filters, g["filters_fallback"], rtol=0, atol=1e-15)


def test_elementwise_match_reference(golden):
    g = golden("elementwise")
    ut, obs = g["ut"], g["obs"]
    np.testing.assert_allclose(orc.prox_quadratic(ut, 0.7, obs), g["pq_0.7"], rtol=1e-14)
    np.testing.assert_array_equal(orc.prox_quadratic(ut, 0.0, obs), g["pq_0"])
    for t in ("0.7", "0", "3.5"):
        np.testing.assert_allclose(orc.prox_idiv(ut, float(t), obs), g[f"pi_{t}"], rtol=1e-14, atol=1e-300)
    np.testing.assert_allclose(orc.anscombe_forward(obs), g["ans_fwd"], rtol=1e-15)
    d = {}
    np.testing.assert_allclose(orc.anscombe_inverse_exact_unbiased(g["z"], d), g["ans_inv"], rtol=1e-14, atol=1e-14)
    assert [d["n_clamped_input"], d["n_clamped_output"]] == list(g["ans_inv_counts"])


def _check_denoise(res, g, name, exact_trace=True):
    ref_img = g[f"{name}_image"]
    tr = g[f"{name}_trace"]
    assert res["branch"] == str(g[f"{name}_branch"])
    np.testing.assert_allclose(res["lam"], g[f"{name}_meta"][1], rtol=1e-15)
    ours = np.array([res["trace"].F, res["trace"].G, res["trace"].L, res["trace"].step_norm]).T
    assert ours.shape[0] == tr.shape[0]
    # identical backtracking decisions => identical L sequence
    np.testing.assert_allclose(ours[:, 2], tr[:, 2], rtol=1e-13)
    np.testing.assert_allclose(ours[:, 0], tr[:, 0], rtol=1e-10)
    peak = g[f"{name}_meta"][0]
    assert np.max(np.abs(res["image"] - ref_img)) <= 1e-8 * peak


def test_denoise_small_matches_reference(golden):
    g = golden("denoise_small")
    table = orc.load_lambda_table(os.path.join(ASSETS, "lambda_table.json"))
    fa = orc.read_foe(os.path.join(ASSETS, "foe_a.foe"))
    fs = orc.read_foe(os.path.join(ASSETS, "foe_s.foe"))
    fb = orc.read_foe(os.path.join(ASSETS, "foe_fallback48x7.foe"))
    jobs = {"t_quad_p4": (fa, "transform", "quadratic"), "t_idiv_p4": (fa, "transform", None),
            "t_quad_p1": (fa, "transform", "quadratic"), "t_idiv_p05": (fa, "transform", None),
            "t_quad_p8": (fa, "transform", None), "d_fa_p8": (fa, "direct", None),
            "d_fs_p8": (fs, "direct", None), "t_fb_p2": (fb, "transform", "quadratic"),
            "t_quad_reltol": (fa, "transform", "quadratic")}
    for name, (model, variant, fbr) in jobs.items():
        meta = g[f"{name}_meta"]
        res = orc.denoise(g[f"{name}_noisy"], meta[0], model, variant, table, force_branch=fbr,
                          rel_tol=meta[5])
        _check_denoise(res, g, name)


@pytest.mark.slow
def test_cfg1_full_size_matches_reference(golden):
    """BASELINE config 1 (256^2, peak 4, quadratic, foe_a): oracle vs reference run."""
    from paper_1609_05722_b200.synth import make_counts
    g = golden("cfg1_256")
    _, y = make_counts(256, 256, 0, 4.0)
    assert y.sum() == g["counts_sum"]
    table = orc.load_lambda_table(os.path.join(ASSETS, "lambda_table.json"))
    fa = orc.read_foe(os.path.join(ASSETS, "foe_a.foe"))
    res = orc.denoise(y, 4.0, fa, "transform", table, force_branch="quadratic", rel_tol=0.0)
    np.testing.assert_allclose(res["trace"].L, g["trace"][:, 2], rtol=1e-13)
    assert np.max(np.abs(res["image"] - g["image"])) <= 1e-5 * 4.0   # golden stored as float32


def test_binned_matches_reference(golden):
    """transform_binned (pipeline.py:214-235) incl. bin3/unbin_bilinear (noise.py:55-113)."""
    g = golden("binned")
    table = orc.load_lambda_table(os.path.join(ASSETS, "lambda_table.json"))
    fa = orc.read_foe(os.path.join(ASSETS, "foe_a.foe"))
    for name, fbr in (("b_p05", None), ("b_p02_quad", "quadratic"), ("b_f1", None), ("b_f2", None)):
        meta = g[f"{name}_meta"]
        np.testing.assert_array_equal(orc.bin3(g[f"{name}_noisy"], int(meta[5])), g[f"{name}_binned"])
        res = orc.denoise(g[f"{name}_noisy"], meta[0], fa, "transform_binned", table, force_branch=fbr,
                          rel_tol=0.0, bin_factor=int(meta[5]))
        assert res["branch"] == str(g[f"{name}_branch"]) and res["peak_used"] == meta[6]
        np.testing.assert_allclose(res["trace"].L, g[f"{name}_trace"][:, 2], rtol=1e-13)
        np.testing.assert_allclose(res["image"], g[f"{name}_image"], rtol=0, atol=1e-8 * meta[0])
        np.testing.assert_allclose(orc.unbin_bilinear(res["transformed"], g[f"{name}_noisy"].shape, int(meta[5])),
                                   g[f"{name}_unbin_of_transformed"], rtol=1e-13, atol=1e-13)


CFG23 = {"cfg2_quad": (1.0, "foe_a", "transform", "quadratic"), "cfg2_idiv": (1.0, "foe_a", "transform", None),
         "cfg3_fa": (8.0, "foe_a_original", "direct", None), "cfg3_fs": (8.0, "foe_s", "direct", None)}


def cfg23_model(name):
    mk = CFG23[name][1]
    if mk == "foe_s":
        return orc.read_foe(os.path.join(ASSETS, "foe_s.foe"))
    fa = orc.read_foe(os.path.join(ASSETS, "foe_a.foe"))
    if mk == "foe_a_original":
        fa = orc.OracleModel(filters=fa.filters, weights=fa.weights, boundary=fa.boundary, domain_tag="original")
    return fa


@pytest.mark.slow
@pytest.mark.parametrize("name", sorted(CFG23))
def test_cfg23_full_size_matches_reference(golden, name):
    """BASELINE configs 2 and 3 at 512^2 (tests/golden/make_golden_512.py ran the reference's own
    denoise): identical L-trace (identical decisions), F to 1e-10, image to the fp32 storage of the
    golden."""
    import hashlib
    from paper_1609_05722_b200.synth import make_counts
    g = golden("cfg23_512")
    peak, _, variant, fb = CFG23[name]
    _, y = make_counts(512, 512, 0, peak)
    assert hashlib.sha256(y.tobytes()).digest() == g[f"{name}_counts_sha"].tobytes()
    table = orc.load_lambda_table(os.path.join(ASSETS, "lambda_table.json"))
    res = orc.denoise(y, peak, cfg23_model(name), variant, table, force_branch=fb, rel_tol=0.0)
    tr = g[f"{name}_trace"]
    assert res["branch"] == str(g[f"{name}_branch"]) and res["lam"] == g[f"{name}_meta"][1]
    np.testing.assert_allclose(res["trace"].L, tr[:, 2], rtol=1e-13)
    np.testing.assert_allclose(res["trace"].F, tr[:, 0], rtol=1e-10)
    np.testing.assert_allclose(res["trace"].G, tr[:, 1], rtol=1e-9)
    np.testing.assert_allclose(res["trace"].step_norm, tr[:, 3], rtol=1e-7)
    assert np.max(np.abs(res["image"] - g[f"{name}_image"])) <= 1e-5 * peak  # golden stored as float32
