"""GPU parity: the sm_100a path vs the CPU oracle and the reference's golden vectors.

Gates (BASELINE.json north_star): per-pass gradient rel-L2 <= 1e-5; after the
full solve max |x_gpu - x_ref| <= 1e-3 * peak and |dPSNR| <= 0.01 dB on the
same counts, filter bank and iteration budget.  fp32 operator tolerances are
stated per test.
"""

import os

import numpy as np
import pytest

import paper_1609_05722_b200 as fp
from oracle import cpu as orc
from paper_1609_05722_b200.synth import make_counts
from tests.conftest import REPO

pytestmark = pytest.mark.gpu

ASSETS = os.path.join(REPO, "paper_1609_05722_b200", "assets")
TABLE = orc.load_lambda_table(os.path.join(ASSETS, "lambda_table.json"))


def psnr(x, ref, peak):
    mse = np.mean((x - ref) ** 2)
    return 10 * np.log10(peak ** 2 / mse)


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def oracle_model(model):
    return orc.OracleModel(filters=model.filters, weights=model.weights, boundary=model.boundary,
                           domain_tag=model.domain_tag)


def test_elementwise_vs_golden(golden):
    g = golden("elementwise")
    ut, obs = g["ut"], g["obs"]
    np.testing.assert_allclose(fp.solver.prox_quadratic(ut, 0.7, obs), g["pq_0.7"], rtol=2e-6, atol=1e-6)
    np.testing.assert_allclose(fp.solver.prox_quadratic(ut, 0.0, obs), g["pq_0"], rtol=1e-6, atol=1e-6)
    for t in ("0.7", "0", "3.5"):
        np.testing.assert_allclose(fp.solver.prox_idiv(ut, float(t), obs), g[f"pi_{t}"], rtol=2e-6, atol=2e-6)
    from paper_1609_05722_b200 import anscombe
    np.testing.assert_allclose(anscombe.anscombe_forward(obs), g["ans_fwd"], rtol=1e-7)
    d = {}
    np.testing.assert_allclose(anscombe.anscombe_inverse_exact_unbiased(g["z"], d), g["ans_inv"], rtol=1e-6,
                               atol=1e-6)
    assert [d["n_clamped_input"], d["n_clamped_output"]] == list(g["ans_inv_counts"])


def test_single_filter_operators_vs_golden(golden):
    """convolve_same / convolve_adjoint (image.py:37-83), fp32: rel-L2 <= 1e-6."""
    g = golden("conv")
    for key in [k[5:] for k in g if k.startswith("same_")]:
        b = key.split("_")[-1]
        assert rel_l2(fp.image.convolve_same(g[f"x_{key}"], g[f"k_{key}"], b), g[f"same_{key}"]) < 1e-6, key
        assert rel_l2(fp.image.convolve_adjoint(g[f"y_{key}"], g[f"k_{key}"], b), g[f"adj_{key}"]) < 1e-6, key


def test_fused_energy_gradient_vs_golden(golden):
    """Fused pass (EVAL mode) vs reference foe_energy/foe_gradient: energy rel 1e-6, grad rel-L2 1e-5."""
    g = golden("prior")
    for name in [k[2:] for k in g if k.startswith("u_")]:
        filt, w = g[f"filters_{name}"], g[f"weights_{name}"]
        m = filt.shape[1]
        basis = fp.dct_basis(m)
        betas = np.tensordot(filt, basis.atoms, axes=([1, 2], [1, 2]))
        model = fp.FoEModel(basis=basis, betas=betas, weights=w, domain_tag="anscombe",
                            boundary=str(g[f"boundary_{name}"]))
        np.testing.assert_allclose(model.filters, filt, atol=1e-12)
        u = g[f"u_{name}"]
        e = fp.foe_energy(u, model)
        gr = fp.foe_gradient(u, model)
        ref_e = float(g[f"energy_{name}"])
        assert abs(e - ref_e) <= 1e-6 * max(abs(ref_e), 1e-3), (name, e, ref_e)
        assert rel_l2(gr, g[f"grad_{name}"]) <= 1e-5, (name, rel_l2(gr, g[f"grad_{name}"]))


@pytest.mark.parametrize("shape", [(7, 9), (47, 45), (48, 93), (130, 97), (512, 512)])
@pytest.mark.parametrize("m,boundary", [(1, "symmetric"), (3, "symmetric"), (5, "symmetric"), (7, "symmetric"),
                                        (3, "periodic"), (5, "periodic"), (7, "periodic")])
def test_fused_gradient_shapes_and_boundaries(shape, m, boundary):
    """Tile edges, partial tiles, the last-tile pull-up and both fold rules vs the C oracle."""
    if min(shape) < m:
        pytest.skip("image smaller than filter")
    rng = np.random.default_rng(hash((shape, m, boundary)) % 2 ** 32)
    basis = fp.dct_basis(m) if m > 1 else None
    if m == 1:
        filt = rng.normal(size=(3, 1, 1))
        w = rng.uniform(0.5, 2, 3)
        model_o = orc.OracleModel(filters=filt, weights=w, boundary=boundary)
        from paper_1609_05722_b200.prior import energy_grad_device
        import torch
        u = rng.normal(scale=3, size=shape)
        # m = 1 has no DCT basis; drive the device bank directly
        from paper_1609_05722_b200.prior import DeviceBank
        bank = DeviceBank(filt, w, boundary)
        from paper_1609_05722_b200 import _lib
        ud = torch.from_numpy(u).to("cuda", torch.float32)[None].contiguous()
        gd = torch.empty_like(ud)
        en = torch.empty(1, dtype=torch.float64, device="cuda")
        ws = torch.empty(_lib.lib().foe_eval_workspace_size(bank.handle, 1, *shape), dtype=torch.uint8,
                         device="cuda")
        _lib.check(_lib.lib().foe_energy_grad(bank.handle, ud.data_ptr(), gd.data_ptr(), en.data_ptr(), 1, *shape,
                                              ws.data_ptr(), ws.numel(), torch.cuda.current_stream().cuda_stream))
        assert rel_l2(gd[0].double().cpu().numpy(), orc.foe_gradient(u, model_o)) <= 1e-5
        assert abs(en.item() - orc.foe_energy(u, model_o)) <= 1e-6 * abs(orc.foe_energy(u, model_o))
        return
    model = fp.FoEModel(basis=basis, betas=rng.normal(scale=0.7, size=(6, basis.n_atoms)),
                        weights=rng.uniform(0.5, 2, 6), domain_tag="anscombe", boundary=boundary)
    u = rng.normal(scale=3, size=shape) + 5
    ref_g = orc.foe_gradient(u, oracle_model(model))
    ref_e = orc.foe_energy(u, oracle_model(model))
    assert rel_l2(fp.foe_gradient(u, model), ref_g) <= 1e-5
    assert abs(fp.foe_energy(u, model) - ref_e) <= 1e-6 * abs(ref_e)


@pytest.mark.parametrize("kernel", ["ffma", "tc"])
def test_gradient_along_oracle_iterates(monkeypatch, kernel):
    """Per-iteration gradient check (north_star, rel-L2 <= 1e-5): at oracle iterates u_k of a 256^2 foe_a solve.

    The device state is fp32, so the oracle gradient is taken at the same fp32-representable
    iterate; rounding u_k itself to fp32 moves the reference gradient by up to ~9e-6 near
    convergence (input quantisation, reported separately and not charged to the operator)."""
    monkeypatch.setenv("FOE_TC", "1" if kernel == "tc" else "0")
    model = fp.load_packaged_model("foe_a")
    om = oracle_model(model)
    _, y = make_counts(256, 256, 0, 4.0)
    v = orc.anscombe_forward(y)
    lam = orc.select_lambda(4.0, "transform", TABLE, "quadratic")
    worst = 0.0
    for k in (1, 3, 10, 40, 150):
        uk, _ = orc.ipiano_foe(v, v, om, lam, "quadratic", max_iters=k, rel_tol=0.0)
        u32 = uk.astype(np.float32).astype(np.float64)
        worst = max(worst, rel_l2(fp.foe_gradient(u32, model), orc.foe_gradient(u32, om)))
    assert worst <= 1e-5, worst


def _check_solve(res_img, ref_img, peak, clean=None, what=""):
    err = np.max(np.abs(res_img - ref_img))
    assert err <= 1e-3 * peak, (what, err / peak)
    if clean is not None:
        d = abs(psnr(res_img, peak * clean, peak) - psnr(ref_img, peak * clean, peak))
        assert d <= 0.01, (what, d)
    return err / peak


def test_denoise_small_vs_reference_golden(golden):
    """Full pipeline on small images vs the reference's own outputs (all branches, both models)."""
    g = golden("denoise_small")
    fa = fp.load_packaged_model("foe_a")
    import dataclasses
    models = {"fa": fa, "fs": fp.load_packaged_model("foe_s"), "fb": fp.load_packaged_model("foe_fallback48x7"),
              "fa_orig": dataclasses.replace(fa, domain_tag="original")}
    jobs = {"t_quad_p4": ("fa", "transform", "quadratic"), "t_idiv_p4": ("fa", "transform", None),
            "t_quad_p1": ("fa", "transform", "quadratic"), "t_idiv_p05": ("fa", "transform", None),
            "t_quad_p8": ("fa", "transform", None), "d_fa_p8": ("fa_orig", "direct", None),
            "d_fs_p8": ("fs", "direct", None), "t_fb_p2": ("fb", "transform", "quadratic"),
            "t_quad_reltol": ("fa", "transform", "quadratic")}
    for name, (mk, variant, fbr) in jobs.items():
        meta = g[f"{name}_meta"]
        peak = meta[0]
        req = fp.DenoiseRequest(noisy=g[f"{name}_noisy"], peak=peak, model=models[mk], variant=variant,
                                force_branch=fbr)
        r = fp.denoise(req, fp.SolverConfig(rel_tol=meta[5]))
        assert r.branch == str(g[f"{name}_branch"])
        assert len(r.trace) == g[f"{name}_trace"].shape[0]
        _check_solve(r.image, g[f"{name}_image"], peak, g[f"{name}_clean"], name)


def test_cfg1_256_vs_reference_golden(golden):
    """BASELINE config 1: 256^2, peak 4, quadratic forced, foe_a, 150 iterations."""
    g = golden("cfg1_256")
    x, y = make_counts(256, 256, 0, 4.0)
    assert y.sum() == g["counts_sum"]
    r = fp.denoise(fp.DenoiseRequest(noisy=y, peak=4.0, model=fp.load_packaged_model("foe_a"),
                                     variant="transform", force_branch="quadratic"), fp.SolverConfig(rel_tol=0.0))
    assert len(r.trace) == 150
    _check_solve(r.image, g["image"].astype(np.float64), 4.0, x, "cfg1")
    assert r.trace.L == g["trace"][:, 2].tolist()  # identical decisions (the exact L-trace)


@pytest.mark.parametrize("peak,branch", [(1.0, "quadratic"), (1.0, None)])
def test_cfg2_512_vs_oracle(peak, branch):
    """BASELINE config 2 (512^2, peak 1): quadratic as named, and the reference's default idiv branch."""
    model = fp.load_packaged_model("foe_a")
    x, y = make_counts(512, 512, 0, peak)
    ref = orc.denoise(y, peak, oracle_model(model), "transform", TABLE, force_branch=branch, rel_tol=0.0)
    r = fp.denoise(fp.DenoiseRequest(noisy=y, peak=peak, model=model, variant="transform", force_branch=branch),
                   fp.SolverConfig(rel_tol=0.0))
    assert len(r.trace) == 150
    _check_solve(r.image, ref["image"], peak, x, f"cfg2 {branch}")


@pytest.mark.parametrize("which", ["foe_a_original", "foe_s"])
def test_cfg3_direct_512_vs_oracle(which):
    """BASELINE config 3: direct Poisson-domain variant, peak 8, 60 iterations."""
    import dataclasses
    fa = fp.load_packaged_model("foe_a")
    model = dataclasses.replace(fa, domain_tag="original") if which == "foe_a_original" else \
        fp.load_packaged_model("foe_s")
    x, y = make_counts(512, 512, 0, 8.0)
    ref = orc.denoise(y, 8.0, oracle_model(model), "direct", TABLE, rel_tol=0.0)
    r = fp.denoise(fp.DenoiseRequest(noisy=y, peak=8.0, model=model, variant="direct"),
                   fp.SolverConfig(rel_tol=0.0))
    assert len(r.trace) == 60 and np.all(r.image >= 0)
    _check_solve(r.image, ref["image"], 8.0, x, f"cfg3 {which}")


def test_batch_equals_single_bitwise():
    """Batched solve (cfg4 layout, per-image peaks/lambda/state) == independent single solves, bitwise."""
    model = fp.load_packaged_model("foe_a")
    ys, peaks = [], []
    for s in range(4):
        peak = [0.5, 1.0, 2.0, 4.0][s % 4]
        ys.append(make_counts(96, 80, s, peak)[1])
        peaks.append(peak)
    imgs, traces, lams, _ = fp.denoise_batch(np.stack(ys), peaks, model, "transform", force_branch="quadratic",
                                             solver=fp.SolverConfig(rel_tol=0.0))
    for s in range(4):
        r = fp.denoise(fp.DenoiseRequest(noisy=ys[s], peak=peaks[s], model=model, variant="transform",
                                         force_branch="quadratic"), fp.SolverConfig(rel_tol=0.0))
        np.testing.assert_array_equal(imgs[s], r.image)
        assert traces[s].L == r.trace.L


def test_solve_is_deterministic():
    model = fp.load_packaged_model("foe_a")
    _, y = make_counts(200, 136, 9, 2.0)
    req = fp.DenoiseRequest(noisy=y, peak=2.0, model=model, variant="transform")
    a = fp.denoise(req, fp.SolverConfig(rel_tol=0.0))
    b = fp.denoise(req, fp.SolverConfig(rel_tol=0.0))
    np.testing.assert_array_equal(a.image, b.image)
    assert a.trace.F == b.trace.F


def test_accepted_steps_satisfy_descent_inequality():
    """test_solver.py:217-229 on the device trace."""
    model = fp.load_packaged_model("foe_a")
    _, y = make_counts(64, 64, 2, 1.0)
    r = fp.denoise(fp.DenoiseRequest(noisy=y, peak=1.0, model=model, variant="transform", force_branch="quadratic"),
                   fp.SolverConfig(rel_tol=0.0))
    assert np.all(np.asarray(r.trace.descent_slack) <= np.asarray(r.trace.slack_tol))
    assert r.trace.n_trials >= len(r.trace)


def test_numerical_failure_raises_with_trace():
    """Stalled backtracking -> NumericalFailure carrying the partial trace (solver.py:159-160)."""
    model = fp.load_packaged_model("foe_a")
    _, y = make_counts(32, 32, 1, 4.0)
    req = fp.DenoiseRequest(noisy=y, peak=4.0, model=model, variant="transform", force_branch="quadratic")
    with pytest.raises(fp.NumericalFailure) as ei:
        fp.denoise(req, fp.SolverConfig(lipschitz_init=1.0, max_lipschitz=1.5))
    assert ei.value.trace is not None


@pytest.mark.parametrize("n_bands,H,W,iters", [(2, 200, 130, 40), (3, 200, 130, 40), (4, 1000, 333, 12),
                                               (4, 8192, 8192, 3)])
def test_row_bands_equal_single_device_bitwise(n_bands, H, W, iters):
    """Config-5 decomposition through the halo/all-gather path (bands in-process on one GPU):
    bitwise identical to the single-device solve, for any band count."""
    import torch
    from paper_1609_05722_b200 import bands
    from paper_1609_05722_b200.anscombe import forward_device
    model = fp.load_packaged_model("foe_a")
    _, y = make_counts(H, W, 7, 2.0)
    v = forward_device(torch.from_numpy(y).cuda())
    cfg = fp.SolverConfig(rel_tol=0.0)
    lam = fp.select_lambda(2.0, "transform", force_branch="quadratic")
    single = fp.solve_device(model, v, v, lam, "quadratic", iters, cfg)
    u, traces, status = bands.solve_image_bands(model, v, v, lam, "quadratic", iters, n_bands, cfg)
    assert status == [0]
    assert traces[0].L == single.traces[0].L and traces[0].F == single.traces[0].F
    assert torch.equal(u[0], single.u)


def test_transform_binned_vs_reference_golden(golden):
    """transform_binned on the device (bin3 / unbin kernels around the solve) vs the reference output."""
    g = golden("binned")
    model = fp.load_packaged_model("foe_a")
    for name, fbr in (("b_p05", None), ("b_p02_quad", "quadratic"), ("b_f1", None), ("b_f2", None)):
        meta = g[f"{name}_meta"]
        peak = meta[0]
        r = fp.denoise(fp.DenoiseRequest(noisy=g[f"{name}_noisy"], peak=peak, model=model, variant="transform_binned",
                                         force_branch=fbr, bin_factor=int(meta[5])), fp.SolverConfig(rel_tol=0.0))
        assert r.branch == str(g[f"{name}_branch"]) and r.peak_used == meta[6]
        assert r.image.shape == g[f"{name}_image"].shape
        _check_solve(r.image, g[f"{name}_image"], peak, g[f"{name}_clean"], name)


def test_tcgen05_primitives_selftest():
    """TMEM alloc / tcgen05.st / TS-form MMA with the hand-built K-major descriptor / commit / tcgen05.ld:
    3xTF32 product matches fp64 to ~fp32 accuracy."""
    import torch
    from paper_1609_05722_b200 import _lib
    rng = np.random.default_rng(3)
    A = rng.normal(size=(128, 32)).astype(np.float32)
    B = rng.normal(size=(32, 32)).astype(np.float32)
    Ad, Bd = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    Dd = torch.zeros((128, 32), dtype=torch.float32, device="cuda")
    _lib.check(_lib.lib().foe_tc_selftest(Ad.data_ptr(), Bd.data_ptr(), Dd.data_ptr(),
                                          torch.cuda.current_stream().cuda_stream))
    ref = A.astype(np.float64) @ B.astype(np.float64).T
    got = Dd.cpu().numpy()
    err = np.abs(got - ref).max() / np.abs(ref).max()
    assert err < 1e-6, err


@pytest.mark.parametrize("kernel", ["ffma", "tc"])
@pytest.mark.parametrize("shape,boundary", [((47, 45), "symmetric"), ((130, 97), "symmetric"), ((512, 512), "symmetric"),
                                            ((200, 136), "periodic"), ((7, 9), "symmetric")])
def test_pass_kernel_gradient_vs_oracle(monkeypatch, shape, boundary, kernel):
    """Both pass kernels -- k_pass (FFMA) and k_pass_tc (tcgen05 implicit GEMMs, 3xTF32) -- fused
    energy / gradient vs the C oracle."""
    monkeypatch.setenv("FOE_TC", "1" if kernel == "tc" else "0")
    rng = np.random.default_rng(hash((shape, boundary)) % 2 ** 32)
    if boundary == "symmetric":
        model = fp.load_packaged_model("foe_a")
        u = orc.anscombe_forward(make_counts(*shape, 4, 2.0)[1])
    else:
        basis = fp.dct_basis(5)
        model = fp.FoEModel(basis=basis, betas=rng.normal(scale=0.7, size=(20, basis.n_atoms)),
                            weights=rng.uniform(0.5, 2, 20), domain_tag="anscombe", boundary=boundary)
        u = rng.normal(scale=3, size=shape) + 5
    u = u.astype(np.float32).astype(np.float64)
    om = oracle_model(model)
    ref_g, ref_e = orc.foe_gradient(u, om), orc.foe_energy(u, om)
    assert rel_l2(fp.foe_gradient(u, model), ref_g) <= 1e-5
    assert abs(fp.foe_energy(u, model) - ref_e) <= 1e-6 * abs(ref_e)


@pytest.mark.parametrize("kernel", ["ffma", "tc"])
@pytest.mark.parametrize("branch", ["quadratic", None])
def test_pass_kernel_solve_cfg2_vs_oracle(monkeypatch, branch, kernel):
    """Config 2 (512^2, peak 1) through each pass kernel: parity gates vs the oracle."""
    monkeypatch.setenv("FOE_TC", "1" if kernel == "tc" else "0")
    model = fp.load_packaged_model("foe_a")
    x, y = make_counts(512, 512, 0, 1.0)
    ref = orc.denoise(y, 1.0, oracle_model(model), "transform", TABLE, force_branch=branch, rel_tol=0.0)
    r = fp.denoise(fp.DenoiseRequest(noisy=y, peak=1.0, model=model, variant="transform", force_branch=branch),
                   fp.SolverConfig(rel_tol=0.0))
    assert len(r.trace) == 150
    _check_solve(r.image, ref["image"], 1.0, x, f"{kernel} cfg2 {branch}")


@pytest.mark.parametrize("kernel", ["ffma", "tc"])
def test_pass_kernel_cfg1_vs_reference_golden(monkeypatch, golden, kernel):
    """Config 1 through each pass kernel vs the reference's own output."""
    monkeypatch.setenv("FOE_TC", "1" if kernel == "tc" else "0")
    g = golden("cfg1_256")
    x, y = make_counts(256, 256, 0, 4.0)
    r = fp.denoise(fp.DenoiseRequest(noisy=y, peak=4.0, model=fp.load_packaged_model("foe_a"),
                                     variant="transform", force_branch="quadratic"), fp.SolverConfig(rel_tol=0.0))
    _check_solve(r.image, g["image"].astype(np.float64), 4.0, x, f"{kernel} cfg1")


def test_device_scores_vs_reference_golden(golden):
    """foe_score (PSNR / MSSIM, metrics.py:30-102) vs the reference's own scores."""
    from paper_1609_05722_b200 import metrics
    g = golden("metrics")
    for i in range(4):
        peak, ref_psnr, ref_mssim = g[f"m{i}_ref"]
        r = metrics.score_denoised(g[f"m{i}_xhat"], g[f"m{i}_g"], peak)
        assert abs(r.psnr_db - ref_psnr) <= 1e-10 * abs(ref_psnr), (i, r.psnr_db, ref_psnr)
        assert abs(r.mssim - ref_mssim) <= 1e-12, (i, r.mssim, ref_mssim)
    # batched scoring equals one call per image
    x = np.stack([g["m2_xhat"], g["m2_g"] * 0.9])
    y = np.stack([g["m2_g"], g["m2_g"]])
    ps, ms = metrics.score_batch(x, y, 0.5)
    assert ps[0] == metrics.score_batch(x[0], y[0], 0.5)[0][0] and ms[1] == metrics.score_batch(x[1], y[1], 0.5)[1][0]


def test_evaluation_grid_vs_reference_golden(golden):
    """benchmark.run_benchmark on a 2 images x 3 peaks x 3 variants grid: batched device solves give
    the reference's rows (seeds, branches, lambdas exact; PSNR within the 0.01 dB gate)."""
    from paper_1609_05722_b200 import evaluate as ev
    g = golden("bench_grid")
    spec = ev.BenchmarkSpec(images=("syn40x36s1", "syn33x47s2"), peaks=(0.5, 2.0, 8.0),
                            variants=("transform", "transform_binned", "direct"),
                            transform_model=fp.load_packaged_model("foe_a"),
                            direct_model=fp.load_packaged_model("foe_s"), base_seed=7)
    rows = ev.run_benchmark(spec)
    assert [f"{r.image}|{r.variant}|{r.branch}" for r in rows] == list(g["rows_key"])
    assert [r.seed for r in rows] == [int(s) for s in g["row_seeds"]]
    num = g["rows_num"]
    for r, (peak, psnr_ref, mssim_ref, lam_ref) in zip(rows, num):
        assert r.peak == peak and r.lam == lam_ref
        assert abs(r.psnr_db - psnr_ref) <= 0.01, (r, psnr_ref)
        assert abs(r.mssim - mssim_ref) <= 1e-3, (r, mssim_ref)


def test_cli_denoise_round_trip(tmp_path):
    """python -m paper_1609_05722_b200 denoise (cli.py:63-85 shim) equals the API call."""
    from paper_1609_05722_b200.__main__ import main
    _, y = make_counts(40, 44, 5, 2.0)
    np.save(tmp_path / "in.npy", y)
    assert main(["denoise", str(tmp_path / "in.npy"), str(tmp_path / "out.npy"), "--peak", "2",
                 "--trace", str(tmp_path / "t.csv")]) == 0
    ref = fp.denoise(fp.DenoiseRequest(noisy=y, peak=2.0, model=fp.load_packaged_model("foe_a"), variant="transform"))
    np.testing.assert_array_equal(np.load(tmp_path / "out.npy"), ref.image)
    assert (tmp_path / "t.csv").exists()


def test_fp64_bank_operators_vs_golden(golden):
    """foe_conv_bank64 / foe_adjoint_bank64 (training side, fp64) vs the reference's convolve_same /
    convolve_adjoint at the reference tests' 1e-12 tolerance, m in {1,3,5,7} x both boundaries."""
    import torch
    from paper_1609_05722_b200 import training as tr
    from paper_1609_05722_b200.image import BOUNDARY_CODES
    g = golden("conv")
    for key in [k[5:] for k in g if k.startswith("same_")]:
        b = key.split("_")[-1]
        k = tr._dev(g[f"k_{key}"])[None]
        bank = type("B", (), {})()
        bank.m, bank.boundary, bank.filters = k.shape[-1], BOUNDARY_CODES[b], k
        z = tr._Bank64.conv(bank, tr._dev(g[f"x_{key}"]))[0, 0].cpu().numpy()
        a = tr._Bank64.adjoint(bank, tr._dev(g[f"y_{key}"])[None, None])[0].cpu().numpy()
        assert np.allclose(z, g[f"same_{key}"], rtol=1e-12, atol=1e-12), key
        assert np.allclose(a, g[f"adj_{key}"], rtol=1e-12, atol=1e-12), key
    # adjointness of the whole bank: <K x, y> = <x, K^T y>
    model = fp.load_packaged_model("foe_a")
    bank = tr._Bank64(model)
    rng = np.random.default_rng(3)
    x, y = rng.normal(size=(1, 37, 41)), rng.normal(size=(1, 24, 37, 41))
    lhs = float(torch.sum(bank.conv(tr._dev(x)) * tr._dev(y)).item())
    rhs = float(torch.sum(tr._dev(x) * bank.adjoint(tr._dev(y))).item())
    assert abs(lhs - rhs) <= 1e-12 * abs(lhs)


def _training_case(g, tag):
    from paper_1609_05722_b200 import training as tr
    if tag == "a":
        model, objective = fp.load_packaged_model("foe_a"), "anscombe_domain"
    elif tag == "s":
        model, objective = fp.load_packaged_model("foe_s"), "original_domain"
    else:
        model = fp.FoEModel(basis=fp.dct_basis(5), betas=g["tr_per_betas"], weights=g["tr_per_weights"],
                            domain_tag="anscombe", boundary="periodic")
        objective = "anscombe_domain"
    smp = tr.TrainingSample.create(g["tr_clean"], g["tr_noisy"])
    return model, objective, smp


def test_training_operators_vs_reference_golden(golden):
    """hessian_apply / total_gradient / stationarity_residual (training.py:132-174), fp64 on the
    device, vs the reference on three cases (anscombe foe_a, original-domain foe_s, periodic bank)."""
    from paper_1609_05722_b200 import training as tr
    g = golden("training")
    for tag in ("a", "s", "p"):
        model, objective, smp = _training_case(g, tag)
        w, p = g[f"tr_{tag}_w"], g[f"tr_{tag}_p"]
        assert rel_l2(tr.hessian_apply(w, model, objective, p, smp, lam=1.3), g[f"tr_{tag}_hp"]) <= 1e-12, tag
        assert rel_l2(tr.total_gradient(w, model, smp, objective, lam=1.3), g[f"tr_{tag}_grad"]) <= 1e-12, tag
        st = tr.stationarity_residual(w, model, smp, objective, lam=1.3)
        assert abs(st - float(g[f"tr_{tag}_stat"])) <= 1e-12 * abs(st), tag


def test_hessian_cg_and_param_gradients_vs_reference_golden(golden):
    """solve_hessian_system at the reference's minimiser and param_gradients (training.py:183-356)."""
    from paper_1609_05722_b200 import training as tr
    g = golden("training")
    model, objective, smp = _training_case(g, "a")
    w_star = g["tr_wstar"]
    q, info = tr.solve_hessian_system(w_star, model, objective, g["tr_cg_rhs"], smp, 1.0, tol=1e-9, max_iters=600)
    assert abs(info["iterations"] - int(g["tr_cg_iters"])) <= 3
    assert rel_l2(q, g["tr_cg_q"]) <= 1e-8
    d_beta, d_logw = tr.param_gradients(w_star, model, smp, objective, tr.TrainConfig())
    assert rel_l2(d_beta, g["tr_dbeta"]) <= 1e-8
    assert rel_l2(d_logw, g["tr_dlogw"]) <= 1e-8


@pytest.mark.parametrize("kernel", ["ffma", "tc7"])
def test_fallback_bank_solve_vs_oracle(monkeypatch, kernel):
    """48 x 7 x 7 fallback bank through each 7x7 pass kernel (k_pass<7> FFMA, k_pass_tc7): parity gates vs the
    oracle on a 96 x 112 transform / quadratic solve (150 iterations)."""
    monkeypatch.setenv("FOE_TC7", "1" if kernel == "tc7" else "0")
    model = fp.load_packaged_model("foe_fallback48x7")
    x, y = make_counts(96, 112, 3, 2.0)
    ref = orc.denoise(y, 2.0, oracle_model(model), "transform", TABLE, force_branch="quadratic", rel_tol=0.0)
    r = fp.denoise(fp.DenoiseRequest(noisy=y, peak=2.0, model=model, variant="transform", force_branch="quadratic"),
                   fp.SolverConfig(rel_tol=0.0))
    assert len(r.trace) == 150
    _check_solve(r.image, ref["image"], 2.0, x, f"{kernel} fallback bank")


def test_tc7_matches_ffma_7x7(monkeypatch):
    """k_pass_tc7 and k_pass<7> (different tile grids, hence different fp64 reduction orders) on a 256^2 48 x 7 x 7
    solve: results within the parity gates of each other; the fused gradient at the same iterate to 1e-5."""
    model = fp.load_packaged_model("foe_fallback48x7")
    x, y = make_counts(256, 256, 5, 1.0)
    out = {}
    for k in ("0", "1"):
        monkeypatch.setenv("FOE_TC7", k)
        r = fp.denoise(fp.DenoiseRequest(noisy=y, peak=1.0, model=model, variant="transform",
                                         force_branch="quadratic"), fp.SolverConfig(rel_tol=0.0))
        out[k] = (np.asarray(r.trace.L), r.image, r.transformed.astype(np.float32).astype(np.float64))
    assert len(out["0"][0]) == len(out["1"][0]) == 150
    _check_solve(out["1"][1], out["0"][1], 1.0, x, "tc7 vs ffma")
    u = out["0"][2]  # both kernels' gradients at the same (converged, fp32) iterate
    g = {}
    for k in ("0", "1"):
        monkeypatch.setenv("FOE_TC7", k)
        g[k] = fp.foe_gradient(u, model)
    assert rel_l2(g["1"], g["0"]) <= 1e-5


def test_device_cg_restarts_and_free_set_vs_reference_golden(golden):
    """solve_hessian_system's restart rule (six escalating H + eps I attempts after non-positive curvature)
    and its free set (pinned pixels act as the identity), run as device-resident CG attempts, vs the
    reference's own outputs (tests/golden/make_golden_cg.py)."""
    import warnings
    from paper_1609_05722_b200 import training as tr
    g = golden("cg")
    smp = tr.TrainingSample.create(g["cg_clean"], g["cg_noisy"])
    fs, fa = fp.load_packaged_model("foe_s"), fp.load_packaged_model("foe_a")
    hp = tr.hessian_apply(g["brk_w"], fs, "original_domain", g["cg_rhs"], smp, lam=0.1)
    assert rel_l2(hp, g["brk_hp"]) <= 1e-12
    with warnings.catch_warnings(record=True) as wl:
        warnings.simplefilter("always")
        q, info = tr.solve_hessian_system(g["brk_w"], fs, "original_domain", g["cg_rhs"], smp, lam=0.1, tol=1e-9,
                                          max_iters=80)
    assert sum("non-positive curvature" in str(x.message) for x in wl) == 6
    assert info["iterations"] == int(g["brk_iters"])
    assert abs(info["regularization"] - float(g["brk_reg"])) <= 1e-12 * float(g["brk_reg"])
    assert len(info["residuals"]) == len(g["brk_res"])
    np.testing.assert_allclose(info["residuals"], g["brk_res"], rtol=1e-8)
    assert rel_l2(q, g["brk_q"]) <= 1e-8
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        q, info = tr.solve_hessian_system(g["free_w"], fa, "anscombe_domain", g["cg_rhs"], smp, lam=1.0, tol=1e-9,
                                          max_iters=600, free=g["free_mask"])
    assert info["iterations"] == int(g["free_iters"])
    assert abs(info["regularization"] - float(g["free_reg"])) <= 1e-12 * float(g["free_reg"])
    assert len(info["residuals"]) == len(g["free_res"])
    np.testing.assert_allclose(info["residuals"], g["free_res"], rtol=1e-6)
    assert rel_l2(q, g["free_q"]) <= 1e-8
    np.testing.assert_array_equal(q[~g["free_mask"]], g["free_q"][~g["free_mask"]])


def test_fused_hessian_apply_matches_composed_bank_operators():
    """foe_hessian_apply64 (one fused kernel) == the product composed from the fp64 bank kernels
    (conv, rho'' weighting, adjoint) + d2D, for both objectives, both boundaries, m in {3, 5, 7}, a free
    set and the eps term, to 1e-13 relative."""
    import torch
    from paper_1609_05722_b200 import training as tr
    rng = np.random.default_rng(21)
    for m, boundary, objective, shape in ((3, "symmetric", "original_domain", (37, 53)),
                                          (5, "periodic", "anscombe_domain", (40, 33)),
                                          (7, "symmetric", "anscombe_domain", (64, 70)),
                                          (5, "symmetric", "original_domain", (17, 19))):
        basis = fp.dct_basis(m)
        model = fp.FoEModel(basis=basis, betas=rng.normal(scale=0.5, size=(6, basis.n_atoms)),
                            weights=rng.uniform(0.5, 2, 6),
                            domain_tag="original" if objective == "original_domain" else "anscombe", boundary=boundary)
        bank = tr._Bank64(model)
        w = tr._dev(np.abs(rng.normal(2.0, 1.0, shape)) + 0.1)
        p = tr._dev(rng.normal(size=shape))
        f = tr._dev(rng.poisson(2.0, shape).astype(np.float64))
        free = torch.as_tensor(rng.random(shape) < 0.7, device="cuda")
        lam, eps = 0.7, 0.3
        pm = torch.where(free, p, torch.zeros_like(p))
        raw = bank.adjoint(bank.weights[None, :, None, None] * tr._rho2(bank.conv(w)) * bank.conv(pm))[0]
        if objective == "anscombe_domain":
            raw = raw + pm
        else:
            raw = raw + torch.where(f > 0, lam * f / torch.clamp(w, min=1e-150) ** 2, torch.zeros_like(w)) * pm
        want = torch.where(free, raw, p) + eps * p
        got = tr._hvp_fused(bank, w, p, objective, lam, f if objective == "original_domain" else None,
                            free.to(torch.uint8), eps)
        assert rel_l2(got.cpu().numpy(), want.cpu().numpy()) <= 1e-13, (m, boundary, objective)
