"""Generate golden vectors from the REFERENCE implementation (run in the dev container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Imports the reference ``foepoisson`` package read-only from /root/reference and
writes small .npz fixtures next to this script, plus the packaged model banks
and lambda table (re-serialised with the reference's own ``save_model`` / json)
into ``paper_1609_05722_b200/assets``.  The GPU box never runs this script; the
committed outputs travel instead.
"""

from __future__ import annotations

import dataclasses
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from foepoisson import anscombe, fileio, image, pipeline, prior, solver  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
from paper_1609_05722_b200.synth import make_counts  # noqa: E402

ASSETS = os.path.join(REPO, "paper_1609_05722_b200", "assets")


def trace_arrays(tr):
    return np.array([tr.F, tr.G, tr.L, tr.step_norm, tr.descent_slack, tr.slack_tol]).T


def fallback_bank(seed: int = 1609):
    """48 zero-mean unit-norm 7x7 filters (dct7, unit-norm beta rows), alpha ~ U[0.5, 2]."""
    rng = np.random.Generator(np.random.Philox(key=seed))
    basis = image.dct_basis(7)
    betas = rng.standard_normal((48, basis.n_atoms))
    betas /= np.linalg.norm(betas, axis=1, keepdims=True)
    weights = rng.uniform(0.5, 2.0, size=48)
    return prior.FoEModel(basis=basis, betas=betas, weights=weights, domain_tag="anscombe")


def random_model(rng, n_filters, m, domain_tag="original", boundary="symmetric"):
    basis = image.dct_basis(m)
    betas = rng.normal(scale=0.5, size=(n_filters, basis.n_atoms))
    weights = rng.uniform(0.5, 2.0, size=n_filters)
    return prior.FoEModel(basis=basis, betas=betas, weights=weights, domain_tag=domain_tag, boundary=boundary)


def main():
    os.makedirs(ASSETS, exist_ok=True)
    foe_a = fileio.load_packaged_model("foe_a")
    foe_s = fileio.load_packaged_model("foe_s")
    fileio.save_model(os.path.join(ASSETS, "foe_a.foe"), foe_a)
    fileio.save_model(os.path.join(ASSETS, "foe_s.foe"), foe_s)
    fileio.save_model(os.path.join(ASSETS, "foe_fallback48x7.foe"), fallback_bank())
    with open(os.path.join(ASSETS, "lambda_table.json"), "w") as fh:
        json.dump(pipeline._load_table(), fh, indent=1)

    # --- convolution operators (image.py:37-83) -------------------------------------------
    out = {}
    rng = np.random.default_rng(7)
    for shape in [(12, 17), (31, 26)]:
        x = rng.normal(size=shape)
        y = rng.normal(size=shape)
        for m in (1, 3, 5, 7):
            k = rng.normal(size=(m, m))
            for b in image.BOUNDARY_RULES:
                key = f"{shape[0]}x{shape[1]}_m{m}_{b}"
                out[f"x_{key}"] = x
                out[f"y_{key}"] = y
                out[f"k_{key}"] = k
                out[f"same_{key}"] = image.convolve_same(x, k, b)
                out[f"adj_{key}"] = image.convolve_adjoint(y, k, b)
    np.savez_compressed(os.path.join(HERE, "conv.npz"), **out)

    # --- FoE energy / gradient (prior.py:95-110) --------------------------------------------
    out = {}
    _, y = make_counts(40, 36, 3, 4.0)
    v = anscombe.anscombe_forward(y)
    cases = {
        "foe_a": (foe_a, v),
        "foe_s": (foe_s, y + 0.5),
        "fallback": (fallback_bank(), v),
        "rand_periodic": (random_model(np.random.default_rng(5), 3, 5, boundary="periodic"), v),
        "rand_m7_sym": (random_model(np.random.default_rng(6), 4, 7), v[:13, :11].copy()),
        "rand_m3_periodic_tiny": (random_model(np.random.default_rng(8), 2, 3, boundary="periodic"),
                                  np.random.default_rng(9).normal(size=(5, 7)) + 3.0),
    }
    for name, (model, u) in cases.items():
        out[f"u_{name}"] = u
        out[f"filters_{name}"] = model.filters
        out[f"weights_{name}"] = model.weights
        out[f"boundary_{name}"] = np.array(model.boundary)
        out[f"energy_{name}"] = np.array(prior.foe_energy(u, model))
        out[f"grad_{name}"] = prior.foe_gradient(u, model)
    np.savez_compressed(os.path.join(HERE, "prior.npz"), **out)

    # --- prox + anscombe (solver.py:92-125, anscombe.py:19-51) -------------------------------
    rng = np.random.default_rng(11)
    ut = rng.normal(scale=3.0, size=(9, 11))
    obs = rng.poisson(2.0, size=(9, 11)).astype(float)
    obs[0, :4] = 0.0
    ut[0, :2] = -1.0
    z = np.concatenate([np.linspace(0.0, 3.0, 61), np.array([1.2247, 1.2248, 10.0, 100.0, 1e4])])
    diag = {}
    out = {"ut": ut, "obs": obs, "z": z,
           "pq_0.7": solver.prox_quadratic(ut, 0.7, obs), "pq_0": solver.prox_quadratic(ut, 0.0, obs),
           "pi_0.7": solver.prox_idiv(ut, 0.7, obs), "pi_0": solver.prox_idiv(ut, 0.0, obs),
           "pi_3.5": solver.prox_idiv(ut, 3.5, obs),
           "ans_fwd": anscombe.anscombe_forward(obs),
           "ans_inv": anscombe.anscombe_inverse_exact_unbiased(z, diag)}
    out["ans_inv_counts"] = np.array([diag["n_clamped_input"], diag["n_clamped_output"]])
    np.savez_compressed(os.path.join(HERE, "elementwise.npz"), **out)

    # --- full denoise, small images (pipeline.py:152-244) -------------------------------------
    out = {}
    cfg = solver.SolverConfig(rel_tol=0.0)
    foe_a_orig = dataclasses.replace(foe_a, domain_tag="original")
    jobs = [
        ("t_quad_p4", 37, 45, 0, 4.0, foe_a, "transform", "quadratic", cfg),
        ("t_idiv_p4", 37, 45, 0, 4.0, foe_a, "transform", None, cfg),
        ("t_quad_p1", 32, 32, 1, 1.0, foe_a, "transform", "quadratic", cfg),
        ("t_idiv_p05", 29, 33, 2, 0.5, foe_a, "transform", None, cfg),
        ("t_quad_p8", 33, 29, 4, 8.0, foe_a, "transform", None, cfg),
        ("d_fa_p8", 32, 40, 1, 8.0, foe_a_orig, "direct", None, cfg),
        ("d_fs_p8", 32, 40, 1, 8.0, foe_s, "direct", None, cfg),
        ("t_fb_p2", 30, 30, 5, 2.0, fallback_bank(), "transform", "quadratic", cfg),
        ("t_quad_reltol", 24, 24, 6, 2.0, foe_a, "transform", "quadratic", solver.SolverConfig()),
    ]
    for name, H, W, seed, peak, model, variant, fb, scfg in jobs:
        x, y = make_counts(H, W, seed, peak)
        req = pipeline.DenoiseRequest(noisy=y, peak=peak, model=model, variant=variant, force_branch=fb)
        r = pipeline.denoise(req, scfg)
        out[f"{name}_noisy"] = y
        out[f"{name}_clean"] = x
        out[f"{name}_image"] = r.image
        out[f"{name}_transformed"] = r.transformed if r.transformed is not None else np.zeros(0)
        out[f"{name}_trace"] = trace_arrays(r.trace)
        out[f"{name}_meta"] = np.array([peak, r.lam, H, W, seed, float(scfg.rel_tol)])
        out[f"{name}_branch"] = np.array(r.branch)
        print(name, r.branch, r.lam, len(r.trace))
    np.savez_compressed(os.path.join(HERE, "denoise_small.npz"), **out)

    # --- transform_binned (pipeline.py:214-235, noise.py:55-113) -----------------------------------
    out = {}
    for name, H, W, seed, peak, fb, bf in [("b_p05", 61, 50, 3, 0.5, None, 3), ("b_p02_quad", 49, 47, 8, 0.2, "quadratic", 3),
                                           ("b_f1", 30, 31, 9, 1.0, None, 1), ("b_f2", 41, 37, 10, 0.4, None, 2)]:
        x, y = make_counts(H, W, seed, peak)
        req = pipeline.DenoiseRequest(noisy=y, peak=peak, model=foe_a, variant="transform_binned", force_branch=fb,
                                      bin_factor=bf)
        r = pipeline.denoise(req, cfg)
        from foepoisson import noise
        out[f"{name}_noisy"] = y
        out[f"{name}_clean"] = x
        out[f"{name}_binned"] = noise.bin3(y, bf)
        out[f"{name}_image"] = r.image
        out[f"{name}_trace"] = trace_arrays(r.trace)
        out[f"{name}_meta"] = np.array([peak, r.lam, H, W, seed, bf, r.peak_used])
        out[f"{name}_branch"] = np.array(r.branch)
        up = noise.unbin_bilinear(r.transformed, (H, W), bf)
        out[f"{name}_unbin_of_transformed"] = up
        print(name, r.branch, r.lam, len(r.trace), r.peak_used)
    np.savez_compressed(os.path.join(HERE, "binned.npz"), **out)

    # --- scoring (metrics.py:30-102) and the evaluation grid (benchmark.py:32-122) ------------------
    # benchmark.py imports data.py, which needs scikit-image (absent here) only for its image
    # roster; the grid below passes its own loader, so a stub module satisfies the import
    import types
    if "skimage" not in sys.modules:
        stub = types.ModuleType("skimage")
        stub.data = types.ModuleType("skimage.data")
        sys.modules["skimage"], sys.modules["skimage.data"] = stub, stub.data
    from foepoisson import benchmark, metrics
    out = {}
    rng = np.random.default_rng(5)
    for i, (H, W, peak) in enumerate([(11, 11, 1.0), (37, 53, 4.0), (64, 64, 0.5), (20, 90, 40.0)]):
        g = rng.uniform(0, peak, size=(H, W))
        xh = np.clip(g + rng.normal(scale=0.1 * peak, size=(H, W)), 0, None)
        sc = metrics.score_denoised(xh, g, peak)
        out[f"m{i}_xhat"], out[f"m{i}_g"] = xh, g
        out[f"m{i}_ref"] = np.array([peak, sc.psnr_db, sc.mssim])
    np.savez_compressed(os.path.join(HERE, "metrics.npz"), **out)
    from paper_1609_05722_b200.evaluate import synthetic_eval_image
    foe_s = fileio.load_packaged_model("foe_s")
    spec = benchmark.BenchmarkSpec(images=("syn40x36s1", "syn33x47s2"), peaks=(0.5, 2.0, 8.0),
                                   variants=("transform", "transform_binned", "direct"), transform_model=foe_a,
                                   direct_model=foe_s, base_seed=7)
    rows = benchmark.run_benchmark(spec, image_loader=synthetic_eval_image, workers=1)
    out = {"rows_num": np.array([[r.peak, r.psnr_db, r.mssim, r.lam] for r in rows]),
           "rows_key": np.array([f"{r.image}|{r.variant}|{r.branch}" for r in rows]),
           "row_seeds": np.array([r.seed for r in rows], dtype=np.uint64),
           "seeds": np.array([benchmark.job_seed(n, p, v, 7) for n in ("a", "syn40x36s1") for p in (0.5, 40.0)
                              for v in ("transform", "direct")], dtype=np.uint64)}
    np.savez_compressed(os.path.join(HERE, "bench_grid.npz"), **out)
    for r in rows:
        print("grid", r.image, r.peak, r.variant, r.branch, round(r.psnr_db, 4), round(r.mssim, 5))

    # --- training operators (training.py:132-356), small patches -----------------------------------
    from foepoisson import training
    from paper_1609_05722_b200.synth import synthetic_clean, sample_poisson
    out = {}
    rng = np.random.default_rng(11)
    clean = 4.0 * synthetic_clean(24, 28, 5)
    noisy = sample_poisson(clean, 5)
    smp = training.TrainingSample.create(clean, noisy)
    out["tr_clean"], out["tr_noisy"] = clean, noisy
    foe_s = fileio.load_packaged_model("foe_s")
    per = random_model(rng, 6, 5, domain_tag="anscombe", boundary="periodic")
    out["tr_per_betas"], out["tr_per_weights"] = per.betas, per.weights
    for tag, model, objective in (("a", foe_a, "anscombe_domain"), ("s", foe_s, "original_domain"),
                                  ("p", per, "anscombe_domain")):
        w = smp.transformed + rng.normal(scale=0.3, size=clean.shape) if objective == "anscombe_domain" \
            else noisy + 0.5 + rng.uniform(0, 0.5, size=clean.shape)
        pv = rng.normal(size=clean.shape)
        out[f"tr_{tag}_w"], out[f"tr_{tag}_p"] = w, pv
        out[f"tr_{tag}_hp"] = training.hessian_apply(w, model, objective, pv, smp, lam=1.3)
        out[f"tr_{tag}_grad"] = training.total_gradient(w, model, smp, objective, lam=1.3)
        out[f"tr_{tag}_stat"] = np.array(training.stationarity_residual(w, model, smp, objective, lam=1.3))
    cfg_t = training.TrainConfig()
    w_star = training.lower_solve(smp, foe_a, "anscombe_domain", cfg_t)
    rhs = rng.normal(size=clean.shape)
    q, info = training.solve_hessian_system(w_star, foe_a, "anscombe_domain", rhs, smp, 1.0, tol=1e-9, max_iters=600)
    out["tr_cg_rhs"], out["tr_cg_q"], out["tr_cg_iters"] = rhs, q, np.array(info["iterations"])
    d_beta, d_logw = training.param_gradients(w_star, foe_a, smp, "anscombe_domain", cfg_t)
    out["tr_wstar"], out["tr_dbeta"], out["tr_dlogw"] = w_star, d_beta, d_logw
    np.savez_compressed(os.path.join(HERE, "training.npz"), **out)
    print("training", info["iterations"], float(np.abs(d_beta).max()), float(np.abs(d_logw).max()))

    if os.environ.get("GOLDEN_SKIP_CFG1"):
        return
    # --- BASELINE config 1 at full size (256^2, peak 4, quadratic forced, foe_a) ----------------
    x, y = make_counts(256, 256, 0, 4.0)
    req = pipeline.DenoiseRequest(noisy=y, peak=4.0, model=foe_a, variant="transform", force_branch="quadratic")
    r = pipeline.denoise(req, cfg)
    np.savez_compressed(os.path.join(HERE, "cfg1_256.npz"), image=r.image.astype(np.float32),
                        trace=trace_arrays(r.trace), counts_sum=np.array(y.sum()),
                        counts_hash=np.array(float(np.sum(y * np.arange(y.size).reshape(y.shape) % 1009))),
                        lam=np.array(r.lam))
    print("cfg1", r.lam, len(r.trace))


if __name__ == "__main__":
    main()
