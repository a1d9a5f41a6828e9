/*
 * foe_b200.h -- C ABI of the B200-native FoE Poisson-denoise hot path.
 *
 * The reference (foepoisson, pure Python) has no FFI layer; its operator
 * boundary is a set of numpy functions.  Each entry point below replaces one
 * of them and keeps its argument meaning and error behaviour; citations are
 * /root/reference/pkg/src/foepoisson/<file>:<line>.
 *
 * Conventions
 *  - All image pointers are DEVICE pointers (row-major, contiguous), sizes are
 *    plain ints; `stream` is a cudaStream_t passed as void* (NULL = legacy).
 *  - Every call returns FOE_OK (0) or a negative FOE_E* code; the message of the
 *    last failure on the calling host thread is available from foe_last_error().
 *  - Calls are stream-ordered and re-entrant across host threads as long as
 *    each call gets its own workspace (reference: independent denoise() jobs may
 *    run concurrently, benchmark.py:117-121).
 *  - Arithmetic is fp32 on device with fp64 reductions and fp64 solver scalars;
 *    host-visible scalars (energies, trace) are fp64 like the reference.
 */
#ifndef FOE_B200_H
#define FOE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum foe_status {
    FOE_OK = 0,
    FOE_E_INVALID = -1,   /* ValueError in the reference (image.py:23-34, prior.py:87-92, solver.py:94-118) */
    FOE_E_CUDA = -2,      /* CUDA runtime failure */
    FOE_E_NUMERICAL = -3, /* NumericalFailure (solver.py:26-31) -- per-image detail in foe_image_status */
    FOE_E_UNSUPPORTED = -4
};

enum foe_boundary { FOE_SYMMETRIC = 0, FOE_PERIODIC = 1 }; /* image.py:17 BOUNDARY_RULES */
enum foe_branch { FOE_QUADRATIC = 0, FOE_IDIV = 1 };       /* pipeline.py:193-204 */

/* per-image solver outcome (solver.py:128-175) */
enum foe_solve_status {
    FOE_SOLVE_OK = 0,
    FOE_SOLVE_NONFINITE = 1, /* non-finite smooth energy (solver.py:143-144) */
    FOE_SOLVE_STALLED = 2    /* backtracking past max_lipschitz (solver.py:159-160) */
};

typedef struct foe_bank foe_bank; /* opaque device-resident filter bank */

/* SolverConfig (solver.py:34-65) */
typedef struct foe_solver_cfg {
    double gamma;            /* inertial weight, default 0.8 */
    double lipschitz_init;   /* L_{-1}, default 1.0 */
    double backtrack_factor; /* eta, default 1.2 */
    double relax_factor;     /* default 1.05 */
    double rel_tol;          /* default 1e-6 */
    double max_lipschitz;    /* default 1e15 */
} foe_solver_cfg;

/* per-image result of foe_solve; trace rows are in the caller's trace buffer */
typedef struct foe_image_status {
    int status;     /* foe_solve_status */
    int n_iters;    /* accepted iterations == len(SolverTrace) */
    int n_trials;   /* trial energies evaluated (backtracking included) */
    int failed_at;  /* iteration index of the failure, -1 if none */
} foe_image_status;

int foe_abi_version(void);
const char *foe_last_error(void);
int foe_device_sm_count(int device);
/* DenoiseRequest's count validation (pipeline.py:50-56) on a host float64 array: 0 if every value
 * is >= 0 and integral, 1 otherwise (negative, NaN or fractional); host only, no device work. */
int foe_counts_check(const double *x, size_t n);
/* the same validation that also writes every count as a float into dst (a page-locked staging buffer of the
 * binding: the H2D copy of the counts then needs no separate host pass): 0 valid, 1 invalid, 2 valid but some
 * count >= 2^24 (not exact as a float: stage the doubles instead); host only. */
int foe_counts_check_stage(const double *x, size_t n, float *dst);
/* number of CUDA kernels this library has launched in the process (launch accounting for bench.py) */
long long foe_kernel_launch_count(void);

/* ---- filter bank: FoEModel.filters (prior.py:75-78) + weights --------------------------------
 * filters: host float64 (n, m, m) in true-convolution orientation (what convolve_same takes,
 * image.py:37-58); weights: host float64 (n), strictly positive (prior.py:64-66).
 * m odd in {1,3,5,7}; n*m*m <= 4096.  Uploaded to the current device. */
int foe_bank_create(const double *filters, const double *weights, int n, int m, int boundary,
                    foe_bank **out);
int foe_bank_destroy(foe_bank *bank);
int foe_bank_info(const foe_bank *bank, int *n, int *m, int *boundary);

/* ---- elementwise ------------------------------------------------------------------------------ */
/* anscombe_forward, anscombe.py:19-24: v = 2 sqrt(y + 3/8) (y validated >= 0 by the caller) */
int foe_anscombe_forward(const double *y, float *v, int64_t n, void *stream);
/* the same from counts staged as exact floats (foe_counts_check_stage) */
int foe_anscombe_forward_f32(const float *y, float *v, int64_t n, void *stream);
/* denoise_direct obs, pipeline.py:165: obs = where(y == 0, c, y) */
int foe_direct_obs(const double *y, float *obs, double c, int64_t n, void *stream);
/* anscombe_inverse_exact_unbiased, anscombe.py:33-51; fp64 output from fp32 z.
 * counts (device, 2 x uint64, nullable): [n_clamped_input, n_clamped_output] (added to) */
int foe_anscombe_inverse_exact_unbiased(const float *z, double *x, int64_t n,
                                        unsigned long long *counts, void *stream);
/* prox_quadratic, solver.py:92-100 and prox_idiv, solver.py:103-125 (t >= 0) */
int foe_prox_quadratic(const float *u_tilde, const float *v, float *out, double t, int64_t n,
                       void *stream);
int foe_prox_idiv(const float *u_tilde, const float *obs, float *out, double t, int64_t n,
                  void *stream);

/* transform_binned (pipeline.py:214-235): bin3 (noise.py:55-71) -- factor x factor block sums with
 * bottom/right replicate padding -> yb (ceil(H/f), ceil(W/f)); unbin_bilinear (noise.py:98-113) --
 * divide by f^2, corner-aligned bilinear upsampling to the padded size, crop to (H, W).  fp64. */
int foe_bin(const double *y, double *yb, int H, int W, int factor, void *stream);
int foe_unbin_bilinear(const double *xb, double *out, int h, int w, int H, int W, int factor,
                       void *stream);

/* estimate_peak (pipeline.py:247-254, used by cli.py:69-73 when --peak is omitted): max of the 3 x 3
 * median filter (scipy "reflect" = edge-inclusive mirror boundary) of y (H x W fp64, device).
 * scratch: 8 bytes of device memory; *peak (host) is written after a stream synchronise. */
int foe_estimate_peak(const double *y, int H, int W, unsigned long long *scratch, double *peak, void *stream);

/* ---- operators ---------------------------------------------------------------------------------
 * convolve_same (image.py:37-58) / convolve_adjoint (image.py:68-83) with filter `index` of the
 * bank, B images of H x W.  Reference-operator surface for tests; the solve uses the fused pass. */
int foe_convolve_same(const foe_bank *bank, int index, const float *x, float *out, int B, int H,
                      int W, void *stream);
int foe_convolve_adjoint(const foe_bank *bank, int index, const float *y, float *out, int B, int H,
                         int W, void *stream);

/* foe_energy (prior.py:95-101) + foe_gradient (prior.py:104-110) fused in one pass.
 * u, grad: device (B, H, W) fp32; energy: device fp64 (B).  workspace >= foe_eval_workspace_size. */
size_t foe_eval_workspace_size(const foe_bank *bank, int B, int H, int W);
int foe_energy_grad(const foe_bank *bank, const float *u, float *grad, double *energy, int B, int H,
                    int W, void *workspace, size_t workspace_bytes, void *stream);

/* ---- the solver --------------------------------------------------------------------------------
 * ipiano_minimize (solver.py:128-175) with FoE callbacks (pipeline.py:167-172, 205-208) for B
 * independent images, fully device-resident: every backtracking decision is taken on the device.
 *   u0, obs      device (B,H,W) fp32: start point and data-term observation (v or y-with-c)
 *   lam, branch, max_iters   host arrays (B): data weight, foe_branch, iteration budget
 *   u_out        device (B,H,W) fp32: final iterate
 *   status       host (B) results;  trace  host (B, trace_cap, 6) fp64 rows F,G,L,step,slack,tol
 *   trace_cap >= max(max_iters).  Returns FOE_E_NUMERICAL if any image failed (others valid). */
size_t foe_solve_workspace_size(const foe_bank *bank, int B, int H, int W, int trace_cap);
int foe_solve(const foe_bank *bank, const foe_solver_cfg *cfg, int B, int H, int W,
              const float *u0, const float *obs, const double *lam, const int *branch,
              const int *max_iters, float *u_out, foe_image_status *status, double *trace,
              int trace_cap, void *workspace, size_t workspace_bytes, void *stream);

/* benchmark hook: run `reps` back-to-back trial passes of the fused kernel on the state left by
 * the last foe_solve in `workspace` without changing it (decisions suppressed). */
int foe_bench_trial_pass(const foe_bank *bank, int B, int H, int W, int trace_cap, int reps,
                         void *workspace, size_t workspace_bytes, void *stream);
/* ---- fp64 bank operators for the training side -------------------
 * filters: n x m x m fp64 in the reference orientation (FoEModel.filters), device memory.
 * foe_conv_bank64:    out[B][n][H][W] = convolve_same(x[b], filters[i])        (image.py:37-58)
 * foe_adjoint_bank64: out[B][H][W] = sum_i convolve_adjoint(y[b][i], filters[i]) (image.py:68-83)
 * boundary FOE_SYMMETRIC / FOE_PERIODIC; H, W >= m. */
int foe_conv_bank64(const double *filters, int n, int m, int boundary, const double *x, double *out, int B, int H,
                    int W, void *stream);
int foe_adjoint_bank64(const double *filters, int n, int m, int boundary, const double *y, double *out, int B, int H,
                       int W, void *stream);

/* hessian_apply (training.py:158-174), fused fp64: out = H p (+ eps p), H = sum_i wgt_i K_i^T diag(rho''(K_i w))
 * K_i + d2D, d2D = I (objective 0, anscombe_domain) or diag(lam f / max(w, 1e-150)^2 where f > 0) (objective 1,
 * original_domain); free_mask (nullable, uint8 H x W): outside it H acts as the identity and p is zeroed
 * inside the operator (solve_hessian_system's `free`, training.py:196-200).  filters: (n, m, m) reference
 * orientation, device; w, f, p, out: device H x W fp64.  One kernel per call, no N x H x W intermediate. */
int foe_hessian_apply64(const double *filters, const double *weights, int n, int m, int boundary, int objective,
                        double lam, const double *w, const double *f, const unsigned char *free_mask, const double *p,
                        double eps, double *out, int H, int W, void *stream);
/* one conjugate-gradient attempt of solve_hessian_system (training.py:203-237) on (H + eps I) q = rhs, entirely on
 * the device (rhs already masked by the caller's free set): status 1 converged (relative residual <= tol),
 * 2 non-positive curvature (the caller restarts with a larger eps, as the reference), 3 iteration cap;
 * residuals (host, max_iters + 1): relative residual history, [0] = 1; iterations = entries after [0]. */
size_t foe_cg_workspace_size(int H, int W, int max_iters);
int foe_cg_solve64(const double *filters, const double *weights, int n, int m, int boundary, int objective, double lam,
                   const double *w, const double *f, const unsigned char *free_mask, const double *rhs, double eps,
                   double tol, int max_iters, double *q, int *status, int *iterations, double *residuals,
                   int H, int W, void *workspace, size_t workspace_bytes, void *stream);

/* ---- scoring (metrics.py:30-102) ------------------------------------
 * Per image b of B (H x W fp64, row-major, device): psnr[b] and mssim[b] of x_hat against g after the
 * reference's convention (both scaled by 255 / peak, data_range 255; 11 x 11 Gaussian window,
 * sigma 1.5, valid-mode statistics, K1 = 0.01, K2 = 0.03).  fp64 arithmetic, fixed-order sums
 * (deterministic).  H, W >= 11 (ValueError in the reference otherwise). */
size_t foe_score_workspace_size(int B, int H, int W);
int foe_score(const double *x_hat, const double *g, int B, int H, int W, double peak, double *psnr,
              double *mssim, void *workspace, size_t workspace_bytes, void *stream);

/* FP32 FFMA throughput probe for the roofline denominator: launches a kernel of independent FMA
 * chains on every SM; *flop_out receives the FLOPs it executes (time it with events on `stream`).
 * `scratch` is one device float. */
int foe_measure_ffma_peak(int iters, float *scratch, double *flop_out, void *stream);
/* which fused pass a bank of m x m filters, nf of them, runs on: 1 = k_pass_tc (tcgen05 3xTF32
 * implicit GEMMs; 5 x 5 banks of <= 32 filters, default), 0 = k_pass (FFMA).  The environment
 * variable FOE_TC=0 forces the FFMA pass, FOE_TC=1 the tensor-core pass where eligible. */
int foe_pass_uses_tensor_cores(int m, int nf);
/* diagnostics: cycles (clock64, into device out_cycles[0]) for one thread to issue `nmma`
 * accumulating kind::tf32 MMAs of M = 128, N = n (32 / 64 / 128), K = 8, A in TMEM (ts = 1) or
 * shared memory (ts = 0), and observe their commit */
int foe_debug_tc_rate(int n, int ts, int nmma, int nchain, int every, long long *out_cycles, void *stream);
/* diagnostics: tcgen05.ld / st throughput with nwarps warps (out_cycles[0] = cycles for iters x 4 x 512 B per warp) */
int foe_debug_tmem_rate(int nwarps, int store, int iters, long long *out_cycles, void *stream);
/* diagnostics: the tcgen05 / TMEM primitives of the tensor-core pass on one 128 x 32 x 32 product,
 * D = A . B^T in 3xTF32 (A: 128 x 32, B: 32 x 32 row-major fp32 device arrays) */
int foe_tc_selftest(const float *A, const float *B, float *D, void *stream);
/* diagnostics: one such pass recording per-CTA %globaltimer [start, end-of-compute, exit] (ns) into
 * device `times` (3 x CTAs) */
int foe_debug_pass_times(const foe_bank *bank, int B, int H, int W, int trace_cap, void *workspace,
                         size_t workspace_bytes, unsigned long long *times, void *stream);
/* diagnostics: n_passes such passes back to back (stream order / PDL as in a solve), pass k recording
 * into times + k * (3 x CTAs + 512) */
int foe_debug_pass_times_seq(const foe_bank *bank, int B, int H, int W, int trace_cap, void *workspace,
                             size_t workspace_bytes, unsigned long long *times, int n_passes, void *stream);


/* ---- row-band decomposition (BASELINE config 5; reference has none) -------
 * A band owns global tile rows [ty0, ty1) of a B x H x W problem and keeps local rows
 * [lrow0, lrow0 + Hl) = owned rows +- halo (halo = 2r).  Per pass each band runs foe_band_trial,
 * the caller all-gathers the per-tile partials chunk [partials_offset, +partials_count) of
 * `partials` into every band's array and swaps the halo send buffers with the neighbouring bands
 * (dir 0 <-> band above, dir 1 <-> band below), then foe_band_commit takes the decision.  The
 * reduction order equals the single-device path, so any band count gives bitwise-identical
 * results.  Symmetric boundary only. */
typedef struct foe_band_desc {
    int B, H, W;          /* batch and GLOBAL image size */
    int ty0, ty1;         /* global tile rows owned by the band */
    int tiles_x, tiles_y; /* global tile grid */
    int row0, row1;       /* owned global rows */
    int lrow0, Hl;        /* local rows [lrow0, lrow0 + Hl) */
    int halo;             /* rows exchanged with each neighbour per pass */
} foe_band_desc;

typedef struct foe_band_buffers {
    double *partials;       /* device [tiles_y*tiles_x][B][8] fp64 */
    size_t partials_offset; /* doubles: this band's chunk */
    size_t partials_count;
    size_t partials_total;
    float *sendbuf, *recvbuf; /* device [2 dir][B][2 field][halo][W] */
    size_t halo_count;        /* floats per direction */
    int *n_active;            /* device live-image counter */
} foe_band_buffers;

/* tile grid / band geometry for filter side m (host-only, no device needed) */
int foe_tile_grid(int m, int H, int W, int *tiles_x, int *tiles_y);
int foe_band_geometry(int m, int B, int H, int W, int ty0, int ty1, foe_band_desc *out);
int foe_band_describe(const foe_bank *bank, int B, int H, int W, int ty0, int ty1, foe_band_desc *out);
size_t foe_band_workspace_size(const foe_bank *bank, const foe_band_desc *d, int trace_cap);
int foe_band_buffers_get(const foe_bank *bank, const foe_band_desc *d, int trace_cap, void *workspace,
                         foe_band_buffers *out);
/* u0_local, obs_local: device (B, Hl, W) rows [lrow0, lrow0+Hl) of the start point / observation */
int foe_band_begin(const foe_bank *bank, const foe_solver_cfg *cfg, const foe_band_desc *d,
                   const float *u0_local, const float *obs_local, const double *lam, const int *branch,
                   const int *max_iters, int trace_cap, void *workspace, size_t workspace_bytes,
                   void *stream);
int foe_band_trial(const foe_bank *bank, const foe_solver_cfg *cfg, const foe_band_desc *d, int trace_cap,
                   void *workspace, size_t workspace_bytes, void *stream);
int foe_band_commit(const foe_bank *bank, const foe_solver_cfg *cfg, const foe_band_desc *d, int trace_cap,
                    int init, void *workspace, size_t workspace_bytes, void *stream);
/* after the last pass: F at the final iterate, tile partials only (all-gather them as after a trial,
 * then foe_band_end sums them in the fixed order and anchors the trace's F column as foe_solve does) */
int foe_band_final_pass(const foe_bank *bank, const foe_solver_cfg *cfg, const foe_band_desc *d, int trace_cap,
                        void *workspace, size_t workspace_bytes, void *stream);
/* u_owned: device (B, row1-row0, W) final iterate rows; status/trace as foe_solve */
int foe_band_end(const foe_bank *bank, const foe_band_desc *d, int trace_cap, void *workspace,
                 size_t workspace_bytes, float *u_owned, foe_image_status *status, double *trace,
                 void *stream);

#ifdef __cplusplus
}
#endif
#endif /* FOE_B200_H */
