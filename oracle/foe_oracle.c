/*
 * foe_oracle.c -- TEST INFRASTRUCTURE ONLY (parity checker / CPU baseline).
 *
 * A plain-C, float64 restatement of the reference `foepoisson` denoise hot path
 * (arXiv 1609.05722 reference package, /root/reference/pkg/src/foepoisson).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * arm may load this library; the product path (paper_1609_05722_b200) never does.
 *
 * Every function cites the reference lines it restates.  Arithmetic is float64
 * like the reference (image.py:48, prior.py:88, solver.py:136).  Convolutions
 * are direct loops (the reference delegates them to cv2.filter2D, pinned by its
 * own naive-loop oracle in test_image.py:17-39); results agree with the
 * reference to ~1e-14 relative, which tests/test_oracle.py checks against the
 * committed golden vectors generated from the reference itself.
 *
 * OpenMP parallelises the row loops; build with oracle/Makefile.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

enum { ORC_SYMMETRIC = 0, ORC_PERIODIC = 1 };

/* np.pad "symmetric" (edge-inclusive mirror) / "wrap" index map for a padded
 * coordinate q in [-r, n + r): image.py:61-65 (_pad_index_map) and
 * image.py:54-58 (BORDER_REFLECT == np.pad symmetric; periodic via wrap). */
static inline int src_index(int q, int n, int boundary) {
    if (boundary == ORC_PERIODIC) {
        int s = q % n;
        return s < 0 ? s + n : s;
    }
    if (q < 0) return -1 - q;
    if (q >= n) return 2 * n - 1 - q;
    return q;
}

int orc_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void orc_set_num_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

/* pad x by r on every side with the boundary's index map (np.pad symmetric / wrap, image.py:54-65) */
static void pad_image(const double *x, int H, int W, int r, int boundary, double *xp) {
    const int Hp = H + 2 * r, Wp = W + 2 * r;
    int *cmap = (int *)malloc(sizeof(int) * Wp);
    for (int j = 0; j < Wp; ++j) cmap[j] = src_index(j - r, W, boundary);
#pragma omp parallel for schedule(static)
    for (int i = 0; i < Hp; ++i) {
        const double *row = x + (size_t)src_index(i - r, H, boundary) * W;
        double *o = xp + (size_t)i * Wp;
        for (int j = 0; j < Wp; ++j) o[j] = row[cmap[j]];
    }
    free(cmap);
}

/* out[y][x] = sum_{a,b} kf[a][b] xp[y + a][x + b] over the padded image (row pitch Wp), accumulated tap
 * by tap in (a, b) order */
static void conv_padded(const double *xp, int Wp, int H, int W, const double *kf, int m, double *out) {
#pragma omp parallel for schedule(static)
    for (int y = 0; y < H; ++y) {
        double *o = out + (size_t)y * W;
        for (int xx = 0; xx < W; ++xx) o[xx] = 0.0;
        for (int a = 0; a < m; ++a) {
            const double *in = xp + (size_t)(y + a) * Wp;
            for (int b = 0; b < m; ++b) {
                const double w = kf[a * m + b];
                const double *inb = in + b;
                for (int xx = 0; xx < W; ++xx) o[xx] += w * inb[xx];
            }
        }
    }
}

static void flip_kernel(const double *k, int m, double *kf) {
    for (int a = 0; a < m; ++a)
        for (int b = 0; b < m; ++b) kf[a * m + b] = k[(m - 1 - a) * m + (m - 1 - b)];
}

/* convolve_same, image.py:37-58: true 2-D convolution, "same" output,
 * z[p] = sum_{a,b} kf[a,b] * u_ext[p + (a - r, b - r)],  kf = k[::-1, ::-1]. */
void orc_convolve_same(const double *x, int H, int W, const double *k, int m,
                       int boundary, double *out) {
    const int r = m / 2;
    if (r == 0) { /* image.py:51-52 */
        for (long i = 0; i < (long)H * W; ++i) out[i] = x[i] * k[0];
        return;
    }
    const int Hp = H + 2 * r, Wp = W + 2 * r;
    double *xp = (double *)malloc(sizeof(double) * (size_t)Hp * Wp);
    pad_image(x, H, W, r, boundary, xp);
    double kf[49];
    flip_kernel(k, m, kf);
    conv_padded(xp, Wp, H, W, kf, m, out);
    free(xp);
}

/* convolve_adjoint, image.py:68-83: V^T psi = full correlation of the
 * zero-padded input with the unflipped kernel on the padded domain
 * (image.py:76-79), then P^T folds every padded pixel onto its source pixel
 * in padded row-major order (image.py:80-83, np.bincount).  The fold runs in
 * parallel over destination rows; each destination pixel still receives its
 * contributions in padded row-major order, so the sums are the serial ones. */
void orc_convolve_adjoint(const double *y, int H, int W, const double *k, int m,
                          int boundary, double *out) {
    const int r = m / 2;
    if (r == 0) { /* image.py:82-83 */
        for (long i = 0; i < (long)H * W; ++i) out[i] = y[i] * k[0];
        return;
    }
    const int Hp = H + 2 * r, Wp = W + 2 * r;
    /* zero-padded by r (np.pad(y, r)), then a further r of zero border so the
     * correlation window never leaves the buffer (BORDER_CONSTANT) */
    const int Hz = Hp + 2 * r, Wz = Wp + 2 * r;
    double *yz = (double *)calloc((size_t)Hz * Wz, sizeof(double));
#pragma omp parallel for schedule(static)
    for (int i = 0; i < H; ++i)
        memcpy(yz + (size_t)(i + 2 * r) * Wz + 2 * r, y + (size_t)i * W, sizeof(double) * W);
    double *g = (double *)malloc(sizeof(double) * (size_t)Hp * Wp);
#pragma omp parallel for schedule(static)
    for (int q = 0; q < Hp; ++q) {
        double *o = g + (size_t)q * Wp;
        for (int xx = 0; xx < Wp; ++xx) o[xx] = 0.0;
        for (int a = 0; a < m; ++a) {
            const double *in = yz + (size_t)(q + a) * Wz;
            for (int b = 0; b < m; ++b) {
                const double w = k[a * m + b];
                const double *inb = in + b;
                for (int xx = 0; xx < Wp; ++xx) o[xx] += w * inb[xx];
            }
        }
    }
    int *cmap = (int *)malloc(sizeof(int) * Wp);
    for (int j = 0; j < Wp; ++j) cmap[j] = src_index(j - r, W, boundary);
    /* source padded rows of every destination row, ascending (at most 3: itself and two folds) */
    int *nsrc = (int *)calloc(H, sizeof(int));
    int *srcs = (int *)malloc(sizeof(int) * 4 * (size_t)H);
    for (int q = 0; q < Hp; ++q) {
        const int d = src_index(q - r, H, boundary);
        if (nsrc[d] < 4) srcs[4 * d + nsrc[d]++] = q;
    }
#pragma omp parallel for schedule(static)
    for (int d = 0; d < H; ++d) {
        double *dst = out + (size_t)d * W;
        for (int j = 0; j < W; ++j) dst[j] = 0.0;
        for (int t = 0; t < nsrc[d]; ++t) {
            const double *s = g + (size_t)srcs[4 * d + t] * Wp;
            for (int j = 0; j < Wp; ++j) dst[cmap[j]] += s[j];
        }
    }
    free(srcs);
    free(nsrc);
    free(cmap);
    free(g);
    free(yz);
}

/* sum of log1p(z^2) over an H x W response: per-row sums in parallel, then the rows in order -- the
 * same result for any thread count (numpy's pairwise sum differs by ~1e-16 relative, covered by the
 * golden tolerances) */
static double sum_log1p_sq(const double *z, int H, int W, double *row_sums) {
#pragma omp parallel for schedule(static)
    for (int y = 0; y < H; ++y) {
        const double *zr = z + (size_t)y * W;
        double s = 0.0;
        for (int x = 0; x < W; ++x) s += log1p(zr[x] * zr[x]);
        row_sums[y] = s;
    }
    double t = 0.0;
    for (int y = 0; y < H; ++y) t += row_sums[y];
    return t;
}

/* foe_energy, prior.py:95-101: sum_i w_i sum_p log1p((k_i * u)_p^2)
 * (potential order 0, prior.py:23-35).  u is padded once for all filters. */
double orc_foe_energy(const double *u, int H, int W, const double *filters,
                      const double *weights, int N, int m, int boundary) {
    const long n = (long)H * W;
    const int r = m / 2, Hp = H + 2 * r, Wp = W + 2 * r;
    double *z = (double *)malloc(sizeof(double) * n);
    double *xp = (double *)malloc(sizeof(double) * (size_t)Hp * Wp);
    double *rs = (double *)malloc(sizeof(double) * H);
    pad_image(u, H, W, r, boundary, xp);
    double total = 0.0;
    for (int i = 0; i < N; ++i) {
        double kf[49];
        flip_kernel(filters + (size_t)i * m * m, m, kf);
        conv_padded(xp, Wp, H, W, kf, m, z);
        total += weights[i] * sum_log1p_sq(z, H, W, rs);
    }
    free(rs);
    free(xp);
    free(z);
    return total;
}

/* foe_gradient, prior.py:104-110: sum_i w_i K_i^T rho'(K_i u),
 * rho'(z) = 2z / (1 + z^2) (prior.py:31-32). */
void orc_foe_gradient(const double *u, int H, int W, const double *filters,
                      const double *weights, int N, int m, int boundary, double *grad) {
    const long n = (long)H * W;
    const int r = m / 2, Hp = H + 2 * r, Wp = W + 2 * r;
    double *z = (double *)malloc(sizeof(double) * n);
    double *a = (double *)malloc(sizeof(double) * n);
    double *xp = (double *)malloc(sizeof(double) * (size_t)Hp * Wp);
    pad_image(u, H, W, r, boundary, xp);
#pragma omp parallel for schedule(static)
    for (long p = 0; p < n; ++p) grad[p] = 0.0;
    for (int i = 0; i < N; ++i) {
        const double *k = filters + (size_t)i * m * m;
        double kf[49];
        flip_kernel(k, m, kf);
        if (r == 0) {
            for (long p = 0; p < n; ++p) z[p] = u[p] * k[0];
        } else {
            conv_padded(xp, Wp, H, W, kf, m, z);
        }
#pragma omp parallel for schedule(static)
        for (long p = 0; p < n; ++p) z[p] = 2.0 * z[p] / (1.0 + z[p] * z[p]);
        orc_convolve_adjoint(z, H, W, k, m, boundary, a);
        const double w = weights[i];
#pragma omp parallel for schedule(static)
        for (long p = 0; p < n; ++p) grad[p] += w * a[p];
    }
    free(xp);
    free(a);
    free(z);
}

/* prox_quadratic, solver.py:92-100: (u_tilde + t v) / (1 + t). */
void orc_prox_quadratic(const double *ut, const double *v, double t, long n, double *out) {
#pragma omp parallel for schedule(static)
    for (long i = 0; i < n; ++i) out[i] = (ut[i] + t * v[i]) / (1.0 + t);
}

/* prox_idiv, solver.py:103-125: cancellation-free root of
 * u^2 - (u_tilde - t) u - t obs = 0; 0 where obs == 0 and a < 0; t == 0 copies. */
void orc_prox_idiv(const double *ut, const double *obs, double t, long n, double *out) {
    if (t == 0.0) {
        memcpy(out, ut, sizeof(double) * n);
        return;
    }
#pragma omp parallel for schedule(static)
    for (long i = 0; i < n; ++i) {
        const double a = ut[i] - t;
        const double root = sqrt(a * a + 4.0 * t * obs[i]);
        double o = (a >= 0.0) ? (a + root) / 2.0 : 2.0 * t * obs[i] / (root - a);
        if (obs[i] == 0.0 && a < 0.0) o = 0.0;
        out[i] = o;
    }
}

/* anscombe_forward, anscombe.py:19-24 (caller validates y >= 0). */
void orc_anscombe_forward(const double *y, long n, double *v) {
    for (long i = 0; i < n; ++i) v[i] = 2.0 * sqrt(y[i] + 0.375);
}

/* anscombe_inverse_exact_unbiased, anscombe.py:33-51; counts[0] = inputs
 * clamped up to sqrt(1.5), counts[1] = outputs clamped to 0 (not already low). */
void orc_anscombe_inverse_exact_unbiased(const double *z, long n, double *x, long *counts) {
    const double S = sqrt(1.5);
    long c0 = 0, c1 = 0;
    for (long i = 0; i < n; ++i) {
        const int low = z[i] < S;
        const double zc = low ? S : z[i];
        const double v = zc * zc / 4.0 + S / (4.0 * zc) - 11.0 / (8.0 * zc * zc) +
                         5.0 * S / (8.0 * zc * zc * zc) - 0.125;
        const int neg = v < 0.0;
        c0 += low;
        c1 += (neg && !low);
        x[i] = neg ? 0.0 : v;
    }
    if (counts) {
        counts[0] = c0;
        counts[1] = c1;
    }
}

/* energy_G of the two data terms: quadratic 0.5*lam*|u - v|^2 (pipeline.py:200)
 * and _idiv_energy (pipeline.py:141-149). */
static double energy_G(const double *u, const double *obs, long n, double lam, int branch) {
    if (branch == 0) {
        double s = 0.0;
        for (long i = 0; i < n; ++i) {
            const double d = u[i] - obs[i];
            s += d * d;
        }
        return 0.5 * lam * s;
    }
    double val = 0.0, lg = 0.0;
    for (long i = 0; i < n; ++i) {
        val += u[i];
        if (obs[i] > 0) {
            if (u[i] <= 0) return INFINITY;
            lg += obs[i] * log(u[i]);
        }
    }
    return lam * (val - lg);
}

/* ipiano_minimize, solver.py:128-175, with the FoE callbacks of
 * pipeline.py:167-172 / 205-208 and prox by branch (0 quadratic, 1 idiv).
 * trace rows (per accepted iteration): F, G, L, step_norm, slack, slack_tol.
 * Returns 0 ok, 1 non-finite f_u (solver.py:143-144), 2 backtracking stalled
 * (solver.py:159-160).  *n_iters = accepted iterations; *n_trials = energy
 * evaluations of trial points. */
/* iterates (nullable): (max_iters, H * W) fp32 copies of each accepted iterate, for the per-iteration
 * gradient check of the GPU path (the device state is fp32, so the check runs at the fp32 iterate). */
int orc_ipiano_foe_ex(const double *u0, const double *obs, int H, int W,
                      const double *filters, const double *weights, int N, int m, int boundary,
                      double lam, int branch, double gamma, double L0, double eta, double relax,
                      int max_iters, double rel_tol, double max_L,
                      double *u_out, double *trace, int *n_iters, int *n_trials, float *iterates) {
    const double SLACK_RTOL = 1e-12; /* solver.py:23 */
    const long n = (long)H * W;
    double *u = (double *)malloc(sizeof(double) * n);
    double *up = (double *)malloc(sizeof(double) * n);
    double *un = (double *)malloc(sizeof(double) * n);
    double *ut = (double *)malloc(sizeof(double) * n);
    double *g = (double *)malloc(sizeof(double) * n);
    memcpy(u, u0, sizeof(double) * n);
    memcpy(up, u0, sizeof(double) * n);
    double L = L0;
    int status = 0, it = 0, trials = 0;
    for (int k = 0; k < max_iters; ++k) {
        const double f_u = orc_foe_energy(u, H, W, filters, weights, N, m, boundary);
        if (!isfinite(f_u)) { status = 1; break; }
        orc_foe_gradient(u, H, W, filters, weights, N, m, boundary, g);
        double f_new, sq, gd, slack, tol;
        for (;;) {
            const double tau = 1.99 * (1.0 - gamma) / L; /* solver.py:64-65 */
            for (long i = 0; i < n; ++i) ut[i] = u[i] - tau * g[i] + gamma * (u[i] - up[i]);
            if (branch == 0) orc_prox_quadratic(ut, obs, tau * lam, n, un);
            else orc_prox_idiv(ut, obs, tau * lam, n, un);
            f_new = orc_foe_energy(un, H, W, filters, weights, N, m, boundary);
            ++trials;
            sq = 0.0;
            gd = 0.0;
            for (long i = 0; i < n; ++i) {
                const double du = un[i] - u[i];
                sq += du * du;
                gd += g[i] * du;
            }
            slack = f_new - (f_u + gd + 0.5 * L * sq);
            tol = SLACK_RTOL * (fabs(f_u) + fabs(f_new) + fabs(gd) + 0.5 * L * sq);
            if (isfinite(f_new) && slack <= tol) break;
            L *= eta;
            if (L > max_L) { status = 2; break; }
        }
        if (status) break;
        const double step = sqrt(sq);
        double *row = trace + (size_t)it * 6;
        row[0] = f_new;
        row[1] = energy_G(un, obs, n, lam, branch);
        row[2] = L;
        row[3] = step;
        row[4] = slack;
        row[5] = tol;
        if (iterates) {
            float *dst = iterates + (size_t)it * n;
            for (long i = 0; i < n; ++i) dst[i] = (float)un[i];
        }
        ++it;
        double unorm = 0.0;
        for (long i = 0; i < n; ++i) unorm += u[i] * u[i];
        unorm = sqrt(unorm);
        double *tmp = up;
        up = u;
        u = un;
        un = tmp;
        L /= relax;
        if (step < rel_tol * (unorm > 1e-300 ? unorm : 1e-300)) break;
    }
    memcpy(u_out, u, sizeof(double) * n);
    *n_iters = it;
    *n_trials = trials;
    free(u); free(up); free(un); free(ut); free(g);
    return status;
}

int orc_ipiano_foe(const double *u0, const double *obs, int H, int W,
                   const double *filters, const double *weights, int N, int m, int boundary,
                   double lam, int branch, double gamma, double L0, double eta, double relax,
                   int max_iters, double rel_tol, double max_L,
                   double *u_out, double *trace, int *n_iters, int *n_trials) {
    return orc_ipiano_foe_ex(u0, obs, H, W, filters, weights, N, m, boundary, lam, branch, gamma, L0, eta, relax,
                             max_iters, rel_tol, max_L, u_out, trace, n_iters, n_trials, NULL);
}
