// foe_train64.cuh -- training-side Hessian operator and its conjugate-gradient solve, fp64 (included by
// foe_b200.cu after the bank64 kernels).  Reference: training.py:158-237.
//
//   H p = sum_i wgt_i K_i^T diag(rho''(K_i w)) K_i p + d2D p            (hessian_apply, training.py:158-174)
//
// k_cg_hvp computes H p for a 16 x 16 output tile in one pass: w and p are staged with a 2r ring (the
// boundary's index map), and per filter the tile + r ring gets c_i = wgt_i rho''(K_i w) (K_i p) (zero
// outside the image for the symmetric rule, psi_0 of image.py:76-79), whose exact adjoint -- with the
// P^T fold of image.py:80-83 resolved per output pixel -- accumulates into H p.  No N x H x W response
// is materialised: K_i w is recomputed per call (constant over the CG solve, but 24 x 8 B per pixel
// of HBM traffic would cost as much as the recompute).
//
// The CG of solve_hessian_system (training.py:183-237) runs on the device: a CUDA graph whose
// conditional WHILE node repeats [k_cg_hvp -> k_cg_update] until the residual test, a non-positive-
// curvature breakdown or the iteration cap ends the attempt.  k_cg_hvp also forms the search direction
// d = r + beta d_prev while staging (double-buffered d) and its CTAs' partial <d, Hd>, <d, d>; the last
// CTA (ticket) reduces them in a fixed order into alpha (or flags the breakdown).  k_cg_update applies
// q += alpha d, r -= alpha Hd and its last CTA reduces <r, r> into the residual history, the stop test
// and beta.  The host sees one synchronise per CG attempt; restarts with H + eps I stay on the host,
// as in the reference (at most six).

constexpr int kHT = 16;          // output tile side (256 threads)
constexpr int kCgUpdCtas = 296;  // 2 x 148 SMs, grid-stride elementwise update

enum CgStatus { CG_RUNNING = 0, CG_CONVERGED = 1, CG_BREAKDOWN = 2, CG_MAXITER = 3 };

struct CgState {  // device scalars of one CG attempt
    double rs, alpha, beta, rhs_norm, tol;
    int it, max_iters, status, parity;
};

struct CgArgs {
    int H, W, n, objective;  // objective: 0 anscombe_domain (d2D = I), 1 original_domain (diag lam f / w^2)
    double lam, eps;         // data weight; regularisation of the restart (H + eps I)
    const double *kf, *wgt;  // filters (n, m, m) in the reference orientation, weights (n)
    const double *w, *f;     // lower iterate, observed counts (original objective)
    const unsigned char *free_mask;  // nullable: pixels outside it act as the identity (training.py:196-200)
    // operands: H p with p = r + beta * d_prev (hessian_apply: r = p, d_prev = null), written to d_next
    const double *r, *d_prev;
    double *d_next, *hp;
    double *q;  // CG iterate
    double *r_mut;
    double *part;          // [2][ctas] partial sums
    unsigned *tickets;     // [2]
    CgState *st;           // null: plain hessian_apply (beta = 0, no reductions)
    double *residuals;     // [max_iters + 1]
    cudaGraphConditionalHandle cond;
    int use_cond;
};

__device__ __forceinline__ double rho2_64(double z) {  // prior.py:33-34
    const double q = 1.0 + z * z;
    return 2.0 * (1.0 - z * z) / (q * q);
}

// fixed-order block sum of two doubles (256 threads) -> thread 0
__device__ __forceinline__ void block_sum2(double &a, double &b, double (*red)[2]) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        a += __shfl_down_sync(0xffffffffu, a, off);
        b += __shfl_down_sync(0xffffffffu, b, off);
    }
    if (lane == 0) { red[warp][0] = a; red[warp][1] = b; }
    __syncthreads();
    if (threadIdx.x == 0) {
        a = 0.0; b = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { a += red[w][0]; b += red[w][1]; }
    }
}

template <int M, bool SYM>
__global__ void __launch_bounds__(256) k_cg_hvp(const CgArgs a) {
    constexpr int R = M / 2, SP = kHT + 4 * R, SC = kHT + 2 * R;
    __shared__ double ws[SP * SP], ps[SP * SP], cs[SC * SC];
    __shared__ double red[8][2];
    __shared__ int s_last;
    const int tid = threadIdx.x, H = a.H, W = a.W;
    if (a.st && a.st->status != CG_RUNNING) return;
    const double beta = a.st ? a.st->beta : 0.0;
    const double *dprev = a.d_prev;
    double *dnext = a.d_next;
    if (a.st && a.st->parity) {  // double-buffered search direction: the pair swaps every iteration
        dprev = a.d_next;
        dnext = const_cast<double *>(a.d_prev);
    }
    const int y0 = blockIdx.y * kHT, x0 = blockIdx.x * kHT;
    // stage w and the direction p = r + beta d_prev (zero outside the free set) with a 2r ring
    for (int e = tid; e < SP * SP; e += 256) {
        const int sy = src_idx<SYM>(y0 - 2 * R + e / SP, H), sx = src_idx<SYM>(x0 - 2 * R + e % SP, W);
        const size_t o = (size_t)sy * W + sx;
        ws[e] = a.w[o];
        double p = a.r[o];
        if (dprev && beta != 0.0) p = fma(beta, dprev[o], p);  // training.py:231
        if (a.free_mask && !a.free_mask[o]) p = 0.0;
        ps[e] = p;
    }
    const int ty = tid / kHT, tx = tid % kHT, qy = y0 + ty, qx = x0 + tx;
    const bool inside = qy < H && qx < W;
    // P^-1(q): padded positions whose source pixel is q (image.py:61-66); periodic: q only
    int Qy[2], Qx[2], nqy = 1, nqx = 1;
    Qy[0] = qy;
    Qx[0] = qx;
    if (SYM) {
        if (qy < R) Qy[nqy++] = -1 - qy;
        else if (qy >= H - R) Qy[nqy++] = 2 * H - 1 - qy;
        if (qx < R) Qx[nqx++] = -1 - qx;
        else if (qx >= W - R) Qx[nqx++] = 2 * W - 1 - qx;
    }
    double acc = 0.0;
    // c positions: thread t < SC * SC / 2 owns column t % SC, rows 2 (t / SC) and 2 (t / SC) + 1 (the two
    // rows share M (M - 1) of their 2 M^2 staged operands); taps live in registers (warp-uniform loads)
    static_assert(SC % 2 == 0 && SC * SC / 2 <= 256, "two c rows per thread");
    const int ccol = tid % SC, crow = 2 * (tid / SC);
    const bool cworker = tid < SC * SC / 2;
    for (int i = 0; i < a.n; ++i) {
        double k[M * M];
#pragma unroll
        for (int e = 0; e < M * M; ++e) k[e] = __ldg(a.kf + (size_t)i * M * M + e);
        const double wgt = __ldg(a.wgt + i);
        __syncthreads();  // staging done / previous filter's c consumed
        if (cworker) {
            double z0 = 0.0, z1 = 0.0, p0 = 0.0, p1 = 0.0;  // z(x) = sum_{a,b} k[a,b] w_ext(x - (a - r, b - r))
#pragma unroll
            for (int aa = 0; aa < M; ++aa)
#pragma unroll
                for (int bb = 0; bb < M; ++bb) {
                    const int s0 = (crow + 2 * R - aa) * SP + (ccol + 2 * R - bb);
                    const double kk = k[aa * M + bb];
                    z0 = fma(kk, ws[s0], z0);
                    z1 = fma(kk, ws[s0 + SP], z1);
                    p0 = fma(kk, ps[s0], p0);
                    p1 = fma(kk, ps[s0 + SP], p1);
                }
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int gy = y0 - R + crow + h, gx = x0 - R + ccol;
                const bool in = !SYM || (gy >= 0 && gy < H && gx >= 0 && gx < W);  // psi_0 = 0 outside (symmetric)
                cs[(crow + h) * SC + ccol] = in ? wgt * rho2_64(h ? z1 : z0) * (h ? p1 : p0) : 0.0;
            }
        }
        __syncthreads();
        if (!inside) continue;
        for (int u = 0; u < nqy; ++u)
            for (int v = 0; v < nqx; ++v) {
                const int ly = Qy[u] - y0, lx = Qx[v] - x0;  // c(Q + (a - r, b - r)) at c index ly + a
#pragma unroll
                for (int aa = 0; aa < M; ++aa) {
                    const int iy = ly + aa;
                    if (iy < 0 || iy >= SC) continue;  // outside the c tile: outside the image (psi_0 = 0)
#pragma unroll
                    for (int bb = 0; bb < M; ++bb) {
                        const int ix = lx + bb;
                        if (ix < 0 || ix >= SC) continue;
                        acc = fma(k[aa * M + bb], cs[iy * SC + ix], acc);
                    }
                }
            }
    }
    double dhd = 0.0, dd = 0.0;
    if (inside) {
        const size_t o = (size_t)qy * W + qx;
        const double p = ps[(ty + 2 * R) * SP + tx + 2 * R];  // this pixel's direction (0 outside the free set)
        double out;
        if (a.objective == 0) {
            out = acc + p;  // anscombe: d2D = I
        } else {
            const double fo = a.f[o];
            const double wc = fmax(a.w[o], 1e-150);
            out = acc + ((fo > 0.0) ? a.lam * fo / (wc * wc) : 0.0) * p;  // training.py:170-172
        }
        double dfull = p;
        if (a.free_mask && !a.free_mask[o]) {  // identity outside the free set (training.py:199-200)
            dfull = a.r[o];
            if (dprev && beta != 0.0) dfull = fma(beta, dprev[o], dfull);
            out = dfull;
        }
        out = fma(a.eps, dfull, out);  // H + eps I on a restart (training.py:216)
        a.hp[o] = out;
        if (dnext) dnext[o] = dfull;
        dhd = dfull * out;
        dd = dfull * dfull;
    }
    if (!a.st) return;
    block_sum2(dhd, dd, red);
    const int nct = gridDim.x * gridDim.y, cta = blockIdx.y * gridDim.x + blockIdx.x;
    if (tid == 0) {
        a.part[cta] = dhd;
        a.part[nct + cta] = dd;
        s_last = ticket_acq_rel(a.tickets) == (unsigned)(nct - 1);
    }
    __syncthreads();
    if (!s_last) return;
    double sdhd = 0.0, sdd = 0.0;  // fixed order: thread t sums CTAs t, t + 256, ..., then a fixed tree
    for (int k = tid; k < nct; k += 256) {
        sdhd += __ldcg(a.part + k);
        sdd += __ldcg(a.part + nct + k);
    }
    block_sum2(sdhd, sdd, red);
    if (tid != 0) return;
    a.tickets[0] = 0u;
    CgState *st = a.st;
    if (sdhd <= 1e-14 * sdd) st->status = CG_BREAKDOWN;  // training.py:220-222
    else st->alpha = st->rs / sdhd;
}

__global__ void __launch_bounds__(256) k_cg_update(const CgArgs a) {
    __shared__ double red[8][2];
    __shared__ int s_last;
    CgState *st = a.st;
    const int tid = threadIdx.x;
    if (st->status != CG_RUNNING) {
        if (a.use_cond && blockIdx.x == 0 && tid == 0) cudaGraphSetConditional(a.cond, 0u);
        return;
    }
    const double alpha = st->alpha;
    const double *d = st->parity ? a.d_prev : a.d_next;  // the direction k_cg_hvp just wrote
    const size_t n = (size_t)a.H * a.W;
    double rs = 0.0, unused = 0.0;
    for (size_t i = blockIdx.x * 256 + tid; i < n; i += (size_t)gridDim.x * 256) {
        a.q[i] = fma(alpha, d[i], a.q[i]);              // training.py:224
        const double r = fma(-alpha, a.hp[i], a.r_mut[i]);  // training.py:225
        a.r_mut[i] = r;
        rs = fma(r, r, rs);
    }
    block_sum2(rs, unused, red);
    if (tid == 0) {
        a.part[blockIdx.x] = rs;
        s_last = ticket_acq_rel(a.tickets + 1) == gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last) return;
    double rs_new = 0.0, unused2 = 0.0;  // fixed order, as in k_cg_hvp
    for (int k = tid; k < (int)gridDim.x; k += 256) rs_new += __ldcg(a.part + k);
    block_sum2(rs_new, unused2, red);
    if (tid != 0) return;
    a.tickets[1] = 0u;
    const double res = sqrt(rs_new) / st->rhs_norm;  // training.py:226-227
    st->it += 1;
    a.residuals[st->it] = res;
    if (res <= st->tol) st->status = CG_CONVERGED;
    else if (st->it >= st->max_iters) st->status = CG_MAXITER;
    st->beta = rs_new / st->rs;  // training.py:231-232
    st->rs = rs_new;
    st->parity ^= 1;
    if (a.use_cond) cudaGraphSetConditional(a.cond, st->status == CG_RUNNING ? 1u : 0u);
}

__global__ void k_cg_init(CgState *st, const double *rhs, double *r, double *q, size_t n, double tol, int max_iters,
                          double *residuals, double *part) {
    // r = rhs, q = 0, rs = <r, r> (fixed order: block 0 only, grid-stride by thread then a tree)
    __shared__ double red[8][2];
    double s = 0.0, unused = 0.0;
    for (size_t i = threadIdx.x; i < n; i += 256) {
        const double v = rhs[i];
        r[i] = v;
        q[i] = 0.0;
        s = fma(v, v, s);
    }
    block_sum2(s, unused, red);
    if (threadIdx.x == 0) {
        st->rs = s;
        st->rhs_norm = sqrt(s);
        st->tol = tol;
        st->alpha = 0.0;
        st->beta = 0.0;
        st->it = 0;
        st->max_iters = max_iters;
        st->status = max_iters > 0 ? CG_RUNNING : CG_MAXITER;
        st->parity = 0;
        residuals[0] = 1.0;  // sqrt(rs) / rhs_norm at the start
        (void)part;
    }
}
