// foe_b200.cu -- B200 (sm_100a) kernels and C ABI for the FoE Poisson-denoise hot path.
//
// Reference path (/root/reference/pkg/src/foepoisson):
//   denoise (pipeline.py:242-244) -> anscombe_forward (anscombe.py:19-24)
//   -> ipiano_minimize (solver.py:128-175) over foe_energy / foe_gradient (prior.py:95-110)
//      with prox_quadratic / prox_idiv (solver.py:92-125)
//   -> anscombe_inverse_exact_unbiased (anscombe.py:33-51)
//
// Design:
//  * One fused "pass" kernel evaluates one iPiano trial for every live image of a batch:
//    trial point + prox (elementwise, in a shared-memory tile with a 2r halo), the forward
//    responses K_i u_new and K_i du of all filters, rho'(z), the exact adjoint K_i^T with the
//    symmetric-boundary fold done in-tile, the energy change dF = sum a_i log1p(dz(2z_o+dz)/(1+z_o^2))
//    and the dot products <du,du>, <g,du>, |u|^2, G(u_new) -- one HBM pass per trial.
//  * Per-tile fp64 partials are summed in a fixed order by the last CTA of each image, which also
//    takes the accept/reject decision, updates L and rotates the state buffers: no host round trip.
//  * A trial that is accepted already carries grad F(u_new) for the next iteration (speculative
//    gradient), so every pass is one trial: ~1.37 passes per accepted iteration.
#include "foe_b200.h"

#ifndef FOE_ABLATE
#define FOE_ABLATE 0  // timing ablations of the tensor-core pass (1: no shifted sums, 2: no energy series)
#endif
#ifndef FOE_STAMPS
#define FOE_STAMPS 0  // per-block cycle stamps of the tensor-core pass (timing diagnostic builds only)
#endif

#include <cuda_runtime.h>
#include <math_constants.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <type_traits>
#include <vector>

struct foe_bank {
    int n, m, boundary, device, zero_mean;
    float *d_kf, *d_alpha;
    float *d_tc_img;  // operand image of the tensor-core 5x5 pass (foe_pass_tc.cuh), null for other banks
};

namespace {

thread_local std::string g_err;
std::atomic<long long> g_launches{0};  // kernels launched by this library (bench accounting)

int fail(int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define FOE_CUDA(x)                                                                              \
    do {                                                                                         \
        cudaError_t e_ = (x);                                                                    \
        if (e_ != cudaSuccess) return fail(FOE_E_CUDA, "%s: %s", #x, cudaGetErrorString(e_));    \
    } while (0)

constexpr int kMaxTaps = 4096;
constexpr int kMaxFilters = 512;
constexpr int kNumPartials = 7;  // dF|F, sq, gd, |u|^2, G_a, G_b, G_bad
constexpr int kPartialStride = 8;
constexpr bool kTcDefault = true;  // tensor-core pass for eligible banks unless FOE_TC=0

enum PassMode { MODE_EVAL = 0, MODE_INIT = 1, MODE_TRIAL = 2 };

struct ImgCtl {
    double L, f_u, lam;
    int n, max_iters, trials, status, done, branch, failed_at;
    int iu, iup, inew, ig, ignew;
    // step size tau = step_num / L (solver.py:64-65), prox weight t = tau * lam and 1 / (1 + t), kept in step
    // with L: the trial point is formed in fp64 from these (trial_point) and rounded once to fp32
    double tau, t, inv1pt;
};

// the trial step of the current L, computed once per change of L rather than by every thread of a pass
__host__ __device__ inline void set_step(ImgCtl &c, double step_num) {
    const double tau = step_num / c.L;  // SolverConfig.step_size, solver.py:64-65
    c.tau = tau;
    c.t = tau * c.lam;
    c.inv1pt = 1.0 / (1.0 + c.t);
}

struct PassArgs {
    int B, H, W, n_filters, tiles_x, tiles_y, mode, no_decide, zero_mean;
    // row-band decomposition (single device: ty0 = 0, lrow0 = 0, Hl = H, band = 0)
    int ty0;    // first global tile row of this launch (tiles_y is the global count)
    int tiles_yl;  // tile rows in this launch
    int lrow0;  // global row stored in local row 0
    int Hl;     // local rows per image (plane stride = Hl * W)
    int band;   // 1: write partials only, decisions by k_decide after the all-gather
    unsigned long long *dbg_times;  // optional per-CTA [start, end-of-compute, exit] %globaltimer (ns)
    size_t plane;  // B*H*W: distance between state slots
    const float *kf;     // (n, M*M) flipped taps (correlation orientation of the forward conv)
    const float *alpha;  // (n)
    const float *tc_img; // k_pass_tc's shared-memory operand image (5x5 banks with <= 32 filters), else null
    // state (solve modes)
    float *U;        // 3 slots
    float *Gs;       // 2 slots
    const float *obs;
    ImgCtl *ctl;
    double *trace;
    int trace_cap;
    int *n_active;
    // eval mode
    const float *u_in;
    float *g_out;
    double *energy_out;
    // reductions
    double *partials;     // (B, tiles, kPartialStride)
    unsigned *tickets;    // (B)
    // solver constants
    double gamma, step_num, eta, relax, rel_tol, max_L;
};

// ------------------------------------------------------------------------------------------------
// geometry

// Owned-row partition of the image into tiles of T rows; the last tile is pulled up so it owns at
// least r rows: every pixel within r of the far edge then lies in a tile whose region also holds
// the padded pixels that fold onto it (symmetric boundary, image.py:61-83).
__host__ __device__ __forceinline__ int tile_start(int k, int nt, int T, int n, int r) {
    if (k >= nt) return n;
    int s = k * T;
    if (k == nt - 1 && nt > 1) s = (s < n - r) ? s : n - r;
    return s;
}

// np.pad index map (image.py:61-65): "symmetric" (edge-inclusive mirror) or "wrap"; clamped so
// far-out (don't-care) positions of partial tiles stay in bounds.
template <bool SYM>
__device__ __forceinline__ int src_idx(int q, int n) {
    if (SYM) {
        if (q < 0) q = -1 - q;
        if (q >= n) q = 2 * n - 1 - q;
        return q < 0 ? 0 : (q >= n ? n - 1 : q);
    } else {
        q %= n;
        return q < 0 ? q + n : q;
    }
}


template <int W>
__device__ __forceinline__ void load_row(const float *p, float (&r)[W]) {
#pragma unroll
    for (int k = 0; k + 4 <= W; k += 4) {
        const float4 v = *reinterpret_cast<const float4 *>(p + k);
        r[k] = v.x; r[k + 1] = v.y; r[k + 2] = v.z; r[k + 3] = v.w;
    }
    if constexpr ((W & 3) >= 2) {
        const float2 v = *reinterpret_cast<const float2 *>(p + (W & ~3));
        r[W & ~3] = v.x; r[(W & ~3) + 1] = v.y;
    }
    if constexpr ((W & 1) == 1) r[W - 1] = p[W - 1];
}

__device__ __forceinline__ float prox_quad(float ut, float t, float v) {
    return (ut + t * v) / (1.0f + t);  // solver.py:100
}

// prox_idiv (solver.py:103-125) in fp64 for the trial point
__device__ __forceinline__ double prox_idv64(double ut, double t, double ob) {
    if (t == 0.0) return ut;  // solver.py:119-120
    const double a = ut - t;
    const double root = sqrt(fma(a, a, 4.0 * t * ob));
    double o = (a >= 0.0) ? 0.5 * (a + root) : (2.0 * t * ob) / (root - a);  // solver.py:121-124
    if (ob == 0.0 && a < 0.0) o = 0.0;                                        // solver.py:125
    return o;
}

__device__ __forceinline__ float prox_idv(float ut, float t, float ob) {
    if (t == 0.0f) return ut;  // solver.py:119-120
    const float a = ut - t;
    const float root = sqrtf(fmaf(a, a, 4.0f * t * ob));
    float o = (a >= 0.0f) ? 0.5f * (a + root) : (2.0f * t * ob) / (root - a);  // solver.py:121-124
    if (ob == 0.0f && a < 0.0f) o = 0.0f;                                      // solver.py:125
    return o;
}

// ------------------------------------------------------------------------------------------------
// decision (the body of the backtracking loop, solver.py:147-174), run by one thread per image

__device__ void finish_image(const PassArgs &a, ImgCtl &c, bool primary) {
    c.done = 1;
    if (primary) atomicSub(a.n_active, 1);
}

// Apply one pass's summed partials s[0..6] to image b's control block c.  `primary` = this copy of
// the control block is the authoritative one (writes the trace row and the live counter).
__device__ void decide_ctl(const PassArgs &a, int b, const double *s, ImgCtl &c, bool primary, int mode) {
    if (mode == MODE_INIT) {
        c.f_u = s[0];
        if (!isfinite(s[0])) {  // solver.py:142-144
            c.status = FOE_SOLVE_NONFINITE;
            c.failed_at = c.n;
            finish_image(a, c, primary);
        }
        return;
    }
    const double L = c.L;
    const double dF = s[0], sq = s[1], gd = s[2], un2 = s[3];
    const double f_new = c.f_u + dF;
    // slack = f_new - (f_u + gd + L/2 sq), evaluated from dF directly (solver.py:154-155)
    const double slack = dF - (gd + 0.5 * L * sq);
    const double tol = 1e-12 * (fabs(c.f_u) + fabs(f_new) + fabs(gd) + 0.5 * L * sq);
    c.trials++;
    if (isfinite(f_new) && slack <= tol) {  // solver.py:156
        if (primary) {
            double Gv;
            if (c.branch == FOE_QUADRATIC) Gv = 0.5 * c.lam * s[4];  // pipeline.py:200
            else Gv = (s[6] > 0.0) ? INFINITY : c.lam * (s[4] - s[5]);  // pipeline.py:141-149
            double *row = a.trace + ((size_t)b * a.trace_cap + c.n) * 6;  // solver.py:162-169
            row[0] = f_new; row[1] = Gv; row[2] = L; row[3] = sqrt(sq); row[4] = slack; row[5] = tol;
        }
        const double step = sqrt(sq);
        const int old_up = c.iup;  // u_prev, u = u, u_new (solver.py:171)
        c.iup = c.iu; c.iu = c.inew; c.inew = old_up;
        const int og = c.ig; c.ig = c.ignew; c.ignew = og;
        c.f_u = f_new;
        c.L = L / a.relax;  // solver.py:172
        set_step(c, a.step_num);
        c.n++;
        const double un = sqrt(un2);
        if (step < a.rel_tol * fmax(un, 1e-300) || c.n >= c.max_iters) finish_image(a, c, primary);  // :173-174
    } else {
        c.L = L * a.eta;  // solver.py:158-160
        set_step(c, a.step_num);
        if (c.L > a.max_L) {
            c.status = FOE_SOLVE_STALLED;
            c.failed_at = c.n;
            finish_image(a, c, primary);
        }
    }
}

// on a register copy: one batch of loads, the logic, one batch of stores (operating on the global block in
// place serialised L2 round trips behind the trace-row stores, which may alias it)
__device__ void decide(const PassArgs &a, int b, const double *s) {
    ImgCtl c = a.ctl[b];
    decide_ctl(a, b, s, c, true, a.mode);
    a.ctl[b] = c;
}

// fixed-order block reduction of kNumPartials doubles (deterministic), in two halves that a kernel may
// run at different times: per-warp shuffle sums of partials [K0, K1) into red[warp][k], then one warp's
// shuffle tree over the per-warp sums into out[] (complete for every thread on return)
template <int K0, int K1>
__device__ __forceinline__ void warp_partials(const double (&v)[kNumPartials], double (*red)[kNumPartials]) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double x[K1 - K0];
#pragma unroll
    for (int k = K0; k < K1; ++k) x[k - K0] = v[k];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1)
#pragma unroll
        for (int k = K0; k < K1; ++k) x[k - K0] += __shfl_down_sync(0xffffffffu, x[k - K0], off);
    if (lane == 0)
#pragma unroll
        for (int k = K0; k < K1; ++k) red[warp][k] = x[k - K0];
}

// the per-warp sums through shared memory instead of shuffles (SHFL issues at one warp-instruction per
// SM clock, so a whole CTA's fp64 shuffle trees cost ~1.5k cycles): each lane parks its values in the
// warp's scratch (K1 - K0) x 32 doubles, lanes 4k..4k+3 add partial k's four groups of 8 lanes in order,
// then two shuffle steps combine the groups.  Deterministic, a fixed association of its own.
// Scratch row r (32 doubles) starts at scratch + r * PITCH doubles; warp w uses rows w * NK .. w * NK + NK - 1.
template <int K0, int K1, int PITCH>
__device__ __forceinline__ void warp_partials_smem(const double (&v)[kNumPartials], double (*red)[kNumPartials],
                                                   double *scratch) {
    constexpr int NK = K1 - K0;
    static_assert(4 * NK <= 32 && PITCH >= 32, "four lanes per partial, 32 doubles per row");
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double *sc = scratch + warp * NK * PITCH;
#pragma unroll
    for (int k = 0; k < NK; ++k) sc[k * PITCH + lane] = v[K0 + k];
    __syncwarp();
    const int kk = lane >> 2, q = lane & 3;
    double s = 0.0;
    if (kk < NK) {
#pragma unroll
        for (int i = 0; i < 8; ++i) s += sc[kk * PITCH + 8 * q + i];
    }
    s += __shfl_down_sync(0xffffffffu, s, 2);
    s += __shfl_down_sync(0xffffffffu, s, 1);
    if (q == 0 && kk < NK) red[warp][K0 + kk] = s;
    __syncwarp();
}

// one warp (any) combines the NT / 32 per-warp sums in a fixed tree; the result is in lane 0's x (and in out)
template <int NT>
__device__ __forceinline__ void warp_combine(double (*red)[kNumPartials], double *out, double (&x)[kNumPartials]) {
    const int lane = threadIdx.x & 31;
    static_assert(NT / 32 <= 32, "one warp combines the per-warp sums");
#pragma unroll
    for (int k = 0; k < kNumPartials; ++k) x[k] = lane < NT / 32 ? red[lane][k] : 0.0;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1)
#pragma unroll
        for (int k = 0; k < kNumPartials; ++k) x[k] += __shfl_down_sync(0xffffffffu, x[k], off);
    if (lane == 0)
#pragma unroll
        for (int k = 0; k < kNumPartials; ++k) out[k] = x[k];
}

template <int NT>
__device__ __forceinline__ void block_combine(double (*red)[kNumPartials], double *out) {
    const int warp = threadIdx.x >> 5;
    __syncthreads();
    if (warp == 0) {
        double x[kNumPartials];
        warp_combine<NT>(red, out, x);
    }
    __syncthreads();
}

template <int NT>
__device__ __forceinline__ void block_reduce(double (&v)[kNumPartials], double (*red)[kNumPartials],
                                             double *out) {
    warp_partials<0, kNumPartials>(v, red);
    block_combine<NT>(red, out);
}

// fixed-order sum of one image's tile partials (layout [tile][B][8]) into s_sum, by a whole CTA:
// thread k < 384 sums tiles k, k+384, ... then a fixed tree.  Shared by the last-CTA path and
// k_decide, so a band-decomposed solve reduces in exactly the single-device order.
// The tile stride is a fixed 384 whatever the block size (threads beyond it add exact zeros), so
// every kernel that decides -- k_pass, k_pass_tc, k_decide -- reduces in the same order.
// Up to kFastReduceTiles tiles (every single-image configuration up to ~2k x 2k) take the one-warp-
// per-partial path below instead.
constexpr int kReduceNT = 384, kFastReduceTiles = 1024;

// lane l's ordered sum of partial k over tiles l, l + 32, ...: eight loads in flight at a time (a loop of
// dependent load-add pairs costs one L2 round trip per tile: 4-5 of them, ~2 us, at 144 tiles), added in
// the same order (absent tiles add an exact zero)
__device__ __forceinline__ double lane_tile_sum(const double *partials, int ntiles, int B, int b, int k, int lane) {
    double x = 0.0;
    for (int base = 0; base < ntiles; base += 256) {
        double v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int tt = base + lane + 32 * i;
            v[i] = tt < ntiles ? __ldcg(partials + ((size_t)tt * B + b) * kPartialStride + k) : 0.0;
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) x += v[i];
    }
    return x;
}

template <int NT>
__device__ void reduce_tiles(const double *partials, int ntiles, int B, int b, double (*red)[kNumPartials],
                             double *s_sum) {
    static_assert(NT >= kReduceNT && NT % 32 == 0, "reducing block narrower than the fixed tile stride");
    if (ntiles <= kFastReduceTiles) {
        // one warp per partial: lane l adds tiles l, l + 32, ... in order, then a shuffle tree -- one L2
        // round trip and ~10 shuffles on the decision's critical path (the order depends on ntiles only)
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        __syncthreads();
        if (warp < kNumPartials) {
            double x = lane_tile_sum(partials, ntiles, B, b, warp, lane);
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) x += __shfl_down_sync(0xffffffffu, x, off);
            if (lane == 0) s_sum[warp] = x;
        }
        __syncthreads();
        return;
    }
    double tot[kNumPartials];
#pragma unroll
    for (int k = 0; k < kNumPartials; ++k) tot[k] = 0.0;
    for (int tt = threadIdx.x; threadIdx.x < kReduceNT && tt < ntiles; tt += kReduceNT)
#pragma unroll
        for (int k = 0; k < kNumPartials; ++k) tot[k] += __ldcg(partials + ((size_t)tt * B + b) * kPartialStride + k);
    __syncthreads();
    block_reduce<NT>(tot, red, s_sum);
    __syncthreads();
}

#include "foe_pass.cuh"
#include "foe_tc.cuh"
#include "foe_pass_tc.cuh"
#include "foe_pass_tc7.cuh"

// ------------------------------------------------------------------------------------------------
// elementwise kernels

__global__ void k_anscombe_fwd(const double *__restrict__ y, float *__restrict__ v, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        v[i] = (float)(2.0 * sqrt(y[i] + 0.375));  // anscombe.py:24
}

__global__ void k_anscombe_fwd_f32(const float *__restrict__ y, float *__restrict__ v, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        v[i] = (float)(2.0 * sqrt((double)y[i] + 0.375));  // anscombe.py:24, counts staged as exact floats
}

__global__ void k_direct_obs(const double *__restrict__ y, float *__restrict__ obs, double c, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        obs[i] = (float)(y[i] == 0.0 ? c : y[i]);  // pipeline.py:165
}

__global__ void k_inverse_exact_unbiased(const float *__restrict__ z, double *__restrict__ x, int64_t n,
                                         unsigned long long *counts) {
    const double S = 1.2247448713915890491;  // sqrt(3/2), anscombe.py:13
    unsigned c_low = 0, c_neg = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double zi = (double)z[i];
        const bool low = zi < S;
        const double zc = low ? S : zi;
        const double v = zc * zc / 4.0 + S / (4.0 * zc) - 11.0 / (8.0 * zc * zc) + 5.0 * S / (8.0 * zc * zc * zc) - 0.125;
        const bool neg = v < 0.0;
        c_low += low;
        c_neg += (neg && !low);
        x[i] = neg ? 0.0 : v;  // anscombe.py:48-51
    }
    if (counts) {
        for (int off = 16; off > 0; off >>= 1) {
            c_low += __shfl_down_sync(0xffffffffu, c_low, off);
            c_neg += __shfl_down_sync(0xffffffffu, c_neg, off);
        }
        if ((threadIdx.x & 31) == 0) {
            if (c_low) atomicAdd(counts, (unsigned long long)c_low);
            if (c_neg) atomicAdd(counts + 1, (unsigned long long)c_neg);
        }
    }
}

__global__ void k_prox_quadratic(const float *__restrict__ ut, const float *__restrict__ v, float *__restrict__ out,
                                 float t, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = prox_quad(ut[i], t, v[i]);
}

__global__ void k_prox_idiv(const float *__restrict__ ut, const float *__restrict__ ob, float *__restrict__ out,
                            float t, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = prox_idv(ut[i], t, ob[i]);
}

// single-filter reference operators (image.py:37-83); simple gathers, not on the solve path
template <bool SYM>
__global__ void k_conv_same(const float *__restrict__ x, float *__restrict__ out, const float *__restrict__ kf, int m,
                            int B, int H, int W) {
    const int r = m / 2;
    const int64_t n = (int64_t)B * H * W;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = i / ((int64_t)H * W);
        const int p = (int)(i - b * H * W), y = p / W, xx = p - y * W;
        const float *img = x + b * H * W;
        float s = 0.0f;
        for (int a = 0; a < m; ++a)
            for (int c = 0; c < m; ++c)
                s = fmaf(kf[a * m + c], img[(size_t)src_idx<SYM>(y + a - r, H) * W + src_idx<SYM>(xx + c - r, W)], s);
        out[i] = s;
    }
}

template <bool SYM>
__global__ void k_conv_adjoint(const float *__restrict__ yv, float *__restrict__ out, const float *__restrict__ k,
                               int m, int B, int H, int W) {
    const int r = m / 2;
    const int64_t n = (int64_t)B * H * W;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = i / ((int64_t)H * W);
        const int p = (int)(i - b * H * W), y = p / W, xx = p - y * W;
        const float *img = yv + b * H * W;
        // padded positions q with src(q) == p (image.py:80-83)
        int qy[3], qx[3], ny = 0, nx = 0;
        const int cy[3] = {y, SYM ? -1 - y : y - H, SYM ? 2 * H - 1 - y : y + H};
        const int cx[3] = {xx, SYM ? -1 - xx : xx - W, SYM ? 2 * W - 1 - xx : xx + W};
        for (int e = 0; e < 3; ++e) {
            if (cy[e] >= -r && cy[e] < H + r && (e == 0 || cy[e] != y)) qy[ny++] = cy[e];
            if (cx[e] >= -r && cx[e] < W + r && (e == 0 || cx[e] != xx)) qx[nx++] = cx[e];
        }
        float s = 0.0f;
        for (int ey = 0; ey < ny; ++ey)
            for (int ex = 0; ex < nx; ++ex)
                for (int a = 0; a < m; ++a) {
                    const int py = qy[ey] + a - r;
                    if (py < 0 || py >= H) continue;
                    for (int c = 0; c < m; ++c) {
                        const int px = qx[ex] + c - r;
                        if (px < 0 || px >= W) continue;
                        s = fmaf(k[a * m + c], img[(size_t)py * W + px], s);
                    }
                }
        out[i] = s;
    }
}

__global__ void k_gather_final(const float *__restrict__ U, size_t plane, const ImgCtl *__restrict__ ctl,
                               float *__restrict__ out, size_t HW, int B) {
    const int b = blockIdx.y;
    const float *src = U + (size_t)ctl[b].iu * plane + (size_t)b * HW;
    float *dst = out + (size_t)b * HW;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < HW; i += (size_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
}



// ------------------------------------------------------------------------------------------------
// transform_binned (pipeline.py:214-235): bin3 and unbin_bilinear (noise.py:55-113)

// sum of factor x factor blocks, bottom/right replicate-padded (noise.py:55-71); exact for counts
__global__ void k_bin(const double *__restrict__ y, double *__restrict__ yb, int H, int W, int f, int Hb, int Wb) {
    const int64_t n = (int64_t)Hb * Wb;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int r = (int)(i / Wb), c = (int)(i - (int64_t)r * Wb);
        double s = 0.0;
        for (int a = 0; a < f; ++a) {
            const double *row = y + (size_t)min(r * f + a, H - 1) * W;
            for (int b = 0; b < f; ++b) s += row[min(c * f + b, W - 1)];
        }
        yb[i] = s;
    }
}

// divide by factor^2, corner-aligned bilinear upsampling to the padded size, crop (noise.py:74-113)
__global__ void k_unbin(const double *__restrict__ xb, double *__restrict__ out, int h, int w, int H, int W, int f) {
    const int Hp = (H + f - 1) / f * f, Wp = (W + f - 1) / f * f;
    const double inv = 1.0 / (double)(f * f);
    const int64_t n = (int64_t)H * W;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int Y = (int)(i / W), X = (int)(i - (int64_t)Y * W);
        int i0 = 0, j0 = 0;
        double di = 0.0, dj = 0.0;
        if (h > 1) {
            const double row = Hp > 1 ? (double)Y * ((double)(h - 1) / (double)(Hp - 1)) : 0.0;
            i0 = min((int)row, h - 2);
            di = row - i0;
        }
        if (w > 1) {
            const double col = Wp > 1 ? (double)X * ((double)(w - 1) / (double)(Wp - 1)) : 0.0;
            j0 = min((int)col, w - 2);
            dj = col - j0;
        }
        const int i1 = min(i0 + 1, h - 1), j1 = min(j0 + 1, w - 1);
        const double tl = xb[(size_t)i0 * w + j0] * inv, tr = xb[(size_t)i0 * w + j1] * inv;
        const double bl = xb[(size_t)i1 * w + j0] * inv, br = xb[(size_t)i1 * w + j1] * inv;
        const double top = tl + (tr - tl) * dj, bot = bl + (br - bl) * dj;
        out[i] = top + (bot - top) * di;
    }
}

// estimate_peak (pipeline.py:247-254): the max over pixels of the 3 x 3 median filter of the counts, with
// scipy.ndimage.median_filter's default "reflect" boundary (edge-inclusive mirror, the symmetric rule of
// src_idx).  The median is the 19-exchange selection network for 9 values; the max is an atomicMax on an
// order-preserving integer image of the double.
__device__ __forceinline__ unsigned long long ordered_bits(double x) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(x);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ void cswap(double &a, double &b) {
    const double lo = fmin(a, b), hi = fmax(a, b);
    a = lo;
    b = hi;
}
__global__ void k_median3_max(const double *__restrict__ y, int H, int W, unsigned long long *out) {
    const int64_t n = (int64_t)H * W;
    unsigned long long best = 0ull;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int Y = (int)(i / W), X = (int)(i - (int64_t)Y * W);
        double p[9];
#pragma unroll
        for (int dy = 0; dy < 3; ++dy)
#pragma unroll
            for (int dx = 0; dx < 3; ++dx)
                p[3 * dy + dx] = y[(size_t)src_idx<true>(Y + dy - 1, H) * W + src_idx<true>(X + dx - 1, W)];
        cswap(p[1], p[2]); cswap(p[4], p[5]); cswap(p[7], p[8]);
        cswap(p[0], p[1]); cswap(p[3], p[4]); cswap(p[6], p[7]);
        cswap(p[1], p[2]); cswap(p[4], p[5]); cswap(p[7], p[8]);
        cswap(p[0], p[3]); cswap(p[5], p[8]); cswap(p[4], p[7]);
        cswap(p[3], p[6]); cswap(p[1], p[4]); cswap(p[2], p[5]);
        cswap(p[4], p[7]); cswap(p[4], p[2]); cswap(p[6], p[4]);
        cswap(p[4], p[2]);
        const unsigned long long o = ordered_bits(p[4]);
        best = o > best ? o : best;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const unsigned long long v = __shfl_down_sync(0xffffffffu, best, off);
        best = v > best ? v : best;
    }
    if ((threadIdx.x & 31) == 0 && best) atomicMax(out, best);
}

// ------------------------------------------------------------------------------------------------
// row-band decomposition (BASELINE config 5): decisions after the partials all-gather, halo rows

// one CTA per image: the same fixed-order reduction as the last-CTA path, then the decision
__global__ void __launch_bounds__(PassCfg<5>::NT) k_decide(const PassArgs a) {
    constexpr int NT = PassCfg<5>::NT;
    __shared__ double red[NT / 32][kNumPartials];
    __shared__ double s_sum[kNumPartials];
    const int b = blockIdx.x;
    if (a.ctl[b].done) return;
    reduce_tiles<NT>(a.partials, a.tiles_x * a.tiles_y, a.B, b, red, s_sum);
    if (threadIdx.x == 0) decide(a, b, s_sum);
}

// boundary rows -> send buffer [dir][B][field][halo][W]; dir 0 = first owned rows (to the band
// above), dir 1 = last owned rows (to the band below); field 0 = u, 1 = grad.  init: the gradient of
// the start point (u halos come with the input); otherwise the trial slots.
// the final-energy reduction of a band solve: image b's all-gathered tile partials in the fixed order
__global__ void __launch_bounds__(PassCfg<5>::NT) k_band_energy(const PassArgs a, double *energy) {
    constexpr int NT = PassCfg<5>::NT;
    __shared__ double red[NT / 32][kNumPartials];
    __shared__ double s_sum[kNumPartials];
    const int b = blockIdx.x;
    reduce_tiles<NT>(a.partials, a.tiles_x * a.tiles_y, a.B, b, red, s_sum);
    if (threadIdx.x == 0) energy[b] = s_sum[0];
}

__global__ void k_band_pack(const PassArgs a, float *send, int halo, int row0, int row1, int init) {
    const int b = blockIdx.y;
    const ImgCtl &c = a.ctl[b];
    const float *U = a.U + (init ? c.iu : c.inew) * a.plane + (size_t)b * a.Hl * a.W;
    const float *G = a.Gs + (init ? c.ig : c.ignew) * a.plane + (size_t)b * a.Hl * a.W;
    const size_t per = (size_t)halo * a.W;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < 2 * per; i += (size_t)gridDim.x * blockDim.x) {
        const int dir = (int)(i / per);
        const size_t e = i - dir * per;
        const int row = (dir == 0 ? row0 : row1 - halo) + (int)(e / a.W);
        const size_t src = (size_t)(row - a.lrow0) * a.W + e % a.W;
        float *dst = send + ((size_t)dir * a.B + b) * 2 * per;
        dst[e] = U[src];
        dst[per + e] = G[src];
    }
}

// receive buffer [dir][B][field][halo][W] -> halo rows; dir 0 came from the band above (rows
// [row0-halo, row0)), dir 1 from the band below (rows [row1, row1+halo)).
__global__ void k_band_unpack(const PassArgs a, const float *recv, int halo, int row0, int row1, int init) {
    const int b = blockIdx.y;
    const ImgCtl &c = a.ctl[b];
    float *U = a.U + (init ? c.iu : c.inew) * a.plane + (size_t)b * a.Hl * a.W;
    float *G = a.Gs + (init ? c.ig : c.ignew) * a.plane + (size_t)b * a.Hl * a.W;
    const size_t per = (size_t)halo * a.W;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < 2 * per; i += (size_t)gridDim.x * blockDim.x) {
        const int dir = (int)(i / per);
        if (dir == 0 && row0 == 0) continue;
        if (dir == 1 && row1 == a.H) continue;
        const size_t e = i - dir * per;
        const int row = (dir == 0 ? row0 - halo : row1) + (int)(e / a.W);
        const size_t dst = (size_t)(row - a.lrow0) * a.W + e % a.W;
        const float *src = recv + ((size_t)dir * a.B + b) * 2 * per;
        if (!init) U[dst] = src[e];
        G[dst] = src[per + e];
    }
}

// gather the owned rows of the final iterate
__global__ void k_gather_band(const float *__restrict__ U, size_t plane, const ImgCtl *__restrict__ ctl,
                              float *__restrict__ out, int Hl, int W, int row0, int row1, int lrow0) {
    const int b = blockIdx.y;
    const float *src = U + (size_t)ctl[b].iu * plane + (size_t)b * Hl * W + (size_t)(row0 - lrow0) * W;
    float *dst = out + (size_t)b * (row1 - row0) * W;
    const size_t n = (size_t)(row1 - row0) * W;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
}

// ------------------------------------------------------------------------------------------------
// host side

int grid_1d(int64_t n, int block = 256) {
    int64_t g = (n + block - 1) / block;
    return (int)std::max<int64_t>(1, std::min<int64_t>(g, 148 * 32));
}

template <int M>
size_t pass_smem_bytes(int nf, bool trial) {
    return sizeof(float) * smem_floats<M>(nf, trial);
}

// programmatic dependent launch of a pass kernel: its CTAs may start (bank staging, TMEM, barriers)
// while the previous kernel in the stream drains; the kernel waits (griddepcontrol.wait) before
// reading the state that kernel wrote.
// raise a kernel's dynamic shared-memory limit once per device (the bitmask is shared by concurrent
// host threads; a race only repeats the idempotent attribute call)
template <class K>
int ensure_smem(K kernel, int bytes, std::atomic<unsigned long long> &configured) {
    int dev = 0;
    FOE_CUDA(cudaGetDevice(&dev));
    const unsigned long long bit = 1ull << (dev & 63);
    if (!(configured.load(std::memory_order_acquire) & bit)) {
        FOE_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
        configured.fetch_or(bit, std::memory_order_release);
    }
    return FOE_OK;
}

template <class K>
cudaError_t launch_pdl(K kernel, dim3 grid, dim3 block, size_t smem, cudaStream_t st, const PassArgs &a) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, a);
}

template <int M, bool TRIAL, bool SYM>
int launch_pass_t(const PassArgs &a, cudaStream_t st) {
    using C = PassCfg<M>;
    const size_t smem = pass_smem_bytes<M>(a.n_filters, TRIAL);
    static std::atomic<unsigned long long> configured{0};  // one bit per device
    if (int rc = ensure_smem(k_pass<M, TRIAL, SYM>, 200 * 1024, configured)) return rc;
    FOE_CUDA(launch_pdl(k_pass<M, TRIAL, SYM>, dim3(a.tiles_x * a.tiles_yl, a.B), dim3(C::NT), smem, st, a));
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return FOE_OK;
}

template <bool TRIAL, bool SYM>
int launch_pass_m(int m, const PassArgs &a, cudaStream_t st) {
    switch (m) {
        case 1: return launch_pass_t<1, TRIAL, SYM>(a, st);
        case 3: return launch_pass_t<3, TRIAL, SYM>(a, st);
        case 5: return launch_pass_t<5, TRIAL, SYM>(a, st);
        case 7: return launch_pass_t<7, TRIAL, SYM>(a, st);
        default: return fail(FOE_E_UNSUPPORTED, "filter size %d not compiled (1,3,5,7)", m);
    }
}

// tensor-core pass (k_pass_tc): 5x5 banks with <= 32 filters; FOE_TC=0 forces the FFMA pass
bool use_tc(int m, int nf) {
    const char *e = getenv("FOE_TC");
    const int env = (e && e[0] == '0') ? 0 : (e && e[0] == '1') ? 1 : 2;
    return env != 0 && m == 5 && nf <= 32 && (env == 1 || kTcDefault);
}

template <int NF, bool TRIAL, bool SYM>
int launch_pass_tc_t(const PassArgs &a, cudaStream_t st) {
    using T = TcCfg<32>;
    // >= 116 KB keeps one CTA per SM: the 512 TMEM columns it allocates are the whole SM's
    const size_t smem = std::max<size_t>(sizeof(float) * (tc_smem_floats<32>() + 64), 116 * 1024);
    static std::atomic<unsigned long long> configured{0};  // one bit per device
    if (int rc = ensure_smem(k_pass_tc<NF, TRIAL, SYM>, (int)smem, configured)) return rc;
    FOE_CUDA(launch_pdl(k_pass_tc<NF, TRIAL, SYM>, dim3(a.tiles_x * a.tiles_yl, a.B), dim3(T::NT), smem, st, a));
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return FOE_OK;
}

// tensor-core pass for 7x7 banks with <= 48 filters (k_pass_tc7); FOE_TC7=0 (or FOE_TC=0) forces the FFMA pass
bool tc7_enabled();
bool use_tc7(int m, int nf) { return m == 7 && nf <= 48 && tc7_enabled(); }

template <bool TRIAL, bool SYM>
int launch_pass_tc7_t(const PassArgs &a, cudaStream_t st) {
    const size_t smem = sizeof(float) * (tc7_smem_floats() + 64);
    static std::atomic<unsigned long long> configured{0};  // one bit per device
    if (int rc = ensure_smem(k_pass_tc7<TRIAL, SYM>, (int)smem, configured)) return rc;
    FOE_CUDA(launch_pdl(k_pass_tc7<TRIAL, SYM>, dim3(a.tiles_x * a.tiles_yl, a.B), dim3(TcCfg7::NT), smem, st, a));
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return FOE_OK;
}

int launch_pass(int m, bool sym, const PassArgs &a, cudaStream_t st) {
    const bool trial = a.mode == MODE_TRIAL;
    if (m == 7 && tc7_enabled() && a.n_filters > 48)
        return fail(FOE_E_UNSUPPORTED, "7x7 banks with more than 48 filters need FOE_TC7=0 (FFMA pass)");
    if (use_tc7(m, a.n_filters))
        return trial ? (sym ? launch_pass_tc7_t<true, true>(a, st) : launch_pass_tc7_t<true, false>(a, st))
                     : (sym ? launch_pass_tc7_t<false, true>(a, st) : launch_pass_tc7_t<false, false>(a, st));
    if (use_tc(m, a.n_filters)) {
        switch ((a.n_filters + 7) / 8) {
            case 1: return trial ? (sym ? launch_pass_tc_t<8, true, true>(a, st) : launch_pass_tc_t<8, true, false>(a, st))
                                 : (sym ? launch_pass_tc_t<8, false, true>(a, st) : launch_pass_tc_t<8, false, false>(a, st));
            case 2: return trial ? (sym ? launch_pass_tc_t<16, true, true>(a, st) : launch_pass_tc_t<16, true, false>(a, st))
                                 : (sym ? launch_pass_tc_t<16, false, true>(a, st) : launch_pass_tc_t<16, false, false>(a, st));
            case 3: return trial ? (sym ? launch_pass_tc_t<24, true, true>(a, st) : launch_pass_tc_t<24, true, false>(a, st))
                                 : (sym ? launch_pass_tc_t<24, false, true>(a, st) : launch_pass_tc_t<24, false, false>(a, st));
            default: return trial ? (sym ? launch_pass_tc_t<32, true, true>(a, st) : launch_pass_tc_t<32, true, false>(a, st))
                                  : (sym ? launch_pass_tc_t<32, false, true>(a, st) : launch_pass_tc_t<32, false, false>(a, st));
        }
    }
    if (trial) return sym ? launch_pass_m<true, true>(m, a, st) : launch_pass_m<true, false>(m, a, st);
    return sym ? launch_pass_m<false, true>(m, a, st) : launch_pass_m<false, false>(m, a, st);
}

// region rows of the pass kernel that runs filter side m: 7x7 banks take the tensor-core pass's 40-row
// regions unless it is switched off (FOE_TC7=0 / FOE_TC=0: the FFMA k_pass<7>'s 48)
bool tc7_enabled() {
    const char *e = getenv("FOE_TC7"), *e5 = getenv("FOE_TC");
    return !(e && e[0] == '0') && !(e5 && e5[0] == '0');
}
int region_rows(int m) {
    if (m == 7) return tc7_enabled() ? TcCfg7::RH : PassCfg<7>::RH;
    return PassCfg<1>::RH;
}

void tile_counts(int m, int H, int W, int *tx, int *ty) {
    const int r = m / 2;
    const int TH = region_rows(m) - 2 * r, TW = PassCfg<1>::RW - 2 * r;  // owned tile
    *ty = (H + TH - 1) / TH;
    *tx = (W + TW - 1) / TW;
}

size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

struct SolveLayout {
    size_t U, G, O, ctl, partials, tickets, trace, n_active, energy, send, recv, total;
    size_t halo_floats;  // per direction
};

// Hl = local rows per image (H unless a row band), halo = rows exchanged per side (0 unless banded)
SolveLayout solve_layout(int m, int B, int H, int W, int trace_cap, int Hl = -1, int halo = 0) {
    if (Hl < 0) Hl = H;
    int tx, ty;
    tile_counts(m, H, W, &tx, &ty);
    const size_t plane = (size_t)B * Hl * W * sizeof(float);
    SolveLayout L;
    size_t off = 0;
    L.U = off; off = align_up(off + 3 * plane);
    L.G = off; off = align_up(off + 2 * plane);
    L.O = off; off = align_up(off + plane);
    L.ctl = off; off = align_up(off + sizeof(ImgCtl) * B);
    L.partials = off; off = align_up(off + sizeof(double) * kPartialStride * (size_t)B * tx * ty);
    L.tickets = off; off = align_up(off + sizeof(unsigned) * B);
    L.trace = off; off = align_up(off + sizeof(double) * 6 * (size_t)B * trace_cap);
    L.n_active = off; off = align_up(off + sizeof(int) * 4);
    L.energy = off; off = align_up(off + sizeof(double) * B);
    L.halo_floats = (size_t)B * 2 * halo * W;
    L.send = off; off = align_up(off + sizeof(float) * 2 * L.halo_floats);
    L.recv = off; off = align_up(off + sizeof(float) * 2 * L.halo_floats);
    L.total = off;
    return L;
}

int check_dims(const foe_bank *bank, int B, int H, int W) {
    if (!bank) return fail(FOE_E_INVALID, "null bank");
    if (B < 1 || B > 65535) return fail(FOE_E_INVALID, "batch %d out of range", B);
    if (H < bank->m || W < bank->m)  // prior.py:87-92
        return fail(FOE_E_INVALID, "image shape (%d, %d) smaller than filter size %d", H, W, bank->m);
    return FOE_OK;
}


// The trace's F column (solver.py:163) is the device's running f_u + dF: every dF is accurate to its own
// scale, but their sum carries the absolute rounding of the large early energies (F falls ~150x over a
// solve, so the last rows were ~3e-5 off relative).  Anchoring the column on F(u_final), evaluated
// directly, turns F_k into F(u_final) - sum_{j > k} dF_j (the same dF values; the accept decisions,
// which use dF only, are untouched).
void anchor_f_column(double *trace, int trace_cap, const std::vector<ImgCtl> &hc, const std::vector<double> &e) {
    for (size_t b = 0; b < hc.size(); ++b) {
        const int n = hc[b].n;
        if (n < 1 || !std::isfinite(e[b])) continue;
        double *rows = trace + b * (size_t)trace_cap * 6;
        const double delta = e[b] - rows[(size_t)(n - 1) * 6];
        if (!std::isfinite(delta)) continue;
        for (int k = 0; k < n; ++k) rows[(size_t)k * 6] += delta;
    }
}

}  // namespace

// ------------------------------------------------------------------------------------------------
// device-side solve loop: a CUDA graph whose conditional WHILE node runs [kGraphChunk trial passes ->
// k_loop_cond] until no image is live, so the tail of a solve needs no host round trip.  n_active[1]
// counts the passes the loop ran, n_active[2] flags the safety cap.

constexpr int kGraphChunk = 8;  // trial passes per evaluation of the loop condition

__global__ void k_loop_cond(cudaGraphConditionalHandle h, int *n_active, int cap, int chunk) {
    const int passes = (n_active[1] += chunk);
    const bool live = n_active[0] > 0;
    if (live && passes >= cap) n_active[2] = 1;
    cudaGraphSetConditional(h, (live && passes < cap) ? 1u : 0u);
}

struct LoopGraph {
    PassArgs key{};
    int m = 0, sym = 0, cap = 0, tc = 0;  // tc: which pass kernel the graph captured
    cudaGraphExec_t exec = nullptr;
};

struct LoopGraphCache {
    std::vector<LoopGraph> entries;
    cudaStream_t cap_stream = nullptr;
    ~LoopGraphCache() {
        for (auto &e : entries)
            if (e.exec) cudaGraphExecDestroy(e.exec);
        if (cap_stream) cudaStreamDestroy(cap_stream);
    }
};
thread_local LoopGraphCache t_graphs;

// the instantiated loop graph for these pass arguments (captured once, reused while the workspace,
// shape and solver constants stay the same)
int loop_graph(int m, bool sym, const PassArgs &a, int cap, cudaGraphExec_t *out) {
    const int tc = use_tc(m, a.n_filters) ? 1 : use_tc7(m, a.n_filters) ? 2 : 0;
    for (auto &e : t_graphs.entries)
        if (e.m == m && e.sym == (int)sym && e.cap == cap && e.tc == tc && !memcmp(&e.key, &a, sizeof(PassArgs))) {
            *out = e.exec;
            return FOE_OK;
        }
    if (!t_graphs.cap_stream) FOE_CUDA(cudaStreamCreateWithFlags(&t_graphs.cap_stream, cudaStreamNonBlocking));
    cudaGraph_t g = nullptr;
    FOE_CUDA(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle h;
    FOE_CUDA(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t node;
    FOE_CUDA(cudaGraphAddNode(&node, g, nullptr, 0, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    cudaStream_t cs = t_graphs.cap_stream;
    FOE_CUDA(cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    const long long before = g_launches.load();
    int rc = FOE_OK;
    const int chunk = kGraphChunk;
    for (int k = 0; k < chunk && rc == FOE_OK; ++k) rc = launch_pass(m, sym, a, cs);
    if (rc == FOE_OK) k_loop_cond<<<1, 1, 0, cs>>>(h, a.n_active, cap, chunk);
    cudaGraph_t captured = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(cs, &captured);
    g_launches.store(before);  // captured launches run (and are counted) per graph execution
    if (rc != FOE_OK) {
        cudaGraphDestroy(g);
        return rc;
    }
    if (ce != cudaSuccess) {
        cudaGraphDestroy(g);
        return fail(FOE_E_CUDA, "loop graph capture: %s", cudaGetErrorString(ce));
    }
    cudaGraphExec_t exec = nullptr;
    const cudaError_t ie = cudaGraphInstantiate(&exec, g, 0);
    cudaGraphDestroy(g);
    if (ie != cudaSuccess) return fail(FOE_E_CUDA, "loop graph instantiate: %s", cudaGetErrorString(ie));
    if (t_graphs.entries.size() >= 8) {
        cudaGraphExecDestroy(t_graphs.entries.front().exec);
        t_graphs.entries.erase(t_graphs.entries.begin());
    }
    LoopGraph e;
    memcpy(&e.key, &a, sizeof(PassArgs));  // bytewise, padding included (the cache compares bytes)
    e.m = m;
    e.sym = sym;
    e.cap = cap;
    e.tc = tc;
    e.exec = exec;
    t_graphs.entries.push_back(e);
    *out = exec;
    return FOE_OK;
}

// ------------------------------------------------------------------------------------------------
// scoring (metrics.py:30-102): PSNR and mean SSIM of x_hat against g after the [0, 255] convention
// (both scaled by 255 / peak, data_range 255), fp64 throughout.  SSIM: 11 x 11 Gaussian window
// (sigma 1.5, the outer product of the normalised 1-D window), valid-mode local statistics.  Per-CTA
// fp64 partials are summed in a fixed order by k_score_final, so the result is deterministic.

constexpr int kSsimW = 11, kSsimT = 32, kSsimIn = kSsimT + kSsimW - 1;
__constant__ double c_ssim_g[kSsimW];

__global__ void __launch_bounds__(256) k_ssim_tiles(const double *__restrict__ xh, const double *__restrict__ gt,
                                                    int H, int W, double scale, double c1, double c2,
                                                    double *__restrict__ part) {
    extern __shared__ double ssm[];
    double *X = ssm, *Y = X + kSsimIn * kSsimIn;          // scaled inputs of the tile
    double *Hs = Y + kSsimIn * kSsimIn;                   // horizontal sums [5][kSsimIn][kSsimT]
    const int b = blockIdx.z, tid = threadIdx.x;
    const int Hv = H - kSsimW + 1, Wv = W - kSsimW + 1;
    const int oy0 = blockIdx.y * kSsimT, ox0 = blockIdx.x * kSsimT;
    const double *xb = xh + (size_t)b * H * W, *gb = gt + (size_t)b * H * W;
    for (int e = tid; e < kSsimIn * kSsimIn; e += 256) {
        const int r = e / kSsimIn, c = e - r * kSsimIn;
        const int y = min(oy0 + r, H - 1), x = min(ox0 + c, W - 1);
        X[e] = xb[(size_t)y * W + x] * scale;
        Y[e] = gb[(size_t)y * W + x] * scale;
    }
    __syncthreads();
    for (int e = tid; e < kSsimIn * kSsimT; e += 256) {
        const int r = e / kSsimT, c = e - r * kSsimT;
        double sx = 0, sy = 0, sxx = 0, syy = 0, sxy = 0;
#pragma unroll
        for (int k = 0; k < kSsimW; ++k) {
            const double w = c_ssim_g[k], a = X[r * kSsimIn + c + k], d = Y[r * kSsimIn + c + k];
            sx += w * a;
            sy += w * d;
            sxx += w * a * a;
            syy += w * d * d;
            sxy += w * a * d;
        }
        const int o = r * kSsimT + c, P = kSsimIn * kSsimT;
        Hs[o] = sx;
        Hs[P + o] = sy;
        Hs[2 * P + o] = sxx;
        Hs[3 * P + o] = syy;
        Hs[4 * P + o] = sxy;
    }
    __syncthreads();
    double acc = 0.0;
    for (int e = tid; e < kSsimT * kSsimT; e += 256) {
        const int r = e / kSsimT, c = e - r * kSsimT;
        if (oy0 + r >= Hv || ox0 + c >= Wv) continue;
        const int P = kSsimIn * kSsimT;
        double ux = 0, uy = 0, mxx = 0, myy = 0, mxy = 0;
#pragma unroll
        for (int k = 0; k < kSsimW; ++k) {
            const double w = c_ssim_g[k];
            const int o = (r + k) * kSsimT + c;
            ux += w * Hs[o];
            uy += w * Hs[P + o];
            mxx += w * Hs[2 * P + o];
            myy += w * Hs[3 * P + o];
            mxy += w * Hs[4 * P + o];
        }
        const double vx = mxx - ux * ux, vy = myy - uy * uy, vxy = mxy - ux * uy;
        acc += ((2 * ux * uy + c1) * (2 * vxy + c2)) / ((ux * ux + uy * uy + c1) * (vx + vy + c2));
    }
    // fixed-order block sum
    __shared__ double red[256];
    red[tid] = acc;
    __syncthreads();
    for (int sft = 128; sft > 0; sft >>= 1) {
        if (tid < sft) red[tid] += red[tid + sft];
        __syncthreads();
    }
    if (tid == 0) part[((size_t)b * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = red[0];
}

__global__ void __launch_bounds__(256) k_sqdiff(const double *__restrict__ xh, const double *__restrict__ gt,
                                                int64_t n, double scale, double *__restrict__ part) {
    const int b = blockIdx.y, tid = threadIdx.x;
    const double *xb = xh + (size_t)b * n, *gb = gt + (size_t)b * n;
    double acc = 0.0;
    for (int64_t i = blockIdx.x * 256 + tid; i < n; i += (int64_t)gridDim.x * 256) {
        const double d = xb[i] * scale - gb[i] * scale;
        acc += d * d;
    }
    __shared__ double red[256];
    red[tid] = acc;
    __syncthreads();
    for (int sft = 128; sft > 0; sft >>= 1) {
        if (tid < sft) red[tid] += red[tid + sft];
        __syncthreads();
    }
    if (tid == 0) part[(size_t)b * gridDim.x + blockIdx.x] = red[0];
}

// per image: PSNR from the squared-difference partials, mean SSIM from the tile partials
__global__ void k_score_final(const double *__restrict__ sq_part, int n_sq, const double *__restrict__ ss_part,
                              int n_ss, int64_t n_px, int64_t n_valid, double data_range, double *psnr,
                              double *mssim) {
    const int b = blockIdx.x;
    if (threadIdx.x != 0) return;
    double sq = 0.0, ss = 0.0;
    for (int i = 0; i < n_sq; ++i) sq += sq_part[(size_t)b * n_sq + i];
    for (int i = 0; i < n_ss; ++i) ss += ss_part[(size_t)b * n_ss + i];
    const double mse = sq / (double)n_px;
    psnr[b] = mse == 0.0 ? CUDART_INF : 10.0 * log10(data_range * data_range / mse);
    mssim[b] = ss / (double)n_valid;
}

// ------------------------------------------------------------------------------------------------
// fp64 filter-bank operators for the training side (training.py runs in
// fp64 with 1e-9 CG / stationarity tolerances, so these stay fp64):
//   k_conv_bank64: out[b][i] = convolve_same(x[b], k_i)          (image.py:37-58, true convolution)
//   k_adj_bank64:  out[b]    = sum_i convolve_adjoint(y[b][i], k_i)  (image.py:68-83, exact adjoint:
//                  V^T psi on the padded domain with psi_0 = 0 outside the image, folded by P^T)
// Filters in the reference orientation (model.filters), n x m x m fp64, device memory.  16 x 16
// output tiles; the adjoint resolves P^-1(q) per output pixel (single reflection: H, W >= m).

constexpr int kT64 = 16;

template <int M, bool SYM>
__global__ void __launch_bounds__(256) k_conv_bank64(const double *__restrict__ kf, int n, const double *__restrict__ x,
                                                     double *__restrict__ out, int H, int W) {
    constexpr int R = M / 2, S = kT64 + 2 * R, FC = 8;
    __shared__ double xs[S * S];
    __shared__ double ks[FC * M * M];
    const int tid = threadIdx.x, nch = (n + FC - 1) / FC;
    const int b = blockIdx.z / nch, f0 = (blockIdx.z % nch) * FC, nfc = min(FC, n - f0);
    const int y0 = blockIdx.y * kT64, x0 = blockIdx.x * kT64;
    const double *xb = x + (size_t)b * H * W;
    for (int e = tid; e < S * S; e += 256) {
        const int i = e / S, j = e - i * S;
        xs[e] = xb[(size_t)src_idx<SYM>(y0 - R + i, H) * W + src_idx<SYM>(x0 - R + j, W)];
    }
    for (int e = tid; e < nfc * M * M; e += 256) ks[e] = kf[(size_t)f0 * M * M + e];
    __syncthreads();
    const int ty = tid / kT64, tx = tid % kT64, y = y0 + ty, xx = x0 + tx;
    if (y >= H || xx >= W) return;
    for (int fi = 0; fi < nfc; ++fi) {
        double acc = 0.0;
#pragma unroll
        for (int a = 0; a < M; ++a)
#pragma unroll
            for (int c = 0; c < M; ++c)  // z(p) = sum_{a,b} k[a,b] u_ext(p - (a - r, b - r))
                acc += ks[fi * M * M + a * M + c] * xs[(ty + 2 * R - a) * S + (tx + 2 * R - c)];
        out[(((size_t)b * n + f0 + fi) * H + y) * W + xx] = acc;
    }
}

template <int M, bool SYM>
__global__ void __launch_bounds__(256) k_adj_bank64(const double *__restrict__ kf, int n, const double *__restrict__ y,
                                                    double *__restrict__ out, int H, int W) {
    constexpr int R = M / 2, S = kT64 + 2 * R;
    __shared__ double ps[S * S];
    __shared__ double ks[M * M];
    const int tid = threadIdx.x, b = blockIdx.z;
    const int y0 = blockIdx.y * kT64, x0 = blockIdx.x * kT64;
    const int ty = tid / kT64, tx = tid % kT64, qy = y0 + ty, qx = x0 + tx;
    // P^-1(q): the padded positions Q in [-r, n + r) whose source pixel is q (image.py:61-66)
    int Qy[3], Qx[3], nqy = 1, nqx = 1;
    Qy[0] = qy;
    Qx[0] = qx;
    if (SYM) {
        if (qy < R) Qy[nqy++] = -1 - qy;
        if (qy >= H - R) Qy[nqy++] = 2 * H - 1 - qy;
        if (qx < R) Qx[nqx++] = -1 - qx;
        if (qx >= W - R) Qx[nqx++] = 2 * W - 1 - qx;
    }
    double acc = 0.0;
    for (int i = 0; i < n; ++i) {
        __syncthreads();
        const double *yb = y + ((size_t)b * n + i) * H * W;
        for (int e = tid; e < S * S; e += 256) {
            const int gy = y0 - R + e / S, gx = x0 - R + e % S;
            double v;
            if (SYM) v = (gy >= 0 && gy < H && gx >= 0 && gx < W) ? yb[(size_t)gy * W + gx] : 0.0;  // psi_0
            else v = yb[(size_t)src_idx<false>(gy, H) * W + src_idx<false>(gx, W)];  // circular adjoint
            ps[e] = v;
        }
        for (int e = tid; e < M * M; e += 256) ks[e] = kf[(size_t)i * M * M + e];
        __syncthreads();
        if (qy >= H || qx >= W) continue;
        for (int u = 0; u < nqy; ++u)
            for (int v = 0; v < nqx; ++v) {
                const int ly = Qy[u] - y0, lx = Qx[v] - x0;  // psi_0(Q + (a - r, b - r)) at ring index ly + a
#pragma unroll
                for (int a = 0; a < M; ++a) {
                    const int iy = ly + a;
                    if (iy < 0 || iy >= S) continue;  // outside the staged ring: outside the image
#pragma unroll
                    for (int c = 0; c < M; ++c) {
                        const int ix = lx + c;
                        if (ix < 0 || ix >= S) continue;
                        acc += ks[a * M + c] * ps[iy * S + ix];
                    }
                }
            }
    }
    if (qy < H && qx < W) out[((size_t)b * H + qy) * W + qx] = acc;
}

template <bool ADJ, int M>
int launch_bank64(const double *kf, int n, int boundary, const double *in, double *out, int B, int H, int W,
                  cudaStream_t st) {
    const dim3 tiles((W + kT64 - 1) / kT64, (H + kT64 - 1) / kT64);
    const bool sym = boundary == FOE_SYMMETRIC;
    if (ADJ) {
        const dim3 grid(tiles.x, tiles.y, B);
        if (sym) k_adj_bank64<M, true><<<grid, 256, 0, st>>>(kf, n, in, out, H, W);
        else k_adj_bank64<M, false><<<grid, 256, 0, st>>>(kf, n, in, out, H, W);
    } else {
        const dim3 grid(tiles.x, tiles.y, B * ((n + 7) / 8));
        if (sym) k_conv_bank64<M, true><<<grid, 256, 0, st>>>(kf, n, in, out, H, W);
        else k_conv_bank64<M, false><<<grid, 256, 0, st>>>(kf, n, in, out, H, W);
    }
    FOE_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return FOE_OK;
}

template <bool ADJ>
int bank64(const double *kf, int n, int m, int boundary, const double *in, double *out, int B, int H, int W,
           void *stream) {
    if (n < 1 || B < 1 || (boundary != FOE_SYMMETRIC && boundary != FOE_PERIODIC))
        return fail(FOE_E_INVALID, "bad bank arguments");
    if (H < m || W < m) return fail(FOE_E_INVALID, "fp64 bank operators need H, W >= m (got %dx%d, m=%d)", H, W, m);
    cudaStream_t st = (cudaStream_t)stream;
    switch (m) {
        case 1: return launch_bank64<ADJ, 1>(kf, n, boundary, in, out, B, H, W, st);
        case 3: return launch_bank64<ADJ, 3>(kf, n, boundary, in, out, B, H, W, st);
        case 5: return launch_bank64<ADJ, 5>(kf, n, boundary, in, out, B, H, W, st);
        case 7: return launch_bank64<ADJ, 7>(kf, n, boundary, in, out, B, H, W, st);
        default: return fail(FOE_E_UNSUPPORTED, "filter size %d not compiled (1,3,5,7)", m);
    }
}

#include "foe_train64.cuh"

template <int M, bool SYM>
int launch_cg_hvp(const CgArgs &a, cudaStream_t st) {
    const dim3 grid((a.W + kHT - 1) / kHT, (a.H + kHT - 1) / kHT);
    k_cg_hvp<M, SYM><<<grid, 256, 0, st>>>(a);
    FOE_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return FOE_OK;
}

int cg_hvp(int m, bool sym, const CgArgs &a, cudaStream_t st) {
    switch (m) {
        case 1: return sym ? launch_cg_hvp<1, true>(a, st) : launch_cg_hvp<1, false>(a, st);
        case 3: return sym ? launch_cg_hvp<3, true>(a, st) : launch_cg_hvp<3, false>(a, st);
        case 5: return sym ? launch_cg_hvp<5, true>(a, st) : launch_cg_hvp<5, false>(a, st);
        case 7: return sym ? launch_cg_hvp<7, true>(a, st) : launch_cg_hvp<7, false>(a, st);
        default: return fail(FOE_E_UNSUPPORTED, "filter size %d not compiled (1,3,5,7)", m);
    }
}

int check_cg_model(const double *filters, const double *weights, int n, int m, int boundary, int objective,
                   const double *w, const double *f, int H, int W) {
    if (!filters || !weights || !w) return fail(FOE_E_INVALID, "null argument");
    if (n < 1 || m < 1 || m > 7 || m % 2 != 1) return fail(FOE_E_INVALID, "bad bank (%d filters, side %d)", n, m);
    if (boundary != FOE_SYMMETRIC && boundary != FOE_PERIODIC) return fail(FOE_E_INVALID, "bad boundary");
    if (objective != 0 && objective != 1) return fail(FOE_E_INVALID, "objective must be 0 (anscombe) or 1 (original)");
    if (objective == 1 && !f) return fail(FOE_E_INVALID, "the original-domain objective needs the counts");
    if (H < m || W < m) return fail(FOE_E_INVALID, "image shape (%d, %d) smaller than filter size %d", H, W, m);
    return FOE_OK;
}

struct CgLayout {
    size_t r, da, db, hp, part, tickets, state, resid, total;
};
CgLayout cg_layout(int H, int W, int max_iters) {
    const size_t plane = sizeof(double) * (size_t)H * W;
    const size_t nct = (size_t)((W + kHT - 1) / kHT) * ((H + kHT - 1) / kHT);
    CgLayout L;
    size_t off = 0;
    L.r = off; off = align_up(off + plane);
    L.da = off; off = align_up(off + plane);
    L.db = off; off = align_up(off + plane);
    L.hp = off; off = align_up(off + plane);
    L.part = off; off = align_up(off + sizeof(double) * 2 * std::max<size_t>(nct, kCgUpdCtas));
    L.tickets = off; off = align_up(off + 2 * sizeof(unsigned));
    L.state = off; off = align_up(off + sizeof(CgState));
    L.resid = off; off = align_up(off + sizeof(double) * ((size_t)max_iters + 1));
    L.total = off;
    return L;
}

// FP32 FFMA throughput probe: 8 independent FMA chains per thread, 4 warps per SMSP, enough CTAs for
// every SM; the result feeds the roofline peak (MEASURED_PEAKS.json has no FP32 figure)
__global__ void __launch_bounds__(512) k_ffma_peak(float *out, int iters, float a, float b) {
    float x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3f + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 16; ++r)
#pragma unroll
            for (int i = 0; i < 8; ++i) x[i] = fmaf(x[i], a, b);
    }
    float s = 0.0f;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 1234.5f) out[0] = s;  // keeps the chains live
}

// Shared-memory operand image of k_pass_tc (TcCfg<32>::IMG_*), built once per bank: forward B1 / B2 (N = 32
// filters x K = 56 A columns, K-major SWIZZLE_NONE), adjoint Kt hi / lo (N = 32 taps x K = 32 filters), alpha,
// 2 alpha.  tf32 hi / lo both rounded to nearest-even, as cvt.rn.tf32.f32 does.
namespace {
float tf32_rn_host(float x) {
    uint32_t b;
    memcpy(&b, &x, 4);
    b += 0xFFFu + ((b >> 13) & 1u);
    b &= 0xffffe000u;
    memcpy(&x, &b, 4);
    return x;
}
template <int NF>
void tc_operand_image_t(std::vector<float> &img, const float *kf, const float *al, int nf) {
    using T = TcCfg<32>;
    using CL = TcCols<NF>;
    // K-major SWIZZLE_NONE operand of N rows: 8-row groups 128 B apart, 16-byte K chunks (N / 8) * 128 B apart
    auto boff = [](int N, int n, int k) { return (n & 7) * 4 + (k & 3) + (n >> 3) * 32 + (k >> 2) * (N / 8) * 32; };
    for (int f = 0; f < nf; ++f)
        for (int t = 0; t < T::KT; ++t) {
            const float v = kf[f * T::KT + t], h = tf32_rn_host(v), l = tf32_rn_host(v - h);
            img[T::IMG_BF + boff(CL::NZ, CL::brow(f, 0), tc_acol(t, 0))] = h;  // z1: u_hi k_hi
            img[T::IMG_BF + boff(CL::NZ, CL::brow(f, 0), tc_acol(t, 1))] = h;  //     u_lo k_hi
            img[T::IMG_BF + boff(CL::NZ, CL::brow(f, 1), tc_acol(t, 0))] = l;  // z2: u_hi k_lo
        }
    // adjoint: Kt[t][f] = 2 a_f k_f[t] with the unflipped k_f[t] = kf_f[24 - t]; K1 and K2 are N = 32 row operands
    for (int t = 0; t < T::KT; ++t)
        for (int f = 0; f < nf; ++f) {
            const float v = 2.0f * al[f] * kf[f * T::KT + (T::KT - 1 - t)], h = tf32_rn_host(v), l = tf32_rn_host(v - h);
            img[T::IMG_KT + boff(32, t, CL::kcol(f, 0))] = h;   // K1: psi_hi kt_hi
            img[T::IMG_KT + boff(32, t, CL::kcol(f, 1))] = h;   //     psi_lo kt_hi
            img[T::IMG_KT2 + boff(32, t, CL::kcol(f, 0))] = l;  // K2: psi_hi kt_lo
        }
    for (int f = 0; f < nf; ++f) {
        img[T::IMG_AL + f] = al[f];
        img[T::IMG_AL2 + f] = 2.0f * al[f];
    }
}
std::vector<float> tc_operand_image(const float *kf, const float *al, int nf) {
    std::vector<float> img(TcCfg<32>::IMG_FLOATS, 0.0f);
    switch ((nf + 7) / 8) {  // the kernel instantiation (launch_pass)
        case 1: tc_operand_image_t<8>(img, kf, al, nf); break;
        case 2: tc_operand_image_t<16>(img, kf, al, nf); break;
        case 3: tc_operand_image_t<24>(img, kf, al, nf); break;
        default: tc_operand_image_t<32>(img, kf, al, nf); break;
    }
    return img;
}
}  // namespace

extern "C" {

int foe_abi_version(void) { return 1; }
long long foe_kernel_launch_count(void) { return g_launches.load(); }
const char *foe_last_error(void) { return g_err.c_str(); }

// DenoiseRequest's count check (pipeline.py:50-56): every value >= 0 (NaN fails) and integral.  One
// branch-free pass the compiler vectorises: below 2^52, (v + 2^52) - 2^52 is v rounded to an integer
// (round-to-nearest-even, as np.rint); from 2^52 up every double is an integer (and +inf = rint(+inf)).
int foe_counts_check(const double *x, size_t n) {
    if (!x && n) return fail(FOE_E_INVALID, "null argument");
    constexpr double k52 = 4503599627370496.0;
    for (size_t i0 = 0; i0 < n; i0 += 8192) {
        const size_t i1 = std::min(n, i0 + 8192);
        int bad = 0;
        for (size_t i = i0; i < i1; ++i) {
            const double v = x[i];
            const double r = (v + k52) - k52;
            bad |= !(v >= 0.0) | ((v < k52) & (r != v));
        }
        if (bad) return 1;
    }
    return 0;
}

// The same check, writing every count as a float into dst (the caller's page-locked staging buffer) in the same
// pass: the H2D copy then moves 4 bytes per pixel and needs no separate host copy.  Returns 1 for invalid
// counts, 2 if every count is valid but one is too large for an exact float (>= 2^24; dst is then unusable),
// else 0.
int foe_counts_check_stage(const double *x, size_t n, float *dst) {
    if ((!x || !dst) && n) return fail(FOE_E_INVALID, "null argument");
    constexpr double k52 = 4503599627370496.0;
    int big = 0;
    for (size_t i0 = 0; i0 < n; i0 += 8192) {
        const size_t i1 = std::min(n, i0 + 8192);
        int bad = 0;
        for (size_t i = i0; i < i1; ++i) {
            const double v = x[i];
            const double r = (v + k52) - k52;
            bad |= !(v >= 0.0) | ((v < k52) & (r != v));
            big |= !(v < 16777216.0);
            dst[i] = (float)v;
        }
        if (bad) return 1;
    }
    return big ? 2 : 0;
}

int foe_device_sm_count(int device) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return -1;
    return v;
}

int foe_bank_create(const double *filters, const double *weights, int n, int m, int boundary, foe_bank **out) {
    if (!filters || !weights || !out) return fail(FOE_E_INVALID, "null argument");
    if (n < 1 || n > kMaxFilters) return fail(FOE_E_INVALID, "filter count %d out of range", n);
    if (m < 1 || m % 2 != 1) return fail(FOE_E_INVALID, "kernel side must be odd, got %d", m);  // image.py:23-29
    if (m > 7) return fail(FOE_E_UNSUPPORTED, "filter size %d not compiled (1,3,5,7)", m);
    if (n * m * m > kMaxTaps) return fail(FOE_E_UNSUPPORTED, "bank too large (%d taps)", n * m * m);
    if (boundary != FOE_SYMMETRIC && boundary != FOE_PERIODIC)
        return fail(FOE_E_INVALID, "boundary must be symmetric or periodic");
    for (int i = 0; i < n; ++i)
        if (!(weights[i] > 0)) return fail(FOE_E_INVALID, "expert weights must be strictly positive");
    std::vector<float> kf((size_t)n * m * m), al(n);
    int zero_mean = m > 1;
    for (int i = 0; i < n; ++i) {
        al[i] = (float)weights[i];
        double sum = 0.0, asum = 0.0;
        for (int a = 0; a < m; ++a)
            for (int b = 0; b < m; ++b) {  // cv2.filter2D correlates with the flipped kernel, image.py:49-50
                const double v = filters[(size_t)i * m * m + (m - 1 - a) * m + (m - 1 - b)];
                kf[(size_t)i * m * m + a * m + b] = (float)v;
                sum += v;
                asum += fabs(v);
            }
        if (!(fabs(sum) <= 1e-9 * asum)) zero_mean = 0;
    }
    if (zero_mean) {
        // the fp32 taps of a zero-mean filter are made to sum to zero as well (adjust the largest tap
        // by the exact fp32 residual), so shifting the input by a constant leaves K u unchanged
        for (int i = 0; i < n; ++i) {
            float *k = kf.data() + (size_t)i * m * m;
            double s32 = 0.0;
            int big = 0;
            for (int e = 0; e < m * m; ++e) {
                s32 += (double)k[e];
                if (fabsf(k[e]) > fabsf(k[big])) big = e;
            }
            k[big] = (float)((double)k[big] - s32);
        }
    }
    foe_bank *bk = new foe_bank();
    bk->n = n; bk->m = m; bk->boundary = boundary; bk->zero_mean = zero_mean;
    cudaGetDevice(&bk->device);
    if (cudaMalloc(&bk->d_kf, kf.size() * sizeof(float)) != cudaSuccess ||
        cudaMalloc(&bk->d_alpha, al.size() * sizeof(float)) != cudaSuccess) {
        delete bk;
        return fail(FOE_E_CUDA, "cudaMalloc failed for the filter bank");
    }
    FOE_CUDA(cudaMemcpy(bk->d_kf, kf.data(), kf.size() * sizeof(float), cudaMemcpyHostToDevice));
    FOE_CUDA(cudaMemcpy(bk->d_alpha, al.data(), al.size() * sizeof(float), cudaMemcpyHostToDevice));
    if (m == 5 && n <= 32) {
        const std::vector<float> img = tc_operand_image(kf.data(), al.data(), n);
        if (cudaMalloc(&bk->d_tc_img, img.size() * sizeof(float)) != cudaSuccess) {
            foe_bank_destroy(bk);
            return fail(FOE_E_CUDA, "cudaMalloc failed for the operand image");
        }
        FOE_CUDA(cudaMemcpy(bk->d_tc_img, img.data(), img.size() * sizeof(float), cudaMemcpyHostToDevice));
    }
    *out = bk;
    return FOE_OK;
}

int foe_bank_destroy(foe_bank *bank) {
    if (!bank) return FOE_OK;
    cudaFree(bank->d_kf);
    cudaFree(bank->d_alpha);
    cudaFree(bank->d_tc_img);
    delete bank;
    return FOE_OK;
}

int foe_bank_info(const foe_bank *bank, int *n, int *m, int *boundary) {
    if (!bank) return fail(FOE_E_INVALID, "null bank");
    if (n) *n = bank->n;
    if (m) *m = bank->m;
    if (boundary) *boundary = bank->boundary;
    return FOE_OK;
}

int foe_anscombe_forward(const double *y, float *v, int64_t n, void *stream) {
    if (n <= 0) return FOE_OK;
    g_launches.fetch_add(1, std::memory_order_relaxed);
    k_anscombe_fwd<<<grid_1d(n), 256, 0, (cudaStream_t)stream>>>(y, v, n);
    FOE_CUDA(cudaGetLastError());
    return FOE_OK;
}

int foe_anscombe_forward_f32(const float *y, float *v, int64_t n, void *stream) {
    if (n <= 0) return FOE_OK;
    g_launches.fetch_add(1, std::memory_order_relaxed);
    k_anscombe_fwd_f32<<<grid_1d(n), 256, 0, (cudaStream_t)stream>>>(y, v, n);
    FOE_CUDA(cudaGetLastError());
    return FOE_OK;
}

int foe_direct_obs(const double *y, float *obs, double c, int64_t n, void *stream) {
    if (c < 0) return fail(FOE_E_INVALID, "zero_offset_c must be non-negative");
    if (n <= 0) return FOE_OK;
    g_launches.fetch_add(1, std::memory_order_relaxed);
    k_direct_obs<<<grid_1d(n), 256, 0, (cudaStream_t)stream>>>(y, obs, c, n);
    FOE_CUDA(cudaGetLastError());
    return FOE_OK;
}

int foe_anscombe_inverse_exact_unbiased(const float *z, double *x, int64_t n, unsigned long long *counts,
                                        void *stream) {
    if (n <= 0) return FOE_OK;
    g_launches.fetch_add(1, std::memory_order_relaxed);
    k_inverse_exact_unbiased<<<grid_1d(n), 256, 0, (cudaStream_t)stream>>>(z, x, n, counts);
    FOE_CUDA(cudaGetLastError());
    return FOE_OK;
}

int foe_prox_quadratic(const float *ut, const float *v, float *out, double t, int64_t n, void *stream) {
    if (t < 0) return fail(FOE_E_INVALID, "t must be >= 0, got %g", t);  // solver.py:94-95
    if (n <= 0) return FOE_OK;
    g_launches.fetch_add(1, std::memory_order_relaxed);
    k_prox_quadratic<<<grid_1d(n), 256, 0, (cudaStream_t)stream>>>(ut, v, out, (float)t, n);
    FOE_CUDA(cudaGetLastError());
    return FOE_OK;
}

int foe_prox_idiv(const float *ut, const float *obs, float *out, double t, int64_t n, void *stream) {
    if (t < 0) return fail(FOE_E_INVALID, "t must be >= 0, got %g", t);  // solver.py:111-112
    if (n <= 0) return FOE_OK;
    g_launches.fetch_add(1, std::memory_order_relaxed);
    k_prox_idiv<<<grid_1d(n), 256, 0, (cudaStream_t)stream>>>(ut, obs, out, (float)t, n);
    FOE_CUDA(cudaGetLastError());
    return FOE_OK;
}

int foe_convolve_same(const foe_bank *bank, int index, const float *x, float *out, int B, int H, int W,
                      void *stream) {
    int rc = check_dims(bank, B, H, W);
    if (rc) return rc;
    if (index < 0 || index >= bank->n) return fail(FOE_E_INVALID, "filter index %d out of range", index);
    const int64_t n = (int64_t)B * H * W;
    const float *kf = bank->d_kf + (size_t)index * bank->m * bank->m;
    if (bank->boundary == FOE_SYMMETRIC)
        k_conv_same<true><<<grid_1d(n), 256, 0, (cudaStream_t)stream>>>(x, out, kf, bank->m, B, H, W);
    else
        k_conv_same<false><<<grid_1d(n), 256, 0, (cudaStream_t)stream>>>(x, out, kf, bank->m, B, H, W);
    FOE_CUDA(cudaGetLastError());
    return FOE_OK;
}

int foe_convolve_adjoint(const foe_bank *bank, int index, const float *y, float *out, int B, int H, int W,
                         void *stream) {
    // the adjoint correlates with the unflipped kernel: reverse the stored flipped taps on the fly
    int rc = check_dims(bank, B, H, W);
    if (rc) return rc;
    if (index < 0 || index >= bank->n) return fail(FOE_E_INVALID, "filter index %d out of range", index);
    const int m = bank->m;
    std::vector<float> kf((size_t)m * m), k((size_t)m * m);
    FOE_CUDA(cudaMemcpy(kf.data(), bank->d_kf + (size_t)index * m * m, sizeof(float) * m * m, cudaMemcpyDeviceToHost));
    for (int i = 0; i < m * m; ++i) k[i] = kf[m * m - 1 - i];
    float *dk = nullptr;
    FOE_CUDA(cudaMallocAsync(&dk, sizeof(float) * m * m, (cudaStream_t)stream));
    FOE_CUDA(cudaMemcpyAsync(dk, k.data(), sizeof(float) * m * m, cudaMemcpyHostToDevice, (cudaStream_t)stream));
    const int64_t n = (int64_t)B * H * W;
    if (bank->boundary == FOE_SYMMETRIC)
        k_conv_adjoint<true><<<grid_1d(n), 256, 0, (cudaStream_t)stream>>>(y, out, dk, m, B, H, W);
    else
        k_conv_adjoint<false><<<grid_1d(n), 256, 0, (cudaStream_t)stream>>>(y, out, dk, m, B, H, W);
    FOE_CUDA(cudaGetLastError());
    FOE_CUDA(cudaFreeAsync(dk, (cudaStream_t)stream));
    FOE_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
    return FOE_OK;
}

size_t foe_eval_workspace_size(const foe_bank *bank, int B, int H, int W) {
    if (!bank) return 0;
    int tx, ty;
    tile_counts(bank->m, H, W, &tx, &ty);
    return align_up(sizeof(double) * kPartialStride * (size_t)B * tx * ty) + align_up(sizeof(unsigned) * B);
}

int foe_energy_grad(const foe_bank *bank, const float *u, float *grad, double *energy, int B, int H, int W,
                    void *workspace, size_t workspace_bytes, void *stream) {
    int rc = check_dims(bank, B, H, W);
    if (rc) return rc;
    if (workspace_bytes < foe_eval_workspace_size(bank, B, H, W)) return fail(FOE_E_INVALID, "workspace too small");
    cudaStream_t st = (cudaStream_t)stream;
    PassArgs a{};
    a.B = B; a.H = H; a.W = W; a.n_filters = bank->n; a.zero_mean = bank->zero_mean;
    tile_counts(bank->m, H, W, &a.tiles_x, &a.tiles_y);
    a.tiles_yl = a.tiles_y; a.ty0 = 0; a.lrow0 = 0; a.Hl = H; a.band = 0;
    a.mode = MODE_EVAL;
    a.kf = bank->d_kf; a.alpha = bank->d_alpha; a.tc_img = bank->d_tc_img;
    a.u_in = u; a.g_out = grad; a.energy_out = energy;
    a.partials = (double *)workspace;
    a.tickets = (unsigned *)((char *)workspace + align_up(sizeof(double) * kPartialStride * (size_t)B * a.tiles_x * a.tiles_y));
    FOE_CUDA(cudaMemsetAsync(a.tickets, 0, sizeof(unsigned) * B, st));
    return launch_pass(bank->m, bank->boundary == FOE_SYMMETRIC, a, st);
}

size_t foe_solve_workspace_size(const foe_bank *bank, int B, int H, int W, int trace_cap) {
    if (!bank) return 0;
    return solve_layout(bank->m, B, H, W, trace_cap).total;
}

static void fill_solve_args(PassArgs &a, const foe_bank *bank, const foe_solver_cfg &cfg, int B, int H, int W,
                            int trace_cap, char *ws, const SolveLayout &L, const foe_band_desc *band = nullptr) {
    a.B = B; a.H = H; a.W = W; a.n_filters = bank->n; a.zero_mean = bank->zero_mean;
    tile_counts(bank->m, H, W, &a.tiles_x, &a.tiles_y);
    if (band) {
        a.ty0 = band->ty0; a.tiles_yl = band->ty1 - band->ty0; a.lrow0 = band->lrow0; a.Hl = band->Hl; a.band = 1;
    } else {
        a.ty0 = 0; a.tiles_yl = a.tiles_y; a.lrow0 = 0; a.Hl = H; a.band = 0;
    }
    a.plane = (size_t)B * a.Hl * W;
    a.kf = bank->d_kf; a.alpha = bank->d_alpha; a.tc_img = bank->d_tc_img;
    a.U = (float *)(ws + L.U);
    a.Gs = (float *)(ws + L.G);
    a.obs = (const float *)(ws + L.O);
    a.ctl = (ImgCtl *)(ws + L.ctl);
    a.partials = (double *)(ws + L.partials);
    a.tickets = (unsigned *)(ws + L.tickets);
    a.trace = (double *)(ws + L.trace);
    a.trace_cap = trace_cap;
    a.n_active = (int *)(ws + L.n_active);
    a.gamma = cfg.gamma;
    a.step_num = 1.99 * (1.0 - cfg.gamma);  // solver.py:64-65
    a.eta = cfg.backtrack_factor;
    a.relax = cfg.relax_factor;
    a.rel_tol = cfg.rel_tol;
    a.max_L = cfg.max_lipschitz;
}

int foe_solve(const foe_bank *bank, const foe_solver_cfg *cfgp, int B, int H, int W, const float *u0,
              const float *obs, const double *lam, const int *branch, const int *max_iters, float *u_out,
              foe_image_status *status, double *trace, int trace_cap, void *workspace, size_t workspace_bytes,
              void *stream) {
    int rc = check_dims(bank, B, H, W);
    if (rc) return rc;
    if (!cfgp || !u0 || !obs || !lam || !branch || !max_iters || !u_out || !status || !trace)
        return fail(FOE_E_INVALID, "null argument");
    const foe_solver_cfg cfg = *cfgp;
    // SolverConfig.__post_init__, solver.py:54-62
    if (!(cfg.gamma >= 0.0 && cfg.gamma < 1.0)) return fail(FOE_E_INVALID, "gamma must be in [0, 1), got %g", cfg.gamma);
    if (!(cfg.lipschitz_init > 0)) return fail(FOE_E_INVALID, "lipschitz_init must be positive");
    if (!(cfg.backtrack_factor > 1)) return fail(FOE_E_INVALID, "backtrack_factor must exceed 1");
    int max_it = 0, min_it = 1 << 30;
    for (int b = 0; b < B; ++b) {
        if (max_iters[b] < 1) return fail(FOE_E_INVALID, "max_iters must be at least 1");
        if (!(lam[b] > 0)) return fail(FOE_E_INVALID, "lambda must be positive, got %g", lam[b]);
        if (branch[b] != FOE_QUADRATIC && branch[b] != FOE_IDIV) return fail(FOE_E_INVALID, "bad branch");
        max_it = std::max(max_it, max_iters[b]);
        min_it = std::min(min_it, max_iters[b]);
    }
    if (trace_cap < max_it) return fail(FOE_E_INVALID, "trace_cap %d < max_iters %d", trace_cap, max_it);
    const SolveLayout L = solve_layout(bank->m, B, H, W, trace_cap);
    if (workspace_bytes < L.total) return fail(FOE_E_INVALID, "workspace too small (%zu < %zu)", workspace_bytes, L.total);
    cudaStream_t st = (cudaStream_t)stream;
    char *ws = (char *)workspace;
    PassArgs a{};
    fill_solve_args(a, bank, cfg, B, H, W, trace_cap, ws, L);

    std::vector<ImgCtl> hc(B);
    for (int b = 0; b < B; ++b) {
        ImgCtl &c = hc[b];
        memset(&c, 0, sizeof(c));
        c.L = cfg.lipschitz_init;
        c.lam = lam[b];
        c.max_iters = max_iters[b];
        c.branch = branch[b];
        c.failed_at = -1;
        c.iu = 0; c.iup = 2; c.inew = 1;  // u_prev = u = u0 (solver.py:136-137), distinct slots
        set_step(c, a.step_num);
        c.ig = 0; c.ignew = 1;
    }
    const size_t HWB = (size_t)B * H * W;
    FOE_CUDA(cudaMemcpyAsync(a.ctl, hc.data(), sizeof(ImgCtl) * B, cudaMemcpyHostToDevice, st));
    FOE_CUDA(cudaMemsetAsync(a.tickets, 0, sizeof(unsigned) * B, st));
    {
        const int live[4] = {B, 0, 0, 0};  // live images, loop-graph pass count, loop-graph cap flag
        FOE_CUDA(cudaMemcpyAsync(a.n_active, live, sizeof(live), cudaMemcpyHostToDevice, st));
    }
    FOE_CUDA(cudaMemcpyAsync(a.U, u0, sizeof(float) * HWB, cudaMemcpyDeviceToDevice, st));
    FOE_CUDA(cudaMemcpyAsync(a.U + 2 * a.plane, u0, sizeof(float) * HWB, cudaMemcpyDeviceToDevice, st));
    FOE_CUDA(cudaMemcpyAsync((float *)(ws + L.O), obs, sizeof(float) * HWB, cudaMemcpyDeviceToDevice, st));

    // iteration 0 needs F(u0) and grad F(u0)
    a.mode = MODE_INIT;
    if ((rc = launch_pass(bank->m, bank->boundary == FOE_SYMMETRIC, a, st))) return rc;
    // every image needs >= 1 trial per accepted iteration: min_it passes straight away, then the
    // device-side loop graph until no image is live
    a.mode = MODE_TRIAL;
    for (int k = 0; k < std::max(1, min_it); ++k)
        if ((rc = launch_pass(bank->m, bank->boundary == FOE_SYMMETRIC, a, st))) return rc;
    const int cap = max_it * 200 + 64;
    cudaGraphExec_t exec = nullptr;
    if ((rc = loop_graph(bank->m, bank->boundary == FOE_SYMMETRIC, a, cap, &exec))) return rc;
    FOE_CUDA(cudaGraphLaunch(exec, st));
    // final-energy pass: F at each image's last accepted iterate, evaluated directly (INIT mode on the
    // final slot, no decision), to anchor the trace's F column (anchor_f_column)
    a.mode = MODE_INIT;
    a.no_decide = 1;
    a.energy_out = (double *)(ws + L.energy);
    if ((rc = launch_pass(bank->m, bank->boundary == FOE_SYMMETRIC, a, st))) return rc;
    a.no_decide = 0;
    a.energy_out = nullptr;
    {
        dim3 grid(std::max(1, std::min(148, (int)((size_t)H * W / 1024 + 1))), B);
        g_launches.fetch_add(1, std::memory_order_relaxed);
        k_gather_final<<<grid, 256, 0, st>>>(a.U, a.plane, a.ctl, u_out, (size_t)H * W, B);
        FOE_CUDA(cudaGetLastError());
    }
    FOE_CUDA(cudaMemcpyAsync(hc.data(), a.ctl, sizeof(ImgCtl) * B, cudaMemcpyDeviceToHost, st));
    FOE_CUDA(cudaMemcpyAsync(trace, a.trace, sizeof(double) * 6 * (size_t)B * trace_cap, cudaMemcpyDeviceToHost, st));
    int loop_info[4] = {0, 0, 0, 0};
    std::vector<double> energy(B);
    FOE_CUDA(cudaMemcpyAsync(loop_info, a.n_active, sizeof(loop_info), cudaMemcpyDeviceToHost, st));
    FOE_CUDA(cudaMemcpyAsync(energy.data(), ws + L.energy, sizeof(double) * B, cudaMemcpyDeviceToHost, st));
    FOE_CUDA(cudaStreamSynchronize(st));
    anchor_f_column(trace, trace_cap, hc, energy);
    g_launches.fetch_add(loop_info[1] + loop_info[1] / kGraphChunk, std::memory_order_relaxed);
    if (loop_info[2]) return fail(FOE_E_NUMERICAL, "solver did not terminate after %d passes", loop_info[1]);
    int any_fail = 0;
    for (int b = 0; b < B; ++b) {
        status[b].status = hc[b].status;
        status[b].n_iters = hc[b].n;
        status[b].n_trials = hc[b].trials;
        status[b].failed_at = hc[b].status ? hc[b].failed_at : -1;
        any_fail |= hc[b].status != 0;
    }
    return any_fail ? fail(FOE_E_NUMERICAL, "numerical failure in at least one image") : FOE_OK;
}

int foe_debug_pass_times_seq(const foe_bank *bank, int B, int H, int W, int trace_cap, void *workspace,
                             size_t workspace_bytes, unsigned long long *times, int n_passes, void *stream) {
    int rc = check_dims(bank, B, H, W);
    if (rc) return rc;
    const SolveLayout L = solve_layout(bank->m, B, H, W, trace_cap);
    if (workspace_bytes < L.total) return fail(FOE_E_INVALID, "workspace too small");
    foe_solver_cfg cfg{0.8, 1.0, 1.2, 1.05, 1e-6, 1e15};
    PassArgs a{};
    fill_solve_args(a, bank, cfg, B, H, W, trace_cap, (char *)workspace, L);
    a.mode = MODE_TRIAL;
    a.no_decide = 1;
    // per pass: [cta][start, loop start, ticket seen] | 512 phase stamps | [cta] dependency released | [cta] decider done
    const size_t stride = 5 * (size_t)a.tiles_x * a.tiles_y * B + 512;
    for (int k = 0; k < n_passes; ++k) {
        a.dbg_times = times + k * stride;
        if ((rc = launch_pass(bank->m, bank->boundary == FOE_SYMMETRIC, a, (cudaStream_t)stream))) return rc;
    }
    return FOE_OK;
}

int foe_debug_pass_times(const foe_bank *bank, int B, int H, int W, int trace_cap, void *workspace,
                         size_t workspace_bytes, unsigned long long *times, void *stream) {
    int rc = check_dims(bank, B, H, W);
    if (rc) return rc;
    const SolveLayout L = solve_layout(bank->m, B, H, W, trace_cap);
    if (workspace_bytes < L.total) return fail(FOE_E_INVALID, "workspace too small");
    foe_solver_cfg cfg{0.8, 1.0, 1.2, 1.05, 1e-6, 1e15};
    PassArgs a{};
    fill_solve_args(a, bank, cfg, B, H, W, trace_cap, (char *)workspace, L);
    a.mode = MODE_TRIAL;
    a.no_decide = 1;
    a.dbg_times = times;
    return launch_pass(bank->m, bank->boundary == FOE_SYMMETRIC, a, (cudaStream_t)stream);
}

int foe_bench_trial_pass(const foe_bank *bank, int B, int H, int W, int trace_cap, int reps, void *workspace,
                         size_t workspace_bytes, void *stream) {
    int rc = check_dims(bank, B, H, W);
    if (rc) return rc;
    const SolveLayout L = solve_layout(bank->m, B, H, W, trace_cap);
    if (workspace_bytes < L.total) return fail(FOE_E_INVALID, "workspace too small");
    foe_solver_cfg cfg{0.8, 1.0, 1.2, 1.05, 1e-6, 1e15};
    PassArgs a{};
    fill_solve_args(a, bank, cfg, B, H, W, trace_cap, (char *)workspace, L);
    a.mode = MODE_TRIAL;
    a.no_decide = 1;
    for (int k = 0; k < reps; ++k)
        if ((rc = launch_pass(bank->m, bank->boundary == FOE_SYMMETRIC, a, (cudaStream_t)stream))) return rc;
    return FOE_OK;
}


int foe_tile_grid(int m, int H, int W, int *tiles_x, int *tiles_y) {
    if (m < 1 || m % 2 != 1 || m > 7) return fail(FOE_E_INVALID, "bad filter size %d", m);
    int tx, ty;
    tile_counts(m, H, W, &tx, &ty);
    if (tiles_x) *tiles_x = tx;
    if (tiles_y) *tiles_y = ty;
    return FOE_OK;
}

int foe_band_describe(const foe_bank *bank, int B, int H, int W, int ty0, int ty1, foe_band_desc *d) {
    int rc = check_dims(bank, B, H, W);
    if (rc) return rc;
    if (bank->boundary != FOE_SYMMETRIC)
        return fail(FOE_E_UNSUPPORTED, "row bands support the symmetric boundary only");
    return foe_band_geometry(bank->m, B, H, W, ty0, ty1, d);
}

int foe_band_geometry(int m, int B, int H, int W, int ty0, int ty1, foe_band_desc *d) {
    if (!d || m < 1 || m % 2 != 1 || m > 7 || B < 1 || H < m || W < m) return fail(FOE_E_INVALID, "bad geometry");
    int tx, ty;
    tile_counts(m, H, W, &tx, &ty);
    if (ty0 < 0 || ty1 > ty || ty0 >= ty1) return fail(FOE_E_INVALID, "tile rows [%d, %d) outside [0, %d)", ty0, ty1, ty);
    const int r = m / 2, T = region_rows(m) - 2 * r;
    d->B = B; d->H = H; d->W = W; d->ty0 = ty0; d->ty1 = ty1; d->tiles_x = tx; d->tiles_y = ty;
    d->row0 = tile_start(ty0, ty, T, H, r);
    d->row1 = tile_start(ty1, ty, T, H, r);
    d->halo = 2 * r;  // the trial point is formed on the region + r ring = owned rows +- 2r
    if (ty0 > 0 && d->row1 - d->row0 < d->halo) return fail(FOE_E_INVALID, "band thinner than its halo");
    d->lrow0 = std::max(0, d->row0 - d->halo);
    d->Hl = std::min(H, d->row1 + d->halo) - d->lrow0;
    return FOE_OK;
}

size_t foe_band_workspace_size(const foe_bank *bank, const foe_band_desc *d, int trace_cap) {
    if (!bank || !d) return 0;
    return solve_layout(bank->m, d->B, d->H, d->W, trace_cap, d->Hl, d->halo).total;
}

int foe_band_buffers_get(const foe_bank *bank, const foe_band_desc *d, int trace_cap, void *workspace,
                         foe_band_buffers *out) {
    if (!bank || !d || !out) return fail(FOE_E_INVALID, "null argument");
    const SolveLayout L = solve_layout(bank->m, d->B, d->H, d->W, trace_cap, d->Hl, d->halo);
    char *ws = (char *)workspace;
    out->partials = (double *)(ws + L.partials);
    out->partials_offset = (size_t)d->ty0 * d->tiles_x * d->B * kPartialStride;
    out->partials_count = (size_t)(d->ty1 - d->ty0) * d->tiles_x * d->B * kPartialStride;
    out->partials_total = (size_t)d->tiles_y * d->tiles_x * d->B * kPartialStride;
    out->sendbuf = (float *)(ws + L.send);
    out->recvbuf = (float *)(ws + L.recv);
    out->halo_count = L.halo_floats;
    out->n_active = (int *)(ws + L.n_active);
    return FOE_OK;
}

static int band_args(const foe_bank *bank, const foe_band_desc *d, int trace_cap, void *workspace,
                     size_t workspace_bytes, PassArgs &a, SolveLayout &L, const foe_solver_cfg *cfgp = nullptr) {
    if (!bank || !d || !workspace) return fail(FOE_E_INVALID, "null argument");
    L = solve_layout(bank->m, d->B, d->H, d->W, trace_cap, d->Hl, d->halo);
    if (workspace_bytes < L.total) return fail(FOE_E_INVALID, "band workspace too small");
    static const foe_solver_cfg def{0.8, 1.0, 1.2, 1.05, 1e-6, 1e15};  // only for cfg-free calls
    memset(&a, 0, sizeof(a));
    fill_solve_args(a, bank, cfgp ? *cfgp : def, d->B, d->H, d->W, trace_cap, (char *)workspace, L, d);
    return FOE_OK;
}

int foe_band_begin(const foe_bank *bank, const foe_solver_cfg *cfg, const foe_band_desc *d, const float *u0_local,
                   const float *obs_local, const double *lam, const int *branch, const int *max_iters, int trace_cap,
                   void *workspace, size_t workspace_bytes, void *stream) {
    if (!cfg || !u0_local || !obs_local || !lam || !branch || !max_iters) return fail(FOE_E_INVALID, "null argument");
    PassArgs a;
    SolveLayout L;
    int rc = band_args(bank, d, trace_cap, workspace, workspace_bytes, a, L, cfg);
    if (rc) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    const int B = d->B;
    std::vector<ImgCtl> hc(B);
    for (int b = 0; b < B; ++b) {
        if (max_iters[b] < 1 || max_iters[b] > trace_cap) return fail(FOE_E_INVALID, "bad max_iters");
        if (!(lam[b] > 0)) return fail(FOE_E_INVALID, "lambda must be positive");
        ImgCtl &c = hc[b];
        memset(&c, 0, sizeof(c));
        c.L = cfg->lipschitz_init; c.lam = lam[b]; c.max_iters = max_iters[b]; c.branch = branch[b]; c.failed_at = -1;
        c.iu = 0; c.iup = 2; c.inew = 1; c.ig = 0; c.ignew = 1;
        set_step(c, a.step_num);
    }
    const size_t local = (size_t)B * d->Hl * d->W;
    FOE_CUDA(cudaMemcpyAsync(a.ctl, hc.data(), sizeof(ImgCtl) * B, cudaMemcpyHostToDevice, st));
    FOE_CUDA(cudaMemcpyAsync(a.n_active, &B, sizeof(int), cudaMemcpyHostToDevice, st));
    FOE_CUDA(cudaMemcpyAsync(a.U, u0_local, sizeof(float) * local, cudaMemcpyDeviceToDevice, st));
    FOE_CUDA(cudaMemcpyAsync(a.U + 2 * a.plane, u0_local, sizeof(float) * local, cudaMemcpyDeviceToDevice, st));
    FOE_CUDA(cudaMemcpyAsync((void *)a.obs, obs_local, sizeof(float) * local, cudaMemcpyDeviceToDevice, st));
    a.mode = MODE_INIT;
    if ((rc = launch_pass(bank->m, true, a, st))) return rc;
    g_launches.fetch_add(1, std::memory_order_relaxed);
    k_band_pack<<<dim3(32, B), 256, 0, st>>>(a, (float *)((char *)workspace + L.send), d->halo, d->row0, d->row1, 1);
    FOE_CUDA(cudaGetLastError());
    return FOE_OK;
}

int foe_band_trial(const foe_bank *bank, const foe_solver_cfg *cfg, const foe_band_desc *d, int trace_cap,
                   void *workspace, size_t workspace_bytes, void *stream) {
    PassArgs a;
    SolveLayout L;
    int rc = band_args(bank, d, trace_cap, workspace, workspace_bytes, a, L, cfg);
    if (rc) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    a.mode = MODE_TRIAL;
    if ((rc = launch_pass(bank->m, true, a, st))) return rc;
    g_launches.fetch_add(1, std::memory_order_relaxed);
    k_band_pack<<<dim3(32, d->B), 256, 0, st>>>(a, (float *)((char *)workspace + L.send), d->halo, d->row0, d->row1, 0);
    FOE_CUDA(cudaGetLastError());
    return FOE_OK;
}

int foe_band_commit(const foe_bank *bank, const foe_solver_cfg *cfg, const foe_band_desc *d, int trace_cap, int init,
                    void *workspace, size_t workspace_bytes, void *stream) {
    PassArgs a;
    SolveLayout L;
    int rc = band_args(bank, d, trace_cap, workspace, workspace_bytes, a, L, cfg);
    if (rc) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    a.mode = init ? MODE_INIT : MODE_TRIAL;
    g_launches.fetch_add(2, std::memory_order_relaxed);
    k_band_unpack<<<dim3(32, d->B), 256, 0, st>>>(a, (const float *)((char *)workspace + L.recv), d->halo, d->row0,
                                                 d->row1, init);
    FOE_CUDA(cudaGetLastError());
    k_decide<<<d->B, PassCfg<5>::NT, 0, st>>>(a);
    FOE_CUDA(cudaGetLastError());
    return FOE_OK;
}

int foe_band_final_pass(const foe_bank *bank, const foe_solver_cfg *cfg, const foe_band_desc *d, int trace_cap,
                        void *workspace, size_t workspace_bytes, void *stream) {
    PassArgs a;
    SolveLayout L;
    int rc = band_args(bank, d, trace_cap, workspace, workspace_bytes, a, L, cfg);
    if (rc) return rc;
    a.mode = MODE_INIT;  // F and its tile partials at every image's final slot, no decision
    a.no_decide = 1;
    return launch_pass(bank->m, true, a, (cudaStream_t)stream);
}

int foe_band_end(const foe_bank *bank, const foe_band_desc *d, int trace_cap, void *workspace, size_t workspace_bytes,
                 float *u_owned, foe_image_status *status, double *trace, void *stream) {
    PassArgs a;
    SolveLayout L;
    int rc = band_args(bank, d, trace_cap, workspace, workspace_bytes, a, L);
    if (rc) return rc;
    if (!u_owned || !status || !trace) return fail(FOE_E_INVALID, "null argument");
    cudaStream_t st = (cudaStream_t)stream;
    const int B = d->B;
    g_launches.fetch_add(1, std::memory_order_relaxed);
    k_gather_band<<<dim3(64, B), 256, 0, st>>>(a.U, a.plane, a.ctl, u_owned, d->Hl, d->W, d->row0, d->row1, d->lrow0);
    FOE_CUDA(cudaGetLastError());
    // final energy from the all-gathered partials of foe_band_final_pass (the same fixed order on every
    // band and in the single-device solve), to anchor the F column exactly as foe_solve does
    g_launches.fetch_add(1, std::memory_order_relaxed);
    k_band_energy<<<B, PassCfg<5>::NT, 0, st>>>(a, (double *)((char *)workspace + L.energy));
    FOE_CUDA(cudaGetLastError());
    std::vector<ImgCtl> hc(B);
    std::vector<double> energy(B);
    FOE_CUDA(cudaMemcpyAsync(hc.data(), a.ctl, sizeof(ImgCtl) * B, cudaMemcpyDeviceToHost, st));
    FOE_CUDA(cudaMemcpyAsync(trace, a.trace, sizeof(double) * 6 * (size_t)B * trace_cap, cudaMemcpyDeviceToHost, st));
    FOE_CUDA(cudaMemcpyAsync(energy.data(), (char *)workspace + L.energy, sizeof(double) * B, cudaMemcpyDeviceToHost, st));
    FOE_CUDA(cudaStreamSynchronize(st));
    anchor_f_column(trace, trace_cap, hc, energy);
    int any_fail = 0;
    for (int b = 0; b < B; ++b) {
        status[b].status = hc[b].status;
        status[b].n_iters = hc[b].n;
        status[b].n_trials = hc[b].trials;
        status[b].failed_at = hc[b].status ? hc[b].failed_at : -1;
        any_fail |= hc[b].status != 0;
    }
    return any_fail ? fail(FOE_E_NUMERICAL, "numerical failure in at least one image") : FOE_OK;
}


int foe_bin(const double *y, double *yb, int H, int W, int factor, void *stream) {
    if (factor < 1 || H < 1 || W < 1) return fail(FOE_E_INVALID, "bad bin arguments");
    const int Hb = (H + factor - 1) / factor, Wb = (W + factor - 1) / factor;
    g_launches.fetch_add(1, std::memory_order_relaxed);
    k_bin<<<grid_1d((int64_t)Hb * Wb), 256, 0, (cudaStream_t)stream>>>(y, yb, H, W, factor, Hb, Wb);
    FOE_CUDA(cudaGetLastError());
    return FOE_OK;
}

int foe_unbin_bilinear(const double *xb, double *out, int h, int w, int H, int W, int factor, void *stream) {
    if (factor < 1 || h < 1 || w < 1 || H < h || W < w) return fail(FOE_E_INVALID, "bad unbin arguments");
    g_launches.fetch_add(1, std::memory_order_relaxed);
    k_unbin<<<grid_1d((int64_t)H * W), 256, 0, (cudaStream_t)stream>>>(xb, out, h, w, H, W, factor);
    FOE_CUDA(cudaGetLastError());
    return FOE_OK;
}



int foe_estimate_peak(const double *y, int H, int W, unsigned long long *scratch, double *peak, void *stream) {
    if (!y || !scratch || !peak || H < 1 || W < 1) return fail(FOE_E_INVALID, "bad estimate_peak arguments");
    cudaStream_t st = (cudaStream_t)stream;
    unsigned long long host = 0ull;
    FOE_CUDA(cudaMemsetAsync(scratch, 0, sizeof(unsigned long long), st));
    g_launches.fetch_add(1, std::memory_order_relaxed);
    k_median3_max<<<grid_1d((int64_t)H * W), 256, 0, st>>>(y, H, W, scratch);
    FOE_CUDA(cudaGetLastError());
    FOE_CUDA(cudaMemcpyAsync(&host, scratch, sizeof(host), cudaMemcpyDeviceToHost, st));
    FOE_CUDA(cudaStreamSynchronize(st));
    const unsigned long long b = (host >> 63) ? (host & 0x7fffffffffffffffull) : ~host;
    double v;
    memcpy(&v, &b, sizeof(v));
    *peak = v;
    return FOE_OK;
}

int foe_measure_ffma_peak(int iters, float *scratch, double *flop_out, void *stream) {
    int dev = 0, sms = 0;
    FOE_CUDA(cudaGetDevice(&dev));
    FOE_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int blocks = sms * 4;
    k_ffma_peak<<<blocks, 512, 0, (cudaStream_t)stream>>>(scratch, iters, 0.999f, 1e-4f);
    FOE_CUDA(cudaGetLastError());
    if (flop_out) *flop_out = 2.0 * 8 * 16 * (double)iters * 512 * blocks;
    return FOE_OK;
}

size_t foe_score_workspace_size(int B, int H, int W) {
    if (B < 1 || H < kSsimW || W < kSsimW) return 0;
    const size_t tiles = (size_t)((W - kSsimW + 1 + kSsimT - 1) / kSsimT) * ((H - kSsimW + 1 + kSsimT - 1) / kSsimT);
    return sizeof(double) * (size_t)B * (tiles + 256);
}

int foe_score(const double *x_hat, const double *g, int B, int H, int W, double peak, double *psnr,
              double *mssim, void *workspace, size_t workspace_bytes, void *stream) {
    if (B < 1 || H < kSsimW || W < kSsimW) return fail(FOE_E_INVALID, "images must be at least %d pixels per side", kSsimW);
    if (!(peak > 0)) return fail(FOE_E_INVALID, "peak must be positive");
    if (workspace_bytes < foe_score_workspace_size(B, H, W)) return fail(FOE_E_INVALID, "workspace too small");
    static bool init = false;
    if (!init) {  // metrics.py:41-45: normalised 1-D Gaussian, sigma 1.5; the 2-D window is its outer product
        double gw[kSsimW], sum = 0.0;
        for (int k = 0; k < kSsimW; ++k) {
            const double d = k - (kSsimW - 1) / 2.0;
            gw[k] = exp(-0.5 * (d / 1.5) * (d / 1.5));
            sum += gw[k];
        }
        for (int k = 0; k < kSsimW; ++k) gw[k] /= sum;
        FOE_CUDA(cudaMemcpyToSymbol(c_ssim_g, gw, sizeof(gw)));
        FOE_CUDA(cudaFuncSetAttribute(k_ssim_tiles, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
        init = true;
    }
    cudaStream_t st = (cudaStream_t)stream;
    const double scale = 255.0 / peak, dr = 255.0;  // metrics.py:93-101 scoring convention
    const int tx = (W - kSsimW + 1 + kSsimT - 1) / kSsimT, ty = (H - kSsimW + 1 + kSsimT - 1) / kSsimT;
    double *ss_part = (double *)workspace, *sq_part = ss_part + (size_t)B * tx * ty;
    const size_t smem = sizeof(double) * (2 * kSsimIn * kSsimIn + 5 * kSsimIn * kSsimT);
    k_ssim_tiles<<<dim3(tx, ty, B), 256, smem, st>>>(x_hat, g, H, W, scale, (0.01 * dr) * (0.01 * dr),
                                                     (0.03 * dr) * (0.03 * dr), ss_part);
    FOE_CUDA(cudaGetLastError());
    k_sqdiff<<<dim3(256, B), 256, 0, st>>>(x_hat, g, (int64_t)H * W, scale, sq_part);
    FOE_CUDA(cudaGetLastError());
    k_score_final<<<B, 32, 0, st>>>(sq_part, 256, ss_part, tx * ty, (int64_t)H * W,
                                    (int64_t)(H - kSsimW + 1) * (W - kSsimW + 1), dr, psnr, mssim);
    FOE_CUDA(cudaGetLastError());
    g_launches.fetch_add(3, std::memory_order_relaxed);
    return FOE_OK;
}

int foe_conv_bank64(const double *filters, int n, int m, int boundary, const double *x, double *out, int B, int H,
                    int W, void *stream) {
    return bank64<false>(filters, n, m, boundary, x, out, B, H, W, stream);
}

int foe_adjoint_bank64(const double *filters, int n, int m, int boundary, const double *y, double *out, int B, int H,
                       int W, void *stream) {
    return bank64<true>(filters, n, m, boundary, y, out, B, H, W, stream);
}

int foe_hessian_apply64(const double *filters, const double *weights, int n, int m, int boundary, int objective,
                        double lam, const double *w, const double *f, const unsigned char *free_mask, const double *p,
                        double eps, double *out, int H, int W, void *stream) {
    int rc = check_cg_model(filters, weights, n, m, boundary, objective, w, f, H, W);
    if (rc) return rc;
    if (!p || !out) return fail(FOE_E_INVALID, "null argument");
    CgArgs a{};
    a.H = H; a.W = W; a.n = n; a.objective = objective; a.lam = lam; a.eps = eps;
    a.kf = filters; a.wgt = weights; a.w = w; a.f = f; a.free_mask = free_mask;
    a.r = p; a.hp = out;
    return cg_hvp(m, boundary == FOE_SYMMETRIC, a, (cudaStream_t)stream);
}

size_t foe_cg_workspace_size(int H, int W, int max_iters) {
    if (H < 1 || W < 1 || max_iters < 0) return 0;
    return cg_layout(H, W, max_iters).total;
}

int foe_cg_solve64(const double *filters, const double *weights, int n, int m, int boundary, int objective, double lam,
                   const double *w, const double *f, const unsigned char *free_mask, const double *rhs, double eps,
                   double tol, int max_iters, double *q, int *status, int *iterations, double *residuals,
                   int H, int W, void *workspace, size_t workspace_bytes, void *stream) {
    int rc = check_cg_model(filters, weights, n, m, boundary, objective, w, f, H, W);
    if (rc) return rc;
    if (!rhs || !q || !status || !iterations || !residuals || !workspace || max_iters < 1)
        return fail(FOE_E_INVALID, "null argument or max_iters < 1");
    const CgLayout L = cg_layout(H, W, max_iters);
    if (workspace_bytes < L.total) return fail(FOE_E_INVALID, "workspace too small (%zu < %zu)", workspace_bytes, L.total);
    cudaStream_t st = (cudaStream_t)stream;
    char *ws = (char *)workspace;
    CgArgs a{};
    a.H = H; a.W = W; a.n = n; a.objective = objective; a.lam = lam; a.eps = eps;
    a.kf = filters; a.wgt = weights; a.w = w; a.f = f; a.free_mask = free_mask;
    a.r = (const double *)(ws + L.r);
    a.r_mut = (double *)(ws + L.r);
    a.d_prev = (const double *)(ws + L.da);
    a.d_next = (double *)(ws + L.db);
    a.hp = (double *)(ws + L.hp);
    a.q = q;
    a.part = (double *)(ws + L.part);
    a.tickets = (unsigned *)(ws + L.tickets);
    a.st = (CgState *)(ws + L.state);
    a.residuals = (double *)(ws + L.resid);
    const size_t npx = (size_t)H * W;
    FOE_CUDA(cudaMemsetAsync(a.tickets, 0, 2 * sizeof(unsigned), st));
    g_launches.fetch_add(1, std::memory_order_relaxed);
    k_cg_init<<<1, 256, 0, st>>>(a.st, rhs, a.r_mut, q, npx, tol, max_iters, a.residuals, a.part);
    FOE_CUDA(cudaGetLastError());
    // the iteration loop: a graph whose WHILE node repeats [H d, update] until k_cg_update clears it
    cudaGraph_t g = nullptr;
    FOE_CUDA(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle h;
    FOE_CUDA(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t node;
    FOE_CUDA(cudaGraphAddNode(&node, g, nullptr, 0, &cp));
    cudaStream_t cs;
    FOE_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    FOE_CUDA(cudaStreamBeginCaptureToGraph(cs, cp.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                           cudaStreamCaptureModeThreadLocal));
    a.cond = h;
    a.use_cond = 1;
    const long long before = g_launches.load();
    rc = cg_hvp(m, boundary == FOE_SYMMETRIC, a, cs);
    if (rc == FOE_OK) {
        k_cg_update<<<kCgUpdCtas, 256, 0, cs>>>(a);
        if (cudaGetLastError() != cudaSuccess) rc = fail(FOE_E_CUDA, "k_cg_update launch failed");
    }
    cudaGraph_t captured = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(cs, &captured);
    cudaStreamDestroy(cs);
    g_launches.store(before);
    cudaGraphExec_t exec = nullptr;
    if (rc == FOE_OK && ce == cudaSuccess) {
        const cudaError_t ie = cudaGraphInstantiate(&exec, g, 0);
        if (ie != cudaSuccess) rc = fail(FOE_E_CUDA, "CG graph instantiate: %s", cudaGetErrorString(ie));
    } else if (rc == FOE_OK) {
        rc = fail(FOE_E_CUDA, "CG graph capture: %s", cudaGetErrorString(ce));
    }
    cudaGraphDestroy(g);
    if (rc) return rc;
    const cudaError_t le = cudaGraphLaunch(exec, st);
    CgState hs{};
    cudaError_t me = cudaMemcpyAsync(&hs, a.st, sizeof(CgState), cudaMemcpyDeviceToHost, st);
    if (me == cudaSuccess)
        me = cudaMemcpyAsync(residuals, a.residuals, sizeof(double) * ((size_t)max_iters + 1), cudaMemcpyDeviceToHost, st);
    const cudaError_t se = cudaStreamSynchronize(st);
    cudaGraphExecDestroy(exec);
    FOE_CUDA(le);
    FOE_CUDA(me);
    FOE_CUDA(se);
    g_launches.fetch_add(2LL * hs.it + (hs.status == CG_BREAKDOWN ? 2 : 0), std::memory_order_relaxed);
    *status = hs.status;
    *iterations = hs.it;
    return FOE_OK;
}

int foe_pass_uses_tensor_cores(int m, int nf) { return (use_tc(m, nf) || use_tc7(m, nf)) ? 1 : 0; }

int foe_debug_tmem_rate(int nwarps, int store, int iters, long long *out_cycles, void *stream) {
    if (nwarps < 4 || nwarps > 32 || nwarps % 4) return fail(FOE_E_INVALID, "nwarps must be a multiple of 4 in 4..32");
    cudaStream_t st = (cudaStream_t)stream;
    if (store) k_tmem_rate<true><<<1, 32 * nwarps, 0, st>>>(iters, out_cycles);
    else k_tmem_rate<false><<<1, 32 * nwarps, 0, st>>>(iters, out_cycles);
    FOE_CUDA(cudaGetLastError());
    return FOE_OK;
}

int foe_debug_tc_rate(int n, int ts, int nmma, int nchain, int every, long long *out_cycles, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (n != 32 && n != 64 && n != 128) return fail(FOE_E_INVALID, "n must be 32, 64 or 128");
    if (nchain < 1 || nchain * n > 256) return fail(FOE_E_INVALID, "nchain accumulators of n columns must fit 256 columns");
    if (ts) {
        if (n == 32) k_tc_rate<32, true><<<1, 128, 0, st>>>(nmma, nchain, every, out_cycles);
        if (n == 64) k_tc_rate<64, true><<<1, 128, 0, st>>>(nmma, nchain, every, out_cycles);
        if (n == 128) k_tc_rate<128, true><<<1, 128, 0, st>>>(nmma, nchain, every, out_cycles);
    } else {
        if (n == 32) k_tc_rate<32, false><<<1, 128, 0, st>>>(nmma, nchain, every, out_cycles);
        if (n == 64) k_tc_rate<64, false><<<1, 128, 0, st>>>(nmma, nchain, every, out_cycles);
        if (n == 128) k_tc_rate<128, false><<<1, 128, 0, st>>>(nmma, nchain, every, out_cycles);
    }
    FOE_CUDA(cudaGetLastError());
    return FOE_OK;
}

int foe_tc_selftest(const float *A, const float *B, float *D, void *stream) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    k_tc_selftest<<<1, 128, 0, (cudaStream_t)stream>>>(A, B, D);
    FOE_CUDA(cudaGetLastError());
    return FOE_OK;
}

}  // extern "C"
