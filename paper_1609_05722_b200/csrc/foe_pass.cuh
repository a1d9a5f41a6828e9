// foe_pass.cuh -- the fused FoE pass (included by foe_b200.cu).
//
// One CTA = one tile of one image.  Region = owned tile + r ring (the pixels whose responses the
// adjoint needs); staged cells = region + another r ring (the inputs of those responses).
//
// Thread layout: 3 filter groups x 6 warps.  A warp covers 8 micro-columns x 4 micro-rows of
// 3x4-pixel micro-tiles, so each 8-lane LDS.128 phase reads 32 consecutive floats of one smem row
// (bank-conflict free for any pitch).  Each group owns a third of the filter bank and a ring of
// psi buffers, synchronised with split-phase mbarriers.
//
// Per filter and thread: forward z = K u_new and dz = K du on 12 pixels from a 5x8 (r=2) window
// streamed from smem (600 FFMA), pointwise psi = 2a z/(1+z^2) and the energy change
// a*log1p(dz(2z_o+dz)/(1+z_o^2)) evaluated as 2a*atanh(t), t = (z^2-z_o^2)/((1+z^2)+(1+z_o^2)),
// then the adjoint K^T psi (300 FFMA).
//
// k_pass: one launch per trial pass (any batch size, row bands); the last CTA of an image reduces
// the tile partials and decides.

template <int M_>
struct PassCfg {
    static constexpr int M = M_;
    static constexpr int R = M / 2;
    // region (owned tile + r ring): 36 x 64 (6 warps per filter group); 7 x 7 banks use 48 rows (8 warps
    // per group) so a 512^2 image is 13 x 9 = 117 tiles, one wave on 148 SMs instead of 162
    static constexpr int RH = (M_ == 7) ? 48 : 36, RW = 64;
    static constexpr int MY = 3, MX = 4;    // micro-tile per thread
    static constexpr int G = 2;             // filter groups per CTA (6 warps each: 3 warps per SMSP)
    static constexpr int NBUF = 3;          // psi buffers per group (pipelined mbarrier ring)
    static constexpr int NTX = RW / MX, NTY = RH / MY, NTG = NTX * NTY, NT = G * NTG;
    static constexpr int CW = RW + 2 * R;       // staged columns
    static constexpr int SH = RH + 2 * R;       // staged rows
    static constexpr int SW = (CW + 3) & ~3;    // row pitch (float4 aligned)
    static constexpr int PLANE = SH * SW;
    static constexpr int NPSI = G * NBUF;       // psi planes
    static constexpr int TH = RH - 2 * R, TW = RW - 2 * R;  // max owned tile
    static constexpr int TAPS = (M * M + 3) & ~3;           // per-filter tap stride (float4)
    static constexpr int NCELL = SH * CW;
    static constexpr int CPT = (NCELL + NT - 1) / NT;       // staged cells per thread
    static_assert(NTX == 16 && (NTY == 12 || NTY == 16), "warp layout: 16 x 12 or 16 x 16 micro-tiles per group");
    static_assert(TH >= 2 * R, "tile too small for the fold rule");
    static_assert(G * RH * RW <= NPSI * PLANE, "group partial-gradient buffer must fit the psi planes");
    static_assert(NT % RW == 0, "fold walk assumes whole region rows per pass");
};


__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ float rcp_approx(float x) {  // MUFU.RCP, no denormal fix-up
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// programmatic dependent launch (the launch carries cudaLaunchAttributeProgrammaticStreamSerialization)
__device__ __forceinline__ void griddep_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
// the image's ticket: release orders this thread's partial stores before it, acquire makes every earlier
// ticket holder's partials visible to the CTA that draws the last one (after a CTA barrier) -- one
// MEMBAR.ALL.GPU + CCTL instead of a seq-cst fence on each side
__device__ __forceinline__ unsigned ticket_acq_rel(unsigned *t) {
    unsigned v;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(v) : "l"(t) : "memory");
    return v;
}
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ void mbar_init(unsigned long long *bar, unsigned count) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_arrive(unsigned long long *bar) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile("{ .reg .b64 st; mbarrier.arrive.release.cta.shared::cta.b64 st, [%0]; }" ::"r"(a) : "memory");
}

__device__ __forceinline__ void mbar_wait(unsigned long long *bar, unsigned parity) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile(
        "{ .reg .pred p;\n"
        "WAIT_%=: mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=; }" ::"r"(a),
        "r"(parity)
        : "memory");
}

// 2*atanh(t) == log1p(x) for t = x / (2 + x).  Series to t^9 for |t| <= 0.2 (rel. error < 1e-8);
// MUFU-based logarithm of (1+t)/(1-t) otherwise (|result| >= 0.4, abs. error ~1e-7).
__device__ __forceinline__ float two_atanh(float t) {
    if (fabsf(t) <= 0.2f) {
        const float s = t * t;
        float p = fmaf(s, 1.0f / 9.0f, 1.0f / 7.0f);
        p = fmaf(s, p, 1.0f / 5.0f);
        p = fmaf(s, p, 1.0f / 3.0f);
        p = fmaf(s, p, 1.0f);
        return 2.0f * t * p;
    }
    return __logf((1.0f + t) * rcp_approx(1.0f - t));
}

// sum over filter pairs i of alpha_i * 2 atanh(t_i) into (e0, e1) (even, odd filters) when a warp's |t| exceeds
// the series range somewhere: two_atanh's two forms (series to t^9 for |t| <= 0.2, MUFU logarithm of
// (1+t)/(1-t) otherwise) evaluated in packed fp32 for both filters of a pair, selected per lane -- the same
// arithmetic without the divergent branch.  al / al2: alpha and 2 alpha of the n filters (shared memory).
template <int N>
__device__ __forceinline__ void two_atanh_pairs(const float *t, const float *al, const float *al2, float &e0,
                                                float &e1) {
    static_assert(N % 2 == 0, "filter pairs");
    float2 e = make_float2(e0, e1);
#pragma unroll
    for (int i = 0; i < N; i += 2) {
        const float2 t1 = make_float2(t[i], t[i + 1]);
        const float2 w = __fmul2_rn(*reinterpret_cast<const float2 *>(al2 + i), t1);
        const float2 sq = __fmul2_rn(t1, t1);
        float2 pp = __ffma2_rn(sq, make_float2(1.0f / 9.0f, 1.0f / 9.0f), make_float2(1.0f / 7.0f, 1.0f / 7.0f));
        pp = __ffma2_rn(sq, pp, make_float2(1.0f / 5.0f, 1.0f / 5.0f));
        pp = __ffma2_rn(sq, pp, make_float2(1.0f / 3.0f, 1.0f / 3.0f));
        pp = __ffma2_rn(sq, pp, make_float2(1.0f, 1.0f));
        const float2 vs = __fmul2_rn(w, pp);
        const float2 num = __fadd2_rn(make_float2(1.0f, 1.0f), t1);
        const float2 den = __fadd2_rn(make_float2(1.0f, 1.0f), make_float2(-t1.x, -t1.y));
        const float2 q = __fmul2_rn(num, make_float2(rcp_approx(den.x), rcp_approx(den.y)));
        const float2 a2 = *reinterpret_cast<const float2 *>(al + i);
        const float2 vl = __fmul2_rn(make_float2(__log2f(q.x), __log2f(q.y)),
                                     __fmul2_rn(a2, make_float2(0.69314718f, 0.69314718f)));
        e = __fadd2_rn(e, make_float2(fabsf(t1.x) <= 0.2f ? vs.x : vl.x, fabsf(t1.y) <= 0.2f ? vs.y : vl.y));
    }
    e0 = e.x;
    e1 = e.y;
}

// ------------------------------------------------------------------------------------------------
// tile geometry and shared-memory carve-up

struct TileGeom {
    int t;                 // global tile index (partials layout [tile][B][8])
    int s0, s1, c0, c1;    // owned rows / cols
    int ry0, rx0;          // region origin; staged cell (i,j) <-> (ry0-R+i, rx0-R+j)
    bool edge;             // touches the image edge (symmetric rule needs the psi ring zeroed)
};

template <int TH, int TW, int R, bool SYM>
__device__ __forceinline__ TileGeom tile_geom_t(const PassArgs &a, int tyl, int txi) {
    TileGeom g;
    const int tyi = a.ty0 + tyl;
    g.t = tyi * a.tiles_x + txi;
    g.s0 = tile_start(tyi, a.tiles_y, TH, a.H, R);
    g.s1 = tile_start(tyi + 1, a.tiles_y, TH, a.H, R);
    g.c0 = tile_start(txi, a.tiles_x, TW, a.W, R);
    g.c1 = tile_start(txi + 1, a.tiles_x, TW, a.W, R);
    g.ry0 = g.s0 - R;
    g.rx0 = g.c0 - R;
    g.edge = SYM && (g.s0 == 0 || g.c0 == 0 || g.s1 == a.H || g.c1 == a.W);
    return g;
}

template <int M, bool SYM>
__device__ __forceinline__ TileGeom tile_geom(const PassArgs &a, int tyl, int txi) {
    using C = PassCfg<M>;
    return tile_geom_t<C::TH, C::TW, C::R, SYM>(a, tyl, txi);
}

template <int M>
struct Smem {
    float *Un, *Du, *Psi, *taps, *alpha;
    __device__ Smem(float *sm, int nf, bool trial_planes) {
        using C = PassCfg<M>;
        Un = sm;
        Du = Un + C::PLANE;
        Psi = trial_planes ? Du + C::PLANE : Du;
        taps = Psi + C::NPSI * C::PLANE;
        alpha = taps + nf * C::TAPS;
    }
};

template <int M>
__host__ __device__ constexpr size_t smem_floats(int nf, bool trial) {
    using C = PassCfg<M>;
    return (size_t)(trial ? 2 : 1) * C::PLANE + (size_t)C::NPSI * C::PLANE + (size_t)nf * C::TAPS +
           (size_t)((nf + 3) & ~3);
}

template <int M>
__device__ void stage_bank(const PassArgs &a, const Smem<M> &S) {
    using C = PassCfg<M>;
    const int nf = a.n_filters;
    for (int k = threadIdx.x; k < nf * C::TAPS; k += C::NT) {
        const int f = k / C::TAPS, e = k - f * C::TAPS;
        S.taps[k] = e < M * M ? a.kf[f * M * M + e] : 0.0f;
    }
    for (int k = threadIdx.x; k < nf; k += C::NT) S.alpha[k] = a.alpha[k];
}

// psi_0 = 0 outside the image: the r ring of every psi plane is read only by outputs on the region
// border, which matter only where they are padded pixels folded back (symmetric rule, tiles on an
// image edge).  Elsewhere the ring feeds discarded outputs and stays unwritten.
template <int M>
__device__ void zero_psi_ring(const Smem<M> &S) {
    using C = PassCfg<M>;
    constexpr int R = C::R, CW = C::CW, SH = C::SH;
    if constexpr (R > 0) {
        constexpr int RING = SH * CW - C::RH * C::RW;
        for (int k = threadIdx.x; k < C::NPSI * RING; k += C::NT) {
            const int pl = k / RING, e = k - pl * RING;
            int i, j;
            if (e < R * CW) { i = e / CW; j = e - i * CW; }
            else if (e < 2 * R * CW) { const int e2 = e - R * CW; i = C::RH + R + e2 / CW; j = e2 % CW; }
            else { const int e3 = e - 2 * R * CW; i = R + e3 / (2 * R); const int jj = e3 % (2 * R); j = jj < R ? jj : C::RW + jj; }
            S.Psi[pl * C::PLANE + i * C::SW + j] = 0.0f;
        }
    }
}

// per-image trial parameters of one pass
struct TrialParams {
    int iu, iup, inew, ig, ignew, branch;
    double tau, t, inv1pt, gam;
};

__device__ __forceinline__ TrialParams trial_params(const PassArgs &a, const ImgCtl &c) {
    TrialParams p;
    p.iu = c.iu; p.iup = c.iup; p.inew = c.inew; p.ig = c.ig; p.ignew = c.ignew; p.branch = c.branch;
    p.tau = c.tau;  // set_step: step_num / L (solver.py:64-65), tau * lam, 1 / (1 + tau * lam)
    p.t = c.t;
    p.inv1pt = c.inv1pt;
    p.gam = a.gamma;
    return p;
}

// the trial point prox(u - tau g + gamma (u - u_prev)) (solver.py:146-149 with prox_quadratic / prox_idiv,
// solver.py:92-125) of one pixel, in fp64 like the reference and rounded once to the fp32 state: the
// state then tracks the reference's iterates to ~1/2 ulp per iteration (fp32 arithmetic here rounded
// several times per pixel and moved the iterates ~2x further, enough to flip a late decision)
__device__ __forceinline__ float trial_point(float u, float up, float g, float ob, const TrialParams &p) {
    const double ud = (double)u;
    const double ut = (ud - p.tau * (double)g) + p.gam * (ud - (double)up);
    if (p.branch == FOE_QUADRATIC) return (float)((ut + p.t * (double)ob) * p.inv1pt);
    return (float)prox_idv64(ut, p.t, (double)ob);
}

// ------------------------------------------------------------------------------------------------
// prologue: stage u (EVAL/INIT) or the trial point u_new and du (TRIAL) into Un/Du
//   global inputs are image-offset pointers to local buffers holding rows [lrow0, lrow0 + Hl)

template <int M, bool TRIAL, bool SYM>
__device__ void stage(const PassArgs &a, const TileGeom &g, const Smem<M> &S, const TrialParams &p, const float *uin,
                      const float *upv, const float *gin, const float *obs, float *uout, float shift,
                      double (&acc)[kNumPartials]) {
    using C = PassCfg<M>;
    constexpr int R = C::R, CW = C::CW, SW = C::SW, NT = C::NT, CPT = C::CPT, NCELL = C::NCELL;
    const int H = a.H, W = a.W, lrow0 = a.lrow0, tid = threadIdx.x;
    // load phase: every global read of this thread's cells in flight before any use
    float lu[CPT], lup[CPT], lg[CPT], lob[CPT];
#pragma unroll
    for (int q = 0; q < CPT; ++q) {
        const int k = tid + q * NT;
        if (k < NCELL) {
            const int i = k / CW, j = k - i * CW;
            const int sy = src_idx<SYM>(g.ry0 - R + i, H), sx = src_idx<SYM>(g.rx0 - R + j, W);
            const size_t o = (size_t)(sy - lrow0) * W + sx;
            lu[q] = __ldg(uin + o);
            if (TRIAL) { lup[q] = __ldg(upv + o); lg[q] = __ldg(gin + o); lob[q] = __ldg(obs + o); }
        }
    }
#pragma unroll
    for (int q = 0; q < CPT; ++q) {
        const int k = tid + q * NT;
        if (k >= NCELL) continue;
        const int i = k / CW, j = k - i * CW;
        if (!TRIAL) {
            S.Un[i * SW + j] = lu[q] - shift;
            continue;
        }
        const int gy = g.ry0 - R + i, gx = g.rx0 - R + j;
        const float u = lu[q], gg = lg[q], ob = lob[q];
        // u - tau g + gamma (u - u_prev)  (solver.py:146-149)
        const float un = trial_point(u, lup[q], gg, ob, p);
        const float du = un - u;
        S.Un[i * SW + j] = un - shift;
        S.Du[i * SW + j] = du;
        if (gy >= g.s0 && gy < g.s1 && gx >= g.c0 && gx < g.c1) {
            uout[(size_t)(gy - lrow0) * W + gx] = un;
            acc[1] += (double)du * (double)du;  // vdot(du, du)  solver.py:152
            acc[2] += (double)gg * (double)du;  // vdot(g, du)   solver.py:153
            acc[3] += (double)u * (double)u;    // |u|^2 for the stop test, solver.py:173
            if (p.branch == FOE_QUADRATIC) {
                const double d = (double)un - (double)ob;
                acc[4] += d * d;
            } else {
                acc[4] += (double)un;
                if (ob > 0.0f) {
                    if (un > 0.0f) acc[5] += (double)ob * (double)logf(un);
                    else acc[6] += 1.0;
                }
            }
        }
    }
}

// ------------------------------------------------------------------------------------------------
// filter loop: per filter forward responses, pointwise, adjoint; returns this thread's owned
// energy terms (fp64) and leaves the group's partial gradient in gacc.  `phase` carries the
// mbarrier parities of the NBUF slots across calls.

template <int M, bool TRIAL, bool SYM>
__device__ double filter_loop(const PassArgs &a, const TileGeom &g, const Smem<M> &S,
                              unsigned long long (*mbar)[PassCfg<M>::NBUF], unsigned &phase,
                              float (&gacc)[PassCfg<M>::MY][PassCfg<M>::MX]) {
    using C = PassCfg<M>;
    constexpr int R = C::R, SW = C::SW, MY = C::MY;
    constexpr int WIN = C::MX + 2 * R;  // window width per micro-tile row
    constexpr int WR = MY + 2 * R;      // window rows
    const int H = a.H, W = a.W, nf = a.n_filters, tid = threadIdx.x;
    const int grp = tid / C::NTG, lt = tid - grp * C::NTG;
    const int wg = lt >> 5, lane = lt & 31;
    const int tx = (wg & 1) * 8 + (lane & 7), ty = (wg >> 1) * 4 + (lane >> 3);
    const int fpg = (nf + C::G - 1) / C::G;
    const int fbeg = grp * fpg, fend = min(nf, fbeg + fpg);
    const int ly0 = ty * MY, lx0 = tx * C::MX;  // region-local origin of this thread's micro-tile

    // edge handling, hoisted out of the filter loop: which of this thread's pixels lie outside the
    // image (psi_0 must be 0 there, symmetric rule) and which it owns (energy terms)
    unsigned out_bits = 0u, own_bits = 0u;
#pragma unroll
    for (int o = 0; o < MY; ++o) {
        const int gy = g.ry0 + ly0 + o;
#pragma unroll
        for (int c = 0; c < C::MX; ++c) {
            const int gx = g.rx0 + lx0 + c;
            if (SYM && !(gy >= 0 && gy < H && gx >= 0 && gx < W)) out_bits |= 1u << (o * C::MX + c);
            if (gy >= g.s0 && gy < g.s1 && gx >= g.c0 && gx < g.c1) own_bits |= 1u << (o * C::MX + c);
        }
    }
    float epx[MY][C::MX];  // per-pixel energy terms summed over this group's filters (fp32)
#pragma unroll
    for (int o = 0; o < MY; ++o)
#pragma unroll
        for (int c = 0; c < C::MX; ++c) { epx[o][c] = 0.0f; gacc[o][c] = 0.0f; }

    const float *ubase = S.Un + ly0 * SW + lx0;
    const float *dbase = S.Du + ly0 * SW + lx0;

    // software-pipelined over this group's filters: forward(k) -> wait(k-1) -> adjoint(k-1) ->
    // arrive(k).  psi of round k lives in buffer k % NBUF.  A thread arrives on round k only after
    // its adjoint(k-1), so the buffer forward(k) overwrites -- last read by adjoint(k-3) -- is free
    // once the writer has passed wait(k-2): NBUF = 3 suffices, and a warp waits only if a peer is a
    // whole forward behind.
#pragma unroll 1
    for (int k = 0; k <= fpg; ++k) {
        if (k < fpg) {
            const int f = fbeg + k;
            const int kb = k % C::NBUF;
            if (f < fend) {
                float w[C::TAPS];
#pragma unroll
                for (int kk = 0; kk < C::TAPS; kk += 4) {
                    const float4 v = *reinterpret_cast<const float4 *>(S.taps + f * C::TAPS + kk);
                    w[kk] = v.x; w[kk + 1] = v.y; w[kk + 2] = v.z; w[kk + 3] = v.w;
                }
                const float al = S.alpha[f];
                float z[MY][C::MX], dz[MY][C::MX];
#pragma unroll
                for (int o = 0; o < MY; ++o)
#pragma unroll
                    for (int c = 0; c < C::MX; ++c) { z[o][c] = 0.0f; dz[o][c] = 0.0f; }
                // forward responses: z = K_f u_new (image.py:37-58), dz = K_f du
#pragma unroll
                for (int i = 0; i < WR; ++i) {
                    float ru[WIN], rd[WIN];
                    load_row<WIN>(ubase + i * SW, ru);
                    if (TRIAL) load_row<WIN>(dbase + i * SW, rd);
#pragma unroll
                    for (int o = 0; o < MY; ++o) {
                        const int aa = i - o;
                        if (aa < 0 || aa >= M) continue;
#pragma unroll
                        for (int bb = 0; bb < M; ++bb) {
                            const float wt = w[aa * M + bb];
#pragma unroll
                            for (int c = 0; c < C::MX; ++c) {
                                z[o][c] = fmaf(wt, ru[c + bb], z[o][c]);
                                if (TRIAL) dz[o][c] = fmaf(wt, rd[c + bb], dz[o][c]);
                            }
                        }
                    }
                }
                // pointwise: psi = a rho'(z) (prior.py:31-32); energy terms
                float *ps = S.Psi + (grp * C::NBUF + kb) * C::PLANE + (ly0 + R) * SW + lx0 + R;
                const float a2 = 2.0f * al;
                float tt[MY][C::MX];
                float tmax = 0.0f;
#pragma unroll
                for (int o = 0; o < MY; ++o) {
#pragma unroll
                    for (int c = 0; c < C::MX; ++c) {
                        const float zz = z[o][c];
                        const float q1 = fmaf(zz, zz, 1.0f);
                        ps[o * SW + c] = (a2 * zz) * rcp_approx(q1);
                        if (TRIAL) {
                            // F(u_new) - F(u) per response: log((1+z^2)/(1+z_o^2)) = 2 atanh(t) with
                            // t = (z^2 - z_o^2) / ((1+z^2) + (1+z_o^2)), z_o = z - dz
                            const float d = dz[o][c];
                            const float zo = zz - d;
                            const float num = d * fmaf(2.0f, zo, d);
                            const float den = fmaf(zo, zo, q1) + 1.0f;
                            tt[o][c] = num * rcp_approx(den);
                            tmax = fmaxf(tmax, fabsf(tt[o][c]));
                        }
                    }
                }
                if (SYM && out_bits) {  // psi_0 = 0 outside the image (only threads on an image edge)
#pragma unroll
                    for (int o = 0; o < MY; ++o)
#pragma unroll
                        for (int c = 0; c < C::MX; ++c)
                            if (out_bits >> (o * C::MX + c) & 1u) ps[o * SW + c] = 0.0f;
                }
                if (TRIAL) {
                    if (__any_sync(0xffffffffu, tmax > 0.2f)) {
#pragma unroll
                        for (int o = 0; o < MY; ++o)
#pragma unroll
                            for (int c = 0; c < C::MX; ++c) epx[o][c] = fmaf(al, two_atanh(tt[o][c]), epx[o][c]);
                    } else {
#pragma unroll
                        for (int o = 0; o < MY; ++o)
#pragma unroll
                            for (int c = 0; c < C::MX; ++c) {
                                const float t1 = tt[o][c], sq = t1 * t1;
                                float pp = fmaf(sq, 1.0f / 9.0f, 1.0f / 7.0f);
                                pp = fmaf(sq, pp, 1.0f / 5.0f);
                                pp = fmaf(sq, pp, 1.0f / 3.0f);
                                pp = fmaf(sq, pp, 1.0f);
                                epx[o][c] = fmaf(a2 * t1, pp, epx[o][c]);
                            }
                    }
                } else {
#pragma unroll
                    for (int o = 0; o < MY; ++o)
#pragma unroll
                        for (int c = 0; c < C::MX; ++c) epx[o][c] = fmaf(al, log1pf(z[o][c] * z[o][c]), epx[o][c]);
                }
            }
        }
        if (k > 0) {
            const int f = fbeg + k - 1;
            const int kb = (k - 1) % C::NBUF;
            mbar_wait(&mbar[grp][kb], (phase >> kb) & 1u);
            phase ^= 1u << kb;
            if (f < fend) {
                float w[C::TAPS];
#pragma unroll
                for (int kk = 0; kk < C::TAPS; kk += 4) {
                    const float4 v = *reinterpret_cast<const float4 *>(S.taps + f * C::TAPS + kk);
                    w[kk] = v.x; w[kk + 1] = v.y; w[kk + 2] = v.z; w[kk + 3] = v.w;
                }
                const float *pb = S.Psi + (grp * C::NBUF + kb) * C::PLANE + ly0 * SW + lx0;
                // adjoint: gacc += K_f^T psi_f  (correlation with the unflipped kernel, image.py:76-79)
#pragma unroll
                for (int i = 0; i < WR; ++i) {
                    float rp[WIN];
                    load_row<WIN>(pb + i * SW, rp);
#pragma unroll
                    for (int o = 0; o < MY; ++o) {
                        const int aa = i - o;
                        if (aa < 0 || aa >= M) continue;
#pragma unroll
                        for (int bb = 0; bb < M; ++bb) {
                            const float wt = w[(M - 1 - aa) * M + (M - 1 - bb)];
#pragma unroll
                            for (int c = 0; c < C::MX; ++c) gacc[o][c] = fmaf(wt, rp[c + bb], gacc[o][c]);
                        }
                    }
                }
            }
        }
        if (k < fpg) {  // one arrival per warp once its lanes' psi stores are ordered (__syncwarp)
            __syncwarp();
            if ((threadIdx.x & 31) == 0) mbar_arrive(&mbar[grp][k % C::NBUF]);
        }
    }
    double e = 0.0;  // owned pixels only, fp64 across pixels
#pragma unroll
    for (int o = 0; o < MY; ++o)
#pragma unroll
        for (int c = 0; c < C::MX; ++c)
            if (own_bits >> (o * C::MX + c) & 1u) e += (double)epx[o][c];
    return e;
}

// combine the group partial gradients, fold padded pixels onto their mirror sources (P^T,
// image.py:76-83) and write the owned gradient
template <int M, bool SYM>
__device__ void fold_and_write(const PassArgs &a, const TileGeom &g, const Smem<M> &S,
                               const float (&gacc)[PassCfg<M>::MY][PassCfg<M>::MX], float *gout) {
    using C = PassCfg<M>;
    constexpr int R = C::R, NT = C::NT, MY = C::MY;
    const int tid = threadIdx.x, H = a.H, W = a.W;
    const int grp = tid / C::NTG, lt = tid - grp * C::NTG;
    const int wg = lt >> 5, lane = lt & 31;
    const int tx = (wg & 1) * 8 + (lane & 7), ty = (wg >> 1) * 4 + (lane >> 3);
    const int ly0 = ty * MY, lx0 = tx * C::MX;
    __syncthreads();  // all groups done with their psi planes
    float *gb = S.Psi;  // G planes of RH x RW
#pragma unroll
    for (int o = 0; o < MY; ++o)
        *reinterpret_cast<float4 *>(gb + grp * C::RH * C::RW + (ly0 + o) * C::RW + lx0) =
            make_float4(gacc[o][0], gacc[o][1], gacc[o][2], gacc[o][3]);
    __syncthreads();
    auto gsum = [&](int ly, int lx) {
        float s = gb[ly * C::RW + lx];
#pragma unroll
        for (int g2 = 1; g2 < C::G; ++g2) s += gb[g2 * C::RH * C::RW + ly * C::RW + lx];
        return s;
    };
    // 2-D ownership walk: column = tid % RW, rows strided by NT / RW (no integer division)
    const int xx = tid % C::RW;
    const int gx = g.c0 + xx;
    if (gx < g.c1) {
        const int lx = gx - g.rx0;
        int mx = -1;
        if (SYM && R > 0) {
            if (gx < R) mx = (-1 - gx) - g.rx0;
            else if (gx >= W - R) mx = (2 * W - 1 - gx) - g.rx0;
        }
        for (int gy = g.s0 + tid / C::RW; gy < g.s1; gy += NT / C::RW) {
            const int ly = gy - g.ry0;
            float val = gsum(ly, lx);
            if (SYM && R > 0) {
                int my = -1;
                if (gy < R) my = (-1 - gy) - g.ry0;
                else if (gy >= H - R) my = (2 * H - 1 - gy) - g.ry0;
                if (my >= 0) val += gsum(my, lx);
                if (mx >= 0) val += gsum(ly, mx);
                if (my >= 0 && mx >= 0) val += gsum(my, mx);
            }
            gout[(size_t)(gy - a.lrow0) * W + gx] = val;
        }
    }
}

// ------------------------------------------------------------------------------------------------
// k_pass: one trial (or eval/init) pass per launch

template <int M, bool TRIAL, bool SYM>
__global__ void __launch_bounds__(PassCfg<M>::NT, 1) k_pass(const PassArgs a) {
    using C = PassCfg<M>;
    constexpr int NT = C::NT;
    extern __shared__ __align__(16) float sm[];
    __shared__ double red[NT / 32][kNumPartials];
    __shared__ double s_sum[kNumPartials];
    __shared__ int s_last;
    __shared__ ImgCtl s_ctl;  // the control block as read at the pass's start (the decision's input)
    __shared__ unsigned long long s_mbar[C::G][C::NBUF];

    const int tid = threadIdx.x;
    const int b = blockIdx.y;
    const size_t cta = (size_t)blockIdx.y * gridDim.x + blockIdx.x;
    if (a.dbg_times && tid == 0) a.dbg_times[cta * 3] = globaltimer_ns();
    // programmatic dependent launch: the next pass may be scheduled once every CTA of this one has
    // started; the bank staging below depends only on the launch arguments
    griddep_launch_dependents();
    const int tyl = blockIdx.x / a.tiles_x, txi = blockIdx.x - tyl * a.tiles_x;
    const TileGeom g = tile_geom<M, SYM>(a, tyl, txi);
    const Smem<M> S(sm, a.n_filters, TRIAL);
    stage_bank<M>(a, S);
    if (tid < C::G * C::NBUF) mbar_init(&s_mbar[tid / C::NBUF][tid % C::NBUF], C::NTG / 32);
    if (g.edge) zero_psi_ring<M>(S);
    griddep_wait();  // the previous pass (control block, iterates, gradients, partials) is complete
    TrialParams p{};
    if (a.mode != MODE_EVAL) {
        const ImgCtl c = a.ctl[b];
        if (c.done && !a.no_decide) return;
        p = trial_params(a, c);
        if (tid == 0) s_ctl = c;
    }
    // local buffers hold global rows [lrow0, lrow0 + Hl) of each image (the whole image unless this
    // launch is one row band of a decomposed image)
    const size_t ioff = (size_t)b * a.Hl * a.W;
    const float *uin, *upv = nullptr, *gin = nullptr, *obs = nullptr;
    float *gout, *uout = nullptr;
    if (a.mode == MODE_EVAL) {
        uin = a.u_in + ioff;
        gout = a.g_out + ioff;
    } else {
        uin = a.U + p.iu * a.plane + ioff;
        if (TRIAL) {
            upv = a.U + p.iup * a.plane + ioff;
            gin = a.Gs + p.ig * a.plane + ioff;
            obs = a.obs + ioff;
            uout = a.U + p.inew * a.plane + ioff;
            gout = a.Gs + p.ignew * a.plane + ioff;
        } else {
            gout = a.Gs + p.ig * a.plane + ioff;
        }
    }
    // Filters are zero-mean (DCT basis without DC, image.py:117-130), so K(u - c) == K u: staging
    // u - c with c = the tile's anchor pixel keeps the fp32 products small (accuracy, not speed).
    const float shift = a.zero_mean ? __ldg(uin + (size_t)(g.s0 - a.lrow0) * a.W + g.c0) : 0.0f;
    double acc[kNumPartials];
#pragma unroll
    for (int k = 0; k < kNumPartials; ++k) acc[k] = 0.0;
    stage<M, TRIAL, SYM>(a, g, S, p, uin, upv, gin, obs, uout, shift, acc);
    __syncthreads();  // staged tile, taps and mbarrier init visible

    float gacc[C::MY][C::MX];
    unsigned phase = 0u;
    acc[0] = filter_loop<M, TRIAL, SYM>(a, g, S, s_mbar, phase, gacc);
    fold_and_write<M, SYM>(a, g, S, gacc, gout);

    if (a.dbg_times && tid == 0) a.dbg_times[cta * 3 + 1] = globaltimer_ns();
    // per-tile partials, last CTA of the image reduces and decides
    block_reduce<NT>(acc, red, s_sum);
    if (tid < kNumPartials) a.partials[((size_t)g.t * a.B + b) * kPartialStride + tid] = s_sum[tid];
    if (a.band) return;  // band mode: partials are all-gathered and decided by k_decide
    const int nlaunch = a.tiles_x * a.tiles_y;
    __syncthreads();
    // thread 0's acq_rel ticket releases the CTA's partial stores (ordered before it by the barrier;
    // release is cumulative) and, in the last CTA, acquires every earlier CTA's
    if (tid == 0) s_last = (ticket_acq_rel(a.tickets + b) == (unsigned)(nlaunch - 1));
    __syncthreads();
    if (a.dbg_times && tid == 0) a.dbg_times[cta * 3 + 2] = globaltimer_ns();
    if (!s_last) return;
    reduce_tiles<NT>(a.partials, a.tiles_x * a.tiles_y, a.B, b, red, s_sum);
    if (tid == 0) {
        a.tickets[b] = 0u;
        if (a.energy_out) a.energy_out[b] = s_sum[0];  // EVAL, and a solve's final-energy pass
        if (a.mode != MODE_EVAL && !a.no_decide) {
            ImgCtl c = s_ctl;  // = a.ctl[b]: read at this pass's start, written only by this decision
            decide_ctl(a, b, s_sum, c, true, a.mode);
            a.ctl[b] = c;
        }
    }
}
