// foe_pass.cuh -- the fused FoE pass kernel (included by foe_b200.cu).
//
// One CTA = one tile of one image.  Region = owned tile + r ring (the pixels whose responses the
// adjoint needs); staged cells = region + another r ring (the inputs of those responses).
//
// Thread layout: 3 filter groups x 6 warps.  A warp covers 8 micro-columns x 4 micro-rows of
// 3x4-pixel micro-tiles, so each 8-lane LDS.128 phase reads 32 consecutive floats of one smem row
// (bank-conflict free for any pitch).  Each group owns every 3rd filter slice of the bank and
// double-buffered psi planes, so groups synchronise only among themselves (named barriers).
//
// Per filter and thread: forward z = K u_new and dz = K du on 12 pixels from a 5x8 (r=2) window
// streamed from smem (600 FFMA), pointwise psi = 2a z/(1+z^2) and the energy change
// a*log1p(dz(2z_o+dz)/(1+z_o^2)) evaluated as 2a*atanh(t), t = (z^2-z_o^2)/((1+z^2)+(1+z_o^2)),
// then the adjoint K^T psi (300 FFMA).

template <int M_>
struct PassCfg {
    static constexpr int M = M_;
    static constexpr int R = M / 2;
    static constexpr int RH = 36, RW = 64;  // region (owned tile + r ring)
    static constexpr int MY = 3, MX = 4;    // micro-tile per thread
    static constexpr int G = 3;             // filter groups per CTA
    static constexpr int NBUF = 4;          // psi buffers per group (pipelined mbarrier ring)
    static constexpr int NTX = RW / MX, NTY = RH / MY, NTG = NTX * NTY, NT = G * NTG;
    static constexpr int WARPS_G = NTG / 32;
    static constexpr int CW = RW + 2 * R;       // staged columns
    static constexpr int SH = RH + 2 * R;       // staged rows
    static constexpr int SW = (CW + 3) & ~3;    // row pitch (float4 aligned)
    static constexpr int PLANE = SH * SW;
    static constexpr int NPSI = G * NBUF;       // psi planes
    static constexpr int TH = RH - 2 * R, TW = RW - 2 * R;  // max owned tile
    static constexpr int TAPS = (M * M + 3) & ~3;           // per-filter tap stride (float4)
    static_assert(NTX == 16 && NTY == 12, "warp layout assumes 16 x 12 micro-tiles per group");
    static_assert(TH >= 2 * R, "tile too small for the fold rule");
    static_assert(G * RH * RW <= NPSI * PLANE, "group partial-gradient buffer must fit the psi planes");
};

__device__ __forceinline__ float rcp_approx(float x) {  // MUFU.RCP, no denormal fix-up
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

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

template <int M, bool TRIAL, bool SYM>
__global__ void __launch_bounds__(PassCfg<M>::NT, 1) k_pass(const PassArgs a) {
    using C = PassCfg<M>;
    constexpr int R = C::R, SW = C::SW, CW = C::CW, SH = C::SH, MY = C::MY, NT = C::NT;
    constexpr int WIN = C::MX + 2 * R;  // window width per micro-tile row
    constexpr int WR = MY + 2 * R;      // window rows

    extern __shared__ __align__(16) float sm[];
    __shared__ double red[NT / 32][kNumPartials];
    __shared__ double s_sum[kNumPartials];
    __shared__ int s_last;
    __shared__ unsigned long long s_mbar[C::G][C::NBUF];

    const int tid = threadIdx.x;
    const int b = blockIdx.y;
    const int H = a.H, W = a.W, nf = a.n_filters;

    int iu = 0, iup = 0, inew = 0, ig = 0, ignew = 0, branch = 0;
    float tau32 = 0.f, t32 = 0.f, gam32 = 0.f;
    if (a.mode != MODE_EVAL) {
        const ImgCtl &c = a.ctl[b];
        if (c.done && !a.no_decide) return;
        iu = c.iu; iup = c.iup; inew = c.inew; ig = c.ig; ignew = c.ignew; branch = c.branch;
        if (TRIAL) {
            const double tau = a.step_num / c.L;  // SolverConfig.step_size, solver.py:64-65
            tau32 = (float)tau;
            t32 = (float)(tau * c.lam);
            gam32 = (float)a.gamma;
        }
    }
    // local buffers hold global rows [lrow0, lrow0 + Hl) of each image (the whole image unless this
    // launch is one row band of a decomposed image)
    const int lrow0 = a.lrow0;
    const size_t ioff = (size_t)b * a.Hl * W;
    const float *uin, *upv = nullptr, *gin = nullptr, *obs = nullptr;
    float *gout, *uout = nullptr;
    if (a.mode == MODE_EVAL) {
        uin = a.u_in + ioff;
        gout = a.g_out + ioff;
    } else {
        uin = a.U + iu * a.plane + ioff;
        if (TRIAL) {
            upv = a.U + iup * a.plane + ioff;
            gin = a.Gs + ig * a.plane + ioff;
            obs = a.obs + ioff;
            uout = a.U + inew * a.plane + ioff;
            gout = a.Gs + ignew * a.plane + ioff;
        } else {
            gout = a.Gs + ig * a.plane + ioff;
        }
    }

    const int tyl = blockIdx.x / a.tiles_x, txi = blockIdx.x - tyl * a.tiles_x;
    const int tyi = a.ty0 + tyl;              // global tile row
    const int t = tyi * a.tiles_x + txi;      // global tile index (partials layout [tile][B][8])
    const int s0 = tile_start(tyi, a.tiles_y, C::TH, H, R), s1 = tile_start(tyi + 1, a.tiles_y, C::TH, H, R);
    const int c0 = tile_start(txi, a.tiles_x, C::TW, W, R), c1 = tile_start(txi + 1, a.tiles_x, C::TW, W, R);
    const int ry0 = s0 - R, rx0 = c0 - R;  // region origin; staged cell (i,j) <-> (ry0-R+i, rx0-R+j)

    float *Un = sm;
    float *Du = Un + C::PLANE;
    float *Psi = TRIAL ? Du + C::PLANE : Du;
    float *s_taps = Psi + C::NPSI * C::PLANE;
    float *s_alpha = s_taps + nf * C::TAPS;

    for (int k = tid; k < nf * C::TAPS; k += NT) {
        const int f = k / C::TAPS, e = k - f * C::TAPS;
        s_taps[k] = e < M * M ? a.kf[f * M * M + e] : 0.0f;
    }
    for (int k = tid; k < nf; k += NT) s_alpha[k] = a.alpha[k];
    if (tid < C::G * C::NBUF) mbar_init(&s_mbar[tid / C::NBUF][tid % C::NBUF], C::NTG);
    // psi_0 = 0 outside the image: the r ring of every psi plane is read only by outputs on the
    // region border, which matter only where they are padded pixels folded back (symmetric rule,
    // tiles on an image edge).  Elsewhere the ring feeds discarded outputs and stays unwritten.
    const bool edge_tile = SYM && (s0 == 0 || c0 == 0 || s1 == H || c1 == W);
    if constexpr (R > 0) {
        if (edge_tile) {
            constexpr int RING = SH * CW - C::RH * C::RW;
            for (int k = tid; k < C::NPSI * RING; k += NT) {
                const int pl = k / RING, e = k - pl * RING;
                int i, j;
                if (e < R * CW) { i = e / CW; j = e - i * CW; }
                else if (e < 2 * R * CW) { const int e2 = e - R * CW; i = C::RH + R + e2 / CW; j = e2 % CW; }
                else { const int e3 = e - 2 * R * CW; i = R + e3 / (2 * R); const int jj = e3 % (2 * R); j = jj < R ? jj : C::RW + jj; }
                Psi[pl * C::PLANE + i * SW + j] = 0.0f;
            }
        }
    }


    // Filters are zero-mean (DCT basis without DC, image.py:117-130), so K(u - c) == K u: staging
    // u - c with c = the tile's anchor pixel keeps the fp32 products small (accuracy, not speed).
    const float shift = a.zero_mean ? __ldg(uin + (size_t)(s0 - lrow0) * W + c0) : 0.0f;

    // ---- prologue: stage u (EVAL/INIT) or the trial point u_new and du (TRIAL) -------------------
    double acc[kNumPartials];
#pragma unroll
    for (int k = 0; k < kNumPartials; ++k) acc[k] = 0.0;
    constexpr int NCELL = SH * CW;
    constexpr int CPT = (NCELL + NT - 1) / NT;  // staged cells per thread
    if (TRIAL) {
        // all global loads of this thread's cells first (4 x CPT in flight), then the arithmetic
        float lu[CPT], lup[CPT], lg[CPT], lob[CPT];
#pragma unroll
        for (int q = 0; q < CPT; ++q) {
            const int k = tid + q * NT;
            if (k < NCELL) {
                const int i = k / CW, j = k - i * CW;
                const size_t o = (size_t)(src_idx<SYM>(ry0 - R + i, H) - lrow0) * W + src_idx<SYM>(rx0 - R + j, W);
                lu[q] = __ldg(uin + o); lup[q] = __ldg(upv + o); lg[q] = __ldg(gin + o); lob[q] = __ldg(obs + o);
            }
        }
#pragma unroll
        for (int q = 0; q < CPT; ++q) {
            const int k = tid + q * NT;
            if (k < NCELL) {
                const int i = k / CW, j = k - i * CW;
                const int gy = ry0 - R + i, gx = rx0 - R + j;
                const float u = lu[q], g = lg[q], ob = lob[q];
                // u - tau g + gamma (u - u_prev)  (solver.py:146-149)
                const float ut = (u - tau32 * g) + gam32 * (u - lup[q]);
                const float un = (branch == FOE_QUADRATIC) ? prox_quad(ut, t32, ob) : prox_idv(ut, t32, ob);
                const float du = un - u;
                Un[i * SW + j] = un - shift;
                Du[i * SW + j] = du;
                if (gy >= s0 && gy < s1 && gx >= c0 && gx < c1) {
                    uout[(size_t)(gy - lrow0) * W + gx] = un;
                    acc[1] += (double)du * (double)du;  // vdot(du, du)  solver.py:152
                    acc[2] += (double)g * (double)du;   // vdot(g, du)   solver.py:153
                    acc[3] += (double)u * (double)u;    // |u|^2 for the stop test, solver.py:173
                    if (branch == FOE_QUADRATIC) {
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
    } else {
        float lu[CPT];
#pragma unroll
        for (int q = 0; q < CPT; ++q) {
            const int k = tid + q * NT;
            if (k < NCELL) {
                const int i = k / CW, j = k - i * CW;
                lu[q] = __ldg(uin + (size_t)(src_idx<SYM>(ry0 - R + i, H) - lrow0) * W + src_idx<SYM>(rx0 - R + j, W));
            }
        }
#pragma unroll
        for (int q = 0; q < CPT; ++q) {
            const int k = tid + q * NT;
            if (k < NCELL) {
                const int i = k / CW, j = k - i * CW;
                Un[i * SW + j] = lu[q] - shift;
            }
        }
    }
    __syncthreads();  // staged tile, taps and mbarrier init visible

    // ---- filter loop -----------------------------------------------------------------------------
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
        const int gy = ry0 + ly0 + o;
#pragma unroll
        for (int c = 0; c < C::MX; ++c) {
            const int gx = rx0 + lx0 + c;
            if (SYM && !(gy >= 0 && gy < H && gx >= 0 && gx < W)) out_bits |= 1u << (o * C::MX + c);
            if (gy >= s0 && gy < s1 && gx >= c0 && gx < c1) own_bits |= 1u << (o * C::MX + c);
        }
    }
    float epx[MY][C::MX];  // per-pixel energy terms summed over this group's filters (fp32)
#pragma unroll
    for (int o = 0; o < MY; ++o)
#pragma unroll
        for (int c = 0; c < C::MX; ++c) epx[o][c] = 0.0f;

    float gacc[MY][C::MX];
#pragma unroll
    for (int o = 0; o < MY; ++o)
#pragma unroll
        for (int c = 0; c < C::MX; ++c) gacc[o][c] = 0.0f;

    const float *ubase = Un + ly0 * SW + lx0;
    const float *dbase = Du + ly0 * SW + lx0;

    // software-pipelined over this group's filters: forward(k) -> arrive(k) -> wait(k-1) ->
    // adjoint(k-1).  psi of round k lives in buffer k % NBUF; a warp waits only if a peer has not
    // finished the previous round's forward.  NBUF = 4 keeps the buffer written by forward(k)
    // clear of readers: its last reader, adjoint(k-4), precedes every thread's arrive(k-2), and a
    // thread at forward(k) has already waited on round k-2.
#pragma unroll 1
    for (int k = 0; k <= fpg; ++k) {
        if (k < fpg) {
            const int f = fbeg + k;
            const int kb = k % C::NBUF;
            if (f < fend) {
                float w[C::TAPS];
#pragma unroll
                for (int kk = 0; kk < C::TAPS; kk += 4) {
                    const float4 v = *reinterpret_cast<const float4 *>(s_taps + f * C::TAPS + kk);
                    w[kk] = v.x; w[kk + 1] = v.y; w[kk + 2] = v.z; w[kk + 3] = v.w;
                }
                const float al = s_alpha[f];
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
                float *ps = Psi + (grp * C::NBUF + kb) * C::PLANE + (ly0 + R) * SW + lx0 + R;
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
            mbar_arrive(&s_mbar[grp][kb]);
        }
        if (k > 0) {
            const int f = fbeg + k - 1;
            const int kb = (k - 1) % C::NBUF;
            mbar_wait(&s_mbar[grp][kb], ((k - 1) / C::NBUF) & 1);
            if (f < fend) {
                float w[C::TAPS];
#pragma unroll
                for (int kk = 0; kk < C::TAPS; kk += 4) {
                    const float4 v = *reinterpret_cast<const float4 *>(s_taps + f * C::TAPS + kk);
                    w[kk] = v.x; w[kk + 1] = v.y; w[kk + 2] = v.z; w[kk + 3] = v.w;
                }
                const float *pb = Psi + (grp * C::NBUF + kb) * C::PLANE + ly0 * SW + lx0;
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
    }
    {
        double e = 0.0;  // owned pixels only, fp64 across pixels
#pragma unroll
        for (int o = 0; o < MY; ++o)
#pragma unroll
            for (int c = 0; c < C::MX; ++c)
                if (own_bits >> (o * C::MX + c) & 1u) e += (double)epx[o][c];
        acc[0] = e;
    }
    __syncthreads();

    // ---- combine filter groups, fold padded pixels (P^T, image.py:88-90), write ------------------
    float *gb = Psi;  // G planes of RH x RW
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
    static_assert(NT % C::RW == 0, "fold walk assumes whole region rows per pass");
    {
        const int xx = tid % C::RW;
        const int gx = c0 + xx;
        if (gx < c1) {
            const int lx = gx - rx0;
            int mx = -1;
            if (SYM && R > 0) {
                if (gx < R) mx = (-1 - gx) - rx0;
                else if (gx >= W - R) mx = (2 * W - 1 - gx) - rx0;
            }
            for (int gy = s0 + tid / C::RW; gy < s1; gy += NT / C::RW) {
                const int ly = gy - ry0;
                float val = gsum(ly, lx);
                if (SYM && R > 0) {
                    int my = -1;
                    if (gy < R) my = (-1 - gy) - ry0;
                    else if (gy >= H - R) my = (2 * H - 1 - gy) - ry0;
                    if (my >= 0) val += gsum(my, lx);
                    if (mx >= 0) val += gsum(ly, mx);
                    if (my >= 0 && mx >= 0) val += gsum(my, mx);
                }
                gout[(size_t)(gy - lrow0) * W + gx] = val;
            }
        }
    }

    // ---- per-tile partials, last CTA of the image reduces and decides ----------------------------
    block_reduce<NT>(acc, red, s_sum);
    if (tid < kNumPartials) {
        a.partials[((size_t)t * a.B + b) * kPartialStride + tid] = s_sum[tid];
        __threadfence();
    }
    if (a.band) return;  // band mode: partials are all-gathered and decided by k_decide
    const int nlaunch = a.tiles_x * a.tiles_y;
    __syncthreads();
    if (tid == 0) s_last = (atomicAdd(a.tickets + b, 1u) == (unsigned)(nlaunch - 1));
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    reduce_tiles<NT>(a.partials, a.tiles_x * a.tiles_y, a.B, b, red, s_sum);
    if (tid == 0) {
        a.tickets[b] = 0u;
        if (a.mode == MODE_EVAL) {
            a.energy_out[b] = s_sum[0];
        } else if (!a.no_decide) {
            decide(a, b, s_sum);
        }
    }
}
