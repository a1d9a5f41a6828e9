// foe_pass_tc7.cuh -- tensor-core (tcgen05, 3xTF32) variant of the fused FoE pass for 7x7 banks with up
// to 48 filters (the BASELINE 48 x 7 x 7 fallback bank; the paper's filter-bank size).  Included by
// foe_b200.cu after foe_pass_tc.cuh; the default for such banks (FOE_TC7=0 forces the FFMA pass).
//
// 40 x 64 regions (34 x 58 owned; the FFMA k_pass<7> uses 48 rows), prologue, fold and reductions as
// k_pass_tc; per 128-pixel block (two region rows, 20 blocks per tile):
//   forward   Z  = A_u  . Kf^T     K = 48 taps (6 K = 8 steps) + one tap-48 step, N = 48 filters
//             dZ = A_du . Kf^T
//   adjoint   Y  = Psi . Kt^T      K = 48 filters, N = 64 (49 taps)
//   g(q) = sum_a H_a(q + (a - 3, 0)),  H_a(p) = sum_b Y(p + (0, b - 3))[7 a + b]
// The 49-tap shifted sum runs in two stages (7 horizontal partial sums per pixel into a ring, then 7
// vertical): a ring of 49-tap Y rows over the 5 blocks one output block touches would not fit in shared
// memory.
//
// TMEM (512 columns): one A stage (u hi / lo, du hi / lo: 4 x 48 = 192 columns) and two D regions of
// 160 (z 48 -> Psi hi, dz 48 -> Psi lo, Y 64).  The tap-48 operand group {u hi, u lo, du hi, du lo, 0, 0,
// 0, 0} of block j is parked in columns 152..159 of its D region -- Y's unused tail, written by the
// adjoint only after the forward has read the group.
//
// Roles (24 warps): operand warps 0-7 (im2col of block j once forward(j-1) has read the A stage, the
// tap-48 group once the D region is drained, warp 0 issues forward(j)); two point sets of 8 warps (set s
// <-> D region s <-> blocks j = s mod 2; 4 lane quarters x 2 filter halves of 24, two chunks of 12):
// psi' / energy terms -> adjoint(j) -> Y(j) drained to a shared-memory block buffer (frees the D region)
// -> H(j) into the ring -> vertical sums of block j-2 (needs H(j-4 .. j); the odd ones are the other
// set's, flagged by mbarriers).

struct TcCfg7 {
    static constexpr int R = 3, M = 7, KT = 49, NFX = 48;
    // 40 x 64 regions (34 x 58 owned): a 512^2 image is 16 x 9 = 144 tiles, one wave on 148 SMs (the FFMA
    // pass's 48-row regions give 117); the host tile grid follows the 7x7 kernel in use (region_rows)
    static constexpr int RH = 40, RW = 64, SH = RH + 2 * R, CW = RW + 2 * R, SW = (CW + 3) & ~3, PLANE = SH * SW;
    static constexpr int NCELL = SH * CW, TH = RH - 2 * R, TW = RW - 2 * R;
    static constexpr int NBLK = RH * RW / 128;  // 20
    static constexpr int W_PT = 8, NWARPS = 24, NT = NWARPS * 32;
    // TMEM columns
    static constexpr int C_AUH = 0, C_AUL = 48, C_ADH = 96, C_ADL = 144;  // A stage
    static constexpr int C_D0 = 192, C_DREG = 160, C_DZ = 0, C_DDZ = 48, C_DY = 96, C_G48 = 152;
    // B operands (floats): Kf [hi | lo] (N = 48, K = 48), tap-48 selectors 4 x (N = 48, K = 8), Kt [hi | lo]
    // (N = 64, K = 48)
    static constexpr int BKF = 48 * 48, BK48 = 48 * 8, BKT = 64 * 48;
    static constexpr int YBW = RW + 6;                 // Y block buffer row (3 zero columns each side)
    static constexpr int YB = KT * 2 * YBW;            // one block's Y: [tap][row][YBW]
    static constexpr int HSLOTS = 8, HROWS = 2 * HSLOTS;  // H ring: [a][ring row][RW] (power of two: masks)
    // named barriers
    static constexpr int BAR_AFREE = 1, BAR_AFULL = 2, BAR_DFREE = 3, BAR_DFULL = 5, BAR_PFULL = 7, BAR_YFULL = 9,
                         BAR_SET = 11;
    static_assert(RW == 64 && NBLK * 128 == RH * RW, "blocks of two 64-pixel region rows");
    static_assert(C_D0 + 2 * C_DREG == 512, "TMEM plan");
};

__host__ __device__ constexpr size_t tc7_smem_floats() {
    using T = TcCfg7;
    // staged cells (float4), Kf hi/lo, tap-48 selectors, Kt hi/lo, two Y block buffers, H ring, region
    // gradient (two a-halves), alpha / 2 alpha (64 each)
    return 4 * (size_t)T::PLANE + 2 * T::BKF + 4 * T::BK48 + 2 * T::BKT + 2 * (size_t)T::YB +
           7 * (size_t)T::HROWS * T::RW + 2 * (size_t)T::RH * T::RW + 128;
}

// im2col of one pixel's tap rounds (bit r: taps 4r .. 4r+3, r < 12) from the staged cells into the A stage
template <unsigned ROUNDS, bool TRIAL, class T>
__device__ __forceinline__ void tc7_im2col(const float4 *sp, uint32_t st) {
#pragma unroll
    for (int rd = 0; rd < 12; ++rd) {
        if (!((ROUNDS >> rd) & 1u)) continue;
        const int c0 = 4 * rd;
        float uh[4], ul[4], dh[4], dl[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int t = c0 + i;
            const float4 c = sp[(t / T::M) * T::SW + (t % T::M)];
            uh[i] = c.x; ul[i] = c.y; dh[i] = c.z; dl[i] = c.w;
        }
        tmem_st4(st + T::C_AUH + c0, uh);
        tmem_st4(st + T::C_AUL + c0, ul);
        if (TRIAL) {
            tmem_st4(st + T::C_ADH + c0, dh);
            tmem_st4(st + T::C_ADL + c0, dl);
        }
    }
}

template <bool TRIAL, bool SYM>
__global__ void __launch_bounds__(TcCfg7::NT, 1) k_pass_tc7(const PassArgs a) {
    using T = TcCfg7;
    using C = TcCfg7;
    constexpr int NT = T::NT, R = T::R, SW = T::SW, NBLK = T::NBLK;
    extern __shared__ __align__(128) float sm[];
    __shared__ double red[NT / 32][kNumPartials];
    __shared__ double s_sum[kNumPartials];
    __shared__ int s_last;
    __shared__ uint32_t s_tmem;
    __shared__ ImgCtl s_ctl;  // the control block as read at the pass's start (the decision's input)
    __shared__ __align__(8) unsigned long long mb_dfull[2], mb_yfull[2];
    __shared__ __align__(8) unsigned long long mb_hfull[NBLK], mb_vdone[NBLK];

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int b = blockIdx.y;
    const int nf = a.n_filters;
#if FOE_STAMPS
    unsigned long long *ph = (a.dbg_times && blockIdx.x == gridDim.x / 2 && blockIdx.y == 0 && lane == 0)
                                 ? a.dbg_times + 3 * (size_t)gridDim.x * gridDim.y : nullptr;
#else
    constexpr unsigned long long *ph = nullptr;
#endif
    griddep_launch_dependents();
    const int tyl = blockIdx.x / a.tiles_x, txi = blockIdx.x - tyl * a.tiles_x;
    const TileGeom g = tile_geom_t<T::TH, T::TW, T::R, SYM>(a, tyl, txi);

    float4 *S4 = reinterpret_cast<float4 *>(sm);
    float *Kf = sm + 4 * T::PLANE;       // [hi | lo]
    float *K48 = Kf + 2 * T::BKF;        // 4 tap-48 selectors
    float *Kt = K48 + 4 * T::BK48;       // [hi | lo]
    float *Yb = Kt + 2 * T::BKT;         // [set][tap][row][YBW]
    float *Hr = Yb + 2 * T::YB;          // [a][ring row][RW]
    float *Gr = Hr + 7 * T::HROWS * T::RW;  // [a-half][RH][RW]
    float *s_al = Gr + 2 * T::RH * T::RW;
    float *s_al2 = s_al + 64;

    if (warp == 0) tmem_alloc(&s_tmem, 512);
    if (tid == 0) {
        for (int s = 0; s < 2; ++s) {
            mbar_init(&mb_dfull[s], 1);
            mbar_init(&mb_yfull[s], 1);
        }
        for (int j = 0; j < NBLK; ++j) {
            mbar_init(&mb_hfull[j], 8);  // one arrival per warp of the set that wrote H(j)
            mbar_init(&mb_vdone[j], 8);  // one arrival per warp of the set that summed block j
        }
    }
    // B operands: Kf[f][t] = kf_f[t] (K = taps 0..47), Kt[t][f] = 2 a_f k_f[t] with k_f[t] = kf_f[48 - t]
    // (N = 64 taps, zero beyond 48), tf32 hi + lo (both rounded to nearest)
    for (int e = tid; e < 48 * 48; e += NT) {
        const int n = e / 48, k = e % 48;
        const float vf = (n < nf) ? a.kf[n * T::KT + k] : 0.0f;
        const float hf = tf32_rn(vf);
        Kf[bsw_offset<48>(n, k)] = hf;
        Kf[T::BKF + bsw_offset<48>(n, k)] = tf32_rn(vf - hf);
    }
    for (int e = tid; e < 64 * 48; e += NT) {
        const int n = e / 48, k = e % 48;
        const float vt = (k < nf && n < T::KT) ? 2.0f * a.alpha[k] * a.kf[k * T::KT + (T::KT - 1 - n)] : 0.0f;
        const float ht = tf32_rn(vt);
        Kt[bsw_offset<64>(n, k)] = ht;
        Kt[T::BKT + bsw_offset<64>(n, k)] = tf32_rn(vt - ht);
    }
    // tap-48 selectors (K rows: u hi, u lo, du hi, du lo, 0 ...): [0] rows 0, 1 = k48 hi; [1] row 0 = k48 lo;
    // [2] / [3] the same on rows 2, 3 (dz)
    for (int e = tid; e < 4 * T::BK48; e += NT) {
        const int mtx = e / T::BK48, rem = e % T::BK48, n = rem / 8, k = rem % 8;
        const float v48 = n < nf ? a.kf[n * T::KT + 48] : 0.0f, h48 = tf32_rn(v48);
        const int row = (mtx >> 1) ? k - 2 : k;
        float val = 0.0f;
        if (row == 0) val = (mtx & 1) ? tf32_rn(v48 - h48) : h48;
        else if (row == 1 && !(mtx & 1)) val = h48;
        K48[mtx * T::BK48 + bsw_offset<48>(n, k)] = val;
    }
    for (int e = tid; e < 64; e += NT) {
        s_al[e] = e < nf ? a.alpha[e] : 0.0f;
        s_al2[e] = e < nf ? 2.0f * a.alpha[e] : 0.0f;
    }
    for (int e = tid; e < 2 * T::KT * 2 * 6; e += NT) {  // zero columns of both Y block buffers
        const int col = e % 6, rr = e / 6;
        Yb[rr * T::YBW + (col < 3 ? col : T::YBW - 6 + col)] = 0.0f;
    }
    griddep_wait();

    // ---- prologue (as k_pass_tc, R = 3) ----
    constexpr int CPT = (C::NCELL + NT - 1) / NT;
    const size_t ioff = (size_t)b * a.Hl * a.W;
    TrialParams p{};
    if (a.mode != MODE_EVAL) {
        const ImgCtl c = a.ctl[b];
        if (c.done && !a.no_decide) {
            __syncthreads();
            if (warp == 0) tmem_dealloc(s_tmem, 512);
            return;
        }
        p = trial_params(a, c);
        if (tid == 0) s_ctl = c;
    }
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
    const float shift = a.zero_mean ? __ldg(uin + (size_t)(g.s0 - a.lrow0) * a.W + g.c0) : 0.0f;
    double acc[kNumPartials];
#pragma unroll
    for (int k = 0; k < kNumPartials; ++k) acc[k] = 0.0;
    {
        float lu[CPT], lup[CPT], lg[CPT], lob[CPT];
#pragma unroll
        for (int q = 0; q < CPT; ++q) {
            const int k = tid + q * NT;
            if (k < C::NCELL) {
                const int i = k / C::CW, j = k - i * C::CW;
                const size_t o = (size_t)(src_idx<SYM>(g.ry0 - R + i, a.H) - a.lrow0) * a.W +
                                 src_idx<SYM>(g.rx0 - R + j, a.W);
                lu[q] = __ldg(uin + o);
                if (TRIAL) {
                    lup[q] = __ldg(upv + o);
                    lg[q] = __ldg(gin + o);
                    lob[q] = __ldg(obs + o);
                }
            }
        }
#pragma unroll
        for (int q = 0; q < CPT; ++q) {
            const int k = tid + q * NT;
            if (k >= C::NCELL) continue;
            const int i = k / C::CW, j = k - i * C::CW;
            if (!TRIAL) {
                const float x = lu[q] - shift, h = tf32_rn(x);
                S4[i * SW + j] = make_float4(h, tf32_rn_operand(x - h), 0.0f, 0.0f);
                continue;
            }
            const int gy = g.ry0 - R + i, gx = g.rx0 - R + j;
            const float u = lu[q], gg = lg[q], ob = lob[q];
            const float un = trial_point(u, lup[q], gg, ob, p);  // solver.py:146-149
            const float du = un - u;
            const float x = un - shift, h = tf32_rn(x), hd = tf32_rn(du);
            S4[i * SW + j] = make_float4(h, tf32_rn_operand(x - h), hd, tf32_rn_operand(du - hd));
            if (gy >= g.s0 && gy < g.s1 && gx >= g.c0 && gx < g.c1) {
                uout[(size_t)(gy - a.lrow0) * a.W + gx] = un;
                acc[1] += (double)du * (double)du;
                acc[2] += (double)gg * (double)du;
                acc[3] += (double)u * (double)u;
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
    // the prologue's partials 1..6 summed per warp through shared memory (the H ring and region gradient are
    // not live yet; CTA-wide fp64 shuffle trees cost ~1.5k cycles of SHFL issue)
    static_assert((NT / 32) * (kNumPartials - 1) * 32 <= (7 * T::HROWS * T::RW + 2 * T::RH * T::RW) / 2, "scratch");
    warp_partials_smem<1, kNumPartials, 32>(acc, red, reinterpret_cast<double *>(Hr));
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    constexpr uint32_t tmem = 0u;
    if (tid == 0 && s_tmem != 0u) __trap();
    if (ph && tid == 0) ph[NBLK * 16] = clock64();  // loop start

    if (warp < T::W_PT) {
        // ================= operand warps =================
        const int pl = tid & 127, v = warp >> 2;
        const uint32_t lane_off = (uint32_t)(32 * (warp & 3)) << 16;
        BDescs<48, 6> kfd;
        kfd.build(smem_u32(Kf), smem_u32(Kf + T::BKF));
        uint64_t k48d[4];
#pragma unroll
        for (int m = 0; m < 4; ++m) k48d[m] = umma_desc_kmajor(smem_u32(K48 + T::BK48 * m), (48 / 8) * 128, 128);
        for (int j = 0; j < NBLK; ++j) {
            const int s = j & 1;
            // A stage: forward(j-1) has read it (warp 0 polls, the OP barrier relays)
            if (warp == 0 && j >= 1) mbar_wait_sleep(&mb_dfull[(j - 1) & 1], ((j - 1) >> 1) & 1);
            named_sync(T::BAR_AFREE, 256);
            tc_fence_after();
            if (ph && warp == 0) ph[j * 16 + 5] = clock64();
            const int lr = 2 * j + (pl >> 6), lc = pl & 63;
            const float4 *sp = S4 + lr * SW + lc;
            // taps 0..47: warps 0-3 rounds 0..5, warps 4-7 rounds 6..11
            if (v == 0)
                tc7_im2col<0x03fu, TRIAL, T>(sp, tmem + lane_off);
            else
                tc7_im2col<0xfc0u, TRIAL, T>(sp, tmem + lane_off);
            // the tap-48 group goes into D region s once Y(j-2) left it (the set arrives on DFREE + s)
            if (j >= 2) named_sync(T::BAR_DFREE + s, 512);
            if (v == 1) {
                const float4 c = sp[(48 / T::M) * T::SW + (48 % T::M)];
                const float g48[8] = {c.x, c.y, c.z, c.w, 0.0f, 0.0f, 0.0f, 0.0f};
                tmem_st8(tmem + lane_off + T::C_D0 + s * T::C_DREG + T::C_G48, g48);
            }
            tc_wait_st();
            tc_fence_before();
            if (warp != 0) {
                named_arrive(T::BAR_AFULL, 256);
            } else {
                named_sync(T::BAR_AFULL, 256);
                tc_fence_after();
                if (elect_one()) {
                    constexpr uint32_t idesc = idesc_tf32(128, 48);
                    const uint32_t sd = tmem + T::C_D0 + s * T::C_DREG, g48 = sd + T::C_G48;
                    umma_3xtf32_pre<48, 6>(sd + T::C_DZ, tmem + T::C_AUH, tmem + T::C_AUL, kfd, 6);
                    umma_tf32_ts(sd + T::C_DZ, g48, k48d[0], idesc, 1u);
                    umma_tf32_ts(sd + T::C_DZ, g48, k48d[1], idesc, 1u);
                    if (TRIAL) {
                        umma_3xtf32_pre<48, 6>(sd + T::C_DDZ, tmem + T::C_ADH, tmem + T::C_ADL, kfd, 6);
                        umma_tf32_ts(sd + T::C_DDZ, g48, k48d[2], idesc, 1u);
                        umma_tf32_ts(sd + T::C_DDZ, g48, k48d[3], idesc, 1u);
                    }
                    umma_commit(&mb_dfull[s]);
                }
                __syncwarp();
                if (ph) ph[j * 16 + 0] = clock64();
            }
        }
    } else {
        // ================= point sets =================
        const int q4 = warp & 3, hf = ((warp - T::W_PT) >> 2) & 1;
        const int set = (warp - T::W_PT) >> 3;
        const int ws = (warp - T::W_PT) & 7;  // warp within the set
        const bool issuer = ws == 0;
        BDescs<64, 6> ktd;
        ktd.build(smem_u32(Kt), smem_u32(Kt + T::BKT));
        const int pl = 32 * q4 + lane;
        const uint32_t lane_off = (uint32_t)(32 * q4) << 16;
        const uint32_t sd = tmem + T::C_D0 + set * T::C_DREG + lane_off;
        float *yb = Yb + set * T::YB;
        double e_own = 0.0;
        const bool inner = !SYM || (g.ry0 >= 0 && g.ry0 + T::RH <= a.H && g.rx0 >= 0 && g.rx0 + T::RW <= a.W);
        for (int j = set; j < NBLK + 2; j += 2) {
            const bool comp = j < NBLK;
            if (comp) {
                if (issuer) {
                    mbar_wait_sleep(&mb_dfull[set], (j >> 1) & 1);
                    named_arrive(T::BAR_DFULL + set, 256);
                } else {
                    named_sync(T::BAR_DFULL + set, 256);
                }
                tc_fence_after();
                if (ph && ws == 0) ph[j * 16 + 1] = clock64();
                const int lr = 2 * j + (pl >> 6), lc = pl & 63;
                const int gy = g.ry0 + lr, gx = g.rx0 + lc;
                const bool in_img = !SYM || (gy >= 0 && gy < a.H && gx >= 0 && gx < a.W);
                const bool owned = gy >= g.s0 && gy < g.s1 && gx >= g.c0 && gx < g.c1;
                const bool keep_all = inner || __all_sync(0xffffffffu, in_img);
                float e0 = 0.0f, e1 = 0.0f;
#pragma unroll 1
                for (int ch = 0; ch < 2; ++ch) {  // this warp's 24 filters in two chunks of 12
                    const int f0 = 24 * hf + 12 * ch;
                    float z[12], dz[12];
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        tmem_ld4(sd + T::C_DZ + f0 + 4 * c, *reinterpret_cast<float(*)[4]>(&z[4 * c]));
                        if (TRIAL) tmem_ld4(sd + T::C_DDZ + f0 + 4 * c, *reinterpret_cast<float(*)[4]>(&dz[4 * c]));
                    }
                    tc_wait_ld();
                    float tmax = 0.0f;
                    if (TRIAL) {  // filter pairs in packed fp32 (FFMA2 / FMUL2 / FADD2), as k_pass_tc
#pragma unroll
                        for (int i = 0; i < 12; i += 2) {
                            const float2 zz = make_float2(z[i], z[i + 1]), d = make_float2(dz[i], dz[i + 1]);
                            const float2 zo = __fadd2_rn(zz, make_float2(-d.x, -d.y));
                            const float2 a1 = __ffma2_rn(zz, zz, make_float2(1.0f, 1.0f));
                            const float2 b1 = __fadd2_rn(__ffma2_rn(zo, zo, a1), make_float2(1.0f, 1.0f));
                            const float2 ps = __fmul2_rn(zz, make_float2(rcp_approx(a1.x), rcp_approx(a1.y)));
                            const float2 tt = __fmul2_rn(__fmul2_rn(d, __fadd2_rn(zz, zo)),
                                                         make_float2(rcp_approx(b1.x), rcp_approx(b1.y)));
                            dz[i] = tt.x;
                            dz[i + 1] = tt.y;
                            tmax = fmaxf(tmax, fmaxf(fabsf(tt.x), fabsf(tt.y)));
                            z[i] = (keep_all || in_img) ? ps.x : 0.0f;
                            z[i + 1] = (keep_all || in_img) ? ps.y : 0.0f;
                        }
                    } else {
#pragma unroll
                        for (int i = 0; i < 12; ++i) {
                            const float zz = z[i];
                            const float ps = zz * rcp_approx(fmaf(zz, zz, 1.0f));
                            dz[i] = zz;
                            z[i] = (keep_all || in_img) ? ps : 0.0f;
                        }
                    }
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        float hi[4], lo[4];
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            hi[i] = tf32_rn(z[4 * c + i]);
                            lo[i] = tf32_rn_operand(z[4 * c + i] - hi[i]);
                        }
                        tmem_st4(sd + T::C_DZ + f0 + 4 * c, hi);
                        tmem_st4(sd + T::C_DDZ + f0 + 4 * c, lo);
                    }
                    if (TRIAL) {
                        const float wmax = __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(tmax)));
                        // series cut per warp as in k_pass_tc (first omitted term below 2^-25 relative)
                        auto series = [&](auto deg) {  // filter pairs packed: (e0, e1) = (even, odd)
                            constexpr int D = decltype(deg)::value;
                            float2 e = make_float2(e0, e1);
#pragma unroll
                            for (int i = 0; i < 12; i += 2) {
                                const float2 t1 = make_float2(dz[i], dz[i + 1]);
                                const float2 w = __fmul2_rn(*reinterpret_cast<const float2 *>(s_al2 + f0 + i), t1);
                                if (D == 1) {
                                    e = __fadd2_rn(e, w);
                                    continue;
                                }
                                const float2 sq = __fmul2_rn(t1, t1);
                                float2 pp;
                                if (D == 9) {
                                    pp = __ffma2_rn(sq, make_float2(1.0f / 9.0f, 1.0f / 9.0f), make_float2(1.0f / 7.0f, 1.0f / 7.0f));
                                    pp = __ffma2_rn(sq, pp, make_float2(1.0f / 5.0f, 1.0f / 5.0f));
                                    pp = __ffma2_rn(sq, pp, make_float2(1.0f / 3.0f, 1.0f / 3.0f));
                                } else if (D == 7) {
                                    pp = __ffma2_rn(sq, make_float2(1.0f / 7.0f, 1.0f / 7.0f), make_float2(1.0f / 5.0f, 1.0f / 5.0f));
                                    pp = __ffma2_rn(sq, pp, make_float2(1.0f / 3.0f, 1.0f / 3.0f));
                                } else if (D == 5) {
                                    pp = __ffma2_rn(sq, make_float2(1.0f / 5.0f, 1.0f / 5.0f), make_float2(1.0f / 3.0f, 1.0f / 3.0f));
                                } else {
                                    pp = make_float2(1.0f / 3.0f, 1.0f / 3.0f);
                                }
                                pp = __ffma2_rn(sq, pp, make_float2(1.0f, 1.0f));
                                e = __ffma2_rn(w, pp, e);
                            }
                            e0 = e.x;
                            e1 = e.y;
                        };
                        if (wmax > 0.2f) {  // lanes mix series-range and larger |t|: both forms, per-lane select
                            two_atanh_pairs<12>(dz, s_al + f0, s_al2 + f0, e0, e1);
                        } else if (wmax > 0.12f) {
                            series(std::integral_constant<int, 9>{});
                        } else if (wmax > 0.04f) {
                            series(std::integral_constant<int, 7>{});
                        } else if (wmax > 0.015f) {
                            series(std::integral_constant<int, 5>{});
                        } else if (wmax > 2.5e-4f) {
                            series(std::integral_constant<int, 3>{});
                        } else {
                            series(std::integral_constant<int, 1>{});
                        }
                    } else {
#pragma unroll
                        for (int i = 0; i < 12; ++i) {
                            const float term = s_al[f0 + i] * log1pf(dz[i] * dz[i]);
                            if (i & 1) e1 += term; else e0 += term;
                        }
                    }
                }
                if (owned) e_own += (double)(e0 + e1);
                tc_wait_st();
                tc_fence_before();
                if (!issuer) {
                    named_arrive(T::BAR_PFULL + set, 256);
                } else {
                    named_sync(T::BAR_PFULL + set, 256);
                    tc_fence_after();
                    if (elect_one()) {
                        const uint32_t sb = tmem + T::C_D0 + set * T::C_DREG;
                        umma_3xtf32_pre<64, 6>(sb + T::C_DY, sb + T::C_DZ, sb + T::C_DDZ, ktd, 6);
                        umma_commit(&mb_yfull[set]);
                    }
                    __syncwarp();
                    if (ph) ph[j * 16 + 2] = clock64();
                }
                // Y(j) -> block buffer (frees the D region for block j + 2)
                if (issuer) {
                    mbar_wait_sleep(&mb_yfull[set], (j >> 1) & 1);
                    named_arrive(T::BAR_YFULL + set, 256);
                } else {
                    named_sync(T::BAR_YFULL + set, 256);
                }
                tc_fence_after();
                {
                    float y[32];
                    tmem_ld32(sd + T::C_DY + 32 * hf, y);
                    tc_wait_ld();
                    tc_fence_before();
                    if (j + 2 < NBLK) named_arrive(T::BAR_DFREE + set, 512);
                    const int rr = pl >> 6, cc = pl & 63;
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        const int t = 32 * hf + i;
                        if (t < T::KT) yb[(t * 2 + rr) * T::YBW + 3 + cc] = y[i];
                    }
                }
                named_sync(T::BAR_SET + set, 256);  // the whole block's Y is in the buffer
                if (ph && ws == 0) ph[j * 16 + 3] = clock64();
                // H(j): thread (pixel, a-half) -> H_a for a in {0..3} / {4..6}; ring slot j % HSLOTS held
                // H(j - 8), last read by the vertical sums of blocks j - 10 .. j - 6 (j - 7 the other set's)
                if (j >= 7) mbar_wait_sleep(&mb_vdone[j - 7], 0);
                {
                    const int p2 = ws * 32 + lane;  // 0..255
                    const int px = p2 & 127, ah = p2 >> 7;
                    const int rr = px >> 6, cc = px & 63;
                    const int hrow = (2 * j + rr) & (T::HROWS - 1);
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const int aa = 4 * ah + k;
                        if (aa >= 7) continue;
                        const float *yrow = yb + ((7 * aa) * 2 + rr) * T::YBW + cc;
                        float h0 = 0.0f, h1 = 0.0f;
#pragma unroll
                        for (int bb = 0; bb < 7; ++bb) {
                            const float vv = yrow[bb * 2 * T::YBW + bb];
                            if (bb & 1) h1 += vv; else h0 += vv;
                        }
                        Hr[(aa * T::HROWS + hrow) * T::RW + cc] = h0 + h1;
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&mb_hfull[j]);
                if (ph && ws == 0) ph[j * 16 + 4] = clock64();
            }
            // vertical sums of block q = j - 2 (rows 2q, 2q+1) once H(q-2 .. q+2) are in the ring
            const int q = j - 2;
            if (q >= 0) {
                for (int n = q - 2; n <= q + 2; ++n)
                    if (n >= 0 && n < NBLK) mbar_wait_sleep(&mb_hfull[n], 0);
                const int p2 = ws * 32 + lane;
                const int px = p2 & 127, ah = p2 >> 7;
                const int r = 2 * q + (px >> 6), c = px & 63;
                float s0 = 0.0f, s1 = 0.0f;
                auto vsum = [&](auto edge) {
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const int aa = 4 * ah + k;
                        if (aa >= 7) continue;
                        const int rr = r + aa - R;
                        if (decltype(edge)::value && (rr < 0 || rr >= T::RH)) continue;
                        const float vv = Hr[(aa * T::HROWS + (rr & (T::HROWS - 1))) * T::RW + c];
                        if (k & 1) s1 += vv; else s0 += vv;
                    }
                };
                if (q < 2 || q >= NBLK - 2)
                    vsum(std::true_type{});
                else
                    vsum(std::false_type{});
                Gr[ah * T::RH * T::RW + r * T::RW + c] = s0 + s1;
                __syncwarp();
                if (lane == 0) mbar_arrive(&mb_vdone[q]);
                if (ph && ws == 0) ph[q * 16 + 6] = clock64();
            }
        }
        acc[0] = e_own;
    }
    tc_fence_before();
    __syncthreads();
    warp_partials_smem<0, 1, 32>(acc, red, reinterpret_cast<double *>(Hr));  // H ring no longer live
    block_combine<NT>(red, s_sum);
    const int nlaunch = a.tiles_x * a.tiles_y;
    int ticket = 0;
    if (tid == 0) {
        double *pp = a.partials + ((size_t)g.t * a.B + b) * kPartialStride;
#pragma unroll
        for (int k = 0; k < kNumPartials; ++k) pp[k] = s_sum[k];
        if (!a.band) ticket = (int)ticket_acq_rel(a.tickets + b);
    }
    // ---- fold padded pixels (symmetric rule) and write the owned gradient ----
    for (int k = tid; k < T::RW * 8; k += NT) {
        const int xx = k % T::RW, rows0 = k / T::RW;
        const int gx = g.c0 + xx;
        if (gx >= g.c1) continue;
        const int lx = gx - g.rx0;
        int mx = -1;
        if (SYM) {
            if (gx < R) mx = (-1 - gx) - g.rx0;
            else if (gx >= a.W - R) mx = (2 * a.W - 1 - gx) - g.rx0;
        }
        for (int gy = g.s0 + rows0; gy < g.s1; gy += 8) {
            const int ly = gy - g.ry0;
            auto gr = [&](int yy, int xx2) { return Gr[yy * T::RW + xx2] + Gr[T::RH * T::RW + yy * T::RW + xx2]; };
            float val = gr(ly, lx);
            if (SYM) {
                int my = -1;
                if (gy < R) my = (-1 - gy) - g.ry0;
                else if (gy >= a.H - R) my = (2 * a.H - 1 - gy) - g.ry0;
                if (my >= 0) val += gr(my, lx);
                if (mx >= 0) val += gr(ly, mx);
                if (my >= 0 && mx >= 0) val += gr(my, mx);
            }
            gout[(size_t)(gy - a.lrow0) * a.W + gx] = val;
        }
    }
    if (a.band) {
        __syncthreads();
        if (warp == 0) tmem_dealloc(tmem, 512);
        return;
    }
    if (tid == 0) s_last = ticket == nlaunch - 1;
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 512);
    if (!s_last) return;
    // (no fence: thread 0's acquiring ticket and the barrier above order the loads below)
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
