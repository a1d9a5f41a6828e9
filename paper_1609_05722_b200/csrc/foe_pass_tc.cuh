// foe_pass_tc.cuh -- tensor-core (tcgen05, 3xTF32) variant of the fused FoE pass for 5x5 banks
// with at most 32 filters (included by foe_b200.cu after foe_pass.cuh / foe_tc.cuh).
//
// Same tile geometry, prologue, fold and reductions as k_pass; the two convolutions become
// implicit GEMMs on the tensor cores, one 128-pixel block (two region rows) at a time:
//   forward   Z  = A_u  . Kf^T    A_u[p][t] = u_new(p + off_t)  (im2col, K = 25 -> 32), N = filters
//             dZ = A_du . Kf^T    (the same for du, for the energy change)
//   adjoint   Y  = Psi  . Kt^T    Psi[p][f] = z/(1+z^2), Kt[t][f] = 2 a_f k_f[t], N = taps
//             g(q) = sum_t Y(q + off_t)[t]       (25-term shifted sum on the CUDA cores)
// A operands are written by their pixel's thread straight into TMEM (tcgen05.st), B operands sit in
// shared memory, D accumulators in TMEM.  fp32 accuracy from tf32 units via the 3xTF32 split.
// Two warpgroups alternate blocks so one builds operands / evaluates the pointwise terms while the
// other's MMAs run.

template <int NF_MAX>
struct TcCfg {
    using P = PassCfg<5>;
    static constexpr int R = 2, M = 5, KT = 25;
    static constexpr int RH = P::RH, RW = P::RW, SH = P::SH, SW = P::SW, PLANE = P::PLANE;
    static constexpr int NBLK = RH * RW / 128;       // 128-pixel blocks (two region rows each)
    static constexpr int NWG = 2, WGT = 256, NT = WGT * NWG;  // 2 warpgroups of 8 warps: warps w and w+4
                                                              // share a TMEM lane quarter (same pixels)
    static constexpr int YROWS = 12, YW = RW + 4;    // Y ring: 6 blocks of 2 rows, 2 zero columns each side
    static constexpr int BSZ = 32 * 32;              // one 32 x 32 B operand (floats)
    // TMEM columns per warpgroup: A_u hi/lo, A_du hi/lo (reused for Psi hi/lo), D_z (reused for
    // D_y), D_dz
    static constexpr int C_AUH = 0, C_AUL = 32, C_ADH = 64, C_ADL = 96, C_DZ = 128, C_DDZ = 160, C_WG = 256;
    static_assert(RW == 64 && NBLK * 128 == RH * RW, "blocks of two 64-pixel region rows");
    static_assert(NF_MAX <= 32, "one N = 32 MMA covers the bank");
};

template <int NF_MAX>
__host__ __device__ constexpr size_t tc_smem_floats() {
    using T = TcCfg<NF_MAX>;
    // Un, Du staged planes; Kf hi/lo, Kt hi/lo; Y ring; region gradient
    return 2 * (size_t)T::PLANE + 4 * (size_t)T::BSZ + (size_t)T::KT * T::YROWS * T::YW + 2 * (size_t)T::RH * T::RW;
}

template <int NF, bool TRIAL, bool SYM>
__global__ void __launch_bounds__(TcCfg<32>::NT, 1) k_pass_tc(const PassArgs a) {
    static_assert(NF % 8 == 0 && NF <= 32, "filter count rounded up to a multiple of 8");
    using T = TcCfg<32>;
    using C = PassCfg<5>;
    constexpr int NT = T::NT, R = T::R, SW = T::SW;
    extern __shared__ __align__(128) float sm[];
    __shared__ double red[NT / 32][kNumPartials];
    __shared__ double s_sum[kNumPartials];
    __shared__ int s_last;
    __shared__ uint32_t s_tmem;
    __shared__ __align__(8) unsigned long long s_mma[T::NWG];       // MMA completion, per warpgroup
    __shared__ __align__(8) unsigned long long s_ready[T::NBLK];    // Y of block j in the ring

    const int tid = threadIdx.x, warp = tid >> 5;
    const int wg = tid / T::WGT, wt = tid % T::WGT;  // warpgroup, thread in warpgroup
    const int hf = wt >> 7, pl = wt & 127;           // half (filters / taps), pixel = TMEM lane
    const int b = blockIdx.y;
    const size_t cta = (size_t)blockIdx.y * gridDim.x + blockIdx.x;
    if (a.dbg_times && tid == 0) a.dbg_times[cta * 3] = globaltimer_ns();
    const int nf = a.n_filters;
    TrialParams p{};
    if (a.mode != MODE_EVAL) {
        const ImgCtl &c = a.ctl[b];
        if (c.done && !a.no_decide) return;
        p = trial_params(a, c);
    }
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
    const int tyl = blockIdx.x / a.tiles_x, txi = blockIdx.x - tyl * a.tiles_x;
    const TileGeom g = tile_geom<5, SYM>(a, tyl, txi);

    float *Un = sm;
    float *Du = Un + T::PLANE;
    float *Kf = Du + T::PLANE;     // [hi | lo], forward B (N = filters, K = taps)
    float *Kt = Kf + 2 * T::BSZ;   // [hi | lo], adjoint B (N = taps, K = filters)
    float *Yr = Kt + 2 * T::BSZ;   // Y ring [tap][ring row][YW]
    float *Gr = Yr + T::KT * T::YROWS * T::YW;  // region gradient (before the fold)
    float *s_al = Gr + 2 * T::RH * T::RW;        // alpha_f, zero-padded to NF (Gr: two tap halves)
    float *s_k24 = s_al + 32;                    // tap 24 of each filter (outside the K = 24 MMAs)

    if (warp == 0) tmem_alloc(&s_tmem, 512);
    if (tid < T::NWG) mbar_init(&s_mma[tid], 1);
    if (tid < T::NBLK) mbar_init(&s_ready[tid], T::WGT);
    // B operands: Kf[f][t] = kf_f[t] (convolution orientation), Kt[t][f] = 2 a_f k_f[t] with the
    // unflipped k_f[t] = kf_f[24 - t]; zero padding to 32 x 32; split into tf32 hi + fp32 lo
    for (int e = tid; e < 32 * 32; e += NT) {
        const int n = e >> 5, k = e & 31;
        const float vf = (n < nf && k < T::KT) ? a.kf[n * T::KT + k] : 0.0f;
        const float vt = (k < nf && n < T::KT) ? 2.0f * a.alpha[k] * a.kf[k * T::KT + (T::KT - 1 - n)] : 0.0f;
        const float hf = tf32_hi(vf), ht = tf32_hi(vt);
        Kf[bsw_offset<32>(n, k)] = hf;
        Kf[T::BSZ + bsw_offset<32>(n, k)] = vf - hf;
        Kt[bsw_offset<32>(n, k)] = ht;
        Kt[T::BSZ + bsw_offset<32>(n, k)] = vt - ht;
    }
    for (int e = tid; e < NF; e += NT) {
        s_al[e] = e < nf ? a.alpha[e] : 0.0f;
        s_k24[e] = e < nf ? a.kf[e * T::KT + 24] : 0.0f;
    }
    // zero columns of the Y ring (padded positions outside the region)
    for (int e = tid; e < T::KT * T::YROWS * 4; e += NT) {
        const int col = e & 3, rr = e >> 2;
        Yr[rr * T::YW + (col < 2 ? col : T::YW - 4 + col)] = 0.0f;
    }
    const float shift = a.zero_mean ? __ldg(uin + (size_t)(g.s0 - a.lrow0) * a.W + g.c0) : 0.0f;
    double acc[kNumPartials];
#pragma unroll
    for (int k = 0; k < kNumPartials; ++k) acc[k] = 0.0;
    // prologue: stage u_new - shift and du for the region + r ring; all loads of a thread in flight
    // before any use (cells strided by NT)
    {
        constexpr int CPT = (C::NCELL + NT - 1) / NT;
        float lu[CPT], lup[CPT], lg[CPT], lob[CPT];
#pragma unroll
        for (int q = 0; q < CPT; ++q) {
            const int k = tid + q * NT;
            if (k < C::NCELL) {
                const int i = k / C::CW, j = k - i * C::CW;
                const size_t o = (size_t)(src_idx<SYM>(g.ry0 - R + i, a.H) - a.lrow0) * a.W +
                                 src_idx<SYM>(g.rx0 - R + j, a.W);
                lu[q] = __ldg(uin + o);
                if (TRIAL) { lup[q] = __ldg(upv + o); lg[q] = __ldg(gin + o); lob[q] = __ldg(obs + o); }
            }
        }
#pragma unroll
        for (int q = 0; q < CPT; ++q) {
            const int k = tid + q * NT;
            if (k >= C::NCELL) continue;
            const int i = k / C::CW, j = k - i * C::CW;
            if (!TRIAL) {
                Un[i * SW + j] = lu[q] - shift;
                continue;
            }
            const int gy = g.ry0 - R + i, gx = g.rx0 - R + j;
            const float u = lu[q], gg = lg[q], ob = lob[q];
            const float ut = (u - p.tau * gg) + p.gam * (u - lup[q]);  // solver.py:146-149
            const float un = (p.branch == FOE_QUADRATIC) ? prox_quad(ut, p.t, ob) : prox_idv(ut, p.t, ob);
            const float du = un - u;
            Un[i * SW + j] = un - shift;
            Du[i * SW + j] = du;
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
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (a.dbg_times && tid == 0) a.dbg_times[cta * 3 + 1] = globaltimer_ns();

    const uint32_t tbase = s_tmem + (uint32_t)(wg * T::C_WG);
    const uint32_t lane_off = (uint32_t)(32 * (warp & 3)) << 16;
    const uint32_t kf_hi = smem_u32(Kf), kf_lo = smem_u32(Kf + T::BSZ);
    const uint32_t kt_hi = smem_u32(Kt), kt_lo = smem_u32(Kt + T::BSZ);
    unsigned mma_phase = 0u;
    double e_own = 0.0;
    constexpr int FH = NF > 16 ? 16 : NF;  // filters per half (half 1 idles for NF <= 16)

    // g(q) over one half of the taps: half 0 taps [0, 13), half 1 taps [13, 25)
    auto shifted_sum = [&](int gb) {
        const int r = 2 * gb + (pl >> 6), c = pl & 63;
        float s = 0.0f;
#pragma unroll
        for (int t = 0; t < T::KT; ++t) {
            if ((t < 13) != (hf == 0)) continue;
            const int aa = t / 5, bb = t % 5;
            const int rr = r + aa - R;
            if (rr < 0 || rr >= T::RH) continue;
            s += Yr[(t * T::YROWS + rr % T::YROWS) * T::YW + 2 + c - R + bb];
        }
        Gr[hf * T::RH * T::RW + r * T::RW + c] = s;
    };

    unsigned long long *ph = (a.dbg_times && blockIdx.x == 0 && blockIdx.y == 0 && wt == 0)
                                 ? a.dbg_times + 3 * (size_t)gridDim.x * gridDim.y : nullptr;
    for (int blk = wg; blk < T::NBLK; blk += T::NWG) {
        if (ph) ph[blk * 8 + 0] = globaltimer_ns();
        const int lr = 2 * blk + (pl >> 6), lc = pl & 63;  // this thread's pixel (region-local)
        const int gy = g.ry0 + lr, gx = g.rx0 + lc;
        const bool in_img = !SYM || (gy >= 0 && gy < a.H && gx >= 0 && gx < a.W);
        const bool owned = gy >= g.s0 && gy < g.s1 && gx >= g.c0 && gx < g.c1;
        // ---- im2col into TMEM, taps 0..23 (K = 24): half 0 u_new, half 1 du ----
        if (hf == 0 || TRIAL) {
            float hi[32], lo[32];
            const float *src = (hf ? Du : Un) + lr * SW + lc;
#pragma unroll
            for (int t = 0; t < 32; ++t) {
                const float x = t < 24 ? src[(t / 5) * SW + (t % 5)] : 0.0f;
                hi[t] = tf32_hi(x);
                lo[t] = x - hi[t];
            }
            tmem_st32(tbase + lane_off + (hf ? T::C_ADH : T::C_AUH), hi);
            tmem_st32(tbase + lane_off + (hf ? T::C_ADL : T::C_AUL), lo);
        }
        if (ph) ph[blk * 8 + 1] = globaltimer_ns();
        tc_wait_st();
        tc_fence_before();
        asm volatile("bar.sync %0, %1;" ::"r"(1 + wg), "r"(T::WGT) : "memory");
        if (ph) ph[blk * 8 + 2] = globaltimer_ns();
        if (wt == 0) {
            tc_fence_after();
            umma_3xtf32<32>(tbase + T::C_DZ, tbase + T::C_AUH, tbase + T::C_AUL, kf_hi, kf_lo, 3, false);
            if (TRIAL) umma_3xtf32<32>(tbase + T::C_DDZ, tbase + T::C_ADH, tbase + T::C_ADL, kf_hi, kf_lo, 3, false);
            umma_commit(&s_mma[wg]);
        }
        // while the forward MMAs run: shifted sums of block blk-3 (its Y neighbours finished an
        // iteration ago; the 6-block ring keeps blk-4 .. blk+1 live)
        if (blk >= 3) {
            mbar_wait(&s_ready[blk - 3], 0);
            shifted_sum(blk - 3);
        }
        // tap 24 (a = b = 4) on the CUDA cores: the MMAs cover K = 24
        const float u24 = Un[(lr + 4) * SW + lc + 4];
        const float d24 = TRIAL ? Du[(lr + 4) * SW + lc + 4] : 0.0f;
        if (ph) ph[blk * 8 + 3] = globaltimer_ns();
        mbar_wait(&s_mma[wg], mma_phase);
        mma_phase ^= 1u;
        tc_fence_after();
        if (ph) ph[blk * 8 + 4] = globaltimer_ns();
        // ---- pointwise on this half's filters [16 hf, 16 hf + 16): psi' -> Psi operand, then the
        //      energy terms while the adjoint MMAs run ----
        {
            const int f0 = 16 * hf;
            float z[16], dz[16];
            tmem_ld16(tbase + lane_off + T::C_DZ + f0, z);
            if (TRIAL) tmem_ld16(tbase + lane_off + T::C_DDZ + f0, dz);
            tc_wait_ld();
            float hi[16], lo[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const int f = f0 + i;
                if (i < FH && f < NF) {
                    const float k24 = s_k24[f];
                    z[i] = fmaf(k24, u24, z[i]);
                    if (TRIAL) dz[i] = fmaf(k24, d24, dz[i]);
                    const float zz = z[i];
                    const float ps = in_img ? zz * rcp_approx(fmaf(zz, zz, 1.0f)) : 0.0f;
                    hi[i] = tf32_hi(ps);
                    lo[i] = ps - hi[i];
                } else {
                    hi[i] = 0.0f;
                    lo[i] = 0.0f;
                }
            }
            tmem_st16(tbase + lane_off + T::C_AUH + f0, hi);
            tmem_st16(tbase + lane_off + T::C_AUL + f0, lo);
            tc_wait_st();
            tc_fence_before();
            asm volatile("bar.sync %0, %1;" ::"r"(1 + wg), "r"(T::WGT) : "memory");
            if (wt == 0) {
                tc_fence_after();
                umma_3xtf32<32>(tbase + T::C_DZ, tbase + T::C_AUH, tbase + T::C_AUL, kt_hi, kt_lo, NF / 8, false);
                umma_commit(&s_mma[wg]);
            }
            float e0 = 0.0f, e1 = 0.0f;
            if (TRIAL) {
                float tt[16];
                float tmax = 0.0f;
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    if (!(i < FH && f0 + i < NF)) { tt[i] = 0.0f; continue; }
                    const float zz = z[i], d = dz[i];
                    const float zo = zz - d;
                    const float num = d * fmaf(2.0f, zo, d);
                    const float den = fmaf(zo, zo, fmaf(zz, zz, 2.0f));
                    tt[i] = num * rcp_approx(den);
                    tmax = fmaxf(tmax, fabsf(tt[i]));
                }
                if (__any_sync(0xffffffffu, tmax > 0.2f)) {
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        if (!(i < FH && f0 + i < NF)) continue;
                        const float term = s_al[f0 + i] * two_atanh(tt[i]);
                        if (i & 1) e1 += term; else e0 += term;
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        if (!(i < FH && f0 + i < NF)) continue;
                        const float t1 = tt[i], sq = t1 * t1;
                        float pp = fmaf(sq, 1.0f / 9.0f, 1.0f / 7.0f);
                        pp = fmaf(sq, pp, 1.0f / 5.0f);
                        pp = fmaf(sq, pp, 1.0f / 3.0f);
                        pp = fmaf(sq, pp, 1.0f);
                        const float term = (2.0f * s_al[f0 + i]) * t1 * pp;
                        if (i & 1) e1 += term; else e0 += term;
                    }
                }
            } else {
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    if (!(i < FH && f0 + i < NF)) continue;
                    const float term = s_al[f0 + i] * log1pf(z[i] * z[i]);
                    if (i & 1) e1 += term; else e0 += term;
                }
            }
            if (owned) e_own += (double)(e0 + e1);
        }
        if (ph) ph[blk * 8 + 5] = globaltimer_ns();
        mbar_wait(&s_mma[wg], mma_phase);
        mma_phase ^= 1u;
        tc_fence_after();
        if (ph) ph[blk * 8 + 6] = globaltimer_ns();
        // ---- Y rows of this block into the ring: half 0 taps 0..15, half 1 taps 16..24 ----
        {
            float y[16];
            tmem_ld16(tbase + lane_off + T::C_DZ + 16 * hf, y);
            tc_wait_ld();
            float *yrow = Yr + (lr % T::YROWS) * T::YW + 2 + lc;
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const int t = 16 * hf + i;
                if (t < T::KT) yrow[t * T::YROWS * T::YW] = y[i];
            }
        }
        tc_fence_before();
        mbar_arrive(&s_ready[blk]);
        if (ph) ph[blk * 8 + 7] = globaltimer_ns();
    }
    // the last three blocks' rows (their later Y neighbours exist only now)
    for (int gb = T::NBLK - 3 + wg; gb < T::NBLK; gb += T::NWG) {
        for (int q = gb - 1; q <= gb + 1; ++q)
            if (q >= 0 && q < T::NBLK) mbar_wait(&s_ready[q], 0);
        shifted_sum(gb);
    }
    acc[0] = e_own;
    tc_fence_before();
    __syncthreads();
    if (a.dbg_times && tid == 0) a.dbg_times[cta * 3 + 2] = globaltimer_ns();
    if (warp == 0) tmem_dealloc(s_tmem, 512);

    // ---- fold padded pixels (symmetric rule) and write the owned gradient ----
    {
        const int xx = tid % T::RW;
        const int gx = g.c0 + xx;
        if (gx < g.c1) {
            const int lx = gx - g.rx0;
            int mx = -1;
            if (SYM) {
                if (gx < R) mx = (-1 - gx) - g.rx0;
                else if (gx >= a.W - R) mx = (2 * a.W - 1 - gx) - g.rx0;
            }
            for (int gy = g.s0 + tid / T::RW; gy < g.s1; gy += NT / T::RW) {
                const int ly = gy - g.ry0;
                auto gsum2 = [&](int yy, int xx2) { return Gr[yy * T::RW + xx2] + Gr[T::RH * T::RW + yy * T::RW + xx2]; };
                float val = gsum2(ly, lx);
                if (SYM) {
                    int my = -1;
                    if (gy < R) my = (-1 - gy) - g.ry0;
                    else if (gy >= a.H - R) my = (2 * a.H - 1 - gy) - g.ry0;
                    if (my >= 0) val += gsum2(my, lx);
                    if (mx >= 0) val += gsum2(ly, mx);
                    if (my >= 0 && mx >= 0) val += gsum2(my, mx);
                }
                gout[(size_t)(gy - a.lrow0) * a.W + gx] = val;
            }
        }
    }

    // ---- per-tile partials, last CTA of the image reduces and decides (as k_pass) ----
    block_reduce<NT>(acc, red, s_sum);
    if (tid < kNumPartials) {
        a.partials[((size_t)g.t * a.B + b) * kPartialStride + tid] = s_sum[tid];
        __threadfence();
    }
    if (a.band) return;
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
