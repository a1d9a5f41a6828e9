// foe_pass_tc.cuh -- tensor-core (tcgen05, 3xTF32) variant of the fused FoE pass for 5x5 banks
// with at most 32 filters (included by foe_b200.cu after foe_pass.cuh / foe_tc.cuh).
//
// Same tile geometry, prologue, fold and reductions as k_pass; the two convolutions become implicit
// GEMMs on the tensor cores, one 128-pixel block (two region rows) at a time:
//   forward   Z  = A_u  . Kf^T    A_u[p][t] = u_new(p + off_t)  (im2col, K = 24 taps + one tap-24 step)
//             dZ = A_du . Kf^T    (the same for du, for the energy change)
//   adjoint   Y  = Psi  . Kt^T    Psi[p][f] = z/(1+z^2), Kt[t][f] = 2 a_f k_f[t]
//             g(q) = sum_t Y(q + off_t)[t]       (25-term shifted sum on the CUDA cores)
// A operands are written by their pixel's thread straight into TMEM (tcgen05.st), B operands sit in
// shared memory, D accumulators in TMEM; fp32 accuracy from tf32 units via the 3xTF32 split.
//
// Warp-specialised pipeline over the 18 blocks of a tile; block j uses A stage j%2 (im2col operands,
// 96 TMEM columns: u / du hi / lo, K = 24 each) and D region j%3 (its forward accumulators, Psi in
// place over them, its adjoint accumulator; 3 x 96 columns):
//   im2col (warps 0-7)      warps 0-3 A_u, warps 4-7 A_du of block j (once forward(j-2) released the
//                           stage) -> a_full[s]; warp 0 issues forward(j) once block j-3 has left the
//                           D region (d_free[j%3]) -> d_full[j%3]
//   point set s (8 warps)   blocks j = s, s+2, ...: z, dz -> energy terms and Psi (written over z, dz)
//                           -> p_full[s]; the set's first warp issues adjoint(j) -> y_full[j%3]; Y ->
//                           d_free[j%3] -> shared ring -> ring_full[j]; then g(j-1) = shifted sum over
//                           the warp's tap half once Y(j-2 .. j) are in the ring -> sum_done[j-1]
// so the tensor core, the operand build, two blocks' pointwise work and the shifted sums overlap; with
// three D regions the region a set's next block needs was freed by the other set one block earlier.
// Within a point set, warps w and w+4 share a TMEM lane quarter (same 32 pixels) and split the
// filters (forward side, NF/2 each) and taps (adjoint side, 16 + 9).  24 warps: 80 registers/thread.

#ifndef FOE_MMA_SLEEP
#define FOE_MMA_SLEEP 0  // ns between the MMA warp's polls of its mbarriers
#endif
#ifndef FOE_ISSUER_SPIN
#define FOE_ISSUER_SPIN 1  // MMA issuers: mbarrier.test_wait spin instead of try_wait (a suspended try_wait wakes
                            // ~300 cycles after the phase completes: 21.25 -> 20.8 us per pass)
#endif
__device__ __forceinline__ void tc_issuer_wait(unsigned long long *bar) {
#if FOE_ISSUER_SPIN
    while (!mbar_test(bar, 0u)) {
    }
#else
    mbar_wait(bar, 0u);
#endif
}
#ifndef FOE_SPIN_POINT
#define FOE_SPIN_POINT 2  // point sets' waits for MMA completions spin: bit 0 forward (z, dz), bit 1 adjoint (Y)
                          // (measured, with spinning issuers: 0 -> 20.8, 1 -> 20.75, 2 -> 20.5, 3 -> 20.6 us per pass)
#endif
#ifndef FOE_SPIN_MOVER
#define FOE_SPIN_MOVER 0  // movers' waits spin: bit 0 stage free, bit 1 ring (measured no different: 20.76 us)
#endif
template <bool SPIN>
__device__ __forceinline__ void tc_wait(unsigned long long *bar, unsigned parity) {
    if (SPIN) {
        while (!mbar_test(bar, parity)) {
        }
    } else {
        mbar_wait_sleep(bar, parity);
    }
}
#ifndef FOE_TAPSPLIT
#define FOE_TAPSPLIT 10  // the u movers sum taps [0, FOE_TAPSPLIT), the du movers the rest (whole filter rows; the u
                         // movers are the later ones: measured 8 -> 20.45, 10 -> 20.38, 12 -> 20.54, 15 -> 20.43 us per pass)
#endif
#ifndef FOE_ABLATE
#define FOE_ABLATE 0  // timing diagnostics only (results wrong): 1 no shifted sums, 2 no energy series, 4 no psi math, 8 one MMA per sweep, 16 no im2col, 32 im2col without its shared-memory loads, 64 im2col without its TMEM stores
#endif

template <int NF_MAX>
struct TcCfg {
    using P = PassCfg<5>;
    static constexpr int R = 2, M = 5, KT = 25;
    static constexpr int RH = P::RH, RW = P::RW, SH = P::SH, SW = P::SW, PLANE = P::PLANE;
    static constexpr int NBLK = RH * RW / 128;  // 128-pixel blocks (two region rows each)
    // warps 0-7 movers (im2col, shifted sums), 8-15 / 16-23 the two point sets (psi', energy terms, Y drain),
    // 24 / 25 / 26 the MMA issuers of z, dz and the adjoint
    static constexpr int W_PT = 8, W_MMA = 24, NWARPS = 27, NT = NWARPS * 32;
    // named barriers: the movers' per-block barrier (ring writes before ring reads), the epilogue's
    static constexpr int BAR_MOVERS = 1, BAR_EPI = 14;
    static constexpr int RING = 4;                       // Y ring: 4 blocks = 8 region rows
    static constexpr int SUMLAG = 4;                     // the movers sum g(j - SUMLAG) after im2col(j)
    static constexpr int YROWS = 2 * RING, YW = RW + 4;  // 2 zero columns each side
    static constexpr int BSZ = 32 * 32;                  // one 32 x 32 B operand (floats)
    // A operands (TMEM, lane = pixel): two quantities (u, du) of KA = 56 columns each.  Column order = the
    // order the im2col loads deliver them, so every tcgen05.st takes consecutive registers: per filter row
    // dy the pairs {hi, lo} of taps dx 0..3 (8 columns, two LDS.128 of the pair-replicated staged cells),
    // then the {hi, lo} pairs of tap dx = 4 of the five rows (10 columns), then 6 zero columns.
    //   column 8 dy + 2 dx + part (dx < 4);  40 + 2 dy + part (dx = 4);  part 0 = tf32 hi, 1 = tf32 lo
    static constexpr int KA = 56, KSTEPS = KA / 8, NDREG = 3;
    // A tcgen05.mma of this shape (M = 128, K = 8, tf32) occupies the tensor pipe ~51 cycles for any N <= 64
    // (tools/tc_rate.py), so the block loop is bound by the MMA *count*: the two sweeps of a 3xTF32 product
    // are merged along N instead of being issued one after the other --
    //   forward  [z1 | z2] = A . [B1 | B2]^T,  B1[k] = k_hi[tap(k)] on both parts (u_hi k_hi + u_lo k_hi),
    //            B2[k] = k_lo[tap(k)] on part 0 (u_hi k_lo): N = 2 NF, 7 MMAs per quantity, z = z1 + z2
    //   adjoint  Y = Psi . K1^T + Psi . K2^T, Psi = {hi, lo} pairs per filter (K = 2 NF), K1 = Kt_hi on both
    //            parts, K2 = Kt_lo on part 0: N = 32, a sweep of NF / 4 MMAs and one over the K steps that hold a hi
    //            column (4 of 6 at NF = 24) into the same columns (a merged N = 64 adjoint would cost 16 more TMEM
    //            columns per D region -- the second du stage)
    // (24 MMAs per 128-pixel block at NF = 24; ~23 / 28 / 32 pipe cycles per MMA at N = 32 / 48 / 64, tools/tc_rate.py).
    // operand image built once per bank on the host (foe_bank_create) and copied into shared memory by one
    // bulk copy per CTA: [forward (2 NF x 56) | adjoint K1 (32 x 2 NF) | K2 | alpha (64) | 2 alpha (32)] floats,
    // sized for NF = 32
    static constexpr int IMG_BF = 0, IMG_KT = 64 * KA, IMG_KT2 = IMG_KT + 32 * 64, IMG_AL = IMG_KT2 + 32 * 64, IMG_AL2 = IMG_AL + 64;
    static constexpr int IMG_FLOATS = IMG_AL2 + 32;
    static_assert(IMG_FLOATS % 4 == 0, "bulk copy: multiple of 16 bytes");
    static_assert(RW == 64 && NBLK * 128 == RH * RW, "blocks of two 64-pixel region rows");
    static_assert(NF_MAX <= 32, "one N = 32 MMA covers the bank");
};

// TMEM plan for a bank of NF (multiple of 8) filters.  D region of a block: [Z: z1 | z2 per filter half, then Psi
// pairs in place, 2 NF columns][W: dz1 | dz2 per filter half, then Y (32 columns) over them].  Within Z (and
// W) the point thread of filter half h owns columns [h NF, (h + 1) NF): part p of its filter i at h NF + p NF/2 + i,
// its Psi parts at h NF + part NF/2 + i (the same columns) -- so a thread overwrites only what it has read itself.  Three regions at
// the top of TMEM, the A operands below them: NU u stages and ND du stages of KA columns.
template <int NF>
struct TcCols {
    using T = TcCfg<32>;
    static constexpr int FH = NF / 2, NZ = 2 * NF, REGION = NZ + (NZ > 32 ? NZ : 32), C_Z = 0, C_W = NZ;
    static constexpr int C_D0 = 512 - T::NDREG * REGION;
    // both quantities double-buffered when TMEM allows (a single du stage puts im2col -> dz -> its completion
    // on a one-block cycle)
    static constexpr int NU = C_D0 >= 4 * T::KA ? 2 : 1, ND = NU;
    static constexpr int C_AU = 0, C_AD = NU * T::KA;
    static_assert(NF % 8 == 0 && NF <= 32, "filter count rounded up to a multiple of 8");
    static_assert((NU + ND) * T::KA <= C_D0 && NZ <= 64, "TMEM budget");
    // forward operand row of (filter f, part p); adjoint operand K column of (filter f, part)
    __host__ __device__ static constexpr int brow(int f, int p) { return (f / FH) * NF + p * FH + f % FH; }
    // (per filter half: the FH hi parts, then the FH lo parts -- a thread's own columns, and the K steps of the
    // second adjoint sweep, which multiplies hi parts only, shrink to those that hold a hi column)
    __host__ __device__ static constexpr int kcol(int f, int part) { return (f / FH) * NF + part * FH + f % FH; }
    __host__ __device__ static constexpr bool kstep_has_hi(int k) { return (8 * k) % NF < FH; }
};

// A-stage column of (tap, part) in the order above
__host__ __device__ constexpr int tc_acol(int tap, int part) {
    return (tap % 5 < 4) ? 8 * (tap / 5) + 2 * (tap % 5) + part : 40 + 2 * (tap / 5) + part;
}

template <int NF_MAX>
__host__ __device__ constexpr size_t tc_smem_floats() {
    using T = TcCfg<NF_MAX>;
    // staged cells (u and du, pair-replicated: 4 floats each); operand image; Y ring; region gradient (two tap halves)
    return 8 * (size_t)T::PLANE + (size_t)T::IMG_FLOATS + (size_t)T::KT * T::YROWS * T::YW + 2 * (size_t)T::RH * T::RW;
}

// sum over taps [T0, T1) of Y(row r + a - R, column c + b - R)[a M + b] from the Y ring: one ring-row
// offset per filter row a, then an immediate-offset load per tap.  EDGE (first / last block only): rows
// outside the region contribute zero.
template <int T0, int T1, bool EDGE, class T>
__device__ __forceinline__ float tc_tap_sum(const float *Yr, int r, int c) {
    static_assert((T::YROWS & (T::YROWS - 1)) == 0, "ring rows: power of two");
    float s0 = 0.0f, s1 = 0.0f;
    const float *base = Yr + 2 + c - T::R;
#pragma unroll
    for (int aa = T0 / T::M; aa <= (T1 - 1) / T::M; ++aa) {
        const int rr = r + aa - T::R;
        if (EDGE && (rr < 0 || rr >= T::RH)) continue;  // warp-uniform (a warp covers one region row)
        const float *rowp = base + (rr & (T::YROWS - 1)) * T::YW;
#pragma unroll
        for (int bb = 0; bb < T::M; ++bb) {
            const int t = aa * T::M + bb;
            if (t < T0 || t >= T1) continue;
            const float v = rowp[t * T::YROWS * T::YW + bb];
            if (t & 1) s1 += v; else s0 += v;
        }
    }
    return s0 + s1;
}

// im2col of one pixel's 25 taps of one quantity (u or du) from its pair-replicated staged cells X[p] =
// {hi(p), lo(p), hi(p+1), lo(p+1)} into the quantity's KA columns of an A stage (TMEM lane = pixel): per
// filter row two LDS.128 (taps dx 0..3) and one LDS.64 (dx 4), five tcgen05.st of consecutive registers
template <class T>
__device__ __forceinline__ void tc_im2col(const float4 *xp, uint32_t st) {
    float q[40], c[10];
    const int e2 = 8 - ((threadIdx.x >> 3) & 1);
#pragma unroll
    for (int dy = 0; dy < T::M; ++dy) {
        if (FOE_ABLATE & 32) {
#pragma unroll
            for (int i = 0; i < 8; ++i) q[8 * dy + i] = __int_as_float(st + i);
            c[2 * dy] = c[2 * dy + 1] = __int_as_float(st);
            continue;
        }
        const float4 a = xp[dy * T::SW], b = xp[dy * T::SW + 2];
        // the pair of p + 4: the left half of cell p + 4 or the right half of cell p + 3 (the same values), by
        // groups of 8 lanes -- 8-byte loads at a 16-byte stride alone use half the banks (2-way conflict)
        const float2 e = reinterpret_cast<const float2 *>(xp + dy * T::SW)[e2];
        q[8 * dy + 0] = a.x; q[8 * dy + 1] = a.y; q[8 * dy + 2] = a.z; q[8 * dy + 3] = a.w;
        q[8 * dy + 4] = b.x; q[8 * dy + 5] = b.y; q[8 * dy + 6] = b.z; q[8 * dy + 7] = b.w;
        c[2 * dy] = e.x; c[2 * dy + 1] = e.y;
    }
    if (FOE_ABLATE & 64) {  // keep the loads live
        float s = 0.0f;
#pragma unroll
        for (int i = 0; i < 40; ++i) s += q[i];
#pragma unroll
        for (int i = 0; i < 10; ++i) s += c[i];
        if (s == 1234.5f) tmem_st2(st + 48, s, s);
        return;
    }
    tmem_st16(st, *reinterpret_cast<const float(*)[16]>(q));
    tmem_st16(st + 16, *reinterpret_cast<const float(*)[16]>(q + 16));
    tmem_st8(st + 32, *reinterpret_cast<const float(*)[8]>(q + 32));
    tmem_st8(st + 40, *reinterpret_cast<const float(*)[8]>(c));
    tmem_st2(st + 48, c[8], c[9]);
}

// forward product of one quantity, both 3xTF32 sweeps in one N = 2 NF operand: [z1 | z2] = A . [B1 | B2]^T over the
// KA columns, one MMA per K step (issued by one thread); bd: descriptor of K step 0, the next 16-byte K chunk
// pair LBO2 bytes further
template <class T, int N>
__device__ __forceinline__ void tc_forward(uint32_t d_tmem, uint32_t a_tmem, uint64_t bd) {
    constexpr uint32_t idesc = idesc_tf32(128, N);
    constexpr uint64_t step = (uint64_t)(2 * (N / 8) * 128 / 16);  // two K chunks, in 16-byte units
#pragma unroll
    for (int j = 0; j < ((FOE_ABLATE & 8) ? 1 : T::KSTEPS); ++j) umma_tf32_ts(d_tmem, a_tmem + 8 * j, bd + j * step, idesc, j > 0 ? 1u : 0u);
}

// shared-memory carve-up of the tensor-core pass (dynamic buffers + the static arrays of the kernel)
struct TcSmem {
    float4 *XU, *XD;                      // staged cells, pair-replicated: {hi(p), lo(p), hi(p+1), lo(p+1)} of u / du
    float *img, *Kt, *Yr, *Gr, *s_al, *s_al2;
    double (*red)[kNumPartials];
    double *s_sum;
    unsigned long long *mb_dfull, *mb_yfull, *mb_aufull, *mb_adfull, *mb_zfull, *mb_pfull, *mb_dfree, *mb_ring, *mb_sum, *mb_img, *mb_edone;
    int *s_ticket;
};

template <int NF>
__device__ __forceinline__ TcSmem tc_carve(float *sm, double (*red)[kNumPartials], double *s_sum,
                                           unsigned long long *mb_dfull, unsigned long long *mb_yfull,
                                           unsigned long long *mb_aufull, unsigned long long *mb_adfull,
                                           unsigned long long *mb_zfull, unsigned long long *mb_pfull,
                                           unsigned long long *mb_dfree, unsigned long long *mb_ring,
                                           unsigned long long *mb_sum, unsigned long long *mb_img,
                                           unsigned long long *mb_edone, int *s_ticket) {
    using T = TcCfg<32>;
    TcSmem S;
    // staged planes, split once into tf32 hi + lo (both rounded to nearest): u_new - shift and du, each cell
    // also carrying its right neighbour's pair (one 16-byte load = two taps in the im2col)
    S.XU = reinterpret_cast<float4 *>(sm);
    S.XD = S.XU + T::PLANE;
    S.img = sm + 8 * T::PLANE;     // operand image (bulk-copied): forward [B1 | B2], adjoint [K1 | K2], alpha, 2 alpha
    S.Kt = S.img + T::IMG_KT;      // adjoint B operands K1 | K2 (N = 32 taps, K = {hi, lo} pairs of the filters)
    S.s_al = S.img + T::IMG_AL;    // alpha_f, zero-padded
    S.s_al2 = S.img + T::IMG_AL2;  // 2 alpha_f
    S.Yr = S.img + T::IMG_FLOATS;  // Y ring [tap][ring row][YW]
    S.Gr = S.Yr + T::KT * T::YROWS * T::YW;  // region gradient (before the fold), two tap halves
    S.red = red;
    S.s_sum = s_sum;
    S.mb_dfull = mb_dfull; S.mb_yfull = mb_yfull; S.mb_aufull = mb_aufull; S.mb_adfull = mb_adfull; S.mb_zfull = mb_zfull;
    S.mb_pfull = mb_pfull; S.mb_dfree = mb_dfree; S.mb_ring = mb_ring; S.mb_sum = mb_sum;
    S.mb_img = mb_img;
    S.mb_edone = mb_edone;
    S.s_ticket = s_ticket;
    return S;
}

// once per CTA: TMEM, barriers, the operand image (one bulk copy), the Y ring's zero columns (launch
// arguments only: runs before the dependency on the previous pass is awaited)
template <int NF>
__device__ __forceinline__ void tc_setup(const PassArgs &a, const TcSmem &S, uint32_t *s_tmem) {
    using T = TcCfg<32>;
    constexpr int NT = T::NT;
    const int tid = threadIdx.x, warp = tid >> 5;
    if (tid == 32) {  // warp 1: the bank's operand image, global -> shared (TMA bulk copy, completes on mb_img)
        mbar_init(S.mb_img, 1);
        fence_mbar_init();
        mbar_expect_tx(S.mb_img, T::IMG_FLOATS * 4);
        bulk_g2s(S.img, a.tc_img, T::IMG_FLOATS * 4, S.mb_img);
    }
    if (warp == 0) tmem_alloc(s_tmem, 512);
    if (tid < T::NBLK) {
        // one single-phase barrier per block and event (no index arithmetic or phase bookkeeping in the loop)
        const int j = tid;
        mbar_init(&S.mb_aufull[j], 4);  // u columns of the block's A stage built: one arrival per u mover warp
        mbar_init(&S.mb_adfull[j], 4);  // du columns built: one arrival per du mover warp
        mbar_init(&S.mb_zfull[j], 1);   // z MMAs committed
        mbar_init(&S.mb_dfull[j], 1);   // dz MMAs committed
        mbar_init(&S.mb_pfull[j], 8);   // Psi written: one arrival per warp of the block's point set
        mbar_init(&S.mb_yfull[j], 1);   // adjoint MMAs committed
        mbar_init(&S.mb_dfree[j], 8);   // Y drained from its D region: one arrival per warp of the point set
        mbar_init(&S.mb_ring[j], 8);    // Y(j) in the ring: one arrival per warp of the point set
        mbar_init(&S.mb_sum[j], 8);     // g(j) summed: one arrival per mover warp
    }
    if (tid == T::NBLK) mbar_init(S.mb_edone, 16);  // the energy change summed per warp: one arrival per point warp
    for (int e = tid; e < T::KT * T::YROWS * 4; e += NT) {  // zero columns of the Y ring
        const int col = e & 3, rr = e >> 2;
        S.Yr[rr * T::YW + (col < 2 ? col : T::YW - 4 + col)] = 0.0f;
    }
}

// staged cells per thread, and their source offsets within an image (np.pad index maps of image.py:61-65):
// launch arguments only, so the kernel computes them before it awaits the previous pass
struct TcCells {
    static constexpr int CPT = (PassCfg<5>::NCELL + TcCfg<32>::NT - 1) / TcCfg<32>::NT;
};
template <bool SYM>
__device__ __forceinline__ void tc_cell_offsets(const PassArgs &a, const TileGeom &g, int (&coff)[TcCells::CPT]) {
    using C = PassCfg<5>;
#pragma unroll
    for (int q = 0; q < TcCells::CPT; ++q) {
        const int k = threadIdx.x + q * TcCfg<32>::NT;
        const int i = k / C::CW, j = k - i * C::CW;
        coff[q] = k < C::NCELL ? (src_idx<SYM>(g.ry0 - C::R + i, a.H) - a.lrow0) * a.W + src_idx<SYM>(g.rx0 - C::R + j, a.W) : 0;
    }
}

// One trial (TRIAL) or evaluation pass of this CTA's tile: stage the trial point, the 18-block tensor-core
// loop, the fold; the z issuer's lane 0 publishes the tile's fp64 partials in buffer `pbuf` of a.partials.
// ctl: the image's control block (null in MODE_EVAL); rpar: phase parity of the once-per-pass ring
// mbarriers; take_ticket: that lane then takes the image's ticket (the last CTA reduces and decides) and
// parks it in *S.s_ticket, valid after the caller's next CTA-wide or BAR_EPI barrier.  Returns -1, before
// touching shared state, if the image is done; else 0.
template <int NF, bool TRIAL, bool SYM>
__device__ __forceinline__ int tc_body(const PassArgs &a, const TcSmem &S, const TileGeom &g, const ImgCtl *ctl,
                                       const int (&coff)[TcCells::CPT], const float (&pob)[TcCells::CPT], unsigned rpar,
                                       int pbuf, bool take_ticket,
                                       int fold_t0, unsigned long long *ph, ImgCtl *ctl_keep = nullptr) {
    using T = TcCfg<32>;
    using CL = TcCols<NF>;
    using C = PassCfg<5>;
    constexpr int NT = T::NT, R = T::R, SW = T::SW, NBLK = T::NBLK;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int b = blockIdx.y;
    float2 *xu2 = reinterpret_cast<float2 *>(S.XU), *xd2 = reinterpret_cast<float2 *>(S.XD);
    float *Kt = S.Kt, *Yr = S.Yr, *Gr = S.Gr, *s_al = S.s_al, *s_al2 = S.s_al2;
    double(*red)[kNumPartials] = S.red;
    double *s_sum = S.s_sum;
    unsigned long long *mb_dfull = S.mb_dfull, *mb_yfull = S.mb_yfull;
    (void)C::NCELL; (void)R; (void)SW; (void)lane; (void)Kt; (void)s_al; (void)s_al2; (void)xd2;
    static_assert(C::CW == SW, "staged cells are stored without row padding: cell index = i * SW + j");
    constexpr int CPT = TcCells::CPT;
    const size_t ioff = (size_t)b * a.Hl * a.W;
    // the control block's trial fields first: their L2 round trip overlaps the candidate loads below
    TrialParams p{};
    int c_done = 0;
    if (a.mode != MODE_EVAL) {
        p = trial_params(a, *ctl);
        c_done = ctl->done;
    }
    // TRIAL: every candidate slot (3 iterate planes, 2 gradient planes) and the observation are loaded
    // before the control block that names the slots is read, so the two L2 round trips overlap
    float cu[TRIAL ? 3 : 1][CPT], cg[TRIAL ? 2 : 1][CPT], canc[TRIAL ? 3 : 1];
    if (TRIAL) {
#pragma unroll
        for (int q = 0; q < CPT; ++q) {
            const int k = tid + q * NT;
            if (k < C::NCELL) {
                const size_t o = ioff + (size_t)coff[q];
#pragma unroll
                for (int sl = 0; sl < 3; ++sl) cu[sl][q] = __ldg(a.U + sl * a.plane + o);
#pragma unroll
                for (int sl = 0; sl < 2; ++sl) cg[sl][q] = __ldg(a.Gs + sl * a.plane + o);
            }
        }
        const size_t oa = ioff + (size_t)(g.s0 - a.lrow0) * a.W + g.c0;
#pragma unroll
        for (int sl = 0; sl < 3; ++sl) canc[sl] = a.zero_mean ? __ldg(a.U + sl * a.plane + oa) : 0.0f;
    }
    if (ph && tid == 0) ph[NBLK * 16 + 10] = clock64();  // candidate loads issued
    if (a.mode != MODE_EVAL) {
        if (c_done && !a.no_decide) return -1;  // image converged
        // ctl_keep: the whole block parked in shared memory for this pass's decision (the deciding CTA then
        // needs no L2 round trip for it on the pass-to-pass critical path; only that CTA writes it)
        if (ctl_keep && tid == 0) *ctl_keep = *ctl;
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
    if (ph && tid == 0) ph[NBLK * 16 + 11] = clock64();  // control block read
    const float shift = TRIAL ? (p.iu == 0 ? canc[0] : p.iu == 1 ? canc[1] : canc[2])
                              : a.zero_mean ? __ldg(uin + (size_t)(g.s0 - a.lrow0) * a.W + g.c0) : 0.0f;
    double acc[kNumPartials];
#pragma unroll
    for (int k = 0; k < kNumPartials; ++k) acc[k] = 0.0;
    // ---- prologue: stage u_new - shift and du for the region + r ring (all loads in flight first) ----
    {
        float lu[CPT], lup[CPT], lg[CPT], lob[CPT];
#pragma unroll
        for (int q = 0; q < CPT; ++q) {
            const int k = tid + q * NT;
            if (TRIAL) {  // select the slots named by the control block
                lu[q] = p.iu == 0 ? cu[0][q] : p.iu == 1 ? cu[1][q] : cu[2][q];
                lup[q] = p.iup == 0 ? cu[0][q] : p.iup == 1 ? cu[1][q] : cu[2][q];
                lg[q] = p.ig == 0 ? cg[0][q] : cg[1][q];
                lob[q] = pob[q];
            } else if (k < C::NCELL) {
                lu[q] = __ldg(uin + coff[q]);
            }
        }
#pragma unroll
        for (int q = 0; q < CPT; ++q) {
            const int k = tid + q * NT;
            if (k >= C::NCELL) continue;
            const int i = k / C::CW, j = k - i * C::CW;
            const int k1 = (tid & 8) ? 2 * k - 1 : 2 * k, k2 = (tid & 8) ? 2 * k : 2 * k - 1;
            if (!TRIAL) {
                const float x = lu[q] - shift, h = tf32_rn(x);
                const float2 pu = make_float2(h, tf32_rn_operand(x - h));
                // cell k's own pair and its copy as cell k - 1's right neighbour: lanes 8..15 / 24..31 store
                // the copy first, so that each half-warp's 8-byte stores cover all 32 banks (no 2-way conflict)
                if (k1 >= 0) xu2[k1] = pu;
                if (k2 >= 0) xu2[k2] = pu;
                continue;
            }
            const int gy = g.ry0 - R + i, gx = g.rx0 - R + j;
            const float u = lu[q], gg = lg[q], ob = lob[q];
            const float un = trial_point(u, lup[q], gg, ob, p);  // solver.py:146-149
            const float du = un - u;
            const float x = un - shift, h = tf32_rn(x), hd = tf32_rn(du);
            const float2 pu = make_float2(h, tf32_rn_operand(x - h)), pd = make_float2(hd, tf32_rn_operand(du - hd));
            if (k1 >= 0) {
                xu2[k1] = pu;
                xd2[k1] = pd;
            }
            if (k2 >= 0) {
                xu2[k2] = pu;
                xd2[k2] = pd;
            }
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
    if (ph && tid == 0) ph[NBLK * 16 + 12] = clock64();  // cells staged
    // the prologue's partials 1..6 are summed per warp now (the block loop only adds partial 0)
    // scratch: the Y ring's data columns 2 .. 65 (its zero columns stay intact), one 32-double row per ring row
    static_assert(T::YW % 2 == 0 && (NT / 32) * (kNumPartials - 1) <= T::KT * T::YROWS, "partial scratch");
    warp_partials_smem<1, kNumPartials, T::YW / 2>(acc, red, reinterpret_cast<double *>(Yr + 2));
    if (lane == 0 && (warp < T::W_PT || warp >= T::W_MMA)) red[warp][0] = 0.0;  // partial 0 comes from the point sets
    if (ph && tid == 0) ph[NBLK * 16 + 13] = clock64();  // warp partials
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    mbar_wait_sleep(S.mb_img, 0u);  // the operand image has landed (bulk copy issued in tc_setup)
    if (a.dbg_times && tid == 0) a.dbg_times[((size_t)blockIdx.y * gridDim.x + blockIdx.x) * 3 + 1] = globaltimer_ns();
    // the CTA owns all 512 columns (one CTA per SM), so the allocation starts at column 0: constant
    // TMEM addresses keep the MMA operands in uniform registers
    constexpr uint32_t tmem = 0u;
    // per-block role stamps: [block][im2col, fwd, point, sum]
    if (ph && tid == 0) ph[NBLK * 16] = clock64();  // loop start (cycles)
    unsigned long long *pw = ph ? ph + 304 + 8 * warp : nullptr;  // per-warp stamps of blocks 8 / 9
    (void)pw;

    // warp-uniform role index (a shuffle result lets the compiler keep it, and the TMEM addresses derived from
    // it, in uniform registers)
    const int wu = __shfl_sync(0xffffffffu, warp, 0);
    int early_ticket = 0;
    if (wu >= T::W_MMA) {
        // ================= MMA issuers: one warp each for z(j), dz(j) and the adjoint(j) =================
        // A warp that has issued a batch of tcgen05.mma stalls on its next uniform-datapath instructions until the
        // batch has consumed its descriptors, so a single issuer serialises its own polling and fences with the
        // tensor pipe (measured: ~450 cycles of overhead per batch, three batches per block); three issuers
        // overlap theirs.  forward operand: K-major, N = 2 NF rows; adjoint operands K1, K2: N = 32 rows, K = 2 NF
        const int role = wu - T::W_MMA;  // 0: z, 1: dz, 2: adjoint
        if (role < 2) {
            const uint64_t bfd = umma_desc_kmajor(smem_u32(S.img + T::IMG_BF), (CL::NZ / 8) * 128, 128);
            if (role == 0 || TRIAL) {
                uint32_t sd = tmem + CL::C_D0;  // D region j % 3
                int st = 0;                     // A stage j % NU
                for (int j = 0; j < NBLK; ++j, sd = sd + CL::REGION == tmem + CL::C_D0 + T::NDREG * CL::REGION ? tmem + CL::C_D0 : sd + CL::REGION,
                         st = st + 1 == CL::NU ? 0 : st + 1) {
                    // its A stage is built and block j-3's Y has left D region j%3
                    tc_issuer_wait(role == 0 ? &S.mb_aufull[j] : &S.mb_adfull[j]);
                    if (j >= T::NDREG) tc_issuer_wait(&S.mb_dfree[j - T::NDREG]);
                    tc_fence_after();
                    if (ph) ph[j * 16 + (role == 0 ? 10 : 12)] = clock64();  // z / dz issue starts
                    if (elect_one()) {
                        if (role == 0) {
                            tc_forward<T, CL::NZ>(sd + CL::C_Z, tmem + CL::C_AU + st * T::KA, bfd);
                            umma_commit(&S.mb_zfull[j]);
                        } else {
                            tc_forward<T, CL::NZ>(sd + CL::C_W, tmem + CL::C_AD + st * T::KA, bfd);
                            umma_commit(&mb_dfull[j]);
                        }
                    }
                    __syncwarp();
                    if (ph) ph[j * 16 + (role == 0 ? 11 : 0)] = clock64();  // z / dz issued
                }
            }
            if (role == 0) {
                // the z issuer is idle from here: it publishes the tile's partials and takes the image's ticket as
                // soon as the point sets have summed the last energy terms -- the movers' last shifted sums, the
                // fold and the ticket's round trip then overlap (the ticket is read after the loop's barrier)
                tc_issuer_wait(S.mb_edone);
                double x[kNumPartials];
                warp_combine<NT>(red, s_sum, x);
                if (lane == 0) {
                    double *parts = a.partials + (((size_t)pbuf * a.tiles_x * a.tiles_y + g.t) * a.B + b) * kPartialStride;
#pragma unroll
                    for (int k = 0; k < kNumPartials; ++k) parts[k] = x[k];
                    // release: this thread's partial stores; acquire: every earlier CTA's
                    if (take_ticket) early_ticket = (int)ticket_acq_rel(a.tickets + b);
                }
                if (ph && lane == 0) ph[NBLK * 16 + 5] = clock64();  // partials published, ticket requested
            }
        } else {
            const uint64_t ktd = umma_desc_kmajor(smem_u32(Kt), 512, 128);
            const uint64_t kt2d = umma_desc_kmajor(smem_u32(S.img + T::IMG_KT2), 512, 128);
            uint32_t sb = tmem + CL::C_D0;  // D region j % 3
            for (int j = 0; j < NBLK; ++j, sb = sb + CL::REGION == tmem + CL::C_D0 + T::NDREG * CL::REGION ? tmem + CL::C_D0 : sb + CL::REGION) {
                // adjoint(j) once its point set wrote the Psi pairs over z1 | z2
                tc_issuer_wait(&S.mb_pfull[j]);
                tc_fence_after();
                if (ph) ph[j * 16 + 13] = clock64();  // adjoint issue starts
                if (elect_one()) {
                    constexpr uint32_t idesc = idesc_tf32(128, 32);
#pragma unroll
                    for (int k = 0; k < ((FOE_ABLATE & 8) ? 1 : CL::NZ / 8); ++k)  // K = 2 NF; two 16-byte K chunks (2 x 512 B) per step
                        umma_tf32_ts(sb + CL::C_W, sb + CL::C_Z + 8 * k, ktd + (uint64_t)(k * 64), idesc, k > 0 ? 1u : 0u);
#pragma unroll
                    for (int k = 0; k < ((FOE_ABLATE & 8) ? 1 : CL::NZ / 8); ++k)  // K2 is zero on the lo parts: hi steps only
                        if (CL::kstep_has_hi(k)) umma_tf32_ts(sb + CL::C_W, sb + CL::C_Z + 8 * k, kt2d + (uint64_t)(k * 64), idesc, 1u);
                    umma_commit(&mb_yfull[j]);
                }
                __syncwarp();
                if (ph) ph[j * 16 + 2] = clock64();  // adjoint issued
            }
        }
    } else if (wu < T::W_PT) {
        // ================= movers: im2col(j), shifted sum g(j-3) =================
        // warps 0-3 build the u columns, warps 4-7 the du columns; warps w and w+4 share a TMEM lane quarter (the
        // same 128 pixels) and split the taps of the sum (10 + 15)
        auto mover = [&](auto HFc) {
        constexpr int hf = decltype(HFc)::value;  // 0: u columns, taps 0..9; 1: du columns, taps 10..24
        const int pl = tid & 127;
        const uint32_t lane_off = (uint32_t)(32 * (wu & 3)) << 16;
        const int nst = hf == 0 ? CL::NU : CL::ND;
        const uint32_t abase = tmem + lane_off + (hf == 0 ? CL::C_AU : CL::C_AD);
        {  // zero columns KA-8 .. KA-1 of every stage once (48, 49 are rewritten per block; the rest pad K to 56)
            const float z8[8] = {0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f};
            if (hf == 0 || TRIAL) {
                for (int st = 0; st < nst; ++st) tmem_st8(abase + st * T::KA + T::KA - 8, z8);
                tc_wait_st();
            }
        }
        const float4 *xsrc = (hf == 0 ? S.XU : S.XD) + (pl >> 6) * SW + (pl & 63);
        const int prow = pl >> 6, pcol = pl & 63;
        // (the last iteration sums the last two blocks together: both wait for Y(NBLK-1) and each sum is a
        // latency-bound step of its own)
        for (int j = 0; j < NBLK + T::SUMLAG - 1; ++j) {
            if (j < NBLK) {
                const int s = nst == 2 ? (j & 1) : 0, jp = j - nst;  // block jp used this stage last
                if (jp >= 0) {  // its MMAs have read it: the z MMAs (u stage) / the whole forward (du stage)
                    if (hf == 0) tc_wait<(FOE_SPIN_MOVER & 1) != 0>(&S.mb_zfull[jp], 0u);
                    else if (TRIAL) tc_wait<(FOE_SPIN_MOVER & 1) != 0>(&mb_dfull[jp], 0u);
                }
                tc_fence_after();
                if (ph && wu == 0) ph[j * 16 + 5] = clock64();  // im2col start
                if (pw && j == 8) pw[0] = clock64();
                if ((hf == 0 || TRIAL) && !(FOE_ABLATE & 16)) {
                    tc_im2col<T>(xsrc + 2 * j * SW, abase + s * T::KA);
                    tc_wait_st();
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(hf == 0 ? &S.mb_aufull[j] : &S.mb_adfull[j]);
                if (ph && wu == 0) ph[j * 16 + 7] = clock64();  // A stage built
                if (pw && j == 8) pw[1] = clock64();
            }
            const int js = j - T::SUMLAG;
            if (js >= 0 && js < NBLK) {  // g(js) over this warp's tap half once Y(js-1 .. js+1) are in the ring
                // (Y(js-1) and Y(js) were awaited by the two previous sums)
                if (js == 0) tc_wait<(FOE_SPIN_MOVER & 2) != 0>(&S.mb_ring[0], rpar);
                if (js + 1 < NBLK) tc_wait<(FOE_SPIN_MOVER & 2) != 0>(&S.mb_ring[js + 1], rpar);
                if (pw && j == 8) pw[2] = clock64();
                const int r = 2 * js + prow;
                float gsum;
                if (FOE_ABLATE & 1)
                    gsum = 0.0f;
                else if (js == 0 || js == NBLK - 1)
                    gsum = hf ? tc_tap_sum<FOE_TAPSPLIT, 25, true, T>(Yr, r, pcol) : tc_tap_sum<0, FOE_TAPSPLIT, true, T>(Yr, r, pcol);
                else
                    gsum = hf ? tc_tap_sum<FOE_TAPSPLIT, 25, false, T>(Yr, r, pcol) : tc_tap_sum<0, FOE_TAPSPLIT, false, T>(Yr, r, pcol);
                if (js == NBLK - 2) {
                    const float gl = hf ? tc_tap_sum<FOE_TAPSPLIT, 25, true, T>(Yr, r + 2, pcol) : tc_tap_sum<0, FOE_TAPSPLIT, true, T>(Yr, r + 2, pcol);
                    Gr[hf * T::RH * T::RW + (r + 2) * T::RW + pcol] = (FOE_ABLATE & 1) ? 0.0f : gl;
                }
                Gr[hf * T::RH * T::RW + r * T::RW + pcol] = gsum;
                __syncwarp();
                if (lane == 0) mbar_arrive(&S.mb_sum[js]);
                if (ph && wu == 0) ph[js * 16 + 4] = clock64();  // g summed
                if (pw && j == 8) pw[3] = clock64();
            }
        }
        };
        if (wu >> 2) mover(std::integral_constant<int, 1>{});
        else mover(std::integral_constant<int, 0>{});
    } else {
        // ================= point sets: psi', energy terms, shifted sums =================
        // set s handles blocks j = s (mod 2): z, dz -> psi' (tf32 hi / lo written over them as the adjoint's A
        // operand) -> p_full; then the energy terms while the adjoint runs.  Warps w and w+4 of a set share a
        // TMEM lane quarter (same 32 pixels) and split the filters.
        const int q4 = wu & 3, hf = ((wu - T::W_PT) >> 2) & 1;  // lane quarter; filter half
        const int set = (wu - T::W_PT) >> 3;                     // blocks j = set (mod 2)
        const int pl = 32 * q4 + lane;
        const uint32_t lane_off = (uint32_t)(32 * q4) << 16;
        constexpr int FH = NF / 2;  // filters per half
        const int f0 = FH * hf;
        const uint32_t own = (uint32_t)(hf * NF);  // this thread's columns within Z and W
        const int lc = pl & 63, gx = g.rx0 + lc;
        const bool col_in = !SYM || (gx >= 0 && gx < a.W), col_own = gx >= g.c0 && gx < g.c1;
        double e_own = 0.0;
        int rg = set;  // D region of block j: j % 3
        for (int j = set; j < NBLK; j += 2, rg = rg == 0 ? 2 : rg - 1) {
            tc_wait<(FOE_SPIN_POINT & 1) != 0>(&S.mb_zfull[j], 0u);            // z(j) committed
            if (TRIAL) tc_wait<(FOE_SPIN_POINT & 1) != 0>(&mb_dfull[j], 0u);  // dz(j) committed
            tc_fence_after();
            const bool pst = ph && (wu - T::W_PT) % 8 == 0;
            if (pst) ph[j * 16 + 1] = clock64();  // forward seen
            if (pw && (j >> 1) == 4) pw[0] = clock64();
            const uint32_t sd = tmem + CL::C_D0 + rg * CL::REGION + lane_off + own;
            const int gy = g.ry0 + 2 * j + (pl >> 6);
            const bool in_img = col_in && (!SYM || (gy >= 0 && gy < a.H));
            const bool owned = col_own && gy >= g.s0 && gy < g.s1;
            // this half's filters: all z / dz loads in flight at once; psi' (tf32 hi / lo, written over
            // the z / dz columns as the adjoint's A operand, whose K covers filters < NF only) and the
            // atanh arguments for every filter with full ILP; Psi is handed to the adjoint MMA before
            // the energy series are evaluated
            float z[FH], dz[FH];
            {  // z = z1 + z2, dz = dz1 + dz2 (the two sweeps of the 3xTF32 products)
                float zz[NF], dd[TRIAL ? NF : 2];
                tmem_ldn<NF>(sd + CL::C_Z, zz);
                if (TRIAL) tmem_ldn<NF>(sd + CL::C_W, *reinterpret_cast<float(*)[NF]>(dd));
                tc_wait_ld();
                if (pw && (j >> 1) == 4) pw[1] = clock64();
#pragma unroll
                for (int i = 0; i < FH; i += 2) {
                    const float2 t2 = __fadd2_rn(make_float2(zz[i], zz[i + 1]), make_float2(zz[FH + i], zz[FH + i + 1]));
                    z[i] = t2.x;
                    z[i + 1] = t2.y;
                    if (TRIAL) {
                        const float2 d2 = __fadd2_rn(make_float2(dd[i], dd[i + 1]), make_float2(dd[FH + i], dd[FH + i + 1]));
                        dz[i] = d2.x;
                        dz[i + 1] = d2.y;
                    }
                }
            }
            float tmax = 0.0f;
            // psi' (zero on padded cells outside the image: a warp-uniform test, edge tiles only)
            auto point = [&](auto keep_all) {
                if (TRIAL) {  // filter pairs in packed fp32 (FFMA2 / FMUL2 / FADD2: one issue slot per pair)
#pragma unroll
                    for (int i = 0; i < FH; i += 2) {
                        const float2 zz = make_float2(z[i], z[i + 1]), d = make_float2(dz[i], dz[i + 1]);
                        // psi' = z / (1+z^2) and t = (z^2 - zo^2) / (2+z^2+zo^2) with zo = z - d:
                        // z^2 - zo^2 = d (2z - d) and 2+z^2+zo^2 = 2 (1+z^2) - (z^2 - zo^2); two MUFU
                        // reciprocals (the XU pipe has room; fewer issue slots than one reciprocal of the product)
                        const float2 a1 = __ffma2_rn(zz, zz, make_float2(1.0f, 1.0f));
                        const float2 s2 = __ffma2_rn(zz, make_float2(2.0f, 2.0f), make_float2(-d.x, -d.y));
                        const float2 nm = __fmul2_rn(d, s2);
                        const float2 b1 = __ffma2_rn(a1, make_float2(2.0f, 2.0f), make_float2(-nm.x, -nm.y));
                        const float2 ps = __fmul2_rn(zz, make_float2(rcp_approx(a1.x), rcp_approx(a1.y)));
                        const float2 tt = __fmul2_rn(nm, make_float2(rcp_approx(b1.x), rcp_approx(b1.y)));
                        dz[i] = tt.x;
                        dz[i + 1] = tt.y;
                        tmax = fmaxf(tmax, fmaxf(fabsf(tt.x), fabsf(tt.y)));
                        z[i] = (decltype(keep_all)::value || in_img) ? ps.x : 0.0f;
                        z[i + 1] = (decltype(keep_all)::value || in_img) ? ps.y : 0.0f;
                    }
                    return;
                }
#pragma unroll
                for (int i = 0; i < FH; ++i) {
                    const float zz = z[i];
                    const float ps = zz * rcp_approx(fmaf(zz, zz, 1.0f));
                    dz[i] = zz;  // keep z for log1p(z^2)
                    z[i] = (decltype(keep_all)::value || in_img) ? ps : 0.0f;
                }
            };
            if (FOE_ABLATE & 4) {
            } else if (__all_sync(0xffffffffu, in_img))
                point(std::true_type{});
            else
                point(std::false_type{});
            {  // Psi: the FH hi parts, then the FH lo parts, over this thread's z1 | z2 columns
                float pr[NF];
#pragma unroll
                for (int i = 0; i < FH; i += 2) {
                    const float h0 = tf32_rn(z[i]), h1 = tf32_rn(z[i + 1]);
                    const float2 l2 = __fadd2_rn(make_float2(z[i], z[i + 1]), make_float2(-h0, -h1));
                    pr[i] = h0;
                    pr[i + 1] = h1;
                    pr[FH + i] = tf32_rn_operand(l2.x);
                    pr[FH + i + 1] = tf32_rn_operand(l2.y);
                }
                tmem_stn<NF>(sd + CL::C_Z, pr);
            }
            // the series' 2 alpha, loaded while the Psi stores drain (the asm statements below are compiler
            // barriers: left after them, these loads queue behind the movers' im2col traffic on the energy path)
            float2 al2r[TRIAL ? FH / 2 : 1];
            if (TRIAL) {
#pragma unroll
                for (int i = 0; i < FH; i += 2) al2r[i / 2] = *reinterpret_cast<const float2 *>(s_al2 + f0 + i);
            }
            tc_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&S.mb_pfull[j]);
            if (pst) ph[j * 16 + 6] = clock64();  // Psi handed over
            if (pw && (j >> 1) == 4) pw[2] = clock64();
            // energy terms while the adjoint MMAs run
            float e0 = 0.0f, e1 = 0.0f;
            if (FOE_ABLATE & 2) {
            } else if (TRIAL) {
                // 2 a atanh(t) = 2 a (t + t^3/3 + ...): the series is cut where the next term is below fp32
                // rounding for the warp's largest |t| (degree 9 up to 0.2, then 5, 3, 1); MUFU log beyond
                const float wmax = __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(tmax)));  // tmax >= 0
                auto series = [&](auto deg) {  // filter pairs packed: (e0, e1) = (even, odd) filters
                    constexpr int D = decltype(deg)::value;
                    float2 e = make_float2(e0, e1);
#pragma unroll
                    for (int i = 0; i < FH; i += 2) {
                        const float2 t1 = make_float2(dz[i], dz[i + 1]);
                        const float2 w = __fmul2_rn(al2r[i / 2], t1);  // 2 alpha t
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
                    two_atanh_pairs<FH>(dz, s_al + f0, s_al2 + f0, e0, e1);
                } else if (wmax > 0.04f) {
                    series(std::integral_constant<int, 9>{});
                } else if (wmax > 0.004f) {
                    series(std::integral_constant<int, 5>{});
                } else if (wmax > 1e-4f) {
                    series(std::integral_constant<int, 3>{});
                } else {
                    series(std::integral_constant<int, 1>{});
                }
            } else {
#pragma unroll
                for (int i = 0; i < FH; ++i) {
                    const float term = s_al[f0 + i] * log1pf(dz[i] * dz[i]);
                    if (i & 1) e1 += term; else e0 += term;
                }
            }
            if (owned) e_own += (double)(e0 + e1);
            if (pst) ph[j * 16 + 9] = clock64();  // energy terms done
            if (pw && (j >> 1) == 4) pw[3] = clock64();
            {  // Y(j) (the adjoint ran meanwhile): half 0 taps 0..15, half 1 taps 16..24, into ring slot j % RING
                tc_wait<(FOE_SPIN_POINT & 2) != 0>(&mb_yfull[j], 0u);
                tc_fence_after();
                if (pst) ph[j * 16 + 8] = clock64();  // adjoint seen
                if (pw && (j >> 1) == 4) pw[4] = clock64();
                float y[16];
                tmem_ld16(tmem + CL::C_D0 + rg * CL::REGION + lane_off + CL::C_W + 16 * hf, y);
                tc_wait_ld();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&S.mb_dfree[j]);  // for forward(j + 3)
                // the slot held Y(j - 4), read by g(j - 5) .. g(j - 3), which the movers sum in that order
                if (j >= T::RING) mbar_wait_sleep(&S.mb_sum[j - 3], rpar);
                float *yrow = Yr + ((2 * j + (pl >> 6)) & (T::YROWS - 1)) * T::YW + 2 + lc;
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const int t = 16 * hf + i;
                    if (t < T::KT) yrow[t * T::YROWS * T::YW] = y[i];
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&S.mb_ring[j]);
                if (pst) ph[j * 16 + 3] = clock64();  // Y in the ring
                if (pw && (j >> 1) == 4) pw[5] = clock64();
            }
        }
        acc[0] = e_own;
        // the set's warp sums of the energy change, for the z issuer (scratch: the staged u cells, dead once the
        // last block's operands are built)
        mbar_wait_sleep(&S.mb_aufull[NBLK - 1], 0u);
        warp_partials_smem<0, 1, 32>(acc, red, reinterpret_cast<double *>(S.XU));
        if (lane == 0) mbar_arrive(S.mb_edone);
    }
    tc_fence_before();
    __syncthreads();
    if (ph && tid == 0) ph[NBLK * 16 + 1] = clock64();  // loop end (cycles), CTA (0, 0)
    // ---- the tile's partials were published and the ticket requested by the z issuer (above); its lane 0 parks
    // the ticket in shared memory for the CTA's decision path ----
    if (tid == T::W_MMA * 32) *S.s_ticket = early_ticket;

    // ---- fold padded pixels (symmetric rule) and write the owned gradient: threads [fold_t0, 32 W_MMA) (the
    // rest return to run the image's reduction and decision meanwhile if this CTA is the last) ----
    if (tid < fold_t0 || tid >= T::W_MMA * 32) return 0;
    for (int k = tid - fold_t0; k < T::RW * 8; k += T::W_MMA * 32 - fold_t0) {
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
            if (ph && tid == fold_t0 && gy == g.s0) ph[NBLK * 16 + 8] = clock64();  // first value folded
            gout[(size_t)(gy - a.lrow0) * a.W + gx] = val;
            if (ph && tid == fold_t0 && gy == g.s0) ph[NBLK * 16 + 9] = clock64();  // first store issued
        }
    }

    if (ph && tid == fold_t0) ph[NBLK * 16 + 4] = clock64();  // fold done
    return 0;
}

template <int NF, bool TRIAL, bool SYM>
__global__ void __launch_bounds__(TcCfg<32>::NT, 1) k_pass_tc(const PassArgs a) {
    static_assert(NF % 8 == 0 && NF <= 32, "filter count rounded up to a multiple of 8");
    using T = TcCfg<32>;
    constexpr int NT = T::NT, NBLK = T::NBLK;
    extern __shared__ __align__(128) float sm[];
    __shared__ double red[NT / 32][kNumPartials];
    __shared__ double s_sum[kNumPartials];
    __shared__ uint32_t s_tmem;
    __shared__ __align__(8) unsigned long long mb_dfull[NBLK], mb_yfull[NBLK], mb_aufull[NBLK], mb_adfull[NBLK], mb_zfull[NBLK];
    __shared__ __align__(8) unsigned long long mb_pfull[NBLK], mb_dfree[NBLK], mb_img;
    __shared__ __align__(8) unsigned long long mb_ring[NBLK], mb_sum[NBLK];

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int b = blockIdx.y;
    const size_t cta = (size_t)blockIdx.y * gridDim.x + blockIdx.x;
    if (a.dbg_times && tid == 0) a.dbg_times[cta * 3] = globaltimer_ns();
    // per-block / per-phase cycle stamps of CTA (0, 0) for the timing diagnostic (compiled in only with
    // -DFOE_STAMPS=1: the predicated-off stamps cost ~3 % of the pass's issue slots)
#if FOE_STAMPS
    unsigned long long *ph = (a.dbg_times && blockIdx.x == gridDim.x / 2 && blockIdx.y == 0 && lane == 0)
                                 ? a.dbg_times + 3 * (size_t)gridDim.x * gridDim.y : nullptr;
#else
    constexpr unsigned long long *ph = nullptr;
    (void)lane;
#endif
    if (ph && tid == 0) ph[NBLK * 16 + 2] = clock64();  // kernel start (cycles)
    // programmatic dependent launch: the next pass may be scheduled as soon as every CTA of this one
    // has started; everything up to griddep_wait() below depends only on the launch arguments
    griddep_launch_dependents();
    const int tyl = blockIdx.x / a.tiles_x, txi = blockIdx.x - tyl * a.tiles_x;
    const TileGeom g = tile_geom<5, SYM>(a, tyl, txi);
    __shared__ __align__(8) unsigned long long mb_edone;
    __shared__ int s_ticket;
    const TcSmem S = tc_carve<NF>(sm, red, s_sum, mb_dfull, mb_yfull, mb_aufull, mb_adfull, mb_zfull, mb_pfull, mb_dfree, mb_ring, mb_sum, &mb_img,
                                  &mb_edone, &s_ticket);
    tc_setup<NF>(a, S, &s_tmem);
    int coff[TcCells::CPT];
    tc_cell_offsets<SYM>(a, g, coff);
    // the observation never changes during a solve: its cells are loaded before the dependency is awaited
    float pob[TcCells::CPT];
#pragma unroll
    for (int q = 0; q < TcCells::CPT; ++q)
        pob[q] = (TRIAL && tid + q * NT < PassCfg<5>::NCELL) ? __ldg(a.obs + (size_t)b * a.Hl * a.W + coff[q]) : 0.0f;
    griddep_wait();  // the previous pass (control block, iterates, gradients, partials) is complete
    if (a.dbg_times && tid == 0) a.dbg_times[3 * (size_t)gridDim.x * gridDim.y + 512 + cta] = globaltimer_ns();
    if (ph && tid == 0) ph[NBLK * 16 + 3] = clock64();  // dependency resolved
    if (tid == 0 && s_tmem != 0u) __trap();
    constexpr uint32_t tmem = 0u;
    const int nlaunch = a.tiles_x * a.tiles_y;
    // warps 0-7 skip the fold when the image's reduction fits the one-warp-per-partial path: the last CTA
    // reduces and decides while warps 8-23 fold (RW * 8 = 512 items, one each)
    const bool split = !a.band && nlaunch <= kFastReduceTiles && T::RW * 8 <= NT - 256;
    __shared__ ImgCtl s_ctl;
    const int live = tc_body<NF, TRIAL, SYM>(a, S, g, a.mode == MODE_EVAL ? nullptr : a.ctl + b, coff, pob, 0u, 0, !a.band,
                                             split ? 256 : 0, ph, &s_ctl);
    if (live < 0) {
        __syncthreads();  // image converged: release TMEM and leave
        if (warp == 0) tmem_dealloc(tmem, 512);
        return;
    }
    // TMEM is released at the very end (tcgen05.dealloc right after the loop stalled warp 0, and with it
    // the whole epilogue, for ~6,500 cycles)
    if (a.band) {
        if (warp == 0) tmem_dealloc(tmem, 512);
        return;
    }
    if (split) {
        // warps 8..23 folded, the dz / adjoint issuers are idle; the movers wait for the z issuer's ticket
        if (warp >= 8 && warp != T::W_MMA) return;
        named_sync(T::BAR_EPI, 288);
        if (warp == T::W_MMA) return;
        if (a.dbg_times && tid == 0) a.dbg_times[cta * 3 + 2] = globaltimer_ns();
        if (ph && tid == 0) ph[NBLK * 16 + 6] = clock64();  // ticket seen
        // TMEM is released by warp 7, which takes no part in the reduction (tcgen05.dealloc blocks its warp:
        // on warp 0 it sat on the deciding CTA's critical path)
        static_assert(kNumPartials <= 7, "warp 7 is free of the tile reduction");
        if (warp == 7) {
            tmem_dealloc(tmem, 512);
            return;
        }
        if (s_ticket != nlaunch - 1) return;
        // (no fence: the z issuer's acquiring ticket and the barrier above order the loads below)
        {  // warps 0..6: the fixed order of reduce_tiles' fast path
            double x = lane_tile_sum(a.partials, nlaunch, a.B, b, warp, lane);
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) x += __shfl_down_sync(0xffffffffu, x, off);
            if (lane == 0) s_sum[warp] = x;
        }
        named_sync(T::BAR_EPI, 224);
    } else {
        __syncthreads();
        if (a.dbg_times && tid == 0) a.dbg_times[cta * 3 + 2] = globaltimer_ns();
        if (ph && tid == 0) ph[NBLK * 16 + 6] = clock64();  // ticket seen
        if (warp == 0) tmem_dealloc(tmem, 512);
        if (s_ticket != nlaunch - 1) return;
        reduce_tiles<NT>(a.partials, nlaunch, a.B, b, red, s_sum);
    }
    if (tid == 0) {
        a.tickets[b] = 0u;
        if (a.energy_out) a.energy_out[b] = s_sum[0];  // EVAL, and a solve's final-energy pass
        if (a.mode != MODE_EVAL && !a.no_decide) {
            ImgCtl c = s_ctl;  // = a.ctl[b]: read at this pass's start, written only by this decision
            decide_ctl(a, b, s_sum, c, true, a.mode);
            a.ctl[b] = c;
        }
        if (a.dbg_times) a.dbg_times[4 * (size_t)gridDim.x * gridDim.y + 512 + cta] = globaltimer_ns();  // decider done
    }
}
