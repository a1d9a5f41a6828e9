// foe_tc.cuh -- tcgen05 / TMEM primitives for the tensor-core FoE pass (included by foe_b200.cu).
//
// Operand conventions used by the implicit-GEMM pass:
//  * A (M = 128 pixels x K) lives in TMEM: lane = pixel, one fp32/tf32 element per column.  Written
//    by the owning thread with tcgen05.st (32x32b), no shared-memory staging (the "TS" MMA form).
//  * B (N x K, K-major) lives in shared memory in the SWIZZLE_NONE canonical layout: core matrices
//    of 8 rows x 16 bytes, 8-row groups SBO bytes apart, 16-byte K chunks LBO bytes apart.
//  * D (128 x N fp32) in TMEM, read back with tcgen05.ld 32x32b (thread = pixel, register = column).
//  * fp32 accuracy from tf32 units: x = hi + lo with hi = x truncated to tf32, lo = x - hi (exact);
//    A.B ~= A_hi.B_hi + A_lo.B_hi + A_hi.B_lo (3xTF32, the A_lo.B_lo term is below fp32 rounding).

__device__ __forceinline__ float tf32_hi(float x) { return __uint_as_float(__float_as_uint(x) & 0xffffe000u); }
// nearest tf32: the 3xTF32 split x = hi + lo with hi = rn(x), lo = rn(x - hi) leaves |lo| <= 2^-11 |x|
// and a lo error <= 2^-22 |x| (the MMA truncates fp32 inputs to tf32).  cvt.rn.tf32.f32 is one
// instruction on sm_100a (F2FP.TF32.F32), where cvt.rna (and the integer add-and-mask form) take two.
__device__ __forceinline__ float tf32_rn(float x) {
    uint32_t r;
    asm("cvt.rn.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

// lo operand of a split: x + half a tf32 ulp, left for the MMA to truncate -- the tensor core reads the
// top 19 bits, so this is rn(x) as an operand without the masking instruction (never used otherwise)
__device__ __forceinline__ float tf32_rn_operand(float x) { return __uint_as_float(__float_as_uint(x) + 0x1000u); }

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// tcgen05.alloc by one full warp; the allocated base address is written to *slot (shared memory)
__device__ __forceinline__ void tmem_alloc(uint32_t *slot, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)), "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void tmem_dealloc(uint32_t base, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base), "r"(ncols) : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tc_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// generic-proxy shared-memory writes -> visible to the tensor core (async proxy)
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// 32 consecutive columns of this warp's 32 lanes: thread t <-> lane (32*(warp%4) + t)
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float (&v)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr),
        "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]), "f"(v[9]),
        "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15]), "f"(v[16]), "f"(v[17]), "f"(v[18]),
        "f"(v[19]), "f"(v[20]), "f"(v[21]), "f"(v[22]), "f"(v[23]), "f"(v[24]), "f"(v[25]), "f"(v[26]), "f"(v[27]),
        "f"(v[28]), "f"(v[29]), "f"(v[30]), "f"(v[31])
        : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7]), "=f"(v[8]),
          "=f"(v[9]), "=f"(v[10]), "=f"(v[11]), "=f"(v[12]), "=f"(v[13]), "=f"(v[14]), "=f"(v[15]), "=f"(v[16]),
          "=f"(v[17]), "=f"(v[18]), "=f"(v[19]), "=f"(v[20]), "=f"(v[21]), "=f"(v[22]), "=f"(v[23]), "=f"(v[24]),
          "=f"(v[25]), "=f"(v[26]), "=f"(v[27]), "=f"(v[28]), "=f"(v[29]), "=f"(v[30]), "=f"(v[31])
        : "r"(taddr)
        : "memory");
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float (&v)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16};" ::"r"(taddr),
        "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]), "f"(v[9]),
        "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15])
        : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15}, [%16];"
        : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7]), "=f"(v[8]),
          "=f"(v[9]), "=f"(v[10]), "=f"(v[11]), "=f"(v[12]), "=f"(v[13]), "=f"(v[14]), "=f"(v[15])
        : "r"(taddr)
        : "memory");
}

__device__ __forceinline__ void tmem_st8(uint32_t taddr, const float (&v)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
                 "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
                 : "memory");
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float (&v)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
                 : "r"(taddr)
                 : "memory");
}

__device__ __forceinline__ void tmem_st2(uint32_t taddr, float v0, float v1) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(taddr), "f"(v0), "f"(v1) : "memory");
}

__device__ __forceinline__ void tmem_st4(uint32_t taddr, const float (&v)[4]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr), "f"(v[0]), "f"(v[1]),
                 "f"(v[2]), "f"(v[3])
                 : "memory");
}

__device__ __forceinline__ void tmem_ld4(uint32_t taddr, float (&v)[4]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3])
                 : "r"(taddr)
                 : "memory");
}

// N = 4 .. 32 (multiple of 4) consecutive columns in the fewest instructions
template <int N>
__device__ __forceinline__ void tmem_ldn(uint32_t taddr, float (&v)[N]) {
    static_assert(N % 4 == 0 && N >= 4 && N <= 32, "column count");
    if constexpr (N == 32) {
        tmem_ld32(taddr, v);
    } else if constexpr (N >= 16) {
        tmem_ld16(taddr, *reinterpret_cast<float(*)[16]>(&v[0]));
        if constexpr (N > 16) tmem_ldn<N - 16>(taddr + 16, *reinterpret_cast<float(*)[N - 16]>(&v[16]));
    } else if constexpr (N >= 8) {
        tmem_ld8(taddr, *reinterpret_cast<float(*)[8]>(&v[0]));
        if constexpr (N > 8) tmem_ldn<N - 8>(taddr + 8, *reinterpret_cast<float(*)[N - 8]>(&v[8]));
    } else {
        tmem_ld4(taddr, v);
    }
}
template <int N>
__device__ __forceinline__ void tmem_stn(uint32_t taddr, const float (&v)[N]) {
    static_assert(N % 4 == 0 && N >= 4 && N <= 32, "column count");
    if constexpr (N == 32) {
        tmem_st32(taddr, v);
    } else if constexpr (N >= 16) {
        tmem_st16(taddr, *reinterpret_cast<const float(*)[16]>(&v[0]));
        if constexpr (N > 16) tmem_stn<N - 16>(taddr + 16, *reinterpret_cast<const float(*)[N - 16]>(&v[16]));
    } else if constexpr (N >= 8) {
        tmem_st8(taddr, *reinterpret_cast<const float(*)[8]>(&v[0]));
        if constexpr (N > 8) tmem_stn<N - 8>(taddr + 8, *reinterpret_cast<const float(*)[N - 8]>(&v[8]));
    } else {
        tmem_st4(taddr, v);
    }
}

// mbarrier wait: a non-blocking probe, then probes with a short nanosleep backoff so waiting warps
// leave the issue slots to the working ones
__device__ __forceinline__ bool mbar_test(unsigned long long *bar, unsigned parity) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    uint32_t ok;
    asm volatile(
        "{ .reg .pred p;\n"
        "mbarrier.test_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
    return ok != 0u;
}
#ifndef FOE_SLEEP_NS
#define FOE_SLEEP_NS -1  // < 0: mbarrier.try_wait (hardware-suspended; measured best: 5.40 vs 5.52 ms per cfg2 solve with 32 ns sleeps, 5.44 spinning)
#endif
__device__ __forceinline__ void mbar_wait_sleep(unsigned long long *bar, unsigned parity) {
#if FOE_SLEEP_NS < 0
    // hardware-suspended wait (mbarrier.try_wait blocks up to a system-defined time per probe)
    const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile(
        "{ .reg .pred p;\n"
        "WAITS_%=: mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAITS_%=; }" ::"r"(a),
        "r"(parity)
        : "memory");
#else
    while (!mbar_test(bar, parity)) {
        if (FOE_SLEEP_NS > 0) __nanosleep(FOE_SLEEP_NS);
    }
#endif
}

// TMA bulk copy global -> shared (cp.async.bulk, no tensor map): one thread issues it, the bytes land through
// the async proxy and complete the transaction count armed on the mbarrier
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(unsigned long long *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst_smem, const void *src_gmem, uint32_t bytes, unsigned long long *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst_smem)),
                 "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// hardware named barriers: producers arrive without blocking, the consumer warp blocks in sync
// (no issue slots spent waiting); every participant passes the same thread count
__device__ __forceinline__ void named_arrive(int id, int nthreads) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void named_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// one lane of a converged warp (tcgen05.mma / commit are single-thread instructions; issuing them
// from converged code keeps their operands in uniform registers)
__device__ __forceinline__ bool elect_one() {
    uint32_t pred;
    asm volatile(
        "{ .reg .pred p;\n"
        "elect.sync _|p, 0xffffffff;\n"
        "selp.u32 %0, 1, 0, p; }"
        : "=r"(pred));
    return pred != 0u;
}

// UMMA shared-memory descriptor, K-major, SWIZZLE_NONE (sm_100 "version 1" format)
__device__ __forceinline__ uint64_t umma_desc_kmajor(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1u << 46;  // version
    // base_offset 0, lbo_mode 0, layout_type 0 (SWIZZLE_NONE)
    return d;
}

// instruction descriptor: kind::tf32, D fp32, A/B tf32 K-major, M x N
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// D[tmem] (+)= A[tmem] . B[smem]^T   (one K = 8 slice)
__device__ __forceinline__ void umma_tf32_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                             uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, {%5, %6, %7, %8}, p;\n\t}\n" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate), "r"(0u), "r"(0u), "r"(0u), "r"(0u)
        : "memory");
}

// arrive on an mbarrier when all previously issued tcgen05.mma of this thread have completed
__device__ __forceinline__ void umma_commit(unsigned long long *mbar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(mbar))
                 : "memory");
}

// B operand (N rows x K cols, K-major) element offset in floats within the SWIZZLE_NONE layout with
// SBO = 128 B (8-row groups contiguous) and LBO = (N/8) * 128 B (next 16-byte K chunk)
template <int N>
__device__ __forceinline__ int bsw_offset(int n, int k) {
    return (n & 7) * 4 + (k & 3) + (n >> 3) * 32 + (k >> 2) * (N / 8) * 32;
}

// 3xTF32 product of one 128 x K (TMEM) by N x K (smem) pair, K = 8 * nk; a_hi/a_lo are TMEM column
// bases of the split A, b_hi/b_lo shared addresses of the split B.  Issued by one thread.
template <int N>
__device__ __forceinline__ void umma_3xtf32(uint32_t d_tmem, uint32_t a_hi, uint32_t a_lo, uint32_t b_hi, uint32_t b_lo,
                                            int nk, bool accumulate) {
    constexpr uint32_t LBO = (N / 8) * 128, SBO = 128;
    const uint32_t idesc = idesc_tf32(128, N);
    for (int j = 0; j < nk; ++j) {
        const uint64_t dh = umma_desc_kmajor(b_hi + 2 * j * LBO, LBO, SBO);
        const uint64_t dl = umma_desc_kmajor(b_lo + 2 * j * LBO, LBO, SBO);
        umma_tf32_ts(d_tmem, a_hi + 8 * j, dh, idesc, (accumulate || j > 0) ? 1u : 0u);
        umma_tf32_ts(d_tmem, a_lo + 8 * j, dh, idesc, 1u);
        umma_tf32_ts(d_tmem, a_hi + 8 * j, dl, idesc, 1u);
    }
}

// the same product with the B descriptors built once (db[2 j] = hi, db[2 j + 1] = lo of K step j):
// the issuing thread then spends three instructions per K step
template <int N, int NK>
struct BDescs {
    uint64_t d[2 * NK];
    __device__ __forceinline__ void build(uint32_t b_hi, uint32_t b_lo) {
        constexpr uint32_t LBO = (N / 8) * 128, SBO = 128;
#pragma unroll
        for (int j = 0; j < NK; ++j) {
            d[2 * j] = umma_desc_kmajor(b_hi + 2 * j * LBO, LBO, SBO);
            d[2 * j + 1] = umma_desc_kmajor(b_lo + 2 * j * LBO, LBO, SBO);
        }
    }
};
template <int N, int NK>
__device__ __forceinline__ void umma_3xtf32_pre(uint32_t d_tmem, uint32_t a_hi, uint32_t a_lo, const BDescs<N, NK> &b,
                                                int nk) {
    constexpr uint32_t idesc = idesc_tf32(128, N);
#pragma unroll
    for (int j = 0; j < NK; ++j) {
        if (j >= nk) break;
        umma_tf32_ts(d_tmem, a_hi + 8 * j, b.d[2 * j], idesc, j > 0 ? 1u : 0u);
        umma_tf32_ts(d_tmem, a_lo + 8 * j, b.d[2 * j], idesc, 1u);
        umma_tf32_ts(d_tmem, a_hi + 8 * j, b.d[2 * j + 1], idesc, 1u);
    }
}

// ------------------------------------------------------------------------------------------------
// self-test: D (128 x 32) = A (128 x 32) . B (32 x 32)^T through the exact primitives of the pass

__global__ void __launch_bounds__(128) k_tc_selftest(const float *__restrict__ A, const float *__restrict__ B,
                                                     float *__restrict__ D) {
    __shared__ __align__(128) float sB[2][32 * 32];
    __shared__ uint32_t s_tmem;
    __shared__ __align__(8) unsigned long long s_mbar;
    const int tid = threadIdx.x, warp = tid >> 5;
    if (warp == 0) tmem_alloc(&s_tmem, 128);
    if (tid == 0) mbar_init(&s_mbar, 1);
    for (int e = tid; e < 32 * 32; e += 128) {
        const int n = e / 32, k = e % 32;
        const float x = B[e];
        const float h = tf32_hi(x);
        sB[0][bsw_offset<32>(n, k)] = h;
        sB[1][bsw_offset<32>(n, k)] = x - h;
    }
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = s_tmem;
    const uint32_t lane_base = (uint32_t)(32 * (warp & 3)) << 16;
    {
        float hi[32], lo[32];
#pragma unroll
        for (int k = 0; k < 32; ++k) {
            const float x = A[tid * 32 + k];
            hi[k] = tf32_hi(x);
            lo[k] = x - hi[k];
        }
        tmem_st32(tbase + lane_base + 0, hi);   // A_hi: columns [0, 32)
        tmem_st32(tbase + lane_base + 32, lo);  // A_lo: columns [32, 64)
    }
    tc_wait_st();
    tc_fence_before();
    __syncthreads();
    if (tid == 0) {
        tc_fence_after();
        umma_3xtf32<32>(tbase + 64, tbase + 0, tbase + 32, smem_u32(sB[0]), smem_u32(sB[1]), 4, false);
        umma_commit(&s_mbar);
    }
    mbar_wait(&s_mbar, 0);
    tc_fence_after();
    float d[32];
    tmem_ld32(tbase + lane_base + 64, d);
    tc_wait_ld();
#pragma unroll
    for (int n = 0; n < 32; ++n) D[tid * 32 + n] = d[n];
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tbase, 128);
}

// ------------------------------------------------------------------------------------------------
// MMA issue/throughput probe: one thread issues nmma accumulating kind::tf32 MMAs (M = 128, N, K = 8)
// with A in TMEM (ts = true) or shared memory, then waits for their commit; clock64 cycles -> out[0]

__device__ __forceinline__ void umma_tf32_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                             uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}

template <int N, bool TS>
__global__ void __launch_bounds__(128) k_tc_rate(int nmma, int nchain, int every, long long *out) {
    __shared__ __align__(128) float sA[128 * 8];
    __shared__ __align__(128) float sB[N * 8];
    __shared__ uint32_t s_tmem;
    __shared__ __align__(8) unsigned long long s_mbar, s_mid[128];
    const int tid = threadIdx.x, warp = tid >> 5;
    if (warp == 0) tmem_alloc(&s_tmem, 512);
    if (tid == 0) mbar_init(&s_mbar, 1);
    mbar_init(&s_mid[tid], 1);
    for (int e = tid; e < 128 * 8; e += 128) sA[e] = 0.0f;
    for (int e = tid; e < N * 8; e += 128) sB[e] = 0.0f;
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t t0 = s_tmem;
    if (warp == 0) {
        const uint64_t bd = umma_desc_kmajor(smem_u32(sB), (N / 8) * 128, 128);
        const uint64_t ad = umma_desc_kmajor(smem_u32(sA), (128 / 8) * 128, 128);
        const uint32_t idesc = idesc_tf32(128, N);
        const long long c0 = clock64();
        if (elect_one()) {
            // nchain independent accumulators (D columns 256 + N c), issued round robin: a dependent chain of
            // small MMAs exposes the pipeline's accumulate latency, independent chains overlap
            if (every <= 0) {
                int c = 0;
                for (int i = 0; i < nmma; ++i) {
                    const uint32_t d = t0 + 256 + (uint32_t)(c * N);
                    if (TS) umma_tf32_ts(d, t0, bd, idesc, i >= nchain);
                    else umma_tf32_ss(d, ad, bd, idesc, i >= nchain);
                    c = c + 1 == nchain ? 0 : c + 1;
                }
            } else {
                // a tcgen05.commit (to an mbarrier nobody waits on) after each group of `every` MMAs
                for (int g = 0; g * every < nmma; ++g) {
                    for (int k = 0; k < every; ++k) {
                        if (TS) umma_tf32_ts(t0 + 256, t0, bd, idesc, (g | k) != 0);
                        else umma_tf32_ss(t0 + 256, ad, bd, idesc, (g | k) != 0);
                    }
                    if ((g + 1) * every < nmma) umma_commit(&s_mid[g & 127]);
                }
            }
            umma_commit(&s_mbar);
        }
        __syncwarp();
        mbar_wait(&s_mbar, 0);
        const long long c1 = clock64();
        if (tid == 0) out[0] = c1 - c0;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(t0, 512);
}

// ------------------------------------------------------------------------------------------------
// TMEM read / write throughput probe: nwarps warps (4 per lane quarter group) each issue `iters` rounds of four
// tcgen05.ld (or st) .32x32b.x32 (512 bytes per lane quarter per instruction); clock64 cycles -> out[0]
template <bool STORE>
__global__ void __launch_bounds__(1024) k_tmem_rate(int iters, long long *out) {
    __shared__ uint32_t s_tmem;
    __shared__ long long s_t[32];
    const int tid = threadIdx.x, warp = tid >> 5;
    if (warp == 0) tmem_alloc(&s_tmem, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t base = s_tmem + ((uint32_t)(32 * (warp & 3)) << 16);
    float v[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = 0.0f;
    tmem_st32(base, v);
    tmem_st32(base + 32, v);
    tmem_st32(base + 64, v);
    tmem_st32(base + 96, v);
    tc_wait_st();
    __syncthreads();
    const long long c0 = clock64();
    float acc = 0.0f;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if (STORE) {
                tmem_st32(base + 32 * k, v);
            } else {
                float w[32];
                tmem_ld32(base + 32 * k, w);
                tc_wait_ld();
                acc += w[0] + w[31];
            }
        }
        if (STORE) tc_wait_st();
    }
    const long long c1 = clock64();
    if ((tid & 31) == 0) s_t[warp] = c1 - c0;
    tc_fence_before();
    __syncthreads();
    if (tid == 0) {
        long long m = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m = s_t[w] > m ? s_t[w] : m;
        out[0] = m;
        out[1] = (long long)acc;
    }
    if (warp == 0) tmem_dealloc(s_tmem, 512);
}

