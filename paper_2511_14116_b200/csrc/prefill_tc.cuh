// K8, tcgen05 variant: the chunked-prefill GQA tile on the 5th-generation
// tensor cores with the accumulators in TMEM (included by prefill.cu inside
// namespace fs).
//
// Tile = NQ x 128 query rows (NQ*128 / q_per_kv chunk tokens x q_per_kv
// heads); each 128-row half is one UMMA M and has its own 4 softmax warps,
// so with NQ = 2 the K/V blocks in smem feed two independent S / P / O
// streams and the tensor pipe always has the other half's MMAs to run while
// one half is in softmax (FA4's two-tile ping-pong).  KV is consumed in
// blocks of 64 keys (4 pages).  Per block j and half h:
//     S_j[128 x 64]   = Q[128 x 128] . K_j^T     tcgen05.mma, bf16, -> TMEM
//     P_j             = exp2(S_j*scale - m)       softmax warps, bf16 hi + lo -> TMEM
//     O[128 x 128]   += P_j . V_j                 2 x tcgen05.mma (hi, lo), bf16, TMEM acc
// Roles (NQ*128 + 64 threads): warps 0..4NQ-1 = softmax / correction /
// epilogue (thread = row = TMEM lane; half h = warp / 4), warp 4NQ = TMA
// producer (each page = 4 bulk copies of
// 2 KB atoms, so the K / V blocks land as UMMA-canonical SWIZZLE_128B tiles:
// K as the K-major B of S, V as the MN-major B of P.V), warp 5 = MMA issuer
// (one thread) + TMEM owner.  S is double-buffered in TMEM so S_{j+2} is
// computed while the softmax warps work on S_{j+1}; the softmax warps store
// P (bf16 hi | lo halves) over S_j's columns and P.V_j reads its A operands from TMEM (no
// shared-memory round trip).  The running max is rescaled lazily (FA4): O and l are only
// rescaled when a row's max grows by more than 2^8 (P <= 256) and most
// blocks never touch O.  P is split into bf16 hi + lo (~16 mantissa bits;
// bf16 P alone costs ~1.5e-3 mean relative error at 4k context, over the
// north star's 1e-3) against the bf16 V pages, so P.V is two MMAs.
//
// TMEM (half h at column 256h): O at [0, 128), S buffers at [128, 192) and
// [192, 256).

constexpr int kTcRows = 128;                      // rows per Q half-tile (UMMA M)
constexpr int kTcQBytes = kTcRows * 256;          // 32 KB: 2 atoms x 128 rows x 128 B
// keys per block BK = 64 (4 pages) or 128 (8 pages); per BK: K/V ring depth
// and S buffers per half (TMEM: O 128 columns + kTcSBuf x BK per half)
// separate K and V rings: K_j is released once S_j ran, V_j once P.V_j ran,
// so K can run further ahead (S_{j+1} is issued before P.V_j's inputs are free)
template <int BK> constexpr int tc_kstages() { return BK == 64 ? 5 : 3; }
template <int BK> constexpr int tc_vstages() { return BK == 64 ? 5 : 2; }
template <int BK> constexpr int tc_sbuf() { return BK == 64 ? 2 : 1; }
template <int NQ, int BK>
constexpr int tc_smem() {
    return NQ * kTcQBytes + (tc_kstages<BK>() + tc_vstages<BK>()) * (BK * 256) + 1024 + 512;
}
constexpr float kTcRescale = 8.f;                 // lazy-rescale threshold (log2)

// kind::f16 instruction descriptors: D fp32; S: A = Q bf16 K-major, B = K
// bf16 K-major, M 128, N 64; PV: A = P bf16 K-major, B = V bf16 MN-major,
// M 128, N 128
template <int BK>
constexpr uint32_t tc_idesc_s() {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BK >> 3) << 17) | ((uint32_t)(kTcRows >> 4) << 24);
}
constexpr uint32_t kIdescPV = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) |
                              ((uint32_t)(kHeadDim >> 3) << 17) | ((uint32_t)(kTcRows >> 4) << 24);

__device__ __forceinline__ uint64_t tc_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
    d |= (uint64_t)2 << 61;  // SWIZZLE_128B
    return d;
}

__device__ __forceinline__ void tc_mma_f16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                           uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// D[tmem] (+)= A[tmem] . B[smem]: A (K-major, 2 f16 per 32-bit column) read
// straight from TMEM -- the softmax warps store P over their S columns
__device__ __forceinline__ void tc_mma_f16_ta(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                              uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}

__device__ __forceinline__ void tc_commit_bar(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     bar)
                 : "memory");
}

// one lane of the (converged) warp: true on exactly one lane
__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}"
                 : "=r"(pred));
    return pred != 0;
}

// packed fp32x2 arithmetic (FFMA2 / FADD2) and the 3-input max (FMNMX3) of
// sm_100: half the softmax's FMA-pipe instructions per element
__device__ __forceinline__ uint64_t f2(float a, float b) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void f2_split(uint64_t v, float &a, float &b) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
    uint64_t d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {
    float d;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}

// 2^x on the FMA pipe for a pair (FA4's MUFU offload): x = n + f with n =
// round(x), f in [-0.5, 0.5]; near-minimax cubic for 2^f (max rel err
// 7.5e-5, below f16's half ulp); n added to the exponent field.  x >= -125
// keeps that field positive (such P underflow to 0 in f16 anyway).
__device__ __forceinline__ void exp2_fma2(float x0, float x1, float &e0, float &e1) {
    const uint64_t x = f2(fmaxf(x0, -125.f), fmaxf(x1, -125.f));
    const uint64_t magic = f2(12582912.f, 12582912.f);  // 1.5 * 2^23
    const uint64_t t = fadd2(x, magic);
    const uint64_t r = fadd2(t, f2(-12582912.f, -12582912.f));  // round(x)
    const uint64_t f = fadd2(x, r ^ 0x8000000080000000ull);        // x - round(x)
    uint64_t p = ffma2(f2(0.05517166f, 0.05517166f), f, f2(0.24261114f, 0.24261114f));
    p = ffma2(p, f, f2(0.69326097f, 0.69326097f));
    p = ffma2(p, f, f2(0.99992806f, 0.99992806f));
    float t0, t1, p0, p1;
    f2_split(t, t0, t1);
    f2_split(p, p0, p1);
    e0 = __int_as_float(__float_as_int(p0) + (__float_as_int(t0) << 23));
    e1 = __int_as_float(__float_as_int(p1) + (__float_as_int(t1) << 23));
}

__device__ __forceinline__ void tc_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// 32 lanes x 32 consecutive fp32 columns (thread = lane = row)
__device__ __forceinline__ void tc_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
        "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
          "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
          "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
}

__device__ __forceinline__ void tc_st32(uint32_t taddr, const uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
        "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
        "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
        "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]),
        "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]),
        "r"(r[29]), "r"(r[30]), "r"(r[31])
        : "memory");
}

__device__ __forceinline__ void tc_st16(uint32_t taddr, const uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
        "%14,%15,%16};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
        "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}

__device__ __forceinline__ void tc_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tc_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void bulk_g2s_plain(uint32_t dst, const void *src, uint32_t bytes,
                                               uint32_t bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            dst),
        "l"(src), "r"(bytes), "r"(bar)
        : "memory");
}

template <int NQ, int BK>
__global__ void __launch_bounds__(NQ * 128 + 64, 1) prefill_tc_kernel(const PrefillParams p) {
    constexpr int kTcKeys = BK, kPB = BK / 16;        // keys / pages per block
    constexpr int kKS = tc_kstages<BK>(), kVS = tc_vstages<BK>(), kSBuf = tc_sbuf<BK>();
    constexpr int kTcKVBytes = BK * 256;              // K or V of a block: 2 atoms x BK rows x 128 B
    constexpr int kAtom = BK * 128;                   // one 64-dim atom of a block
    constexpr uint32_t kIdescS = tc_idesc_s<BK>();
    constexpr int kSoftWarps = 4 * NQ;
    constexpr int kTmemCols = 256 * NQ;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t sb = smem_u32(smem);
    const uint32_t q_s = sb;                                       // half h at + h*32K
    const uint32_t k_s = q_s + NQ * kTcQBytes;                     // K stage s at + s * kTcKVBytes
    const uint32_t v_s = k_s + kKS * kTcKVBytes;                   // V stage s at + s * kTcKVBytes
    const uint32_t bars = v_s + kVS * kTcKVBytes;
    const uint32_t k_full = bars, k_empty = k_full + 8 * kKS;
    const uint32_t v_full = k_empty + 8 * kKS, v_empty = v_full + 8 * kVS;
    // per half h and buffer b: barrier + 8 * (2h + b)
    const uint32_t s_full = v_empty + 8 * kVS;
    const uint32_t p_full = s_full + 16 * NQ, o_done = p_full + 16 * NQ, q_ready = o_done + 16 * NQ;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(smem + (q_ready + 8 - sb));

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int t = blockIdx.x;
    const int item = p.tile_item[t];
    const int tok0 = p.tile_tok0[t];
    const int pg0 = p.tile_page0[t];
    const int npg = p.tile_page1[t] - pg0;
    const int nb = (npg + kPB - 1) / kPB;  // key blocks
    // the item's parameters, loaded before the setup barrier so their
    // latency overlaps barrier init and the TMEM allocation
    const int it_seq = p.item_seq[item], it_start = p.item_start[item], it_len = p.item_len[item];
    const int it_qoff = p.item_qoff[item];

    if (threadIdx.x == 0) {
        for (int s = 0; s < kKS; ++s) {
            mbar_init(k_full + 8 * s, 1);
            mbar_init(k_empty + 8 * s, 1);
        }
        for (int s = 0; s < kVS; ++s) {
            mbar_init(v_full + 8 * s, 1);
            mbar_init(v_empty + 8 * s, 1);
        }
        for (int b = 0; b < 2 * NQ; ++b) {
            mbar_init(s_full + 8 * b, 1);
            mbar_init(p_full + 8 * b, 4);
            mbar_init(o_done + 8 * b, 1);
        }
        mbar_init(q_ready, kSoftWarps);
        fence_barrier_init();
    }
    if (warp == kSoftWarps + 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)), "n"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_before();
    __syncthreads();
    tc_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == kSoftWarps) {
        // ---------------- TMA producer ----------------
        const int64_t row = (int64_t)it_seq * p.bt_stride + pg0;
        // page ids 32 at a time (lane = page), the next 32 prefetched a
        // chunk ahead so the block-table load latency stays off the ring
        int64_t ids = lane < npg ? p.bt[row + lane] : 0;
        int64_t ids_next = 32 + lane < npg ? p.bt[row + 32 + lane] : 0;
        for (int j = 0; j < nb; ++j) {
            if (j > 0 && (j % (32 / kPB)) == 0) {
                ids = ids_next;
                const int k = kPB * j + 32 + lane;
                ids_next = k < npg ? p.bt[row + k] : 0;
            }
            const int np = min(kPB, npg - kPB * j);
            // lane l < 2 * np copies one 2 KB atom of K (then of V): page
            // l >> 1, atom l & 1
            const int pp = lane >> 1, a = lane & 1;
            const int64_t pg = __shfl_sync(0xffffffffu, ids, (kPB * j + pp) & 31);
            const uint8_t *src = p.kv + pg * kPageBytes + a * kAtomBytes;
            {
                const int st = j % kKS;
                if (j >= kKS) mbar_wait(k_empty + 8 * st, ((j / kKS) - 1) & 1);
                if (lane == 0) mbar_expect_tx(k_full + 8 * st, np * kHalfPage);
                __syncwarp();
                if (lane < 2 * np)
                    bulk_g2s_plain(k_s + st * kTcKVBytes + a * kAtom + pp * 2048, src, kAtomBytes,
                                   k_full + 8 * st);
            }
            {
                const int st = j % kVS;
                if (j >= kVS) mbar_wait(v_empty + 8 * st, ((j / kVS) - 1) & 1);
                const uint32_t vs = v_s + st * kTcKVBytes;
                if (np < kPB) {
                    // keys of missing pages are masked; their V rows must be finite
                    const int per_atom = (kPB - np) * 128;  // 16-byte chunks past page np-1
                    for (int c = lane; c < 2 * per_atom; c += 32) {
                        const int aa = c / per_atom, w = c - aa * per_atom;
                        reinterpret_cast<uint4 *>(smem + (vs - sb) + aa * kAtom + np * 2048)[w] =
                            make_uint4(0, 0, 0, 0);
                    }
                    fence_proxy_async();
                }
                if (lane == 0) mbar_expect_tx(v_full + 8 * st, np * kHalfPage);
                __syncwarp();
                if (lane < 2 * np)
                    bulk_g2s_plain(vs + a * kAtom + pp * 2048, src + kHalfPage, kAtomBytes, v_full + 8 * st);
            }
        }
        // consume the ring-slot releases of the last blocks (the MMA warp
        // commits them; they retire before o_done, so these waits return at
        // once): no barrier phase is left unconsumed at exit (synccheck)
        for (int j = max(nb - kKS, 0); j < nb; ++j) mbar_wait(k_empty + 8 * (j % kKS), (j / kKS) & 1);
        for (int j = max(nb - kVS, 0); j < nb; ++j) mbar_wait(v_empty + 8 * (j % kVS), (j / kVS) & 1);
    } else if (warp == kSoftWarps + 1) {
        // ---------------- MMA issuer ----------------
        // The whole warp runs the loop so descriptors and TMEM addresses are
        // warp-uniform (uniform datapath, no per-MMA R2UR waterfall); one
        // elected lane issues.  Issuing from lane 0 alone measured ~1.4x
        // slower than the tensor pipe (tools/ubench/mma_rate.cu, twohalf).
        mbar_wait(q_ready, 0);
        tc_after();
        // S_h(j) into buffer j % kSBuf of half h
        auto issue_s_half = [&](int j, int h) {
            const int b = j % kSBuf;
            const uint32_t ks = k_s + (j % kKS) * kTcKVBytes;
            // S_j overwrites the TMEM columns P_{j-kSBuf} occupied: the
            // tensor pipe runs this warp's MMAs in issue order, so
            // P.V_{j-kSBuf} (issued earlier) has read them
            tc_after();
            const uint32_t qh = q_s + h * kTcQBytes;
            const uint32_t s_t = tmem + 256 * h + kHeadDim + b * kTcKeys;
            if (elect_one()) {
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const uint64_t ad = tc_desc(qh + (k >> 2) * (kTcRows * 128) + (k & 3) * 32, 16, 1024);
                    const uint64_t bd = tc_desc(ks + (k >> 2) * kAtom + (k & 3) * 32, 16, 1024);
                    tc_mma_f16(s_t, ad, bd, kIdescS, k > 0);
                }
                tc_commit_bar(s_full + 8 * (2 * h + b));
                if (h == NQ - 1) tc_commit_bar(k_empty + 8 * (j % kKS));  // K_j read by S_j
            }
            __syncwarp();
        };
        auto wait_kv = [&](int j) { mbar_wait(k_full + 8 * (j % kKS), (j / kKS) & 1); };
        for (int j = 0; j < kSBuf && j < nb; ++j) {
            wait_kv(j);
#pragma unroll
            for (int h = 0; h < NQ; ++h) issue_s_half(j, h);
        }
        for (int j = 0; j < nb; ++j) {
            const int st = j % kVS, b = j % kSBuf;
            const uint32_t vs = v_s + st * kTcKVBytes;
            const bool more = j + kSBuf < nb;
            mbar_wait(v_full + 8 * st, (j / kVS) & 1);
#pragma unroll
            for (int h = 0; h < NQ; ++h) {
                mbar_wait(p_full + 8 * (2 * h + b), (j / kSBuf) & 1);
                tc_after();
                const uint32_t pt = tmem + 256 * h + kHeadDim + b * kTcKeys;  // P over S_j
                if (elect_one()) {
#pragma unroll
                    for (int k = 0; k < kTcKeys / 16; ++k) {
                        const uint64_t bd = tc_desc(vs + k * 2048, kAtom, 1024);
                        tc_mma_f16_ta(tmem + 256 * h, pt + k * 8, bd, kIdescPV, (j > 0 || k > 0) ? 1u : 0u);
                        tc_mma_f16_ta(tmem + 256 * h, pt + kTcKeys / 2 + k * 8, bd, kIdescPV, 1u);
                    }
                    tc_commit_bar(o_done + 8 * (2 * h + b));
                }
                __syncwarp();
                if (kSBuf == 1 && more) {
                    // one S buffer per half: S_h(j+1) right behind P.V_h(j),
                    // so half h's softmax restarts while the other half's
                    // MMAs run
                    if (h == 0) wait_kv(j + 1);
                    issue_s_half(j + 1, h);
                }
            }
            if (elect_one()) tc_commit_bar(v_empty + 8 * st);  // V_j read by P.V_j
            __syncwarp();
            if (kSBuf == 2 && more) {
                wait_kv(j + 2);
#pragma unroll
                for (int h = 0; h < NQ; ++h) issue_s_half(j + 2, h);
            }
        }
    } else {
        // ---------------- softmax / correction / epilogue (row = thread) ----------------
        const int h = warp >> 2;                          // Q half
        const int r = threadIdx.x & 127;                  // row within the half = TMEM lane
        const int R = h * kTcRows + r;                    // row within the tile
        const int qpk = p.qpk, rows_used = p.tpt * qpk;
        const int start = it_start, n = it_len;
        const int tl = min(R, rows_used - 1) / qpk;
        const int tok = min(tok0 + tl, n - 1);
        const int pos = start + tok;                     // causal limit of this row
        const int kv_lim = (pg0 + npg) * kPageTokens;    // keys past the range: masked
        // smallest row position of this half (rows of a half are in token order)
        const int pos_min = start + min(tok0 + min(h * kTcRows, rows_used - 1) / qpk, n - 1);
        const float scale = p.scale_log2;
        // ---- Q row -> smem (2 SW128 atoms of this half) ----
        {
            // the warp loads its 32 rows cooperatively, two 256-B rows per
            // instruction (rows of one token are adjacent heads: coalesced),
            // all 16 loads in flight before the swizzled smem stores
            const __nv_bfloat16 *qb = p.q + it_qoff;
            const int c = lane & 15;
            uint4 v[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const int Ri = h * kTcRows + (warp & 3) * 32 + 2 * i + (lane >> 4);
                const int tki = min(tok0 + min(Ri, rows_used - 1) / qpk, n - 1);
                v[i] = __ldg(reinterpret_cast<const uint4 *>(qb + (int64_t)tki * p.q_stride +
                                                             (Ri % qpk) * kHeadDim) + c);
            }
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const int ri = (warp & 3) * 32 + 2 * i + (lane >> 4);  // row within the half
                const uint32_t off = h * kTcQBytes + (c >> 3) * (kTcRows * 128) + ri * 128 +
                                     (((c & 7) ^ (ri & 7)) << 4);
                *reinterpret_cast<uint4 *>(smem + (q_s - sb) + off) = v[i];
            }
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) mbar_arrive_cta(q_ready);
        }
        const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
        const uint32_t o_t = tmem + 256 * h + lane_base, s_t = o_t + kHeadDim;
        float m_used = -INFINITY, l = 0.f;
        for (int j = 0; j < nb; ++j) {
            const int b = j % kSBuf, hb = 2 * h + b;
            mbar_wait(s_full + 8 * hb, (j / kSBuf) & 1);
            // consume o_done of block j - kSBuf: S_j was issued after that
            // block's P.V, so it has retired (returns at once) -- every
            // o_done phase is observed (the epilogue takes the last ones)
            if (j >= kSBuf) mbar_wait(o_done + 8 * hb, ((j - kSBuf) / kSBuf) & 1);
            tc_after();
            constexpr int kC = kTcKeys / 32;  // 32-column groups of S
            uint32_t sr[kC][32];
#pragma unroll
            for (int hh = 0; hh < kC; ++hh) tc_ld32(s_t + b * kTcKeys + 32 * hh, sr[hh]);
            tc_wait_ld();
            const int kb0 = (pg0 + kPB * j) * kPageTokens;
            // raw scores: the scale is folded into the exponent's FFMA; the
            // mask only runs on blocks crossing a row's diagonal or the range
            // end (warp-uniform test on the half's smallest row position)
            if (kb0 + kTcKeys - 1 > pos_min || kb0 + kTcKeys > kv_lim) {
#pragma unroll
                for (int hh = 0; hh < kC; ++hh)
#pragma unroll
                    for (int c = 0; c < 32; ++c) {
                        const int key = kb0 + hh * 32 + c;
                        if (key > pos || key >= kv_lim) sr[hh][c] = __float_as_uint(-INFINITY);
                    }
            }
            float mxs[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) mxs[i] = -INFINITY;
#pragma unroll
            for (int hh = 0; hh < kC; ++hh)
#pragma unroll
                for (int c = 0; c < 32; c += 2)
                    mxs[(c >> 1) & 3] = fmax3(mxs[(c >> 1) & 3], __uint_as_float(sr[hh][c]),
                                              __uint_as_float(sr[hh][c + 1]));
            const float mx = fmax3(fmaxf(mxs[0], mxs[1]), mxs[2], mxs[3]) * scale;
            float alpha = 1.f;
            const bool grow = mx > m_used + kTcRescale;
            if (grow) {
                alpha = m_used == -INFINITY ? 0.f : fast_exp2(m_used - mx);
                m_used = mx;
                l *= alpha;
            }
            const float mu = m_used == -INFINITY ? 0.f : m_used;
            uint64_t ls2[2] = {f2(0.f, 0.f), f2(0.f, 0.f)};
            const uint64_t scale2 = f2(scale, scale), nmu2 = f2(-mu, -mu);
            // P_j (bf16 hi in the first half of the S_j columns, lo in the
            // second; 2 keys per 32-bit column) over the S_j columns in
            // TMEM: the A operand of P.V_j; one 32-column S group -> 16
            // packed P columns at a time, so each group's registers die as
            // soon as it is stored
#pragma unroll
            for (int hh = 0; hh < kC; ++hh) {
                uint32_t pk[16], pl[16];
#pragma unroll
                for (int c = 0; c < 16; ++c) {
                    float x0, x1;
                    f2_split(ffma2(f2(__uint_as_float(sr[hh][2 * c]), __uint_as_float(sr[hh][2 * c + 1])),
                                   scale2, nmu2), x0, x1);
                    float e0, e1;
                    if (BK == 128 && (c & 3) == 3) {
                        exp2_fma2(x0, x1, e0, e1);  // a quarter of the pairs off the MUFU
                    } else {
                        e0 = fast_exp2(x0);
                        e1 = fast_exp2(x1);
                    }
                    const uint64_t e2 = f2(e0, e1);
                    ls2[c & 1] = fadd2(ls2[c & 1], e2);
                    split_bf16x2(e0, e1, pk[c], pl[c]);
                }
                tc_st16(s_t + b * kTcKeys + 16 * hh, pk);
                tc_st16(s_t + b * kTcKeys + kTcKeys / 2 + 16 * hh, pl);
            }
            tc_wait_st();
            float ls[4];
            f2_split(ls2[0], ls[0], ls[1]);
            f2_split(ls2[1], ls[2], ls[3]);
            if (j > 0 && __any_sync(0xffffffffu, grow)) {
                // rescale this warp's O rows once P_{j-1} . V_{j-1} landed
                // (after P_j is stored: S_j's registers are dead by now;
                // P.V_j waits for p_full below)
                mbar_wait(o_done + 8 * (2 * h + ((j - 1) % kSBuf)), ((j - 1) / kSBuf) & 1);
                tc_after();
#pragma unroll
                for (int cc = 0; cc < 4; ++cc) {
                    uint32_t ov[32];
                    tc_ld32(o_t + cc * 32, ov);
                    tc_wait_ld();
#pragma unroll
                    for (int c = 0; c < 32; ++c) ov[c] = __float_as_uint(__uint_as_float(ov[c]) * alpha);
                    tc_st32(o_t + cc * 32, ov);
                }
                tc_wait_st();
            }
            l += (ls[0] + ls[1]) + (ls[2] + ls[3]);
            tc_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cta(p_full + 8 * hb);
        }
        // ---- epilogue: O / l (or the split partial) ----
        grid_launch_dependents();  // the combine launch (PDL) may be scheduled now
        mbar_wait(o_done + 8 * (2 * h + ((nb - 1) % kSBuf)), ((nb - 1) / kSBuf) & 1);
        // (two S buffers: also consume the other buffer's last commit, which
        // retired earlier, so no barrier phase is left unconsumed at exit)
        if (kSBuf == 2 && nb >= 2) mbar_wait(o_done + 8 * (2 * h + ((nb - 2) % kSBuf)), ((nb - 2) / kSBuf) & 1);
        tc_after();
        const float inv = l > 0.f ? 1.f / l : 0.f;
        const int slot = p.tile_slot[t];
        const int rows = p.rows;
        // O / l -> this warp's 16 KB staging tile (fp32 rows of 512 B, 16-B
        // chunks XOR-swizzled by row), then the warp stores whole rows: a
        // thread-per-row store is 32 scattered 16-B pieces per instruction
        // and measured ~4.5 us per tile.  The staging tiles sit over Q and
        // the K ring, which every S MMA has finished reading once o_done
        // fired (the V ring may still feed the other half's last P.V).
        float *stg = reinterpret_cast<float *>(smem) + warp * 32 * kHeadDim;
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {
            uint32_t ov[32];
            tc_ld32(o_t + cc * 32, ov);
            tc_wait_ld();
#pragma unroll
            for (int c = 0; c < 8; ++c)
                reinterpret_cast<float4 *>(stg + lane * kHeadDim)[(cc * 8 + c) ^ (lane & 7)] =
                    make_float4(__uint_as_float(ov[4 * c]) * inv, __uint_as_float(ov[4 * c + 1]) * inv,
                                __uint_as_float(ov[4 * c + 2]) * inv, __uint_as_float(ov[4 * c + 3]) * inv);
        }
        __syncwarp();
        const int wrow0 = h * kTcRows + (warp & 3) * 32;  // tile row of this warp's lane 0
        for (int rr = 0; rr < 32; ++rr) {
            const float4 v = reinterpret_cast<const float4 *>(stg + rr * kHeadDim)[lane ^ (rr & 7)];
            const int Rr = wrow0 + rr;
            if (slot >= 0) {  // fp32 partial: 4 dims = 16 B per lane
                reinterpret_cast<float4 *>(p.part_o + ((int64_t)slot * rows + Rr) * kHeadDim)[lane] = v;
                continue;
            }
            const int tk = tok0 + Rr / qpk;
            if (Rr >= rows_used || tk >= n) continue;
            const int64_t o = p.item_ooff[item] + (int64_t)tk * p.o_stride + (Rr % qpk) * kHeadDim;
            if (p.out_fp32) {
                reinterpret_cast<float4 *>(static_cast<float *>(p.out) + o)[lane] = v;
            } else {
                uint2 pk;
                pk.x = pack_bf16(v.x, v.y);
                pk.y = pack_bf16(v.z, v.w);
                reinterpret_cast<uint2 *>(static_cast<__nv_bfloat16 *>(p.out) + o)[lane] = pk;
            }
        }
        if (slot >= 0) p.part_lse[(int64_t)slot * rows + R] = l > 0.f ? m_used + __log2f(l) : -INFINITY;
    }
    tc_before();
    __syncthreads();
    if (warp == kSoftWarps + 1) {
        tc_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kTmemCols));
    }
}
