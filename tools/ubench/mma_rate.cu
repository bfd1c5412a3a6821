// Microbenchmark: issue rate / throughput of tcgen05.mma.cta_group::1.kind::f16
// for the shapes K8 uses (one CTA per SM, one issuing thread, operands in smem,
// accumulator in TMEM).  Usage: ./mma_rate
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}

__device__ volatile int g_stop;

template <int N, int ACC_CHAINS, bool A_TMEM, bool LD = false>
__global__ void __launch_bounds__(256, 1) k(long long *out, int iters) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t bar;
    const uint32_t sb = (uint32_t)__cvta_generic_to_shared(smem);
    const uint32_t sb_al = (sb + 1023) & ~1023u;
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tslot;
    constexpr uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
    if (threadIdx.x == 0) {
        const uint32_t a = sb_al, b = sb_al + 32768;
        long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                const uint32_t d = tmem + (uint32_t)((kk % ACC_CHAINS) * N);
                const uint64_t bd = desc(b + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024);
                if (A_TMEM) {
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
                                 ::"r"(d), "r"(tmem + 384 + kk * 8), "l"(bd), "r"(idesc), "r"(1) : "memory");
                } else {
                    const uint64_t ad = desc(a + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024);
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                                 ::"r"(d), "l"(ad), "l"(bd), "r"(idesc), "r"(1) : "memory");
                }
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&bar)) : "memory");
        asm volatile("{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n}"
                     ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
        long long t1 = clock64();
        out[blockIdx.x] = t1 - t0;
        __threadfence_block();
        g_stop = 1;
    } else if (LD && threadIdx.x >= 128) {
        // interference: 4 warps stream tcgen05.ld over columns 256..319
        const uint32_t t = tmem + ((uint32_t)(((threadIdx.x >> 5) & 3) * 32) << 16) + 256;
        uint32_t acc = 0;
        for (int it = 0; it < iters * 4 && !g_stop; ++it) {
            uint32_t r[32];
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
                "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                  "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
                  "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
                  "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
                  "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                : "r"(t));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            for (int i = 0; i < 32; ++i) acc += r[i];
        }
        if (acc == 12345) out[1000] = acc;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// K8's per-half sequence: 4 x P.V (N128, A in TMEM, B MN-major) then 8 x S
// (N64, A/B in smem, K-major), repeated
__global__ void __launch_bounds__(128, 1) mixed(long long *out, int iters, int commit_every, int overlap) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t bar;
    const uint32_t sb = (uint32_t)__cvta_generic_to_shared(smem);
    const uint32_t sb_al = (sb + 1023) & ~1023u;
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tslot;
    constexpr uint32_t idS = (1u << 4) | (1u << 7) | (1u << 10) | (8u << 17) | (8u << 24);
    constexpr uint32_t idPV = (1u << 4) | (1u << 16) | (16u << 17) | (8u << 24);
    uint32_t phase = 0;
    if (threadIdx.x == 0) {
        const uint32_t a = sb_al, b = sb_al + 32768, v = sb_al + 49152;
        long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                const uint64_t bd = desc(v + kk * 2048, 8192, 1024);
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
                             ::"r"(tmem), "r"(tmem + 128 + kk * 8), "l"(bd), "r"(idPV), "r"(1) : "memory");
            }
            if (commit_every) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                (uint32_t)__cvta_generic_to_shared(&bar)) : "memory");
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                const uint64_t ad = desc(a + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024);
                const uint64_t bd = desc(b + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024);
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                             ::"r"(tmem + (overlap ? 128u : 256u)), "l"(ad), "l"(bd), "r"(idS), "r"(1) : "memory");
            }
            if (commit_every) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                (uint32_t)__cvta_generic_to_shared(&bar)) : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&bar)) : "memory");
        // wait for the last commit's phase: count commits
        const int commits = (commit_every ? 2 * iters : 0) + 1;
        phase = (commits - 1) & 1;
        asm volatile("{\n\t.reg .pred p;\nW2:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W2;\n}"
                     ::"r"((uint32_t)__cvta_generic_to_shared(&bar)), "r"(phase));
        long long t1 = clock64();
        out[blockIdx.x] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// K8's block order with both halves: PV h0, PV h1 (A = P in TMEM buffer b),
// then S h0, S h1 written into buffer b (mode 0: over the P just read, as
// K8 does) or buffer b^1 (mode 1)
__global__ void __launch_bounds__(128, 1) twohalf(long long *out, int iters, int mode, const uint8_t *gsrc) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ __align__(8) uint64_t cbar[4];
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t bar;
    const uint32_t sb = (uint32_t)__cvta_generic_to_shared(smem);
    const uint32_t sb_al = (sb + 1023) & ~1023u;
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
        for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&cbar[i])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tslot;
    constexpr uint32_t idS = (1u << 4) | (1u << 7) | (1u << 10) | (8u << 17) | (8u << 24);
    constexpr uint32_t idPV = (1u << 4) | (1u << 16) | (16u << 17) | (8u << 24);
    if (mode & 2) {
        // random bf16 / f16 operands in [-2, 2]
        uint32_t *w = reinterpret_cast<uint32_t *>(smem + (sb_al - sb));
        for (int i = threadIdx.x; i < 100 * 1024 / 4; i += blockDim.x) {
            uint32_t x = i * 2654435761u + 12345u;
            x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
            w[i] = (x & 0xbfffbfffu) | 0x3c003c00u;  // exponents near 1
        }
        asm volatile("fence.proxy.async.shared::cta;");
        // random P in TMEM columns 128..255 and 384..511
        const uint32_t lane_base = (uint32_t)((threadIdx.x >> 5) * 32) << 16;
        for (int c = 0; c < 8; ++c) {
            uint32_t r[16];
            for (int i = 0; i < 16; ++i) { uint32_t x = (threadIdx.x * 131 + c * 16 + i) * 2654435761u; x ^= x >> 13; r[i] = (x & 0x3bff3bffu) | 0x30003000u; }
            for (int h = 0; h < 2; ++h)
            asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                         ::"r"(tmem + lane_base + 256 * h + 128 + c * 16), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
                           "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]));
        }
        asm volatile("tcgen05.wait::st.sync.aligned;");
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;");
    }
    if ((mode & 4) && threadIdx.x == 32) {
        // a TMA-like producer: 2 KB bulk copies into a separate 64 KB region
        __shared__ __align__(8) uint64_t tbar;
        const uint32_t tb = (uint32_t)__cvta_generic_to_shared(&tbar);
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(tb));
        asm volatile("fence.mbarrier_init.release.cluster;");
        const uint32_t dst = sb_al + 131072;
        uint32_t ph = 0;
        for (int it = 0; !g_stop && it < iters * 4; ++it) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tb), "r"(16384));
            for (int c = 0; c < 8; ++c)
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 2048, [%2];"
                             ::"r"(dst + (it & 3) * 16384 + c * 2048), "l"(gsrc + ((size_t)(blockIdx.x * 64 + it % 64) * 16384) + c * 2048), "r"(tb) : "memory");
            asm volatile("{\n\t.reg .pred p;\nW4:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W4;\n}" ::"r"(tb), "r"(ph));
            ph ^= 1;
        }
    }
    if (threadIdx.x == 0) {
        const uint32_t a = sb_al, b = sb_al + 65536, v = sb_al + 81920;
        long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            const uint32_t bb = it & 1;
            for (int h = 0; h < 2; ++h) {
                if (mode & 8) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                    const uint64_t bd = desc(v + kk * 2048, 8192, 1024);
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
                                 ::"r"(tmem + 256 * h), "r"(tmem + 256 * h + 128 + bb * 64 + kk * 8), "l"(bd), "r"(idPV), "r"(1) : "memory");
                }
                if (mode & 16) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                    (uint32_t)__cvta_generic_to_shared(&cbar[h])) : "memory");
            }
            const uint32_t sbuf = mode == 0 ? bb : (bb ^ 1);
            for (int h = 0; h < 2; ++h) {
                if (mode & 8) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint64_t ad = desc(a + h * 32768 + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024);
                    const uint64_t bd = desc(b + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024);
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                                 ::"r"(tmem + 256 * h + 128 + sbuf * 64), "l"(ad), "l"(bd), "r"(idS), "r"((uint32_t)(kk > 0)) : "memory");
                }
                if (mode & 16) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                    (uint32_t)__cvta_generic_to_shared(&cbar[2 + h])) : "memory");
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&bar)) : "memory");
        asm volatile("{\n\t.reg .pred p;\nW3:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W3;\n}"
                     ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
        long long t1 = clock64();
        out[blockIdx.x] = t1 - t0;
        g_stop = 1;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

void run_twohalf(int mode) {
    long long *d;
    cudaMalloc(&d, 1024 * sizeof(long long));
    const int iters = 1000, smem = 200 * 1024;
    static uint8_t *g = nullptr;
    if (!g) { cudaMalloc(&g, (size_t)148 * 64 * 16384); cudaMemset(g, 0x3c, (size_t)148 * 64 * 16384); }
    int zero = 0;
    cudaFuncSetAttribute(twohalf, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaMemcpyToSymbol(g_stop, &zero, sizeof(int));
    twohalf<<<148, 128, smem>>>(d, 10, mode, g);
    cudaMemcpyToSymbol(g_stop, &zero, sizeof(int));
    twohalf<<<148, 128, smem>>>(d, iters, mode, g);
    cudaError_t e = cudaDeviceSynchronize();
    long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("two halves PVh0 PVh1 Sh0 Sh1, S %s%s%s%s%s: %s  %.0f cyc per block (ideal 1280)\n",
           (mode & 1) ? "into the other buffer" : "over the P just read (K8)", (mode & 2) ? " +random data" : "",
           (mode & 4) ? " +bulk copies" : "", (mode & 8) ? " +fence::after_thread_sync" : "", (mode & 16) ? " +commits" : "", cudaGetErrorString(e), (double)h / iters);
    cudaFree(d);
}

__device__ __forceinline__ uint32_t elect_one() {
    uint32_t pred = 0;
    asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}" : "=r"(pred));
    return pred;
}

// twohalf with the whole warp running the issue loop (uniform operands) and
// elect.sync picking the issuing lane
__global__ void __launch_bounds__(128, 1) twohalf_warp(long long *out, int iters) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t bar;
    __shared__ __align__(8) uint64_t cbar[4];
    const uint32_t sb = (uint32_t)__cvta_generic_to_shared(smem);
    const uint32_t sb_al = (sb + 1023) & ~1023u;
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
        for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&cbar[i])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tslot;
    constexpr uint32_t idS = (1u << 4) | (1u << 7) | (1u << 10) | (8u << 17) | (8u << 24);
    constexpr uint32_t idPV = (1u << 4) | (1u << 16) | (16u << 17) | (8u << 24);
    if (threadIdx.x < 32) {
        const uint32_t a = sb_al, b = sb_al + 65536, v = sb_al + 81920;
        long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            const uint32_t bb = it & 1;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                if (elect_one()) {
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        const uint64_t bd = desc(v + kk * 2048, 8192, 1024);
                        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                     "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
                                     ::"r"(tmem + 256 * h), "r"(tmem + 256 * h + 128 + bb * 64 + kk * 8), "l"(bd), "r"(idPV), "r"(1) : "memory");
                    }
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                        (uint32_t)__cvta_generic_to_shared(&cbar[h])) : "memory");
                }
                __syncwarp();
            }
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                if (elect_one()) {
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk) {
                        const uint64_t ad = desc(a + h * 32768 + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024);
                        const uint64_t bd = desc(b + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024);
                        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                                     ::"r"(tmem + 256 * h + 128 + bb * 64), "l"(ad), "l"(bd), "r"(idS), "r"((uint32_t)(kk > 0)) : "memory");
                    }
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                        (uint32_t)__cvta_generic_to_shared(&cbar[2 + h])) : "memory");
                }
                __syncwarp();
            }
        }
        if (elect_one()) {
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                (uint32_t)__cvta_generic_to_shared(&bar)) : "memory");
        }
        __syncwarp();
        asm volatile("{\n\t.reg .pred p;\nW5:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W5;\n}"
                     ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
        long long t1 = clock64();
        if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

void run_twohalf_warp() {
    long long *d;
    cudaMalloc(&d, 1024 * sizeof(long long));
    const int iters = 1000, smem = 200 * 1024;
    cudaFuncSetAttribute(twohalf_warp, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    twohalf_warp<<<148, 128, smem>>>(d, 10);
    twohalf_warp<<<148, 128, smem>>>(d, iters);
    cudaError_t e = cudaDeviceSynchronize();
    long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("two halves, whole-warp uniform issue + elect.sync: %s  %.0f cyc per block (ideal 1280)\n",
           cudaGetErrorString(e), (double)h / iters);
    cudaFree(d);
}

void run_mixed(int commit_every, int overlap = 0) {
    long long *d;
    cudaMalloc(&d, 1024 * sizeof(long long));
    const int iters = 1000, smem = 100 * 1024;
    cudaFuncSetAttribute(mixed, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    mixed<<<148, 128, smem>>>(d, 10, commit_every, overlap);
    mixed<<<148, 128, smem>>>(d, iters, commit_every, overlap);
    cudaError_t e = cudaDeviceSynchronize();
    long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("mixed 4xPV(N128,tmemA)+8xS(N64) commits=%d S-over-P=%d: %s  %.0f cyc per group (ideal 640)\n",
           commit_every, overlap, cudaGetErrorString(e), (double)h / iters);
    cudaFree(d);
}

template <int N, int C, bool AT, bool LD = false>
void run(const char *name) {
    long long *d;
    cudaMalloc(&d, 1024 * sizeof(long long));
    const int iters = 2000, smem = 80 * 1024;
    cudaFuncSetAttribute(k<N, C, AT, LD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int zero = 0;
    cudaMemcpyToSymbol(g_stop, &zero, sizeof(int));
    k<N, C, AT, LD><<<148, 256, smem>>>(d, 10);
    cudaMemcpyToSymbol(g_stop, &zero, sizeof(int));
    k<N, C, AT, LD><<<148, 256, smem>>>(d, iters);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    const double per = (double)h[0] / (iters * 8.0);
    const double macs = 128.0 * N * 16;
    printf("%-28s %s cycles/mma %7.1f  MAC/clk/SM %7.0f\n", name, cudaGetErrorString(e), per, macs / per);
    cudaFree(d);
}

int main() {
    run<64, 1, false>("N64 smemA 1 chain");
    run<64, 4, false>("N64 smemA 4 chains");
    run<64, 1, true>("N64 tmemA 1 chain");
    run<128, 1, false>("N128 smemA 1 chain");
    run<128, 2, false>("N128 smemA 2 chains");
    run<128, 1, true>("N128 tmemA 1 chain");
    run<256, 1, false>("N256 smemA 1 chain");
    run<64, 1, false, true>("N64 smemA + LDTM 4 warps");
    run<128, 1, true, true>("N128 tmemA + LDTM 4 warps");
    run_mixed(0);
    run_mixed(1);
    run_mixed(0, 1);
    run_twohalf(0);
    run_twohalf(1);
    run_twohalf(24);
    run_twohalf_warp();
    return 0;
}
