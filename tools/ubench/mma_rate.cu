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
__global__ void __launch_bounds__(128, 1) mixed(long long *out, int iters, int commit_every) {
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
                             ::"r"(tmem + 256), "l"(ad), "l"(bd), "r"(idS), "r"(1) : "memory");
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

void run_mixed(int commit_every) {
    long long *d;
    cudaMalloc(&d, 1024 * sizeof(long long));
    const int iters = 1000, smem = 100 * 1024;
    cudaFuncSetAttribute(mixed, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    mixed<<<148, 128, smem>>>(d, 10, commit_every);
    mixed<<<148, 128, smem>>>(d, iters, commit_every);
    cudaError_t e = cudaDeviceSynchronize();
    long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("mixed 4xPV(N128,tmemA)+8xS(N64) commits=%d: %s  %.0f cyc per group (ideal 640)\n",
           commit_every, cudaGetErrorString(e), (double)h / iters);
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
    return 0;
}
