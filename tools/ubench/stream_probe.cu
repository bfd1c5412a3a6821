// Per-SM HBM streaming probe: G CTAs (one per SM, forced by shared memory),
// each streaming its own contiguous region through a ring of S slots of B
// bytes filled by cp.async.bulk (one producer thread, slots recycled as soon
// as they land).  Reports per-CTA and aggregate GB/s for a sweep of (G, S, B),
// to tell whether one SM's stream is capped (and at what in-flight depth).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_probe stream_probe.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__global__ void stream_kernel(const uint8_t *src, int64_t per_cta, int S, int B, int split,
                              unsigned long long *t) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ __align__(8) uint64_t bars[32];
    const int nprod = split;  // producer threads (each owns S/split slots)
    if (threadIdx.x < S) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[threadIdx.x])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    unsigned long long t0;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
    const uint8_t *base = src + (int64_t)blockIdx.x * per_cta;
    const int64_t chunks = per_cta / B;
    if (threadIdx.x < nprod && (threadIdx.x & 0) == 0) {
        // producer p owns slots p, p+nprod, ... and chunks p, p+nprod, ...
        const int p = threadIdx.x;
        const int my_slots = S / nprod;
        uint32_t phase[32];
        for (int i = 0; i < 32; ++i) phase[i] = 0;
        int64_t c = p;
        // prime
        for (int i = 0; i < my_slots && c < chunks; ++i, c += nprod) {
            const int s = p + i * nprod;
            const uint32_t bar = smem_u32(&bars[s]);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(B) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(smem_u32(smem + (int64_t)s * B)), "l"(base + c * B), "r"(B), "r"(bar) : "memory");
        }
        int i = 0;
        for (int64_t d = p; d < chunks; d += nprod) {
            const int s = p + i * nprod;
            const uint32_t bar = smem_u32(&bars[s]);
            asm volatile(
                "{\n\t.reg .pred q;\nW_%=:\n\t"
                "mbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1;\n\t"
                "@!q bra W_%=;\n}" ::"r"(bar), "r"(phase[i]) : "memory");
            phase[i] ^= 1u;
            if (c < chunks) {
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(B) : "memory");
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                             ::"r"(smem_u32(smem + (int64_t)s * B)), "l"(base + c * B), "r"(B), "r"(bar) : "memory");
                c += nprod;
            }
            if (++i == my_slots) i = 0;
        }
    }
    __syncthreads();
    unsigned long long t1;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t1));
    if (threadIdx.x == 0) { t[2 * blockIdx.x] = t0; t[2 * blockIdx.x + 1] = t1; }
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int64_t total = 4ll << 30;  // 4 GiB source (>> L2)
    uint8_t *src;
    cudaMalloc(&src, total);
    cudaMemset(src, 1, total);
    unsigned long long *t;
    cudaMalloc(&t, 2 * 1024 * sizeof(unsigned long long));
    cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    std::vector<unsigned long long> h(2 * 1024);
    const int grids[] = {1, 8, 32, 64, 96, 128, 148};
    struct Cfg { int S, B, split; } cfgs[] = {
        {4, 8192, 1}, {8, 8192, 1}, {16, 8192, 1}, {4, 16384, 1}, {8, 16384, 1},
        {12, 16384, 1}, {8, 16384, 4}, {6, 32768, 1}, {4, 49152, 1}, {16, 8192, 4}, {24, 8192, 4}};
    printf("grid,S,B,split,inflight_KB,per_cta_MB,mean_cta_GBs,min_cta_GBs,max_cta_GBs,agg_GBs\n");
    for (int G : grids) {
        for (auto cf : cfgs) {
            const int64_t per_cta = ((int64_t)std::min<int64_t>(total / G, 64ll << 20) / cf.B) * cf.B;
            const int64_t per = std::min<int64_t>(per_cta, (int64_t)(G <= 32 ? (16ll << 20) : (8ll << 20)));
            const int64_t p2 = (per / cf.B) * cf.B;
            size_t smem = (size_t)cf.S * cf.B + 1024;
            for (int rep = 0; rep < 3; ++rep) {
                cudaEvent_t e0, e1;
                cudaEventCreate(&e0); cudaEventCreate(&e1);
                // flush L2 by touching a different region
                cudaMemsetAsync(src + (3ll << 30), rep, 512ll << 20);
                cudaEventRecord(e0);
                stream_kernel<<<G, 32, smem>>>(src, p2, cf.S, cf.B, cf.split, t);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms; cudaEventElapsedTime(&ms, e0, e1);
                cudaMemcpy(h.data(), t, 2 * G * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
                double mn = 1e30, mx = 0, sum = 0;
                unsigned long long lo = ~0ull, hi = 0;
                for (int i = 0; i < G; ++i) {
                    double ns = (double)(h[2 * i + 1] - h[2 * i]);
                    double gbs = p2 / ns;
                    mn = std::min(mn, gbs); mx = std::max(mx, gbs); sum += gbs;
                    lo = std::min(lo, h[2 * i]); hi = std::max(hi, h[2 * i + 1]);
                }
                if (rep == 2)
                    printf("%d,%d,%d,%d,%d,%.1f,%.1f,%.1f,%.1f,%.1f\n", G, cf.S, cf.B, cf.split,
                           cf.S * cf.B / 1024, p2 / 1048576.0, sum / G, mn, mx,
                           (double)p2 * G / (double)(hi - lo));
                cudaEventDestroy(e0); cudaEventDestroy(e1);
            }
        }
    }
    cudaError_t e = cudaGetLastError();
    printf("err=%s sms=%d\n", cudaGetErrorString(e), sms);
    return 0;
}
