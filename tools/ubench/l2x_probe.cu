// Does the activation (x) traffic of the skinny GEMM cost weight bandwidth?
// G CTAs stream their own W region (HBM, 32 KB bulk copies) and, per W copy,
// an x copy of r * 32 KB from a small L2-resident buffer shared by all CTAs
// (as the GEMM's per-stage x tiles).  Aggregate W GB/s for r = 0, 1/4, 1/2.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2x_probe l2x_probe.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__global__ void probe(const uint8_t *w, int64_t per_cta, const uint8_t *x, int64_t x_bytes,
                      int xb, unsigned long long *t) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ __align__(8) uint64_t bars[4];
    constexpr int S = 4, WB = 32768;
    if (threadIdx.x < S) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[threadIdx.x])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    unsigned long long t0;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
    if (threadIdx.x == 0) {
        const uint8_t *base = w + (int64_t)blockIdx.x * per_cta;
        const int64_t n = per_cta / WB;
        uint32_t ph[S] = {0, 0, 0, 0};
        int64_t xo = xb ? (int64_t)blockIdx.x * 8192 % (x_bytes - xb) : 0;
        auto issue = [&](int s, int64_t c) {
            const uint32_t bar = smem_u32(&bars[s]);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(WB + xb) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(smem_u32(smem + s * (WB + 16384))), "l"(base + c * WB), "r"(WB), "r"(bar) : "memory");
            if (xb) {
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                             ::"r"(smem_u32(smem + s * (WB + 16384) + WB)), "l"(x + xo), "r"(xb), "r"(bar) : "memory");
                xo += xb;
                if (xo + xb > x_bytes) xo = 0;
            }
        };
        int64_t c = 0;
        for (int s = 0; s < S && c < n; ++s, ++c) issue(s, c);
        for (int64_t d = 0; d < n; ++d) {
            const int s = d % S;
            const uint32_t bar = smem_u32(&bars[s]);
            asm volatile("{\n\t.reg .pred q;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1;\n\t@!q bra W_%=;\n}"
                         ::"r"(bar), "r"(ph[s]) : "memory");
            ph[s] ^= 1u;
            if (c < n) { issue(s, c); ++c; }
        }
    }
    __syncthreads();
    unsigned long long t1;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t1));
    if (threadIdx.x == 0) { t[2 * blockIdx.x] = t0; t[2 * blockIdx.x + 1] = t1; }
}

int main() {
    const int64_t total = 4ll << 30;
    uint8_t *w, *x;
    cudaMalloc(&w, total);
    cudaMemset(w, 1, total);
    const int64_t x_bytes = 1 << 20;  // L2-resident activations
    cudaMalloc(&x, x_bytes);
    cudaMemset(x, 2, x_bytes);
    unsigned long long *t;
    cudaMalloc(&t, 2 * 1024 * sizeof(unsigned long long));
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    std::vector<unsigned long long> h(2 * 1024);
    printf("ctas,x_per_w,w_agg_GBs,x_agg_GBs\n");
    for (int G : {112, 128, 148}) {
        for (int xb : {0, 8192, 16384}) {
            const int64_t per = 1 << 20;  // 1 MB of W per CTA
            for (int rep = 0; rep < 3; ++rep) {
                cudaMemsetAsync(w + (3ll << 30), rep, 512ll << 20);  // evict
                probe<<<G, 32, 4 * (32768 + 16384) + 1024>>>(w, per, x, x_bytes, xb, t);
                cudaDeviceSynchronize();
                cudaMemcpy(h.data(), t, 2 * G * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
                unsigned long long lo = ~0ull, hi = 0;
                for (int i = 0; i < G; ++i) { lo = std::min(lo, h[2 * i]); hi = std::max(hi, h[2 * i + 1]); }
                const double ns = (double)(hi - lo);
                if (rep == 2)
                    printf("%d,%.2f,%.1f,%.1f\n", G, xb / 32768.0, per * (double)G / ns,
                           per / 32768.0 * xb * G / ns);
            }
        }
    }
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
