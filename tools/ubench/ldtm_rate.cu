// Microbenchmark: tcgen05.ld (32x32b.x32) throughput per SM with 4 or 8 warps.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 1) k(long long *out, float *sink, int iters) {
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tslot + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * 256;
    float acc = 0.f;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        uint32_t r[32];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
                "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                  "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
                  "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
                  "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
                  "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                : "r"(tmem + c * 32));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int i = 0; i < 32; ++i) acc += __uint_as_float(r[i]);
        }
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    if (acc == 1234.5f) sink[threadIdx.x] = acc;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tslot));
}

template <int W>
void run() {
    long long *d; float *s;
    cudaMalloc(&d, 148 * 8); cudaMalloc(&s, 4096);
    const int iters = 4000;
    k<W><<<148, W * 32>>>(d, s, 10);
    k<W><<<148, W * 32>>>(d, s, iters);
    cudaError_t e = cudaDeviceSynchronize();
    long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    const double bytes = (double)iters * W * 32 * 64 * 4;  // per CTA
    printf("%d warps: %s  %.1f B/clk/SM  (%.1f cyc per 64-col x 32-lane warp load)\n", W,
           cudaGetErrorString(e), bytes / h, (double)h / (iters * 2.0) );
}
int main() { run<4>(); run<8>(); return 0; }
