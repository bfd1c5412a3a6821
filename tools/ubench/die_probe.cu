// Probe: load latency from one SM to every 4 KB chunk of a buffer, to see
// whether B200's two dies show up as an address -> "near / far" pattern.
// One launch per target SM (the CTA on that SM does the work, others exit),
// L2 flushed between launches.  Output: CSV sm,chunk,cycles.
#include <cstdio>
#include <cstdint>
#include <vector>

__global__ void probe(const uint64_t *buf, int64_t n_chunks, int64_t stride_words, int target,
                      uint32_t *lat) {
    uint32_t sm;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    if ((int)sm != target || threadIdx.x != 0) return;
    uint64_t acc = 0;
    for (int64_t j = 0; j < n_chunks; ++j) {
        const uint64_t *p = buf + j * stride_words + (acc & 1);  // acc is 0: keeps the dependency
        long long t0 = clock64();
        uint64_t v;
        asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
        acc += v;
        long long t1 = clock64();
        lat[j] = (uint32_t)(t1 - t0);
    }
    if (acc == 12345) lat[0] = 0;
}

__global__ void flush(uint4 *f, int64_t n) {
    for (int64_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        f[i] = make_uint4(i, 0, 0, 0);
}

int main(int argc, char **argv) {
    const int64_t chunk = 4096, n_chunks = argc > 1 ? atoll(argv[1]) : 8192;
    const int n_targets = 8;
    const int targets[n_targets] = {0, 1, 2, 36, 73, 74, 110, 147};
    uint64_t *buf;
    cudaMalloc(&buf, n_chunks * chunk);
    cudaMemset(buf, 0, n_chunks * chunk);
    uint4 *f;
    const int64_t fn = (512ll << 20) / 16;
    cudaMalloc(&f, fn * 16);
    uint32_t *lat;
    cudaMalloc(&lat, n_chunks * 4);
    std::vector<uint32_t> h(n_chunks);
    printf("sm,chunk,cycles\n");
    for (int t = 0; t < n_targets; ++t) {
        flush<<<592, 512>>>(f, fn);
        probe<<<148 * 4, 32>>>(buf, n_chunks, chunk / 8, targets[t], lat);
        cudaMemcpy(h.data(), lat, n_chunks * 4, cudaMemcpyDeviceToHost);
        for (int64_t j = 0; j < n_chunks; ++j) printf("%d,%lld,%u\n", targets[t], (long long)j, h[j]);
    }
    return 0;
}
