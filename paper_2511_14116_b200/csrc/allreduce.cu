// The exchange step of the hybrid decode step (the reference's ordered sum of
// the per-rank partials, refexec.py:283-307) as ONE kernel over peer memory:
// every rank's projection GEMM writes its partial straight into a symmetric
// buffer (cudaMalloc'd, shared with the peers by CUDA IPC, mapped over
// NVLink / NVSwitch), and fs_ar_residual then
//   1. publishes "my partial is ready" to every peer (a release store of the
//      buffer's use counter into each peer's flag slot for this rank),
//   2. waits until every peer's flag reached this use (acquire loads),
//   3. reads the partials of all ranks IN RANK ORDER, sums them in fp32,
//      rounds once to bf16 and adds them to the residual stream x in place:
//      x += bf16(sum_r partial_r) -- the reference's exact ordered sum, and
//      bit-identical on every rank (unlike a ring / tree all-reduce).
// No second barrier: a caller alternates two buffers between consecutive
// exchanges (attention / MLP), and a rank can only rewrite buffer A after
// its exchange on buffer B passed its barrier, i.e. after every peer
// finished reading A.  The use counter and flags live in device memory, so
// the launch is CUDA-graph capturable.  A peer that never arrives makes the
// kernel trap after 20 s instead of hanging the GPU.
//
// Two forms, the same bits:
//   one-shot: every rank reads every peer's whole partial (N-1 remote reads
//     of the vector per rank; one flag round) -- lowest latency, for small
//     vectors or two ranks;
//   two-shot: rank r sums only ITS 1/N slice over all ranks (in rank order,
//     fp32, one bf16 rounding) into the sum area of its own buffer, the last
//     CTA releases a second flag, and every rank then gathers the rounded
//     slices from their owners and adds them to x -- (N-1)/N of the vector
//     read twice instead of N-1 times (8 GPUs: 1.75 vs 7 vectors of NVLink
//     reads), for one more flag round.  The summation order per element is
//     the one-shot's, so x is bit-identical either way.
// Buffer layout: [partial: D bytes][slice sums: D bytes][flags: 256 bytes],
// data_bytes = 2D = the flag offset.
#include <cuda_bf16.h>

#include <cstdlib>
#include <cstring>

#include "common.cuh"

namespace fs {

constexpr int64_t kSpinNs = 20000000000LL;  // 20 s

struct ArParams {
    uint8_t *peer[FS_AR_MAX_WORLD];
    int32_t rank, world;
    int64_t n;          // bf16 elements (multiple of 8)
    int64_t data_bytes; // offset of the flag area inside every buffer
    __nv_bfloat16 *x;
};

// flag area words: [0, 16) partial-ready flags per rank, 16 use counter,
// 17 CTA-done counter, [32, 48) slice-sum-ready flags per rank (two-shot),
// 48 two-shot phase-1 CTA-done counter
constexpr int kFlagSums = 32;
constexpr int kDone1 = 48;

__device__ __forceinline__ void st_release_sys(uint32_t *p, uint32_t v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long now_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// flag area of a buffer: [FS_AR_MAX_WORLD] arrival flags, then the use
// counter and the CTA-done counter
__device__ __forceinline__ uint32_t *flags_of(uint8_t *buf, int64_t data_bytes) {
    return reinterpret_cast<uint32_t *>(buf + data_bytes);
}

__global__ void __launch_bounds__(256) ar_residual_kernel(const ArParams p) {
    __shared__ uint32_t s_use;
    // programmatic dependent launch: the next projection's CTAs may start
    // staging their weights while this exchange waits for the peers; this
    // kernel's own reads (the partial, x) wait for the producing GEMM
    grid_launch_dependents();
    grid_dependency_wait();
    uint32_t *mine = flags_of(p.peer[p.rank], p.data_bytes);
    uint32_t *use_ctr = mine + FS_AR_MAX_WORLD, *done_ctr = use_ctr + 1;
    if (threadIdx.x == 0) s_use = *reinterpret_cast<volatile uint32_t *>(use_ctr) + 1u;
    __syncthreads();
    const uint32_t use = s_use;
    if (blockIdx.x == 0 && threadIdx.x < p.world) {
        __threadfence_system();  // my partial (written by the GEMM) before the flag
        st_release_sys(flags_of(p.peer[threadIdx.x], p.data_bytes) + p.rank, use);
    }
    if (threadIdx.x < p.world) {
        const unsigned long long t0 = now_ns();
        while (ld_acquire_sys(mine + threadIdx.x) < use) {
            if (now_ns() - t0 > (unsigned long long)kSpinNs) asm volatile("trap;");
        }
    }
    __syncthreads();
    const int64_t n8 = p.n / 8;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8;
         i += (int64_t)gridDim.x * blockDim.x) {
        float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        for (int r = 0; r < p.world; ++r) {  // rank order: deterministic everywhere
            const uint4 v = __ldcv(reinterpret_cast<const uint4 *>(p.peer[r]) + i);
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                acc[2 * k] += __uint_as_float(w[k] << 16);
                acc[2 * k + 1] += __uint_as_float(w[k] & 0xffff0000u);
            }
        }
        uint4 *xp = reinterpret_cast<uint4 *>(p.x) + i;
        uint4 xv = *xp;
        uint32_t xw[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            // x + bf16(sum): the reference's residual with the rounded total
            const uint32_t t = pack_bf16(acc[2 * k], acc[2 * k + 1]);
            const float lo = __uint_as_float(xw[k] << 16) + __uint_as_float(t << 16);
            const float hi = __uint_as_float(xw[k] & 0xffff0000u) + __uint_as_float(t & 0xffff0000u);
            xw[k] = pack_bf16(lo, hi);
        }
        *xp = make_uint4(xw[0], xw[1], xw[2], xw[3]);
    }
    // the last CTA out advances the use counter for the next exchange on
    // this buffer (read by this rank only, after this kernel)
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(done_ctr, 1u) == gridDim.x - 1) {
            *use_ctr = use;
            *done_ctr = 0;
        }
    }
}


// x[i] += bf16(sum_r partial_r[i]) for the 8 elements of uint4 index i,
// given the already-summed (fp32) values
__device__ __forceinline__ uint4 add_rounded(uint4 xv, const float (&acc)[8]) {
    uint32_t xw[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const uint32_t t = pack_bf16(acc[2 * k], acc[2 * k + 1]);
        const float lo = __uint_as_float(xw[k] << 16) + __uint_as_float(t << 16);
        const float hi = __uint_as_float(xw[k] & 0xffff0000u) + __uint_as_float(t & 0xffff0000u);
        xw[k] = pack_bf16(lo, hi);
    }
    return make_uint4(xw[0], xw[1], xw[2], xw[3]);
}

__device__ __forceinline__ void spin_flags(const uint32_t *f, int world, uint32_t use) {
    if (threadIdx.x < world) {
        const unsigned long long t0 = now_ns();
        while (ld_acquire_sys(f + threadIdx.x) < use) {
            if (now_ns() - t0 > (unsigned long long)kSpinNs) asm volatile("trap;");
        }
    }
    __syncthreads();
}

// two-shot form (see the file comment).  Every CTA of the grid must be
// resident at once (phase 2 waits for phase 1 of all ranks' CTAs): the host
// caps the grid well below one CTA per SM.
__global__ void __launch_bounds__(256) ar_residual_2shot_kernel(const ArParams p) {
    __shared__ uint32_t s_use;
    grid_launch_dependents();  // as ar_residual_kernel
    grid_dependency_wait();
    uint32_t *mine = flags_of(p.peer[p.rank], p.data_bytes);
    uint32_t *use_ctr = mine + FS_AR_MAX_WORLD, *done_ctr = use_ctr + 1, *done1 = mine + kDone1;
    if (threadIdx.x == 0) s_use = *reinterpret_cast<volatile uint32_t *>(use_ctr) + 1u;
    __syncthreads();
    const uint32_t use = s_use;
    if (blockIdx.x == 0 && threadIdx.x < p.world) {
        __threadfence_system();  // my partial (written by the GEMM) before the flag
        st_release_sys(flags_of(p.peer[threadIdx.x], p.data_bytes) + p.rank, use);
    }
    spin_flags(mine, p.world, use);
    // phase 1: the slice this rank owns, summed over ranks in rank order
    const int64_t n8 = p.n / 8;
    const int64_t half = p.data_bytes / 2;
    const int64_t s0 = n8 * p.rank / p.world, s1 = n8 * (p.rank + 1) / p.world;
    uint4 *my_sums = reinterpret_cast<uint4 *>(p.peer[p.rank] + half);
    for (int64_t i = s0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < s1;
         i += (int64_t)gridDim.x * blockDim.x) {
        float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        for (int r = 0; r < p.world; ++r) {
            const uint4 v = __ldcv(reinterpret_cast<const uint4 *>(p.peer[r]) + i);
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                acc[2 * k] += __uint_as_float(w[k] << 16);
                acc[2 * k + 1] += __uint_as_float(w[k] & 0xffff0000u);
            }
        }
        my_sums[i] = make_uint4(pack_bf16(acc[0], acc[1]), pack_bf16(acc[2], acc[3]),
                                pack_bf16(acc[4], acc[5]), pack_bf16(acc[6], acc[7]));
    }
    // the last CTA of this rank publishes "my slice sums are ready"
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        if (atomicAdd(done1, 1u) == gridDim.x - 1) {
            *done1 = 0;
            __threadfence_system();
            for (int r = 0; r < p.world; ++r)
                st_release_sys(flags_of(p.peer[r], p.data_bytes) + kFlagSums + p.rank, use);
        }
    }
    spin_flags(mine + kFlagSums, p.world, use);
    // phase 2: gather every slice from its owner, add to the residual
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8;
         i += (int64_t)gridDim.x * blockDim.x) {
        int owner = (int)(((i + 1) * p.world + n8 - 1) / n8) - 1;  // largest r: n8*r/world <= i
        while (owner > 0 && n8 * owner / p.world > i) --owner;
        while (owner + 1 < p.world && n8 * (owner + 1) / p.world <= i) ++owner;
        const uint4 sv = __ldcv(reinterpret_cast<const uint4 *>(p.peer[owner] + half) + i);
        const uint32_t w[4] = {sv.x, sv.y, sv.z, sv.w};
        float sum[8];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            sum[2 * k] = __uint_as_float(w[k] << 16);
            sum[2 * k + 1] = __uint_as_float(w[k] & 0xffff0000u);
        }
        uint4 *xp = reinterpret_cast<uint4 *>(p.x) + i;
        *xp = add_rounded(*xp, sum);  // bf16(sum) is exactly sum: the rounding happened once
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(done_ctr, 1u) == gridDim.x - 1) {
            *use_ctr = use;
            *done_ctr = 0;
        }
    }
}

}  // namespace fs

using namespace fs;

extern "C" int64_t fs_ar_buffer_bytes(int64_t max_elems) {
    if (max_elems < 0) return -1;
    const int64_t data = ((max_elems * 2 + 255) / 256) * 256;
    return 2 * data + 256;  // partial, slice sums (two-shot), flags + counters
}

extern "C" int fs_ar_alloc(int device, int64_t bytes, void **ptr) {
    FS_CHECK_ARG(ptr && bytes > 0, "bad arguments");
    int prev = 0;
    FS_CUDA(cudaGetDevice(&prev));
    FS_CUDA(cudaSetDevice(device));
    void *p = nullptr;
    cudaError_t e = cudaMalloc(&p, (size_t)bytes);
    if (e == cudaSuccess) e = cudaMemset(p, 0, (size_t)bytes);
    cudaSetDevice(prev);
    FS_CUDA(e);
    *ptr = p;
    return FS_OK;
}

extern "C" int fs_ar_free(void *ptr) {
    if (ptr) FS_CUDA(cudaFree(ptr));
    return FS_OK;
}

extern "C" int fs_ar_ipc_handle(void *ptr, void *handle) {
    FS_CHECK_ARG(ptr && handle, "null pointer");
    cudaIpcMemHandle_t h;
    FS_CUDA(cudaIpcGetMemHandle(&h, ptr));
    memcpy(handle, &h, sizeof(h));
    return FS_OK;
}

extern "C" int fs_ar_ipc_open(const void *handle, void **ptr) {
    FS_CHECK_ARG(ptr && handle, "null pointer");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    FS_CUDA(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
    return FS_OK;
}

extern "C" int fs_ar_ipc_close(void *ptr) {
    if (ptr) FS_CUDA(cudaIpcCloseMemHandle(ptr));
    return FS_OK;
}

// one-shot below this many bytes per rank or at two ranks (latency-bound
// there); two-shot above (NVLink-read-bound).  FS_AR_TWO_SHOT_BYTES overrides.
static int64_t two_shot_min_bytes() {
    static int64_t v = [] {
        const char *e = getenv("FS_AR_TWO_SHOT_BYTES");
        return e ? (int64_t)atoll(e) : (int64_t)(256 * 1024);
    }();
    return v;
}

extern "C" int fs_ar_residual_mode(void *const *peers, int32_t rank, int32_t world, int64_t n,
                                   int64_t data_bytes, void *x, int32_t ctas, int32_t mode,
                                   void *stream) {
    FS_CHECK_ARG(world >= 1 && world <= FS_AR_MAX_WORLD, "world must be in [1, %d]", FS_AR_MAX_WORLD);
    FS_CHECK_ARG(rank >= 0 && rank < world, "rank out of range");
    FS_CHECK_ARG(data_bytes > 0 && data_bytes % 512 == 0, "data_bytes must be the flag offset "
                 "of an fs_ar_buffer_bytes buffer");
    FS_CHECK_ARG(n >= 0 && n % 8 == 0 && n * 2 <= data_bytes / 2,
                 "n must be a multiple of 8 that fits");
    FS_CHECK_ARG(mode >= 0 && mode <= 2, "mode must be 0 (auto), 1 (one-shot) or 2 (two-shot)");
    FS_CHECK_ARG(peers && x && (reinterpret_cast<uintptr_t>(x) & 15) == 0, "bad pointers");
    ArParams prm = {};
    for (int r = 0; r < world; ++r) {
        FS_CHECK_ARG(peers[r] && (reinterpret_cast<uintptr_t>(peers[r]) & 255) == 0,
                     "peer buffer %d missing or misaligned", r);
        prm.peer[r] = static_cast<uint8_t *>(peers[r]);
    }
    prm.rank = rank;
    prm.world = world;
    prm.n = n;
    prm.data_bytes = data_bytes;
    prm.x = static_cast<__nv_bfloat16 *>(x);
    if (mode == 0) mode = (world > 2 && n * 2 >= two_shot_min_bytes()) ? 2 : 1;
    const int64_t need = (n / 8 + 255) / 256;
    // launched with PDL: 256 threads and no shared memory, so the grid is
    // resident next to a projection GEMM's CTAs (one per SM): neither the
    // early start nor the two-shot form's all-CTAs-resident wait can be
    // starved by the dependent launch
    cudaLaunchConfig_t lc = {};
    lc.blockDim = dim3(256);
    lc.stream = static_cast<cudaStream_t>(stream);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = attr;
    lc.numAttrs = 1;
    if (mode == 2) {
        // every CTA resident at once (phase 2 waits on phase 1 of the grid)
        int grid = ctas > 0 ? ctas : 64;
        if (grid > 64) grid = 64;
        if (grid > need) grid = (int)(need > 0 ? need : 1);
        lc.gridDim = dim3(grid);
        FS_CUDA(cudaLaunchKernelEx(&lc, ar_residual_2shot_kernel, prm));
        return FS_OK;
    }
    int grid = ctas > 0 ? ctas : 148;
    if (grid > need) grid = (int)(need > 0 ? need : 1);
    lc.gridDim = dim3(grid);
    FS_CUDA(cudaLaunchKernelEx(&lc, ar_residual_kernel, prm));
    return FS_OK;
}

extern "C" int fs_ar_residual(void *const *peers, int32_t rank, int32_t world, int64_t n,
                              int64_t data_bytes, void *x, int32_t ctas, void *stream) {
    return fs_ar_residual_mode(peers, rank, world, n, data_bytes, x, ctas, 0, stream);
}
