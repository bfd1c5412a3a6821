// MLP helpers of the decode step and the synthetic-weight initialiser.
//
// fs_swiglu:      act[r, c] = silu(h[r, c]) * h[r, C + c] -- the gated-FFN
//                 nonlinearity of the TP MLP partial (the gated 3-matrix FFN the
//                 reference's byte accounting assumes, core.py:93-95), one
//                 vectorised launch between the gate/up and down GEMMs.
// fs_fill_normal: counter-based N(0,1)*scale fill keyed by (seed, salt, GLOBAL
//                 row, GLOBAL col): every rank of every world size materialises
//                 bit-identical slices of one global weight matrix without
//                 generating the whole matrix (hybrid/cyclic/on-demand shards).
#include <cuda_bf16.h>

#include <algorithm>

#include "common.cuh"

namespace fs {

__global__ void __launch_bounds__(256) swiglu_kernel(const __nv_bfloat16 *h, int64_t rows,
                                                     int64_t cols, int64_t ld,
                                                     __nv_bfloat16 *out, int64_t ld_out) {
    const int64_t vec = cols / 8;  // 8 bf16 per 16 B
    const int64_t n = rows * vec;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / vec, c = (i % vec) * 8;
        const uint4 g = *reinterpret_cast<const uint4 *>(h + r * ld + c);
        const uint4 u = *reinterpret_cast<const uint4 *>(h + r * ld + cols + c);
        const __nv_bfloat162 *g2 = reinterpret_cast<const __nv_bfloat162 *>(&g);
        const __nv_bfloat162 *u2 = reinterpret_cast<const __nv_bfloat162 *>(&u);
        uint4 o;
        __nv_bfloat162 *o2 = reinterpret_cast<__nv_bfloat162 *>(&o);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const float2 gf = __bfloat1622float2(g2[k]);
            const float2 uf = __bfloat1622float2(u2[k]);
            const float a = gf.x / (1.f + __expf(-gf.x)) * uf.x;
            const float b = gf.y / (1.f + __expf(-gf.y)) * uf.y;
            o2[k] = __floats2bfloat162_rn(a, b);
        }
        *reinterpret_cast<uint4 *>(out + r * ld_out + c) = o;
    }
}

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__global__ void __launch_bounds__(256) fill_normal_kernel(__nv_bfloat16 *out, int64_t rows,
                                                          int64_t cols, int64_t ld,
                                                          const int32_t *row_map, int64_t row_off,
                                                          const int32_t *col_map, int64_t col_off,
                                                          uint64_t key, float scale) {
    const int64_t n = rows * cols;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / cols, c = i % cols;
        const uint64_t gr = row_map ? (uint64_t)row_map[r] : (uint64_t)(row_off + r);
        const uint64_t gc = col_map ? (uint64_t)col_map[c] : (uint64_t)(col_off + c);
        const uint64_t h = mix64(key ^ mix64((gr << 32) ^ gc));
        const float u1 = ((h >> 40) + 0.5f) * (1.0f / 16777216.0f);          // (0,1)
        const float u2 = ((h & 0xFFFFFFull) + 0.5f) * (1.0f / 16777216.0f);
        const float z = sqrtf(-2.f * __logf(u1)) * __cosf(6.283185307f * u2);
        out[r * ld + c] = __float2bfloat16_rn(z * scale);
    }
}

static uint64_t mix64_host(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

}  // namespace fs

using namespace fs;

extern "C" int fs_swiglu(const void *h, int64_t rows, int64_t cols, int64_t ld, void *out,
                         int64_t ld_out, void *stream) {
    FS_CHECK_ARG(rows >= 0 && cols >= 0, "negative shape");
    if (rows == 0 || cols == 0) return FS_OK;
    FS_CHECK_ARG(h && out, "null pointer");
    FS_CHECK_ARG(cols % 8 == 0 && ld % 8 == 0 && ld_out % 8 == 0 && ld >= 2 * cols,
                 "swiglu needs cols, ld multiples of 8 and ld >= 2*cols");
    const int64_t n = rows * cols / 8;
    const int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
    swiglu_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<const __nv_bfloat16 *>(h), rows, cols, ld, static_cast<__nv_bfloat16 *>(out),
        ld_out);
    return cuda_status(cudaGetLastError(), "swiglu_kernel launch");
}

extern "C" int fs_fill_normal(void *out, int64_t rows, int64_t cols, int64_t ld,
                              const int32_t *row_map, int64_t row_off, const int32_t *col_map,
                              int64_t col_off, uint64_t seed, uint64_t salt, float scale,
                              void *stream) {
    FS_CHECK_ARG(rows >= 0 && cols >= 0 && ld >= cols, "bad shape");
    if (rows == 0 || cols == 0) return FS_OK;
    FS_CHECK_ARG(out, "null pointer");
    const uint64_t key = mix64_host(seed) ^ (salt * 0xD1B54A32D192ED03ull);
    const int64_t n = rows * cols;
    const int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
    fill_normal_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<__nv_bfloat16 *>(out), rows, cols, ld, row_map, row_off, col_map, col_off, key,
        scale);
    return cuda_status(cudaGetLastError(), "fill_normal_kernel launch");
}
