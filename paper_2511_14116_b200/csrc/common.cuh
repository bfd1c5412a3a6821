// Shared helpers for libfailsafe_b200: status handling and sm_100a PTX
// wrappers (TMA bulk copy, mbarrier, ldmatrix, mma.sync, movmatrix).
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <string>

#include "../../include/failsafe_b200.h"

namespace fs {

void set_error(const std::string &msg);
int fail(int code, const char *fmt, ...);

// Returns FS_ECUDA with a message when the last launch / call failed.
int cuda_status(cudaError_t e, const char *what);

#define FS_CHECK_ARG(cond, ...)                                   \
    do {                                                          \
        if (!(cond)) return ::fs::fail(FS_EVALIDATION, __VA_ARGS__); \
    } while (0)

#define FS_CUDA(call)                                             \
    do {                                                          \
        cudaError_t _e = (call);                                  \
        if (_e != cudaSuccess) return ::fs::cuda_status(_e, #call); \
    } while (0)

constexpr int kPageTokens = FS_PAGE_TOKENS;
constexpr int kHeadDim = FS_HEAD_DIM;
constexpr int kPageBytes = FS_PAGE_BYTES;
constexpr int kHalfPage = FS_PAGE_BYTES / 2;   // K rows, then V rows

// byte offset of 16-byte chunk `c` (0..15) of row `r` inside a K or V half:
// two 2 KB atoms (dims 0-63, 64-127), each 16 rows x 128 B with the 128 B
// swizzle (chunk c&7 of row r at c&7 ^ r&7).  Each atom is a UMMA-canonical
// SWIZZLE_128B block, so pages TMA'd atom by atom into consecutive smem
// rows are tcgen05 operands as is; ldmatrix over 8 rows stays conflict-free.
constexpr int kAtomBytes = 2048;
__host__ __device__ __forceinline__ uint32_t swz(uint32_t r, uint32_t c) {
    return ((c >> 3) * kAtomBytes) + r * 128 + (((c & 7u) ^ (r & 7u)) << 4);
}

int sm_count(int device);

#ifdef __CUDACC__
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}

__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Programmatic dependent launch: block until the preceding grid in the
// stream has completed and its writes are visible (no-op without PDL).
__device__ __forceinline__ void grid_dependency_wait() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

// Programmatic dependent launch: let the next grid in the stream be
// scheduled now (it still waits in griddepcontrol.wait for this grid's
// completion before touching our results).
__device__ __forceinline__ void grid_launch_dependents() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive_cta(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "FS_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra FS_WAIT_%=;\n}" ::"r"(bar),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

// TMA bulk (non-tensor) global -> shared copy completing on an mbarrier.
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes,
                                         uint32_t bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1], %2, [%3], %4;" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(bar), "l"(pol)
        : "memory");
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t &r0, uint32_t &r1, uint32_t &r2,
                                        uint32_t &r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}

__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t &r0, uint32_t &r1,
                                          uint32_t &r2, uint32_t &r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}

// D = A(16x16 bf16, row) * B(16x8 bf16, col) + D, fp32 accumulate
__device__ __forceinline__ void mma_bf16(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 "
        "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t movmatrix_t(uint32_t a) {
    uint32_t d;
    asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(d) : "r"(a));
    return d;
}

__device__ __forceinline__ float fast_exp2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}

// D = A(16x16 f16, row) * B(16x8 f16, col) + D, fp32 accumulate
__device__ __forceinline__ void mma_f16(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                        uint32_t a3, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 "
        "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t pack_f16(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}

// as pack_f16, saturating to +-65504 (split partials O / l: a convex
// combination of f16 V rows, marginally above 65504 at most from the f16 P
// vs fp32 l rounding -- never Inf)
__device__ __forceinline__ uint32_t pack_f16_sat(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.satfinite.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}

// (lo, hi) as a bf16x2 pair plus the bf16x2 pair of its rounding residual:
// h + l carries ~16 mantissa bits (two bf16 MMAs instead of one)
__device__ __forceinline__ void split_bf16x2(float lo, float hi, uint32_t &h, uint32_t &l) {
    h = pack_bf16(lo, hi);
    l = pack_bf16(lo - __uint_as_float(h << 16), hi - __uint_as_float(h & 0xffff0000u));
}

// two bf16 -> two f16: exact for |x| in f16's normal range, saturated to
// +-65504 outside it (no Inf reaches the tensor cores); one F2FP
__device__ __forceinline__ uint32_t bf16x2_to_f16x2(uint32_t v) {
    uint32_t r;
    asm("cvt.rn.satfinite.f16x2.f32 %0, %1, %2;"
        : "=r"(r)
        : "f"(__uint_as_float(v & 0xffff0000u)), "f"(__uint_as_float(v << 16)));
    return r;
}

// 8 bf16 -> 8 f16 (the V half of a page is stored in f16)
__device__ __forceinline__ uint4 bf16x8_to_f16x8(uint4 v) {
    v.x = bf16x2_to_f16x2(v.x);
    v.y = bf16x2_to_f16x2(v.y);
    v.z = bf16x2_to_f16x2(v.z);
    v.w = bf16x2_to_f16x2(v.w);
    return v;
}

// two f16 -> two bf16 (exact for values that came from bf16)
__device__ __forceinline__ uint32_t f16x2_to_bf16x2(uint32_t v) {
    __half2 h = *reinterpret_cast<__half2 *>(&v);
    float2 f = __half22float2(h);
    return pack_bf16(f.x, f.y);
}
#endif

}  // namespace fs
