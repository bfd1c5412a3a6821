// K3 (KV append into pages), K5 (backup page gather), K6 (restore page
// scatter) and K7 (peer copy) of the FailSafe B200 hot path.
//
// Pages are opaque 8 KiB blocks to K5/K6/K7, so backup/restore/recovery
// move exactly the bytes the decode kernel reads.  K3/read apply the page
// swizzle (chunk c of row r at c ^ (r & 7)) documented in failsafe_b200.h.
#include <cuda_bf16.h>

#include "common.cuh"

namespace fs {

// one warp per token: lanes 0-15 move the 16 K chunks, lanes 16-31 the V chunks
__global__ void __launch_bounds__(256) kv_write_kernel(uint8_t *pool, const int32_t *bt,
                                                       int64_t bt_stride, const int32_t *tok_seq,
                                                       const int32_t *tok_pos,
                                                       const int32_t *tok_src, int32_t n_tok,
                                                       const uint8_t *k_src, const uint8_t *v_src,
                                                       int64_t src_stride_bytes) {
    const int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (t >= n_tok) return;
    const int32_t pos = tok_pos[t];
    const int64_t page = bt[(int64_t)tok_seq[t] * bt_stride + pos / kPageTokens];
    const uint32_t r = pos % kPageTokens, c = lane & 15, half = lane >> 4;
    const uint8_t *src = (half ? v_src : k_src) + (int64_t)tok_src[t] * src_stride_bytes + c * 16;
    uint8_t *dst = pool + page * kPageBytes + half * kHalfPage + swz(r, c);
    const uint4 v = *reinterpret_cast<const uint4 *>(src);
    *reinterpret_cast<uint4 *>(dst) = half ? bf16x8_to_f16x8(v) : v;  // V pages hold f16
}

// K3 over token runs: warp = token; the run is found by a binary search of
// the run prefix (a few hundred runs per layer)
__global__ void __launch_bounds__(256) kv_write_runs_kernel(
    uint8_t *pool, const int32_t *bt, int64_t bt_stride, const int32_t *run_seq,
    const int32_t *run_pos, const int32_t *run_src, const int32_t *run_off, int32_t n_runs,
    int32_t src_step, const uint8_t *k_src, const uint8_t *v_src, int64_t src_stride_bytes) {
    const int32_t base = run_off[0];
    const int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (t >= (int64_t)run_off[n_runs] - base) return;
    int lo = 0, hi = n_runs;  // run_off[lo] - base <= t < run_off[hi] - base
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (run_off[mid] - base <= t) lo = mid;
        else hi = mid;
    }
    const int32_t i = (int32_t)(t - (run_off[lo] - base));
    const int32_t pos = run_pos[lo] + i;
    const int64_t page = bt[(int64_t)run_seq[lo] * bt_stride + pos / kPageTokens];
    const uint32_t r = pos % kPageTokens, c = lane & 15, half = lane >> 4;
    const uint8_t *src = (half ? v_src : k_src) +
                         ((int64_t)run_src[lo] + (int64_t)i * src_step) * src_stride_bytes + c * 16;
    uint8_t *dst = pool + page * kPageBytes + half * kHalfPage + swz(r, c);
    const uint4 v = *reinterpret_cast<const uint4 *>(src);
    *reinterpret_cast<uint4 *>(dst) = half ? bf16x8_to_f16x8(v) : v;  // V pages hold f16
}

__global__ void __launch_bounds__(256) kv_read_kernel(const uint8_t *pool, const int32_t *bt,
                                                      int64_t bt_stride, const int32_t *tok_seq,
                                                      const int32_t *tok_pos,
                                                      const int32_t *tok_dst, int32_t n_tok,
                                                      uint8_t *k_dst, uint8_t *v_dst,
                                                      int64_t dst_stride_bytes) {
    const int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (t >= n_tok) return;
    const int32_t pos = tok_pos[t];
    const int64_t page = bt[(int64_t)tok_seq[t] * bt_stride + pos / kPageTokens];
    const uint32_t r = pos % kPageTokens, c = lane & 15, half = lane >> 4;
    uint8_t *dst = (half ? v_dst : k_dst) + (int64_t)tok_dst[t] * dst_stride_bytes + c * 16;
    const uint8_t *src = pool + page * kPageBytes + half * kHalfPage + swz(r, c);
    uint4 v = *reinterpret_cast<const uint4 *>(src);
    if (half) {
        v.x = f16x2_to_bf16x2(v.x);
        v.y = f16x2_to_bf16x2(v.y);
        v.z = f16x2_to_bf16x2(v.z);
        v.w = f16x2_to_bf16x2(v.w);
    }
    *reinterpret_cast<uint4 *>(dst) = v;
}

// K5/K6: page-granular gather (pool -> contiguous) / scatter (contiguous ->
// pool).  The contiguous side may be mapped pinned host memory, in which case
// the 16-byte loads/stores travel over PCIe (zero-copy), so a backup or
// restore of scattered pages is ONE launch on a side stream.  Each CTA moves
// whole pages; 4 independent 16 B transfers per thread keep PCIe busy.
template <bool GATHER>
__global__ void __launch_bounds__(256) page_copy_kernel(uint8_t *pool, const int32_t *ids,
                                                        int32_t n_pages, uint8_t *flat,
                                                        const int32_t *slots) {
    constexpr int kChunks = kPageBytes / 16;  // 512 per page
    for (int64_t pg = blockIdx.x; pg < n_pages; pg += gridDim.x) {
        const int64_t slot = slots ? slots[pg] : pg;
        uint4 *pp = reinterpret_cast<uint4 *>(pool + (int64_t)ids[pg] * kPageBytes);
        uint4 *fp = reinterpret_cast<uint4 *>(flat + slot * kPageBytes);
        uint4 v[kChunks / 256];
#pragma unroll
        for (int j = 0; j < kChunks / 256; ++j)
            v[j] = GATHER ? pp[threadIdx.x + j * 256] : fp[threadIdx.x + j * 256];
#pragma unroll
        for (int j = 0; j < kChunks / 256; ++j) {
            if (GATHER) fp[threadIdx.x + j * 256] = v[j];
            else pp[threadIdx.x + j * 256] = v[j];
        }
    }
}

}  // namespace fs

using namespace fs;

extern "C" int fs_kv_write(void *kv_pool, const int32_t *block_table, int64_t bt_stride,
                           const int32_t *tok_seq, const int32_t *tok_pos, const int32_t *tok_src,
                           int32_t n_tok, const void *k_src, const void *v_src, int64_t src_stride,
                           void *stream) {
    FS_CHECK_ARG(n_tok >= 0, "n_tok must be nonnegative");
    if (n_tok == 0) return FS_OK;
    FS_CHECK_ARG(kv_pool && block_table && tok_seq && tok_pos && tok_src && k_src && v_src,
                 "null pointer");
    FS_CHECK_ARG(src_stride % 8 == 0 && src_stride >= kHeadDim,
                 "src_stride must be a multiple of 8 and >= %d", kHeadDim);
    const int64_t threads = (int64_t)n_tok * 32;
    kv_write_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<uint8_t *>(kv_pool), block_table, bt_stride, tok_seq, tok_pos, tok_src, n_tok,
        static_cast<const uint8_t *>(k_src), static_cast<const uint8_t *>(v_src), src_stride * 2);
    return cuda_status(cudaGetLastError(), "kv_write_kernel launch");
}

extern "C" int fs_kv_write_runs(void *kv_pool, const int32_t *block_table, int64_t bt_stride,
                                const int32_t *run_seq, const int32_t *run_pos,
                                const int32_t *run_src, const int32_t *run_off, int32_t n_runs,
                                int32_t n_tok, int32_t src_step, const void *k_src,
                                const void *v_src, int64_t src_stride, void *stream) {
    FS_CHECK_ARG(n_runs >= 0 && n_tok >= 0, "n_runs and n_tok must be nonnegative");
    if (n_runs == 0 || n_tok == 0) return FS_OK;
    FS_CHECK_ARG(kv_pool && block_table && run_seq && run_pos && run_src && run_off && k_src &&
                     v_src, "null pointer");
    FS_CHECK_ARG(src_stride % 8 == 0 && src_stride >= kHeadDim,
                 "src_stride must be a multiple of 8 and >= %d", kHeadDim);
    const int64_t threads = (int64_t)n_tok * 32;
    kv_write_runs_kernel<<<(unsigned)((threads + 255) / 256), 256, 0,
                           static_cast<cudaStream_t>(stream)>>>(
        static_cast<uint8_t *>(kv_pool), block_table, bt_stride, run_seq, run_pos, run_src, run_off,
        n_runs, src_step, static_cast<const uint8_t *>(k_src), static_cast<const uint8_t *>(v_src),
        src_stride * 2);
    return cuda_status(cudaGetLastError(), "kv_write_runs_kernel launch");
}

extern "C" int fs_kv_read(const void *kv_pool, const int32_t *block_table, int64_t bt_stride,
                          const int32_t *tok_seq, const int32_t *tok_pos, const int32_t *tok_dst,
                          int32_t n_tok, void *k_dst, void *v_dst, int64_t dst_stride,
                          void *stream) {
    FS_CHECK_ARG(n_tok >= 0, "n_tok must be nonnegative");
    if (n_tok == 0) return FS_OK;
    FS_CHECK_ARG(kv_pool && block_table && tok_seq && tok_pos && tok_dst && k_dst && v_dst,
                 "null pointer");
    FS_CHECK_ARG(dst_stride % 8 == 0 && dst_stride >= kHeadDim,
                 "dst_stride must be a multiple of 8 and >= %d", kHeadDim);
    const int64_t threads = (int64_t)n_tok * 32;
    kv_read_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<const uint8_t *>(kv_pool), block_table, bt_stride, tok_seq, tok_pos, tok_dst,
        n_tok, static_cast<uint8_t *>(k_dst), static_cast<uint8_t *>(v_dst), dst_stride * 2);
    return cuda_status(cudaGetLastError(), "kv_read_kernel launch");
}

static int page_copy(bool gather, void *pool, const int32_t *ids, int32_t n, void *flat,
                     const int32_t *slots, int32_t max_ctas, void *stream) {
    FS_CHECK_ARG(n >= 0, "n_pages must be nonnegative");
    if (n == 0) return FS_OK;
    FS_CHECK_ARG(pool && ids && flat, "null pointer");
    FS_CHECK_ARG((reinterpret_cast<uintptr_t>(flat) & 15) == 0, "flat buffer must be 16B aligned");
    int grid = max_ctas > 0 ? max_ctas : 4 * 148;
    if (grid > n) grid = n;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (gather)
        page_copy_kernel<true><<<grid, 256, 0, st>>>(static_cast<uint8_t *>(pool), ids, n,
                                                     static_cast<uint8_t *>(flat), slots);
    else
        page_copy_kernel<false><<<grid, 256, 0, st>>>(static_cast<uint8_t *>(pool), ids, n,
                                                      static_cast<uint8_t *>(flat), slots);
    return cuda_status(cudaGetLastError(), "page_copy_kernel launch");
}

extern "C" int fs_pages_gather(const void *kv_pool, const int32_t *page_ids, int32_t n_pages,
                               void *dst, const int32_t *dst_slots, int32_t max_ctas,
                               void *stream) {
    return page_copy(true, const_cast<void *>(kv_pool), page_ids, n_pages, dst, dst_slots,
                     max_ctas, stream);
}

extern "C" int fs_pages_scatter(void *kv_pool, const int32_t *page_ids, int32_t n_pages,
                                const void *src, const int32_t *src_slots, int32_t max_ctas,
                                void *stream) {
    return page_copy(false, kv_pool, page_ids, n_pages, const_cast<void *>(src), src_slots,
                     max_ctas, stream);
}

extern "C" int fs_enable_peer(int device, int peer) {
    if (device == peer) return FS_OK;
    int can = 0;
    FS_CUDA(cudaDeviceCanAccessPeer(&can, device, peer));
    if (!can) return fail(FS_ESIMULATION, "device %d cannot access peer %d", device, peer);
    int prev = 0;
    FS_CUDA(cudaGetDevice(&prev));
    FS_CUDA(cudaSetDevice(device));
    cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
    cudaSetDevice(prev);
    if (e == cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();
        return FS_OK;
    }
    return cuda_status(e, "cudaDeviceEnablePeerAccess");
}

extern "C" int fs_copy_peer(void *dst, int dst_device, const void *src, int src_device,
                            int64_t bytes, void *stream) {
    FS_CHECK_ARG(bytes >= 0, "bytes must be nonnegative");
    if (bytes == 0) return FS_OK;
    FS_CHECK_ARG(dst && src, "null pointer");
    FS_CUDA(cudaMemcpyPeerAsync(dst, dst_device, src, src_device, (size_t)bytes,
                                static_cast<cudaStream_t>(stream)));
    return FS_OK;
}
