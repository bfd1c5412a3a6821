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
    *reinterpret_cast<uint4 *>(dst) = v;
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
    *reinterpret_cast<uint4 *>(dst) = v;
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
    *reinterpret_cast<uint4 *>(dst) = *reinterpret_cast<const uint4 *>(src);
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

// K5, token-granular: the token at item_len[i]-1 of every item -> the same
// page slot of the host mirror (slot == page id).  A token is 4 x 128 B of
// the page (K / V half x the two 64-dim atoms; the swizzle permutes chunks
// only within a 128-B row piece): one warp per item, lane = 16-B chunk.
__global__ void __launch_bounds__(256) kv_backup_tokens_kernel(const uint8_t *pool,
                                                               const int32_t *bt, int64_t bt_stride,
                                                               const int32_t *item_seq,
                                                               const int32_t *item_len,
                                                               int32_t n_items, uint8_t *mirror) {
    const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (i >= n_items) return;
    const int32_t len = item_len[i];
    if (len <= 0) return;
    const int32_t pos = len - 1;
    const int64_t page = bt[(int64_t)item_seq[i] * bt_stride + pos / kPageTokens];
    const int piece = lane >> 3;
    const int64_t off = page * kPageBytes + (piece >> 1) * kHalfPage + (piece & 1) * 2048 +
                        (pos % kPageTokens) * 128 + (lane & 7) * 16;
    *reinterpret_cast<uint4 *>(mirror + off) = *reinterpret_cast<const uint4 *>(pool + off);
}

// K7 executor: many 2-D copies in ONE launch.  Each segment is `height`
// rows of `width` bytes; a warp copies one row (16-B lanes when source,
// destination, pitches and width are 16-B aligned, bytes otherwise), rows
// are dealt to warps round-robin over the flattened row space (row_off =
// exclusive prefix of heights).  Sources / destinations may be local HBM,
// a peer's HBM mapped by CUDA IPC (the reads then run over NVLink) or
// mapped pinned host memory (PCIe): the SMs keep ~thousands of 16-B loads
// in flight, which is what a P2P or zero-copy stream needs.
__global__ void __launch_bounds__(256) copy_segments_kernel(const fs_copy_seg *segs,
                                                            const int64_t *row_off, int32_t n_segs) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    const int64_t total = row_off[n_segs];
    for (int64_t g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; g < total; g += warps) {
        int lo = 0, hi = n_segs;  // row_off[lo] <= g < row_off[hi]
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (row_off[mid] <= g) lo = mid;
            else hi = mid;
        }
        const fs_copy_seg sg = segs[lo];
        const int64_t row = g - row_off[lo];
        const uint8_t *src = static_cast<const uint8_t *>(sg.src) + row * sg.spitch;
        uint8_t *dst = static_cast<uint8_t *>(sg.dst) + row * sg.dpitch;
        const bool vec = ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst) |
                           (uintptr_t)sg.width) & 15) == 0;
        if (vec) {
            const int64_t n16 = sg.width >> 4;
            const uint4 *s4 = reinterpret_cast<const uint4 *>(src);
            uint4 *d4 = reinterpret_cast<uint4 *>(dst);
            int64_t i = lane;
            for (; i + 96 < n16; i += 128) {  // 4 loads in flight per lane
                const uint4 a = s4[i], b = s4[i + 32], c = s4[i + 64], d = s4[i + 96];
                d4[i] = a;
                d4[i + 32] = b;
                d4[i + 64] = c;
                d4[i + 96] = d;
            }
            for (; i < n16; i += 32) d4[i] = s4[i];
        } else {
            for (int64_t i = lane; i < sg.width; i += 32) dst[i] = src[i];
        }
    }
}

}  // namespace fs

using namespace fs;

extern "C" int fs_copy_segments(const fs_copy_seg *segs, const int64_t *row_off, int32_t n_segs,
                                int32_t ctas, void *stream) {
    FS_CHECK_ARG(n_segs >= 0, "n_segs must be nonnegative");
    if (n_segs == 0) return FS_OK;
    FS_CHECK_ARG(segs && row_off, "null pointer");
    copy_segments_kernel<<<ctas > 0 ? ctas : 4 * 148, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        segs, row_off, n_segs);
    return cuda_status(cudaGetLastError(), "copy_segments_kernel launch");
}

extern "C" int fs_kv_backup_tokens(const void *kv_pool, const int32_t *block_table,
                                   int64_t bt_stride, const int32_t *item_seq,
                                   const int32_t *item_len, int32_t n_items, void *mirror,
                                   void *stream) {
    FS_CHECK_ARG(n_items >= 0, "n_items must be nonnegative");
    if (n_items == 0) return FS_OK;
    FS_CHECK_ARG(kv_pool && block_table && item_seq && item_len && mirror, "null pointer");
    FS_CHECK_ARG((reinterpret_cast<uintptr_t>(mirror) & 15) == 0, "mirror must be 16B aligned");
    const int64_t threads = (int64_t)n_items * 32;
    kv_backup_tokens_kernel<<<(unsigned)((threads + 255) / 256), 256, 0,
                              static_cast<cudaStream_t>(stream)>>>(
        static_cast<const uint8_t *>(kv_pool), block_table, bt_stride, item_seq, item_len,
        n_items, static_cast<uint8_t *>(mirror));
    return cuda_status(cudaGetLastError(), "kv_backup_tokens_kernel launch");
}

extern "C" int fs_host_register(void *ptr, int64_t bytes, void **dev_ptr) {
    FS_CHECK_ARG(ptr && bytes > 0 && dev_ptr, "null pointer or empty range");
    FS_CUDA(cudaHostRegister(ptr, (size_t)bytes, cudaHostRegisterPortable | cudaHostRegisterMapped));
    FS_CUDA(cudaHostGetDevicePointer(dev_ptr, ptr, 0));
    return FS_OK;
}

extern "C" int fs_host_unregister(void *ptr) {
    FS_CHECK_ARG(ptr, "null pointer");
    FS_CUDA(cudaHostUnregister(ptr));
    return FS_OK;
}

extern "C" int fs_copy_2d(void *dst, int64_t dpitch, const void *src, int64_t spitch,
                          int64_t width, int64_t height, void *stream) {
    FS_CHECK_ARG(width >= 0 && height >= 0, "negative extent");
    if (width == 0 || height == 0) return FS_OK;
    FS_CHECK_ARG(dst && src, "null pointer");
    FS_CHECK_ARG(dpitch >= width && spitch >= width, "pitch smaller than width");
    FS_CUDA(cudaMemcpy2DAsync(dst, (size_t)dpitch, src, (size_t)spitch, (size_t)width,
                              (size_t)height, cudaMemcpyDefault, static_cast<cudaStream_t>(stream)));
    return FS_OK;
}

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
