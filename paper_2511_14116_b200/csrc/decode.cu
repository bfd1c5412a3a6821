// K1 / K2 / K4: stream-K paged GQA decode for the FailSafe hybrid-attention
// step (the attention half of refexec.parallel_forward, refexec.py:281-297,
// with the per-head math of _head_attention, refexec.py:85-103).
//
// Work = a list of items (one per (kv head, request) pair a rank serves:
// every request for its TP heads, only routed requests for replicated
// heads).  All items' pages are flattened into one page space of P pages
// and split EVENLY over every warp of a persistent grid (W = SMs x WARPS):
// warp w owns pages [w*P/W, (w+1)*P/W).  A warp streams its pages through
// a private ring of STAGES x 8 KiB shared-memory slots filled by TMA bulk
// copies (one cp.async.bulk per page, mbarrier completion), so the HBM
// pipeline never drains at item boundaries and ragged lengths cost nothing
// in balance.  Per 16-token page the warp runs
//     S^T[16 tok x 8 q]   = K[16 x 128]   . Q^T[128 x 8]   (8 mma.m16n8k16)
//     O^T[128 dim x 8 q] += V^T[128 x 16] . P^T[16 x 8]    (8 mma.m16n8k16)
// i.e. tensor cores for the GQA query-group tile (q_per_kv <= 8 queries as
// the mma N dimension), online softmax on the S^T fragments, and P^T made
// from S^T with movmatrix.trans.  A warp that covers a whole item writes
// the normalized output; otherwise it writes (O/l, lse) to a partial slot
// `item + w` and K2 merges the slots of that item.
#include <cuda_bf16.h>
#include <cub/block/block_scan.cuh>

#include "common.cuh"

namespace fs {

struct DecodeParams {
    const __nv_bfloat16 *q;
    const uint8_t *kv;
    const int32_t *bt;
    int64_t bt_stride;
    const int32_t *item_seq, *item_len, *item_qrow, *item_orow, *page_off;
    int32_t n_items;
    int32_t qpk;
    float scale_log2;
    int32_t out_fp32;
    void *out;
    float *part_o, *part_lse;
    int64_t n_warps;  // W of the stream-K partition
};

__device__ __forceinline__ int64_t owner_warp(int64_t x, int64_t W, int64_t P) {
    return ((x + 1) * W + P - 1) / P - 1;
}

// largest i in [0, n) with off[i] <= x (off is nondecreasing, off[n] > x)
__device__ __forceinline__ int find_item(const int32_t *off, int n, int64_t x) {
    int lo = 0, hi = n;  // invariant: off[lo] <= x < off[hi]
    while (hi - lo > 1) {
        int mid = (lo + hi) >> 1;
        if (off[mid] <= x) lo = mid; else hi = mid;
    }
    return lo;
}

template <int WARPS, int STAGES>
__global__ void __launch_bounds__(WARPS * 32, 1) decode_kernel(const DecodeParams p) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gid = lane >> 2, tig = lane & 3;

    const int64_t P = p.page_off[p.n_items];
    const int64_t W = p.n_warps;
    const int64_t w = (int64_t)blockIdx.x * WARPS + warp;
    const int64_t x0 = w * P / W, x1 = (w + 1) * P / W;
    if (x0 >= x1) return;  // warp-uniform; no CTA-wide barriers below

    const uint32_t buf0 = smem_u32(smem) + warp * STAGES * kPageBytes;
    const uint32_t bar0 = smem_u32(smem) + WARPS * STAGES * kPageBytes + warp * STAGES * 8;
    if (lane == 0) {
        for (int s = 0; s < STAGES; ++s) mbar_init(bar0 + 8 * s, 1);
        fence_barrier_init();
        fence_proxy_async();
    }
    __syncwarp();

    const int32_t *off = p.page_off;
    const int first = find_item(off, p.n_items, x0);

    // ---- producer state (lane 0 only) ----
    int pitem = first;
    int64_t px = x0;
    const uint64_t pol = policy_evict_first();
    auto issue = [&](int stage) {
        while (px >= off[pitem + 1]) ++pitem;
        const int64_t pg = p.bt[(int64_t)p.item_seq[pitem] * p.bt_stride + (px - off[pitem])];
        const uint32_t bar = bar0 + 8 * stage;
        mbar_expect_tx(bar, kPageBytes);
        bulk_g2s(buf0 + stage * kPageBytes, p.kv + pg * kPageBytes, kPageBytes, bar, pol);
        ++px;
    };
    if (lane == 0) {
        for (int s = 0; s < STAGES && px < x1; ++s) issue(s);
    }

    // ---- consumer state ----
    int item = first;
    int64_t item_begin = off[item], item_end = off[item + 1];
    int64_t seg_begin = x0;
    int len = p.item_len[item];
    uint32_t qf[8][2];
    float m0, m1, l0, l1;
    float o[8][4];

    auto load_q = [&]() {
        const __nv_bfloat16 *qb = p.q + ((int64_t)p.item_qrow[item] * p.qpk + gid) * kHeadDim;
        const bool ok = gid < p.qpk;
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
            qf[ks][0] = ok ? *reinterpret_cast<const uint32_t *>(qb + ks * 16 + 2 * tig) : 0u;
            qf[ks][1] = ok ? *reinterpret_cast<const uint32_t *>(qb + ks * 16 + 8 + 2 * tig) : 0u;
        }
        m0 = m1 = -INFINITY;
        l0 = l1 = 0.f;
#pragma unroll
        for (int mt = 0; mt < 8; ++mt) o[mt][0] = o[mt][1] = o[mt][2] = o[mt][3] = 0.f;
    };
    load_q();

    int stage = 0;
    uint32_t phase = 0;
    for (int64_t x = x0; x < x1; ++x) {
        const uint32_t kb = buf0 + stage * kPageBytes;
        const uint32_t vb = kb + kHalfPage;
        const int valid = min(kPageTokens, len - (int)(x - item_begin) * kPageTokens);
        mbar_wait(bar0 + 8 * stage, phase);
        if (valid < kPageTokens) {
            // tail page: rows >= valid may hold stale bytes; zero the V rows
            // so 0-probability tokens cannot inject NaN/Inf into P.V
            uint8_t *vrow = smem + (vb - smem_u32(smem));
            for (int c = valid * 16 + lane; c < kPageTokens * 16; c += 32)
                reinterpret_cast<uint4 *>(vrow)[c] = make_uint4(0, 0, 0, 0);
            fence_proxy_async();
            __syncwarp();
        }

        // ---- S^T = K . Q^T ----
        float sa[4] = {0.f, 0.f, 0.f, 0.f}, sb[4] = {0.f, 0.f, 0.f, 0.f};
        {
            const int i = lane >> 3;
            const uint32_t r = (lane & 7) + ((i & 1) << 3);
#pragma unroll
            for (int ks = 0; ks < 8; ks += 2) {
                uint32_t a0, a1, a2, a3, c0, c1, c2, c3;
                ldsm_x4(kb + swz(r, 2 * ks + (i >> 1)), a0, a1, a2, a3);
                ldsm_x4(kb + swz(r, 2 * ks + 2 + (i >> 1)), c0, c1, c2, c3);
                mma_bf16(sa, a0, a1, a2, a3, qf[ks][0], qf[ks][1]);
                mma_bf16(sb, c0, c1, c2, c3, qf[ks + 1][0], qf[ks + 1][1]);
            }
        }
        float s0 = sa[0] + sb[0], s1 = sa[1] + sb[1], s2 = sa[2] + sb[2], s3 = sa[3] + sb[3];
        s0 = gid < valid ? s0 * p.scale_log2 : -INFINITY;
        s1 = gid < valid ? s1 * p.scale_log2 : -INFINITY;
        s2 = gid + 8 < valid ? s2 * p.scale_log2 : -INFINITY;
        s3 = gid + 8 < valid ? s3 * p.scale_log2 : -INFINITY;

        // ---- online softmax (per query column; tokens live on gid) ----
        float mx0 = fmaxf(s0, s2), mx1 = fmaxf(s1, s3);
#pragma unroll
        for (int sh = 4; sh < 32; sh <<= 1) {
            mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, sh));
            mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, sh));
        }
        const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
        const float al0 = fast_exp2(m0 - mn0), al1 = fast_exp2(m1 - mn1);
        const float p0 = fast_exp2(s0 - mn0), p1 = fast_exp2(s1 - mn1);
        const float p2 = fast_exp2(s2 - mn0), p3 = fast_exp2(s3 - mn1);
        l0 = l0 * al0 + p0 + p2;
        l1 = l1 * al1 + p1 + p3;
        m0 = mn0;
        m1 = mn1;
#pragma unroll
        for (int mt = 0; mt < 8; ++mt) {
            o[mt][0] *= al0;
            o[mt][1] *= al1;
            o[mt][2] *= al0;
            o[mt][3] *= al1;
        }
        const uint32_t pb0 = movmatrix_t(pack_bf16(p0, p1));
        const uint32_t pb1 = movmatrix_t(pack_bf16(p2, p3));

        // ---- O^T += V^T . P^T ----
        {
            const int i = lane >> 3;
            const uint32_t r = (lane & 7) + ((i >> 1) << 3);
#pragma unroll
            for (int mt = 0; mt < 8; ++mt) {
                uint32_t a0, a1, a2, a3;
                ldsm_x4_t(vb + swz(r, 2 * mt + (i & 1)), a0, a1, a2, a3);
                mma_bf16(o[mt], a0, a1, a2, a3, pb0, pb1);
            }
        }
        __syncwarp();
        if (lane == 0 && px < x1) issue(stage);
        if (++stage == STAGES) {
            stage = 0;
            phase ^= 1u;
        }

        // ---- end of this warp's segment of the item ----
        if (x + 1 == item_end || x + 1 == x1) {
            float t0 = l0, t1 = l1;
#pragma unroll
            for (int sh = 4; sh < 32; sh <<= 1) {
                t0 += __shfl_xor_sync(0xffffffffu, t0, sh);
                t1 += __shfl_xor_sync(0xffffffffu, t1, sh);
            }
            const float inv0 = 1.f / t0, inv1 = 1.f / t1;
            const int q0 = 2 * tig, q1 = 2 * tig + 1;
            const bool whole = seg_begin == item_begin && x + 1 == item_end;
            if (whole) {
                const int64_t ob = (int64_t)p.item_orow[item] * p.qpk * kHeadDim;
#pragma unroll
                for (int mt = 0; mt < 8; ++mt) {
                    const int d0 = mt * 16 + gid, d1 = d0 + 8;
                    if (p.out_fp32) {
                        float *out = static_cast<float *>(p.out) + ob;
                        if (q0 < p.qpk) {
                            out[q0 * kHeadDim + d0] = o[mt][0] * inv0;
                            out[q0 * kHeadDim + d1] = o[mt][2] * inv0;
                        }
                        if (q1 < p.qpk) {
                            out[q1 * kHeadDim + d0] = o[mt][1] * inv1;
                            out[q1 * kHeadDim + d1] = o[mt][3] * inv1;
                        }
                    } else {
                        __nv_bfloat16 *out = static_cast<__nv_bfloat16 *>(p.out) + ob;
                        if (q0 < p.qpk) {
                            out[q0 * kHeadDim + d0] = __float2bfloat16_rn(o[mt][0] * inv0);
                            out[q0 * kHeadDim + d1] = __float2bfloat16_rn(o[mt][2] * inv0);
                        }
                        if (q1 < p.qpk) {
                            out[q1 * kHeadDim + d0] = __float2bfloat16_rn(o[mt][1] * inv1);
                            out[q1 * kHeadDim + d1] = __float2bfloat16_rn(o[mt][3] * inv1);
                        }
                    }
                }
            } else {
                const int64_t slot = (int64_t)item + w;
                float *po = p.part_o + slot * p.qpk * kHeadDim;
#pragma unroll
                for (int mt = 0; mt < 8; ++mt) {
                    const int d0 = mt * 16 + gid, d1 = d0 + 8;
                    if (q0 < p.qpk) {
                        po[q0 * kHeadDim + d0] = o[mt][0] * inv0;
                        po[q0 * kHeadDim + d1] = o[mt][2] * inv0;
                    }
                    if (q1 < p.qpk) {
                        po[q1 * kHeadDim + d0] = o[mt][1] * inv1;
                        po[q1 * kHeadDim + d1] = o[mt][3] * inv1;
                    }
                }
                if (gid == 0) {
                    if (q0 < p.qpk) p.part_lse[slot * p.qpk + q0] = m0 + __log2f(t0);
                    if (q1 < p.qpk) p.part_lse[slot * p.qpk + q1] = m1 + __log2f(t1);
                }
            }
            if (x + 1 < x1) {
                do { ++item; } while (off[item + 1] <= x + 1);
                item_begin = off[item];
                item_end = off[item + 1];
                seg_begin = x + 1;
                len = p.item_len[item];
                load_q();
            }
        }
    }
}

// K2: merge the partial slots of items split across warps (one warp/item).
__global__ void __launch_bounds__(256) combine_kernel(const DecodeParams p) {
    const int item = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (item >= p.n_items) return;
    const int64_t P = p.page_off[p.n_items];
    const int64_t b = p.page_off[item], e = p.page_off[item + 1];
    if (b == e) return;
    const int64_t wlo = owner_warp(b, p.n_warps, P), whi = owner_warp(e - 1, p.n_warps, P);
    if (wlo == whi) return;
    const int64_t ob = (int64_t)p.item_orow[item] * p.qpk * kHeadDim;
    for (int q = 0; q < p.qpk; ++q) {
        float mx = -INFINITY;
        for (int64_t s = wlo; s <= whi; ++s) mx = fmaxf(mx, p.part_lse[(item + s) * p.qpk + q]);
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        float den = 0.f;
        for (int64_t s = wlo; s <= whi; ++s) {
            const float wt = fast_exp2(p.part_lse[(item + s) * p.qpk + q] - mx);
            const float4 v = reinterpret_cast<const float4 *>(
                p.part_o + ((item + s) * p.qpk + q) * kHeadDim)[lane];
            acc.x += wt * v.x;
            acc.y += wt * v.y;
            acc.z += wt * v.z;
            acc.w += wt * v.w;
            den += wt;
        }
        const float inv = 1.f / den;
        if (p.out_fp32) {
            reinterpret_cast<float4 *>(static_cast<float *>(p.out) + ob + q * kHeadDim)[lane] =
                make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
        } else {
            __nv_bfloat162 lo = __floats2bfloat162_rn(acc.x * inv, acc.y * inv);
            __nv_bfloat162 hi = __floats2bfloat162_rn(acc.z * inv, acc.w * inv);
            uint2 pk;
            pk.x = *reinterpret_cast<uint32_t *>(&lo);
            pk.y = *reinterpret_cast<uint32_t *>(&hi);
            reinterpret_cast<uint2 *>(static_cast<__nv_bfloat16 *>(p.out) + ob + q * kHeadDim)[lane] = pk;
        }
    }
}

// K4: segmented exclusive prefix of pages per item (one CTA per segment).
__global__ void __launch_bounds__(1024) plan_pages_kernel(const int32_t *item_len,
                                                          const int32_t *seg_items,
                                                          int32_t *page_off) {
    using Scan = cub::BlockScan<int32_t, 1024>;
    __shared__ typename Scan::TempStorage tmp;
    const int s = blockIdx.x;
    const int a = seg_items[s], b = seg_items[s + 1];
    int32_t *out = page_off + a + s;
    int32_t carry = 0;
    for (int base = a; base < b; base += 1024) {
        const int i = base + threadIdx.x;
        const int32_t len = i < b ? item_len[i] : 0;
        const int32_t pages = len > 0 ? (len + kPageTokens - 1) / kPageTokens : 0;
        int32_t excl, total;
        Scan(tmp).ExclusiveSum(pages, excl, total);
        if (i < b) out[i - a] = carry + excl;
        carry += total;
        __syncthreads();
    }
    if (threadIdx.x == 0) out[b - a] = carry;
}

// ------------------------------------------------------------- configs ---
struct KernelCfg {
    int warps, stages;
};
// index = desc.config; 0 is the default
static const KernelCfg kCfgs[] = {{4, 6}, {4, 4}, {8, 3}, {8, 2}, {2, 12}, {4, 8}};
constexpr int kNumCfgs = sizeof(kCfgs) / sizeof(kCfgs[0]);

template <int WARPS, int STAGES>
static int launch_decode(const DecodeParams &prm, int grid, cudaStream_t st) {
    const size_t smem = (size_t)WARPS * STAGES * (kPageBytes + 8);
    static bool attr_set[64] = {false};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!attr_set[dev & 63]) {
        FS_CUDA(cudaFuncSetAttribute(decode_kernel<WARPS, STAGES>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr_set[dev & 63] = true;
    }
    decode_kernel<WARPS, STAGES><<<grid, WARPS * 32, smem, st>>>(prm);
    return cuda_status(cudaGetLastError(), "decode_kernel launch");
}

static int warps_of(int config) { return kCfgs[config].warps; }

}  // namespace fs

using namespace fs;

extern "C" int64_t fs_decode_partial_slots(int device, int32_t n_items, int32_t config) {
    if (config < 0 || config >= kNumCfgs) return -1;
    const int sms = sm_count(device);
    if (sms <= 0) return -1;
    return (int64_t)n_items + (int64_t)sms * warps_of(config);
}

extern "C" int fs_plan_pages(const int32_t *item_len, const int32_t *seg_items, int n_segs,
                             int32_t *page_off, void *stream) {
    FS_CHECK_ARG(n_segs >= 0, "n_segs must be nonnegative");
    if (n_segs == 0) return FS_OK;
    FS_CHECK_ARG(item_len && seg_items && page_off, "null pointer");
    plan_pages_kernel<<<n_segs, 1024, 0, static_cast<cudaStream_t>(stream)>>>(item_len, seg_items,
                                                                              page_off);
    return cuda_status(cudaGetLastError(), "plan_pages_kernel launch");
}

extern "C" int fs_decode_attention(const fs_decode_desc *d, void *stream) {
    FS_CHECK_ARG(d != nullptr, "null descriptor");
    FS_CHECK_ARG(d->q_per_kv >= 1 && d->q_per_kv <= FS_MAX_Q_PER_KV,
                 "q_per_kv must be in [1, %d], got %d", FS_MAX_Q_PER_KV, d->q_per_kv);
    FS_CHECK_ARG(d->n_items >= 0, "n_items must be nonnegative");
    FS_CHECK_ARG(d->config >= 0 && d->config < kNumCfgs, "unknown kernel config %d", d->config);
    if (d->n_items == 0) return FS_OK;
    FS_CHECK_ARG(d->q && d->kv_pool && d->block_table && d->item_seq && d->item_len &&
                     d->item_qrow && d->item_orow && d->page_off && d->out && d->part_o &&
                     d->part_lse,
                 "null pointer in decode descriptor");
    FS_CHECK_ARG((reinterpret_cast<uintptr_t>(d->kv_pool) & 15) == 0, "kv_pool must be 16B aligned");
    const int sms = sm_count(d->device);
    if (sms <= 0) return fail(FS_ECUDA, "cannot query SM count of device %d", d->device);
    const KernelCfg cfg = kCfgs[d->config];
    const int64_t W = (int64_t)sms * cfg.warps;
    FS_CHECK_ARG(d->partial_slots >= (int64_t)d->n_items + W,
                 "partial_slots %lld < required %lld", (long long)d->partial_slots,
                 (long long)(d->n_items + W));
    DecodeParams prm;
    prm.q = static_cast<const __nv_bfloat16 *>(d->q);
    prm.kv = static_cast<const uint8_t *>(d->kv_pool);
    prm.bt = d->block_table;
    prm.bt_stride = d->bt_stride;
    prm.item_seq = d->item_seq;
    prm.item_len = d->item_len;
    prm.item_qrow = d->item_qrow;
    prm.item_orow = d->item_orow;
    prm.page_off = d->page_off;
    prm.n_items = d->n_items;
    prm.qpk = d->q_per_kv;
    prm.scale_log2 = d->scale * 1.4426950408889634f;
    prm.out_fp32 = d->out_fp32;
    prm.out = d->out;
    prm.part_o = d->part_o;
    prm.part_lse = d->part_lse;
    prm.n_warps = W;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    int rc;
    switch (d->config) {
        case 0: rc = launch_decode<4, 6>(prm, sms, st); break;
        case 1: rc = launch_decode<4, 4>(prm, sms, st); break;
        case 2: rc = launch_decode<8, 3>(prm, sms, st); break;
        case 3: rc = launch_decode<8, 2>(prm, sms, st); break;
        case 4: rc = launch_decode<2, 12>(prm, sms, st); break;
        default: rc = launch_decode<4, 8>(prm, sms, st); break;
    }
    if (rc != FS_OK) return rc;
    const int blocks = (d->n_items * 32 + 255) / 256;
    combine_kernel<<<blocks, 256, 0, st>>>(prm);
    return cuda_status(cudaGetLastError(), "combine_kernel launch");
}
