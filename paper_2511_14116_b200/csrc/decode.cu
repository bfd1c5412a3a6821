// K1 (+ fused K2 combine and K3 append) and K4 of the FailSafe B200 hot
// path: a stream-K paged GQA decode for the hybrid-attention step (the
// attention half of refexec.parallel_forward, refexec.py:281-297, with the
// per-head math of _head_attention, refexec.py:85-103).
//
// Work = a list of items, one per (kv head, request) pair a rank serves:
// every request for its TP heads, only routed requests for replicated
// heads.  All items' pages are flattened into one page space of P pages
// and split EVENLY over every warp of a persistent grid (W = SMs x CTAS x
// WARPS): warp w owns pages [w*P/W, (w+1)*P/W).  A warp streams its pages
// through a private ring of STAGES x 8 KiB shared-memory slots filled by TMA
// bulk copies (one cp.async.bulk per page, mbarrier completion), so the
// HBM pipeline never drains at item boundaries and ragged lengths cost
// nothing in balance.  Per 16-token page the warp runs
//     S^T[16 tok x 8 q]   = K[16 x 128]   . Q^T[128 x 8]   (8 mma.m16n8k16)
//     O^T[128 dim x 8 q] += V^T[128 x 16] . P^T[16 x 8]    (8 mma.m16n8k16)
// i.e. tensor cores for the GQA query-group tile (q_per_kv <= 8 queries as
// the mma N dimension), online softmax on the S^T fragments, and P^T made
// from S^T with movmatrix.trans.
//
// Fusions (one launch per layer):
//  * append: the warp holding the page of position len-1 patches the new
//    token's K/V (from the projection output) into the landed smem page and
//    writes it to HBM -- no separate KV-append launch;
//  * combine: a warp covering a whole item writes the normalized output;
//    otherwise it writes (O/l, lse) to partial slot `item + w`, bumps the
//    item's semaphore, and the LAST warp of the item merges the slots and
//    resets the semaphore to 0 (self-cleaning across launches).
#include <cuda_bf16.h>
#include <cub/block/block_scan.cuh>

#include "common.cuh"

namespace fs {

struct DecodeParams {
    const __nv_bfloat16 *q;
    const uint8_t *kv;
    const int32_t *bt;
    int64_t bt_stride;
    const int32_t *item_seq, *item_len, *item_qoff, *item_ooff, *page_off;
    const __nv_bfloat16 *kv_new;            // nullptr: no fused append
    const int32_t *item_koff, *item_voff;
    int32_t *item_sem;
    int32_t n_items;
    int32_t qpk;
    float scale_log2;
    int32_t out_fp32;
    void *out;
    float *part_o, *part_lse;
    int64_t n_warps;  // W of the stream-K partition
    int32_t tab_cache;  // decode_cta_kernel: page_off / item_seq staged in smem (n_items <= kTabItems)
    int32_t early;      // FS_DECODE_EARLY_PREFETCH: tables + first pages read before griddepcontrol.wait
    int32_t l2_pf;      // (early) pages per warp past the ring prefetched into L2 before the wait
};

// items whose page offsets and block-table rows decode_cta_kernel stages in
// shared memory at launch (one load round trip instead of the dependent
// P -> search -> item -> block-table chain before the first page copy)
constexpr int kTabItems = 1024;

__device__ __forceinline__ int64_t owner_warp(int64_t x, int64_t W, int64_t P) {
    return ((x + 1) * W + P - 1) / P - 1;
}

__device__ __forceinline__ bool warp_live(int64_t w, int64_t W, int64_t P) {
    return w * P / W < (w + 1) * P / W;
}

// largest i in [0, n) with off[i] <= x (off is nondecreasing, off[n] > x):
// a warp-cooperative 32-ary search (2 dependent rounds for <= 1024 items)
__device__ __forceinline__ int find_item(const int32_t *off, int n, int64_t x, int lane) {
    int lo = 0, hi = n;  // invariant: off[lo] <= x < off[hi]
    while (hi - lo > 1) {
        const int step = (hi - lo + 31) >> 5;
        const int cand = lo + lane * step;
        const bool ok = cand < hi && off[cand] <= x;
        const unsigned m = __ballot_sync(0xffffffffu, ok);
        const int k = 31 - __clz(m);
        lo += k * step;
        hi = min(hi, lo + step);
    }
    return lo;
}

__device__ __forceinline__ void store_out(const DecodeParams &p, int64_t idx, float v) {
    if (p.out_fp32) static_cast<float *>(p.out)[idx] = v;
    else static_cast<__nv_bfloat16 *>(p.out)[idx] = __float2bfloat16_rn(v);
}

// merge the partial slots of `item` (called by its last-finishing warp).
// Lanes first scan the segments in parallel (lse max / weights per query),
// then stream the partial blocks with 8-16 independent float4 loads in
// flight per lane; the merge sits on the kernel tail, so it is latency-
// optimised rather than bandwidth-optimised.
__device__ __forceinline__ void combine_item(const DecodeParams &p, int item, int64_t wlo,
                                          int64_t whi, int64_t P, int lane) {
    const int qpk = p.qpk;
    const bool all_live = P >= p.n_warps;  // every warp owns >= 1 page
    const int nseg = (int)(whi - wlo + 1);
    const float *lse = p.part_lse + (item + wlo) * qpk;
    const float4 *po = reinterpret_cast<const float4 *>(p.part_o + (item + wlo) * qpk * kHeadDim);
    float mx[FS_MAX_Q_PER_KV], den[FS_MAX_Q_PER_KV];
    float4 acc[FS_MAX_Q_PER_KV];
#pragma unroll
    for (int q = 0; q < FS_MAX_Q_PER_KV; ++q) {
        mx[q] = -INFINITY;
        den[q] = 0.f;
        acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    for (int base = 0; base < nseg; base += 32) {
        const int k = base + lane;
        const bool ok = k < nseg && (all_live || warp_live(wlo + k, p.n_warps, P));
#pragma unroll
        for (int q = 0; q < FS_MAX_Q_PER_KV; ++q)
            if (q < qpk && ok) mx[q] = fmaxf(mx[q], __ldcg(lse + k * qpk + q));
    }
#pragma unroll
    for (int q = 0; q < FS_MAX_Q_PER_KV; ++q)
        for (int sh = 1; sh < 32; sh <<= 1)
            mx[q] = fmaxf(mx[q], __shfl_xor_sync(0xffffffffu, mx[q], sh));
    for (int base = 0; base < nseg; base += 32) {
        const int k = base + lane;
        const bool ok = k < nseg && (all_live || warp_live(wlo + k, p.n_warps, P));
        float wt[FS_MAX_Q_PER_KV];
#pragma unroll
        for (int q = 0; q < FS_MAX_Q_PER_KV; ++q) {
            wt[q] = (q < qpk && ok) ? fast_exp2(__ldcg(lse + k * qpk + q) - mx[q]) : 0.f;
            den[q] += wt[q];
        }
        const unsigned live_mask = __ballot_sync(0xffffffffu, ok);
        const int cnt = min(32, nseg - base);
        const int any_live = __ffs(live_mask) - 1;  // dead slots are never read
        // two segments per round: all 2 x qpk float4 loads are issued before
        // any is consumed, so a round costs one L2 round trip
        for (int j = 0; j < cnt; j += 2) {
            const int ja = ((live_mask >> j) & 1u) ? j : any_live;
            const int jb = (j + 1 < cnt && ((live_mask >> (j + 1)) & 1u)) ? j + 1 : any_live;
            const float4 *ba = po + (int64_t)(base + ja) * qpk * (kHeadDim / 4) + lane;
            const float4 *bb = po + (int64_t)(base + jb) * qpk * (kHeadDim / 4) + lane;
            float4 va[FS_MAX_Q_PER_KV], vb[FS_MAX_Q_PER_KV];
#pragma unroll
            for (int q = 0; q < FS_MAX_Q_PER_KV; ++q) {
                if (q < qpk) {
                    va[q] = __ldcg(ba + q * (kHeadDim / 4));
                    vb[q] = __ldcg(bb + q * (kHeadDim / 4));
                }
            }
#pragma unroll
            for (int q = 0; q < FS_MAX_Q_PER_KV; ++q) {
                if (q < qpk) {
                    // weights of dead / out-of-range segments are 0
                    const float wa = __shfl_sync(0xffffffffu, wt[q], j);
                    const float wb = __shfl_sync(0xffffffffu, j + 1 < 32 ? wt[q] : 0.f,
                                                 (j + 1) & 31);
                    const float wbb = (j + 1 < cnt) ? wb : 0.f;
                    acc[q].x += wa * va[q].x + wbb * vb[q].x;
                    acc[q].y += wa * va[q].y + wbb * vb[q].y;
                    acc[q].z += wa * va[q].z + wbb * vb[q].z;
                    acc[q].w += wa * va[q].w + wbb * vb[q].w;
                }
            }
        }
    }
    const int64_t ob = p.item_ooff[item];
#pragma unroll
    for (int q = 0; q < FS_MAX_Q_PER_KV; ++q) {
        if (q >= qpk) break;
        float d = den[q];
        for (int sh = 1; sh < 32; sh <<= 1) d += __shfl_xor_sync(0xffffffffu, d, sh);
        const float inv = 1.f / d;
        const int64_t o = ob + q * kHeadDim + lane * 4;
        if (p.out_fp32) {
            *reinterpret_cast<float4 *>(static_cast<float *>(p.out) + o) =
                make_float4(acc[q].x * inv, acc[q].y * inv, acc[q].z * inv, acc[q].w * inv);
        } else {
            __nv_bfloat162 lo = __floats2bfloat162_rn(acc[q].x * inv, acc[q].y * inv);
            __nv_bfloat162 hi = __floats2bfloat162_rn(acc[q].z * inv, acc[q].w * inv);
            uint2 pk;
            pk.x = *reinterpret_cast<uint32_t *>(&lo);
            pk.y = *reinterpret_cast<uint32_t *>(&hi);
            *reinterpret_cast<uint2 *>(static_cast<__nv_bfloat16 *>(p.out) + o) = pk;
        }
    }
}

template <int WARPS, int STAGES, int CTAS>
__global__ void __launch_bounds__(WARPS * 32, CTAS) decode_kernel(const DecodeParams p) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gid = lane >> 2, tig = lane & 3;
    // without the caller's guarantee that the preceding kernel writes none
    // of the tables / pages, every read stays behind the PDL wait
    if (!p.early) grid_dependency_wait();

    const int64_t P = p.page_off[p.n_items];
    const int64_t W = p.n_warps;
    const int64_t w = (int64_t)blockIdx.x * WARPS + warp;
    const int64_t x0 = w * P / W, x1 = (w + 1) * P / W;
    grid_launch_dependents();  // the next launch may stage its pages early
    if (x0 >= x1) return;  // warp-uniform; no CTA-wide barriers below

    const uint32_t sbase = smem_u32(smem);
    const uint32_t buf0 = sbase + warp * STAGES * kPageBytes;
    const uint32_t bar0 = sbase + WARPS * STAGES * kPageBytes + warp * STAGES * 8;
    if (lane == 0) {
        for (int s = 0; s < STAGES; ++s) mbar_init(bar0 + 8 * s, 1);
        fence_barrier_init();
        fence_proxy_async();
    }
    __syncwarp();

    const int32_t *off = p.page_off;
    const int first = find_item(off, p.n_items, x0, lane);

    // ---- producer: lane-parallel page-id windows ----
    // lane l holds the page id of page win+l (cur) and win+32+l (nxt); the
    // block-table loads of a window are issued 32 pages before their use,
    // so no global-load latency sits on the per-page critical path.
    const uint64_t pol = policy_evict_first();
    int64_t win = x0;
    int wit = first;  // an item <= the item of page win (walk start)
    auto window_ids = [&](int64_t base) -> int64_t {
        const int64_t y = base + lane;
        int it = wit;
        int64_t pg = 0;
        if (y < x1) {
            while (y >= off[it + 1]) ++it;
            pg = p.bt[(int64_t)p.item_seq[it] * p.bt_stride + (y - off[it])];
        }
        const int last = __shfl_sync(0xffffffffu, it, 31);
        wit = max(wit, last);  // lanes past x1 kept `it` at the walk start
        return pg;
    };
    int64_t cur_pg = window_ids(win);
    int64_t nxt_pg = window_ids(win + 32);
    int64_t px = x0;
    auto issue = [&](int stage) {  // warp-uniform
        if (px - win == 32) {
            win += 32;
            cur_pg = nxt_pg;
            nxt_pg = window_ids(win + 32);
        }
        const int64_t pg = __shfl_sync(0xffffffffu, cur_pg, (int)(px - win));
        if (lane == 0) {
            const uint32_t bar = bar0 + 8 * stage;
            mbar_expect_tx(bar, kPageBytes);
            bulk_g2s(buf0 + stage * kPageBytes, p.kv + pg * kPageBytes, kPageBytes, bar, pol);
        }
        ++px;
    };
    for (int s = 0; s < STAGES && px < x1; ++s) issue(s);

    // ---- consumer state ----
    int item = first;
    int64_t item_begin = off[item], item_end = off[item + 1];
    int64_t seg_begin = x0;
    int len = p.item_len[item];
    uint32_t qf[8][2];
    float m0, m1, l0, l1;
    float o[8][4];

    auto load_q = [&]() {
        const __nv_bfloat16 *qb = p.q + p.item_qoff[item] + gid * kHeadDim;
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
    grid_dependency_wait();  // q / kv_new come from the preceding GEMM
    load_q();

    int stage = 0;
    uint32_t phase = 0;
    for (int64_t x = x0; x < x1; ++x) {
        const uint32_t kb = buf0 + stage * kPageBytes;
        const uint32_t vb = kb + kHalfPage;
        const int pidx = (int)(x - item_begin);
        const int valid = min(kPageTokens, len - pidx * kPageTokens);
        mbar_wait(bar0 + 8 * stage, phase);
        const bool tail = valid < kPageTokens;
        const bool append = p.kv_new != nullptr && valid > 0 &&
                            (len - 1) / kPageTokens == pidx;
        if (tail | append) {
            uint8_t *page_s = smem + (kb - sbase);
            if (tail) {
                // rows >= valid may hold stale bytes; zero the V rows so
                // 0-probability tokens cannot inject NaN/Inf into P.V
                for (int c = valid * 8 + lane; c < kPageTokens * 16; c += 32)
                    if ((c & 127) >= valid * 8)  // both atoms: rows >= valid
                        reinterpret_cast<uint4 *>(page_s + kHalfPage)[c] = make_uint4(0, 0, 0, 0);
            }
            if (append) {
                // fused K3: the new token (position len-1) from the
                // projection output into the landed page (smem) and HBM
                const uint32_t r = (len - 1) % kPageTokens, c = lane & 15, half = lane >> 4;
                const int64_t src = (half ? p.item_voff[item] : p.item_koff[item]) + c * 8;
                uint4 v = *reinterpret_cast<const uint4 *>(p.kv_new + src);
                const uint32_t ofs = half * kHalfPage + swz(r, c);
                *reinterpret_cast<uint4 *>(page_s + ofs) = v;
                const int64_t pg = p.bt[(int64_t)p.item_seq[item] * p.bt_stride + pidx];
                *reinterpret_cast<uint4 *>(const_cast<uint8_t *>(p.kv) + pg * kPageBytes + ofs) = v;
            }
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
        // P^T as a bf16 hi + lo pair (~16 mantissa bits) against the bf16 V
        // pages: two bf16 MMAs per V block (bf16 P alone costs ~1.5e-3 mean
        // relative error on long contexts; north star: 1e-3)
        uint32_t h01, l01, h23, l23;
        split_bf16x2(p0, p1, h01, l01);
        split_bf16x2(p2, p3, h23, l23);
        const uint32_t pb0 = movmatrix_t(h01), pb1 = movmatrix_t(h23);
        const uint32_t pl0 = movmatrix_t(l01), pl1 = movmatrix_t(l23);

        // ---- O^T += V^T . P^T ----
        {
            const int i = lane >> 3;
            const uint32_t r = (lane & 7) + ((i >> 1) << 3);
#pragma unroll
            for (int mt = 0; mt < 8; ++mt) {
                uint32_t a0, a1, a2, a3;
                ldsm_x4_t(vb + swz(r, 2 * mt + (i & 1)), a0, a1, a2, a3);
                mma_bf16(o[mt], a0, a1, a2, a3, pb0, pb1);
                mma_bf16(o[mt], a0, a1, a2, a3, pl0, pl1);
            }
        }
        __syncwarp();
        if (px < x1) issue(stage);
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
                const int64_t ob = p.item_ooff[item];
#pragma unroll
                for (int mt = 0; mt < 8; ++mt) {
                    const int d0 = mt * 16 + gid, d1 = d0 + 8;
                    if (q0 < p.qpk) {
                        store_out(p, ob + q0 * kHeadDim + d0, o[mt][0] * inv0);
                        store_out(p, ob + q0 * kHeadDim + d1, o[mt][2] * inv0);
                    }
                    if (q1 < p.qpk) {
                        store_out(p, ob + q1 * kHeadDim + d0, o[mt][1] * inv1);
                        store_out(p, ob + q1 * kHeadDim + d1, o[mt][3] * inv1);
                    }
                }
            } else {
                const int64_t slot = (int64_t)item + w;
                float *po = p.part_o + slot * p.qpk * kHeadDim;
#pragma unroll
                for (int mt = 0; mt < 8; ++mt) {
                    const int d0 = mt * 16 + gid, d1 = d0 + 8;
                    if (q0 < p.qpk) {
                        __stcg(po + q0 * kHeadDim + d0, o[mt][0] * inv0);
                        __stcg(po + q0 * kHeadDim + d1, o[mt][2] * inv0);
                    }
                    if (q1 < p.qpk) {
                        __stcg(po + q1 * kHeadDim + d0, o[mt][1] * inv1);
                        __stcg(po + q1 * kHeadDim + d1, o[mt][3] * inv1);
                    }
                }
                if (gid == 0) {
                    if (q0 < p.qpk) __stcg(p.part_lse + slot * p.qpk + q0, m0 + __log2f(t0));
                    if (q1 < p.qpk) __stcg(p.part_lse + slot * p.qpk + q1, m1 + __log2f(t1));
                }
                // publish, count, and let the last warp of the item merge
                __threadfence();
                __syncwarp();
                int prev = 0;
                if (lane == 0) prev = atomicAdd(p.item_sem + item, 1);
                prev = __shfl_sync(0xffffffffu, prev, 0);
                const int64_t wlo = owner_warp(item_begin, W, P);
                const int64_t whi = owner_warp(item_end - 1, W, P);
                int nseg = (int)(whi - wlo + 1);
                if (P < W) {  // some warps own no page; count the live ones
                    nseg = 0;
                    for (int64_t s = wlo; s <= whi; ++s) nseg += warp_live(s, W, P);
                }
                if (prev == nseg - 1) {
                    __threadfence();
                    combine_item(p, item, wlo, whi, P, lane);
                    if (lane == 0) p.item_sem[item] = 0;
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

#include "decode_cta.cuh"

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
// (warps per CTA, ring stages per warp, CTAs per SM); index = desc.config.
// Pages in flight per SM = warps * stages * ctas (8 KiB each).
// kind 0: warp-level stream-K (decode_kernel); kind 1: CTA-level stream-K
// (decode_cta_kernel, per-CTA smem merge).
#define FS_DECODE_CONFIGS(X) \
    X(0, 8, 2, 1, 1)         \
    X(1, 4, 4, 1, 1)         \
    X(2, 8, 3, 1, 1)         \
    X(3, 16, 1, 1, 1)        \
    X(4, 12, 1, 1, 1)        \
    X(5, 6, 2, 1, 1)         \
    X(6, 4, 2, 2, 1)         \
    X(7, 4, 4, 1, 0)         \
    X(8, 4, 3, 1, 0)         \
    X(9, 8, 2, 1, 0)         \
    X(10, 2, 8, 1, 0)

struct KernelCfg {
    int warps, stages, ctas, kind;
};
#define FS_CFG_ROW(i, w, s, c, k) {w, s, c, k},
static const KernelCfg kCfgs[] = {FS_DECODE_CONFIGS(FS_CFG_ROW)};
#undef FS_CFG_ROW
constexpr int kNumCfgs = sizeof(kCfgs) / sizeof(kCfgs[0]);

template <int WARPS, int STAGES, int CTAS, int KIND>
static int launch_decode(const DecodeParams &prm, int sms, cudaStream_t st) {
    size_t smem = (size_t)WARPS * STAGES * (kPageBytes + 8);
    if (KIND == 1)
        smem += (size_t)WARPS * (2 * FS_MAX_Q_PER_KV + FS_MAX_Q_PER_KV * kMergeStride) * 4;
    // the item-table stage (decode_cta_kernel) when it fits next to the
    // ring and the merge area; the smem size is fixed per kernel either way
    const bool tab_fits = KIND == 1 && smem + (size_t)(2 * kTabItems + 1) * 4 <= 227 * 1024;
    if (tab_fits) smem += (size_t)(2 * kTabItems + 1) * 4;
    DecodeParams prm2 = prm;
    prm2.tab_cache = tab_fits && prm.n_items <= kTabItems;
    static bool attr_set[64] = {false};
    int dev = 0;
    cudaGetDevice(&dev);
    auto fn = KIND == 0 ? decode_kernel<WARPS, STAGES, CTAS> : decode_cta_kernel<WARPS, STAGES>;
    if (!attr_set[dev & 63]) {
        FS_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        FS_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout,
                                     (int)cudaSharedmemCarveoutMaxShared));
        attr_set[dev & 63] = true;
    }
    // PDL: with FS_DECODE_EARLY_PREFETCH the prologue (table lookups, first
    // TMA page loads) may overlap the tail of the preceding kernel and the
    // kernel waits (griddepcontrol.wait) before its first read of q / kv_new
    // and before any global write; without it the wait comes first.
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(sms * CTAS);
    lc.blockDim = dim3(WARPS * 32);
    lc.dynamicSmemBytes = smem;
    lc.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = attr;
    lc.numAttrs = 1;
    FS_CUDA(cudaLaunchKernelEx(&lc, fn, prm2));
    return cuda_status(cudaGetLastError(), "decode_kernel launch");
}

// stream-K partition units (warps for kind 0, CTAs for kind 1) per SM
static int units_of(int config) {
    const KernelCfg &k = kCfgs[config];
    return k.kind == 0 ? k.warps * k.ctas : k.ctas;
}

}  // namespace fs

using namespace fs;

extern "C" int64_t fs_decode_partial_slots(int device, int32_t n_items, int32_t config) {
    if (config < -1 || config >= kNumCfgs) return -1;
    const int sms = sm_count(device);
    if (sms <= 0) return -1;
    int warps = 0;  // config -1: enough for every configuration
    for (int c = 0; c < kNumCfgs; ++c)
        if (config == -1 || c == config) warps = warps > units_of(c) ? warps : units_of(c);
    return (int64_t)n_items + (int64_t)sms * warps;
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
                     d->item_qoff && d->item_ooff && d->page_off && d->out && d->part_o &&
                     d->part_lse && d->item_sem,
                 "null pointer in decode descriptor");
    FS_CHECK_ARG(!d->kv_new || (d->item_koff && d->item_voff),
                 "fused append needs item_koff and item_voff");
    FS_CHECK_ARG((reinterpret_cast<uintptr_t>(d->kv_pool) & 15) == 0, "kv_pool must be 16B aligned");
    const int sms = sm_count(d->device);
    if (sms <= 0) return fail(FS_ECUDA, "cannot query SM count of device %d", d->device);
    const int64_t W = (int64_t)sms * units_of(d->config);
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
    prm.item_qoff = d->item_qoff;
    prm.item_ooff = d->item_ooff;
    prm.page_off = d->page_off;
    prm.kv_new = static_cast<const __nv_bfloat16 *>(d->kv_new);
    prm.item_koff = d->item_koff;
    prm.item_voff = d->item_voff;
    prm.item_sem = d->item_sem;
    prm.n_items = d->n_items;
    prm.qpk = d->q_per_kv;
    prm.scale_log2 = d->scale * 1.4426950408889634f;
    prm.out_fp32 = d->out_fp32;
    prm.out = d->out;
    prm.part_o = d->part_o;
    prm.part_lse = d->part_lse;
    prm.n_warps = W;
    prm.early = (d->flags & FS_DECODE_EARLY_PREFETCH) ? 1 : 0;
    // (early) each warp also sends its 2 pages past the ring to L2 before
    // griddepcontrol.wait, while the QKV GEMM leaves HBM under-used: C3 N=8
    // rank step -1.8%, N=5 -0.9%, C2 -0.4%; 6+ pages, or a standing L2
    // prefetch distance ahead of the ring, are slower
    // (profiles/r02_k1_experiments/README.md).  FS_K1_L2_PREFETCH overrides.
    static const int l2_pf = [] {
        const char *e = getenv("FS_K1_L2_PREFETCH");
        return e ? std::max(0, std::min(28, atoi(e))) : 2;
    }();
    prm.l2_pf = prm.early ? l2_pf : 0;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    switch (d->config) {
#define FS_CFG_CASE(i, w, s, c, k) \
    case i: return launch_decode<w, s, c, k>(prm, sms, st);
        FS_DECODE_CONFIGS(FS_CFG_CASE)
#undef FS_CFG_CASE
        default: return fail(FS_EVALIDATION, "unknown kernel config %d", d->config);
    }
}
