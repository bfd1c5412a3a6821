// K8: paged chunked-prefill GQA attention for Alg. 1 batches (the multi-row
// form of refexec._head_attention, refexec.py:85-103, over the batches of
// scheduler.build_prefill_batch, scheduler.py:189-245).
//
// Tile = 64 query rows = (64 / q_per_kv) consecutive chunk tokens x the
// q_per_kv query heads of one KV head, so every K/V page a tile streams
// feeds 64 rows of tensor-core work (the GQA group shares it).  A CTA is 4
// consumer warps (16 rows each) + 2 producer warps; warp 4 streams the
// tile's pages with TMA bulk copies into a STAGES-deep ring (full barrier:
// transaction bytes; empty barrier: one arrive per consumer warp).  Per
// 16-token page each consumer warp runs FlashAttention-2 style
//     S[16 x 16]   = Q[16 x 128] . K^T      (16 mma.m16n8k16, K via ldmatrix)
//     O[16 x 128] += P[16 x 16]  . V        (16 mma, V via ldmatrix.trans)
// with the causal mask (key position <= row position) applied only on the
// pages that straddle the tile's diagonal.  The page layout (swizzled 16 B
// chunks) is the one the decode kernel and the writers share.
//
// P.V: P is split into a bf16 hi + lo pair (~16 mantissa bits) against the
// bf16 V pages -- two MMAs; bf16 P alone costs ~1.5e-3 mean relative error
// on long contexts, above the 1e-3 the north star allows.  The producer warps zero
// stale rows past an item's last token and publish each page on a third
// barrier.
//
// Long causal ranges are split into page ranges (fs_plan_prefill_tiles) so
// a handful of long requests still fill 148 SMs; split tiles write
// (O/l, log2-sum-exp) partials that prefill_combine_kernel merges in the
// same call.
#include <cuda_bf16.h>

#include <algorithm>
#include <functional>
#include <numeric>
#include <vector>

#include "common.cuh"

namespace fs {

constexpr int kTileRows = 64;
constexpr int kConsumerWarps = 4;
constexpr int kPrefillStages = 6;

struct PrefillParams {
    const __nv_bfloat16 *q;
    void *out;
    int64_t q_stride, o_stride;
    int32_t out_fp32;
    const uint8_t *kv;
    const int32_t *bt;
    int64_t bt_stride;
    const int32_t *item_seq, *item_start, *item_len, *item_qoff, *item_ooff;
    const int32_t *tile_item, *tile_tok0, *tile_page0, *tile_page1, *tile_slot;
    const int32_t *comb_item, *comb_tok0, *comb_slot0, *comb_nsplit;
    int32_t qpk, tpt;  // q heads per kv head, chunk tokens per tile
    int32_t rows;      // query rows per tile (= partial rows per slot): 64 or 128
    float scale_log2;
    float *part_o;      // split partials O / l (fp32)
    float *part_lse;
};

template <int STAGES>
__global__ void __launch_bounds__((kConsumerWarps + 2) * 32) prefill_kernel(const PrefillParams p) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int t = blockIdx.x;
    const int item = p.tile_item[t];
    const int tok0 = p.tile_tok0[t];
    const int pg0 = p.tile_page0[t];
    const int npg = p.tile_page1[t] - pg0;
    const uint32_t buf0 = smem_u32(smem);
    const uint32_t full0 = buf0 + STAGES * kPageBytes;
    const uint32_t empty0 = full0 + STAGES * 8;
    const uint32_t ready0 = empty0 + STAGES * 8;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(full0 + 8 * s, 1);
            mbar_init(empty0 + 8 * s, kConsumerWarps);
            mbar_init(ready0 + 8 * s, 2);
        }
        fence_barrier_init();
    }
    __syncthreads();

    if (warp >= kConsumerWarps) {
        // ---- producer warps: warp 4 issues the TMA ring (refilling the
        // stage released two pages ago, so the refill never waits on the
        // page being computed); warps 4 and 5 each zero the stale rows of
        // half of every landed V half-page and arrive on `ready` ----
        const int cw = warp - kConsumerWarps;
        const int64_t row = (int64_t)p.item_seq[item] * p.bt_stride + pg0;
        const int kv_end = p.item_start[item] + p.item_len[item];
        const uint64_t pol = policy_evict_first();
        int64_t ids = 0;  // lane l: page id of page (k & ~31) + l
        auto page_id = [&](int k) -> int64_t {  // warp-uniform k
            if ((k & 31) == 0) ids = k + lane < npg ? p.bt[row + k + lane] : 0;
            return __shfl_sync(0xffffffffu, ids, k & 31);
        };
        auto issue = [&](int k, int64_t pg) {
            if (lane == 0) {
                const int s = k % STAGES;
                mbar_expect_tx(full0 + 8 * s, kPageBytes);
                bulk_g2s(buf0 + s * kPageBytes, p.kv + pg * kPageBytes, kPageBytes, full0 + 8 * s,
                         pol);
            }
        };
        int issued = 0;
        if (cw == 0)
            for (; issued < min(STAGES, npg); ++issued) issue(issued, page_id(issued));
        for (int k = 0; k < npg; ++k) {
            if (cw == 0 && k >= 2 && issued < npg) {
                const int kr = k - 2, sr = kr % STAGES;
                const int64_t pg = page_id(issued);  // warp-uniform, before the wait
                if (lane == 0) mbar_wait(empty0 + 8 * sr, (kr / STAGES) & 1);
                __syncwarp();
                issue(issued, pg);
                ++issued;
            }
            const int s = k % STAGES;
            mbar_wait(full0 + 8 * s, (k / STAGES) & 1);
            // rows past the item's last written position may hold stale
            // bytes: zero them in this warp's atom (their P is 0, but 0 *
            // NaN/Inf is not)
            const int rows_ok = kv_end - (pg0 + k) * kPageTokens;
            if (rows_ok < kPageTokens) {
                uint4 *vh = reinterpret_cast<uint4 *>(smem + s * kPageBytes + kHalfPage +
                                                      cw * kAtomBytes);
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const int idx = c * 32 + lane;  // row idx >> 3 of the atom
                    if ((idx >> 3) >= rows_ok) vh[idx] = make_uint4(0, 0, 0, 0);
                }
            }
            // the stage is refilled by TMA (async proxy) later: order these
            // generic-proxy writes before it
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) mbar_arrive_cta(ready0 + 8 * s);
        }
        return;
    }

    // ---- consumer warp: rows warp*16 + gid (row a) and + 8 (row b) ----
    const int gid = lane >> 2, tig = lane & 3;
    const int start = p.item_start[item], n = p.item_len[item];
    const int qpk = p.qpk;
    const int rows_used = p.tpt * qpk;
    const int ra = warp * 16 + gid, rb = ra + 8;
    // padding rows (r >= rows_used) and tokens past the chunk reuse the
    // chunk's last valid token so no row is fully masked; they are not stored
    const int ta = min(tok0 + min(ra, rows_used - 1) / qpk, n - 1);
    const int tb = min(tok0 + min(rb, rows_used - 1) / qpk, n - 1);
    const int ha = ra % qpk, hb = rb % qpk;
    const bool va = ra < rows_used && tok0 + ra / qpk < n;
    const bool vb = rb < rows_used && tok0 + rb / qpk < n;
    const int pa = start + ta, pb = start + tb;  // row positions (causal limit)

    uint32_t qf[8][4];
    {
        const __nv_bfloat16 *qa = p.q + p.item_qoff[item] + (int64_t)ta * p.q_stride + ha * kHeadDim;
        const __nv_bfloat16 *qb = p.q + p.item_qoff[item] + (int64_t)tb * p.q_stride + hb * kHeadDim;
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
            qf[ks][0] = *reinterpret_cast<const uint32_t *>(qa + ks * 16 + 2 * tig);
            qf[ks][1] = *reinterpret_cast<const uint32_t *>(qb + ks * 16 + 2 * tig);
            qf[ks][2] = *reinterpret_cast<const uint32_t *>(qa + ks * 16 + 8 + 2 * tig);
            qf[ks][3] = *reinterpret_cast<const uint32_t *>(qb + ks * 16 + 8 + 2 * tig);
        }
    }
    float o[16][4];
#pragma unroll
    for (int nt = 0; nt < 16; ++nt) o[nt][0] = o[nt][1] = o[nt][2] = o[nt][3] = 0.f;
    float ma = -INFINITY, mb = -INFINITY, la = 0.f, lb = 0.f;
    const int pmin = start + tok0;  // smallest row position of the tile
    const int mi = lane >> 3;
    const uint32_t krow = (lane & 7) + ((mi >> 1) << 3), kch = mi & 1;
    const uint32_t vrow = (lane & 7) + ((mi & 1) << 3), vch = mi >> 1;

    for (int k = 0; k < npg; ++k) {
        const int s = k % STAGES;
        const uint32_t kb = buf0 + s * kPageBytes, vbuf = kb + kHalfPage;
        mbar_wait(ready0 + 8 * s, (k / STAGES) & 1);

        float sc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
            uint32_t b0, b1, b2, b3;
            ldsm_x4(kb + swz(krow, 2 * ks + kch), b0, b1, b2, b3);
            mma_bf16(sc[0], qf[ks][0], qf[ks][1], qf[ks][2], qf[ks][3], b0, b1);
            mma_bf16(sc[1], qf[ks][0], qf[ks][1], qf[ks][2], qf[ks][3], b2, b3);
        }
        const int kp0 = (pg0 + k) * kPageTokens;
        const bool diag = kp0 + kPageTokens - 1 > pmin;  // warp-uniform
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                float v = sc[nt][e] * p.scale_log2;
                if (diag) {
                    const int key = kp0 + nt * 8 + 2 * tig + (e & 1);
                    if (key > (e < 2 ? pa : pb)) v = -INFINITY;
                }
                sc[nt][e] = v;
            }
        }
        float xa = fmaxf(fmaxf(sc[0][0], sc[0][1]), fmaxf(sc[1][0], sc[1][1]));
        float xb = fmaxf(fmaxf(sc[0][2], sc[0][3]), fmaxf(sc[1][2], sc[1][3]));
        xa = fmaxf(xa, __shfl_xor_sync(0xffffffffu, xa, 1));
        xa = fmaxf(xa, __shfl_xor_sync(0xffffffffu, xa, 2));
        xb = fmaxf(xb, __shfl_xor_sync(0xffffffffu, xb, 1));
        xb = fmaxf(xb, __shfl_xor_sync(0xffffffffu, xb, 2));
        const float na = fmaxf(ma, xa), nb = fmaxf(mb, xb);
        const float ua = na == -INFINITY ? 0.f : na, ub = nb == -INFINITY ? 0.f : nb;
        const float aa = fast_exp2(ma - ua), ab = fast_exp2(mb - ub);
        ma = na;
        mb = nb;
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
            sc[nt][0] = fast_exp2(sc[nt][0] - ua);
            sc[nt][1] = fast_exp2(sc[nt][1] - ua);
            sc[nt][2] = fast_exp2(sc[nt][2] - ub);
            sc[nt][3] = fast_exp2(sc[nt][3] - ub);
        }
        la = la * aa + sc[0][0] + sc[0][1] + sc[1][0] + sc[1][1];
        lb = lb * ab + sc[0][2] + sc[0][3] + sc[1][2] + sc[1][3];
#pragma unroll
        for (int nt = 0; nt < 16; ++nt) {
            o[nt][0] *= aa;
            o[nt][1] *= aa;
            o[nt][2] *= ab;
            o[nt][3] *= ab;
        }
        // P as a bf16 hi + lo pair against the bf16 V page (two MMAs)
        uint32_t a0, a1, a2, a3, e0, e1, e2, e3;
        split_bf16x2(sc[0][0], sc[0][1], a0, e0);
        split_bf16x2(sc[0][2], sc[0][3], a1, e1);
        split_bf16x2(sc[1][0], sc[1][1], a2, e2);
        split_bf16x2(sc[1][2], sc[1][3], a3, e3);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            uint32_t b0, b1, b2, b3;
            ldsm_x4_t(vbuf + swz(vrow, 2 * j + vch), b0, b1, b2, b3);
            mma_bf16(o[2 * j], a0, a1, a2, a3, b0, b1);
            mma_bf16(o[2 * j + 1], a0, a1, a2, a3, b2, b3);
            mma_bf16(o[2 * j], e0, e1, e2, e3, b0, b1);
            mma_bf16(o[2 * j + 1], e0, e1, e2, e3, b2, b3);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive_cta(empty0 + 8 * s);
    }

    la += __shfl_xor_sync(0xffffffffu, la, 1);
    la += __shfl_xor_sync(0xffffffffu, la, 2);
    lb += __shfl_xor_sync(0xffffffffu, lb, 1);
    lb += __shfl_xor_sync(0xffffffffu, lb, 2);
    const float ia = la > 0.f ? 1.f / la : 0.f, ib = lb > 0.f ? 1.f / lb : 0.f;
    const int slot = p.tile_slot[t];
    if (slot < 0) {
        const int64_t oa = p.item_ooff[item] + (int64_t)ta * p.o_stride + ha * kHeadDim;
        const int64_t ob = p.item_ooff[item] + (int64_t)tb * p.o_stride + hb * kHeadDim;
        if (p.out_fp32) {
            float *o32 = static_cast<float *>(p.out);
#pragma unroll
            for (int nt = 0; nt < 16; ++nt) {
                const int d = nt * 8 + 2 * tig;
                if (va) *reinterpret_cast<float2 *>(o32 + oa + d) = make_float2(o[nt][0] * ia, o[nt][1] * ia);
                if (vb) *reinterpret_cast<float2 *>(o32 + ob + d) = make_float2(o[nt][2] * ib, o[nt][3] * ib);
            }
        } else {
            __nv_bfloat16 *o16 = static_cast<__nv_bfloat16 *>(p.out);
#pragma unroll
            for (int nt = 0; nt < 16; ++nt) {
                const int d = nt * 8 + 2 * tig;
                if (va) *reinterpret_cast<uint32_t *>(o16 + oa + d) = pack_bf16(o[nt][0] * ia, o[nt][1] * ia);
                if (vb) *reinterpret_cast<uint32_t *>(o16 + ob + d) = pack_bf16(o[nt][2] * ib, o[nt][3] * ib);
            }
        }
    } else {
        float *po = p.part_o + (int64_t)slot * kTileRows * kHeadDim;
#pragma unroll
        for (int nt = 0; nt < 16; ++nt) {
            const int d = nt * 8 + 2 * tig;
            *reinterpret_cast<float2 *>(po + ra * kHeadDim + d) = make_float2(o[nt][0] * ia, o[nt][1] * ia);
            *reinterpret_cast<float2 *>(po + rb * kHeadDim + d) = make_float2(o[nt][2] * ib, o[nt][3] * ib);
        }
        if (tig == 0) {
            p.part_lse[(int64_t)slot * kTileRows + ra] = la > 0.f ? ma + __log2f(la) : -INFINITY;
            p.part_lse[(int64_t)slot * kTileRows + rb] = lb > 0.f ? mb + __log2f(lb) : -INFINITY;
        }
    }
}

// merge the page-range splits of one (item, token tile); grid.y = 64-row
// slabs of the tile: 4 threads per row,
// 32 dims each, log-sum-exp weights in base 2
// One CTA = 16 rows x 16 threads of one combine group; a thread owns 8 dims
// of its row (a warp reads two contiguous 512-B partial rows per load).  The
// split loop keeps 4 splits' loads in flight (the merge is latency-bound, not
// bandwidth-bound, at the few-hundred-KB-per-SM sizes K8 produces).  Launched
// with PDL: it is scheduled during the attention kernel's tail and waits in
// griddepcontrol.wait for its partials.
constexpr int kCombRows = 16;

__global__ void __launch_bounds__(256) prefill_combine_kernel(const PrefillParams p) {
    grid_dependency_wait();
    const int g = blockIdx.x;
    const int item = p.comb_item[g], tok0 = p.comb_tok0[g];
    const int slot0 = p.comb_slot0[g], ns = p.comb_nsplit[g];
    const int r = blockIdx.y * kCombRows + (threadIdx.x >> 4), c = threadIdx.x & 15;
    const int qpk = p.qpk, rows_used = p.tpt * qpk;
    if (r >= rows_used) return;
    const int tok = tok0 + r / qpk, h = r % qpk;
    if (tok >= p.item_len[item]) return;
    const float *lse = p.part_lse + (int64_t)slot0 * p.rows + r;
    float mx = -INFINITY;
    for (int s0 = 0; s0 < ns; s0 += 8) {
        float v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = s0 + i < ns ? __ldg(lse + (int64_t)(s0 + i) * p.rows) : -INFINITY;
#pragma unroll
        for (int i = 0; i < 8; ++i) mx = fmaxf(mx, v[i]);
    }
    // this thread's 8 dims of every split: two float4 per split slot
    const float4 *po = reinterpret_cast<const float4 *>(p.part_o + ((int64_t)slot0 * p.rows + r) * kHeadDim) + 2 * c;
    const int64_t sstr = (int64_t)p.rows * (kHeadDim / 4);  // float4s per split slot
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    float den = 0.f;
    for (int s0 = 0; s0 < ns; s0 += 4) {
        float w[4];
        float4 va[4], vb[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            w[i] = 0.f;
            va[i] = vb[i] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (s0 + i < ns) {
                const float l = __ldg(lse + (int64_t)(s0 + i) * p.rows);
                w[i] = l == -INFINITY ? 0.f : fast_exp2(l - mx);
                va[i] = __ldg(po + (s0 + i) * sstr);
                vb[i] = __ldg(po + (s0 + i) * sstr + 1);
            }
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            den += w[i];
            acc[0] += w[i] * va[i].x;
            acc[1] += w[i] * va[i].y;
            acc[2] += w[i] * va[i].z;
            acc[3] += w[i] * va[i].w;
            acc[4] += w[i] * vb[i].x;
            acc[5] += w[i] * vb[i].y;
            acc[6] += w[i] * vb[i].z;
            acc[7] += w[i] * vb[i].w;
        }
    }
    const float inv = den > 0.f ? 1.f / den : 0.f;
    const int64_t o = p.item_ooff[item] + (int64_t)tok * p.o_stride + h * kHeadDim + c * 8;
    if (p.out_fp32) {
        float4 *dst = reinterpret_cast<float4 *>(static_cast<float *>(p.out) + o);
        dst[0] = make_float4(acc[0] * inv, acc[1] * inv, acc[2] * inv, acc[3] * inv);
        dst[1] = make_float4(acc[4] * inv, acc[5] * inv, acc[6] * inv, acc[7] * inv);
        return;
    }
    uint4 pk;
    pk.x = pack_bf16(acc[0] * inv, acc[1] * inv);
    pk.y = pack_bf16(acc[2] * inv, acc[3] * inv);
    pk.z = pack_bf16(acc[4] * inv, acc[5] * inv);
    pk.w = pack_bf16(acc[6] * inv, acc[7] * inv);
    *reinterpret_cast<uint4 *>(static_cast<__nv_bfloat16 *>(p.out) + o) = pk;
}

#include "prefill_tc.cuh"

// query rows per tile of each kernel variant (0: tcgen05 with two 128-row
// halves, 1: mma.sync, 2: tcgen05 with one 128-row half)
static int variant_rows(int variant) {
    return variant == 0 || variant == 3 ? 2 * kTcRows : variant == 1 ? kTileRows : variant == 2 ? kTcRows : -1;
}

}  // namespace fs

using namespace fs;

extern "C" int fs_prefill_tokens_per_tile(int q_per_kv, int variant) {
    if (q_per_kv < 1 || q_per_kv > FS_MAX_Q_PER_KV || variant_rows(variant) < 0) return -1;
    return variant_rows(variant) / q_per_kv;
}

extern "C" int fs_plan_prefill_tiles(int32_t n_items, const int32_t *item_start,
                                     const int32_t *item_len, int32_t q_per_kv, int32_t variant,
                                     int32_t target_units, int32_t max_tiles, int32_t *tile_item,
                                     int32_t *tile_tok0, int32_t *tile_page0, int32_t *tile_page1,
                                     int32_t *tile_slot, int32_t *n_tiles, int32_t max_comb,
                                     int32_t *comb_item, int32_t *comb_tok0, int32_t *comb_slot0,
                                     int32_t *comb_nsplit, int32_t *n_comb, int32_t *n_slots) {
    FS_CHECK_ARG(n_items >= 0, "n_items must be nonnegative");
    FS_CHECK_ARG(q_per_kv >= 1 && q_per_kv <= FS_MAX_Q_PER_KV, "q_per_kv must be in [1, %d]",
                 FS_MAX_Q_PER_KV);
    FS_CHECK_ARG(variant_rows(variant) > 0, "unknown prefill kernel variant %d", variant);
    FS_CHECK_ARG(n_tiles && n_comb && n_slots, "null pointer");
    FS_CHECK_ARG(n_items == 0 || (item_start && item_len), "null item arrays");
    const int tpt = variant_rows(variant) / q_per_kv;
    struct Tok { int32_t item, tok0, pages; };
    std::vector<Tok> toks;
    int64_t work = 0;
    for (int i = 0; i < n_items; ++i) {
        FS_CHECK_ARG(item_start[i] >= 0 && item_len[i] >= 0, "item %d: negative start/len", i);
        for (int t0 = 0; t0 < item_len[i]; t0 += tpt) {
            const int last = std::min(t0 + tpt, item_len[i]) - 1;
            const int pages = (item_start[i] + last + 1 + kPageTokens - 1) / kPageTokens;
            toks.push_back({i, t0, pages});
            work += pages;
        }
    }
    // Pages per split: at least 32 (a split below that is all pipeline
    // fill).  target_units is the number of CTAs that run at once (one
    // tcgen05 CTA per SM); the split size is the one whose tiles, dispatched
    // heaviest first onto target_units slots (what the block scheduler does
    // with the sorted tile list), finish earliest -- each tile costing its
    // pages plus kTileOverheadPages for its prologue / epilogue / combine
    // share (measured: ~8 us per tile vs ~0.28 us per page on B200).
    constexpr int64_t kTileOverheadPages = 28;
    const int64_t units = std::max<int64_t>(1, target_units);
    int32_t max_pages = 1;
    for (const Tok &tk : toks) max_pages = std::max(max_pages, tk.pages);
    std::vector<int64_t> sizes, load;
    auto makespan = [&](int32_t q) {
        sizes.clear();
        for (const Tok &tk : toks) {
            const int ns = (tk.pages + q - 1) / q;
            for (int s = 0; s < ns; ++s)
                sizes.push_back((int64_t)tk.pages * (s + 1) / ns - (int64_t)tk.pages * s / ns);
        }
        std::sort(sizes.begin(), sizes.end(), std::greater<int64_t>());
        load.assign((size_t)std::min<int64_t>(units, (int64_t)sizes.size()), 0);
        std::make_heap(load.begin(), load.end(), std::greater<int64_t>());
        int64_t worst = 0;
        for (int64_t w : sizes) {  // least-loaded slot takes the next tile
            std::pop_heap(load.begin(), load.end(), std::greater<int64_t>());
            load.back() += w + kTileOverheadPages;
            worst = std::max(worst, load.back());
            std::push_heap(load.begin(), load.end(), std::greater<int64_t>());
        }
        return worst;
    };
    int32_t per = std::max<int32_t>(32, max_pages);
    int64_t best = makespan(per);
    for (int32_t q = 32; q < max_pages; q += std::max(1, q / 12)) {
        const int64_t m = makespan(q);
        if (m < best) best = m, per = q;
    }
    struct Tile { int32_t item, tok0, p0, p1, slot; };
    std::vector<Tile> tiles;
    int32_t slots = 0, nc = 0;
    for (const Tok &tk : toks) {
        const int ns = (tk.pages + per - 1) / per;
        if (ns <= 1) {
            tiles.push_back({tk.item, tk.tok0, 0, tk.pages, -1});
            continue;
        }
        FS_CHECK_ARG(nc < max_comb, "combine list too small (%d)", max_comb);
        comb_item[nc] = tk.item;
        comb_tok0[nc] = tk.tok0;
        comb_slot0[nc] = slots;
        comb_nsplit[nc] = ns;
        ++nc;
        for (int s = 0; s < ns; ++s) {
            const int32_t a = (int32_t)((int64_t)tk.pages * s / ns);
            const int32_t b = (int32_t)((int64_t)tk.pages * (s + 1) / ns);
            tiles.push_back({tk.item, tk.tok0, a, b, slots + s});
        }
        slots += ns;
    }
    FS_CHECK_ARG((int64_t)tiles.size() <= max_tiles, "tile list too small (%d < %zu)", max_tiles,
                 tiles.size());
    std::stable_sort(tiles.begin(), tiles.end(),
                     [](const Tile &x, const Tile &y) { return x.p1 - x.p0 > y.p1 - y.p0; });
    for (size_t i = 0; i < tiles.size(); ++i) {
        tile_item[i] = tiles[i].item;
        tile_tok0[i] = tiles[i].tok0;
        tile_page0[i] = tiles[i].p0;
        tile_page1[i] = tiles[i].p1;
        tile_slot[i] = tiles[i].slot;
    }
    *n_tiles = (int32_t)tiles.size();
    *n_comb = nc;
    *n_slots = slots;
    return FS_OK;
}

extern "C" int fs_prefill_attention(const fs_prefill_desc *d, void *stream) {
    FS_CHECK_ARG(d != nullptr, "null descriptor");
    FS_CHECK_ARG(d->q_per_kv >= 1 && d->q_per_kv <= FS_MAX_Q_PER_KV,
                 "q_per_kv must be in [1, %d], got %d", FS_MAX_Q_PER_KV, d->q_per_kv);
    FS_CHECK_ARG(d->n_tiles >= 0 && d->n_comb >= 0, "negative tile / combine count");
    if (d->n_tiles == 0) return FS_OK;
    FS_CHECK_ARG(d->q && d->out && d->kv_pool && d->block_table && d->item_seq && d->item_start &&
                     d->item_len && d->item_qoff && d->item_ooff && d->tile_item && d->tile_tok0 &&
                     d->tile_page0 && d->tile_page1 && d->tile_slot,
                 "null pointer in prefill descriptor");
    FS_CHECK_ARG(d->n_comb == 0 || (d->comb_item && d->comb_tok0 && d->comb_slot0 &&
                                    d->comb_nsplit && d->part_o && d->part_lse),
                 "split tiles need the combine list and partial buffers");
    FS_CHECK_ARG((d->q_stride % 8) == 0 && (d->o_stride % 8) == 0,
                 "q_stride and o_stride must be multiples of 8 elements");
    FS_CHECK_ARG((reinterpret_cast<uintptr_t>(d->kv_pool) & 15) == 0, "kv_pool must be 16B aligned");
    PrefillParams prm;
    prm.q = static_cast<const __nv_bfloat16 *>(d->q);
    prm.out = d->out;
    prm.out_fp32 = d->out_fp32;
    prm.q_stride = d->q_stride;
    prm.o_stride = d->o_stride;
    prm.kv = static_cast<const uint8_t *>(d->kv_pool);
    prm.bt = d->block_table;
    prm.bt_stride = d->bt_stride;
    prm.item_seq = d->item_seq;
    prm.item_start = d->item_start;
    prm.item_len = d->item_len;
    prm.item_qoff = d->item_qoff;
    prm.item_ooff = d->item_ooff;
    prm.tile_item = d->tile_item;
    prm.tile_tok0 = d->tile_tok0;
    prm.tile_page0 = d->tile_page0;
    prm.tile_page1 = d->tile_page1;
    prm.tile_slot = d->tile_slot;
    prm.comb_item = d->comb_item;
    prm.comb_tok0 = d->comb_tok0;
    prm.comb_slot0 = d->comb_slot0;
    prm.comb_nsplit = d->comb_nsplit;
    prm.qpk = d->q_per_kv;
    FS_CHECK_ARG(variant_rows(d->variant) > 0, "unknown prefill kernel variant %d", d->variant);
    prm.rows = variant_rows(d->variant);
    prm.tpt = prm.rows / d->q_per_kv;
    prm.scale_log2 = d->scale * 1.4426950408889634f;
    prm.part_o = static_cast<float *>(d->part_o);
    prm.part_lse = d->part_lse;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    static bool attr_set[4][64] = {{false}};
    int dev = 0;
    cudaGetDevice(&dev);
    if (d->variant == 0 || d->variant == 2 || d->variant == 3) {
        // tcgen05: 0 = two 128-row halves x 64-key blocks, 2 = one half,
        // 3 = two halves x 128-key blocks
        const int v = d->variant;
        auto kfn = v == 0 ? prefill_tc_kernel<2, 64> : v == 2 ? prefill_tc_kernel<1, 64> : prefill_tc_kernel<2, 128>;
        const int smem = v == 0 ? tc_smem<2, 64>() : v == 2 ? tc_smem<1, 64>() : tc_smem<2, 128>();
        const int threads = (v == 2 ? 1 : 2) * 128 + 64;
        if (!attr_set[v][dev & 63]) {
            FS_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
            attr_set[v][dev & 63] = true;
        }
        kfn<<<d->n_tiles, threads, smem, st>>>(prm);
    } else {
        constexpr int S = kPrefillStages;
        const size_t smem = (size_t)S * kPageBytes + 3 * S * 8;
        if (!attr_set[1][dev & 63]) {
            FS_CUDA(cudaFuncSetAttribute(prefill_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem));
            attr_set[1][dev & 63] = true;
        }
        prefill_kernel<S><<<d->n_tiles, (kConsumerWarps + 2) * 32, smem, st>>>(prm);
    }
    FS_CUDA(cudaGetLastError());
    if (d->n_comb > 0) {
        cudaLaunchConfig_t lc = {};
        lc.gridDim = dim3(d->n_comb, prm.rows / kCombRows);
        lc.blockDim = dim3(256);
        lc.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        lc.attrs = attr;
        lc.numAttrs = 1;
        FS_CUDA(cudaLaunchKernelEx(&lc, prefill_combine_kernel, prm));
        FS_CUDA(cudaGetLastError());
    }
    return FS_OK;
}
