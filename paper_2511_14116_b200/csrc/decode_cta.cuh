// K1, CTA-cooperative variant: the stream-K unit is a CTA, not a warp.
//
// CTA c owns pages [c*P/C, (c+1)*P/C) of the flattened page space; its
// WARPS warps take the pages round-robin (warp k: x0+k, x0+k+WARPS, ...),
// each through its own TMA ring exactly like decode_kernel.  At the end of
// every item the CTA range touches, the warps merge their (m, l, O) in
// shared memory (one named barrier) and the CTA writes either the final
// output (item entirely inside the CTA range) or ONE partial per (item, CTA)
// -- ~WARPS x fewer partials than the warp-level split, so the in-kernel
// global merge on the kernel tail reads ~2-3 blocks per item instead of ~10
// at Llama-70B / 8-GPU shapes.  The last CTA of an item (semaphore) merges
// with all its warps in parallel (one query per warp per round).
#pragma once

// (included inside namespace fs by decode.cu)

__device__ __forceinline__ void named_bar(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

constexpr int kMergeStride = kHeadDim + 4;  // padded fp32 row (bank-conflict free)

template <int WARPS, int STAGES>
__global__ void __launch_bounds__(WARPS * 32, 1) decode_cta_kernel(const DecodeParams p) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gid = lane >> 2, tig = lane & 3;
    constexpr int NT = WARPS * 32;
    if (!p.early) grid_dependency_wait();  // see decode_kernel

    // page offsets + block-table rows of all items -> smem in one round
    // trip (the first page copy then waits for one dependent load, the
    // block-table entry, instead of P -> search -> walk -> row -> entry)
    int32_t *tab = reinterpret_cast<int32_t *>(smem + WARPS * STAGES * (kPageBytes + 8) +
                                               WARPS * (2 * FS_MAX_Q_PER_KV + FS_MAX_Q_PER_KV * kMergeStride) * 4);
    const int32_t *off = p.page_off, *iseq = p.item_seq;
    if (p.tab_cache) {
        const int n = p.n_items;
        for (int i = threadIdx.x; i <= n; i += NT) {
            tab[i] = p.page_off[i];
            if (i < n) tab[kTabItems + 1 + i] = p.item_seq[i];
        }
        __syncthreads();
        off = tab;
        iseq = tab + kTabItems + 1;
    }
    const int64_t P = off[p.n_items];
    const int64_t C = p.n_warps;  // partition units = CTAs
    const int64_t c = blockIdx.x;
    const int64_t x0 = c * P / C, x1 = (c + 1) * P / C;
    grid_launch_dependents();  // the next launch may stage its pages early
    if (x0 >= x1) return;  // CTA-uniform

    const uint32_t sbase = smem_u32(smem);
    const uint32_t buf0 = sbase + warp * STAGES * kPageBytes;
    const uint32_t bar0 = sbase + WARPS * STAGES * kPageBytes + warp * STAGES * 8;
    // merge area: per warp m[8], l[8], O[8][132] fp32
    float *merge = reinterpret_cast<float *>(smem + WARPS * STAGES * (kPageBytes + 8));
    constexpr int kSlot = 2 * FS_MAX_Q_PER_KV + FS_MAX_Q_PER_KV * kMergeStride;
    __shared__ int s_prev;
    if (lane == 0) {
        for (int s = 0; s < STAGES; ++s) mbar_init(bar0 + 8 * s, 1);
        fence_barrier_init();
        fence_proxy_async();
    }
    __syncwarp();

    const int first = find_item(off, p.n_items, x0, lane);
    const int64_t span = x1 - x0;
    const int64_t n_my = span > warp ? (span - warp + WARPS - 1) / WARPS : 0;
    auto page_of = [&](int64_t j) { return x0 + warp + (int64_t)WARPS * j; };

    // ---- producer: lane-parallel page-id windows over MY pages ----
    const uint64_t pol = policy_evict_first();
    int64_t win = 0;
    int wit = first;
    auto window_ids = [&](int64_t base) -> int64_t {
        const int64_t j = base + lane;
        int it = wit;
        int64_t pg = 0;
        if (j < n_my) {
            const int64_t y = page_of(j);
            while (y >= off[it + 1]) ++it;
            pg = p.bt[(int64_t)iseq[it] * p.bt_stride + (y - off[it])];
        }
        wit = max(wit, __shfl_sync(0xffffffffu, it, 31));
        return pg;
    };
    int64_t cur_pg = 0, nxt_pg = 0;
    if (n_my > 0) {
        cur_pg = window_ids(0);
        nxt_pg = window_ids(32);
    }
    int64_t px = 0;
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
    for (int s = 0; s < STAGES && px < n_my; ++s) issue(s);
    if (lane >= STAGES && lane < STAGES + p.l2_pf && lane < n_my)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p.kv + cur_pg * kPageBytes),
                     "r"(kPageBytes) : "memory");
    grid_dependency_wait();  // q / kv_new come from the preceding GEMM

    // ---- consumer: items of the CTA range in order ----
    int item = first;
    int64_t jx = 0;
    int stage = 0;
    uint32_t phase = 0;
    uint32_t qf[8][2];
    float o[8][4];
    while (true) {
        const int64_t ib = off[item], ie = off[item + 1];
        const int64_t seg_hi = min(ie, x1);
        const int len = p.item_len[item];
        float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
#pragma unroll
        for (int mt = 0; mt < 8; ++mt) o[mt][0] = o[mt][1] = o[mt][2] = o[mt][3] = 0.f;
        if (jx < n_my && page_of(jx) < seg_hi) {
            const __nv_bfloat16 *qb = p.q + p.item_qoff[item] + gid * kHeadDim;
            const bool ok = gid < p.qpk;
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
                qf[ks][0] = ok ? *reinterpret_cast<const uint32_t *>(qb + ks * 16 + 2 * tig) : 0u;
                qf[ks][1] = ok ? *reinterpret_cast<const uint32_t *>(qb + ks * 16 + 8 + 2 * tig) : 0u;
            }
        }
        for (; jx < n_my && page_of(jx) < seg_hi; ++jx) {
            const int64_t x = page_of(jx);
            const uint32_t kb = buf0 + stage * kPageBytes;
            const uint32_t vb = kb + kHalfPage;
            const int pidx = (int)(x - ib);
            const int valid = min(kPageTokens, len - pidx * kPageTokens);
            mbar_wait(bar0 + 8 * stage, phase);
            const bool tail = valid < kPageTokens;
            const bool append = p.kv_new != nullptr && valid > 0 && (len - 1) / kPageTokens == pidx;
            if (tail | append) {
                uint8_t *page_s = smem + (kb - sbase);
                if (tail)
                    for (int cc = valid * 8 + lane; cc < kPageTokens * 16; cc += 32)
                        if ((cc & 127) >= valid * 8)  // both atoms: rows >= valid
                            reinterpret_cast<uint4 *>(page_s + kHalfPage)[cc] = make_uint4(0, 0, 0, 0);
                if (append) {
                    const uint32_t r = (len - 1) % kPageTokens, ch = lane & 15, half = lane >> 4;
                    const int64_t src = (half ? p.item_voff[item] : p.item_koff[item]) + ch * 8;
                    uint4 v = *reinterpret_cast<const uint4 *>(p.kv_new + src);
                    const uint32_t ofs = half * kHalfPage + swz(r, ch);
                    *reinterpret_cast<uint4 *>(page_s + ofs) = v;
                    const int64_t pg = p.bt[(int64_t)p.item_seq[item] * p.bt_stride + pidx];
                    *reinterpret_cast<uint4 *>(const_cast<uint8_t *>(p.kv) + pg * kPageBytes + ofs) = v;
                }
                fence_proxy_async();
                __syncwarp();
            }
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
            if (px < n_my) issue(stage);
            if (++stage == STAGES) {
                stage = 0;
                phase ^= 1u;
            }
        }

        // ---- CTA merge of this item's warp states ----
#pragma unroll
        for (int sh = 4; sh < 32; sh <<= 1) {
            l0 += __shfl_xor_sync(0xffffffffu, l0, sh);
            l1 += __shfl_xor_sync(0xffffffffu, l1, sh);
        }
        float *slot = merge + warp * kSlot;
        float *om = slot + 2 * FS_MAX_Q_PER_KV;
        const int q0 = 2 * tig, q1 = q0 + 1;
        if (gid == 0) {
            slot[q0] = m0;
            slot[q1] = m1;
            slot[FS_MAX_Q_PER_KV + q0] = l0;
            slot[FS_MAX_Q_PER_KV + q1] = l1;
        }
#pragma unroll
        for (int mt = 0; mt < 8; ++mt) {
            const int d0 = mt * 16 + gid, d1 = d0 + 8;
            om[q0 * kMergeStride + d0] = o[mt][0];
            om[q1 * kMergeStride + d0] = o[mt][1];
            om[q0 * kMergeStride + d1] = o[mt][2];
            om[q1 * kMergeStride + d1] = o[mt][3];
        }
        named_bar(1, NT);
        const bool whole = ib >= x0 && ie <= x1;
        for (int q = warp; q < p.qpk; q += WARPS) {
            float M = -INFINITY;
#pragma unroll
            for (int k = 0; k < WARPS; ++k) M = fmaxf(M, merge[k * kSlot + q]);
            float L = 0.f;
            float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int k = 0; k < WARPS; ++k) {
                const float mk = merge[k * kSlot + q];
                const float wk = mk == -INFINITY ? 0.f : fast_exp2(mk - M);
                L += wk * merge[k * kSlot + FS_MAX_Q_PER_KV + q];
                const float4 v = *reinterpret_cast<const float4 *>(
                    merge + k * kSlot + 2 * FS_MAX_Q_PER_KV + q * kMergeStride + lane * 4);
                acc.x += wk * v.x;
                acc.y += wk * v.y;
                acc.z += wk * v.z;
                acc.w += wk * v.w;
            }
            const float inv = 1.f / L;
            acc = make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
            if (whole) {
                const int64_t ob = (int64_t)p.item_ooff[item] + q * kHeadDim + lane * 4;
                if (p.out_fp32) {
                    *reinterpret_cast<float4 *>(static_cast<float *>(p.out) + ob) = acc;
                } else {
                    __nv_bfloat162 lo = __floats2bfloat162_rn(acc.x, acc.y);
                    __nv_bfloat162 hi = __floats2bfloat162_rn(acc.z, acc.w);
                    uint2 pk;
                    pk.x = *reinterpret_cast<uint32_t *>(&lo);
                    pk.y = *reinterpret_cast<uint32_t *>(&hi);
                    *reinterpret_cast<uint2 *>(static_cast<__nv_bfloat16 *>(p.out) + ob) = pk;
                }
            } else {
                const int64_t sl = (int64_t)item + c;
                __stcg(reinterpret_cast<float4 *>(p.part_o + (sl * p.qpk + q) * kHeadDim) + lane,
                       acc);
                if (lane == 0) __stcg(p.part_lse + sl * p.qpk + q, M + __log2f(L));
            }
        }
        if (!whole) {
            __threadfence();
            named_bar(1, NT);
            if (threadIdx.x == 0) s_prev = atomicAdd(p.item_sem + item, 1);
            named_bar(1, NT);
            const int64_t clo = owner_warp(ib, C, P), chi = owner_warp(ie - 1, C, P);
            int nseg = (int)(chi - clo + 1);
            if (P < C) {
                nseg = 0;
                for (int64_t s = clo; s <= chi; ++s) nseg += warp_live(s, C, P);
            }
            if (s_prev == nseg - 1) {
                // last CTA of the item: merge its (up to ~all-CTA) partials.
                // Warp w streams segments clo+w, clo+w+WARPS, ... issuing each
                // segment's lse and O loads together and folding them into a
                // running log-sum-exp (m, l, acc) per query -- one L2 round
                // trip for the usual <= WARPS segments -- then the warps'
                // states are combined in smem.
                __threadfence();
                const bool all_live = P >= C;
                const int qpk = p.qpk;
                float mw[FS_MAX_Q_PER_KV], lw[FS_MAX_Q_PER_KV];
                float4 acc[FS_MAX_Q_PER_KV];
#pragma unroll
                for (int q = 0; q < FS_MAX_Q_PER_KV; ++q) {
                    mw[q] = -INFINITY;
                    lw[q] = 0.f;
                    acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
                }
                for (int64_t s = clo + warp; s <= chi; s += WARPS) {
                    if (!all_live && !warp_live(s, C, P)) continue;
                    const float *ls = p.part_lse + (item + s) * qpk;
                    const float4 *os = reinterpret_cast<const float4 *>(p.part_o + (item + s) * qpk * kHeadDim);
                    float lv[FS_MAX_Q_PER_KV];
                    float4 v[FS_MAX_Q_PER_KV];
#pragma unroll
                    for (int q = 0; q < FS_MAX_Q_PER_KV; ++q) {
                        if (q < qpk) {
                            lv[q] = __ldcg(ls + q);
                            v[q] = __ldcg(os + q * (kHeadDim / 4) + lane);
                        }
                    }
#pragma unroll
                    for (int q = 0; q < FS_MAX_Q_PER_KV; ++q) {
                        if (q < qpk) {
                            const float mn = fmaxf(mw[q], lv[q]);
                            const float a0 = fast_exp2(mw[q] - mn), a1 = fast_exp2(lv[q] - mn);
                            mw[q] = mn;
                            lw[q] = lw[q] * a0 + a1;
                            acc[q].x = acc[q].x * a0 + v[q].x * a1;
                            acc[q].y = acc[q].y * a0 + v[q].y * a1;
                            acc[q].z = acc[q].z * a0 + v[q].z * a1;
                            acc[q].w = acc[q].w * a0 + v[q].w * a1;
                        }
                    }
                }
                float *slot = merge + warp * kSlot;
                float *om = slot + 2 * FS_MAX_Q_PER_KV;
#pragma unroll
                for (int q = 0; q < FS_MAX_Q_PER_KV; ++q) {
                    if (q < qpk) {
                        if (lane == 0) {
                            slot[q] = mw[q];
                            slot[FS_MAX_Q_PER_KV + q] = lw[q];
                        }
                        *reinterpret_cast<float4 *>(om + q * kMergeStride + lane * 4) = acc[q];
                    }
                }
                named_bar(1, NT);
                for (int q = warp; q < qpk; q += WARPS) {
                    float M = -INFINITY;
#pragma unroll
                    for (int k = 0; k < WARPS; ++k) M = fmaxf(M, merge[k * kSlot + q]);
                    float L = 0.f;
                    float4 sum = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                    for (int k = 0; k < WARPS; ++k) {
                        const float mk = merge[k * kSlot + q];
                        const float wk = mk == -INFINITY ? 0.f : fast_exp2(mk - M);
                        L += wk * merge[k * kSlot + FS_MAX_Q_PER_KV + q];
                        const float4 t = *reinterpret_cast<const float4 *>(
                            merge + k * kSlot + 2 * FS_MAX_Q_PER_KV + q * kMergeStride + lane * 4);
                        sum.x += wk * t.x;
                        sum.y += wk * t.y;
                        sum.z += wk * t.z;
                        sum.w += wk * t.w;
                    }
                    const float inv = 1.f / L;
                    const int64_t ob = (int64_t)p.item_ooff[item] + q * kHeadDim + lane * 4;
                    if (p.out_fp32) {
                        *reinterpret_cast<float4 *>(static_cast<float *>(p.out) + ob) =
                            make_float4(sum.x * inv, sum.y * inv, sum.z * inv, sum.w * inv);
                    } else {
                        __nv_bfloat162 lo = __floats2bfloat162_rn(sum.x * inv, sum.y * inv);
                        __nv_bfloat162 hi = __floats2bfloat162_rn(sum.z * inv, sum.w * inv);
                        uint2 pk;
                        pk.x = *reinterpret_cast<uint32_t *>(&lo);
                        pk.y = *reinterpret_cast<uint32_t *>(&hi);
                        *reinterpret_cast<uint2 *>(static_cast<__nv_bfloat16 *>(p.out) + ob) = pk;
                    }
                }
                if (threadIdx.x == 0) p.item_sem[item] = 0;
            }
        }
        named_bar(1, NT);  // merge area and s_prev are reused by the next item
        if (seg_hi >= x1) break;
        do { ++item; } while (off[item + 1] <= seg_hi);
    }
}


