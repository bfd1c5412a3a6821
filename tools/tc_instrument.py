"""Dev tool: patch a copy of csrc/prefill_tc.cuh with per-CTA globaltimer stamps
(kernel start, first S issue, MMA loop end, CTA end, SM id, #blocks) written to
part_lse + 1e6 (tools/tl_dbg2.py reads them) and/or a softmax ablation
(FS_TC_EXP=1: publish P without computing it).  Never commit the patched file."""
import sys
p = "paper_2511_14116_b200/csrc/prefill_tc.cuh"
s = open(p).read()
mode = sys.argv[1]
if "timeline" in mode:
    s = s.replace('''    const int nb = (npg + kPB - 1) / kPB;  // key blocks
''', '''    const int nb = (npg + kPB - 1) / kPB;  // key blocks
    long long *dbgp = reinterpret_cast<long long *>(p.part_lse) + 1000000 + blockIdx.x * 8;
    auto gtm = []() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return (long long)t; };
    if (threadIdx.x == 0) { unsigned sm; asm volatile("mov.u32 %0, %%smid;" : "=r"(sm)); dbgp[0] = gtm(); dbgp[4] = sm; dbgp[5] = nb; }
''', 1)
    s = s.replace('''        for (int j = 0; j < kSBuf && j < nb; ++j) {
            wait_kv(j);''', '''        if (lane == 0) dbgp[1] = gtm();
        for (int j = 0; j < kSBuf && j < nb; ++j) {
            wait_kv(j);''', 1)
    s = s.replace('''                for (int h = 0; h < NQ; ++h) issue_s_half(j + 2, h);
            }
        }''', '''                for (int h = 0; h < NQ; ++h) issue_s_half(j + 2, h);
            }
        }
        if (lane == 0) dbgp[2] = gtm();''', 1)
    s = s.replace('''    tc_before();
    __syncthreads();
    if (warp == kSoftWarps + 1) {
        tc_after();
        asm volatile("tcgen05.dealloc''', '''    tc_before();
    __syncthreads();
    if (threadIdx.x == 0) dbgp[3] = gtm();
    if (warp == kSoftWarps + 1) {
        tc_after();
        asm volatile("tcgen05.dealloc''', 1)
    assert s.count("dbgp") >= 6, "timeline patch failed"
if "waits" in mode:
    # cycles the MMA warp spends waiting for K/V (kv_full) and for P (p_full)
    s = s.replace("""        auto wait_kv = [&](int j) { mbar_wait(k_full + 8 * (j % kKS), (j / kKS) & 1); };""", """        long long w_kv = 0, w_p = 0, c_loop0 = clock64();
        auto wait_kv = [&](int j) { long long c0 = clock64(); mbar_wait(k_full + 8 * (j % kKS), (j / kKS) & 1); w_kv += clock64() - c0; };""", 1)
    s = s.replace("""                mbar_wait(p_full + 8 * (2 * h + b), (j / kSBuf) & 1);
                tc_after();
                const uint32_t pt""", """                { long long c0 = clock64(); mbar_wait(p_full + 8 * (2 * h + b), (j / kSBuf) & 1); w_p += clock64() - c0; }
                tc_after();
                const uint32_t pt""", 1)
    s = s.replace("""        if (lane == 0) dbgp[2] = gtm();""", """        if (lane == 0) { dbgp[2] = gtm(); dbgp[6] = w_kv; dbgp[7] = w_p; dbgp[5] |= (clock64() - c_loop0) << 16; }""", 1)
    s = s.replace("""            mbar_wait(v_full + 8 * st, (j / kVS) & 1);""", """            { long long c0 = clock64(); mbar_wait(v_full + 8 * st, (j / kVS) & 1); w_v += clock64() - c0; }""", 1)
    s = s.replace("long long w_kv = 0, w_p = 0,", "long long w_kv = 0, w_v = 0, w_p = 0,", 1)
    s = s.replace("dbgp[6] = w_kv;", "dbgp[6] = w_kv | (w_v << 32);", 1)
    assert s.count("w_kv") == 3 and s.count("w_v +=") == 1, s.count("w_kv")
if "prologue" in mode:
    # dbg[6] = after setup barrier (thread 0), dbg[7] = softmax warp 0 Q rows stored
    s = s.replace("""    const uint32_t tmem = *tmem_slot;
""", """    const uint32_t tmem = *tmem_slot;
    if (threadIdx.x == 0) dbgp[6] = gtm();
""", 1)
    s = s.replace("""            if (lane == 0) mbar_arrive_cta(q_ready);""", """            if (lane == 0) mbar_arrive_cta(q_ready);
            if (threadIdx.x == 0) dbgp[7] = gtm();""", 1)
if "qload" in mode:
    # dbg[1] (reused) = params loaded, dbg[2] = Q loads returned, dbg[7] = Q stored (thread 0)
    s = s.replace("""            uint4 v[16];""", """            if (threadIdx.x == 0) { dbgp[1] = gtm() + 0 * (start + n + (long long)qb); }
            uint4 v[16];""", 1) if "qload" in mode else s
    s = s.replace("""#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const int ri = (warp & 3) * 32""", """            if (threadIdx.x == 0) { uint32_t x = 0; for (int i = 0; i < 16; ++i) x ^= v[i].x; dbgp[2] = gtm() + (x == 0x12345 ? 1 : 0); }
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const int ri = (warp & 3) * 32""", 1)
    s = s.replace("""            if (lane == 0) mbar_arrive_cta(q_ready);""", """            if (lane == 0) mbar_arrive_cta(q_ready);
            if (threadIdx.x == 0) dbgp[7] = gtm();""", 1)
    s = s.replace("""    const uint32_t tmem = *tmem_slot;
""", """    const uint32_t tmem = *tmem_slot;
    if (threadIdx.x == 0) dbgp[6] = gtm();
""", 1)
if "noexp" in mode:
    # ablation: the exponentials replaced by an FFMA (wrong P, same data flow)
    old = "fast_exp2("
    n = s.count(old)
    i = s.index("uint32_t pk[32];")
    s = s[:i] + s[i:].replace("fast_exp2(", "(1.0f + 0.5f * ", 2)
if "epi" in mode:
    # dbg[6] = last P.V landed (softmax thread 0), dbg[7] = partial stores issued
    s = s.replace("""        mbar_wait(o_done + 8 * (2 * h + ((nb - 1) % kSBuf)), ((nb - 1) / kSBuf) & 1);""", """        mbar_wait(o_done + 8 * (2 * h + ((nb - 1) % kSBuf)), ((nb - 1) / kSBuf) & 1);
        if (threadIdx.x == 0) dbgp[6] = gtm();""", 1)
    s = s.replace("""        if (slot >= 0) p.part_lse[(int64_t)slot * rows + R] = l > 0.f ? m_used + __log2f(l) : -INFINITY;""", """        if (slot >= 0) p.part_lse[(int64_t)slot * rows + R] = l > 0.f ? m_used + __log2f(l) : -INFINITY;
        if (threadIdx.x == 0) dbgp[7] = gtm();""", 1)
    assert s.count("dbgp[6]") == 1 and s.count("dbgp[7]") == 1
if "smphase" in mode:
    # softmax thread 0 of each half: accumulated cycles per phase (wait for S,
    # TMEM load, max, exp + P store, rest) -> dbg slots 8.. of a second area
    s = s.replace("""        float m_used = -INFINITY, l = 0.f;
        for (int j = 0; j < nb; ++j) {""", """        float m_used = -INFINITY, l = 0.f;
        long long ph_w = 0, ph_ld = 0, ph_mx = 0, ph_ex = 0, ph_rest = 0, c_prev = clock64();
        for (int j = 0; j < nb; ++j) {""", 1)
    s = s.replace("""            mbar_wait(s_full + 8 * hb, (j / kSBuf) & 1);
            tc_after();""", """            { long long c = clock64(); ph_rest += c - c_prev; c_prev = c; }
            mbar_wait(s_full + 8 * hb, (j / kSBuf) & 1);
            tc_after();
            { long long c = clock64(); ph_w += c - c_prev; c_prev = c; }""", 1)
    s = s.replace("""            for (int hh = 0; hh < kC; ++hh) tc_ld32(s_t + b * kTcKeys + 32 * hh, sr[hh]);
            tc_wait_ld();""", """            for (int hh = 0; hh < kC; ++hh) tc_ld32(s_t + b * kTcKeys + 32 * hh, sr[hh]);
            tc_wait_ld();
            { long long c = clock64(); ph_ld += c - c_prev; c_prev = c; }""", 1)
    s = s.replace("""            const float mx = fmax3(fmaxf(mxs[0], mxs[1]), mxs[2], mxs[3]) * scale;""", """            const float mx = fmax3(fmaxf(mxs[0], mxs[1]), mxs[2], mxs[3]) * scale;
            { long long c = clock64() + (mx == 12345.f ? 1 : 0); ph_mx += c - c_prev; c_prev = c; }""", 1)
    s = s.replace("""            tc_wait_st();
            float ls[4];""", """            tc_wait_st();
            { long long c = clock64(); ph_ex += c - c_prev; c_prev = c; }
            float ls[4];""", 1)
    s = s.replace("""        // ---- epilogue: O / l (or the split partial) ----""", """        if ((threadIdx.x & 127) == 0) {
            long long *q = dbgp + 8 * gridDim.x + blockIdx.x * 16 + h * 8;
            q[0] = ph_w; q[1] = ph_ld; q[2] = ph_mx; q[3] = ph_ex; q[4] = ph_rest; q[5] = nb;
        }
        // ---- epilogue: O / l (or the split partial) ----""", 1)
    assert s.count("ph_ex") == 3, s.count("ph_ex")
if "nosoftmax" in mode:
    old = '''            uint32_t sr[2][32];
            tc_ld32(s_t + b * kTcKeys, sr[0]);'''
    assert old in s
    s = s.replace(old, '''            if (true) {
                tc_before();
                __syncwarp();
                if (lane == 0) mbar_arrive_cta(p_full + 8 * hb);
                continue;
            }
''' + old, 1)
open(p, "w").write(s)
