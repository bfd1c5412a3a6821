"""Dev tool: patch a copy of csrc/decode_cta.cuh (config 0's kernel) with
per-CTA globaltimer stamps (CTA start, first page landed, end) written to
part_lse + 2^24 floats; tools/dec_tl.py reads them.  Never commit the
patched file."""
p = "paper_2511_14116_b200/csrc/decode_cta.cuh"
s = open(p).read()
s = s.replace("""    grid_launch_dependents();  // the next launch may stage its pages early
    if (x0 >= x1) return;  // CTA-uniform
""", """    grid_launch_dependents();  // the next launch may stage its pages early
    long long *dbg = reinterpret_cast<long long *>(p.part_lse + (1 << 24)) + c * 4;
    auto gtm = []() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return (long long)t; };
    if (threadIdx.x == 0) { unsigned sm; asm volatile("mov.u32 %0, %%smid;" : "=r"(sm)); dbg[0] = gtm(); dbg[3] = sm; }
    bool first_pg = true;
    if (x0 >= x1) return;  // CTA-uniform
""", 1)
s = s.replace("""            mbar_wait(bar0 + 8 * stage, phase);
            const bool tail = valid < kPageTokens;""", """            mbar_wait(bar0 + 8 * stage, phase);
            if (first_pg && threadIdx.x == 0) dbg[1] = gtm();
            first_pg = false;
            const bool tail = valid < kPageTokens;""", 1)
s = s.replace("""        named_bar(1, NT);  // merge area and s_prev are reused by the next item
        if (seg_hi >= x1) break;
        do { ++item; } while (off[item + 1] <= seg_hi);
    }
}""", """        named_bar(1, NT);  // merge area and s_prev are reused by the next item
        if (seg_hi >= x1) break;
        do { ++item; } while (off[item + 1] <= seg_hi);
    }
    if (threadIdx.x == 0) dbg[2] = gtm();
}""", 1)
assert s.count("dbg[") == 4, s.count("dbg[")
open(p, "w").write(s)
