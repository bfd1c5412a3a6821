// Skinny weight-streaming GEMM for the decode step on sm_100a:
//     out[n, c] (+)= sum_k x[n, k] * W[k, c]        n < 64 (the decode batch)
// computed as D^T[128 cols x 64 rows] = W^T-tile . x^T with tcgen05.mma
// (M = 128 weight columns, N = 64 batch rows, K = 16 per instruction; A = the
// W tile, MN-major, B = x, K-major, both TMA-loaded with 128B swizzle; the
// fp32 accumulator lives in TMEM, double-buffered).
//
// Work decomposition is stream-K over (column tile, 64-wide k-step) units:
// the persistent grid (one CTA per SM) splits the U = tiles x K/64 units
// evenly, so skinny shapes with few column tiles (Llama-70B qkv at 8 GPUs:
// 10 tiles) still use every SM and every byte of W is read exactly once.  A
// CTA that covers a whole tile applies the epilogue directly; otherwise it
// writes an fp32 partial to slot `tile + cta`, and gemm_reduce_kernel (the
// next launch, PDL) sums each split tile's partials in CTA order
// (deterministic) and applies the epilogue.
//
// Roles (192 threads): warp 4 = TMA producer, warp 5 = MMA issuer, warps 0-3
// = epilogue (TMEM lane quadrant = warp index).  Fused epilogues: plain
// store, residual add (x += ...), and SwiGLU (tile = 64 gate + 64 up
// columns -> 64 activations).  Launched with programmatic dependent launch:
// W tiles of the first stages are fetched before griddepcontrol.wait, so the
// weight stream starts while the previous kernel drains.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <mutex>
#include <unordered_map>

#include "common.cuh"

namespace fs {

constexpr int kGemmStages = 8;
constexpr int kTileM = 128;        // weight columns per tile (UMMA M)
constexpr int kRowsN = 64;         // batch rows (UMMA N)
constexpr int kStepK = 64;         // k per stage (one 128B swizzle row)
constexpr int kStageA = kTileM * kStepK * 2;   // 16 KB (two 64-col boxes)
constexpr int kStageB = kRowsN * kStepK * 2;   // 8 KB
constexpr int kStageBytes = kStageA + kStageB;
constexpr int kUpPitch = 64 + 4;              // fp32 row pitch of the swiglu 'up' stage
constexpr int kGemmThreads = 192;
constexpr int kPrefetchA = 3;   // W stages issued before the PDL wait

enum GemmEpilogue { EPI_STORE = 0, EPI_RESIDUAL = 1, EPI_SWIGLU = 2 };

struct GemmParams {
    int32_t rows;       // valid batch rows (<= 64)
    int32_t K;          // multiple of 64
    int32_t tiles;      // output column tiles of 128
    int64_t n_units;    // tiles * K/64
    int32_t epilogue;
    int32_t w_packed;   // 1: W pre-packed in UMMA-canonical 16 KB blocks
    const uint8_t *w_raw;
    __nv_bfloat16 *out;
    int64_t ld_out;
    const __nv_bfloat16 *res;
    int64_t ld_res;
    float *ws;          // partial slots, each [64][128] fp32
    int32_t *sems;      // reserved (ABI): split tiles are reduced by gemm_reduce_kernel
    unsigned long long *dbg;  // optional per-CTA phase timestamps (ns)
};

// ---------------------------------------------------------------- PTX ----
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap *map, int c0, int c1,
                                            uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
        : "memory");
}

__device__ __forceinline__ void prefetch_tmap(const CUtensorMap *map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

__device__ __forceinline__ void tc_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     bar)
                 : "memory");
}

__device__ __forceinline__ void tc_mma(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                       uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// 32 lanes x 32 bit, 32 consecutive columns per thread
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
        "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
          "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
          "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// UMMA shared-memory descriptor (Blackwell version 1); layout 2 =
// SWIZZLE_128B, 0 = no swizzle (canonical core-matrix interleave)
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo,
                                              uint32_t layout) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;           // version
    d |= (uint64_t)layout << 61;
    return d;
}

// kind::f16 instruction descriptor: BF16 x BF16 -> F32, A MN-major, B K-major
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) |
                            ((uint32_t)(kRowsN >> 3) << 17) | ((uint32_t)(kTileM >> 4) << 24);

__device__ __forceinline__ int64_t gemm_owner(int64_t u, int64_t C, int64_t U) {
    return ((u + 1) * C + U - 1) / U - 1;
}
__device__ __forceinline__ bool gemm_live(int64_t c, int64_t C, int64_t U) {
    return c * U / C < (c + 1) * U / C;
}

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ int ld_acquire(const int32_t *p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ float silu(float g) { return g / (1.f + __expf(-g)); }

// final epilogue straight from the accumulator registers: thread m owns
// column m of the tile for all 64 rows, so for a fixed row a warp stores 32
// consecutive bf16.  SwiGLU: warps 2-3 (the 'up' columns) stage through
// shared memory, warps 0-1 (gate) combine and store the 64 activations.
__device__ __forceinline__ void gemm_epilogue(const GemmParams &p, const float (&acc)[kRowsN],
                                              int tile, int m, float *up) {
    if (p.epilogue == EPI_SWIGLU) {
        if (m >= 64) {
#pragma unroll
            for (int n = 0; n < kRowsN; ++n) up[n * kUpPitch + (m - 64)] = acc[n];
        }
        named_bar_sync(2, 128);
        if (m < 64) {
#pragma unroll
            for (int n = 0; n < kRowsN; ++n)
                if (n < p.rows)
                    p.out[n * p.ld_out + tile * 64 + m] =
                        __float2bfloat16_rn(silu(acc[n]) * up[n * kUpPitch + m]);
        }
        return;
    }
    const int64_t col = (int64_t)tile * kTileM + m;
    if (p.epilogue == EPI_RESIDUAL) {
#pragma unroll
        for (int n = 0; n < kRowsN; ++n)
            if (n < p.rows)
                p.out[n * p.ld_out + col] =
                    __float2bfloat16_rn(acc[n] + __bfloat162float(p.res[n * p.ld_res + col]));
    } else {
#pragma unroll
        for (int n = 0; n < kRowsN; ++n)
            if (n < p.rows) p.out[n * p.ld_out + col] = __float2bfloat16_rn(acc[n]);
    }
}

__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm_skinny_kernel(const __grid_constant__ CUtensorMap map_w,
                       const __grid_constant__ CUtensorMap map_x, const GemmParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 1024-byte aligned base for the swizzled stages
    uint8_t *smem = reinterpret_cast<uint8_t *>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t sbase = smem_u32(smem);
    float *up = reinterpret_cast<float *>(smem + kGemmStages * kStageBytes);
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + kGemmStages * kStageBytes +
                                                  kRowsN * kUpPitch * 4);
    const uint32_t bar_full = smem_u32(bars);
    const uint32_t bar_empty = bar_full + 8 * kGemmStages;
    const uint32_t bar_acc_full = bar_empty + 8 * kGemmStages;   // [2]
    const uint32_t bar_acc_empty = bar_acc_full + 16;            // [2]
    __shared__ uint32_t s_tmem;


    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t C = gridDim.x, U = p.n_units, c = blockIdx.x;
    const int64_t u0 = c * U / C, u1 = (c + 1) * U / C;
    const int nk = p.K / kStepK;

    if (warp == 4 && lane == 0) {
        prefetch_tmap(&map_w);
        prefetch_tmap(&map_x);
        for (int s = 0; s < kGemmStages; ++s) {
            mbar_init(bar_full + 8 * s, 1);
            mbar_init(bar_empty + 8 * s, 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(bar_acc_full + 8 * b, 1);
            mbar_init(bar_acc_empty + 8 * b, 128);
        }
        fence_barrier_init();
        fence_proxy_async();
    }
    if (warp == 0) {  // TMEM: two 64-column fp32 accumulators
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(&s_tmem)),
                     "r"(128));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = s_tmem;
    if (p.dbg && threadIdx.x == 0) p.dbg[blockIdx.x * 8 + 0] = gtimer();

    if (u0 < u1) {
        if (warp == 4) {
            // ---------------- TMA producer ----------------
            if (lane == 0) {
                const uint64_t pol = policy_evict_first();
                int stage = 0;
                uint32_t phase = 0;
                int issued = 0;
                bool waited = false;
                int t = (int)(u0 / nk), ks = (int)(u0 % nk);  // advanced incrementally
                for (int64_t u = u0; u < u1; ++u, ks = (ks + 1 == nk) ? (++t, 0) : ks + 1) {
                    mbar_wait(bar_empty + 8 * stage, phase ^ 1u);
                    const uint32_t a = sbase + stage * kStageBytes, b = a + kStageA;
                    mbar_expect_tx(bar_full + 8 * stage, kStageBytes);
                    if (p.w_packed) {  // one contiguous 16 KB block, one bulk copy
                        bulk_g2s(a, p.w_raw + ((int64_t)t * nk + ks) * kStageA, kStageA,
                                 bar_full + 8 * stage, pol);
                    } else {
                        tma_load_2d(a, &map_w, t * kTileM, ks * kStepK, bar_full + 8 * stage);
                        tma_load_2d(a + kStageA / 2, &map_w, t * kTileM + 64, ks * kStepK,
                                    bar_full + 8 * stage);
                    }
                    if (!waited && (++issued == kPrefetchA || u + 1 == u1)) {
                        // x comes from the preceding kernel: PDL wait, then
                        // the B halves of every stage issued so far
                        if (p.dbg) p.dbg[blockIdx.x * 8 + 5] = gtimer();
                        grid_dependency_wait();
                        waited = true;
                        if (p.dbg) p.dbg[blockIdx.x * 8 + 6] = gtimer();
                        int st = stage, vks = ks;
                        for (int i = 0; i < issued; ++i) {
                            tma_load_2d(sbase + st * kStageBytes + kStageA, &map_x, vks * kStepK,
                                        0, bar_full + 8 * st);
                            st = st == 0 ? kGemmStages - 1 : st - 1;
                            vks = vks == 0 ? nk - 1 : vks - 1;
                        }
                    } else if (waited) {
                        tma_load_2d(b, &map_x, ks * kStepK, 0, bar_full + 8 * stage);
                    }
                    if (++stage == kGemmStages) {
                        stage = 0;
                        phase ^= 1u;
                    }
                }
                asm volatile("griddepcontrol.launch_dependents;");
            }
        } else if (warp == 5) {
            // ---------------- MMA issuer ----------------
            if (lane == 0) {
                int stage = 0;
                uint32_t phase = 0;
                int seg = 0;
                int64_t u = u0;
                while (u < u1) {
                    const int t = (int)(u / nk);
                    const int64_t seg_end = min(u1, (int64_t)(t + 1) * nk);
                    const int buf = seg & 1;
                    mbar_wait(bar_acc_empty + 8 * buf, ((seg >> 1) & 1) ^ 1u);
                    tc_fence_after();
                    const uint32_t d = tmem + buf * kRowsN;
                    bool first = true;
                    for (; u < seg_end; ++u) {
                        mbar_wait(bar_full + 8 * stage, phase);
                        if (p.dbg && u == u0) p.dbg[blockIdx.x * 8 + 1] = gtimer();
                        tc_fence_after();
                        const uint32_t a = sbase + stage * kStageBytes, b = a + kStageA;
#pragma unroll
                        for (int j = 0; j < kStepK / 16; ++j) {
                            // packed: no-swizzle canonical MN-major (k-group
                            // stride 2048 B = LBO, m-group stride 128 B = SBO)
                            const uint64_t ad = p.w_packed
                                                    ? umma_desc(a + j * 4096, 2048, 128, 0)
                                                    : umma_desc(a + j * 2048, kStageA / 2, 1024, 2);
                            const uint64_t bd = umma_desc(b + j * 32, 16, 1024, 2);
                            tc_mma(d, ad, bd, kIdesc, first ? 0u : 1u);
                            first = false;
                        }
                        tc_commit(bar_empty + 8 * stage);
                        if (++stage == kGemmStages) {
                            stage = 0;
                            phase ^= 1u;
                        }
                    }
                    tc_commit(bar_acc_full + 8 * buf);
                    if (p.dbg) p.dbg[blockIdx.x * 8 + 2] = gtimer();
                    ++seg;
                }
            }
        } else {
            // ---------------- epilogue (warps 0-3) ----------------
            const int m = warp * 32 + lane;
            int seg = 0;
            int64_t u = u0;
            while (u < u1) {
                const int t = (int)(u / nk);
                const int64_t tb = (int64_t)t * nk, te = tb + nk;
                const int64_t seg_end = min(u1, te);
                const bool whole = u == tb && seg_end == te;
                const int buf = seg & 1;
                mbar_wait(bar_acc_full + 8 * buf, (seg >> 1) & 1);
                tc_fence_after();
                float acc[kRowsN];
                {
                    float v[32];
                    const uint32_t taddr = tmem + buf * kRowsN + ((uint32_t)(warp * 32) << 16);
                    tmem_ld32(taddr, v);
#pragma unroll
                    for (int i = 0; i < 32; ++i) acc[i] = v[i];
                    tmem_ld32(taddr + 32, v);
#pragma unroll
                    for (int i = 0; i < 32; ++i) acc[32 + i] = v[i];
                }
                tc_fence_before();
                mbar_arrive(bar_acc_empty + 8 * buf);
                if (whole) {
                    gemm_epilogue(p, acc, t, m, up);
                    named_bar_sync(2, 128);  // 'up' staging reused by the next segment
                } else {
                    // split tile: this CTA's fp32 partial goes to slot
                    // tile + cta; gemm_reduce_kernel (the next launch, PDL)
                    // sums a tile's partials in CTA order -- no CTA of this
                    // grid ever waits for another
                    const int64_t slot = (int64_t)t + c;
                    float *wsl = p.ws + slot * (kRowsN * kTileM);
#pragma unroll
                    for (int n = 0; n < kRowsN; ++n) __stcg(wsl + n * kTileM + m, acc[n]);
                }
                if (p.dbg && threadIdx.x == 0) p.dbg[blockIdx.x * 8 + 3] = gtimer();
                u = seg_end;
                ++seg;
            }
            if (p.dbg && threadIdx.x == 0) p.dbg[blockIdx.x * 8 + 3] = gtimer();
        }
    }
    if (p.dbg && threadIdx.x == 0) p.dbg[blockIdx.x * 8 + 4] = gtimer();
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(128));
    }
}

// Split tiles of a stream-K launch: block (tile, 8-row group); thread m sums
// column m of the tile over the contributors' partials in CTA order
// (deterministic) and applies the epilogue.  Blocks of whole tiles exit.
// Launched with PDL right behind gemm_skinny_kernel: scheduled during its
// tail, waits in griddepcontrol.wait for its partials.
constexpr int kRedRows = 8;

__global__ void __launch_bounds__(kTileM) gemm_reduce_kernel(const GemmParams p, int32_t grid) {
    const int t = blockIdx.x, r0 = blockIdx.y * kRedRows, m = threadIdx.x;
    const int nk = p.K / kStepK;
    const int64_t C = grid, U = p.n_units;
    const int64_t tb = (int64_t)t * nk, te = tb + nk;
    const int64_t clo = gemm_owner(tb, C, U), chi = gemm_owner(te - 1, C, U);
    grid_launch_dependents();
    if (clo == chi || r0 >= p.rows) return;  // whole tile: the GEMM stored it
    const bool swiglu = p.epilogue == EPI_SWIGLU;
    if (swiglu && m >= 64) return;
    grid_dependency_wait();
    float g[kRedRows], uu[kRedRows];
#pragma unroll
    for (int r = 0; r < kRedRows; ++r) g[r] = uu[r] = 0.f;
    // 4 contributors' rows in flight per round (a split tile of a small GEMM
    // has up to ~15 contributors; one round trip per contributor was the
    // whole cost), summed in CTA order
    const bool all_live = U >= C;
    for (int64_t s0 = clo; s0 <= chi; s0 += 4) {
        float vg[4][kRedRows], vu[4][kRedRows];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int64_t s = s0 + i;
            const bool ok = s <= chi && (all_live || gemm_live(s, C, U));
            const float *src = p.ws + (t + (ok ? s : clo)) * (kRowsN * kTileM) + r0 * kTileM + m;
#pragma unroll
            for (int r = 0; r < kRedRows; ++r) {
                vg[i][r] = ok ? __ldcg(src + r * kTileM) : 0.f;
                vu[i][r] = ok && swiglu ? __ldcg(src + r * kTileM + 64) : 0.f;
            }
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int r = 0; r < kRedRows; ++r) {
                g[r] += vg[i][r];
                uu[r] += vu[i][r];
            }
    }
#pragma unroll
    for (int r = 0; r < kRedRows; ++r) {
        const int n = r0 + r;
        if (n >= p.rows) break;
        if (swiglu) {
            p.out[n * p.ld_out + t * 64 + m] = __float2bfloat16_rn(silu(g[r]) * uu[r]);
        } else {
            const int64_t col = (int64_t)t * kTileM + m;
            float v = g[r];
            if (p.epilogue == EPI_RESIDUAL) v += __bfloat162float(p.res[n * p.ld_res + col]);
            p.out[n * p.ld_out + col] = __float2bfloat16_rn(v);
        }
    }
}

// ------------------------------------------------------------ host side ---
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                  const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                  const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    });
    return fn;
}

// 2-D bf16 row-major [rows][cols] (row stride ld elements), box 64 x box_rows
static int make_map(CUtensorMap *map, const void *ptr, int64_t rows, int64_t cols, int64_t ld,
                    int box_rows) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return fail(FS_ECUDA, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(ptr), dims,
                    strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(FS_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    return FS_OK;
}

static unsigned long long *g_gemm_dbg = nullptr;  // fs_gemm_debug_timestamps

static size_t gemm_smem() {
    return 1024 + (size_t)kGemmStages * kStageBytes + (size_t)kRowsN * kUpPitch * 4 + 8 * 40;
}

}  // namespace fs

using namespace fs;

// testing hook (not in the public header): per-CTA phase timestamps
extern "C" void fs_gemm_debug_timestamps(unsigned long long *dev_buf) { g_gemm_dbg = dev_buf; }

extern "C" int64_t fs_gemm_workspace_floats(int device, int32_t N, int32_t epilogue) {
    const int sms = sm_count(device);
    if (sms <= 0 || N <= 0) return -1;
    const int64_t tiles = (int64_t)N / kTileM;
    (void)epilogue;
    return (tiles + sms) * (int64_t)kRowsN * kTileM;  // sems: 2 * tiles int32
}

extern "C" int fs_gemm_skinny(const void *x, int64_t ld_x, int32_t rows, int32_t K, const void *w,
                              int64_t ld_w, int32_t w_layout, int32_t N, void *out, int64_t ld_out, const void *res,
                              int64_t ld_res, int32_t epilogue, float *workspace,
                              int64_t ws_floats, int32_t *sems, int32_t device, void *stream) {
    FS_CHECK_ARG(rows >= 1 && rows <= kRowsN, "rows must be in [1, %d], got %d", kRowsN, rows);
    FS_CHECK_ARG(K > 0 && K % kStepK == 0, "K must be a positive multiple of %d", kStepK);
    FS_CHECK_ARG(N > 0 && N % kTileM == 0, "N must be a positive multiple of %d", kTileM);
    FS_CHECK_ARG(epilogue >= EPI_STORE && epilogue <= EPI_SWIGLU, "unknown epilogue %d", epilogue);
    FS_CHECK_ARG(x && w && out && workspace && sems, "null pointer");
    FS_CHECK_ARG(epilogue != EPI_RESIDUAL || res, "residual epilogue needs res");
    FS_CHECK_ARG(ld_x % 8 == 0 && ld_w % 8 == 0 && ld_x >= K && (w_layout == 1 || ld_w >= N),
                 "leading dimensions must be multiples of 8 and cover the matrix");
    const int sms = sm_count(device);
    if (sms <= 0) return fail(FS_ECUDA, "cannot query SM count");
    FS_CHECK_ARG(ws_floats >= fs_gemm_workspace_floats(device, N, epilogue), "workspace too small");
    CUtensorMap mw, mx;
    FS_CHECK_ARG(w_layout == 0 || w_layout == 1, "unknown W layout %d", w_layout);
    if (int rc = make_map(&mx, x, rows, K, ld_x, kRowsN)) return rc;
    if (w_layout == 1) {
        FS_CHECK_ARG((reinterpret_cast<uintptr_t>(w) & 15) == 0, "packed W must be 16B aligned");
        mw = mx;  // unused: packed blocks are moved with 1-D bulk copies
    } else {
        if (int rc = make_map(&mw, w, K, N, ld_w, kStepK)) return rc;
    }
    GemmParams prm;
    prm.rows = rows;
    prm.K = K;
    prm.tiles = N / kTileM;
    prm.n_units = (int64_t)prm.tiles * (K / kStepK);
    prm.epilogue = epilogue;
    prm.w_packed = w_layout;
    prm.w_raw = static_cast<const uint8_t *>(w);
    prm.dbg = g_gemm_dbg;
    prm.out = static_cast<__nv_bfloat16 *>(out);
    prm.ld_out = ld_out;
    prm.res = static_cast<const __nv_bfloat16 *>(res);
    prm.ld_res = ld_res;
    prm.ws = workspace;
    prm.sems = sems;
    const size_t smem = gemm_smem();
    static bool attr_set[64] = {false};
    if (!attr_set[device & 63]) {
        FS_CUDA(cudaFuncSetAttribute(gemm_skinny_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
        attr_set[device & 63] = true;
    }
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(sms);
    lc.blockDim = dim3(kGemmThreads);
    lc.dynamicSmemBytes = smem;
    lc.stream = static_cast<cudaStream_t>(stream);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = attr;
    lc.numAttrs = 1;
    FS_CUDA(cudaLaunchKernelEx(&lc, gemm_skinny_kernel, mw, mx, prm));
    // the split-tile reduction (blocks of whole tiles exit at once)
    {
        cudaLaunchConfig_t lr = lc;
        lr.gridDim = dim3(prm.tiles, (rows + kRedRows - 1) / kRedRows);
        lr.blockDim = dim3(kTileM);
        lr.dynamicSmemBytes = 0;
        FS_CUDA(cudaLaunchKernelEx(&lr, gemm_reduce_kernel, prm, (int32_t)sms));
    }
    return FS_OK;
}
