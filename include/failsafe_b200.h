/*
 * failsafe_b200.h -- C ABI of the B200-native FailSafe hybrid-attention
 * decode hot path (libfailsafe_b200.so).
 *
 * Plain C: fixed-width integers, raw pointers, sizes; no torch / CUDA types
 * in the signatures (streams are passed as `void*` = cudaStream_t).  Every
 * entry point returns an int status:
 *
 *   FS_OK            0
 *   FS_EVALIDATION   1  -> failsafe.ValidationError  (reference core.py:17-22)
 *   FS_ESIMULATION   2  -> failsafe.SimulationError  (reference core.py:25-26)
 *   FS_ECUDA         3  -> CUDA error, surfaced as SimulationError
 *
 * with a thread-local message in fs_last_error().  All buffers are caller
 * owned; nothing allocates on the hot path; no internal threads; results
 * are deterministic for a fixed device (the stream-K split depends only on
 * the SM count).
 *
 * Reference interfaces replaced (all in /root/reference/pkg/src/failsafe):
 *   fs_plan_placement   <- placement.make_placement        placement.py:180-186
 *                          (naive/cyclic _block_plan 117-135, hybrid 148-170)
 *   fs_plan_ffn         <- placement.ffn_assignment        placement.py:94-114
 *   fs_plan_on_demand   <- recovery.plan_weight_recovery(.., "on_demand")
 *                          target placement               recovery.py:323-340, 396-427
 *   fs_kv_footprint     <- placement.memory_footprint      placement.py:206-236
 *   fs_plan_pages       <- (new) device page/work table for one decode step;
 *                          the device form of the per-rank head residency of
 *                          refexec.ShardedView            refexec.py:136-148
 *   fs_decode_attention <- the attention half of refexec.parallel_forward
 *                          (TP heads on owners, DP heads on routed rank)
 *                                                          refexec.py:281-297, 85-103
 *   fs_prefill_attention <- the multi-row (chunked-prefill) form of
 *                          refexec._head_attention for Alg. 1 batches
 *                          (scheduler.build_prefill_batch) refexec.py:85-103,
 *                                                          scheduler.py:189-245
 *   fs_plan_prefill_tiles <- (new) host tile/split planner of that launch
 *   fs_ar_residual      <- the ordered sum of parallel_forward's per-rank
 *                          partials (+ residual), refexec.py:283-307, as one
 *                          kernel over IPC-mapped peer memory
 *   fs_kv_write / fs_kv_read <- (new) KV append into / read from pages
 *   fs_pages_gather     <- recovery.advance_backup executed as an incremental
 *                          page copy to pinned host       recovery.py:193-247
 *   fs_pages_scatter    <- recovery.plan_kv_recovery "pcie_host" kv_slice
 *                          transfers executed             recovery.py:430-504
 *   fs_copy_peer        <- recovery.plan_weight_recovery transfers executed
 *                          peer-to-peer over NVLink       recovery.py:396-427
 *   fs_kv_backup_tokens <- advance_backup's drain of the tokens a decode step
 *                          appends (token-granular)       recovery.py:193-247
 *   fs_host_register    <- (new) the shared host mirrors the plans read from
 *   fs_copy_2d / fs_copy_segments <- apply_weight_plan's pcie_host /
 *                          nvlink_peer slices into the survivors' weights
 *                                                          recovery.py:396-427, 591-600
 */
#ifndef FAILSAFE_B200_H
#define FAILSAFE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FS_OK 0
#define FS_EVALIDATION 1
#define FS_ESIMULATION 2
#define FS_ECUDA 3

#define FS_ABI_VERSION 1

/* owner-table value of a replicated (data-parallel) head */
#define FS_REPLICATED (-1)

/* placement modes (placement.py:173-177) */
#define FS_MODE_NAIVE 0
#define FS_MODE_CYCLIC 1
#define FS_MODE_HYBRID 2

/* Page format: one page holds FS_PAGE_TOKENS tokens of ONE kv head:
 * K rows [0,16) then V rows [0,16).  Each half is two 2 KB atoms (head
 * dims 0-63, then 64-127); an atom is 16 rows x 128 B with the 16-byte chunk
 * c (0..7) of row r stored at chunk position c ^ (r & 7) -- the tcgen05 /
 * TMA SWIZZLE_128B pattern, and bank-conflict-free for ldmatrix.  K and
 * V are bf16, stored exactly as given (any finite bf16 value round-trips);
 * the kernels run P.V with P split into a bf16 hi + lo pair.  8 KiB per
 * page. */
#define FS_PAGE_TOKENS 16
#define FS_HEAD_DIM 128
#define FS_PAGE_BYTES 8192
#define FS_MAX_Q_PER_KV 8

int fs_abi_version(void);
const char *fs_last_error(void);
/* number of SMs of `device` (sizes the stream-K partition), or <0 */
int fs_device_sms(int device);

/* ---------------------------------------------------------------- host --- */

/* owner[L*H] <- GPU id of each (layer, head), FS_REPLICATED for hybrid's
 * replicated heads.  alive: n_alive distinct GPU ids (any order). */
int fs_plan_placement(int mode, int num_layers, int num_kv_heads,
                      const int32_t *alive, int n_alive, int32_t *owner);

/* shard_owner[num_shards] <- GPU id of each FFN shard */
int fs_plan_ffn(int num_shards, const int32_t *alive, int n_alive,
                int32_t *shard_owner);

/* On-demand shrink target: survivors keep their heads/shards, departed
 * GPUs' TP heads become replicated, lost shards go to the least-loaded
 * survivor (ties -> lowest id). */
int fs_plan_on_demand(int num_layers, int num_kv_heads, const int32_t *owner,
                      int num_shards, const int32_t *shard_owner,
                      const int32_t *survivors, int n_surv,
                      int32_t *new_owner, int32_t *new_shard_owner);

/* Per-GPU KV bytes of a placement for given request token counts and
 * routing (routing[r] = GPU of request r; may be NULL if no replicated
 * heads).  out_bytes[i] corresponds to alive[i]. */
int fs_kv_footprint(int num_layers, int num_kv_heads, const int32_t *owner,
                    const int32_t *alive, int n_alive, const int64_t *tokens,
                    const int32_t *routing, int n_req, int64_t unit,
                    int64_t *out_bytes);

/* -------------------------------------------------------------- device --- */

/* K4: page prefix per segment (one segment = one layer's work items).
 * For segment s with items [seg_items[s], seg_items[s+1]) it writes the
 * exclusive prefix of ceil(item_len/16) to
 * page_off[seg_items[s] + s .. seg_items[s+1] + s] (n+1 entries). */
int fs_plan_pages(const int32_t *item_len, const int32_t *seg_items, int n_segs,
                  int32_t *page_off, void *stream);

typedef struct fs_decode_desc {
    const void *q;             /* bf16; item i's q_per_kv x 128 query block
                                  starts at element item_qoff[i]            */
    const void *kv_pool;       /* pages, FS_PAGE_BYTES each                 */
    const int32_t *block_table;/* [n_seq][bt_stride] page ids               */
    int64_t bt_stride;
    const int32_t *item_seq;   /* [n_items] block-table row                 */
    const int32_t *item_len;   /* [n_items] tokens attended (>=0), incl. the
                                  new token at position len-1               */
    const int32_t *item_qoff;  /* [n_items] element offset into q           */
    const int32_t *item_ooff;  /* [n_items] element offset into out         */
    const int32_t *page_off;   /* [n_items+1] from fs_plan_pages            */
    const void *kv_new;        /* bf16 new-token K/V source, or NULL: when
                                  set, the token at len-1 is first written
                                  into its page (fused KV append)           */
    const int32_t *item_koff;  /* [n_items] element offset of the new K row */
    const int32_t *item_voff;  /* [n_items] element offset of the new V row */
    int32_t *item_sem;         /* [n_items] zero-initialised; left zero     */
    int32_t n_items;
    int32_t q_per_kv;          /* 1..8                                      */
    float scale;               /* softmax scale, normally 1/sqrt(head_dim)  */
    int32_t out_fp32;          /* 0: bf16 out, 1: fp32 out                  */
    void *out;                 /* q_per_kv x 128 block per item at ooff     */
    float *part_o;             /* [partial_slots][q_per_kv][128] fp32       */
    float *part_lse;           /* [partial_slots][q_per_kv]                 */
    int64_t partial_slots;     /* >= fs_decode_partial_slots(n_items)       */
    int32_t device;            /* CUDA device ordinal the launch runs on    */
    int32_t config;            /* 0 = default kernel configuration          */
    int32_t flags;             /* FS_DECODE_* bits                          */
} fs_decode_desc;

/* fs_decode_desc.flags: the caller guarantees that the kernel launched
 * immediately before on the stream writes none of page_off, item_len,
 * item_seq, block_table or the pages (e.g. it is the projection GEMM), so
 * the launch may read them and stage its first pages before its
 * programmatic-dependent-launch wait.  Without the bit every read waits
 * for the preceding kernel to complete (K3 / K4 / restores may precede). */
#define FS_DECODE_EARLY_PREFETCH 1

/* partial-result slots the stream-K split needs for n_items items
 * (config -1: enough for every kernel configuration) */
int64_t fs_decode_partial_slots(int device, int32_t n_items, int32_t config);

/* K1 (+ fused K2 combine, + optional fused K3 append): split-KV (stream-K
 * over pages) paged GQA decode with the log-sum-exp merge of split items
 * done in-kernel by the item's last warp.  ONE launch.  Output blocks not
 * named by any item are untouched. */
int fs_decode_attention(const fs_decode_desc *d, void *stream);

/* K8: paged chunked-prefill GQA attention.  Item i is one (kv head,
 * request chunk): item_len[i] new tokens at prompt positions item_start[i]
 * .. item_start[i]+item_len[i]-1 of block-table row item_seq[i] (their K/V
 * already in the pages); chunk token j attends causally, including itself,
 * to positions 0..item_start[i]+j (refexec.py:92-97).  A tile = up to
 * fs_prefill_tokens_per_tile(q_per_kv, variant) consecutive chunk tokens x
 * all q_per_kv heads (128 or 64 query rows) over the KV page range
 * [page0, page1);
 * tile_slot < 0 -> the tile covers its whole causal range and writes the
 * output; otherwise it writes a partial (O/l, log2-sum-exp) to that slot and
 * the combine list merges slots comb_slot0 .. +comb_nsplit-1 of each
 * (item, tok0) in the same call.  Tiles come from fs_plan_prefill_tiles. */
typedef struct fs_prefill_desc {
    const void *q;             /* bf16: block of (item i, token j) at element
                                  item_qoff[i] + j*q_stride, q_per_kv x 128 */
    void *out;                 /* bf16 (fp32 if out_fp32): item_ooff[i] +
                                  j*o_stride                                */
    int64_t q_stride, o_stride;
    int32_t out_fp32;
    const void *kv_pool;
    const int32_t *block_table;
    int64_t bt_stride;
    const int32_t *item_seq, *item_start, *item_len, *item_qoff, *item_ooff;
    const int32_t *tile_item, *tile_tok0, *tile_page0, *tile_page1, *tile_slot;
    int32_t n_tiles;
    const int32_t *comb_item, *comb_tok0, *comb_slot0, *comb_nsplit;
    int32_t n_comb;
    int32_t q_per_kv;          /* 1..8                                      */
    float scale;
    void *part_o;              /* [partial_slots][rows][128] fp32 (split
                                  partials O / l)                           */
    float *part_lse;           /* [partial_slots][rows]                     */
    int64_t partial_slots;
    int32_t variant;           /* 0: tcgen05 (TMEM accumulators, 256-row
                                  tiles = two 128-row halves, 64-key
                                  blocks); 1: mma.sync (64-row tiles);
                                  2: tcgen05, 128 rows; 3: as 0 with
                                  128-key blocks                           */
} fs_prefill_desc;

/* chunk tokens per tile (rows / q_per_kv; rows = 256 / 64 / 128 / 256 for
 * variants 0 / 1 / 2 / 3), or <0 */
int fs_prefill_tokens_per_tile(int q_per_kv, int variant);

/* Host planner of the K8 launch: token tiles of every item, each split into
 * equal KV page ranges so the grid has >= ~target_units similar-sized
 * tiles (pass 4*SMs); heaviest tiles first.  Output arrays sized by the
 * caller with max_tiles / max_comb entries; returns the tile count in
 * *n_tiles, combine groups in *n_comb and the partial slots used in
 * *n_slots.  FS_EVALIDATION if the arrays are too small. */
int fs_plan_prefill_tiles(int32_t n_items, const int32_t *item_start, const int32_t *item_len,
                          int32_t q_per_kv, int32_t variant, int32_t target_units, int32_t max_tiles,
                          int32_t *tile_item, int32_t *tile_tok0, int32_t *tile_page0,
                          int32_t *tile_page1, int32_t *tile_slot, int32_t *n_tiles,
                          int32_t max_comb, int32_t *comb_item, int32_t *comb_tok0,
                          int32_t *comb_slot0, int32_t *comb_nsplit, int32_t *n_comb,
                          int32_t *n_slots);

int fs_prefill_attention(const fs_prefill_desc *d, void *stream);

/* K3: write n_tok (K,V) rows into pages: token t goes to sequence
 * tok_seq[t] at position tok_pos[t]; its K/V are rows tok_src[t] of
 * k_src/v_src (bf16, row stride src_stride elements, 128 used). */
int fs_kv_write(void *kv_pool, const int32_t *block_table, int64_t bt_stride,
                const int32_t *tok_seq, const int32_t *tok_pos,
                const int32_t *tok_src, int32_t n_tok, const void *k_src,
                const void *v_src, int64_t src_stride, void *stream);

/* K3 over runs of consecutive tokens (the serving iteration's form: one
 * run per (prefill chunk or decode token, head slot)): run r covers tokens
 * run_off[r] - run_off[0] .. run_off[r+1] - run_off[0] - 1 of this launch;
 * its i-th token goes to sequence run_seq[r] at position run_pos[r] + i and
 * its K/V are rows run_src[r] + i * src_step of k_src / v_src.  run_off:
 * n_runs + 1 nondecreasing entries (a slice of a prefix sum is fine);
 * n_tok = run_off[n_runs] - run_off[0] (the host's copy: sizes the grid). */
int fs_kv_write_runs(void *kv_pool, const int32_t *block_table, int64_t bt_stride,
                     const int32_t *run_seq, const int32_t *run_pos, const int32_t *run_src,
                     const int32_t *run_off, int32_t n_runs, int32_t n_tok, int32_t src_step,
                     const void *k_src, const void *v_src, int64_t src_stride, void *stream);

/* inverse of fs_kv_write (tests / debugging) */
int fs_kv_read(const void *kv_pool, const int32_t *block_table, int64_t bt_stride,
               const int32_t *tok_seq, const int32_t *tok_pos,
               const int32_t *tok_dst, int32_t n_tok, void *k_dst, void *v_dst,
               int64_t dst_stride, void *stream);

/* K5: backup gather.  Page page_ids[i] -> slot (dst_slots ? dst_slots[i] : i)
 * of dst (FS_PAGE_BYTES per slot).  dst may be mapped pinned host memory:
 * the copy then runs over PCIe from a single launch on a side stream. */
int fs_pages_gather(const void *kv_pool, const int32_t *page_ids, int32_t n_pages,
                    void *dst, const int32_t *dst_slots, int32_t max_ctas, void *stream);

/* K6: restore scatter.  Slot (src_slots ? src_slots[i] : i) of src -> page
 * page_ids[i].  src may be mapped pinned host memory (the KV backup). */
int fs_pages_scatter(void *kv_pool, const int32_t *page_ids, int32_t n_pages,
                     const void *src, const int32_t *src_slots, int32_t max_ctas,
                     void *stream);

/* K5, token-granular (decode steps): for every item the token at
 * item_len[i]-1 (512 B: its K and V rows) is copied from its page to the
 * same page slot of `mirror` (FS_PAGE_BYTES per slot, slot == page id;
 * typically mapped pinned host memory shared with the other ranks).
 * Replaces advance_backup's per-step drain (recovery.py:193-247) of the
 * tokens a decode step appends. */
int fs_kv_backup_tokens(const void *kv_pool, const int32_t *block_table, int64_t bt_stride,
                        const int32_t *item_seq, const int32_t *item_len, int32_t n_items,
                        void *mirror, void *stream);

/* Page-lock a host range (e.g. a /dev/shm mapping shared by the ranks of a
 * node: the KV backup mirror and the weight store outlive the process that
 * wrote them) for zero-copy / DMA access; *dev_ptr = its device address. */
int fs_host_register(void *ptr, int64_t bytes, void **dev_ptr);
int fs_host_unregister(void *ptr);

/* K7 transfer primitive: 2-D copy (rows of `width` bytes) between any of
 * registered host memory, local device memory and a peer's device memory
 * mapped by CUDA IPC (NVLink); apply_weight_plan's pcie_host and
 * nvlink_peer slices (recovery.py:396-427, 591-600). */
int fs_copy_2d(void *dst, int64_t dpitch, const void *src, int64_t spitch, int64_t width,
               int64_t height, void *stream);

/* K7 executor: ONE launch performing n_segs 2-D copies (segs and row_off
 * in device memory; row_off[i] = sum of heights before segment i, n_segs+1
 * entries).  src / dst may be local HBM, peer HBM mapped by CUDA IPC
 * (NVLink) or mapped pinned host memory (fs_host_register; PCIe).  Used to
 * execute apply_weight_plan (recovery.py:591-600): the plan's pcie_host
 * slices, its nvlink_peer remainders and the scatter of the recovered
 * shards into a survivor's fused weight tensors.  ctas <= 0: 4 per SM. */
typedef struct fs_copy_seg {
    const void *src;
    void *dst;
    int64_t spitch, dpitch;   /* bytes between rows                        */
    int64_t width, height;    /* bytes per row, rows                       */
} fs_copy_seg;
int fs_copy_segments(const fs_copy_seg *segs, const int64_t *row_off, int32_t n_segs,
                     int32_t ctas, void *stream);

/* Skinny weight-streaming GEMM of the decode step (tcgen05.mma + TMA):
 *   STORE    (0): out[n, c]  = sum_k x[n, k] W[k, c]
 *   RESIDUAL (1): out[n, c]  = res[n, c] + sum_k x[n, k] W[k, c]  (out may == res)
 *   SWIGLU   (2): out[n, 64t+j] = silu(g) * u with g, u the columns 128t+j and
 *                 128t+64+j of x.W (gate/up interleaved in 64-column blocks)
 * Replaces the projection matmuls of refexec.py:287-307 (q/k/v, o, gated
 * FFN; _ffn_partial refexec.py:106-108) for the decode batch.
 * x: bf16 [rows <= 64][K] (row stride ld_x), W: bf16 [K][N] row-major (row
 * stride ld_w, w_layout 0) or pre-packed (gemm.PackedWeight): w_layout 1 =
 * 16 KB UMMA-canonical K-major SWIZZLE_128B blocks per (128-column tile,
 * 64-k step) ordered [tile][step]; w_layout 2 = the same blocks for pairs of
 * tiles, ordered [pair][step][tile] (used when the tiles outnumber the SMs).
 * K % 64 == 0, N % 128 == 0; out / res 16-byte aligned with row strides
 * that are multiples of 8.  One launch per call: grid = column groups x S
 * k-splits <= SMs, each split group a thread-block cluster whose partial
 * tiles are summed over distributed shared memory in split order
 * (deterministic); programmatic dependent launch (the first weight stages
 * are fetched while the previous kernel drains).  workspace / sems are
 * reserved (must be non-null; fs_gemm_workspace_floats returns 1). */
int64_t fs_gemm_workspace_floats(int device, int32_t N, int32_t epilogue);
int fs_gemm_skinny(const void *x, int64_t ld_x, int32_t rows, int32_t K, const void *w,
                   int64_t ld_w, int32_t w_layout, int32_t N, void *out, int64_t ld_out, const void *res,
                   int64_t ld_res, int32_t epilogue, float *workspace, int64_t ws_floats,
                   int32_t *sems, int32_t device, void *stream);

/* k-split count (CTAs per column group; grid = N / 128 / G x splits) that
 * fs_gemm_skinny uses for this shape and W layout on `device` (>= 1), or a
 * negative status. */
int fs_gemm_plan(int32_t device, int32_t K, int32_t N, int32_t w_layout);

/* TP MLP partial nonlinearity: out[r, c] = silu(h[r, c]) * h[r, cols + c]
 * (bf16; h row stride ld >= 2*cols; gated FFN of core.py:93-95). */
int fs_swiglu(const void *h, int64_t rows, int64_t cols, int64_t ld, void *out,
              int64_t ld_out, void *stream);

/* Synthetic weights: out[i, j] = scale * N(0,1) keyed by (seed, salt, global
 * row, global col); global row = row_map ? row_map[i] : row_off + i (same for
 * columns), so every rank materialises identical slices of one model. */
int fs_fill_normal(void *out, int64_t rows, int64_t cols, int64_t ld,
                   const int32_t *row_map, int64_t row_off, const int32_t *col_map,
                   int64_t col_off, uint64_t seed, uint64_t salt, float scale, void *stream);

/* ---- the exchange: ordered-sum all-reduce + residual over peer memory ----
 * (refexec.py:283-307).  Each rank owns symmetric buffers of
 * fs_ar_buffer_bytes(max_elems) bytes (fs_ar_alloc: zeroed cudaMalloc;
 * layout [partial][slice sums][flags]), shares them with CUDA IPC
 * (fs_ar_ipc_handle -> 64-byte handle -> fs_ar_ipc_open on every peer) and
 * writes its bf16 partial to the first n elements of its own buffer.
 * fs_ar_residual then signals / waits on the peers' flags and does
 * x[i] += bf16(sum over ranks 0..world-1, in order, in fp32, of
 * partial_r[i]) in ONE launch (peers[r] = buffer of rank r as mapped in
 * this process, data_bytes = the buffer's flag offset =
 * fs_ar_buffer_bytes(max_elems) - 256).  Consecutive exchanges must
 * alternate between two buffers.  Traps (no hang) if a peer never arrives.
 * fs_ar_residual_mode: mode 1 = one-shot (every rank reads every partial),
 * 2 = two-shot (each rank sums its 1/world slice, then gathers the rounded
 * slices: (world-1)/world of the vector read twice instead of world-1
 * times), 0 = auto (two-shot for world > 2 and >= 256 KiB); identical
 * bits in every mode.  fs_ar_residual = mode 0. */
#define FS_AR_MAX_WORLD 16
int64_t fs_ar_buffer_bytes(int64_t max_elems);
int fs_ar_alloc(int device, int64_t bytes, void **ptr);
int fs_ar_free(void *ptr);
int fs_ar_ipc_handle(void *ptr, void *handle64);
int fs_ar_ipc_open(const void *handle64, void **ptr);
int fs_ar_ipc_close(void *ptr);
int fs_ar_residual(void *const *peers, int32_t rank, int32_t world, int64_t n,
                   int64_t data_bytes, void *x, int32_t ctas, void *stream);
int fs_ar_residual_mode(void *const *peers, int32_t rank, int32_t world, int64_t n,
                        int64_t data_bytes, void *x, int32_t ctas, int32_t mode, void *stream);

/* K7: enable peer access (idempotent) and peer copy */
int fs_enable_peer(int device, int peer);
int fs_copy_peer(void *dst, int dst_device, const void *src, int src_device,
                 int64_t bytes, void *stream);

/* Debugging (tools/gemm_tl.py): per-CTA globaltimer phase stamps of the
 * skinny GEMM are written to dev_buf while it is non-NULL. */
void fs_gemm_debug_timestamps(unsigned long long *dev_buf);

#ifdef __cplusplus
}
#endif
#endif /* FAILSAFE_B200_H */
