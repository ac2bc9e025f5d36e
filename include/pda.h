/*
 * pda.h -- C ABI of the B200 paged decode attention library (libpda.so).
 *
 * The hot path of arXiv 2504.06319 ("L2-cache-oriented asynchronous KV cache
 * prefetching"): decode-phase attention of one query token per sequence over
 * a paged KV cache gathered block by block through a block table, with the
 * K/V blocks a tunable distance ahead prefetched into L2 while the current
 * block is being computed.  Citations: P:n = PAPER.md line n.
 *
 *   out[b, h, :] = sum_t softmax_t(scale * q[b,h,:] . k_t) * v_t,
 *   t in [0, context_lens[b]),  k_t/v_t gathered through block_tables[b]
 *   ("logits . V"; QK^T with resident Q; Alg. 1).
 *
 * General conventions (apply to every entry point):
 *  - Tensor pointers passed to the compute entry points are DEVICE pointers
 *    owned by the caller; the library never allocates, frees or synchronises
 *    them.  Work is enqueued on `stream` (a cudaStream_t passed as void*;
 *    NULL = legacy default stream).  Calls are stateless and thread-safe.
 *  - The split-K kernels are launched with programmatic stream serialization
 *    (PDL): they may be scheduled while the previous grid in the stream
 *    drains and wait for its completion before their first global read.
 *    The split-K grid releases its dependents (griddepcontrol.launch_dependents)
 *    after its main loop, BEFORE its epilogue stores `out`, the workspace and
 *    peer buffers.  For ordinary launches (and for any kernel launched without
 *    the programmatic-serialization attribute) stream order is unchanged; a
 *    caller's own kernel launched WITH that attribute right after this call
 *    may start early and must execute griddepcontrol.wait /
 *    cudaGridDependencySynchronize() before reading this call's outputs.
 *    Environment PDA_PDL=0 disables PDL.
 *  - Host-side argument errors are returned synchronously before any launch;
 *    launch failures map to PDA_ERR_CUDA.  No C++ exception crosses the ABI.
 *  - Device-resident values (block ids, lengths) are not validated: a block
 *    id outside [0, num_blocks) is undefined behaviour; context_lens[b] is
 *    clamped to max_blocks_per_seq * block_size.  pda_validate_inputs is
 *    the debug check that flags them.
 *  - Layouts (all row-major, contiguous):
 *      q, out        [num_seqs, num_q_heads, head_dim]
 *      k_cache/v_cache [num_blocks, num_kv_heads, block_size, head_dim]
 *        -- each (block, kv head) slab is contiguous, "each block exclusively
 *           stores KV Cache data for a single attention head"; its
 *           size is Eq. 1's M_block = b * d_h * T_block bytes.
 *      block_tables  [num_seqs, max_blocks_per_seq] int32 physical block ids
 *                    (one table per sequence, shared by all heads; Alg. 1 bt)
 *      context_lens  [num_seqs] int32, 0 <= L_b
 *  - GQA: q head h reads kv head floor(h / (Hq / Hkv)); Hq % Hkv == 0.
 *  - Supported: head_dim in {64, 128}, block_size == 16,
 *    Hq / Hkv <= 16, dtype fp16 or bf16, out dtype = dtype or fp32.
 *    Base pointers must be 16-byte aligned (TMA / bulk-prefetch requirement).
 *  - context_lens[b] == 0 yields a zero output row.  Tokens >= L_b inside the
 *    last block and blocks not referenced by the table are never read into
 *    the result: they may hold anything, NaN included.
 */
#ifndef PDA_H_
#define PDA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    PDA_OK = 0,
    PDA_ERR_NULL = 1,        /* a required pointer is NULL */
    PDA_ERR_SHAPE = 2,       /* inconsistent or out-of-range sizes */
    PDA_ERR_UNSUPPORTED = 3, /* valid but not implemented (head_dim, block_size, group) */
    PDA_ERR_ALIGN = 4,       /* a base pointer is not 16-byte aligned */
    PDA_ERR_WORKSPACE = 5,   /* workspace NULL or smaller than pda_workspace_bytes() */
    PDA_ERR_CUDA = 6         /* a CUDA runtime/driver call or launch failed */
} pda_status;

typedef enum {
    PDA_F16 = 0,
    PDA_BF16 = 1,
    PDA_F32 = 2, /* out_dtype only */
    PDA_E4M3 = 3 /* kv_dtype only: OCP FP8 E4M3 codes with per-tensor scales */
} pda_dtype;

/* L2 prefetch of upcoming KV blocks (Section 3.2). */
typedef enum {
    PDA_PF_OFF = 0,     /* no prefetch: the ablation baseline */
    PDA_PF_BULK_L2 = 1, /* cp.async.bulk.prefetch.L2 of each K and V slab (one instruction per slab) */
    PDA_PF_LINE_L2 = 2, /* prefetch.global.L2 of every 128-byte line of each slab */
    PDA_PF_AUTO = 3     /* the planner decides where the paper's structure and prefetch pay
                           (measured on B200): with kernel AUTO, a short-context
                           step (one query token, 16-bit KV, contexts of at most 512 tokens)
                           with GQA groups of >= 4 and 128 <= B * Hq <= 512 q-head rows
                           (<= 256 at contexts above 256 tokens) runs the paper-structure
                           kernel -- one CTA per q-head row -- with Alg. 1's line prefetch at
                           distance 4 and evict_last prefetches (eviction AUTO): 1.12-1.52x
                           over split-K there; every other step runs split-K without prefetch,
                           where no prefetch variant was ever faster (p10 of the paired speedup
                           < 1 on all cells).  prefetch_distance is ignored.  A step that fuses
                           the KV append or the output gather keeps split-K. */
} pda_prefetch;

/* L2 eviction priority of the KV traffic ("adjusting the cache eviction
 * priority of prefetched data").  Bit 0: demand K/V loads are marked
 * evict_first (each block is read once per step, "can be safely
 * evicted"); bit 1: prefetched lines are marked evict_last. */
typedef enum {
    PDA_EV_NORMAL = 0,
    PDA_EV_DEMAND_FIRST = 1,
    PDA_EV_PREFETCH_LAST = 2,
    PDA_EV_BOTH = 3,
    PDA_EV_AUTO = 4 /* planner: DEMAND_FIRST when the step's KV bytes (upper bound
                       B * max_blocks * Hkv * M_block * 2) are <= 2 GiB, else NORMAL
                       (measured on B200) */
} pda_eviction;

typedef enum {
    PDA_KERNEL_AUTO = 0,   /* = PDA_KERNEL_SPLITK (fastest measured on B200) */
    PDA_KERNEL_PAPER = 1,  /* the paper's structure: grid [Hq, B], 4 warps, warp-per-block,
                              K/V loaded to registers (Section 3.1) */
    PDA_KERNEL_SPLITK = 2, /* B200 kernel: split-K over context partitions, TMA ring in
                              shared memory, mma.sync, GQA group per CTA; a small combine
                              kernel merges partitions when P_max > 1 */
    PDA_KERNEL_STREAM = 3, /* B200 persistent kernel: every warp a self-pipelined stream over an
                              equal share of all KV blocks of the step (load-balanced for any
                              length mix), partial rows merged in-kernel; one launch */
    PDA_KERNEL_BALANCED = 4, /* B200 persistent split-K kernel: one wave of CTAs (producer warp +
                              4 consumer warps each), CTA c owns an equal share of all KV blocks
                              of the step, rows merged in-kernel (ticket); one launch */
    PDA_KERNEL_TC = 5      /* B200 tcgen05 kernel (decode_tc.cu): one persistent CTA per SM owning
                              an equal share of the step's KV blocks; QK^T and PV on the 5th-gen
                              tensor core (tcgen05.mma, accumulators in TMEM), 128-token tiles;
                              split rows merged by a combine kernel.  16-bit KV, head_dim 128,
                              one query token, no fused append / gather, no trace */
} pda_kernel;

typedef struct {
    int32_t num_seqs;           /* B */
    int32_t num_q_heads;        /* Hq */
    int32_t num_kv_heads;       /* Hkv */
    int32_t head_dim;           /* D */
    int32_t block_size;         /* tokens per KV block (16) */
    int32_t num_blocks;         /* physical blocks in k_cache / v_cache */
    int32_t max_blocks_per_seq; /* columns of block_tables */
    int32_t dtype;              /* pda_dtype of q (and of the caches unless kv_dtype says e4m3) */
    int32_t out_dtype;          /* pda_dtype of out */
    int32_t kv_dtype;           /* pda_dtype of k_cache / v_cache: == dtype, or PDA_E4M3 (1 byte per
                                   element; value = k_scale|v_scale * e4m3(code); head_dim 128 and the
                                   split-K kernel only; a bf16 q is converted to fp16 for the MMAs) */
    int32_t q_len;              /* query tokens per sequence (0 or 1 = single-token decode).  > 1:
                                   multi-token (speculative) decode, q and out are [B, q_len, Hq, D],
                                   context_lens counts the q_len new tokens (already in the cache) and
                                   query token i attends to tokens [0, L - q_len + i]; split-K kernel
                                   only, q_len * (Hq / Hkv) <= 16 */
} pda_shape;

typedef struct {
    int32_t prefetch;          /* pda_prefetch */
    int32_t prefetch_distance; /* blocks ahead of the block being issued; >= 1 when prefetch on.
                                  Paper kernel: d = 4 (= warps) reproduces Alg. 1 exactly;
                                  stream / balanced kernels and e4m3 caches: d <= 32 */
    int32_t partition_tokens;  /* split-K partition size P in tokens; 0 = planner's choice;
                                  otherwise a positive multiple of block_size */
    int32_t smem_stages;       /* shared-memory ring depth in blocks; 0 = planner's choice.
                                  split-K: 4, 8, 12 per CTA (auto: 8, or 4 when the grid fits two
                                  waves at 4 CTAs/SM but not one at 3); e4m3 cache: 8, 16, 24
                                  (blocks consumed in pairs) or 12 (one at a time, 4 CTAs/SM)
                                  (auto: 12 up to 1 GiB of e4m3 KV, else 16);
                                  balanced: 4, 8 (default), 12 (per CTA; multiples of the 4 consumer warps);
                                  stream: per warp, with stream_warps: (8,1), (4,2), (6,2) default, (4,4) */
    int32_t kernel;            /* pda_kernel */
    int32_t num_sms;           /* SMs the planner assumes; 0 = 148 (B200) */
    int32_t stream_warps;      /* stream kernel: warps (streams) per CTA; 0 = default (2) */
    int32_t eviction;          /* pda_eviction (0 = normal) */
    int32_t issue_mode;        /* split-K ring refill: 0 = auto (= 2), 1 = a producer warp, 2 = each
                                  consumer warp refills its own stages (always for e4m3);
                                  self-issue limits prefetch_distance to 32 */
    float k_scale;             /* e4m3 cache only: K dequantisation scale (0 = 1.0) */
    float v_scale;             /* e4m3 cache only: V dequantisation scale (0 = 1.0) */
    int32_t merge;             /* split-K partition merge (S8) when P_max > 1: 0 = auto (cluster
                                  when P_max <= 8, the grid is one wave with at least one CTA
                                  per SM and the device can hold all its clusters at once --
                                  cudaOccupancyMaxActiveClusters, asked when num_sms is 0 --
                                  else combine kernel), 1 = combine kernel
                                  through the workspace, 2 = cluster (P_max <= 16): the
                                  partitions of a (seq, kv head) row run as one thread-block
                                  cluster and merge through distributed shared memory, no
                                  workspace, no second launch.  Bitwise-identical results. */
} pda_options;

/* Result of the (host-only, deterministic) split-K planner. */
typedef struct {
    int32_t kernel;           /* the kernel that will run (PDA_KERNEL_PAPER or _SPLITK) */
    int32_t partition_tokens; /* P (split-K) or max_blocks_per_seq * block_size (paper) */
    int32_t p_max;            /* partitions per sequence = ceil(max_blocks*bs / P) */
    int32_t smem_stages;      /* ring depth */
    int32_t grid_x, grid_y, grid_z; /* main kernel grid (stream: grid_x CTAs x stream_warps) */
    int32_t threads;          /* main kernel block size */
    int32_t trace_rec_len;    /* int32 words per trace record (see paged_decode_attention_trace) */
    int32_t trace_records;    /* number of trace records */
    int32_t eviction;         /* resolved pda_eviction (never PDA_EV_AUTO) */
    int32_t cluster;          /* split-K: CTAs per cluster (= p_max) when partitions merge in a
                                 cluster, else 0 (combine kernel when p_max > 1) */
    size_t workspace_bytes;   /* == pda_workspace_bytes() */
} pda_plan_info;

/* Host-only validation of shape and options (no CUDA context needed). */
pda_status pda_check_args(const pda_shape* shape, const pda_options* opt);

/* Plan the launch (host-only, deterministic; no CUDA context needed). */
pda_status pda_plan(const pda_shape* shape, const pda_options* opt, pda_plan_info* plan);

/* Bytes of device workspace paged_decode_attention needs: the split-K
 * partials (o_p fp32 [B, Hq, P_max, D] and lse_p fp32 [B, Hq, P_max]);
 * 0 when P_max == 1 or for the paper kernel.  Stream kernel: partials of
 * the streams' (balanced: CTAs') first/last segments (fp32 [NS, 2, 8*ceil(g/8), D + 1]) and one
 * uint32 arrival ticket per (seq, kv head) at the end of the buffer: the
 * whole workspace must be ZERO before its first use (every completed call
 * leaves the tickets zero again; applies to the stream and balanced kernels).
 * Returns 0 on invalid args. */
size_t pda_workspace_bytes(const pda_shape* shape, const pda_options* opt);

/* The decode attention step (the method's hot path).
 *   q            [B, Hq, D] dtype                      (device, read)
 *   k_cache      [num_blocks, Hkv, bs, D] dtype        (device, read)
 *   v_cache      [num_blocks, Hkv, bs, D] dtype        (device, read)
 *   block_tables [B, max_blocks_per_seq] int32         (device, read)
 *   context_lens [B] int32                             (device, read)
 *   scale        softmax scale, applied in fp32 to q.k (never folded into q)
 *   out          [B, Hq, D] out_dtype                  (device, written)
 *   workspace    device scratch of >= pda_workspace_bytes() (may be NULL if 0)
 * Results are bit-identical for every prefetch mode and distance and
 * run-to-run (no atomics; fixed-order combine). */
pda_status paged_decode_attention(const void* q, const void* k_cache, const void* v_cache,
                                  const int32_t* block_tables, const int32_t* context_lens,
                                  float scale, void* out, const pda_shape* shape,
                                  const pda_options* opt, void* workspace,
                                  size_t workspace_bytes, void* stream);

/* Same computation, additionally writing the kernel's own bookkeeping trace
 * to the device buffer `trace` (int32, plan.trace_records * plan.trace_rec_len
 * words, R = (trace_rec_len - 4) / 2):
 *   split-K: one record per unit u = (b * Hkv + kvh) * P_max + p;
 *            rec[0..1] = token range [s, e) (s = e = min(p*P, L) when empty)
 *   paper:   one record per (b, h, warp) u = (b * Hq + h) * 4 + warp;
 *            rec[0] = first block index (= warp), rec[1] = e = ceil(L / bs)
 *   stream / balanced: one record per row u = b * Hkv + kvh, R = max_blocks_per_seq;
 *            rec[0] = 0, rec[1] = L; visited[j] and prefetch target[j] are
 *            indexed by the block j that issued them (not issue order);
 *            rows with L = 0 stay all -1
 *   rec[2] = visited block count, rec[3] = prefetch count,
 *   rec[4 .. 4+R)   visited physical block ids in issue order, rest -1,
 *   rec[4+R .. 4+2R) prefetch targets (physical ids) in issue order, rest -1.
 * The caller fills nothing; the library initialises the buffer to -1 first. */
pda_status paged_decode_attention_trace(const void* q, const void* k_cache, const void* v_cache,
                                        const int32_t* block_tables,
                                        const int32_t* context_lens, float scale, void* out,
                                        const pda_shape* shape, const pda_options* opt,
                                        void* workspace, size_t workspace_bytes, int32_t* trace,
                                        size_t trace_words, void* stream);

/* Measurement only: paged_decode_attention_trace (split-K kernel; other
 * kernels return PDA_ERR_UNSUPPORTED) that additionally writes, per unit u of
 * the trace (u = (b * Hkv + kvh) * P_max + p), the unit CTA's timeline to the
 * device buffer `stamps` (uint64, >= 3 * plan.trace_records words):
 *   stamps[3u] = %globaltimer (ns) at CTA entry, stamps[3u+1] = at its exit,
 *   stamps[3u+2] = the SM it ran on.
 * Used to see the grid's ramp, drain and per-CTA stream rate (tools/timeline.py);
 * the trace instantiation runs a few percent slower than the product kernel.
 * NULL trace or stamps: PDA_ERR_NULL; short stamp buffer: PDA_ERR_SHAPE. */
pda_status paged_decode_attention_timeline(const void* q, const void* k_cache, const void* v_cache,
                                           const int32_t* block_tables,
                                           const int32_t* context_lens, float scale, void* out,
                                           const pda_shape* shape, const pda_options* opt,
                                           void* workspace, size_t workspace_bytes, int32_t* trace,
                                           size_t trace_words, uint64_t* stamps,
                                           size_t stamp_words, void* stream);

/* The decode step with the tensor-parallel output all-gather fused into its
 * stores (S9 fused): every output element this rank
 * computes is written directly into the output buffer of each of the n_peers
 * ranks of its group, over NVLink.
 *   out_peers      HOST array of n_peers (1..8) device pointers, each rank's
 *                  [B, q_len, total_q_heads, D] out_dtype buffer, mapped into
 *                  this device's address space (e.g. symmetric memory)
 *   head_offset    first global q head of this rank's shard (its Hq heads land
 *                  at [head_offset, head_offset + Hq) of every buffer)
 * Other arguments as paged_decode_attention; split-K kernel only.  Completion
 * is ordered on `stream`.  Two cross-rank hazards are the caller's to order:
 *   read-after-write  before any rank reads its buffer, the group must pass a
 *                     cross-device barrier after every rank's call (e.g. the
 *                     symmetric-memory barrier);
 *   write-after-read  a rank's call writes into its PEERS' buffers, so no rank
 *                     may start the call that overwrites a buffer while a peer
 *                     still reads that buffer's previous contents.  Either
 *                     alternate two buffer sets between consecutive steps (step
 *                     k writes set k % 2; the barrier ending step k+1 then
 *                     orders every peer's reads of step k before anyone's step
 *                     k+2 writes -- what TPDecodeAttention does), or pass a
 *                     second barrier before the call. */
pda_status paged_decode_attention_gather(const void* q, const void* k_cache, const void* v_cache,
                                         const int32_t* block_tables, const int32_t* context_lens,
                                         float scale, void* const* out_peers, int32_t n_peers,
                                         int32_t head_offset, int32_t total_q_heads,
                                         const pda_shape* shape, const pda_options* opt, void* workspace,
                                         size_t workspace_bytes, void* stream);

/* KV append, the decode step's cache write ("each decoding step requires
 * loading the KV Cache" of all tokens so far; paged layout P:105): the
 * step's q_len new tokens (q_len = shape->q_len, 0 means 1) of each sequence
 * are written into their paged slots.  Token i of sequence b goes to position
 * t = L_b - q_len + i (L_b = context_lens[b] counts the new tokens), i.e. slot
 * t % bs of physical block block_tables[b][t / bs], for every kv head;
 * positions t < 0 are skipped.
 *   k_new, v_new  [B, q_len, Hkv, D] dtype             (device, read)
 *   k_cache, v_cache                                   (device, written)
 * 16-bit caches receive the bit patterns; an e4m3 cache (kv_dtype E4M3)
 * receives code = e4m3(fp32(x) / opt->k_scale) (resp. v_scale): IEEE fp32
 * division, then round to nearest even, saturating to +-448 (scales must be
 * > 0: PDA_ERR_SHAPE otherwise).  The written slots must not be shared with
 * another sequence of the same call (they never are in a paged cache: a
 * sequence's last block is its own). */
pda_status pda_kv_append(const void* k_new, const void* v_new, void* k_cache, void* v_cache,
                         const int32_t* block_tables, const int32_t* context_lens, const pda_shape* shape,
                         const pda_options* opt, void* stream);

/* pda_kv_append followed by paged_decode_attention on the updated cache, as
 * one call.  The split-K kernel fuses the append: the CTA whose partition
 * holds a new token writes it before loading its blocks (one launch fewer);
 * the other kernels run pda_kv_append's kernel first on the same stream.
 * Output identical to the two separate calls (bitwise). */
pda_status paged_decode_attention_append(const void* q, const void* k_new, const void* v_new, void* k_cache,
                                         void* v_cache, const int32_t* block_tables,
                                         const int32_t* context_lens, float scale, void* out,
                                         const pda_shape* shape, const pda_options* opt, void* workspace,
                                         size_t workspace_bytes, void* stream);

/* Debug validation of the device-resident inputs the hot path does not check
 * (block ids, lengths): counts (DEVICE, int64 x 3, written) receives
 *   [0] sequences with context_lens[b] outside [0, max_blocks_per_seq * bs],
 *   [1] referenced block ids (block_tables[b][j], j < ceil(min(L_b, max) / bs))
 *       outside [0, num_blocks),
 *   [2] sequences with either problem.
 * Uses num_seqs, max_blocks_per_seq, num_blocks and block_size of `shape`. */
pda_status pda_validate_inputs(const int32_t* block_tables, const int32_t* context_lens,
                               const pda_shape* shape, int64_t* counts, void* stream);

/* End-to-end decode step from HOST buffers: copies this step's inputs
 * (q, block_tables, context_lens; pinned host memory recommended) to the
 * device staging buffers, runs paged_decode_attention against the
 * device-resident caches, and copies out back to host -- all enqueued on
 * `stream`; the caller synchronises the stream before reading out_host.
 *   *_host   host pointers (read: q, block_tables, context_lens; written: out)
 *   *_dev    device staging buffers of the same sizes (caller-owned)
 *   k_cache, v_cache, workspace: device pointers as above. */
pda_status pda_decode_step_host(const void* q_host, const int32_t* block_tables_host,
                                const int32_t* context_lens_host, void* out_host, void* q_dev,
                                int32_t* block_tables_dev, int32_t* context_lens_dev,
                                void* out_dev, const void* k_cache, const void* v_cache,
                                float scale, const pda_shape* shape, const pda_options* opt,
                                void* workspace, size_t workspace_bytes, void* stream);

/* Pipelined form of pda_decode_step_host for back-to-back steps: the input
 * copies and the output copy run on `copy_stream`, the kernels on
 * `compute_stream`, linked by two caller-owned CUDA events (cudaEvent_t):
 *   copy_stream:    H2D q, block_tables, context_lens; record inputs_ready
 *   compute_stream: wait inputs_ready; the decode kernel(s); record step_done
 *   copy_stream:    wait step_done; D2H out
 * With one compute stream and one copy stream + staging slot + event pair per
 * in-flight step (e.g. two, used alternately), a step's copies overlap the
 * previous step's kernels while the kernels themselves stay in issue order.
 * The caller synchronises copy_stream before reading out_host and must not
 * reuse a slot's staging buffers before that slot's previous step finished
 * (issuing the slot's steps on the same copy_stream guarantees it). */
pda_status pda_decode_step_host_async(const void* q_host, const int32_t* block_tables_host,
                                      const int32_t* context_lens_host, void* out_host, void* q_dev,
                                      int32_t* block_tables_dev, int32_t* context_lens_dev, void* out_dev,
                                      const void* k_cache, const void* v_cache, float scale,
                                      const pda_shape* shape, const pda_options* opt, void* workspace,
                                      size_t workspace_bytes, void* compute_stream, void* copy_stream,
                                      void* inputs_ready, void* step_done);

/* Measurement helper (not part of the method): stream-read `bytes` of device
 * memory at `buf` with 16-byte loads on a grid of num_sms * 4 CTAs, writing a
 * checksum word to `sink` (device, 16 B).  Gives the in-run read roofline.
 * Same as pda_read_roofline_mode(buf, bytes, sink, 0, stream). */
pda_status pda_read_roofline(const void* buf, size_t bytes, void* sink, void* stream);

/* The read roofline probe with a choice of load path:
 *   mode 0  16-byte LDG (as pda_read_roofline);
 *   mode 1  1-D bulk copies (TMA engine) of 16 KiB chunks into a 12-stage
 *           shared-memory ring, one CTA per SM;
 *   mode 2  bulk copies shaped like the decode kernel's ring: 8 KiB chunks,
 *           8 stages, 3 CTAs per SM.
 * Bulk modes read floor(bytes / chunk) whole chunks.  `buf` and `sink` must
 * be 16-B aligned (PDA_ERR_ALIGN); mode outside 0..2: PDA_ERR_SHAPE. */
pda_status pda_read_roofline_mode(const void* buf, size_t bytes, void* sink, int32_t mode, void* stream);

/* Human-readable name of a status code (static string). */
const char* pda_status_string(pda_status status);

/* ABI version (bumped on any signature change). */
int32_t pda_abi_version(void);  /* 13: paged_decode_attention_timeline; 12: cluster merge (options.merge, plan.cluster); 11: pda_decode_step_host_async; 10: KV append + validate entries; 9: _gather entry; 8: q_len; 7: issue_mode; 6: e4m3 KV */

#ifdef __cplusplus
}
#endif

#endif /* PDA_H_ */
