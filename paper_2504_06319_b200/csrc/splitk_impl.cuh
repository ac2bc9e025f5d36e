// splitk_impl.cuh -- the split-K decode kernel template and its launch
// dispatch, included by the decode_splitk_m{0,1,2}.cu translation units (one
// per kernel MODE, compiled in parallel) and by decode_splitk.cu (sizes).
//
// context partitions) and its combine kernel.
//
// One CTA per unit (partition p, kv head, sequence b); grid (P_max, Hkv, B).
//  * Ring refill (S1-S3): by default each of the 4 consumer warps refills the
//    shared-memory ring stages it owns (self-issue); alternatively a producer
//    warp (warp 4) does it.  The issuer walks the unit's block-table slice
//    (S1, Alg. 1 line 3 "Lookup bt[block_idx]"), issues TMA tensor
//    loads of the K and V slabs of each 16-token block into an S-stage ring
//    (S3, "Load K Block"), and -- the paper's method, when prefetch is
//    on -- prefetches the K and V slabs of block j + d into L2 with
//    cp.async.bulk.prefetch.L2 iff j + d < e (S2, Alg. 1 lines 5-7,
//    P:132-135; V blocks likewise).
//  * 4 consumer warps take ring stages round-robin and compute, per block,
//    S^T = K Q^T for the GQA group's g heads (S4; tokens as the MMA M dim,
//    heads as N: one m16n8k16 tile covers g <= 8), the online softmax (S5),
//    and O^T += V^T P (S6), all on mma.sync tensor cores with fp32
//    accumulation.  Q stays in registers for the whole unit.
//  * Epilogue (S7): the 4 warps' (m, l, acc) are merged through shared
//    memory; a sequence with a single partition writes `out` directly,
//    otherwise the normalised partial and its log2-sum-exp either go to the
//    workspace for combine_kernel (S8, fixed partition order) or, when the
//    grid was launched as clusters of the P_max partitions of a row, stay in
//    shared memory and are merged over DSMEM by the cluster (same order).
//  * Optional fused KV append: the new tokens' K/V rows are written by the
//    warp that issues their block's load, before it does.
#include "block_math.cuh"
#pragma once
#include "kv_append.cuh"

namespace pda {

namespace {

constexpr uint32_t kFull = kFullMask;

template <int D, bool KV8>
struct Geometry {
    static constexpr int kElem = KV8 ? 1 : 2;             // bytes per K/V element (e4m3 | fp16/bf16)
    static constexpr int kSlab = kBlockSize * D * kElem;  // Eq. 1: M_block = b * d_h * T_block
    static constexpr int kStage = 2 * kSlab;              // K slab + V slab
    static constexpr int kBoxCols = 128 / kElem;          // TMA box: 16 rows x 128 bytes
    static constexpr int kChunks = kSlab / 2048;          // boxes per slab
};

template <bool BF16, int D, int NT, bool KV8, int MS = 1>
struct MathFor {
    using type = BlockMath<BF16, D, NT, false, MS>;
};
template <bool BF16, int D, int NT, int MS>
struct MathFor<BF16, D, NT, true, MS> {
    using type = BlockMathKV8<BF16, NT, MS>;
};

// Self-issue mode (always for e4m3 caches): no producer warp -- each consumer
// warp refills the ring stages it owns (4 issuers instead of 1; the 2 KiB e4m3
// slabs need twice the issue rate of the 16-bit path).
// Split (TS, 16-bit): 8 consumer warps, the two warps w and w + 4 share the
// blocks j = w (mod 4) -- with two head tiles each computes one tile; with
// one tile (D split) both compute S and P and each accumulates half of the
// output rows d of O^T.  The second warp to finish a block refills its stage.
// Less math per warp and twice the warps, at 2 CTAs/SM.
template <bool SELF, bool TS = false>
constexpr int splitk_block_threads() { return TS ? 2 * kConsumerWarps * 32 : (kConsumerWarps + (SELF ? 0 : 1)) * 32; }

// MODE: 0 = plain, 1 = debug trace (+ runtime cluster support), 2 = launched
// as clusters (merge over DSMEM).  The plain instantiation carries no cluster
// code at all (it cost 4 registers and 1-2 us on small steps).
// CTAs per SM the register budget is built for: 3 (<= 170 registers; the
// two-tile 16-bit kernel fits in 166 without spills); the 4-stage one-tile
// 16-bit ring: 4 (<= 128 registers, the planner picks it for 4 CTAs/SM);
// e4m3 with a 12-stage
// ring: blocks one at a time (no pairs), 4 CTAs per SM (16 warps, 4 x 48 KiB
// in flight) instead of 3 x 16 stages consumed in pairs; two-tile e4m3: 2
// (it would spill at 3).
// The producer-warp form (160 threads) keeps 2 CTAs/SM for two tiles (it
// would spill at 3).
template <bool KV8, int STAGES, int NT, bool SELF, bool TS = false>
constexpr int splitk_min_blocks() {
    return TS ? 2
              : KV8 ? (NT == 1 ? (STAGES == 12 ? 4 : 3) : 3)
                    : (NT == 1 ? (STAGES == 4 && SELF ? 4 : 3) : (SELF ? 3 : 2));
}

template <bool BF16, int D, int NT, int STAGES, int MODE, bool KV8, bool SELF, bool TS = false>
__global__ void __launch_bounds__(splitk_block_threads<SELF, TS>(), splitk_min_blocks<KV8, STAGES, NT, SELF, TS>())
    splitk_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                  const SplitKParams p) {
    static_assert(!TS || SELF, "split: self-issue");
    static_assert(!TS || !KV8 || NT == 1, "e4m3 split: D split only");
    constexpr bool TRACE = MODE == 1;
    const bool clustered = MODE != 0 && p.cluster > 1;
    using G = Geometry<D, KV8>;
    constexpr bool DSPLIT = TS && NT == 1;                 // D split (else head-tile split)
    constexpr bool KVS = kKvSplit && SELF && !TS;          // split K / V ring barriers
    constexpr int NTW = TS && !DSPLIT ? 1 : NT;            // head tiles per warp
    constexpr int NW = TS ? 2 * kConsumerWarps : kConsumerWarps;  // consumer warps
    using BM = typename MathFor<BF16, D, NTW, KV8, DSPLIT ? 2 : 1>::type;
    constexpr int NH = 8 * NT;  // padded heads per CTA
    constexpr int MT = D / 16;  // m-tiles of O^T

    extern __shared__ uint8_t smem_raw[];
    // 1024-B alignment for the 128-B swizzle atoms.
    uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
    uint8_t* ring = smem;
    constexpr int kRingBytes = STAGES * G::kStage;
    constexpr int kMergeAccBytes = kConsumerWarps * NH * (D + 4) * 4;
    constexpr int kClBytes = NH * D * 4 + NH * 4;  // this CTA's partial (o, lse) for the cluster merge
    constexpr int kBigBytes =
        kRingBytes > kMergeAccBytes + kClBytes ? kRingBytes : kMergeAccBytes + kClBytes;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kBigBytes);
    uint64_t* empty = full + STAGES;
    float* merge_m = reinterpret_cast<float*>(empty + STAGES);
    float* merge_l = merge_m + kConsumerWarps * NH;
    float* merge_acc = reinterpret_cast<float*>(ring);
    float* cl_o = reinterpret_cast<float*>(ring + kMergeAccBytes);  // [NH][D], after the main loop
    float* cl_lse = cl_o + NH * D;                                   // [NH]

    const int part = blockIdx.x, kvh = blockIdx.y, b = blockIdx.z;
    const int lane = threadIdx.x & 31;
    // TS: warp = block slot (mod 4), sub = which of its two warps; sub is the
    // head tile (two tiles) or the half of d (D split)
    // warp-level indices through a lane-0 shuffle: ptxas then knows they are
    // warp-uniform, and the ring-slot addresses and TMA coordinates derived
    // from them go to uniform registers without a per-load ELECT loop
    const int warp = __shfl_sync(0xffffffffu, TS ? (threadIdx.x >> 5) & (kConsumerWarps - 1) : threadIdx.x >> 5, 0);
    const int sub = __shfl_sync(0xffffffffu, TS ? threadIdx.x >> 7 : 0, 0);
    const int tile = DSPLIT ? 0 : sub;
    const int g = p.g;

    // PDL: everything this grid reads may come from the previous grid in the
    // stream (q, the tables, the appended KV): wait before the first load
    if constexpr (SELF) {
        // the tensor maps are kernel parameters (not produced by a previous
        // grid): fetch the descriptors before anything else, so the first TMA
        // issue does not wait for them
        if (threadIdx.x == 0) {
            prefetch_tmap(&tmK);
            prefetch_tmap(&tmV);
        }
    }
    pdl_wait();
    const int max_tokens = p.max_blocks * kBlockSize;
    // S1 ahead of S0: this partition's first 64 block ids are loaded alongside
    // the sequence length (its start part * P does not depend on it), so the
    // first TMA issue waits for one global round trip, not two.  Ids past the
    // unit's end are never used.
    int pre_w0 = 0, pre_w1 = 0;
    if constexpr (SELF) {
        const int sb0 = part * p.part_tokens / kBlockSize;  // < max_blocks: part < p_max
        const int32_t* bt0 = p.bt + (size_t)b * p.max_blocks + sb0;
        const int lane0 = threadIdx.x & 31, lim = p.max_blocks - sb0;
        pre_w0 = lane0 < lim ? __ldg(bt0 + lane0) : 0;
        pre_w1 = 32 + lane0 < lim ? __ldg(bt0 + 32 + lane0) : 0;
    }
    int L = __shfl_sync(0xffffffffu, p.lens[b], 0);  // (uniform, see warp above)
    // ring barriers initialised while the length is in flight (independent of it)
    // TS: the empty-barrier words are per-stage consumer counters instead
    int* done_cnt = reinterpret_cast<int*>(empty);
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);  // producer's arrive.expect_tx (+ TMA bytes)
            if constexpr (TS)
                done_cnt[s] = 0;
            else
                mbar_init(&empty[s], KVS ? 1 : 32);  // KVS: the V slab's full barrier; else every lane
                                                     // of the consuming warp releases its reads
        }
        fence_barrier_init();
    }
    L = L < max_tokens ? L : max_tokens;
    const int P = p.part_tokens;
    const int s_tok = part * P < L ? part * P : L;
    const int e_tok = (part + 1) * P < L ? (part + 1) * P : L;

    int32_t* rec = nullptr;
    uint64_t t_start = 0;
    if constexpr (TRACE) {
        rec = p.trace + ((size_t)(b * p.Hkv + kvh) * p.p_max + part) * p.trace_rec_len;
        if (threadIdx.x == 0) t_start = globaltimer_ns();
    }
    auto stamp_end = [&]() {  // timeline export (measurement only): thread 0
        if constexpr (TRACE) {
            if (p.stamps != nullptr && threadIdx.x == 0) {
                uint64_t* st = p.stamps + ((size_t)(b * p.Hkv + kvh) * p.p_max + part) * 3;
                st[0] = t_start;
                st[1] = globaltimer_ns();
                st[2] = sm_id();
            }
        }
    };

    const int n_parts = (L + P - 1) / P;

    // S8 inside a cluster (p.cluster > 1: the P_max partitions of this (seq, kv
    // head) row are one thread-block cluster): each CTA merges a slice of the
    // row's outputs from every partition's (o, lse) read over DSMEM -- the
    // same arithmetic, in the same partition order, as combine_kernel.
    auto cluster_merge = [&]() {
        cluster_sync_all();  // every partition's (o, lse) is in its shared memory
        if (threadIdx.x < NW * 32) {
            const int E = p.q_len * g * D;
            const int per = (E + p.cluster - 1) / p.cluster;
            const int e1 = (part + 1) * per < E ? (part + 1) * per : E;
            const uint32_t o_base = smem_u32(cl_o), l_base = smem_u32(cl_lse);
            for (int idx = part * per + threadIdx.x; idx < e1; idx += NW * 32) {
                const int h = idx / D, dd = idx % D;
                float M = -INFINITY;
                for (int q = 0; q < n_parts; ++q) M = fmaxf(M, ld_cluster_f32(cluster_map(l_base + h * 4, q)));
                if (M == -INFINITY) M = 0.f;  // every partition empty for this column
                float acc = 0.f, den = 0.f;
                for (int q = 0; q < n_parts; ++q) {
                    const float w = ex2(ld_cluster_f32(cluster_map(l_base + h * 4, q)) - M);
                    den += w;
                    acc += w * ld_cluster_f32(cluster_map(o_base + (h * D + dd) * 4, q));
                }
                const float inv = den > 0.f ? 1.f / den : 0.f;  // no visible token at all: zero row
                const size_t row = ((size_t)b * p.q_len + h / g) * p.Hq + kvh * g + h % g;
                store_out_peers(p.outs, row, p.Hq, D, dd, acc * inv, p.out_dtype);
            }
        }
        cluster_sync_all();  // partials stay alive until every reader is done
    };

    if (e_tok <= s_tok) {  // empty unit (S0): nothing to read
        if constexpr (TRACE) {
            if (threadIdx.x == 0) {
                rec[0] = s_tok;
                rec[1] = s_tok;
                rec[2] = 0;
                rec[3] = 0;
            }
        }
        if (clustered) {  // still merges its slice of the row
            cluster_merge();
            stamp_end();
            return;
        }
        if (part == 0 && L <= 0) {  // context_len == 0 => zero rows (reading R6), every query token
            for (int i = threadIdx.x; i < p.q_len * g * D; i += blockDim.x) {
                const int col = i / D, dd = i % D;
                const size_t row = ((size_t)b * p.q_len + col / g) * p.Hq + kvh * g + col % g;
                store_out_peers(p.outs, row, p.Hq, D, dd, 0.f, p.out_dtype);
            }
        }
        stamp_end();
        return;
    }
    const int sb = s_tok / kBlockSize;
    const int n = (e_tok + kBlockSize - 1) / kBlockSize - sb;  // blocks in this unit

    // Fused KV append: the step's new tokens in [t_new0, e_tok) are written by
    // the warp that issues the TMA load of their block, before that issue
    // (partitions are whole blocks, so no other CTA reads these slots).  All
    // lanes store, fence the generic->async proxy, __syncwarp; then lane 0
    // issues the load.
    const int first_new = L - p.q_len;
    const int t_new0 = p.app.k_new == nullptr ? e_tok : (first_new > s_tok ? first_new : s_tok);
    auto write_new = [&](int pos) {  // warp-wide: new-token rows of unit block `pos`
        const int lo = (sb + pos) * kBlockSize, hi = lo + kBlockSize;
        const int ta = t_new0 > lo ? t_new0 : lo, tb = e_tok < hi ? e_tok : hi;
        if (ta >= tb) return;
        constexpr int CH = D / 8;
        for (int c = lane; c < (tb - ta) * 2 * CH; c += 32) {
            const int t = ta + c / (2 * CH);
            append_chunk(p.app, p.bt, p.max_blocks, p.q_len, p.Hkv, D, b, t - first_new, kvh, t, (c / CH) & 1,
                         c % CH);
        }
        fence_proxy_async_global();
        __syncwarp();
    };
    // unit blocks holding new tokens: [jn0, jn1]
    const int jn0 = t_new0 < e_tok ? t_new0 / kBlockSize - sb : n;
    const int jn1 = t_new0 < e_tok ? (e_tok - 1) / kBlockSize - sb : n - 1;

    if constexpr (TRACE && SELF) {
        if (threadIdx.x == 0) {
            rec[2] = 0;
            rec[3] = 0;
        }
    }
    __syncthreads();  // the ring barriers (initialised at entry) are visible to every warp

    if (!SELF && warp == kConsumerWarps) {
        // ============================ producer warp ============================
        if (lane == 0) {
            prefetch_tmap(&tmK);
            prefetch_tmap(&tmV);
        }
        const int32_t* btrow = p.bt + (size_t)b * p.max_blocks + sb;
        const int d = p.pf_mode != kPfOff ? p.pf_dist : 0;
        const uint64_t pol_first = policy_evict_first(), pol_last = policy_evict_last();
        for (int j = jn0; j <= jn1; ++j) write_new(j);
        // block ids for 32 blocks at a time, the next chunk loaded one chunk ahead
        int cur = lane < n ? btrow[lane] : 0;
        int pfv = (d > 0 && lane + d < n) ? btrow[lane + d] : -1;
        int npf = 0;
        for (int c = 0; c < n; c += 32) {
            const int nxt = c + 32 + lane < n ? btrow[c + 32 + lane] : 0;
            const int pfn = (d > 0 && c + 32 + lane + d < n) ? btrow[c + 32 + lane + d] : -1;
            const int m = n - c < 32 ? n - c : 32;
            for (int i = 0; i < m; ++i) {
                const int j = c + i;
                const int phys = __shfl_sync(kFull, cur, i);
                const int pf = __shfl_sync(kFull, pfv, i);
                const int stage = j % STAGES;
                const uint32_t round = j / STAGES;
                if (lane == 0) {
                    if (round > 0) mbar_wait(&empty[stage], (round - 1) & 1);
                    mbar_arrive_expect_tx(&full[stage], G::kStage);
                    const int row = (phys * p.Hkv + kvh) * kBlockSize;
                    issue_kv_slabs<G::kSlab, G::kChunks, G::kBoxCols>(ring + stage * G::kStage, &tmK, &tmV,
                                                                       row, &full[stage], p.eviction, pol_first);
                    if constexpr (TRACE) rec[4 + j] = phys;
                }
                __syncwarp();
                if (pf >= 0) {  // warp-uniform: j + d < e (Alg. 1 guard)
                    const size_t off = ((size_t)pf * p.Hkv + kvh) * G::kSlab;
                    prefetch_kv_bytes<G::kSlab>(p.k, p.v, off, p.pf_mode, lane, p.eviction, pol_last);
                    if constexpr (TRACE) {
                        if (lane == 0) rec[4 + (p.trace_rec_len - 4) / 2 + npf] = pf;
                    }
                    ++npf;
                }
            }
            cur = nxt;
            pfv = pfn;
        }
        if constexpr (TRACE) {
            if (lane == 0) {
                rec[0] = s_tok;
                rec[1] = e_tok;
                rec[2] = n;
                rec[3] = npf;
            }
        }
        if (clustered) {  // the cluster barriers count every thread
            cluster_sync_all();
            cluster_sync_all();
        }
        return;
    }

    // ============================== consumer warps ==============================
    BM bm;
    if constexpr (DSPLIT) bm.i0 = sub * (MT / 2);
    bm.set_q_tokens(p.q_len, g, lane, 8 * tile);
    bm.load_q_tokens(p.q, b, kvh, p.Hq, p.q_len, g, lane, 8 * tile);
    bm.reset();
    if constexpr (SELF) {
        // A warp takes blocks in groups of PAIR (e4m3: pairs 2w, 2w+1 mod 8 with
        // one softmax update per pair; 16-bit: j = w mod 4) and refills the
        // stages it just read: it owns every stage s with (s / PAIR) % 4 == w, so
        // no empty barriers are needed and a parity wait always refers to the
        // warp's own previous fill.
        constexpr int PAIR = (KV8 && kKv8Pairs && STAGES % 8 == 0) ? 2 : 1;
        static_assert(STAGES % (PAIR * kConsumerWarps) == 0, "stages must split evenly over the warps");
        const int32_t* btrow = p.bt + (size_t)b * p.max_blocks + sb;
        const int d = p.pf_mode != kPfOff ? p.pf_dist : 0;  // <= 32 (validated)
        const uint64_t pol_first = policy_evict_first(), pol_last = policy_evict_last();
        int wbase = 0;  // block-id window [wbase, wbase + 64) of this unit, 2 ids per lane
        int w0 = pre_w0, w1 = pre_w1;  // loaded at entry (sb == part * P here: the unit is not empty)
        int npf = 0;
        auto id_at = [&](int pos) {
            const int o = pos - wbase;
            const int x = __shfl_sync(kFull, w0, o & 31), y = __shfl_sync(kFull, w1, o & 31);
            return o < 32 ? x : y;
        };
        auto issue = [&](int pos) {  // S1 + S3 (+ S2) for block `pos` of the unit, warp-wide
            while (pos >= wbase + 32) {
                w0 = w1;
                wbase += 32;
                w1 = wbase + 32 + lane < n ? btrow[wbase + 32 + lane] : 0;
            }
            const int phys = id_at(pos);
            const bool pf = d > 0 && pos + d < n;  // Alg. 1 guard against the unit end
            const int tgt = pf ? id_at(pos + d) : -1;
            const int st = pos % STAGES;
            if constexpr (kElectIssue) {  // converged warp: one elected lane issues
                mbar_arrive_expect_tx_elect(&full[st], G::kStage);
                issue_kv_slabs_elect<G::kSlab, G::kChunks, G::kBoxCols>(ring + st * G::kStage, &tmK, &tmV,
                                                                         (phys * p.Hkv + kvh) * kBlockSize,
                                                                         &full[st], p.eviction, pol_first);
                if constexpr (TRACE) {
                    if (lane == 0) rec[4 + pos] = phys;
                }
            } else if (lane == 0) {
                mbar_arrive_expect_tx(&full[st], G::kStage);
                issue_kv_slabs<G::kSlab, G::kChunks, G::kBoxCols>(ring + st * G::kStage, &tmK, &tmV,
                                                                   (phys * p.Hkv + kvh) * kBlockSize, &full[st],
                                                                   p.eviction, pol_first);
                if constexpr (TRACE) rec[4 + pos] = phys;
            }
            if (pf) {
                prefetch_kv_bytes<G::kSlab>(p.k, p.v, ((size_t)tgt * p.Hkv + kvh) * G::kSlab, p.pf_mode, lane,
                                            p.eviction, pol_last);
                if constexpr (TRACE) {
                    // every block below n - d prefetches, so issue order == block order
                    if (lane == 0) rec[4 + (p.trace_rec_len - 4) / 2 + pos] = tgt;
                }
                ++npf;
            }
        };
        // split K / V ring (KVS): the K slab of block `pos` on full[st], its V slab
        // on empty[st] (used as a second full barrier); issue_k returns the id
        auto issue_k = [&](int pos) {
            while (pos >= wbase + 32) {
                w0 = w1;
                wbase += 32;
                w1 = wbase + 32 + lane < n ? btrow[wbase + 32 + lane] : 0;
            }
            const int phys = id_at(pos);
            const bool pf = d > 0 && pos + d < n;  // Alg. 1 guard against the unit end
            const int tgt = pf ? id_at(pos + d) : -1;
            const int st = pos % STAGES;
            if (lane == 0) {
                mbar_arrive_expect_tx(&full[st], G::kSlab);
                issue_slab<G::kSlab, G::kChunks, G::kBoxCols>(ring + st * G::kStage, &tmK,
                                                              (phys * p.Hkv + kvh) * kBlockSize, &full[st],
                                                              p.eviction, pol_first);
                if constexpr (TRACE) rec[4 + pos] = phys;
            }
            if (pf) {
                prefetch_kv_bytes<G::kSlab>(p.k, p.v, ((size_t)tgt * p.Hkv + kvh) * G::kSlab, p.pf_mode, lane,
                                            p.eviction, pol_last);
                if constexpr (TRACE) {
                    if (lane == 0) rec[4 + (p.trace_rec_len - 4) / 2 + pos] = tgt;
                }
                ++npf;
            }
            return phys;
        };
        auto issue_v = [&](int pos, int phys) {
            const int st = pos % STAGES;
            if (lane == 0) {
                mbar_arrive_expect_tx(&empty[st], G::kSlab);
                issue_slab<G::kSlab, G::kChunks, G::kBoxCols>(ring + st * G::kStage + G::kSlab, &tmV,
                                                              (phys * p.Hkv + kvh) * kBlockSize, &empty[st],
                                                              p.eviction, pol_first);
            }
        };
        for (int pos = PAIR * warp; sub == 0 && pos < STAGES && pos < n; pos += PAIR * kConsumerWarps) {
            if (pos >= jn0 && pos <= jn1) write_new(pos);
            if constexpr (KVS)
                issue_v(pos, issue_k(pos));
            else
                issue(pos);
            if (PAIR == 2 && pos + 1 < n) {
                if (pos + 1 >= jn0 && pos + 1 <= jn1) write_new(pos + 1);
                if constexpr (KVS)
                    issue_v(pos + 1, issue_k(pos + 1));
                else
                    issue(pos + 1);
            }
        }
        // new-token blocks past the prologue: written now (overlapping the
        // prologue loads), ahead of their refill issue by this same warp
        for (int j = jn0 > STAGES ? jn0 : STAGES; j <= jn1; ++j)
            if ((j / PAIR) % kConsumerWarps == warp && !TS) write_new(j);  // (TS: no fused append)
        int mine = 0;
        // Software pipeline (kSwp): the scores of the warp's next block(s) are
        // computed before the softmax / PV of the current ones, so two
        // independent chains (next QK^T, current softmax -> PV) interleave in
        // the warp's instruction stream.  Needs the next block's stage to be a
        // different one from the current (ring depth >= 2 strides); one head
        // tile per warp only (the two-tile kernels would spill at 3 CTAs/SM).
        constexpr int STRIDE = PAIR * kConsumerWarps;
        constexpr bool SWP = kSwp && STAGES >= 2 * STRIDE && BM::kNT == 1;  // (two tiles: spills)
        float ca[BM::kNT][4], ca2[BM::kNT][4], cb[BM::kNT][4], cb2[BM::kNT][4];  // current block(s)
        float na[BM::kNT][4], na2[BM::kNT][4], nb[BM::kNT][4], nb2[BM::kNT][4];  // next block(s)
        auto scores = [&](int jj, float (&xa)[BM::kNT][4], float (&xa2)[BM::kNT][4], float (&xb)[BM::kNT][4],
                          float (&xb2)[BM::kNT][4]) {  // wait for block(s) jj (, jj + 1) and run QK^T
            const bool two = PAIR == 2 && jj + 1 < n;
            mbar_wait(&full[jj % STAGES], (jj / STAGES) & 1);
            bm.qk(smem_u32(ring + (jj % STAGES) * G::kStage), lane, xa, xa2);
            if (two) {
                mbar_wait(&full[(jj + 1) % STAGES], ((jj + 1) / STAGES) & 1);
                bm.qk(smem_u32(ring + ((jj + 1) % STAGES) * G::kStage), lane, xb, xb2);
            }
        };
        if constexpr (KVS) {
            for (int j = PAIR * warp; j < n; j += STRIDE) {
                const bool two = PAIR == 2 && j + 1 < n;
                const int st0 = j % STAGES, st1 = (j + 1) % STAGES;
                const uint32_t ph0 = (j / STAGES) & 1, ph1 = ((j + 1) / STAGES) & 1;
                const uint32_t kb0 = smem_u32(ring + st0 * G::kStage), kb1 = smem_u32(ring + st1 * G::kStage);
                mbar_wait(&full[st0], ph0);
                bm.qk(kb0, lane, ca, ca2);
                if (two) {
                    mbar_wait(&full[st1], ph1);
                    bm.qk(kb1, lane, cb, cb2);
                }
                // the K slabs are read (their registers fed QK^T): their stages' next
                // K loads go out now, a softmax + PV before the V loads
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                int nph0 = 0, nph1 = 0;
                if (j + STAGES < n) nph0 = issue_k(j + STAGES);
                if (two && j + 1 + STAGES < n) nph1 = issue_k(j + 1 + STAGES);
                const int v0 = L - (sb + j) * kBlockSize;  // tokens of the context from this block on
                const int val0 = v0 < kBlockSize ? v0 : kBlockSize;
                uint32_t pa[BM::kNT][2], pa_lo[BM::kNT][2];
                if constexpr (PAIR == 2) {
                    if (two) {
                        const int v1 = L - (sb + j + 1) * kBlockSize;
                        const int val1 = v1 < kBlockSize ? v1 : kBlockSize;
                        uint32_t pbb[BM::kNT][2];
                        const bool m = bm.needs_mask(v1);
                        if (m)
                            bm.template softmax2<true>(ca, ca2, cb, cb2, v0, v1, p.scale_log2, lane, pa, pbb);
                        else
                            bm.template softmax2<false>(ca, ca2, cb, cb2, v0, v1, p.scale_log2, lane, pa, pbb);
                        mbar_wait(&empty[st0], ph0);
                        mbar_wait(&empty[st1], ph1);
                        if (m) {
                            bm.template pv8<true>(kb0 + G::kSlab, val0, lane, pa);
                            bm.template pv8<true>(kb1 + G::kSlab, val1, lane, pbb);
                        } else {
                            bm.template pv8<false>(kb0 + G::kSlab, val0, lane, pa);
                            bm.template pv8<false>(kb1 + G::kSlab, val1, lane, pbb);
                        }
                    } else {
                        bm.template softmax<true>(ca, ca2, v0, p.scale_log2, lane, pa, pa_lo);
                        mbar_wait(&empty[st0], ph0);
                        bm.template pv_any<true>(kb0 + G::kSlab, val0, lane, pa, pa_lo);
                    }
                } else {
                    const bool m = bm.needs_mask(v0);
                    if (m)
                        bm.template softmax<true>(ca, ca2, v0, p.scale_log2, lane, pa, pa_lo);
                    else
                        bm.template softmax<false>(ca, ca2, v0, p.scale_log2, lane, pa, pa_lo);
                    mbar_wait(&empty[st0], ph0);
                    if (m)
                        bm.template pv_any<true>(kb0 + G::kSlab, val0, lane, pa, pa_lo);
                    else
                        bm.template pv_any<false>(kb0 + G::kSlab, val0, lane, pa, pa_lo);
                }
                mine += two ? 2 : 1;
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (j + STAGES < n) issue_v(j + STAGES, nph0);
                if (two && j + 1 + STAGES < n) issue_v(j + 1 + STAGES, nph1);
            }
        }
        if (SWP && !KVS && PAIR * warp < n) scores(PAIR * warp, ca, ca2, cb, cb2);
        for (int j = PAIR * warp; !KVS && j < n; j += STRIDE) {
            const bool two = PAIR == 2 && j + 1 < n;
            const int st0 = j % STAGES, st1 = (j + 1) % STAGES;
            if (SWP) {
                if (j + STRIDE < n) scores(j + STRIDE, na, na2, nb, nb2);
            } else {
                scores(j, ca, ca2, cb, cb2);
            }
            const uint32_t kb0 = smem_u32(ring + st0 * G::kStage), kb1 = smem_u32(ring + st1 * G::kStage);
            const int v0 = L - (sb + j) * kBlockSize;  // tokens of the context from this block on
            // masking only where a context / causal limit falls inside the block(s):
            // a warp-uniform branch, so full blocks issue no mask instructions
            if constexpr (PAIR == 2) {
                if (two) {
                    const int v1 = L - (sb + j + 1) * kBlockSize;
                    if (bm.needs_mask(v1))
                        bm.template finish2<true>(ca, ca2, cb, cb2, kb0 + G::kSlab, v0, kb1 + G::kSlab, v1,
                                                  p.scale_log2, lane);
                    else
                        bm.template finish2<false>(ca, ca2, cb, cb2, kb0 + G::kSlab, v0, kb1 + G::kSlab, v1,
                                                   p.scale_log2, lane);
                } else {
                    bm.template finish<true>(ca, ca2, kb0 + G::kSlab, v0, p.scale_log2, lane);
                }
            } else {
                if (bm.needs_mask(v0))
                    bm.template finish<true>(ca, ca2, kb0 + G::kSlab, v0, p.scale_log2, lane);
                else
                    bm.template finish<false>(ca, ca2, kb0 + G::kSlab, v0, p.scale_log2, lane);
            }
            if (SWP) {
#pragma unroll
                for (int nt = 0; nt < BM::kNT; ++nt)
#pragma unroll
                    for (int r = 0; r < 4; ++r) {
                        ca[nt][r] = na[nt][r];
                        ca2[nt][r] = na2[nt][r];
                        if constexpr (PAIR == 2) {
                            cb[nt][r] = nb[nt][r];
                            cb2[nt][r] = nb2[nt][r];
                        }
                    }
            }
            if (sub == 0) mine += two ? 2 : 1;
            // our ldmatrix reads of the stages are complete (their registers fed the
            // MMAs above); order them before the async-proxy refills
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if constexpr (TS) {
                // the second of the stage's two warps to finish refills it (the
                // count per stage alternates odd / even round by round)
                if (j + STAGES < n) {
                    __threadfence_block();
                    int old = 0;
                    if (lane == 0) old = atomicAdd(done_cnt + st0, 1);
                    old = __shfl_sync(kFull, old, 0);
                    if (old & 1) {
                        __threadfence_block();
                        issue(j + STAGES);
                        if (two && j + 1 + STAGES < n) issue(j + 1 + STAGES);  // (e4m3 pairs: st0 counts both)
                    }
                }
            } else {
                if (j + STAGES < n) issue(j + STAGES);
                if (two && j + 1 + STAGES < n) issue(j + 1 + STAGES);
            }
        }
        if constexpr (TRACE) {
            if (lane == 0) {
                atomicAdd(rec + 2, mine);
                atomicAdd(rec + 3, npf);
            }
        }
    } else {
        for (int j = warp; j < n; j += kConsumerWarps) {
            const int stage = j % STAGES;
            const uint32_t round = j / STAGES;
            mbar_wait(&full[stage], round & 1);
            const uint32_t kbase = smem_u32(ring + stage * G::kStage);
            const int vq = L - (sb + j) * kBlockSize;
            if (bm.needs_mask(vq))
                bm.template block<true>(kbase, kbase + G::kSlab, vq, p.scale_log2, lane);
            else
                bm.template block<false>(kbase, kbase + G::kSlab, vq, p.scale_log2, lane);
            mbar_arrive(&empty[stage]);  // ring slot free for the producer (32 lane arrivals)
        }
    }

    if constexpr (TRACE && SELF) {
        if (threadIdx.x == 0) {
            rec[0] = s_tok;
            rec[1] = e_tok;
        }
    }
    // the main loop is done: the next grid may start its prologue (it waits for
    // this grid's completion before reading anything)
    pdl_launch_dependents();
    // ---- S7: merge the consumer warps of this unit
    bm.reduce_l();
    const int r0 = lane >> 2;
    const int t0 = 2 * (lane & 3);
    asm volatile("bar.sync 1, %0;" ::"n"(NW * 32) : "memory");  // ring reads done
    if (lane < 4 && !(DSPLIT && sub == 1)) {  // (D split: both halves hold the same m, l)
#pragma unroll
        for (int nt = 0; nt < NTW; ++nt)
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const int h = (tile + nt) * 8 + 2 * lane + c;
                merge_m[warp * NH + h] = bm.m_run[nt][c];
                merge_l[warp * NH + h] = bm.l_run[nt][c];
            }
    }
#pragma unroll
    for (int i = 0; i < BM::MTL; ++i)
#pragma unroll
        for (int nt = 0; nt < NTW; ++nt)
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int dd = BM::dcol(i, lane, r) + 16 * bm.i0;
                const int h = (tile + nt) * 8 + t0 + (r & 1);
                merge_acc[(warp * NH + h) * (D + 4) + dd] = bm.acc[i][nt][r];
            }
    asm volatile("bar.sync 1, %0;" ::"n"(NW * 32) : "memory");

    const bool direct = n_parts == 1;
    for (int idx = threadIdx.x; idx < p.q_len * g * D; idx += NW * 32) {
        const int h = idx / D, dd = idx % D;  // h: column = (query token, head)
        float M = -INFINITY;
#pragma unroll
        for (int w = 0; w < kConsumerWarps; ++w) M = fmaxf(M, merge_m[w * NH + h]);
        if (M == -INFINITY) M = 0.f;  // column with no visible token in this unit
        float num = 0.f, den = 0.f;
#pragma unroll
        for (int w = 0; w < kConsumerWarps; ++w) {
            const float sc = ex2(merge_m[w * NH + h] - M);
            den += sc * merge_l[w * NH + h];
            num += sc * merge_acc[(w * NH + h) * (D + 4) + dd];
        }
        // den == 0: no visible token for this column in this unit (multi-token decode)
        const float o = den > 0.f ? num / den * p.out_scale : 0.f;  // v_scale for the e4m3 cache, else 1
        const size_t row = ((size_t)b * p.q_len + h / g) * p.Hq + kvh * g + h % g;
        const float lse = den > 0.f ? M + __log2f(den) : -INFINITY;
        if (clustered) {
            cl_o[h * D + dd] = o;
            if (dd == 0) cl_lse[h] = lse;
        } else if (direct) {
            store_out_peers(p.outs, row, p.Hq, D, dd, o, p.out_dtype);
        } else {
            p.ws_o[(row * p.p_max + part) * D + dd] = o;
            if (dd == 0) p.ws_lse[row * p.p_max + part] = lse;
        }
    }
    if (clustered) cluster_merge();
    stamp_end();
}

template <int D, int NT, int STAGES, bool KV8 = false>
constexpr size_t smem_bytes_for() {
    constexpr int ring = STAGES * Geometry<D, KV8>::kStage;
    constexpr int merge = kConsumerWarps * 8 * NT * (D + 4) * 4 + 8 * NT * (D + 1) * 4;  // + cluster partial
    constexpr int big = ring > merge ? ring : merge;
    return 1024 /* alignment slack */ + big + 2 * STAGES * 8 + 2 * kConsumerWarps * 8 * NT * 4;
}

template <bool BF16, int D, int NT, int STAGES, int MODE, bool KV8 = false, bool SELF = KV8, bool TS = false>
cudaError_t launch_one(const CUtensorMap& tmK, const CUtensorMap& tmV, const SplitKParams& p,
                       dim3 grid, cudaStream_t stream) {
    auto kern = splitk_kernel<BF16, D, NT, STAGES, MODE, KV8, SELF, TS>;
    constexpr size_t smem = smem_bytes_for<D, NT, STAGES, KV8>();
    static std::atomic<uint64_t> smem_set{0};
    if (cudaError_t e = ensure_smem_limit(kern, smem, smem_set); e != cudaSuccess) return e;
    if (p.cluster > 8) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
    }
    if (MODE == 2 && p.query_clusters != nullptr) {
        // planner query: how many clusters of p.cluster CTAs of this kernel can be
        // resident at once (GPC placement included -- a count of CTA slots is not
        // enough: 296 CTAs in clusters of 4 on 148 SMs at 2 CTAs/SM do not all fit)
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)p.cluster, 1, 1);
        cfg.blockDim = dim3(splitk_block_threads<SELF, TS>(), 1, 1);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = (unsigned)p.cluster;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        return cudaOccupancyMaxActiveClusters(p.query_clusters, kern, &cfg);
    }
    if (p.cluster > 1 || p.pdl) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = grid;
        cfg.blockDim = dim3(splitk_block_threads<SELF, TS>(), 1, 1);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = stream;
        cudaLaunchAttribute attr[2];
        int na = 0;
        if (p.cluster > 1) {
            // one cluster per (seq, kv head) row: its P_max partition CTAs (grid.x == P_max)
            attr[na].id = cudaLaunchAttributeClusterDimension;
            attr[na].val.clusterDim.x = (unsigned)p.cluster;
            attr[na].val.clusterDim.y = 1;
            attr[na].val.clusterDim.z = 1;
            ++na;
        }
        if (p.pdl) {
            attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            attr[na].val.programmaticStreamSerializationAllowed = 1;
            ++na;
        }
        cfg.attrs = attr;
        cfg.numAttrs = na;
        return cudaLaunchKernelEx(&cfg, kern, tmK, tmV, p);
    }
    kern<<<grid, splitk_block_threads<SELF, TS>(), smem, stream>>>(tmK, tmV, p);
    return cudaGetLastError();
}

template <bool BF16, int D, int NT, int MODE, bool SELF>
cudaError_t dispatch_stages(const CUtensorMap& tmK, const CUtensorMap& tmV, const SplitKParams& p,
                            int stages, dim3 grid, cudaStream_t s) {
    if constexpr (SELF) {
        if (p.tile_split) {
            switch (stages) {
                case 8: return launch_one<BF16, D, NT, 8, MODE, false, true, true>(tmK, tmV, p, grid, s);
                case 12: return launch_one<BF16, D, NT, 12, MODE, false, true, true>(tmK, tmV, p, grid, s);
                default: return cudaErrorInvalidValue;
            }
        }
    }
    switch (stages) {
        case 4: return launch_one<BF16, D, NT, 4, MODE, false, SELF>(tmK, tmV, p, grid, s);
        case 8: return launch_one<BF16, D, NT, 8, MODE, false, SELF>(tmK, tmV, p, grid, s);
        case 12: return launch_one<BF16, D, NT, 12, MODE, false, SELF>(tmK, tmV, p, grid, s);
        default: return cudaErrorInvalidValue;
    }
}

template <bool BF16, int NT, int MODE>
cudaError_t dispatch_stages_kv8(const CUtensorMap& tmK, const CUtensorMap& tmV, const SplitKParams& p,
                                int stages, dim3 grid, cudaStream_t s) {
    // 4 KiB stages, consumed in pairs (depth a multiple of 8) or singly (12)
    if constexpr (NT == 1) {
        if (p.tile_split) {  // D split: 8 consumer warps, two per block pair, 2 CTAs/SM
            switch (stages) {
                case 16: return launch_one<BF16, 128, 1, 16, MODE, true, true, true>(tmK, tmV, p, grid, s);
                case 24: return launch_one<BF16, 128, 1, 24, MODE, true, true, true>(tmK, tmV, p, grid, s);
                default: return cudaErrorInvalidValue;
            }
        }
    }
    switch (stages) {
        case 8: return launch_one<BF16, 128, NT, 8, MODE, true, true>(tmK, tmV, p, grid, s);
        case 12: return launch_one<BF16, 128, NT, 12, MODE, true, true>(tmK, tmV, p, grid, s);
        case 16: return launch_one<BF16, 128, NT, 16, MODE, true, true>(tmK, tmV, p, grid, s);
        case 24: return launch_one<BF16, 128, NT, 24, MODE, true, true>(tmK, tmV, p, grid, s);
        default: return cudaErrorInvalidValue;
    }
}

template <bool BF16, int MODE>
cudaError_t dispatch_kv8(const CUtensorMap& tmK, const CUtensorMap& tmV, const SplitKParams& p, int n_tiles,
                         int stages, dim3 grid, cudaStream_t s) {
    return n_tiles == 1 ? dispatch_stages_kv8<BF16, 1, MODE>(tmK, tmV, p, stages, grid, s)
                        : dispatch_stages_kv8<BF16, 2, MODE>(tmK, tmV, p, stages, grid, s);
}

template <bool BF16, int D, int MODE>
cudaError_t dispatch_nt(const CUtensorMap& tmK, const CUtensorMap& tmV, const SplitKParams& p,
                        int n_tiles, int stages, dim3 grid, cudaStream_t s, bool self_issue) {
    if (self_issue)
        return n_tiles == 1 ? dispatch_stages<BF16, D, 1, MODE, true>(tmK, tmV, p, stages, grid, s)
                            : dispatch_stages<BF16, D, 2, MODE, true>(tmK, tmV, p, stages, grid, s);
    return n_tiles == 1 ? dispatch_stages<BF16, D, 1, MODE, false>(tmK, tmV, p, stages, grid, s)
                        : dispatch_stages<BF16, D, 2, MODE, false>(tmK, tmV, p, stages, grid, s);
}

template <bool BF16, int MODE>
cudaError_t dispatch_d(const CUtensorMap& tmK, const CUtensorMap& tmV, const SplitKParams& p,
                       int head_dim, int n_tiles, int stages, dim3 grid, cudaStream_t s, bool self_issue) {
    return head_dim == 64 ? dispatch_nt<BF16, 64, MODE>(tmK, tmV, p, n_tiles, stages, grid, s, self_issue)
                          : dispatch_nt<BF16, 128, MODE>(tmK, tmV, p, n_tiles, stages, grid, s, self_issue);
}

// All launches of one MODE (0 plain, 1 trace, 2 cluster).
template <int MODE>
cudaError_t launch_splitk_mode(const CUtensorMap& tmK, const CUtensorMap& tmV, const SplitKParams& p, bool bf16,
                               int head_dim, int n_tiles, int stages, dim3 grid, cudaStream_t stream, bool kv8,
                               bool self_issue) {
    if (kv8) {
        if (head_dim != 128) return cudaErrorInvalidValue;
        return bf16 ? dispatch_kv8<true, MODE>(tmK, tmV, p, n_tiles, stages, grid, stream)
                    : dispatch_kv8<false, MODE>(tmK, tmV, p, n_tiles, stages, grid, stream);
    }
    return bf16 ? dispatch_d<true, MODE>(tmK, tmV, p, head_dim, n_tiles, stages, grid, stream, self_issue)
                : dispatch_d<false, MODE>(tmK, tmV, p, head_dim, n_tiles, stages, grid, stream, self_issue);
}

}  // namespace
}  // namespace pda
