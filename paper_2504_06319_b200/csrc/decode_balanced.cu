// decode_balanced.cu -- persistent, load-balanced split-K decode kernel.
//
// Why: HBM is shared between SMs fairly, so a decode step finishes when the
// SM with the most bytes finishes.  A split-K grid of ~256 equal CTAs on 148
// SMs leaves 40 SMs with one CTA and 108 with two; no power-
// of-two split of 128 rows gives every SM the same bytes.  Here every SM gets
// the same number of KV blocks, whatever the batch shape or length mix.
//
// S0 on the device: the KV blocks of the whole step form one ordered item
// list (rows (b, kv head) in order, row r holding n_b = ceil(L_b / 16)
// blocks).  With T items and G resident CTAs (one wave, 2 per SM), CTA c owns
// items [floor(c T / G), floor((c + 1) T / G)) -- +-1 block of every other
// CTA.  The range is cut into segments at row boundaries.
//
// Inside a CTA the split-K machinery is kept (S1-S7): four consumer warps own
// the ring stages i % 4 of the CTA's item positions i and refill them
// themselves (self-issue) -- TMA loads of each block's K and V slabs (S3),
// block ids from a 64-entry window per warp (S1), and, as the paper does
// (Alg. 1; V: P:118), the L2 prefetch of the block d ahead when it
// lies in the same segment (S2, R9, R20).  The ring runs across segment
// boundaries without draining.  At the end of a segment each warp parks its
// (m, l, acc) in a shared-memory slot and moves on; the fourth warp to park
// merges the four states (S7) -- into `out` if the segment is a whole row,
// else into the workspace as the CTA's first (slot 0) or last (slot 1)
// partial.  No CTA-wide barrier anywhere in the main loop.
//
// S8: rows split between CTAs are merged by balanced_combine_kernel (launched
// right after, programmatic dependent launch) from the partials of the CTAs
// covering the row, in CTA order -- deterministic run to run.
#include "balanced_range.cuh"
#include "block_math.cuh"

namespace pda {

namespace {

using namespace br;

template <int D>
struct BGeom {
    static constexpr int kSlab = kBlockSize * D * 2;  // Eq. 1
    static constexpr int kStage = 2 * kSlab;
};

// Per-CTA shared state written by S0 and the segment slots' bookkeeping.
struct BMisc {
    // per slot: parked[] completes when all consumer warps have parked their
    // state for the slot's current segment (the merger waits on it: acquire),
    // freed[] when the merger has read the slot out (the next users wait on it)
    uint64_t parked[2], freed[2];
    long long T, k0, k1;
    int Ge, n_segs, end_j, pad0;
    Cursor start;
    int arrive[2];          // warps parked in the slot for its current segment (elects the merger)
    long long slot_row[2];  // first output row (b * Hq + kvh * g) of the slot's segment
    int slot_kind[2];       // 0: whole row -> out, 1: partial -> workspace slot 0, 2: slot 1
};

template <int D, int NT, int S>
struct BLayout {
    static constexpr int NH = 8 * NT;
    static constexpr int kSlots = NT == 1 ? 2 : 1;  // segment states parked at once
    static constexpr int kAccStride = D + 4;        // floats per (warp, column) row: conflict-free
    static constexpr int kSlotAcc = kConsumerWarps * NH * kAccStride * 4;
    static constexpr int kSlotML = 2 * kConsumerWarps * NH * 4;
    static constexpr int kSlotBytes = kSlotAcc + kSlotML;
    static constexpr int kRing = S * BGeom<D>::kStage;
    static constexpr size_t kBytes = 1024 + kRing + kSlots * kSlotBytes + S * 8 + sizeof(BMisc) + 64;
};

template <bool BF16, int D, int NT, int S, bool TRACE>
__global__ void __launch_bounds__(kConsumerWarps * 32, NT == 1 ? 2 : 1)
    balanced_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                    const BalancedParams p) {
    static_assert(S % kConsumerWarps == 0, "every ring stage must belong to one warp");
    using G = BGeom<D>;
    using Lay = BLayout<D, NT, S>;
    constexpr int NH = Lay::NH;
    constexpr int MT = D / 16;

    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
    uint8_t* ring = smem;
    uint8_t* slots = smem + Lay::kRing;
    uint64_t* full = reinterpret_cast<uint64_t*>(slots + Lay::kSlots * Lay::kSlotBytes);
    BMisc* misc = reinterpret_cast<BMisc*>(full + S);

    // warp index through a lane-0 shuffle: warp-uniform for ptxas (the refill
    // issue then needs no per-load ELECT loop, see splitk_impl.cuh)
    const int warp = __shfl_sync(kFullMask, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
    const int c = blockIdx.x;
    const int max_tokens = p.max_blocks * kBlockSize;
    const int g = p.g;

    // PDL: q, the tables and the caches may come from the previous grid
    pdl_wait();

    // ---- S0 on the device (warp 0): T, this CTA's range, its first item's
    // cursor and the number of segments it spans (balanced_range.cuh)
    if (warp == 0) {
        const br::RangePlan rp = br::plan_range(p.lens, p.B, p.Hkv, max_tokens, c, gridDim.x, p.seq_prefix, lane);
        if (lane == 0) {
            misc->T = rp.T;
            misc->k0 = rp.k0;
            misc->k1 = rp.k1;
            misc->Ge = rp.Ge;
            misc->n_segs = rp.n_segs;
            misc->end_j = rp.end_j;
            misc->start = rp.start;
            for (int s = 0; s < 2; ++s) {
                misc->arrive[s] = 0;
                mbar_init(&misc->parked[s], kConsumerWarps * 32);  // every consumer thread
                mbar_init(&misc->freed[s], 32);                    // the merging warp's threads
            }
            for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
            fence_barrier_init();
        }
    }
    __syncthreads();
    const long long total = __shfl_sync(kFullMask, misc->k1 - misc->k0, 0);
    const int n_segs = __shfl_sync(kFullMask, misc->n_segs, 0), end_j = __shfl_sync(kFullMask, misc->end_j, 0);
    Cursor start = misc->start;
    uniform_cursor(start);

    // context_len == 0 rows: zeros (reading R6), sequences strided over the grid
    for (int b = c; b < p.B; b += gridDim.x) {
        if (__ldg(p.lens + b) <= 0)
            for (int i = threadIdx.x; i < p.Hq * D; i += kConsumerWarps * 32)
                store_out(p.out, (size_t)b * p.Hq * D + i, 0.f, p.out_dtype);
    }
    if (total <= 0) return;

    const int d = p.pf_mode != kPfOff ? p.pf_dist : 0;  // <= 32 (validated)
    const uint64_t pol_first = policy_evict_first(), pol_last = policy_evict_last();
    if (warp == 0 && lane == 0) {
        prefetch_tmap(&tmK);
        prefetch_tmap(&tmV);
    }

    // ---- issue side (S1 + S3 + S2): this warp's positions warp, warp + 4, ...
    Cursor ic = start;
    int iseg = 0;
    long long ipos = warp;
    if (ipos < total) {
        advance(ic, warp, iseg, p.lens, p.B, p.Hkv, max_tokens);
        uniform_cursor(ic);
        iseg = __shfl_sync(kFullMask, iseg, 0);
    }
    int wb = -1, wbase = 0, w0 = 0, w1 = 0;  // block-id window [wbase, wbase + 64) of sequence wb
    auto issue = [&]() {
        const int32_t* row = p.bt + (size_t)ic.b * p.max_blocks;
        if (ic.b != wb || ic.j < wbase) {
            wbase = ic.j & ~31;
            w0 = wbase + lane < p.max_blocks ? __ldg(row + wbase + lane) : 0;
            w1 = wbase + 32 + lane < p.max_blocks ? __ldg(row + wbase + 32 + lane) : 0;
            wb = ic.b;
        }
        while (ic.j >= wbase + 32) {
            w0 = w1;
            wbase += 32;
            w1 = wbase + 32 + lane < p.max_blocks ? __ldg(row + wbase + 32 + lane) : 0;
        }
        auto id_at = [&](int j) {
            const int o = j - wbase;
            const int x = __shfl_sync(kFullMask, w0, o & 31), y = __shfl_sync(kFullMask, w1, o & 31);
            return o < 32 ? x : y;
        };
        const int phys = id_at(ic.j);
        const int st = (int)(ipos % S);
        int32_t* rec = nullptr;
        if constexpr (TRACE) rec = p.trace + ((size_t)ic.b * p.Hkv + ic.kvh) * p.trace_rec_len;
        mbar_arrive_expect_tx_elect(&full[st], G::kStage);  // converged warp: one elected lane issues
        issue_kv_slabs_elect<kBlockSize * D * 2, D / 64, 64>(ring + st * G::kStage, &tmK, &tmV,
                                                             (phys * p.Hkv + ic.kvh) * kBlockSize, &full[st],
                                                             p.eviction, pol_first);
        if (lane == 0) {
            if constexpr (TRACE) {
                rec[4 + ic.j] = phys;
                atomicAdd(rec + 2, ic.j == 0 ? 2 : 1);  // block 0 cancels the -1 fill
                if (ic.j == 0) {
                    rec[0] = 0;
                    rec[1] = ic.L;
                    atomicAdd(rec + 3, 1);
                }
            }
        }
        // Alg. 1 guard against the segment end (R9): the row end, or the range end
        const int seg_end = iseg == n_segs - 1 ? end_j + 1 : ic.n;
        if (d > 0 && ic.j + d < seg_end) {
            const int tgt = id_at(ic.j + d);
            prefetch_kv_slabs<D>(p.k, p.v, ((size_t)tgt * p.Hkv + ic.kvh) * (kBlockSize * D), p.pf_mode, lane,
                                 p.eviction, pol_last);
            if constexpr (TRACE) {
                if (lane == 0) {
                    rec[4 + (p.trace_rec_len - 4) / 2 + ic.j] = tgt;
                    atomicAdd(rec + 3, 1);
                }
            }
        }
        ipos += kConsumerWarps;
        if (ipos < total) {
            advance(ic, kConsumerWarps, iseg, p.lens, p.B, p.Hkv, max_tokens);
            uniform_cursor(ic);
            iseg = __shfl_sync(kFullMask, iseg, 0);
        }
    };
    for (int k = 0; k < S / kConsumerWarps && ipos < total; ++k) issue();

    // ---- consumers (S4-S6) and the parked-state merges (S7)
    BlockMath<BF16, D, NT> bm;
    bm.set_q_tokens(1, g, lane);
    const int t0 = 2 * (lane & 3);
    int nf = 0;  // next segment this warp must park a state for (empty or not)
    // Park this warp's state for segment s (mine: it holds the segment's
    // blocks of this warp, else an empty state); the fourth warp merges.
    auto park = [&](int s, bool mine, const Cursor& row) {
        const int slot = s % Lay::kSlots;
        const int use = s / Lay::kSlots;
        if (use > 0) mbar_wait(&misc->freed[slot], (use - 1) & 1);  // the previous merge read the slot out
        float* acc_s = reinterpret_cast<float*>(slots + slot * Lay::kSlotBytes);
        float* m_s = reinterpret_cast<float*>(slots + slot * Lay::kSlotBytes + Lay::kSlotAcc);
        float* l_s = m_s + kConsumerWarps * NH;
        if (mine) {
            bm.reduce_l();
            if (lane < 4) {
#pragma unroll
                for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                    for (int cc = 0; cc < 2; ++cc) {
                        const int h = nt * 8 + 2 * lane + cc;
                        m_s[warp * NH + h] = bm.m_run[nt][cc];
                        l_s[warp * NH + h] = bm.l_run[nt][cc];
                    }
            }
#pragma unroll
            for (int i = 0; i < MT; ++i)
#pragma unroll
                for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                    for (int r = 0; r < 4; ++r) {
                        const int dd = BlockMath<BF16, D, NT>::dcol(i, lane, r);
                        const int h = nt * 8 + t0 + (r & 1);
                        acc_s[(warp * NH + h) * Lay::kAccStride + dd] = bm.acc[i][nt][r];
                    }
            if (lane == 0) {
                // whole row unless the range starts inside it (first segment) or
                // ends inside it (last segment)
                const bool whole = (s > 0 || start.j == 0) && (s < n_segs - 1 || end_j == row.n - 1);
                misc->slot_row[slot] = (long long)row.b * p.Hq + row.kvh * g;
                misc->slot_kind[slot] = whole ? 0 : (s == 0 ? 1 : 2);
            }
        } else if (lane < NH) {
            m_s[warp * NH + lane] = -INFINITY;  // no block of this segment was this warp's
            l_s[warp * NH + lane] = 0.f;
        }
        mbar_arrive(&misc->parked[slot]);  // release: this thread's slot writes
        __syncwarp();
        int last = 0;
        if (lane == 0) last = atomicAdd(&misc->arrive[slot], 1) == kConsumerWarps - 1;
        last = __shfl_sync(kFullMask, last, 0);
        if (!last) return;
        // the last warp to count itself merges; every thread arrived on
        // parked[] before its warp's atomicAdd, so this wait returns at once --
        // it is the acquire
        mbar_wait(&misc->parked[slot], use & 1);
        const long long row0 = misc->slot_row[slot];
        const int kind = misc->slot_kind[slot];
        for (int idx = lane; idx < g * D; idx += 32) {
            const int h = idx / D, dd = idx % D;
            float M = -INFINITY;
#pragma unroll
            for (int w = 0; w < kConsumerWarps; ++w) M = fmaxf(M, m_s[w * NH + h]);
            float num = 0.f, den = 0.f;
#pragma unroll
            for (int w = 0; w < kConsumerWarps; ++w) {
                const float mw = m_s[w * NH + h];
                if (mw == -INFINITY) continue;  // empty state: its acc is not written
                const float sc = ex2(mw - M);
                den += sc * l_s[w * NH + h];
                num += sc * acc_s[(w * NH + h) * Lay::kAccStride + dd];
            }
            if (kind == 0) {
                store_out(p.out, (size_t)(row0 + h) * D + dd, num / den, p.out_dtype);
            } else {
                const size_t ws = (size_t)c * 2 + (kind - 1);
                p.ws_o[(ws * NH + h) * D + dd] = num / den;
                if (dd == 0) p.ws_lse[ws * NH + h] = M + __log2f(den);
            }
        }
        __syncwarp();
        if (lane == 0) misc->arrive[slot] = 0;
        mbar_arrive(&misc->freed[slot]);  // release: this thread's reads above (lane 0: the reset)
    };

    Cursor cc = start;
    int cseg = 0;
    long long cpos = warp;
    if (cpos < total) {
        advance(cc, warp, cseg, p.lens, p.B, p.Hkv, max_tokens);
        bm.load_q(p.q, (size_t)cc.b * p.Hq + cc.kvh * g, g, lane);
        bm.reset();
    }
    while (cpos < total) {
        const int st = (int)(cpos % S);
        mbar_wait(&full[st], (uint32_t)((cpos / S) & 1));
        const uint32_t kb = smem_u32(ring + st * G::kStage);
        const int vq = cc.L - cc.j * kBlockSize;  // tokens of the context from this block on
        if (bm.needs_mask(vq))
            bm.template block<true>(kb, kb + G::kSlab, vq, p.scale_log2, lane);
        else
            bm.template block<false>(kb, kb + G::kSlab, vq, p.scale_log2, lane);
        // our ldmatrix reads of the stage are complete; order them before the refill
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (ipos < total) issue();
        cpos += kConsumerWarps;
        if (cpos < total) {
            const int before = cseg;
            const Cursor prev = cc;
            advance(cc, kConsumerWarps, cseg, p.lens, p.B, p.Hkv, max_tokens);
            if (cseg != before) {
                for (; nf < cseg; ++nf) park(nf, nf == before, prev);
                bm.load_q(p.q, (size_t)cc.b * p.Hq + cc.kvh * g, g, lane);
                bm.reset();
            }
        }
    }
    // the main loop is done: the combine grid may start its prologue
    pdl_launch_dependents();
    const bool has_state = (long long)warp < total;
    for (; nf < n_segs; ++nf) park(nf, has_state && nf == cseg, cc);
}

// S8 for rows split between CTAs: out = sum_c 2^(lse_c - M) o_c / sum_c 2^(lse_c - M),
// c over the CTAs covering the row in order.  One warp per (sequence, q head).
template <int D>
__global__ void __launch_bounds__(128) balanced_combine_kernel(const BalancedParams p, int G) {
    constexpr int PER = D / 32;
    pdl_wait();  // the partials and seq_prefix come from the main grid
    const int row = blockIdx.x * 4 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= p.B * p.Hq) return;
    const int b = row / p.Hq, h = row % p.Hq;
    const int kvh = h / p.g, hh = h % p.g;
    const int max_tokens = p.max_blocks * kBlockSize;
    const int n = blocks_of(clamp_len(p.lens, b, max_tokens));
    if (n == 0) return;
    const long long T = p.seq_prefix[p.B] * p.Hkv;
    const int Ge = T < (long long)G ? (int)T : G;
    const long long r0 = p.seq_prefix[b] * p.Hkv + (long long)kvh * n;
    const int c_lo = cta_of(r0, T, Ge), c_hi = cta_of(r0 + n - 1, T, Ge);
    if (c_lo == c_hi) return;  // written by the main kernel
    const int NH = p.g <= 8 ? 8 : 16;
    float M = -INFINITY;
    for (int cx = c_lo; cx <= c_hi; ++cx) {
        const int sl = range_start(cx, T, Ge) >= r0 ? 0 : 1;
        M = fmaxf(M, __ldcg(p.ws_lse + ((size_t)cx * 2 + sl) * NH + hh));
    }
    float accv[PER];
#pragma unroll
    for (int e = 0; e < PER; ++e) accv[e] = 0.f;
    float den = 0.f;
    for (int cx = c_lo; cx <= c_hi; ++cx) {
        const int sl = range_start(cx, T, Ge) >= r0 ? 0 : 1;
        const size_t ws = ((size_t)cx * 2 + sl) * NH + hh;
        const float w = ex2(__ldcg(p.ws_lse + ws) - M);
        den += w;
        const float* op = p.ws_o + ws * D + lane * PER;
#pragma unroll
        for (int e = 0; e < PER; ++e) accv[e] += w * __ldcg(op + e);
    }
#pragma unroll
    for (int e = 0; e < PER; ++e) store_out(p.out, (size_t)row * D + lane * PER + e, accv[e] / den, p.out_dtype);
}

template <bool BF16, int D, int NT, int S, bool TRACE>
cudaError_t launch_b_one(const CUtensorMap& tmK, const CUtensorMap& tmV, const BalancedParams& p, int grid,
                         cudaStream_t stream) {
    auto kern = balanced_kernel<BF16, D, NT, S, TRACE>;
    constexpr size_t smem = BLayout<D, NT, S>::kBytes;
    static std::atomic<uint64_t> smem_set{0};
    if (cudaError_t e = ensure_smem_limit(kern, smem, smem_set); e != cudaSuccess) return e;
    if (p.pdl) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid, 1, 1);
        cfg.blockDim = dim3(kConsumerWarps * 32, 1, 1);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        return cudaLaunchKernelEx(&cfg, kern, tmK, tmV, p);
    }
    kern<<<grid, kConsumerWarps * 32, smem, stream>>>(tmK, tmV, p);
    return cudaGetLastError();
}

template <bool BF16, int D, int NT, bool TRACE>
cudaError_t dispatch_b(const CUtensorMap& tmK, const CUtensorMap& tmV, const BalancedParams& p, int stages,
                       int grid, cudaStream_t s) {
    switch (stages) {
        // S must be a multiple of the 4 consumer warps: each ring stage then
        // always belongs to the same warp, which consumed its previous fill, so
        // the full-barrier parity wait cannot see a stale phase (TMA fills
        // complete out of order).
        case 4: return launch_b_one<BF16, D, NT, 4, TRACE>(tmK, tmV, p, grid, s);
        case 8: return launch_b_one<BF16, D, NT, 8, TRACE>(tmK, tmV, p, grid, s);
        case 12: return launch_b_one<BF16, D, NT, 12, TRACE>(tmK, tmV, p, grid, s);
        default: return cudaErrorInvalidValue;
    }
}

template <int D>
cudaError_t launch_b_combine(const BalancedParams& p, int G, cudaStream_t stream) {
    const dim3 grid((p.B * p.Hq + 3) / 4);
    if (p.pdl) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = grid;
        cfg.blockDim = dim3(128, 1, 1);
        cfg.stream = stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        return cudaLaunchKernelEx(&cfg, balanced_combine_kernel<D>, p, G);
    }
    balanced_combine_kernel<D><<<grid, 128, 0, stream>>>(p, G);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_balanced_combine(const BalancedParams& p, int grid, int head_dim, cudaStream_t stream) {
    return head_dim == 64 ? launch_b_combine<64>(p, grid, stream) : launch_b_combine<128>(p, grid, stream);
}

size_t balanced_smem_bytes(int head_dim, int n_tiles, int stages) {
#define PDA_BS(DD, NN, SS) \
    if (head_dim == DD && n_tiles == NN && stages == SS) return BLayout<DD, NN, SS>::kBytes;
    PDA_BS(64, 1, 4) PDA_BS(64, 1, 8) PDA_BS(64, 1, 12) PDA_BS(64, 2, 4) PDA_BS(64, 2, 8)
    PDA_BS(64, 2, 12) PDA_BS(128, 1, 4) PDA_BS(128, 1, 8) PDA_BS(128, 1, 12) PDA_BS(128, 2, 4)
    PDA_BS(128, 2, 8) PDA_BS(128, 2, 12)
#undef PDA_BS
    return 0;
}

cudaError_t launch_balanced(const CUtensorMap& tmK, const CUtensorMap& tmV, const BalancedParams& p, bool bf16,
                            int head_dim, int n_tiles, int stages, bool trace, int grid, cudaStream_t stream) {
#define PDA_BD(BB, TT)                                                                                     \
    (head_dim == 64 ? (n_tiles == 1 ? dispatch_b<BB, 64, 1, TT>(tmK, tmV, p, stages, grid, stream)         \
                                    : dispatch_b<BB, 64, 2, TT>(tmK, tmV, p, stages, grid, stream))        \
                    : (n_tiles == 1 ? dispatch_b<BB, 128, 1, TT>(tmK, tmV, p, stages, grid, stream)        \
                                    : dispatch_b<BB, 128, 2, TT>(tmK, tmV, p, stages, grid, stream)))
    cudaError_t e = bf16 ? (trace ? PDA_BD(true, true) : PDA_BD(true, false))
                         : (trace ? PDA_BD(false, true) : PDA_BD(false, false));
#undef PDA_BD
    if (e != cudaSuccess) return e;
    return head_dim == 64 ? launch_b_combine<64>(p, grid, stream) : launch_b_combine<128>(p, grid, stream);
}

}  // namespace pda
