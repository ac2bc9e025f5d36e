// decode_balanced.cu -- persistent, load-balanced split-K decode kernel.
//
// The KV blocks of the whole step are one ordered item list: rows (b, kv
// head) in order, row r holding its n_b = ceil(L_b / 16) blocks.  With T
// items and G resident CTAs (one wave), CTA c owns items
// [floor(c*T/G), floor((c+1)*T/G)) -- every CTA moves the same number of
// blocks (+-1) whatever the batch's length mix (S0).  Inside a CTA the
// split-K structure is kept: a producer warp walks the range (S1), issues
// TMA loads of each block's K and V slabs into an S-stage ring (S3) and, as
// the paper does (Alg. 1; V: P:118), prefetches the block d
// ahead into L2 when it lies in the same segment (R9, R20); four consumer
// warps take the ring stages round-robin (S4-S6, BlockMath).  The range is
// cut into segments at row boundaries; at the end of each segment the four
// warps merge through shared memory (S7): a row that lies wholly in the
// range is written to `out`, otherwise the segment's (o, lse) partial goes
// to the workspace and the last of the row's CTAs to finish (self-resetting
// atomic ticket) merges the partials in CTA order (S8).  One launch per
// step, no pipeline drain between rows, deterministic.
#include "block_math.cuh"

namespace pda {

namespace {

struct Cursor {
    int b, kvh, j, n, L;  // sequence, kv head, block in row, blocks in row, context length
    long long pre;        // item index of (b, kvh = 0, j = 0)
};

__device__ __forceinline__ int clamp_len(const int32_t* lens, int b, int max_tokens) {
    const int L = __ldg(lens + b);
    return L < max_tokens ? L : max_tokens;
}

__device__ __forceinline__ int blocks_of(int L) { return L > 0 ? (L + kBlockSize - 1) / kBlockSize : 0; }

__device__ __forceinline__ void next_row(Cursor& c, const int32_t* lens, int B, int Hkv, int max_tokens) {
    c.j = 0;
    if (++c.kvh < Hkv) return;
    c.kvh = 0;
    c.pre += (long long)c.n * Hkv;
    while (++c.b < B) {
        const int L = clamp_len(lens, c.b, max_tokens);
        if (L > 0) {
            c.L = L;
            c.n = blocks_of(L);
            return;
        }
    }
}

// CTA owning item k: the largest c with floor(c*T/G) <= k.
__device__ __forceinline__ int cta_of(long long k, long long T, int G) { return (int)(((k + 1) * G - 1) / T); }
__device__ __forceinline__ long long range_start(int c, long long T, int G) { return (long long)c * T / G; }

template <int D>
struct BGeom {
    static constexpr int kSlab = kBlockSize * D * 2;  // Eq. 1
    static constexpr int kStage = 2 * kSlab;
    static constexpr int kChunks = D / 64;
};

template <int D, int NT, int S>
struct BLayout {
    static constexpr int NH = 8 * NT;
    static constexpr int kRing = S * BGeom<D>::kStage;
    static constexpr int kPasses = 2;              // merge in column halves
    static constexpr int kDH = D / kPasses;
    static constexpr int kMergeAcc = kConsumerWarps * NH * (kDH + 4) * 4;
    static constexpr int kMergeML = 2 * kConsumerWarps * NH * 4;
    static constexpr int kBars = 2 * S * 8;
    static constexpr int kMisc = 128;  // T, range, start cursor, ticket broadcast
    static constexpr size_t kBytes = 1024 + kRing + kMergeAcc + kMergeML + kBars + kMisc;
};

template <bool BF16, int D, int NT, int S, bool TRACE>
__global__ void __launch_bounds__((kConsumerWarps + 1) * 32, NT == 1 ? 3 : 2)
    balanced_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                    const BalancedParams p) {
    using G = BGeom<D>;
    using Lay = BLayout<D, NT, S>;
    constexpr int NH = Lay::NH;
    constexpr int kThreadsC = kConsumerWarps * 32;

    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
    uint8_t* ring = smem;
    float* merge_acc = reinterpret_cast<float*>(smem + Lay::kRing);
    float* merge_m = reinterpret_cast<float*>(smem + Lay::kRing + Lay::kMergeAcc);
    float* merge_l = merge_m + kConsumerWarps * NH;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + Lay::kRing + Lay::kMergeAcc + Lay::kMergeML);
    uint64_t* empty = full + S;
    long long* misc = reinterpret_cast<long long*>(empty + S);  // [0] T, [1] k0, [2] k1, [3..] cursor

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int c = blockIdx.x;
    const int max_tokens = p.max_blocks * kBlockSize;
    const int g = p.g;

    // ---- S0 on the device: T, this CTA's range and its first item's (b, kvh, j)
    if (warp == 0) {
        long long T = 0;
        for (int base = 0; base < p.B; base += 256) {
            int part = 0;
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int b = base + u * 32 + lane;
                if (b < p.B) part += blocks_of(clamp_len(p.lens, b, max_tokens));
            }
            T += __reduce_add_sync(kFullMask, (unsigned)part);
        }
        T *= p.Hkv;
        const int Ge = T < (long long)gridDim.x ? (int)T : (int)gridDim.x;
        long long k0 = 0, k1 = 0;
        if (c < Ge) {
            k0 = range_start(c, T, Ge);
            k1 = range_start(c + 1, T, Ge);
        }
        Cursor cur{};
        if (k1 > k0) {
            long long pre = 0;
            for (int base = 0;; base += 32) {
                const int b = base + lane;
                const long long items = b < p.B ? (long long)blocks_of(clamp_len(p.lens, b, max_tokens)) * p.Hkv : 0;
                long long incl = items;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const long long y = __shfl_up_sync(kFullMask, incl, o);
                    if (lane >= o) incl += y;
                }
                const unsigned hit = __ballot_sync(kFullMask, pre + incl > k0);
                if (hit) {
                    const int src = __ffs(hit) - 1;
                    const long long before = pre + __shfl_sync(kFullMask, incl - items, src);
                    cur.b = base + src;
                    cur.L = clamp_len(p.lens, cur.b, max_tokens);
                    cur.n = blocks_of(cur.L);
                    cur.pre = before;
                    const long long off = k0 - before;
                    cur.kvh = (int)(off / cur.n);
                    cur.j = (int)(off % cur.n);
                    break;
                }
                pre += __shfl_sync(kFullMask, incl, 31);
            }
        }
        if (lane == 0) {
            misc[0] = T;
            misc[1] = k0;
            misc[2] = k1;
            misc[3] = Ge;
            misc[4] = cur.b;
            misc[5] = cur.kvh;
            misc[6] = cur.j;
            misc[7] = ((long long)cur.n << 32) | (unsigned)cur.L;
            misc[8] = cur.pre;
            for (int s = 0; s < S; ++s) {
                mbar_init(&full[s], 1);
                mbar_init(&empty[s], 32);
            }
            fence_barrier_init();
        }
    }
    __syncthreads();
    const long long T = misc[0], k0 = misc[1], k1 = misc[2];
    const int Ge = (int)misc[3];
    const long long total = k1 - k0;
    Cursor start{};
    start.b = (int)misc[4];
    start.kvh = (int)misc[5];
    start.j = (int)misc[6];
    start.n = (int)(misc[7] >> 32);
    start.L = (int)(misc[7] & 0xffffffff);
    start.pre = misc[8];

    // context_len == 0 rows: zeros (reading R6), sequences strided over the grid
    if (warp < kConsumerWarps) {
        for (int b = c; b < p.B; b += gridDim.x) {
            if (__ldg(p.lens + b) <= 0)
                for (int i = threadIdx.x; i < p.Hq * D; i += kThreadsC)
                    store_out(p.out, (size_t)b * p.Hq * D + i, 0.f, p.out_dtype);
        }
    }
    if (total <= 0) return;

    if (warp == kConsumerWarps) {
        // ================================ producer ================================
        if (lane == 0) {
            prefetch_tmap(&tmK);
            prefetch_tmap(&tmV);
        }
        Cursor pc = start;
        long long left = total;
        int win_b = -1, win_base = 0, w0 = 0, w1 = 0;
        const int d = p.pf_mode != kPfOff ? p.pf_dist : 0;
        const size_t slab_elems = (size_t)kBlockSize * D;
        const uint64_t pol_first = policy_evict_first(), pol_last = policy_evict_last();
        for (long long i = 0; i < total; ++i) {
            // block-id window: ids [win_base, win_base + 64) of row pc.b, 2 per lane
            if (pc.b != win_b || pc.j < win_base) {
                const int32_t* row = p.bt + (size_t)pc.b * p.max_blocks;
                win_base = pc.j & ~31;
                w0 = win_base + lane < p.max_blocks ? __ldg(row + win_base + lane) : 0;
                w1 = win_base + 32 + lane < p.max_blocks ? __ldg(row + win_base + 32 + lane) : 0;
                win_b = pc.b;
            } else if (pc.j >= win_base + 32) {
                w0 = w1;
                win_base += 32;
                w1 = win_base + 32 + lane < p.max_blocks
                         ? __ldg(p.bt + (size_t)pc.b * p.max_blocks + win_base + 32 + lane)
                         : 0;
            }
            const int o = pc.j - win_base;
            const int ida = __shfl_sync(kFullMask, w0, o & 31), idb = __shfl_sync(kFullMask, w1, o & 31);
            const int phys = o < 32 ? ida : idb;
            const int stage = (int)(i % S);
            const uint32_t round = (uint32_t)(i / S);
            int32_t* rec = nullptr;
            if constexpr (TRACE) rec = p.trace + ((size_t)pc.b * p.Hkv + pc.kvh) * p.trace_rec_len;
            if (lane == 0) {
                if (round > 0) mbar_wait(&empty[stage], (round - 1) & 1);
                mbar_arrive_expect_tx(&full[stage], G::kStage);
                const int rowc = (phys * p.Hkv + pc.kvh) * kBlockSize;
                issue_kv_slabs<D>(ring + stage * G::kStage, &tmK, &tmV, rowc, &full[stage], p.eviction,
                                  pol_first);
                if constexpr (TRACE) {
                    rec[4 + pc.j] = phys;
                    atomicAdd(rec + 2, pc.j == 0 ? 2 : 1);  // block 0 cancels the -1 fill
                    if (pc.j == 0) {
                        rec[0] = 0;
                        rec[1] = pc.L;
                        atomicAdd(rec + 3, 1);
                    }
                }
            }
            __syncwarp();
            // Alg. 1 guard against the segment end (R9); target from the window (d <= 32)
            const long long seg_end = pc.j + (left < (long long)(pc.n - pc.j) ? left : (long long)(pc.n - pc.j));
            if (d > 0 && pc.j + d < seg_end) {
                const int ot = pc.j + d - win_base;
                const int ta = __shfl_sync(kFullMask, w0, ot & 31), tb = __shfl_sync(kFullMask, w1, ot & 31);
                const int tgt = ot < 32 ? ta : tb;
                const size_t off = ((size_t)tgt * p.Hkv + pc.kvh) * slab_elems;
                prefetch_kv_slabs<D>(p.k, p.v, off, p.pf_mode, lane, p.eviction, pol_last);
                if constexpr (TRACE) {
                    if (lane == 0) {
                        rec[4 + (p.trace_rec_len - 4) / 2 + pc.j] = tgt;
                        atomicAdd(rec + 3, 1);
                    }
                }
            }
            --left;
            if (++pc.j == pc.n) next_row(pc, p.lens, p.B, p.Hkv, max_tokens);
        }
        return;
    }

    // ================================ consumers ================================
    BlockMath<BF16, D, NT> bm;
    Cursor cc = start;
    long long left = total;
    long long i_base = 0;
    bool seg_first = true;
    const int tid = threadIdx.x;
    const int r0 = lane >> 2, t0 = 2 * (lane & 3);
    volatile unsigned* s_ticket = reinterpret_cast<volatile unsigned*>(misc + 12);
    while (true) {
        const int seg_len = (int)(left < (long long)(cc.n - cc.j) ? left : (long long)(cc.n - cc.j));
        const int j0 = cc.j;
        const size_t qrow0 = (size_t)cc.b * p.Hq + cc.kvh * g;
        bm.load_q(p.q, qrow0, g, lane);
        bm.reset();
        long long i = i_base + ((warp - i_base % kConsumerWarps) + kConsumerWarps) % kConsumerWarps;
        for (; i < i_base + seg_len; i += kConsumerWarps) {
            const int stage = (int)(i % S);
            mbar_wait(&full[stage], (uint32_t)((i / S) & 1));
            const uint32_t kbase = smem_u32(ring + stage * G::kStage);
            const int j = j0 + (int)(i - i_base);
            const int valid = min(kBlockSize, cc.L - j * kBlockSize);
            bm.block(kbase, kbase + G::kSlab, valid, p.scale_log2, lane);
            mbar_arrive(&empty[stage]);
        }
        // ---- S7: merge the four warps' states of this segment, in kPasses
        // column slices so the merge buffer stays small (3 CTAs/SM at S = 8)
        bm.reduce_l();
        const bool full_row = (j0 == 0 && seg_len == cc.n);
        const int slot = seg_first ? 0 : 1;
#pragma unroll
        for (int pass = 0; pass < Lay::kPasses; ++pass) {
            asm volatile("bar.sync 1, %0;" ::"n"(kThreadsC) : "memory");  // merge buffer free
            if (pass == 0 && lane < 4) {
#pragma unroll
                for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                    for (int cc2 = 0; cc2 < 2; ++cc2) {
                        const int h = nt * 8 + 2 * lane + cc2;
                        merge_m[warp * NH + h] = bm.m_run[nt][cc2];
                        merge_l[warp * NH + h] = bm.l_run[nt][cc2];
                    }
            }
#pragma unroll
            for (int mi = 0; mi < D / 16; ++mi) {
                if (mi / (D / 16 / Lay::kPasses) != pass) continue;
#pragma unroll
                for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                    for (int r = 0; r < 4; ++r) {
                        const int dd = mi * 16 + r0 + 8 * (r >> 1) - pass * Lay::kDH;
                        const int h = nt * 8 + t0 + (r & 1);
                        merge_acc[(warp * NH + h) * (Lay::kDH + 4) + dd] = bm.acc[mi][nt][r];
                    }
            }
            asm volatile("bar.sync 1, %0;" ::"n"(kThreadsC) : "memory");
            for (int idx = tid; idx < g * Lay::kDH; idx += kThreadsC) {
                const int h = idx / Lay::kDH, dl = idx % Lay::kDH;
                const int dd = pass * Lay::kDH + dl;
                float M = -INFINITY;
#pragma unroll
                for (int w = 0; w < kConsumerWarps; ++w) M = fmaxf(M, merge_m[w * NH + h]);
                float num = 0.f, den = 0.f;
#pragma unroll
                for (int w = 0; w < kConsumerWarps; ++w) {
                    const float sc = ex2(merge_m[w * NH + h] - M);
                    den += sc * merge_l[w * NH + h];
                    num += sc * merge_acc[(w * NH + h) * (Lay::kDH + 4) + dl];
                }
                if (full_row) {
                    store_out(p.out, (qrow0 + h) * D + dd, num / den, p.out_dtype);
                } else {
                    p.ws_o[(((size_t)c * 2 + slot) * NH + h) * D + dd] = num / den;
                    if (dd == 0) p.ws_lse[((size_t)c * 2 + slot) * NH + h] = M + __log2f(den);
                }
            }
        }
        if (!full_row) {
            // ---- S8: ticket; the last CTA of the row merges all partials in CTA order
            const long long row_start = cc.pre + (long long)cc.kvh * cc.n;
            const int c_lo = cta_of(row_start, T, Ge), c_hi = cta_of(row_start + cc.n - 1, T, Ge);
            __threadfence();
            asm volatile("bar.sync 1, %0;" ::"n"(kThreadsC) : "memory");
            if (tid == 0)
                *s_ticket = atomicInc(p.tickets + (size_t)cc.b * p.Hkv + cc.kvh, (unsigned)(c_hi - c_lo));
            asm volatile("bar.sync 1, %0;" ::"n"(kThreadsC) : "memory");
            if (*s_ticket == (unsigned)(c_hi - c_lo)) {
                __threadfence();
                for (int idx = tid; idx < g * D; idx += kThreadsC) {
                    const int h = idx / D, dd = idx % D;
                    float M = -INFINITY;
                    for (int cx = c_lo; cx <= c_hi; ++cx) {
                        const int sl = range_start(cx, T, Ge) >= row_start ? 0 : 1;
                        M = fmaxf(M, __ldcg(p.ws_lse + ((size_t)cx * 2 + sl) * NH + h));
                    }
                    float num = 0.f, den = 0.f;
                    for (int cx = c_lo; cx <= c_hi; ++cx) {
                        const int sl = range_start(cx, T, Ge) >= row_start ? 0 : 1;
                        const float w = ex2(__ldcg(p.ws_lse + ((size_t)cx * 2 + sl) * NH + h) - M);
                        den += w;
                        num += w * __ldcg(p.ws_o + (((size_t)cx * 2 + sl) * NH + h) * D + dd);
                    }
                    store_out(p.out, (qrow0 + h) * D + dd, num / den, p.out_dtype);
                }
            }
        }
        left -= seg_len;
        i_base += seg_len;
        if (left <= 0) break;
        next_row(cc, p.lens, p.B, p.Hkv, max_tokens);
        seg_first = false;
    }
}

template <bool BF16, int D, int NT, int S, bool TRACE>
cudaError_t launch_b_one(const CUtensorMap& tmK, const CUtensorMap& tmV, const BalancedParams& p,
                         int grid, cudaStream_t stream) {
    auto kern = balanced_kernel<BF16, D, NT, S, TRACE>;
    constexpr size_t smem = BLayout<D, NT, S>::kBytes;
    static std::atomic<uint64_t> smem_set{0};
    if (cudaError_t e = ensure_smem_limit(kern, smem, smem_set); e != cudaSuccess) return e;
    kern<<<grid, (kConsumerWarps + 1) * 32, smem, stream>>>(tmK, tmV, p);
    return cudaGetLastError();
}

template <bool BF16, int D, int NT, bool TRACE>
cudaError_t dispatch_b(const CUtensorMap& tmK, const CUtensorMap& tmV, const BalancedParams& p,
                       int stages, int grid, cudaStream_t s) {
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

}  // namespace

size_t balanced_smem_bytes(int head_dim, int n_tiles, int stages) {
#define PDA_BS(DD, NN, SS) \
    if (head_dim == DD && n_tiles == NN && stages == SS) return BLayout<DD, NN, SS>::kBytes;
    PDA_BS(64, 1, 4) PDA_BS(64, 1, 8) PDA_BS(64, 1, 12) PDA_BS(64, 2, 4) PDA_BS(64, 2, 8)
    PDA_BS(64, 2, 12) PDA_BS(128, 1, 4) PDA_BS(128, 1, 8) PDA_BS(128, 1, 12) PDA_BS(128, 2, 4)
    PDA_BS(128, 2, 8) PDA_BS(128, 2, 12)
#undef PDA_BS
    return 0;
}

cudaError_t launch_balanced(const CUtensorMap& tmK, const CUtensorMap& tmV, const BalancedParams& p,
                            bool bf16, int head_dim, int n_tiles, int stages, bool trace, int grid,
                            cudaStream_t stream) {
#define PDA_BD(BB, TT)                                                                    \
    (head_dim == 64 ? (n_tiles == 1 ? dispatch_b<BB, 64, 1, TT>(tmK, tmV, p, stages, grid, stream)   \
                                    : dispatch_b<BB, 64, 2, TT>(tmK, tmV, p, stages, grid, stream))  \
                    : (n_tiles == 1 ? dispatch_b<BB, 128, 1, TT>(tmK, tmV, p, stages, grid, stream)  \
                                    : dispatch_b<BB, 128, 2, TT>(tmK, tmV, p, stages, grid, stream)))
    if (bf16) return trace ? PDA_BD(true, true) : PDA_BD(true, false);
    return trace ? PDA_BD(false, true) : PDA_BD(false, false);
#undef PDA_BD
}

}  // namespace pda
