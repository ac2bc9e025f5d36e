// decode_stream.cu -- the persistent, load-balanced decode kernel ("stream").
//
// All KV blocks of the step form one ordered item list: rows r = (b, kv
// head) in order, each row its n_b = ceil(L_b / 16) blocks.  With T items and
// NS streams, stream s owns items [s*T/NS, (s+1)*T/NS) -- every stream moves
// the same number of blocks (+-1), whatever the batch's length mix.  A
// stream is one warp that pipelines itself: a ring of S shared-memory stages
// filled by TMA (S3) from its own block-table window (S1); every time it
// finishes a block it refills that slot with the block S items ahead and,
// as the paper does (Alg. 1; V: P:118), prefetches the block d
// beyond that into L2 if it lies inside the same segment (R9).  The per-block
// math (S4-S6) is BlockMath.  A row whose blocks all fall in one stream is
// written directly (S7); otherwise each stream writes a partial (o, lse) and
// the last of the row's streams to finish (atomic ticket, self-resetting)
// merges them in stream order (S8) -- one launch per step, deterministic.
#include "block_math.cuh"

namespace pda {

namespace {

struct Cursor {
    int b, kvh, j, n, L;  // sequence, kv head, block index in row, blocks in row, context length
    long long pre;        // item index of (b, kvh=0, j=0)
};

__device__ __forceinline__ int seq_blocks(const int32_t* lens, int b, int max_tokens) {
    int L = __ldg(lens + b);
    L = L < max_tokens ? L : max_tokens;
    return L > 0 ? (L + kBlockSize - 1) / kBlockSize : 0;
}

// Advance to the first block of the next non-empty row.
__device__ __forceinline__ void next_row(Cursor& c, const int32_t* lens, int B, int Hkv,
                                         int max_tokens) {
    c.j = 0;
    if (++c.kvh < Hkv) return;
    c.kvh = 0;
    c.pre += (long long)c.n * Hkv;
    while (++c.b < B) {
        int L = __ldg(lens + c.b);
        L = L < max_tokens ? L : max_tokens;
        if (L > 0) {
            c.L = L;
            c.n = (L + kBlockSize - 1) / kBlockSize;
            return;
        }
    }
}

// Stream containing item k (the largest s with floor(s*T/NS) <= k).
__device__ __forceinline__ int stream_of(long long k, long long T, int NS) {
    return (int)(((k + 1) * NS - 1) / T);
}

__device__ __forceinline__ long long stream_start(int s, long long T, int NS) {
    return (long long)s * T / NS;
}

template <int D>
struct StreamGeometry {
    static constexpr int kSlab = kBlockSize * D * 2;
    static constexpr int kStage = 2 * kSlab;
    static constexpr int kChunks = D / 64;
};

template <bool BF16, int D, int NT, int S, int W, bool TRACE>
__global__ void __launch_bounds__(W * 32) stream_kernel(const __grid_constant__ CUtensorMap tmK,
                                                        const __grid_constant__ CUtensorMap tmV,
                                                        const StreamParams p) {
    using G = StreamGeometry<D>;
    constexpr int NH = 8 * NT;
    constexpr int MT = D / 16;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint8_t* ring = smem + warp * S * G::kStage;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + W * S * G::kStage) + warp * S;
    const int max_tokens = p.max_blocks * kBlockSize;
    const int g = p.g;

    // ---- total items T = Hkv * sum_b n_b (warp-wide, 8 sequences per lane per pass)
    long long T = 0;
    for (int base = 0; base < p.B; base += 256) {
        int part = 0;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int b = base + u * 32 + lane;
            if (b < p.B) part += seq_blocks(p.lens, b, max_tokens);
        }
        T += __reduce_add_sync(kFullMask, (unsigned)part);
    }
    T *= p.Hkv;
    const int NS = T < p.NS ? (int)T : p.NS;  // every stream non-empty
    const int sigma = blockIdx.x * W + warp;

    // context_len == 0 rows are written as zeros (reading R6) by stream b % NS_max
    for (int b = sigma; b < p.B; b += p.NS) {
        if (__ldg(p.lens + b) <= 0)
            for (int i = lane; i < p.Hq * D; i += 32)
                store_out(p.out, (size_t)b * p.Hq * D + i, 0.f, p.out_dtype);
    }
    if (sigma >= NS) return;
    const long long k0 = stream_start(sigma, T, NS), k1 = stream_start(sigma + 1, T, NS);
    const long long total = k1 - k0;

    // ---- locate item k0: sequence prefix scan
    Cursor cur{};
    {
        long long pre = 0;
        for (int base = 0;; base += 32) {
            const int b = base + lane;
            const long long items = b < p.B ? (long long)seq_blocks(p.lens, b, max_tokens) * p.Hkv : 0;
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
                cur.n = seq_blocks(p.lens, cur.b, max_tokens);
                int L = __ldg(p.lens + cur.b);
                cur.L = L < max_tokens ? L : max_tokens;
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
        for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
        fence_barrier_init();
        prefetch_tmap(&tmK);
        prefetch_tmap(&tmV);
    }
    __syncwarp();

    // ---- producer state: cursor S items ahead of the consumer, block-id window
    Cursor pc = cur;
    long long p_left = total;  // items the producer has not issued yet
    int win_b = -1, win_base = 0, w0 = 0, w1 = 0;
    const int d = p.pf_mode != kPfOff ? p.pf_dist : 0;
    const size_t slab_elems = (size_t)kBlockSize * D;
    const uint64_t pol_first = policy_evict_first(), pol_last = policy_evict_last();

    auto window_load = [&](int b, int base) {
        const int32_t* row = p.bt + (size_t)b * p.max_blocks;
        w0 = base + lane < p.max_blocks ? __ldg(row + base + lane) : 0;
        w1 = base + 32 + lane < p.max_blocks ? __ldg(row + base + 32 + lane) : 0;
        win_b = b;
        win_base = base;
    };
    auto id_at = [&](int j) {  // requires win_base <= j < win_base + 64 (uniform j)
        const int o = j - win_base;
        const int a = __shfl_sync(kFullMask, w0, o & 31);
        const int c = __shfl_sync(kFullMask, w1, o & 31);
        return o < 32 ? a : c;
    };

    auto issue = [&](long long k) {  // item k (stream-relative) at the producer cursor
        if (pc.b != win_b || pc.j < win_base) {
            window_load(pc.b, pc.j & ~31);
        } else if (pc.j >= win_base + 32) {
            w0 = w1;
            win_base += 32;
            w1 = win_base + 32 + lane < p.max_blocks
                     ? __ldg(p.bt + (size_t)pc.b * p.max_blocks + win_base + 32 + lane)
                     : 0;
        }
        const int phys = id_at(pc.j);
        const int slot = (int)(k % S);
        if (lane == 0) {
            mbar_arrive_expect_tx(&full[slot], G::kStage);
            const int row = (phys * p.Hkv + pc.kvh) * kBlockSize;
            issue_kv_slabs<D>(ring + slot * G::kStage, &tmK, &tmV, row, &full[slot], p.eviction, pol_first);
        }
        int32_t* rec = nullptr;
        if constexpr (TRACE) {
            rec = p.trace + ((size_t)pc.b * p.Hkv + pc.kvh) * p.trace_rec_len;
            if (lane == 0) {
                rec[4 + pc.j] = phys;
                atomicAdd(rec + 2, pc.j == 0 ? 2 : 1);  // the -1 fill is cancelled by block 0
                if (pc.j == 0) {
                    rec[0] = 0;
                    rec[1] = pc.L;
                    atomicAdd(rec + 3, 1);
                }
            }
        }
        // L2 prefetch of block j + d inside this segment (Alg. 1 guard, R9)
        const long long seg_end = pc.j + (p_left < (long long)(pc.n - pc.j) ? p_left : (long long)(pc.n - pc.j));
        if (d > 0 && pc.j + d < seg_end) {
            const int tgt = id_at(pc.j + d);
            const size_t off = ((size_t)tgt * p.Hkv + pc.kvh) * slab_elems;
            prefetch_kv_slabs<D>(p.k, p.v, off, p.pf_mode, lane, p.eviction, pol_last);
            if constexpr (TRACE) {
                if (lane == 0) {
                    rec[4 + (p.trace_rec_len - 4) / 2 + pc.j] = tgt;
                    atomicAdd(rec + 3, 1);
                }
            }
        }
        --p_left;
        if (++pc.j == pc.n) next_row(pc, p.lens, p.B, p.Hkv, max_tokens);
    };

    const long long first = total < S ? total : S;
    for (long long k = 0; k < first; ++k) issue(k);

    // ---- consumer
    BlockMath<BF16, D, NT> bm;
    long long left = total;
    bool seg_first = true;
    int seg_j0 = cur.j;
    bm.load_q(p.q, (size_t)cur.b * p.Hq + cur.kvh * g, g, lane);
    bm.reset();
    for (long long k = 0; k < total; ++k) {
        const int slot = (int)(k % S);
        mbar_wait(&full[slot], (uint32_t)((k / S) & 1));
        const uint32_t kbase = smem_u32(ring + slot * G::kStage);
        const int valid = min(kBlockSize, cur.L - cur.j * kBlockSize);
        bm.block(kbase, kbase + G::kSlab, valid, p.scale_log2, lane);
        if (k + S < total) {
            // the slot's generic-proxy reads are complete (their registers fed
            // the MMAs above); order them before the async-proxy refill
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            issue(k + S);
        }
        --left;
        ++cur.j;
        if (cur.j < cur.n && left > 0) continue;

        // ---- segment epilogue (S7 / S8)
        bm.reduce_l();
        const int r0 = lane >> 2, t0 = 2 * (lane & 3);
        const size_t qrow0 = (size_t)cur.b * p.Hq + cur.kvh * g;
        if (seg_j0 == 0 && cur.j == cur.n) {
            // the whole row in this stream: normalise and write out
#pragma unroll
            for (int i = 0; i < MT; ++i)
#pragma unroll
                for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                    for (int r = 0; r < 4; ++r) {
                        const int h = nt * 8 + t0 + (r & 1);
                        if (h < g)
                            store_out(p.out, (qrow0 + h) * D + i * 16 + r0 + 8 * (r >> 1),
                                      bm.acc[i][nt][r] / bm.l_run[nt][r & 1], p.out_dtype);
                    }
        } else {
            const int slotp = seg_first ? 0 : 1;
            float* o_base = p.ws_o + ((size_t)sigma * 2 + slotp) * NH * D;
            float* lse_base = p.ws_lse + ((size_t)sigma * 2 + slotp) * NH;
#pragma unroll
            for (int i = 0; i < MT; ++i)
#pragma unroll
                for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                    for (int r = 0; r < 4; ++r) {
                        const int h = nt * 8 + t0 + (r & 1);
                        o_base[h * D + i * 16 + r0 + 8 * (r >> 1)] = bm.acc[i][nt][r] / bm.l_run[nt][r & 1];
                    }
            if (lane < 4) {
#pragma unroll
                for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                    for (int c = 0; c < 2; ++c)
                        lse_base[nt * 8 + 2 * lane + c] = bm.m_run[nt][c] + __log2f(bm.l_run[nt][c]);
            }
            // ticket: the last of the row's streams merges the partials
            const long long row_start = cur.pre + (long long)cur.kvh * cur.n;
            const int s_lo = stream_of(row_start, T, NS);
            const int s_hi = stream_of(row_start + cur.n - 1, T, NS);
            __syncwarp();
            __threadfence();
            unsigned ticket = 0;
            if (lane == 0)
                ticket = atomicInc(p.tickets + (size_t)cur.b * p.Hkv + cur.kvh, (unsigned)(s_hi - s_lo));
            ticket = __shfl_sync(kFullMask, ticket, 0);
            if (ticket == (unsigned)(s_hi - s_lo)) {
                __threadfence();
                for (int h = 0; h < g; ++h) {
                    float M = -INFINITY;
                    for (int s = s_lo; s <= s_hi; ++s) {
                        const int sl = stream_start(s, T, NS) >= row_start ? 0 : 1;
                        M = fmaxf(M, __ldcg(p.ws_lse + ((size_t)s * 2 + sl) * NH + h));
                    }
                    float den = 0.f;
                    float num[D / 32];
#pragma unroll
                    for (int e = 0; e < D / 32; ++e) num[e] = 0.f;
                    for (int s = s_lo; s <= s_hi; ++s) {
                        const int sl = stream_start(s, T, NS) >= row_start ? 0 : 1;
                        const float w = ex2(__ldcg(p.ws_lse + ((size_t)s * 2 + sl) * NH + h) - M);
                        den += w;
                        const float* op = p.ws_o + (((size_t)s * 2 + sl) * NH + h) * D;
#pragma unroll
                        for (int e = 0; e < D / 32; ++e) num[e] += w * __ldcg(op + e * 32 + lane);
                    }
                    const float inv = 1.f / den;
#pragma unroll
                    for (int e = 0; e < D / 32; ++e)
                        store_out(p.out, (qrow0 + h) * D + e * 32 + lane, num[e] * inv, p.out_dtype);
                }
            }
        }
        if (left == 0) break;
        // next segment starts at the next row
        next_row(cur, p.lens, p.B, p.Hkv, max_tokens);
        seg_first = false;
        seg_j0 = 0;
        bm.load_q(p.q, (size_t)cur.b * p.Hq + cur.kvh * g, g, lane);
        bm.reset();
    }
}

template <int D, int S, int W>
constexpr size_t stream_smem_for() {
    return 1024 + (size_t)W * S * StreamGeometry<D>::kStage + (size_t)W * S * 8;
}

template <bool BF16, int D, int NT, int S, int W, bool TRACE>
cudaError_t launch_stream_one(const CUtensorMap& tmK, const CUtensorMap& tmV, const StreamParams& p,
                              int grid, cudaStream_t stream) {
    auto kern = stream_kernel<BF16, D, NT, S, W, TRACE>;
    constexpr size_t smem = stream_smem_for<D, S, W>();
    static std::atomic<uint64_t> smem_set{0};
    if (cudaError_t e = ensure_smem_limit(kern, smem, smem_set); e != cudaSuccess) return e;
    kern<<<grid, W * 32, smem, stream>>>(tmK, tmV, p);
    return cudaGetLastError();
}

template <bool BF16, int D, int NT, bool TRACE>
cudaError_t dispatch_sw(const CUtensorMap& tmK, const CUtensorMap& tmV, const StreamParams& p,
                        int stages, int warps, int grid, cudaStream_t s) {
#define PDA_STREAM_CASE(SS, WW)                                                            \
    if (stages == SS && warps == WW)                                                       \
        return launch_stream_one<BF16, D, NT, SS, WW, TRACE>(tmK, tmV, p, grid, s);
    PDA_STREAM_CASE(8, 1) PDA_STREAM_CASE(4, 2) PDA_STREAM_CASE(6, 2) PDA_STREAM_CASE(4, 4)
#undef PDA_STREAM_CASE
    return cudaErrorInvalidValue;
}

}  // namespace

bool stream_config_supported(int stages, int warps) {
    return (stages == 8 && warps == 1) || (stages == 4 && warps == 2) || (stages == 6 && warps == 2) ||
           (stages == 4 && warps == 4);
}

size_t stream_smem_bytes(int head_dim, int stages, int warps) {
    const size_t stage = (size_t)2 * kBlockSize * head_dim * 2;
    return 1024 + (size_t)warps * stages * stage + (size_t)warps * stages * 8;
}

cudaError_t launch_stream(const CUtensorMap& tmK, const CUtensorMap& tmV, const StreamParams& p,
                          bool bf16, int head_dim, int n_tiles, int stages, int warps, bool trace,
                          int grid, cudaStream_t stream) {
#define PDA_D(BB, TT)                                                                               \
    (head_dim == 64                                                                                 \
         ? (n_tiles == 1 ? dispatch_sw<BB, 64, 1, TT>(tmK, tmV, p, stages, warps, grid, stream)     \
                         : dispatch_sw<BB, 64, 2, TT>(tmK, tmV, p, stages, warps, grid, stream))    \
         : (n_tiles == 1 ? dispatch_sw<BB, 128, 1, TT>(tmK, tmV, p, stages, warps, grid, stream)    \
                         : dispatch_sw<BB, 128, 2, TT>(tmK, tmV, p, stages, warps, grid, stream)))
    if (bf16) return trace ? PDA_D(true, true) : PDA_D(true, false);
    return trace ? PDA_D(false, true) : PDA_D(false, false);
#undef PDA_D
}

}  // namespace pda
