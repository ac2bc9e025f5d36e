// decode_tc.cu -- the tcgen05 decode kernel (kernel = PDA_KERNEL_TC, 16-bit KV, D = 128).
//
// Why: the split-K kernel's per-block chain is ~300 warp instructions
// (ldmatrix, mma.sync, softmax, TMA issue) at ~6 cycles each, so a CTA
// streams at most ~30 GB/s and grids with one or two CTAs per SM are SM-bound
// (profiles/r02_l2res_ncu.md).  Here the contractions run on the 5th-gen
// tensor core with the accumulators in TMEM, and a tile of 128 tokens costs
// the softmax warps ~4 instructions per token:
//
//   S4  S^T[t][c] = K[t] . q_c          tcgen05.mma M=128 tokens, N=16 columns
//                                      (heads, padded), K = d in 8 steps of 16;
//                                      A = K tile [chunk][token][128 B] SW128,
//                                      B = q rows (TMA, SW128), D in TMEM
//   S5  thread t of the 4 softmax warps owns token t of the tile: reads its 16
//       scores with tcgen05.ld, p = exp2(s - m) with a running per-column
//       reference m that is raised only when a score exceeds it by more than
//       2^8 (then O and l are rescaled, exactly); P -> shared memory (bf16:
//       hi + lo terms, R19)
//   S6  O^T[d][c] += V^T[d][t] P[t][c]   tcgen05.mma per 16-token block: M=128
//                                      (d), N=32 (16 hi + 16 lo columns),
//                                      A = the block's V slab (MN-major SW128,
//                                      the TMA box as landed), B = P (MN-major
//                                      core matrices); O^T accumulates in TMEM
//
// Work split (S0) as the balanced kernel: one persistent CTA per SM, each
// owning an equal range of the step's KV blocks (balanced_range.cuh), cut into
// segments at row boundaries; split rows are merged by the balanced combine
// kernel (S8).  Roles: warps 0-3 softmax + epilogue (thread = token / d row),
// warp 4 TMA producer (q, K, V of each tile into a 3-stage ring), warp 5 MMA
// issuer (one thread) and TMEM owner.  mbarriers connect the roles; TMEM holds
// two S buffers and two O buffers (segment parity) so that QK^T of tile i+1,
// the softmax of tile i and PV of tile i-1 overlap.
#include "balanced_range.cuh"
#include "block_math.cuh"
#include "tc_ptx.cuh"

namespace pda {

namespace {

using namespace br;

#ifndef PDA_TC_M
#define PDA_TC_M 128  // tokens per tile = UMMA M of QK^T (64 or 128)
#endif
constexpr int kTcTile = PDA_TC_M;                 // tokens per tile = UMMA M of QK^T
constexpr int kTcBlocks = kTcTile / kBlockSize;  // 16-token blocks per tile
#ifndef PDA_TC_STAGES
#define PDA_TC_STAGES (PDA_TC_M == 64 ? 6 : 3)
#endif
#ifndef PDA_TC_HINT
#define PDA_TC_HINT 1
#endif
#ifndef PDA_TC_K4D
#define PDA_TC_K4D 1  // K block = one 4-D box [half][chunk][8 rows][128 B] (else two 2-D boxes)
#endif
#ifndef PDA_TC_PAR
#define PDA_TC_PAR 1  // lane b of the producer warp issues block b's loads (else lane 0 all)
#endif
constexpr int kTcStages = PDA_TC_STAGES;
constexpr int kTcNQ = 16;  // q rows per tile (the GQA group, padded; UMMA N of QK^T)
constexpr int kTcSoftWarps = 4;
constexpr int kTcThreads = (kTcSoftWarps + 2) * 32;
// K tile: K4D [block][8-row half][chunk][8 rows][128 B] (8-row groups of a
// chunk 2048 B apart), else [chunk][tile tokens][128 B] (groups 1024 B apart)
constexpr int kTcKBytes = 2 * kTcTile * 128;
constexpr int kTcKChunk = PDA_TC_K4D ? 1024 : kTcTile * 128;  // chunk 1 offset
constexpr int kTcKSbo = PDA_TC_K4D ? 2048 : 1024;
constexpr int kTcVBytes = kTcBlocks * 4096;        // one slab [chunk][16 tokens][128 B] per block
constexpr int kTcQBytes = 2 * kTcNQ * 128;         // [chunk][16 rows][128 B]
constexpr int kTcStageBytes = kTcKBytes + kTcVBytes + kTcQBytes;
constexpr int kTcPBytes = kTcTile * 32 * 2;        // one P buffer: tile tokens x (16 hi + 16 lo) columns
constexpr int kTcPSbo = (kTcTile / 8) * 128;       // P core-matrix stride between 8-column groups
constexpr uint32_t kTcTmemCols = 128;              // S0 [0,16) S1 [16,32) O0 [32,64) O1 [64,96)
constexpr float kTcRescaleLog2 = 8.f;              // raise m only past m + 8 (p <= 256)

struct TcTileInfo {
    int b, kvh, j0, nblk, L, flags;  // flags: 1 first tile of its segment, 2 last, kind << 2, seg << 4
};

struct TcShared {
    uint64_t full[kTcStages], empty[kTcStages];
    uint64_t s_full[2], s_free[2], p_full[2], p_free[2], o_full[2], o_free[2];
    TcTileInfo info[kTcStages];
    uint32_t tmem;
    int n_tiles;
    long long k0, k1;
    int n_segs, end_j;
    Cursor start;
    int vote[2][kTcSoftWarps];
    float tmax[2][kTcSoftWarps][kTcNQ];
    float lsum[kTcSoftWarps][kTcNQ];
};

constexpr size_t kTcSmemBytes = 1024 + kTcStages * kTcStageBytes + 2 * kTcPBytes + sizeof(TcShared) + 64;

// float -> uint key whose unsigned order is the float order (for redux.max)
__device__ __forceinline__ uint32_t fkey(float x) {
    const uint32_t u = __float_as_uint(x);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float fkey_inv(uint32_t k) {
    return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

__device__ __forceinline__ int tc_kind(int seg, int n_segs, int end_j, int row_n, bool starts_row) {
    // whole row unless the range starts inside it (first segment) or ends inside it (last segment)
    const bool whole = (seg > 0 || starts_row) && (seg < n_segs - 1 || end_j == row_n - 1);
    return whole ? 0 : (seg == 0 ? 1 : 2);
}

template <bool BF16>
__global__ void __launch_bounds__(kTcThreads, 1)
    tc_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
              const __grid_constant__ CUtensorMap tmQ, const BalancedParams p) {
    constexpr int NP = BF16 ? 32 : 16;  // P columns: hi (+ lo)
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
    uint8_t* stages = smem;
    uint8_t* pbuf = smem + kTcStages * kTcStageBytes;
    TcShared* sh = reinterpret_cast<TcShared*>(pbuf + 2 * kTcPBytes);  // P double-buffered by tile parity
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int c = blockIdx.x;
    const int max_tokens = p.max_blocks * kBlockSize;
    const int g = p.g;

    pdl_wait();  // q, tables, caches may come from the previous grid

    // ---- S0 (warp 0): this CTA's range, its segments and tiles
    if (warp == 0) {
        const RangePlan rp = plan_range(p.lens, p.B, p.Hkv, max_tokens, c, gridDim.x, p.seq_prefix, lane);
        int n_tiles = 0;
        if (rp.k1 > rp.k0) {
            Cursor e = rp.start;
            long long rem = rp.k1 - rp.k0;
            for (int s = 0; rem > 0; ++s) {
                const int jend = s == rp.n_segs - 1 ? rp.end_j : e.n - 1;
                const int len = jend - e.j + 1;
                n_tiles += (len + kTcBlocks - 1) / kTcBlocks;
                rem -= len;
                if (rem > 0) next_row(e, p.lens, p.B, p.Hkv, max_tokens);
            }
        }
        if (lane == 0) {
            sh->n_tiles = n_tiles;
            sh->k0 = rp.k0;
            sh->k1 = rp.k1;
            sh->n_segs = rp.n_segs;
            sh->end_j = rp.end_j;
            sh->start = rp.start;
            for (int s = 0; s < kTcStages; ++s) {
                mbar_init(&sh->full[s], 1);
                mbar_init(&sh->empty[s], 1);
            }
            for (int s = 0; s < 2; ++s) {
                mbar_init(&sh->s_full[s], 1);
                mbar_init(&sh->s_free[s], kTcSoftWarps);
                mbar_init(&sh->o_full[s], 1);
                mbar_init(&sh->o_free[s], kTcSoftWarps);
                mbar_init(&sh->p_full[s], kTcSoftWarps);
                mbar_init(&sh->p_free[s], 1);
            }
            fence_barrier_init();
        }
    }
    if (warp == kTcSoftWarps + 1) tc::alloc<kTcTmemCols>(&sh->tmem);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const int n_tiles = sh->n_tiles;
    const uint32_t tm = sh->tmem;

    // context_len == 0 rows: zeros (reading R6), sequences strided over the grid
    if (warp < kTcSoftWarps)
        for (int b = c; b < p.B; b += gridDim.x)
            if (__ldg(p.lens + b) <= 0)
                for (int i = threadIdx.x; i < p.Hq * 128; i += kTcSoftWarps * 32)
                    store_out(p.out, (size_t)b * p.Hq * 128 + i, 0.f, p.out_dtype);

    if (warp == kTcSoftWarps) {
        // ============================ TMA producer ============================
        if (lane == 0) {
            prefetch_tmap(&tmK);
            prefetch_tmap(&tmV);
            prefetch_tmap(&tmQ);
        }
        const uint64_t pol_first = policy_evict_first();
        Cursor cur = sh->start;
        const int n_segs = sh->n_segs, end_j = sh->end_j;
        const bool starts_row = cur.j == 0;
        int tile = 0;
        int wrow = -1, wbase = 0, w0 = 0;  // 32 block ids [wbase, wbase + 32) of row wrow
        for (int seg = 0; tile < n_tiles; ++seg) {
            const int jend = seg == n_segs - 1 ? end_j : cur.n - 1;
            const int kind = tc_kind(seg, n_segs, end_j, cur.n, starts_row);
            const int32_t* btrow = p.bt + (size_t)cur.b * p.max_blocks;
            for (int j = cur.j; j <= jend; j += kTcBlocks, ++tile) {
                const int nblk = jend - j + 1 < kTcBlocks ? jend - j + 1 : kTcBlocks;
                if (cur.b != wrow || j < wbase || j + nblk > wbase + 32) {  // refill the id window
                    wrow = cur.b;
                    wbase = j;
                    w0 = wbase + lane < p.max_blocks ? __ldg(btrow + wbase + lane) : 0;
                }
                const int st = tile % kTcStages;
                if (tile >= kTcStages) mbar_wait(&sh->empty[st], ((tile / kTcStages) - 1) & 1);
                uint8_t* sb = stages + st * kTcStageBytes;
                if (lane == 0) {
                    TcTileInfo& in = sh->info[st];
                    in.b = cur.b;
                    in.kvh = cur.kvh;
                    in.j0 = j;
                    in.nblk = nblk;
                    in.L = cur.L;
                    in.flags = (j == cur.j ? 1 : 0) | (j + kTcBlocks > jend ? 2 : 0) | (kind << 2) | (seg << 4);
                    mbar_arrive_expect_tx(&sh->full[st], kTcQBytes + nblk * 8192);
                    tma_load_3d(sb + kTcKBytes + kTcVBytes, &tmQ, 0, cur.b * p.Hq + cur.kvh * g, 0, &sh->full[st]);
                }
                __syncwarp();  // lane 0's expect_tx precedes every lane's copies
                auto issue_block = [&](int blk, int phys) {
                    const int row = (phys * p.Hkv + cur.kvh) * kBlockSize;
                    uint64_t* bar = &sh->full[st];
                    if (PDA_TC_K4D) {
                        if (PDA_TC_HINT)
                            tma_load_4d_hint(sb + blk * 4096, &tmK, 0, 0, 0, row >> 3, bar, pol_first);
                        else
                            tma_load_4d(sb + blk * 4096, &tmK, 0, 0, 0, row >> 3, bar);
                    } else if (PDA_TC_HINT) {
                        tma_load_2d_hint(sb + blk * 2048, &tmK, 0, row, bar, pol_first);
                        tma_load_2d_hint(sb + kTcTile * 128 + blk * 2048, &tmK, 64, row, bar, pol_first);
                    } else {
                        tma_load_2d(sb + blk * 2048, &tmK, 0, row, bar);
                        tma_load_2d(sb + kTcTile * 128 + blk * 2048, &tmK, 64, row, bar);
                    }
                    if (PDA_TC_HINT)
                        tma_load_3d_hint(sb + kTcKBytes + blk * 4096, &tmV, 0, row, 0, bar, pol_first);
                    else
                        tma_load_3d(sb + kTcKBytes + blk * 4096, &tmV, 0, row, 0, bar);
                };
                if (PDA_TC_PAR) {
                    const int phys = __shfl_sync(kAllLanes, w0, (j - wbase + lane) & 31);
                    if (lane < nblk) issue_block(lane, phys);
                } else {
                    for (int blk = 0; blk < nblk; ++blk) {
                        const int phys = __shfl_sync(kAllLanes, w0, j - wbase + blk);
                        if (lane == 0) issue_block(blk, phys);
                    }
                }
            }
            if (tile < n_tiles) next_row(cur, p.lens, p.B, p.Hkv, max_tokens);
        }
    } else if (warp == kTcSoftWarps + 1) {
        // ============================ MMA issuer ============================
        if (lane == 0) {
            const uint32_t idq = tc::idesc_f16(BF16, kTcTile, kTcNQ, false, false);
            const uint32_t idp = tc::idesc_f16(BF16, 128, NP, true, true);
            const uint32_t pb = smem_u32(pbuf);
            auto pv = [&](int j) {
                const int st = j % kTcStages;
                const TcTileInfo in = sh->info[st];
                mbar_wait(&sh->p_full[j & 1], (j >> 1) & 1);
                tc::fence_after();
                const int seg = in.flags >> 4, ob = seg & 1;
                const bool first = in.flags & 1;
                if (first && seg >= 2) {
                    mbar_wait(&sh->o_free[ob], ((seg >> 1) - 1) & 1);
                    tc::fence_after();
                }
                const uint32_t vb = smem_u32(stages + st * kTcStageBytes + kTcKBytes);
                for (int blk = 0; blk < in.nblk; ++blk) {
                    const uint64_t a = tc::smem_desc(vb + blk * 4096, 2048, 1024, tc::kLayoutSw128);
                    const uint64_t bd = tc::smem_desc(pb + (j & 1) * kTcPBytes + blk * 256, 128, kTcPSbo,
                                                      tc::kLayoutInterleave);
                    tc::mma_f16_ss(tm + 32 + 32 * ob, a, bd, idp, !(first && blk == 0));
                }
                tc::commit(&sh->p_free[j & 1]);
                tc::commit(&sh->empty[st]);
                if (in.flags & 2) tc::commit(&sh->o_full[ob]);
            };
            for (int i = 0; i < n_tiles; ++i) {
                const int st = i % kTcStages, sb = i & 1;
                mbar_wait(&sh->full[st], (i / kTcStages) & 1);
                if (i >= 2) mbar_wait(&sh->s_free[sb], ((i >> 1) - 1) & 1);
                tc::fence_after();
                const uint32_t kb = smem_u32(stages + st * kTcStageBytes);
                const uint32_t qb = kb + kTcKBytes + kTcVBytes;
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint64_t a = tc::smem_desc(kb + (kk >> 2) * kTcKChunk + (kk & 3) * 32, 16, kTcKSbo,
                                                     tc::kLayoutSw128);
                    const uint64_t bd = tc::smem_desc(qb + (kk >> 2) * (kTcNQ * 128) + (kk & 3) * 32, 16, 1024,
                                                      tc::kLayoutSw128);
                    tc::mma_f16_ss(tm + 16 * sb, a, bd, idq, kk > 0);
                }
                tc::commit(&sh->s_full[sb]);
                if (i >= 1) pv(i - 1);
            }
            if (n_tiles > 0) pv(n_tiles - 1);
        }
        __syncwarp();
    } else {
        // ===================== softmax + epilogue (thread = token / d row) =====================
        // the S^T row (token) of this thread: M = 128 -> TMEM lane = row; M = 64 ->
        // rows 16w..16w+15 in lanes 0-15 of warp w's quarter (lanes 16-31 unused)
        const bool mine = kTcTile == 128 || lane < 16;
        const int t = kTcTile == 128 ? threadIdx.x : warp * 16 + (lane & 15);  // token of the tile
        const int t_d = threadIdx.x;                                          // d row of O^T
        const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
        float m_ref[kTcNQ], l[kTcNQ];
        const float scale_log2 = p.scale_log2;
        for (int i = 0; i < n_tiles; ++i) {
            const int st = i % kTcStages, sb = i & 1;
            mbar_wait(&sh->full[st], (i / kTcStages) & 1);  // acquire the producer's tile info
            const TcTileInfo in = sh->info[st];
            mbar_wait(&sh->s_full[sb], (i >> 1) & 1);
            tc::fence_after();
            uint32_t r[16];
            tc::ld_32x32b_x16(tm + lane_base + 16 * sb, r);
            tc::wait_ld();
            tc::fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&sh->s_free[sb]);
            const bool first = in.flags & 1;
            if (first) {
#pragma unroll
                for (int cc = 0; cc < kTcNQ; ++cc) {
                    m_ref[cc] = -INFINITY;
                    l[cc] = 0.f;
                }
            }
            const bool valid = mine && t < in.nblk * kBlockSize && in.j0 * kBlockSize + t < in.L;
            float s[kTcNQ];
            bool need = false;
#pragma unroll
            for (int cc = 0; cc < kTcNQ; ++cc) {
                // select, never arithmetic: rows of unloaded / past-the-end tokens may hold NaN
                s[cc] = valid ? __uint_as_float(r[cc]) * scale_log2 : -INFINITY;
                need |= s[cc] > m_ref[cc] + kTcRescaleLog2;
            }
            // every softmax warp must agree on m: one vote per tile
            const bool wneed = __any_sync(kAllLanes, need);
            if (lane == 0) sh->vote[i & 1][warp] = wneed;
            asm volatile("bar.sync 1, %0;" ::"n"(kTcSoftWarps * 32) : "memory");
            bool any = false;
#pragma unroll
            for (int w = 0; w < kTcSoftWarps; ++w) any |= sh->vote[i & 1][w] != 0;
            bool rescale_o = false;
            float alpha[kTcNQ];
            if (any) {
                // the tile's exact max per column; m = max(m, tile max)
#pragma unroll
                for (int cc = 0; cc < kTcNQ; ++cc) {
                    const uint32_t k = __reduce_max_sync(kAllLanes, fkey(s[cc]));
                    if (lane == cc) sh->tmax[i & 1][warp][cc] = fkey_inv(k);
                }
                asm volatile("bar.sync 1, %0;" ::"n"(kTcSoftWarps * 32) : "memory");
#pragma unroll
                for (int cc = 0; cc < kTcNQ; ++cc) {
                    float mx = m_ref[cc];
#pragma unroll
                    for (int w = 0; w < kTcSoftWarps; ++w) mx = fmaxf(mx, sh->tmax[i & 1][w][cc]);
                    alpha[cc] = m_ref[cc] == -INFINITY ? 0.f : ex2(m_ref[cc] - mx);
                    rescale_o |= alpha[cc] != 1.f;
                    l[cc] *= alpha[cc];
                    m_ref[cc] = mx;
                }
                rescale_o &= !first;
            }
            // P buffer i & 1 is free once PV(i - 2) completed; rescaling O^T
            // needs every PV issued so far complete (PV(i - 1) too)
            if (i >= 2) mbar_wait(&sh->p_free[i & 1], ((i >> 1) - 1) & 1);
            const int ob = (in.flags >> 4) & 1;
            if (rescale_o) {
                mbar_wait(&sh->p_free[(i - 1) & 1], ((i - 1) >> 1) & 1);
                tc::fence_after();
#pragma unroll
                for (int h = 0; h < NP / 16; ++h) {
                    uint32_t o[16];
                    const uint32_t oa = tm + lane_base + 32 + 32 * ob + 16 * h;
                    tc::ld_32x32b_x16(oa, o);
                    tc::wait_ld();
#pragma unroll
                    for (int cc = 0; cc < 16; ++cc) o[cc] = __float_as_uint(__uint_as_float(o[cc]) * alpha[cc]);
                    tc::st_32x32b_x16(oa, o);
                }
                tc::wait_st();
            }
            // P row t: hi (and lo) terms, MN-major core matrices (8 tokens x 16 B)
            uint32_t hi[kTcNQ / 2], lo[kTcNQ / 2];
#pragma unroll
            for (int cc = 0; cc < kTcNQ; cc += 2) {
                const float p0 = ex2(s[cc] - m_ref[cc]), p1 = ex2(s[cc + 1] - m_ref[cc + 1]);
                l[cc] += p0;
                l[cc + 1] += p1;
                const uint32_t w = pack2<BF16>(p0, p1);
                hi[cc / 2] = w;
                if constexpr (BF16) {
                    const float2 hf = unpack2<true>(w);
                    lo[cc / 2] = pack2<true>(p0 - hf.x, p1 - hf.y);
                }
            }
            uint8_t* prow = pbuf + (i & 1) * kTcPBytes + (t & 7) * 16 + (t >> 3) * 128;
            if (mine) {
                *reinterpret_cast<uint4*>(prow) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
                *reinterpret_cast<uint4*>(prow + kTcPSbo) = make_uint4(hi[4], hi[5], hi[6], hi[7]);
                if constexpr (BF16) {
                    *reinterpret_cast<uint4*>(prow + 2 * kTcPSbo) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
                    *reinterpret_cast<uint4*>(prow + 3 * kTcPSbo) = make_uint4(lo[4], lo[5], lo[6], lo[7]);
                }
            }
            if (mine && !valid && t < in.nblk * kBlockSize) {
                // a loaded token past the context end: zero its V row (0 * NaN would poison PV)
                uint8_t* vrow = stages + st * kTcStageBytes + kTcKBytes + (t >> 4) * 4096 + (t & 15) * 128;
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    *reinterpret_cast<uint4*>(vrow + u * 16) = make_uint4(0, 0, 0, 0);
                    *reinterpret_cast<uint4*>(vrow + 2048 + u * 16) = make_uint4(0, 0, 0, 0);
                }
            }
            tc::fence_async_smem();
            tc::fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&sh->p_full[i & 1]);

            if (in.flags & 2) {
                // ---- S7: the segment's output (whole row) or partial (split row)
#pragma unroll
                for (int cc = 0; cc < kTcNQ; ++cc) {
                    float v = l[cc];
#pragma unroll
                    for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(kAllLanes, v, o);
                    if (lane == cc) sh->lsum[warp][cc] = v;
                }
                asm volatile("bar.sync 1, %0;" ::"n"(kTcSoftWarps * 32) : "memory");
                float Lsum[kTcNQ];
#pragma unroll
                for (int cc = 0; cc < kTcNQ; ++cc) {
                    Lsum[cc] = 0.f;
#pragma unroll
                    for (int w = 0; w < kTcSoftWarps; ++w) Lsum[cc] += sh->lsum[w][cc];
                }
                const int seg = in.flags >> 4;
                mbar_wait(&sh->o_full[ob], (seg >> 1) & 1);
                tc::fence_after();
                uint32_t oh[16], ol[16];
                tc::ld_32x32b_x16(tm + lane_base + 32 + 32 * ob, oh);
                if constexpr (BF16) tc::ld_32x32b_x16(tm + lane_base + 32 + 32 * ob + 16, ol);
                tc::wait_ld();
                tc::fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&sh->o_free[ob]);
                const int kind = (in.flags >> 2) & 3;
                const int NH = g <= 8 ? 8 : 16;
                const int d = t_d;
#pragma unroll
                for (int cc = 0; cc < kTcNQ; ++cc) {
                    if (cc >= g) break;
                    float o = __uint_as_float(oh[cc]);
                    if constexpr (BF16) o += __uint_as_float(ol[cc]);
                    o = o / Lsum[cc];
                    if (kind == 0) {
                        store_out(p.out, ((size_t)in.b * p.Hq + in.kvh * g + cc) * 128 + d, o, p.out_dtype);
                    } else {
                        const size_t ws = (size_t)c * 2 + (kind - 1);
                        p.ws_o[(ws * NH + cc) * 128 + d] = o;
                        if (d == 0) p.ws_lse[ws * NH + cc] = m_ref[cc] + __log2f(Lsum[cc]);
                    }
                }
            }
        }
    }
    // the main loop is done: the combine grid may start its prologue
    pdl_launch_dependents();
    tc::fence_before();
    __syncthreads();
    if (warp == kTcSoftWarps + 1) tc::dealloc<kTcTmemCols>(tm);
}

template <bool BF16>
cudaError_t launch_tc_one(const CUtensorMap& tmK, const CUtensorMap& tmV, const CUtensorMap& tmQ,
                          const BalancedParams& p, int grid, cudaStream_t stream) {
    auto kern = tc_kernel<BF16>;
    static std::atomic<uint64_t> smem_set{0};
    if (cudaError_t e = ensure_smem_limit(kern, kTcSmemBytes, smem_set); e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid, 1, 1);
    cfg.blockDim = dim3(kTcThreads, 1, 1);
    cfg.dynamicSmemBytes = kTcSmemBytes;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = p.pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, tmK, tmV, tmQ, p);
}

}  // namespace

size_t tc_smem_bytes() { return kTcSmemBytes; }
bool tc_k4d() { return PDA_TC_K4D != 0; }
int tc_threads() { return kTcThreads; }

cudaError_t launch_tc(const CUtensorMap& tmK, const CUtensorMap& tmV, const CUtensorMap& tmQ,
                      const BalancedParams& p, bool bf16, int grid, cudaStream_t stream) {
    cudaError_t e = bf16 ? launch_tc_one<true>(tmK, tmV, tmQ, p, grid, stream)
                         : launch_tc_one<false>(tmK, tmV, tmQ, p, grid, stream);
    if (e != cudaSuccess) return e;
    return launch_balanced_combine(p, grid, 128, stream);
}

}  // namespace pda
