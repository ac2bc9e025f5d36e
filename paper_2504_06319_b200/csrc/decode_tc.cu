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

constexpr int kTcTile = 128;                      // tokens per tile = UMMA M of QK^T (thread = token)
constexpr int kTcBlocks = kTcTile / kBlockSize;  // 16-token blocks per tile
#ifndef PDA_TC_STAGES
#define PDA_TC_STAGES 3  // K ring 3 x 36 KiB + V ring 3 x 32 KiB of shared memory
#endif
constexpr int kTcStages = PDA_TC_STAGES;
#ifndef PDA_TC_STAMPS
#define PDA_TC_STAMPS 0  // measurement builds only: per-tile clock64 stamps after the workspace
#endif
constexpr int kTcStampTiles = 64, kTcStampEvents = 8;
constexpr int kTcNQ = 16;  // q rows per tile (the GQA group, padded; UMMA N of QK^T)
constexpr int kTcGroupWarps = 4;                       // softmax warps per group (one per TMEM lane quarter)
constexpr int kTcSoftWarps = 2 * kTcGroupWarps;        // two groups, alternating tiles
constexpr int kTcProducerWarp = kTcSoftWarps, kTcMmaWarp = kTcSoftWarps + 1;
constexpr int kTcThreads = (kTcSoftWarps + 2) * 32;
// K tile [block][8-row half][chunk][8 rows][128 B]: the 8-row groups of a
// chunk lie 2048 B apart (one 4-D TMA box per block, encode_k4d_map)
constexpr int kTcKBytes = 2 * kTcTile * 128;
constexpr int kTcVBytes = kTcBlocks * 4096;        // one slab [chunk][16 tokens][128 B] per block
constexpr int kTcQBytes = 2 * kTcNQ * 128;         // [chunk][16 rows][128 B]
// Separate K and V rings (tile granular): a K stage (K tile + q rows) is free
// as soon as QK^T has read it, a V stage only after PV -- so K runs ahead and
// the V ring holds bytes in flight rather than bytes waiting for the softmax
constexpr int kTcKStageBytes = kTcKBytes + kTcQBytes;
constexpr int kTcRing = 16;  // tile descriptors / block rows in flight (K runs <= ~9 tiles ahead of PV)
constexpr int kTcPBytes = kTcTile * 32 * 2;        // one P buffer: tile tokens x (16 hi + 16 lo) columns
constexpr int kTcPSbo = (kTcTile / 8) * 128;       // P core-matrix stride between 8-column groups
// TMEM: S of group 0 / 1 at columns [0,16) / [16,32); O^T of (group, segment parity) 32 columns each
constexpr uint32_t kTcTmemCols = 256;
__device__ __forceinline__ uint32_t tc_ocol(int gr, int ob) { return 32 + 64 * gr + 32 * ob; }
constexpr float kTcRescaleLog2 = 8.f;              // raise m only past m + 8 (p <= 256)

// tile flags (per group: a segment's tiles alternate between the two softmax groups)
constexpr int kFirstG = 1, kLastG = 2, kFinal = 4, kBoth = 8;  // kind << 4, segment parity << 6

struct TcTileInfo {
    int b, kvh, j0, nblk, L, flags;
    int ouse[2];  // how many earlier segments of this parity used O[group][parity] (barrier phases)
    int suse;     // earlier handoffs through st_ready[non-final group][parity]
};

struct TcShared {
    uint64_t kfull[kTcStages], kempty[kTcStages], vfull[kTcStages], vempty[kTcStages];
    uint64_t s_full[2], s_free[2], p_full[2], p_free[2];
    uint64_t o_full[2][2], o_free[2][2], st_ready[2][2];
    TcTileInfo info[kTcRing];
    int rows[kTcRing][kTcBlocks];  // cache row (phys * Hkv + kvh) * 16 of each block of a tile
    uint32_t tmem;
    int n_tiles;
    int n_segs, end_j;
    Cursor start;
    int vote[2][2][kTcGroupWarps];
    float tmax[2][2][kTcGroupWarps][kTcNQ];
    float lsum[2][kTcGroupWarps][kTcNQ];
    // a group's (m, l) handed to the merging group, [group][parity][handoff parity]: the
    // writer may run one handoff ahead of the merger's read
    float st_m[2][2][2][kTcNQ], st_l[2][2][2][kTcNQ];
};

constexpr size_t kTcSmemBytes =
    1024 + kTcStages * (kTcKStageBytes + kTcVBytes) + 2 * kTcPBytes + sizeof(TcShared) + 64;

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
    uint8_t* kst = smem;                                 // K stages [kTcStages][K tile | q rows]
    uint8_t* vst = smem + kTcStages * kTcKStageBytes;    // V stages [kTcStages][8 slabs]
    uint8_t* pbuf = vst + kTcStages * kTcVBytes;
    TcShared* sh = reinterpret_cast<TcShared*>(pbuf + 2 * kTcPBytes);  // P: one buffer per softmax group
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
            sh->n_segs = rp.n_segs;
            sh->end_j = rp.end_j;
            sh->start = rp.start;
            for (int s = 0; s < kTcStages; ++s) {
                mbar_init(&sh->kfull[s], 1);
                // released by QK^T's commit AND by the softmax group having read the
                // tile's info: the group waits kfull on the stage, which must not
                // complete again (K of tile i + 3) before that wait -- parity aliasing
                mbar_init(&sh->kempty[s], 2);
                mbar_init(&sh->vfull[s], 1);
                mbar_init(&sh->vempty[s], 1);
            }
            for (int s = 0; s < 2; ++s) {
                mbar_init(&sh->s_full[s], 1);
                mbar_init(&sh->s_free[s], kTcGroupWarps);
                mbar_init(&sh->p_full[s], kTcGroupWarps);
                mbar_init(&sh->p_free[s], 1);
                for (int ob = 0; ob < 2; ++ob) {
                    mbar_init(&sh->o_full[s][ob], 1);
                    mbar_init(&sh->o_free[s][ob], kTcGroupWarps);
                    mbar_init(&sh->st_ready[s][ob], 1);
                }
            }
            fence_barrier_init();
        }
    }
    if (warp == kTcMmaWarp) tc::alloc<kTcTmemCols>(&sh->tmem);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const int n_tiles = sh->n_tiles;
    // PDA_TC_STAMPS: [cta][tile][event] clock64 right after the seq_prefix region
    unsigned long long* stamps = nullptr;
    if constexpr (PDA_TC_STAMPS != 0)
        stamps = reinterpret_cast<unsigned long long*>(p.seq_prefix + p.B + 1) + (size_t)c * kTcStampTiles * kTcStampEvents;
    auto stamp = [&](int tile, int ev) {
        if constexpr (PDA_TC_STAMPS != 0)
            if (tile < kTcStampTiles) stamps[tile * kTcStampEvents + ev] = clock64();
    };
    const uint32_t tm = sh->tmem;

    // context_len == 0 rows: zeros (reading R6), sequences strided over the grid
    if (warp < kTcSoftWarps)
        for (int b = c; b < p.B; b += gridDim.x)
            if (__ldg(p.lens + b) <= 0)
                for (int i = threadIdx.x; i < p.Hq * 128; i += kTcSoftWarps * 32)
                    store_out(p.out, (size_t)b * p.Hq * 128 + i, 0.f, p.out_dtype);

    if (warp == kTcProducerWarp) {
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
        int wrow = -1, wbase = 0, w0 = 0;  // 32 block ids [wbase, wbase + 32) of row wrow
        int ouse[2][2] = {{0, 0}, {0, 0}}, suse[2][2] = {{0, 0}, {0, 0}};  // barrier use counts
        // the current segment: blocks [j, jend] of row cur; tiles t0 .. t0 + nt - 1
        int seg = 0, j = cur.j, jend = 0, kind = 0, t0 = 0, nt = 0, ob = 0, u0 = 0, u1 = 0, us = 0;
        const int32_t* btrow = nullptr;
        auto start_seg = [&](int first_tile) {
            jend = seg == n_segs - 1 ? end_j : cur.n - 1;
            kind = tc_kind(seg, n_segs, end_j, cur.n, starts_row);
            btrow = p.bt + (size_t)cur.b * p.max_blocks;
            t0 = first_tile;
            nt = (jend - cur.j + kTcBlocks) / kTcBlocks;
            ob = seg & 1;
            const int merger = (t0 + nt - 1) & 1;  // the group of the final tile merges both groups
            // use indices of this segment's O buffers / state handoff (see TcTileInfo)
            u0 = ouse[0][ob];
            u1 = ouse[1][ob];
            us = suse[merger ^ 1][ob];
            for (int gg = 0; gg < 2; ++gg)
                if (nt >= 2 || (t0 & 1) == gg) ++ouse[gg][ob];
            if (nt >= 2) ++suse[merger ^ 1][ob];
        };
        if (n_tiles > 0) start_seg(0);
        // event loop: the next K tile when its K stage is free, the next V tile
        // (never ahead of K) when its V stage is free
        int nk = 0, nv = 0;
        while (nv < n_tiles) {
            if (nk < n_tiles &&
                (nk < kTcStages || mbar_test(&sh->kempty[nk % kTcStages], ((nk / kTcStages) - 1) & 1))) {
                if (j > jend) {  // next segment
                    next_row(cur, p.lens, p.B, p.Hkv, max_tokens);
                    ++seg;
                    j = cur.j;
                    start_seg(nk);
                }
                const int nblk = jend - j + 1 < kTcBlocks ? jend - j + 1 : kTcBlocks;
                if (cur.b != wrow || j < wbase || j + nblk > wbase + 32) {  // refill the id window
                    wrow = cur.b;
                    wbase = j;
                    w0 = wbase + lane < p.max_blocks ? __ldg(btrow + wbase + lane) : 0;
                }
                const int st = nk % kTcStages, ri = nk % kTcRing;
                uint8_t* sb = kst + st * kTcKStageBytes;
                const int phys = __shfl_sync(kAllLanes, w0, (j - wbase + lane) & 31);
                const int row = (phys * p.Hkv + cur.kvh) * kBlockSize;
                if (lane < nblk) sh->rows[ri][lane] = row;
                if (lane == 0) {
                    TcTileInfo& in = sh->info[ri];
                    in.b = cur.b;
                    in.kvh = cur.kvh;
                    in.j0 = j;
                    in.nblk = nblk;
                    in.L = cur.L;
                    const int k = nk - t0;
                    in.flags = (k < 2 ? kFirstG : 0) | (k >= nt - 2 ? kLastG : 0) | (k == nt - 1 ? kFinal : 0) |
                               (nt >= 2 ? kBoth : 0) | (kind << 4) | (ob << 6);
                    in.ouse[0] = u0;
                    in.ouse[1] = u1;
                    in.suse = us;
                    mbar_arrive_expect_tx(&sh->kfull[st], kTcQBytes + nblk * 4096);
                    tma_load_3d(sb + kTcKBytes, &tmQ, 0, cur.b * p.Hq + cur.kvh * g, 0, &sh->kfull[st]);
                }
                __syncwarp();  // lane 0's expect_tx precedes every lane's copies
                // lane b issues block b's K as one 4-D box
                if (lane < nblk) tma_load_4d_hint(sb + lane * 4096, &tmK, 0, 0, 0, row >> 3, &sh->kfull[st], pol_first);
                if (lane == 0) stamp(nk, 0);  // K issued
                j += kTcBlocks;
                ++nk;
                continue;
            }
            if (nv < nk && (nv < kTcStages || mbar_test(&sh->vempty[nv % kTcStages], ((nv / kTcStages) - 1) & 1))) {
                const int st = nv % kTcStages, ri = nv % kTcRing;
                __syncwarp();  // the ring entries this warp wrote
                const int nblk = sh->info[ri].nblk;
                const int row = lane < nblk ? sh->rows[ri][lane] : 0;
                if (lane == 0) mbar_arrive_expect_tx(&sh->vfull[st], nblk * 4096);
                __syncwarp();
                if (lane < nblk)
                    tma_load_3d_hint(vst + st * kTcVBytes + lane * 4096, &tmV, 0, row, 0, &sh->vfull[st], pol_first);
                if (lane == 0) stamp(nv, 1);  // V issued
                ++nv;
            }
        }
    } else if (warp == kTcMmaWarp) {
        // ============================ MMA issuer ============================
        if (lane == 0) {
            const uint32_t idq = tc::idesc_f16(BF16, kTcTile, kTcNQ, false, false);
            const uint32_t idp = tc::idesc_f16(BF16, 128, NP, true, true);
            const uint32_t pb = smem_u32(pbuf);
            auto pv = [&](int j) {
                const int st = j % kTcStages, gj = j & 1;
                const TcTileInfo in = sh->info[j % kTcRing];
                mbar_wait(&sh->p_full[gj], (j >> 1) & 1);
                mbar_wait(&sh->vfull[st], (j / kTcStages) & 1);
                tc::fence_after();
                const int ob = (in.flags >> 6) & 1;
                const bool first = in.flags & kFirstG;
                const int use = gj ? in.ouse[1] : in.ouse[0];
                if (first && use >= 1) {  // O[gj][ob] read out by the previous segment's merge
                    mbar_wait(&sh->o_free[gj][ob], (use - 1) & 1);
                    tc::fence_after();
                }
                const uint32_t vb = smem_u32(vst + st * kTcVBytes);
                for (int blk = 0; blk < in.nblk; ++blk) {
                    const uint64_t a = tc::smem_desc(vb + blk * 4096, 2048, 1024, tc::kLayoutSw128);
                    const uint64_t bd = tc::smem_desc(pb + gj * kTcPBytes + blk * 256, 128, kTcPSbo,
                                                      tc::kLayoutInterleave);
                    tc::mma_f16_ss(tm + tc_ocol(gj, ob), a, bd, idp, !(first && blk == 0));
                }
                tc::commit(&sh->p_free[gj]);
                tc::commit(&sh->vempty[st]);
                if (in.flags & kLastG) tc::commit(&sh->o_full[gj][ob]);
            };
            // event loop: QK^T of tile i as soon as its data and its group's S
            // buffer are there (its group has read the previous S), PV of tile j as soon
            // as its group's P is written -- the two softmax groups never wait
            // for each other through this thread's program order
            int i = 0, j = 0;
            while (j < n_tiles) {
                if (i < n_tiles) {
                    const int st = i % kTcStages, sb = i & 1;
                    if (mbar_test(&sh->kfull[st], (i / kTcStages) & 1) &&
                        (i < 2 || mbar_test(&sh->s_free[sb], ((i >> 1) - 1) & 1))) {
                        tc::fence_after();
                        const uint32_t kb = smem_u32(kst + st * kTcKStageBytes);
                        const uint32_t qb = kb + kTcKBytes;
#pragma unroll
                        for (int kk = 0; kk < 8; ++kk) {
                            const uint64_t a =
                                tc::smem_desc(kb + (kk >> 2) * 1024 + (kk & 3) * 32, 16, 2048, tc::kLayoutSw128);
                            const uint64_t bd = tc::smem_desc(qb + (kk >> 2) * (kTcNQ * 128) + (kk & 3) * 32, 16,
                                                              1024, tc::kLayoutSw128);
                            tc::mma_f16_ss(tm + 16 * sb, a, bd, idq, kk > 0);
                        }
                        tc::commit(&sh->s_full[sb]);
                        stamp(i, 2);  // QK^T issued
                        tc::commit(&sh->kempty[st]);  // QK^T has read the K tile and q
                        ++i;
                        continue;
                    }
                }
                // PV only once its V tile has landed too: a blocking wait here
                // would stall QK^T of later tiles behind the V stream
                if (j < i && mbar_test(&sh->p_full[j & 1], (j >> 1) & 1) &&
                    mbar_test(&sh->vfull[j % kTcStages], (j / kTcStages) & 1)) {
                    stamp(j, 5);  // PV issued
                    pv(j);
                    ++j;
                }
            }
        }
        __syncwarp();
    } else {
        // ========= softmax + epilogue: group gr (warps 4gr..4gr+3) owns tiles i with i % 2 == gr =========
        const int gr = warp / kTcGroupWarps, gw = warp % kTcGroupWarps;  // gw = the warp's TMEM lane quarter
        const int t = gw * 32 + lane;  // token of the tile = S^T row; d row of O^T
        const uint32_t lane_base = (uint32_t)(gw * 32) << 16;
        const int bar_id = 1 + gr;
        float m_ref[kTcNQ], l[kTcNQ];
        const float scale_log2 = p.scale_log2;
        for (int i = gr; i < n_tiles; i += 2) {
            const int st = i % kTcStages, it = i >> 1;
            mbar_wait(&sh->kfull[st], (i / kTcStages) & 1);  // acquire the producer's tile info
            const TcTileInfo in = sh->info[i % kTcRing];
            if (threadIdx.x % (kTcGroupWarps * 32) == 0) mbar_arrive(&sh->kempty[st]);
            mbar_wait(&sh->s_full[gr], it & 1);
            if (threadIdx.x % (kTcGroupWarps * 32) == 0) stamp(i, 3);  // S ready
            tc::fence_after();
            uint32_t r[16];
            tc::ld_32x32b_x16(tm + lane_base + 16 * gr, r);
            tc::wait_ld();
            tc::fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&sh->s_free[gr]);
            const bool first = in.flags & kFirstG;
            if (first) {
#pragma unroll
                for (int cc = 0; cc < kTcNQ; ++cc) {
                    m_ref[cc] = -INFINITY;
                    l[cc] = 0.f;
                }
            }
            const bool valid = t < in.nblk * kBlockSize && in.j0 * kBlockSize + t < in.L;
            float s[kTcNQ];
            bool need = false;
#pragma unroll
            for (int cc = 0; cc < kTcNQ; ++cc) {
                // select, never arithmetic: rows of unloaded / past-the-end tokens may hold NaN
                s[cc] = valid ? __uint_as_float(r[cc]) * scale_log2 : -INFINITY;
                need |= s[cc] > m_ref[cc] + kTcRescaleLog2;
            }
            // every warp of the group must agree on m: one vote per tile
            const bool wneed = __any_sync(kAllLanes, need);
            if (lane == 0) sh->vote[gr][it & 1][gw] = wneed;
            asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "n"(kTcGroupWarps * 32) : "memory");
            bool any = false;
#pragma unroll
            for (int w = 0; w < kTcGroupWarps; ++w) any |= sh->vote[gr][it & 1][w] != 0;
            bool rescale_o = false;
            float alpha[kTcNQ];
            if (any) {
                // the tile's exact max per column; m = max(m, tile max)
#pragma unroll
                for (int cc = 0; cc < kTcNQ; ++cc) {
                    const uint32_t k = __reduce_max_sync(kAllLanes, fkey(s[cc]));
                    if (lane == cc) sh->tmax[gr][it & 1][gw][cc] = fkey_inv(k);
                }
                asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "n"(kTcGroupWarps * 32) : "memory");
#pragma unroll
                for (int cc = 0; cc < kTcNQ; ++cc) {
                    float mx = m_ref[cc];
#pragma unroll
                    for (int w = 0; w < kTcGroupWarps; ++w) mx = fmaxf(mx, sh->tmax[gr][it & 1][w][cc]);
                    alpha[cc] = m_ref[cc] == -INFINITY ? 0.f : ex2(m_ref[cc] - mx);
                    rescale_o |= alpha[cc] != 1.f;
                    l[cc] *= alpha[cc];
                    m_ref[cc] = mx;
                }
                rescale_o &= !first;
            }
            // the group's previous PV is complete: its P buffer and O^T may be touched
            if (it >= 1) mbar_wait(&sh->p_free[gr], (it - 1) & 1);
            const int ob = (in.flags >> 6) & 1;
            if (rescale_o) {
                tc::fence_after();
#pragma unroll
                for (int h = 0; h < NP / 16; ++h) {
                    uint32_t o[16];
                    const uint32_t oa = tm + lane_base + tc_ocol(gr, ob) + 16 * h;
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
            uint8_t* prow = pbuf + gr * kTcPBytes + (t & 7) * 16 + (t >> 3) * 128;
            *reinterpret_cast<uint4*>(prow) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
            *reinterpret_cast<uint4*>(prow + kTcPSbo) = make_uint4(hi[4], hi[5], hi[6], hi[7]);
            if constexpr (BF16) {
                *reinterpret_cast<uint4*>(prow + 2 * kTcPSbo) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
                *reinterpret_cast<uint4*>(prow + 3 * kTcPSbo) = make_uint4(lo[4], lo[5], lo[6], lo[7]);
            }
            const bool zero_v = !valid && t < in.nblk * kBlockSize;
            if (__any_sync(kAllLanes, zero_v)) mbar_wait(&sh->vfull[st], (i / kTcStages) & 1);  // V landed
            if (zero_v) {
                // a loaded token past the context end: zero its V row (0 * NaN would poison PV)
                uint8_t* vrow = vst + st * kTcVBytes + (t >> 4) * 4096 + (t & 15) * 128;
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    *reinterpret_cast<uint4*>(vrow + u * 16) = make_uint4(0, 0, 0, 0);
                    *reinterpret_cast<uint4*>(vrow + 2048 + u * 16) = make_uint4(0, 0, 0, 0);
                }
            }
            tc::fence_async_smem();
            tc::fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&sh->p_full[gr]);
            if (threadIdx.x % (kTcGroupWarps * 32) == 0) stamp(i, 4);  // P written

            if (in.flags & kLastG) {
                // ---- S7: this group's share of the segment: (m, l) per column
#pragma unroll
                for (int cc = 0; cc < kTcNQ; ++cc) {
                    float v = l[cc];
#pragma unroll
                    for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(kAllLanes, v, o);
                    if (lane == cc) sh->lsum[gr][gw][cc] = v;
                }
                asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "n"(kTcGroupWarps * 32) : "memory");
                float Ls[kTcNQ];
#pragma unroll
                for (int cc = 0; cc < kTcNQ; ++cc) {
                    Ls[cc] = 0.f;
#pragma unroll
                    for (int w = 0; w < kTcGroupWarps; ++w) Ls[cc] += sh->lsum[gr][w][cc];
                }
                if (!(in.flags & kFinal)) {
                    // hand the share to the other group, which merges at the segment's final tile
#pragma unroll
                    for (int cc = 0; cc < kTcNQ; ++cc)
                        if (t == cc) {  // (static register indices: no local-memory arrays)
                            sh->st_m[gr][ob][in.suse & 1][cc] = m_ref[cc];
                            sh->st_l[gr][ob][in.suse & 1][cc] = Ls[cc];
                        }
                    asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "n"(kTcGroupWarps * 32) : "memory");
                    if (t == 0) mbar_arrive(&sh->st_ready[gr][ob]);
                } else {
                    // ---- merge both groups' shares (the segment's output or partial)
                    const int og = gr ^ 1;
                    const bool both = in.flags & kBoth;
                    const int use_own = gr ? in.ouse[1] : in.ouse[0], use_oth = gr ? in.ouse[0] : in.ouse[1];
                    if (both) mbar_wait(&sh->st_ready[og][ob], in.suse & 1);
                    mbar_wait(&sh->o_full[gr][ob], use_own & 1);
                    if (both) mbar_wait(&sh->o_full[og][ob], use_oth & 1);
                    tc::fence_after();
                    // O^T row d of both groups (hi + lo terms summed as they are read)
                    float oa[16], ox[16];
                    {
                        uint32_t h[16], lo_[16];
                        tc::ld_32x32b_x16(tm + lane_base + tc_ocol(gr, ob), h);
                        if constexpr (BF16) tc::ld_32x32b_x16(tm + lane_base + tc_ocol(gr, ob) + 16, lo_);
                        tc::wait_ld();
#pragma unroll
                        for (int cc = 0; cc < 16; ++cc)
                            oa[cc] = __uint_as_float(h[cc]) + (BF16 ? __uint_as_float(lo_[cc]) : 0.f);
                        if (both) {
                            tc::ld_32x32b_x16(tm + lane_base + tc_ocol(og, ob), h);
                            if constexpr (BF16) tc::ld_32x32b_x16(tm + lane_base + tc_ocol(og, ob) + 16, lo_);
                            tc::wait_ld();
                        }
#pragma unroll
                        for (int cc = 0; cc < 16; ++cc)
                            ox[cc] = both ? __uint_as_float(h[cc]) + (BF16 ? __uint_as_float(lo_[cc]) : 0.f) : 0.f;
                    }
                    tc::fence_before();
                    __syncwarp();
                    if (lane == 0) {
                        mbar_arrive(&sh->o_free[gr][ob]);
                        if (both) mbar_arrive(&sh->o_free[og][ob]);
                    }
                    const int kind = (in.flags >> 4) & 3;
                    const int NH = g <= 8 ? 8 : 16;
                    const int d = t;
#pragma unroll
                    for (int cc = 0; cc < kTcNQ; ++cc) {
                        if (cc >= g) break;
                        float M = m_ref[cc], den = Ls[cc], num = oa[cc];
                        if (both) {
                            const float mo = sh->st_m[og][ob][in.suse & 1][cc];
                            const float lo2 = sh->st_l[og][ob][in.suse & 1][cc];
                            const float Mn = fmaxf(M, mo);
                            const float wa = ex2(M - Mn), wb = ex2(mo - Mn);
                            num = num * wa + ox[cc] * wb;
                            den = den * wa + lo2 * wb;
                            M = Mn;
                        }
                        const float v = num / den;
                        if (kind == 0) {
                            store_out(p.out, ((size_t)in.b * p.Hq + in.kvh * g + cc) * 128 + d, v, p.out_dtype);
                        } else {
                            const size_t ws = (size_t)c * 2 + (kind - 1);
                            p.ws_o[(ws * NH + cc) * 128 + d] = v;
                            if (d == 0) p.ws_lse[ws * NH + cc] = M + __log2f(den);
                        }
                    }
                }
            }
        }
    }
    // the main loop is done: the combine grid may start its prologue
    pdl_launch_dependents();
    tc::fence_before();
    __syncthreads();
    if (warp == kTcMmaWarp) tc::dealloc<kTcTmemCols>(tm);
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

int tc_threads() { return kTcThreads; }
size_t tc_stamp_bytes(int grid) {
    return PDA_TC_STAMPS ? (size_t)grid * kTcStampTiles * kTcStampEvents * 8 + 256 : 0;
}

cudaError_t launch_tc(const CUtensorMap& tmK, const CUtensorMap& tmV, const CUtensorMap& tmQ,
                      const BalancedParams& p, bool bf16, int grid, cudaStream_t stream) {
    cudaError_t e = bf16 ? launch_tc_one<true>(tmK, tmV, tmQ, p, grid, stream)
                         : launch_tc_one<false>(tmK, tmV, tmQ, p, grid, stream);
    if (e != cudaSuccess) return e;
    return launch_balanced_combine(p, grid, 128, stream);
}

}  // namespace pda
