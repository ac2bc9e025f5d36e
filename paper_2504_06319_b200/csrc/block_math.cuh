// block_math.cuh -- per-16-token-block attention math on mma.sync, shared by
// the split-K and stream kernels.  One warp, one block of K and V resident in
// shared memory (TMA-written, SWIZZLE_128B, D/64 chunks of [16 rows][128 B]).
//
//   S4  S^T[t][h] = sum_d K[t][d] Q[h][d]        (tokens = MMA M, heads = N)
//   S5  online softmax per head column, tokens >= valid masked (select)
//   S6  O^T[d][h] += sum_t V^T[d][t] P[t][h]     (P transposed with movmatrix)
#pragma once

#include "kernels.cuh"
#include "ptx.cuh"

namespace pda {

constexpr uint32_t kFullMask = 0xffffffffu;

// Byte offset of the 16-byte unit holding column `col` of token row `t`
// inside a slab written by TMA with SWIZZLE_128B: unit u of row t sits at
// unit u ^ (t % 8) of its 128-byte row.
__device__ __forceinline__ uint32_t swz(int t, int col) {
    const int ch = col >> 6;
    const int u = (col & 63) >> 3;
    return ch * 2048 + t * 128 + ((u ^ (t & 7)) << 4);
}

__device__ __forceinline__ void store_out(void* out, size_t idx, float x, int out_dtype) {
    if (out_dtype == 2) {
        static_cast<float*>(out)[idx] = x;
    } else if (out_dtype == 1) {
        static_cast<__nv_bfloat16*>(out)[idx] = __float2bfloat16_rn(x);
    } else {
        static_cast<__half*>(out)[idx] = __float2half_rn(x);
    }
}

// Write one output element of (row = (b * q_len + i) * Hq + local head, d) to
// every destination rank (S9 fused: the TP all-gather happens in the store).
__device__ __forceinline__ void store_out_peers(const OutPeers& o, size_t row, int Hq, int D, int dd, float x,
                                                int out_dtype) {
    const size_t bi = row / Hq, h = row % Hq;
    const size_t idx = (bi * o.Hq_out + o.head_off + h) * D + dd;
    for (int r = 0; r < o.n; ++r) store_out(o.ptr[r], idx, x, out_dtype);
}

// S3: TMA loads of one block's K and V slabs (kChunks boxes of 16 rows x
// 128 B each) into a ring stage, completion counted on `bar`; demand loads
// optionally evict_first (the block is not needed again this step).
template <int kSlab, int kChunks, int kBoxCols>
__device__ __forceinline__ void issue_kv_slabs(uint8_t* dst, const CUtensorMap* tmK, const CUtensorMap* tmV,
                                               int row, uint64_t* bar, int eviction, uint64_t pol_first) {
    if constexpr (kChunks > 1 && kTma3d) {
        // one 3-D box per slab: (64 columns, 16 rows, kChunks column chunks)
        // lands as [chunk][row][128 B], the same bytes as kChunks 2-D boxes
        if (eviction & 1) {
            tma_load_3d_hint(dst, tmK, 0, row, 0, bar, pol_first);
            tma_load_3d_hint(dst + kSlab, tmV, 0, row, 0, bar, pol_first);
        } else {
            tma_load_3d(dst, tmK, 0, row, 0, bar);
            tma_load_3d(dst + kSlab, tmV, 0, row, 0, bar);
        }
    } else {
#pragma unroll
        for (int ch = 0; ch < kChunks; ++ch) {
            if (eviction & 1) {
                tma_load_2d_hint(dst + ch * 2048, tmK, ch * kBoxCols, row, bar, pol_first);
                tma_load_2d_hint(dst + kSlab + ch * 2048, tmV, ch * kBoxCols, row, bar, pol_first);
            } else {
                tma_load_2d(dst + ch * 2048, tmK, ch * kBoxCols, row, bar);
                tma_load_2d(dst + kSlab + ch * 2048, tmV, ch * kBoxCols, row, bar);
            }
        }
    }
}

// S3 for one slab (K or V) of a block: the split K / V ring, where a K slab is
// refilled as soon as QK^T has read it and a V slab once PV has.
template <int kSlab, int kChunks, int kBoxCols>
__device__ __forceinline__ void issue_slab(uint8_t* dst, const CUtensorMap* tm, int row, uint64_t* bar,
                                           int eviction, uint64_t pol_first) {
    if constexpr (kChunks > 1 && kTma3d) {
        if (eviction & 1)
            tma_load_3d_hint(dst, tm, 0, row, 0, bar, pol_first);
        else
            tma_load_3d(dst, tm, 0, row, 0, bar);
    } else {
#pragma unroll
        for (int ch = 0; ch < kChunks; ++ch) {
            if (eviction & 1)
                tma_load_2d_hint(dst + ch * 2048, tm, ch * kBoxCols, row, bar, pol_first);
            else
                tma_load_2d(dst + ch * 2048, tm, ch * kBoxCols, row, bar);
        }
    }
}

// issue_kv_slabs from a converged warp: all 32 lanes call it, one elected lane
// issues each load (see ptx.cuh; same loads, same barrier).
template <int kSlab, int kChunks, int kBoxCols>
__device__ __forceinline__ void issue_kv_slabs_elect(uint8_t* dst, const CUtensorMap* tmK, const CUtensorMap* tmV,
                                                     int row, uint64_t* bar, int eviction, uint64_t pol_first) {
    if constexpr (kChunks > 1 && kTma3d) {
        if (eviction & 1) {
            tma_load_3d_hint_elect(dst, tmK, 0, row, 0, bar, pol_first);
            tma_load_3d_hint_elect(dst + kSlab, tmV, 0, row, 0, bar, pol_first);
        } else {
            tma_load_3d_elect(dst, tmK, 0, row, 0, bar);
            tma_load_3d_elect(dst + kSlab, tmV, 0, row, 0, bar);
        }
    } else {
#pragma unroll
        for (int ch = 0; ch < kChunks; ++ch) {
            if (eviction & 1) {
                tma_load_2d_hint_elect(dst + ch * 2048, tmK, ch * kBoxCols, row, bar, pol_first);
                tma_load_2d_hint_elect(dst + kSlab + ch * 2048, tmV, ch * kBoxCols, row, bar, pol_first);
            } else {
                tma_load_2d_elect(dst + ch * 2048, tmK, ch * kBoxCols, row, bar);
                tma_load_2d_elect(dst + kSlab + ch * 2048, tmV, ch * kBoxCols, row, bar);
            }
        }
    }
}

template <int D>
__device__ __forceinline__ void issue_kv_slabs(uint8_t* dst, const CUtensorMap* tmK, const CUtensorMap* tmV,
                                               int row, uint64_t* bar, int eviction, uint64_t pol_first) {
    issue_kv_slabs<kBlockSize * D * 2, D / 64, 64>(dst, tmK, tmV, row, bar, eviction, pol_first);
}

// S2: L2 prefetch of the kSlab-byte K and V slabs at byte offset `off`
// (the paper's cp.async.bulk.prefetch.L2, or per-line prefetch.global.L2),
// optionally evict_last.  Warp-wide call; bulk uses lane 0 only.
template <int kSlab>
__device__ __forceinline__ void prefetch_kv_bytes(const uint8_t* k, const uint8_t* v, size_t off, int pf_mode,
                                                  int lane, int eviction, uint64_t pol_last) {
    if (pf_mode == kPfBulk) {
        if (lane == 0) {
            if (eviction & 2) {
                bulk_prefetch_l2_hint(k + off, kSlab, pol_last);
                bulk_prefetch_l2_hint(v + off, kSlab, pol_last);
            } else {
                bulk_prefetch_l2(k + off, kSlab);
                bulk_prefetch_l2(v + off, kSlab);
            }
        }
    } else {
        constexpr int kLines = kSlab / 128;
        if (lane < kLines) {
            if (eviction & 2) {
                prefetch_line_l2_evict_last(k + off + lane * 128);
                prefetch_line_l2_evict_last(v + off + lane * 128);
            } else {
                prefetch_line_l2(k + off + lane * 128);
                prefetch_line_l2(v + off + lane * 128);
            }
        }
    }
}

// 16-bit element form (element offset `off`).
template <int D>
__device__ __forceinline__ void prefetch_kv_slabs(const uint16_t* k, const uint16_t* v, size_t off,
                                                  int pf_mode, int lane, int eviction, uint64_t pol_last) {
    prefetch_kv_bytes<kBlockSize * D * 2>(reinterpret_cast<const uint8_t*>(k), reinterpret_cast<const uint8_t*>(v),
                                          off * 2, pf_mode, lane, eviction, pol_last);
}

// TOKPERM: MMA row m of S^T holds token tok_of_row(m) (the e4m3 path loads K
// rows in that order so that its V^T fragments come straight from a
// transposing byte ldmatrix, see BlockMathKV8); the contraction over tokens
// is order-free, only the masks need the mapping.
// MS = 2 (D split): this warp accumulates only output rows d in
// [16 i0, 16 i0 + D / 2) of O^T; QK^T and the softmax are computed in full.
template <bool BF16, int D, int NT, bool TOKPERM = false, int MS = 1>
struct BlockMath {
    // rows m = 2c + e -> token 4c + e, rows 8 + 2c + e -> token 4c + 2 + e
    static __device__ __forceinline__ int tok_of_row(int m) {
        return TOKPERM ? 4 * ((m & 7) >> 1) + (m & 1) + ((m >> 3) << 1) : m;
    }

    static constexpr int kNT = NT;
    static constexpr int KSTEPS = D / 16;
    static constexpr int MT = D / 16;
    static constexpr int MTL = MT / MS;               // m-tiles of O^T this warp accumulates
    static constexpr int kSlab = kBlockSize * D * 2;  // Eq. 1

    uint32_t qf[KSTEPS][NT][2];  // Q as the B operand of S^T = K Q^T (register-resident)
    float acc[MTL][NT][4];       // O^T accumulators: (d = 16(i0 + i) + lane/4 + 8(r/2), h = 2(lane%4) + r%2)
    int i0 = 0;                  // first m-tile (D split)
    float m_run[NT][2];          // running max per head column (log2 domain)
    float l_run[NT][2];          // per-lane partial row sums (reduced at the end)
    // multi-token decode: column (query token i, head) of this lane may see
    // tokens < L - qoff, qoff = q_len - 1 - i; qm1 = q_len - 1 (0 = single query)
    int qoff[NT][2] = {};
    int qm1 = 0;

    __device__ __forceinline__ void reset() {
#pragma unroll
        for (int i = 0; i < MTL; ++i)
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                for (int r = 0; r < 4; ++r) acc[i][nt][r] = 0.f;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            m_run[nt][0] = m_run[nt][1] = -INFINITY;
            l_run[nt][0] = l_run[nt][1] = 0.f;
        }
    }

    // Columns = (query token i, head h) pairs, c = i * g + h, c < q_len * g.
    // col0: first column of this warp's tiles (8 with the tile-split kernel's second tile)
    __device__ __forceinline__ void set_q_tokens(int q_len, int g, int lane, int col0 = 0) {
        qm1 = q_len - 1;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const int col = col0 + nt * 8 + 2 * (lane & 3) + c;
                qoff[nt][c] = col < q_len * g ? q_len - 1 - col / g : 0;
            }
    }

    // q rows of the columns (token i, head h) of kv head kvh of sequence b
    // (q [B, q_len, Hq, D]); padded columns are zero.
    __device__ __forceinline__ void load_q_tokens(const uint16_t* q, int b, int kvh, int Hq, int q_len, int g,
                                                  int lane, int col0 = 0) {
        const int dq = 2 * (lane & 3);
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            const int col = col0 + nt * 8 + (lane >> 2);
            const bool ok = col < q_len * g;
            const size_t row = ((size_t)b * q_len + (ok ? col / g : 0)) * Hq + kvh * g + (ok ? col % g : 0);
            const uint32_t* qrow = reinterpret_cast<const uint32_t*>(q + row * D);
#pragma unroll
            for (int kk = 0; kk < KSTEPS; ++kk) {
                qf[kk][nt][0] = ok ? __ldg(qrow + ((kk * 16 + dq) >> 1)) : 0u;
                qf[kk][nt][1] = ok ? __ldg(qrow + ((kk * 16 + dq + 8) >> 1)) : 0u;
            }
        }
    }

    // q rows of the g heads of kv head `kvh` of sequence b; heads >= g are zero.
    __device__ __forceinline__ void load_q(const uint16_t* q, size_t first_row, int g, int lane) {
        const int h = lane >> 2;
        const int dq = 2 * (lane & 3);
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            const int hh = nt * 8 + h;
            const uint32_t* qrow = reinterpret_cast<const uint32_t*>(q + (first_row + hh) * D);
#pragma unroll
            for (int kk = 0; kk < KSTEPS; ++kk) {
                qf[kk][nt][0] = hh < g ? __ldg(qrow + ((kk * 16 + dq) >> 1)) : 0u;
                qf[kk][nt][1] = hh < g ? __ldg(qrow + ((kk * 16 + dq + 8) >> 1)) : 0u;
            }
        }
    }

    // One block: K slab at kbase, V slab at vbase (shared addresses); vq =
    // L - (first token of the block): rows >= vq are outside the context (V
    // zeroed), and column c additionally masks rows >= vq - qoff[c].
    // TAIL = false: the caller guarantees no masking is needed
    // (needs_mask(vq) is false), so the masking code is not even issued
    // (predicated-off masks still cost issue slots every block).
    template <bool TAIL = true>
    __device__ __forceinline__ void block(uint32_t kbase, uint32_t vbase, int vq, float scale_log2,
                                          int lane) {
        float s[NT][4], s2[NT][4];
        qk(kbase, lane, s, s2);
        finish<TAIL>(s, s2, vbase, vq, scale_log2, lane);
    }

    // S5 + S6 of a block whose scores qk() produced earlier: the split-K
    // consumers issue the QK^T of their next block before this one's softmax
    // and PV (two independent dependency chains in flight per warp).
    template <bool TAIL = true>
    __device__ __forceinline__ void finish(float (&s)[NT][4], const float (&s2)[NT][4], uint32_t vbase, int vq,
                                           float scale_log2, int lane) {
        uint32_t pb[NT][2], pb_lo[NT][2];
        softmax<TAIL>(s, s2, vq, scale_log2, lane, pb, pb_lo);
        pv<TAIL>(vbase, vq < kBlockSize ? vq : kBlockSize, lane, pb, pb_lo);
    }

    // Does a block starting vq tokens before the context end need masking
    // (some column's limit, or the context end, inside the block)?
    __device__ __forceinline__ bool needs_mask(int vq) const { return vq - qm1 < kBlockSize; }

    // Mask the scores of rows outside each column's context (select, never
    // arithmetic: masked K rows may hold NaN).
    __device__ __forceinline__ void mask_scores(float (&s)[NT][4], int vq, int lane) const {
        if (vq - qm1 >= kBlockSize) return;  // no column reaches into this block's end
        const int t0 = tok_of_row(lane >> 2), t1 = tok_of_row((lane >> 2) + 8);
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const int lim = vq - qoff[nt][c];
                if (t0 >= lim) s[nt][c] = -INFINITY;
                if (t1 >= lim) s[nt][c + 2] = -INFINITY;
            }
    }

    // ---- S4: S^T = K Q^T (two independent accumulator chains s, s2)
    __device__ __forceinline__ void qk(uint32_t kbase, int lane, float (&s)[NT][4], float (&s2)[NT][4]) {
        const int k_t = (lane & 7) + ((lane >> 3) & 1) * 8;
        const int k_c = (lane >> 4) * 8;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int r = 0; r < 4; ++r) s[nt][r] = s2[nt][r] = 0.f;
#pragma unroll
        for (int kk = 0; kk < KSTEPS; ++kk) {
            uint32_t a[4];
            ldsm_x4(kbase + swz(k_t, kk * 16 + k_c), a[0], a[1], a[2], a[3]);
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
                if (kk & 1)
                    mma_16816<BF16>(s2[nt], a, qf[kk][nt][0], qf[kk][nt][1]);
                else
                    mma_16816<BF16>(s[nt], a, qf[kk][nt][0], qf[kk][nt][1]);
            }
        }
    }

    // ---- S5: scale (fp32), mask t >= valid, online softmax per head column;
    // P leaves as PV B fragments (transposed in registers with movmatrix)
    template <bool TAIL = true>
    __device__ __forceinline__ void softmax(float (&s)[NT][4], const float (&s2)[NT][4], int vq,
                                            float scale_log2, int lane, uint32_t (&pb)[NT][2],
                                            uint32_t (&pb_lo)[NT][2]) {
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int r = 0; r < 4; ++r) s[nt][r] = (s[nt][r] + s2[nt][r]) * scale_log2;
        if constexpr (TAIL) mask_scores(s, vq, lane);
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            float pr[4];
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                float mx = fmaxf(s[nt][c], s[nt][c + 2]);
                mx = fmaxf(mx, __shfl_xor_sync(kFullMask, mx, 4));
                mx = fmaxf(mx, __shfl_xor_sync(kFullMask, mx, 8));
                mx = fmaxf(mx, __shfl_xor_sync(kFullMask, mx, 16));
                const float m_new = fmaxf(m_run[nt][c], mx);
                // a column with no visible token yet stays at -inf: use 0 as the
                // reference so that alpha and p are 0, not NaN
                const float m_ref = m_new == -INFINITY ? 0.f : m_new;
                const float alpha = ex2(m_run[nt][c] - m_ref);
                m_run[nt][c] = m_new;
                pr[c] = ex2(s[nt][c] - m_ref);
                pr[c + 2] = ex2(s[nt][c + 2] - m_ref);
                l_run[nt][c] = l_run[nt][c] * alpha + pr[c] + pr[c + 2];
#pragma unroll
                for (int i = 0; i < MTL; ++i) {
                    acc[i][nt][c] *= alpha;
                    acc[i][nt][c + 2] *= alpha;
                }
            }
            const uint32_t w0 = pack2<BF16>(pr[0], pr[1]);
            const uint32_t w1 = pack2<BF16>(pr[2], pr[3]);
            pb[nt][0] = movmatrix_trans(w0);
            pb[nt][1] = movmatrix_trans(w1);
            if constexpr (BF16) {
                // bf16 P keeps 8 mantissa bits: carry the residual as a second
                // bf16 term so P enters PV with ~16 bits (R19).
                const float2 h0 = unpack2<true>(w0), h1 = unpack2<true>(w1);
                pb_lo[nt][0] = movmatrix_trans(pack2<true>(pr[0] - h0.x, pr[1] - h0.y));
                pb_lo[nt][1] = movmatrix_trans(pack2<true>(pr[2] - h1.x, pr[3] - h1.y));
            }
        }
    }

    // Zero the V^T fragment elements of tokens >= valid (0 * NaN would poison).
    static __device__ __forceinline__ void mask_v(uint32_t (&a)[4], int valid, int lane) {
        const int t0 = 2 * (lane & 3);
        const uint32_t m0 = (t0 < valid ? 0xffffu : 0u) | (t0 + 1 < valid ? 0xffff0000u : 0u);
        const uint32_t m1 = (t0 + 8 < valid ? 0xffffu : 0u) | (t0 + 9 < valid ? 0xffff0000u : 0u);
        a[0] &= m0;
        a[1] &= m0;
        a[2] &= m1;
        a[3] &= m1;
    }

    // S6 with the fragments softmax() produced (the split K / V ring waits for
    // the V slab between the two)
    template <bool TAIL = true>
    __device__ __forceinline__ void pv_any(uint32_t vbase, int valid, int lane, const uint32_t (&pb)[NT][2],
                                           const uint32_t (&pb_lo)[NT][2]) {
        pv<TAIL>(vbase, valid, lane, pb, pb_lo);
    }

    // ---- S6: O^T[d][h] += sum_t V^T[d][t] P[t][h]
    template <bool TAIL = true>
    __device__ __forceinline__ void pv(uint32_t vbase, int valid, int lane, const uint32_t (&pb)[NT][2],
                                       const uint32_t (&pb_lo)[NT][2]) {
        const int v_t = (lane & 7) + (lane >> 4) * 8;
        const int v_c = ((lane >> 3) & 1) * 8;
#pragma unroll
        for (int i = 0; i < MTL; ++i) {
            uint32_t a[4];
            ldsm_x4_trans(vbase + swz(v_t, (i0 + i) * 16 + v_c), a[0], a[1], a[2], a[3]);
            if (TAIL && valid < kBlockSize) mask_v(a, valid, lane);
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
                mma_16816<BF16>(acc[i][nt], a, pb[nt][0], pb[nt][1]);
                if constexpr (BF16) mma_16816<BF16>(acc[i][nt], a, pb_lo[nt][0], pb_lo[nt][1]);
            }
        }
    }

    // Output column d held by accumulator acc[i][*][r] of this lane.
    static __device__ __forceinline__ int dcol(int i, int lane, int r) {
        return i * 16 + (lane >> 2) + 8 * (r >> 1);
    }

    // Reduce the per-lane partial row sums across the 8 lanes of each column.
    __device__ __forceinline__ void reduce_l() {
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                float l = l_run[nt][c];
                l += __shfl_xor_sync(kFullMask, l, 4);
                l += __shfl_xor_sync(kFullMask, l, 8);
                l += __shfl_xor_sync(kFullMask, l, 16);
                l_run[nt][c] = l;
            }
    }
};

// FP8 (e4m3) KV-cache variant, head_dim 128.  K and V
// slabs are 16 x 128 bytes (one TMA box, SWIZZLE_128B); every e4m3 value is
// exact in fp16, so the math runs on fp16 MMAs (P in fp16, no hi/lo split).
//  * QK^T: ldmatrix (b16) over byte rows hands each lane 4 consecutive fp8 of
//    a token; converted pairwise to f16x2 they fill the A fragment with the
//    contraction index d permuted within each 16-column k-step -- Q's B
//    fragment is loaded with the same permutation, so q.k is unchanged.
//  * PV: V^T fragments come straight from ldmatrix.m16n16.x2.trans.b8 (lane
//    (g, c): tokens 4c..4c+3 of columns g, g + 8) -- the K rows of QK^T are
//    loaded in the matching token order (tok_of_row), so P's k index lines
//    up; no movmatrix on V, output rows d in natural order.
// Q_BF16 only selects how q is read (bf16 q is converted to fp16).
__device__ __forceinline__ void cvt_e4m3x4(uint32_t w, uint32_t& lo, uint32_t& hi) {
    asm("{\n\t.reg .b16 l, h;\n\tmov.b32 {l, h}, %2;\n\t"
        "cvt.rn.f16x2.e4m3x2 %0, l;\n\tcvt.rn.f16x2.e4m3x2 %1, h;\n\t}"
        : "=r"(lo), "=r"(hi)
        : "r"(w));
}

// MS = 2 (D split): this warp accumulates output rows d in [16 i0, 16 i0 + 64)
// only (PV converts and multiplies half of V); QK^T and the softmax in full.
template <bool Q_BF16, int NT, int MS = 1>
struct BlockMathKV8 : BlockMath<false, 128, NT, true, MS> {
    using Base = BlockMath<false, 128, NT, true, MS>;
    static constexpr int D = 128;
    static constexpr int MT = D / 16;
    static constexpr int MTL = MT / MS;  // m-tiles of O^T this warp accumulates
    static constexpr int kSlab = kBlockSize * D;  // 1 byte per element

    // Q B fragments: qf[2j + half][nt] = Q[col][32j + 16 half + 4(lane%4) + {0,1 | 2,3}],
    // columns = (query token i, head h), c = i * g + h
    __device__ __forceinline__ void load_q_tokens(const uint16_t* q, int b, int kvh, int Hq, int q_len, int g,
                                                  int lane, int col0 = 0) {
        const int t = lane & 3;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            const int col = col0 + nt * 8 + (lane >> 2);
            const bool ok = col < q_len * g;
            const size_t row = ((size_t)b * q_len + (ok ? col / g : 0)) * Hq + kvh * g + (ok ? col % g : 0);
            const uint16_t* qrow = q + row * D;
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk) {
                uint2 w = make_uint2(0u, 0u);
                if (ok) w = __ldg(reinterpret_cast<const uint2*>(qrow + kk * 16 + 4 * t));
                if constexpr (Q_BF16) {
                    const float2 a = unpack2<true>(w.x), b = unpack2<true>(w.y);
                    w.x = pack2<false>(a.x, a.y);
                    w.y = pack2<false>(b.x, b.y);
                }
                this->qf[kk][nt][0] = w.x;
                this->qf[kk][nt][1] = w.y;
            }
        }
    }

    // ---- S4 on e4m3 K (two accumulator chains: even / odd k-steps)
    __device__ __forceinline__ void qk8(uint32_t kbase, int lane, float (&s)[NT][4], float (&s2)[NT][4]) {
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int r = 0; r < 4; ++r) s[nt][r] = s2[nt][r] = 0.f;
        // MMA row m = (lane & 7) + ((lane >> 3) & 1) * 8 is loaded from token tok_of_row(m)
        const int kr = Base::tok_of_row((lane & 7) + ((lane >> 3) & 1) * 8);
#pragma unroll
        for (int j = 0; j < D / 32; ++j) {
            const int unit = 2 * j + (lane >> 4);
            uint32_t r[4];
            ldsm_x4(kbase + kr * 128 + ((unit ^ (kr & 7)) << 4), r[0], r[1], r[2], r[3]);
            uint32_t a[4], c[4];
            cvt_e4m3x4(r[0], a[0], a[2]);
            cvt_e4m3x4(r[1], a[1], a[3]);
            cvt_e4m3x4(r[2], c[0], c[2]);
            cvt_e4m3x4(r[3], c[1], c[3]);
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
                mma_16816<false>(s[nt], a, this->qf[2 * j][nt][0], this->qf[2 * j][nt][1]);
                mma_16816<false>(s2[nt], c, this->qf[2 * j + 1][nt][0], this->qf[2 * j + 1][nt][1]);
            }
        }
    }

    // ---- S6 on e4m3 V: V^T fragments straight from a transposing byte
    // ldmatrix -- lane (g, c) gets tokens 4c..4c+3 of columns d = g and g + 8,
    // which is the A fragment of O^T += V^T P for the token order
    // tok_of_row() gave the rows of S^T (hence of P's k index); no movmatrix.
    static __device__ __forceinline__ void mask_v8(uint32_t (&a)[4], int valid, int lane) {
        const int t0 = 4 * (lane & 3);
        const uint32_t m0 = (t0 < valid ? 0xffffu : 0u) | (t0 + 1 < valid ? 0xffff0000u : 0u);
        const uint32_t m1 = (t0 + 2 < valid ? 0xffffu : 0u) | (t0 + 3 < valid ? 0xffff0000u : 0u);
        a[0] &= m0;
        a[1] &= m0;
        a[2] &= m1;
        a[3] &= m1;
    }

    template <bool TAIL = true>
    __device__ __forceinline__ void pv8(uint32_t vbase, int valid, int lane, const uint32_t (&pb)[NT][2]) {
        const int vr = lane & 15;
#pragma unroll
        for (int ip = 0; ip < MTL / 2; ++ip) {
            // 16 d columns per matrix: tiles 2 gp, 2 gp + 1 (gp: this warp's first
            // tile pair i0 / 2 on, D split)
            const int unit = 2 * (ip + this->i0 / 2) + (lane >> 4);
            uint32_t r[4];
            ldsm_x2_trans_b8(vbase + vr * 128 + ((unit ^ (vr & 7)) << 4), r[0], r[1], r[2], r[3]);
#pragma unroll
            for (int c2 = 0; c2 < 2; ++c2) {
                uint32_t a[4];
                cvt_e4m3x4(r[2 * c2], a[0], a[2]);      // d = g: tokens (4c, 4c+1) | (4c+2, 4c+3)
                cvt_e4m3x4(r[2 * c2 + 1], a[1], a[3]);  // d = g + 8
                if (TAIL && valid < kBlockSize) mask_v8(a, valid, lane);
#pragma unroll
                for (int nt = 0; nt < NT; ++nt)
                    mma_16816<false>(this->acc[2 * ip + c2][nt], a, pb[nt][0], pb[nt][1]);
            }
        }
    }

    // the split-K consumers' software pipeline calls qk() / finish() / finish2()
    __device__ __forceinline__ void qk(uint32_t kbase, int lane, float (&s)[NT][4], float (&s2)[NT][4]) {
        qk8(kbase, lane, s, s2);
    }

    template <bool TAIL = true>
    __device__ __forceinline__ void finish(float (&s)[NT][4], const float (&s2)[NT][4], uint32_t vbase, int vq,
                                           float scale_log2, int lane) {
        uint32_t pb[NT][2], pb_lo[NT][2];
        this->template softmax<TAIL>(s, s2, vq, scale_log2, lane, pb, pb_lo);
        pv8<TAIL>(vbase, vq < kBlockSize ? vq : kBlockSize, lane, pb);
    }

    template <bool TAIL = true>
    __device__ __forceinline__ void pv_any(uint32_t vbase, int valid, int lane, const uint32_t (&pb)[NT][2],
                                           const uint32_t (&)[NT][2]) {
        pv8<TAIL>(vbase, valid, lane, pb);
    }

    template <bool TAIL = true>
    __device__ __forceinline__ void block(uint32_t kbase, uint32_t vbase, int vq, float scale_log2,
                                          int lane) {
        float s[NT][4], s2[NT][4];
        qk8(kbase, lane, s, s2);
        finish<TAIL>(s, s2, vbase, vq, scale_log2, lane);
    }

    // Two blocks (32 tokens) per step: independent QK chains, ONE online-softmax
    // update (shared max / rescale), two PV tiles -- halves the per-block
    // latency chain, which bounds the e4m3 path (half the bytes per block).
    template <bool TAIL = true>
    __device__ __forceinline__ void block2(uint32_t kb0, uint32_t vb0, int vq0, uint32_t kb1, uint32_t vb1,
                                           int vq1, float scale_log2, int lane) {
        float sa[NT][4], sa2[NT][4], sb[NT][4], sb2[NT][4];
        qk8(kb0, lane, sa, sa2);
        qk8(kb1, lane, sb, sb2);
        finish2<TAIL>(sa, sa2, sb, sb2, vb0, vq0, vb1, vq1, scale_log2, lane);
    }

    // S5 + S6 of a block pair whose scores qk() produced earlier
    template <bool TAIL = true>
    __device__ __forceinline__ void finish2(float (&sa)[NT][4], const float (&sa2)[NT][4], float (&sb)[NT][4],
                                            const float (&sb2)[NT][4], uint32_t vb0, int vq0, uint32_t vb1,
                                            int vq1, float scale_log2, int lane) {
        uint32_t pa[NT][2], pbb[NT][2];
        softmax2<TAIL>(sa, sa2, sb, sb2, vq0, vq1, scale_log2, lane, pa, pbb);
        pv8<TAIL>(vb0, vq0 < kBlockSize ? vq0 : kBlockSize, lane, pa);
        pv8<TAIL>(vb1, vq1 < kBlockSize ? vq1 : kBlockSize, lane, pbb);
    }

    // S5 of a block pair: one online-softmax update for both, P fragments out
    template <bool TAIL = true>
    __device__ __forceinline__ void softmax2(float (&sa)[NT][4], const float (&sa2)[NT][4], float (&sb)[NT][4],
                                             const float (&sb2)[NT][4], int vq0, int vq1, float scale_log2,
                                             int lane, uint32_t (&pa)[NT][2], uint32_t (&pbb)[NT][2]) {
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                sa[nt][r] = (sa[nt][r] + sa2[nt][r]) * scale_log2;
                sb[nt][r] = (sb[nt][r] + sb2[nt][r]) * scale_log2;
            }
        if constexpr (TAIL) {
            this->mask_scores(sa, vq0, lane);
            this->mask_scores(sb, vq1, lane);
        }
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            float pra[4], prb[4];
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                float mx = fmaxf(fmaxf(sa[nt][c], sa[nt][c + 2]), fmaxf(sb[nt][c], sb[nt][c + 2]));
                mx = fmaxf(mx, __shfl_xor_sync(kFullMask, mx, 4));
                mx = fmaxf(mx, __shfl_xor_sync(kFullMask, mx, 8));
                mx = fmaxf(mx, __shfl_xor_sync(kFullMask, mx, 16));
                const float m_new = fmaxf(this->m_run[nt][c], mx);
                const float m_ref = m_new == -INFINITY ? 0.f : m_new;  // column not started yet
                const float alpha = ex2(this->m_run[nt][c] - m_ref);
                this->m_run[nt][c] = m_new;
                pra[c] = ex2(sa[nt][c] - m_ref);
                pra[c + 2] = ex2(sa[nt][c + 2] - m_ref);
                prb[c] = ex2(sb[nt][c] - m_ref);
                prb[c + 2] = ex2(sb[nt][c + 2] - m_ref);
                this->l_run[nt][c] = this->l_run[nt][c] * alpha + (pra[c] + pra[c + 2]) + (prb[c] + prb[c + 2]);
#pragma unroll
                for (int i = 0; i < MTL; ++i) {
                    this->acc[i][nt][c] *= alpha;
                    this->acc[i][nt][c + 2] *= alpha;
                }
            }
            pa[nt][0] = movmatrix_trans(pack2<false>(pra[0], pra[1]));
            pa[nt][1] = movmatrix_trans(pack2<false>(pra[2], pra[3]));
            pbb[nt][0] = movmatrix_trans(pack2<false>(prb[0], prb[1]));
            pbb[nt][1] = movmatrix_trans(pack2<false>(prb[2], prb[3]));
        }
    }

};

}  // namespace pda
