// decode_splitk.cu -- the B200 decode paged-attention kernel (split-K over
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
#include "splitk_impl.cuh"

namespace pda {

namespace {

// S8: out = sum_p 2^(lse_p - M) o_p / sum_p 2^(lse_p - M), partitions in fixed order.
// One warp per output row.  Every load is issued before any result is needed
// -- the sequence length, the row's lse (lane i: partition i) and the first
// kPre partials' o -- so the row costs one memory round trip instead of three
// dependent ones (lens -> lse -> o); entries at or past the row's partition
// count are loaded but never used (they may hold anything).  The arithmetic
// (w_p = 2^(lse_p - M), den and acc accumulated in partition order) is the
// cluster merge's, so the two stay bitwise equal.
template <int D>
__global__ void __launch_bounds__(128) combine_kernel(const CombineParams p) {
    constexpr int PER = D / 32;
    constexpr int kPre = 8;
    pdl_wait();  // the partials come from the split-K grid before this one
    const int row = blockIdx.x * 4 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= p.B * p.q_len * p.Hq) return;
    const int b = row / (p.q_len * p.Hq);
    const float* lse = p.ws_lse + (size_t)row * p.p_max;
    const float* o_base = p.ws_o + (size_t)row * p.p_max * D + lane * PER;
    int L = p.lens[b];
    const float lse_l = lane < p.p_max ? lse[lane] : -INFINITY;
    float pre[kPre][PER];
#pragma unroll
    for (int q = 0; q < kPre; ++q) {
        if (q < p.p_max) {
            if constexpr (PER == 4) {
                const float4 x = *reinterpret_cast<const float4*>(o_base + (size_t)q * D);
                pre[q][0] = x.x;
                pre[q][1] = x.y;
                pre[q][2] = x.z;
                pre[q][3] = x.w;
            } else {
                const float2 x = *reinterpret_cast<const float2*>(o_base + (size_t)q * D);
                pre[q][0] = x.x;
                pre[q][1] = x.y;
            }
        }
    }
    L = L < p.max_tokens ? L : p.max_tokens;
    const int n_parts = (L + p.part_tokens - 1) / p.part_tokens;
    if (n_parts <= 1) return;  // written by the main kernel
    float M = lane < n_parts ? lse_l : -INFINITY;
    for (int i = 32 + lane; i < n_parts; i += 32) M = fmaxf(M, lse[i]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(kFull, M, o));
    if (M == -INFINITY) M = 0.f;  // every partition empty for this column
    float accv[PER];
#pragma unroll
    for (int e = 0; e < PER; ++e) accv[e] = 0.f;
    float den = 0.f;
#pragma unroll
    for (int q = 0; q < kPre; ++q) {
        const float lq = __shfl_sync(kFull, lse_l, q);
        if (q < n_parts) {
            const float w = ex2(lq - M);
            den += w;
#pragma unroll
            for (int e = 0; e < PER; ++e) accv[e] += w * pre[q][e];
        }
    }
    for (int part = kPre; part < n_parts; ++part) {
        const float w = ex2((part < 32 ? __shfl_sync(kFull, lse_l, part) : lse[part]) - M);
        den += w;
        const float* op = o_base + (size_t)part * D;
        if constexpr (PER == 4) {
            const float4 x = *reinterpret_cast<const float4*>(op);
            accv[0] += w * x.x;
            accv[1] += w * x.y;
            accv[2] += w * x.z;
            accv[3] += w * x.w;
        } else {
            const float2 x = *reinterpret_cast<const float2*>(op);
            accv[0] += w * x.x;
            accv[1] += w * x.y;
        }
    }
    const float inv = den > 0.f ? 1.f / den : 0.f;  // no visible token at all: zero row
#pragma unroll
    for (int e = 0; e < PER; ++e)
        store_out_peers(p.outs, row, p.Hq, D, lane * PER + e, accv[e] * inv, p.out_dtype);
}

}  // namespace


int splitk_threads(bool self_issue, bool tile_split) {
    if (tile_split) return splitk_block_threads<true, true>();
    return self_issue ? splitk_block_threads<true>() : splitk_block_threads<false>();
}

cudaError_t launch_splitk(const CUtensorMap& tmK, const CUtensorMap& tmV, const SplitKParams& p,
                          bool bf16, int head_dim, int n_tiles, int stages, bool trace, dim3 grid,
                          cudaStream_t stream, bool kv8, bool self_issue) {
    if (trace)
        return launch_splitk_m1(tmK, tmV, p, bf16, head_dim, n_tiles, stages, grid, stream, kv8, self_issue);
    if (p.cluster > 1)
        return launch_splitk_m2(tmK, tmV, p, bf16, head_dim, n_tiles, stages, grid, stream, kv8, self_issue);
    return launch_splitk_m0(tmK, tmV, p, bf16, head_dim, n_tiles, stages, grid, stream, kv8, self_issue);
}

cudaError_t launch_combine(const CombineParams& p, int head_dim, cudaStream_t stream) {
    // PDL (default, p.pdl): the combine grid may be scheduled while the split-K
    // grid drains and waits (griddepcontrol.wait) before reading the partials.
    // PDL of the combine alone measured neutral to -2 %; of split-K + combine
    // together it is the default.
    const int rows = p.B * p.q_len * p.Hq;
    const dim3 grid((rows + 3) / 4);
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
        return head_dim == 64 ? cudaLaunchKernelEx(&cfg, combine_kernel<64>, p)
                              : cudaLaunchKernelEx(&cfg, combine_kernel<128>, p);
    }
    if (head_dim == 64)
        combine_kernel<64><<<grid, 128, 0, stream>>>(p);
    else
        combine_kernel<128><<<grid, 128, 0, stream>>>(p);
    return cudaGetLastError();
}

}  // namespace pda
