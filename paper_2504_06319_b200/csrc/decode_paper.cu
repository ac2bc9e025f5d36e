// decode_paper.cu -- the paper's kernel structure, re-created for sm_100a as
// the ablation baseline (Section 3.1; Algorithm 1).
//
//  * Grid [H, B, 1]: one CTA per (q head, sequence); 128 threads =
//    4 warps (Table 2 N_thread).
//  * Warp w handles KV blocks block_idx = w, w + 4, ... < e (the
//    warp-per-block split; e = ceil(L / 16)).
//  * Per iteration: bt lookup (Alg. 1 line 3) -> load the K (and V)
//    block into registers with 16-byte coalesced loads (line 4) ->
//    if block_idx + d < e prefetch block bt[block_idx + d] into L2 with
//    cp.async.bulk.prefetch.L2 (lines 5-7; d = w = 4 is the
//    paper; V likewise) -> QK^T on CUDA cores with the register-
//    resident Q (line 8) -> online softmax -> P.V.
//  * The warps' (m, l, acc) are merged through shared memory and the CTA
//    writes its output row directly (no split-K: the paper has none).
#include "block_math.cuh"

namespace pda {

namespace {

constexpr uint32_t kFull = kFullMask;

template <bool BF16>
__device__ __forceinline__ void unpack8(const uint4& w, float (&f)[8]) {
    const uint32_t u[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float2 t = unpack2<BF16>(u[i]);
        f[2 * i] = t.x;
        f[2 * i + 1] = t.y;
    }
}

template <bool BF16, int D, bool TRACE>
__global__ void __launch_bounds__(kPaperWarps * 32) paper_kernel(const PaperParams p) {
    constexpr int CH = D / 8;          // 16-byte chunks per token row
    constexpr int TPI = 32 / CH;       // tokens covered by one warp-wide load
    constexpr int NI = kBlockSize / TPI;

    __shared__ float sm_m[kPaperWarps], sm_l[kPaperWarps];
    __shared__ float sm_acc[kPaperWarps][D];

    const int h = blockIdx.x, b = blockIdx.y;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int kvh = h / p.g;  // GQA
    const int c = lane % CH, tg = lane / CH;
    const int max_tokens = p.max_blocks * kBlockSize;
    int L = p.lens[b];
    L = L < max_tokens ? L : max_tokens;
    const int e = (L + kBlockSize - 1) / kBlockSize;
    const int32_t* btrow = p.bt + (size_t)b * p.max_blocks;
    const int d = p.pf_mode != kPfOff ? p.pf_dist : 0;
    const uint64_t pol_first = policy_evict_first(), pol_last = policy_evict_last();

    float qv[8];
    {
        const uint4 w = *reinterpret_cast<const uint4*>(p.q + ((size_t)b * p.Hq + h) * D + c * 8);
        unpack8<BF16>(w, qv);
    }
    float acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = 0.f;
    float m_run = -INFINITY, l_run = 0.f;
    int nv = 0, npf = 0;
    int32_t* rec = nullptr;
    if constexpr (TRACE)
        rec = p.trace + ((size_t)(b * p.Hq + h) * kPaperWarps + warp) * p.trace_rec_len;
    const int R = (p.trace_rec_len - 4) / 2;

    for (int idx = warp; idx < e; idx += kPaperWarps) {
        const int phys = btrow[idx];  // Alg. 1 line 3
        const size_t base = ((size_t)phys * p.Hkv + kvh) * kBlockSize * D;
        uint4 kr[NI], vr[NI];
        if (p.eviction & 1) {  // demand loads evict_first
#pragma unroll
            for (int i = 0; i < NI; ++i) kr[i] = ld_nc_v4_hint(p.k + base + (size_t)(i * TPI + tg) * D + c * 8, pol_first);
#pragma unroll
            for (int i = 0; i < NI; ++i) vr[i] = ld_nc_v4_hint(p.v + base + (size_t)(i * TPI + tg) * D + c * 8, pol_first);
        } else {
#pragma unroll
            for (int i = 0; i < NI; ++i) {  // Alg. 1 line 4: K block -> registers
                const int t = i * TPI + tg;
                kr[i] = ld_nc_v4(p.k + base + (size_t)t * D + c * 8);
            }
#pragma unroll
            for (int i = 0; i < NI; ++i) {
                const int t = i * TPI + tg;
                vr[i] = ld_nc_v4(p.v + base + (size_t)t * D + c * 8);
            }
        }
        if constexpr (TRACE) {
            if (lane == 0) rec[4 + nv] = phys;
        }
        ++nv;
        if (d > 0 && idx + d < e) {  // Alg. 1 lines 5-7: prefetch the next block to L2
            const int nphys = btrow[idx + d];
            const size_t nb = ((size_t)nphys * p.Hkv + kvh) * kBlockSize * D;
            prefetch_kv_slabs<D>(p.k, p.v, nb, p.pf_mode, lane, p.eviction, pol_last);
            if constexpr (TRACE) {
                if (lane == 0) rec[4 + R + npf] = nphys;
            }
            ++npf;
        }
        // Alg. 1 line 8: QK^T with the register-resident Q
        float s[NI];
#pragma unroll
        for (int i = 0; i < NI; ++i) {
            float kf[8];
            unpack8<BF16>(kr[i], kf);
            float dot = 0.f;
#pragma unroll
            for (int e2 = 0; e2 < 8; ++e2) dot = fmaf(qv[e2], kf[e2], dot);
#pragma unroll
            for (int o = CH / 2; o > 0; o >>= 1) dot += __shfl_xor_sync(kFull, dot, o);
            const int t = idx * kBlockSize + i * TPI + tg;
            s[i] = t < L ? dot * p.scale_log2 : -INFINITY;
        }
        float mx = s[0];
#pragma unroll
        for (int i = 1; i < NI; ++i) mx = fmaxf(mx, s[i]);
#pragma unroll
        for (int o = CH; o < 32; o <<= 1) mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, o));
        const float m_new = fmaxf(m_run, mx);
        const float alpha = ex2(m_run - m_new);
        m_run = m_new;
        l_run *= alpha;
#pragma unroll
        for (int e2 = 0; e2 < 8; ++e2) acc[e2] *= alpha;
#pragma unroll
        for (int i = 0; i < NI; ++i) {
            const int t = idx * kBlockSize + i * TPI + tg;
            if (t < L) {  // never touch masked V (0 * NaN)
                const float pr = ex2(s[i] - m_new);
                l_run += pr;
                float vf[8];
                unpack8<BF16>(vr[i], vf);
#pragma unroll
                for (int e2 = 0; e2 < 8; ++e2) acc[e2] = fmaf(pr, vf[e2], acc[e2]);
            }
        }
    }
    // reduce the token groups of the warp (lanes sharing chunk c)
#pragma unroll
    for (int o = CH; o < 32; o <<= 1) {
        l_run += __shfl_xor_sync(kFull, l_run, o);
#pragma unroll
        for (int e2 = 0; e2 < 8; ++e2) acc[e2] += __shfl_xor_sync(kFull, acc[e2], o);
    }
    if constexpr (TRACE) {
        if (lane == 0) {
            rec[0] = warp;
            rec[1] = e;
            rec[2] = nv;
            rec[3] = npf;
        }
    }
    if (lane == 0) {
        sm_m[warp] = m_run;
        sm_l[warp] = l_run;
    }
    if (tg == 0) {
#pragma unroll
        for (int e2 = 0; e2 < 8; ++e2) sm_acc[warp][c * 8 + e2] = acc[e2];
    }
    __syncthreads();
    for (int dd = threadIdx.x; dd < D; dd += blockDim.x) {
        float o = 0.f;
        if (L > 0) {
            float M = -INFINITY;
#pragma unroll
            for (int w = 0; w < kPaperWarps; ++w) M = fmaxf(M, sm_m[w]);
            float num = 0.f, den = 0.f;
#pragma unroll
            for (int w = 0; w < kPaperWarps; ++w) {
                const float sc = ex2(sm_m[w] - M);
                den += sc * sm_l[w];
                num += sc * sm_acc[w][dd];
            }
            o = num / den;
        }
        store_out(p.out, ((size_t)b * p.Hq + h) * D + dd, o, p.out_dtype);
    }
}

template <bool BF16, int D>
cudaError_t launch_t(const PaperParams& p, bool trace, dim3 grid, cudaStream_t s) {
    if (trace)
        paper_kernel<BF16, D, true><<<grid, kPaperWarps * 32, 0, s>>>(p);
    else
        paper_kernel<BF16, D, false><<<grid, kPaperWarps * 32, 0, s>>>(p);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_paper(const PaperParams& p, bool bf16, int head_dim, bool trace, dim3 grid,
                         cudaStream_t stream) {
    if (bf16)
        return head_dim == 64 ? launch_t<true, 64>(p, trace, grid, stream)
                              : launch_t<true, 128>(p, trace, grid, stream);
    return head_dim == 64 ? launch_t<false, 64>(p, trace, grid, stream)
                          : launch_t<false, 128>(p, trace, grid, stream);
}

}  // namespace pda
