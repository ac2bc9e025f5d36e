// kv_append.cuh -- the decode step's KV-cache write, shared by the fused path
// in the split-K kernel and the standalone append kernel (kv_cache.cu).
//
// "each decoding step requires loading the Key-Value Cache": the step's
// new token(s) must be in the paged cache before attention reads it.
// Token i of sequence b (of q_len new tokens) sits at position
// t = L_b - q_len + i, i.e. slot t % 16 of physical block bt[b][t / 16].
#pragma once

#include "kernels.cuh"
#include "ptx.cuh"

namespace pda {

// Chunk `ch` (8 elements = 16 input bytes) of K (which == 0) or V of new token
// i of (b, kvh), stored at position t.
__device__ __forceinline__ void append_chunk(const AppendParams& a, const int32_t* bt, int max_blocks,
                                             int q_len, int Hkv, int D, int b, int i, int kvh, int t,
                                             int which, int ch) {
    const uint16_t* src = (which ? a.v_new : a.k_new) + (((size_t)b * q_len + i) * Hkv + kvh) * D + ch * 8;
    const int64_t phys = bt[(size_t)b * max_blocks + t / kBlockSize];
    const size_t dst = (((size_t)phys * Hkv + kvh) * kBlockSize + t % kBlockSize) * D + ch * 8;
    const uint4 x = *reinterpret_cast<const uint4*>(src);
    uint8_t* cache = which ? a.v : a.k;
    if (!a.kv8) {
        *reinterpret_cast<uint4*>(cache + dst * 2) = x;
        return;
    }
    // e4m3 cache: code = e4m3_rn_satfinite(fp32(x) / fp32(scale))
    const float sc = which ? a.v_scale : a.k_scale;
    const uint32_t w[4] = {x.x, x.y, x.z, x.w};
    uint32_t codes[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        uint32_t packed = 0;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const uint32_t word = w[2 * h + e];
            float lo, hi;
            if (a.bf16) {
                lo = __uint_as_float(word << 16);
                hi = __uint_as_float(word & 0xffff0000u);
            } else {
                lo = __half2float(__ushort_as_half((unsigned short)(word & 0xffff)));
                hi = __half2float(__ushort_as_half((unsigned short)(word >> 16)));
            }
            packed |= (uint32_t)cvt_e4m3x2(__fdiv_rn(lo, sc), __fdiv_rn(hi, sc)) << (16 * e);
        }
        codes[h] = packed;
    }
    *reinterpret_cast<uint2*>(cache + dst) = make_uint2(codes[0], codes[1]);
}

}  // namespace pda
