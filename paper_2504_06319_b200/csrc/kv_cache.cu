// kv_cache.cu -- KV-cache side kernels: the standalone KV append (the
// decode step's cache write, fused into the split-K kernel when that kernel
// runs; kv_append.cuh) and the debug validation of device-resident block
// tables and lengths (out-of-range values are undefined behaviour
// on the hot path; this kernel flags them on request).
#include "kv_append.cuh"

namespace pda {

namespace {

__global__ void __launch_bounds__(256) kv_append_kernel(const AppendParams a, const int32_t* bt,
                                                        const int32_t* lens, int B, int q_len, int Hkv,
                                                        int D, int max_blocks) {
    const int CH = D / 8;
    const long long total = (long long)B * q_len * Hkv * 2 * CH;
    const int max_tokens = max_blocks * kBlockSize;
    for (long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x; c < total;
         c += (long long)gridDim.x * blockDim.x) {
        const int ch = (int)(c % CH);
        long long r = c / CH;
        const int which = (int)(r & 1);
        r >>= 1;
        const int kvh = (int)(r % Hkv);
        r /= Hkv;
        const int i = (int)(r % q_len);
        const int b = (int)(r / q_len);
        int L = lens[b];
        L = L < max_tokens ? L : max_tokens;
        const int t = L - q_len + i;
        if (t < 0) continue;
        append_chunk(a, bt, max_blocks, q_len, Hkv, D, b, i, kvh, t, which, ch);
    }
}

// One warp per sequence (grid-stride): lengths outside [0, max_tokens], and
// referenced ids (j < ceil(min(L, max)/16)) outside [0, num_blocks).
__global__ void __launch_bounds__(256) validate_kernel(const int32_t* bt, const int32_t* lens, int B,
                                                       int max_blocks, long long num_blocks,
                                                       unsigned long long* counts) {
    const int lane = threadIdx.x & 31;
    const int warps = gridDim.x * (blockDim.x >> 5);
    const long long max_tokens = (long long)max_blocks * kBlockSize;
    for (int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); b < B; b += warps) {
        long long L = lens[b];
        const bool bad_len = L < 0 || L > max_tokens;
        L = L < 0 ? 0 : (L > max_tokens ? max_tokens : L);
        const int n = (int)((L + kBlockSize - 1) / kBlockSize);
        unsigned bad = 0;
        for (int j = lane; j < n; j += 32) {
            const int32_t id = bt[(size_t)b * max_blocks + j];
            bad += (id < 0 || id >= num_blocks) ? 1u : 0u;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) bad += __shfl_xor_sync(0xffffffffu, bad, o);
        if (lane == 0) {
            if (bad_len) atomicAdd(&counts[0], 1ull);
            if (bad) atomicAdd(&counts[1], (unsigned long long)bad);
            if (bad_len || bad) atomicAdd(&counts[2], 1ull);
        }
    }
}

}  // namespace

cudaError_t launch_kv_append(const AppendParams& a, const int32_t* bt, const int32_t* lens, int B,
                             int q_len, int Hkv, int head_dim, int max_blocks, cudaStream_t stream) {
    const long long total = (long long)B * q_len * Hkv * 2 * (head_dim / 8);
    if (total == 0) return cudaSuccess;
    long long blocks = (total + 255) / 256;
    blocks = blocks < 148 * 8 ? blocks : 148 * 8;
    kv_append_kernel<<<(unsigned)blocks, 256, 0, stream>>>(a, bt, lens, B, q_len, Hkv, head_dim, max_blocks);
    return cudaGetLastError();
}

cudaError_t launch_validate(const int32_t* bt, const int32_t* lens, int B, int max_blocks,
                            int64_t num_blocks, long long* counts, cudaStream_t stream) {
    cudaError_t e = cudaMemsetAsync(counts, 0, 3 * sizeof(long long), stream);
    if (e != cudaSuccess || B == 0) return e;
    int blocks = (B + 7) / 8;
    blocks = blocks < 148 * 4 ? blocks : 148 * 4;
    validate_kernel<<<blocks, 256, 0, stream>>>(bt, lens, B, max_blocks, (long long)num_blocks,
                                                reinterpret_cast<unsigned long long*>(counts));
    return cudaGetLastError();
}

}  // namespace pda
