// roofline.cu -- measurement helper (not part of the method): a read-only
// stream over a large device buffer with 16-byte non-allocating loads, used
// by bench.py as the in-run read roofline next to the decode kernel.
#include "kernels.cuh"
#include "ptx.cuh"

namespace pda {

namespace {

__global__ void __launch_bounds__(512) read_roofline_kernel(const uint4* __restrict__ buf,
                                                            size_t n16, uint32_t* sink) {
    constexpr int U = 8;
    uint32_t x = 0;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + (U - 1) * stride < n16; i += U * stride) {
        uint4 r[U];
#pragma unroll
        for (int u = 0; u < U; ++u) r[u] = ld_nc_v4(buf + i + u * stride);
#pragma unroll
        for (int u = 0; u < U; ++u) x ^= r[u].x ^ r[u].y ^ r[u].z ^ r[u].w;
    }
    for (; i < n16; i += stride) {
        const uint4 r = ld_nc_v4(buf + i);
        x ^= r.x ^ r.y ^ r.z ^ r.w;
    }
    if (x == 0x9e3779b9u) sink[0] = x;  // keeps the loads alive; practically never taken
}

}  // namespace

cudaError_t launch_read_roofline(const void* buf, size_t bytes, void* sink, int num_sms,
                                 cudaStream_t stream) {
    read_roofline_kernel<<<num_sms * 4, 512, 0, stream>>>(static_cast<const uint4*>(buf), bytes / 16,
                                                          static_cast<uint32_t*>(sink));
    return cudaGetLastError();
}

}  // namespace pda
