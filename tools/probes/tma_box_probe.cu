// tma_box_probe.cu -- how fast can CTAs drain 4 KiB TMA tensor boxes (one
// 16-token x 128-column bf16 KV slab, the decode kernels' unit of transfer)
// into a shared-memory ring, with NO math behind the ring?  Separates the
// TMA / memory side of a design from its consumers (DESIGN.md 6 tc_kernel:
// one persistent CTA per SM drained ~55 GB/s per SM whatever the source).
//
// W producer warps, one thread (or one lane per box) each, issue boxes of
// scattered block ids into S stages of B boxes; a consumer warp per producer
// waits for each of its stages and releases it.  Mode bulk1d: cp.async.bulk of
// the same 4 KiB (no tensor map, no swizzle).  Grid = 148 x C CTAs (C per SM),
// ring bytes per CTA = S*B*4 KiB.  Pool: 32 MiB (L2-resident) or 4 GiB (HBM);
// block ids are a walk of the pool hashed in registers (an id LOAD per stage in
// the issue path would measure its latency, ~0.5 us, not the TMA).  One JSON
// line per configuration.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2504_06319_b200/csrc \
//        tma_box_probe.cu -o tma_box_probe
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "ptx.cuh"

using namespace pda;

constexpr int kBox = 4096;  // 16 rows x 256 B

// Scattered block id of load x: an odd-multiplier hash, a permutation of the
// power-of-two pool (mask, not a modulo: no integer division in the issue path).
__device__ __forceinline__ int block_id(size_t x, int n) { return (int)(((uint32_t)x * 2654435761u) & (uint32_t)(n - 1)); }

__global__ void __launch_bounds__(512) probe(const __grid_constant__ CUtensorMap tm, const uint8_t* __restrict__ src,
                                             int n_ids, int loads_per_cta, int S, int B, int lane_issue, int W,
                                             int mode, unsigned long long* prof) {
    unsigned long long t_wait = 0, t_issue = 0, t0;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* ring = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
    uint64_t* full = reinterpret_cast<uint64_t*>(ring + (size_t)S * B * kBox);
    uint64_t* empty = full + S;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        fence_barrier_init();
    }
    __syncthreads();
    // producer warp w (< W) and consumer warp W + w own loads i = w (mod W),
    // stages s = i mod S (S % W == 0, so stage s always belongs to pair s mod W)
    const size_t base = (size_t)blockIdx.x * loads_per_cta * B;
    const int w = warp % W;
    if (warp < W) {
        int s = w, ph = 0, rot = 0;  // stage, its phase, lane-set rotation (no divisions)
        for (int i = w; i < loads_per_cta; i += W) {
            t0 = clock64();
            if (i >= S) mbar_wait(&empty[s], ph ^ 1);
            const unsigned long long t1 = clock64();
            t_wait += t1 - t0;
            uint8_t* dst = ring + (size_t)s * B * kBox;
            if (lane_issue) {
                if (lane == 0) mbar_arrive_expect_tx(&full[s], B * kBox);
                __syncwarp();
                // lane_issue 2: the issuing lanes rotate over the warp from
                // stage to stage (lane set (i / W) mod (32 / B))
                const int l0 = lane_issue == 2 ? rot : 0;
                if (lane >= l0 && lane < l0 + B) {
                    const int bx = lane - l0;
                    const int blk = block_id(base + (size_t)i * B + bx, n_ids);
                    if (mode == 0)
                        tma_load_3d(dst + bx * kBox, &tm, 0, blk * 16, 0, &full[s]);
                    else
                        bulk_load_1d(dst + bx * kBox, src + (size_t)blk * kBox, kBox, &full[s]);
                }
            } else if (lane == 0) {
                mbar_arrive_expect_tx(&full[s], B * kBox);
                for (int b = 0; b < B; ++b) {
                    const int blk = block_id(base + (size_t)i * B + b, n_ids);
                    if (mode == 0)
                        tma_load_3d(dst + b * kBox, &tm, 0, blk * 16, 0, &full[s]);
                    else
                        bulk_load_1d(dst + b * kBox, src + (size_t)blk * kBox, kBox, &full[s]);
                }
            }
            __syncwarp();
            t_issue += clock64() - t1;
            s += W;
            if (s >= S) {
                s -= S;
                ph ^= 1;
            }
            rot += B;
            if (rot + B > 32) rot = 0;
        }
        if (blockIdx.x == 0 && lane == 0) {
            prof[4 * w] = t_wait;
            prof[4 * w + 1] = t_issue;
        }
    } else if (warp < 2 * W) {
        int s = w, ph = 0;
        for (int i = w; i < loads_per_cta; i += W) {
            t0 = clock64();
            mbar_wait(&full[s], ph);
            t_wait += clock64() - t0;
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
            s += W;
            if (s >= S) {
                s -= S;
                ph ^= 1;
            }
        }
        if (blockIdx.x == 0 && lane == 0) prof[4 * w + 2] = t_wait;
    }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    EncodeFn enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q);
    if (!enc) {
        printf("no encoder\n");
        return 1;
    }
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t hbm_pool = (size_t)4 << 30, l2_pool = (size_t)32 << 20;
    uint8_t* buf;
    if (cudaMalloc(&buf, hbm_pool) != cudaSuccess) return 1;
    cudaMemset(buf, 1, hbm_pool);
    uint8_t* flush;
    cudaMalloc(&flush, (size_t)256 << 20);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    unsigned long long* prof;
    cudaMalloc(&prof, 64 * 8);
    struct Cfg {
        int C, S, B, lane, W, mode;
    };
    // ring 192 KiB per SM throughout; S % W == 0
    // lane: 0 one thread issues the stage, 1 lanes 0..B-1, 2 rotating lane sets
    const Cfg cfgs[] = {{1, 6, 8, 1, 1, 0},  {1, 6, 8, 2, 1, 0},  {1, 2, 24, 1, 1, 0}, {1, 12, 4, 2, 1, 0},
                        {1, 12, 4, 1, 1, 0}, {1, 6, 8, 1, 2, 0},  {1, 12, 4, 1, 4, 0}, {1, 48, 1, 0, 8, 0},
                        {1, 24, 2, 0, 8, 0}, {2, 3, 8, 1, 1, 0},  {3, 8, 2, 0, 4, 0},  {3, 16, 1, 0, 4, 0},
                        {1, 6, 8, 1, 1, 1},  {1, 6, 8, 2, 1, 1},  {1, 3, 16, 1, 1, 0}, {1, 3, 16, 2, 1, 0}};
    const size_t total = (size_t)2 << 30;  // bytes moved per run
    for (int pool_l2 = 1; pool_l2 >= 0; --pool_l2) {
        const size_t pool = pool_l2 ? l2_pool : hbm_pool;
        const int n_blk = (int)(pool / kBox);
        CUtensorMap tm;
        const cuuint64_t dims[3] = {64, (cuuint64_t)n_blk * 16, 2};
        const cuuint64_t strides[2] = {256, 128};
        const cuuint32_t box[3] = {64u, 16u, 2u};
        const cuuint32_t estr[3] = {1, 1, 1};
        if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT16, 3, buf, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
            printf("encode failed\n");
            return 1;
        }
        for (const Cfg& c : cfgs) {
            const int grid = sms * c.C;
            const size_t ring = (size_t)c.S * c.B * kBox;
            const size_t smem = 1024 + ring + 2 * c.S * 8;
            const int loads = (int)(total / ((size_t)grid * c.B * kBox));
            float best = 1e30f;
            for (int rep = 0; rep < 4; ++rep) {
                cudaMemsetAsync(flush, rep, (size_t)256 << 20);
                cudaEvent_t e0, e1;
                cudaEventCreate(&e0);
                cudaEventCreate(&e1);
                cudaEventRecord(e0);
                probe<<<grid, 64 * c.W, smem>>>(tm, buf, n_blk, loads, c.S, c.B, c.lane, c.W, c.mode, prof);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (rep > 0 && ms < best) best = ms;
                cudaEventDestroy(e0);
                cudaEventDestroy(e1);
            }
            const cudaError_t e = cudaGetLastError();
            unsigned long long hp[4] = {0, 0, 0, 0};
            cudaMemcpy(hp, prof, sizeof hp, cudaMemcpyDeviceToHost);
            const int per_warp = (loads + c.W - 1) / c.W;
            const double bytes = (double)grid * loads * c.B * kBox;
            printf("{\"pool\": \"%s\", \"ctas_per_sm\": %d, \"stages\": %d, \"boxes_per_stage\": %d, "
                   "\"lane_issue\": %d, \"producer_warps\": %d, \"mode\": \"%s\", \"ring_kib_per_sm\": %zu, "
                   "\"us\": %.1f, \"gbs\": %.0f, \"gbs_per_sm\": %.1f, \"w0_cycles_per_stage\": {\"prod_wait\": %.0f, \"prod_issue\": %.0f, \"cons_wait\": %.0f}, \"err\": \"%s\"}\n",
                   pool_l2 ? "l2_32MiB" : "hbm_4GiB", c.C, c.S, c.B, c.lane, c.W, c.mode ? "bulk1d" : "tensor3d",
                   ring * c.C / 1024, best * 1e3, bytes / (best * 1e6), bytes / (best * 1e6) / sms,
                   (double)hp[0] / per_warp, (double)hp[1] / per_warp, (double)hp[2] / per_warp, cudaGetErrorString(e));
            fflush(stdout);
        }
    }
    return 0;
}
