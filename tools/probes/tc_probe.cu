// tc_probe.cu -- checks the tcgen05 operand layouts the tc decode kernel uses,
// on one CTA with data written by threads (no TMA), against a host reference:
//   S^T[t][h] = sum_d K[t][d] Q[h][d]   M=128 tokens, N=16, K-major A (K tile,
//              [chunk][token][128 B], SW128) and B (Q, [chunk][row][128 B], SW128)
//   O^T[d][c] = sum_t V[t][d] P[t][c]   M=128 (d), N=32, K=16 per block:
//              A = V slab, MN-major SW128 ([chunk][token][128 B], TMA's 3-D box
//              layout); B = P, MN-major no-swizzle core matrices
// TMEM read back with tcgen05.ld.32x32b (thread = lane).
//   nvcc -gencode arch=compute_100a,code=sm_100a -I../../paper_2504_06319_b200/csrc tc_probe.cu -o tc_probe
#include <cuda_bf16.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "tc_ptx.cuh"

using namespace pda;

constexpr int D = 128, T = 128, NQ = 16, NP = 32;
constexpr int KT_BYTES = 2 * T * 128;           // K tile: 2 chunks x 128 rows x 128 B
constexpr int Q_BYTES = 2 * NQ * 128;           // Q: 2 chunks x 16 rows x 128 B
constexpr int V_BYTES = (T / 16) * 4096;        // 8 slabs of [2][16][128 B]
constexpr int P_BYTES = T * NP * 2;             // [k group 16][mn group 4] core matrices of 128 B
constexpr int P_LBO = 128, P_SBO = (T / 8) * 128;

__device__ __forceinline__ uint32_t sw(int row, int byte) {  // 128-B swizzle inside a [rows][128 B] chunk
    return row * 128 + ((((byte >> 4) ^ (row & 7)) & 7) << 4) + (byte & 15);
}

__global__ void probe(const __nv_bfloat16* K, const __nv_bfloat16* Q, const __nv_bfloat16* V,
                      const __nv_bfloat16* P, float* S_out, float* O_out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* sm = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
    uint8_t* kt = sm;
    uint8_t* qs = kt + KT_BYTES;
    uint8_t* vs = qs + Q_BYTES;
    uint8_t* ps = vs + V_BYTES;
    uint64_t* bar = reinterpret_cast<uint64_t*>(ps + P_BYTES);
    uint32_t* tbase = reinterpret_cast<uint32_t*>(bar + 1);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // K tile: token t, d -> chunk d/64, row t
    for (int i = tid; i < T * D; i += blockDim.x) {
        const int t = i / D, d = i % D;
        *reinterpret_cast<__nv_bfloat16*>(kt + (d / 64) * (T * 128) + sw(t, (d % 64) * 2)) = K[i];
        *reinterpret_cast<__nv_bfloat16*>(vs + (t / 16) * 4096 + (d / 64) * 2048 + sw(t % 16, (d % 64) * 2)) = V[i];
    }
    for (int i = tid; i < NQ * D; i += blockDim.x) {
        const int h = i / D, d = i % D;
        *reinterpret_cast<__nv_bfloat16*>(qs + (d / 64) * (NQ * 128) + sw(h, (d % 64) * 2)) = Q[i];
    }
    for (int i = tid; i < T * NP; i += blockDim.x) {
        const int t = i / NP, c = i % NP;
        *reinterpret_cast<__nv_bfloat16*>(ps + (t % 8) * 16 + (t / 8) * P_LBO + (c % 8) * 2 + (c / 8) * P_SBO) = P[i];
    }
    if (tid == 0) {
        mbar_init(bar, 1);
        fence_barrier_init();
    }
    if (warp == 0) tc::alloc<64>(tbase);
    tc::fence_async_smem();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tm = *tbase;
    if (tid == 0) {
        const uint32_t idq = tc::idesc_f16(true, 128, NQ, false, false);
        for (int j = 0; j < D / 16; ++j) {
            const uint64_t a = tc::smem_desc(smem_u32(kt) + (j / 4) * (T * 128) + (j % 4) * 32, 16, 1024, tc::kLayoutSw128);
            const uint64_t b = tc::smem_desc(smem_u32(qs) + (j / 4) * (NQ * 128) + (j % 4) * 32, 16, 1024, tc::kLayoutSw128);
            tc::mma_f16_ss(tm, a, b, idq, j > 0);
        }
        const uint32_t idp = tc::idesc_f16(true, 128, NP, true, true);
        for (int blk = 0; blk < T / 16; ++blk) {
            const uint64_t a = tc::smem_desc(smem_u32(vs) + blk * 4096, 2048, 1024, tc::kLayoutSw128);
            const uint64_t b = tc::smem_desc(smem_u32(ps) + blk * 2 * P_LBO, P_LBO, P_SBO, tc::kLayoutInterleave);
            tc::mma_f16_ss(tm + 32, a, b, idp, blk > 0);
        }
        tc::commit(bar);
    }
    mbar_wait(bar, 0);
    tc::fence_after();
    uint32_t r[16];
    const uint32_t lane_addr = (uint32_t)(warp * 32) << 16;
    tc::ld_32x32b_x16(tm + lane_addr, r);
    tc::wait_ld();
    for (int c = 0; c < 16; ++c) S_out[(warp * 32 + lane) * NQ + c] = __uint_as_float(r[c]);
    for (int half = 0; half < 2; ++half) {
        tc::ld_32x32b_x16(tm + lane_addr + 32 + 16 * half, r);
        tc::wait_ld();
        for (int c = 0; c < 16; ++c) O_out[(warp * 32 + lane) * NP + 16 * half + c] = __uint_as_float(r[c]);
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::dealloc<64>(tm);
}

int main() {
    std::vector<__nv_bfloat16> K(T * D), Q(NQ * D), V(T * D), P(T * NP);
    std::vector<float> Kf(T * D), Qf(NQ * D), Vf(T * D), Pf(T * NP);
    srand(1);
    auto rnd = [] { return (float)rand() / RAND_MAX * 2.f - 1.f; };
    for (int i = 0; i < T * D; ++i) { K[i] = __float2bfloat16(rnd()); Kf[i] = __bfloat162float(K[i]); }
    for (int i = 0; i < T * D; ++i) { V[i] = __float2bfloat16(rnd()); Vf[i] = __bfloat162float(V[i]); }
    for (int i = 0; i < NQ * D; ++i) { Q[i] = __float2bfloat16(rnd()); Qf[i] = __bfloat162float(Q[i]); }
    for (int i = 0; i < T * NP; ++i) { P[i] = __float2bfloat16(rnd()); Pf[i] = __bfloat162float(P[i]); }
    __nv_bfloat16 *dK, *dQ, *dV, *dP;
    float *dS, *dO;
    cudaMalloc(&dK, T * D * 2); cudaMalloc(&dQ, NQ * D * 2); cudaMalloc(&dV, T * D * 2); cudaMalloc(&dP, T * NP * 2);
    cudaMalloc(&dS, T * NQ * 4); cudaMalloc(&dO, D * NP * 4);
    cudaMemcpy(dK, K.data(), T * D * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dQ, Q.data(), NQ * D * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dV, V.data(), T * D * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dP, P.data(), T * NP * 2, cudaMemcpyHostToDevice);
    const int smem = 1024 + KT_BYTES + Q_BYTES + V_BYTES + P_BYTES + 64;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    probe<<<1, 128, smem>>>(dK, dQ, dV, dP, dS, dO);
    cudaError_t e = cudaDeviceSynchronize();
    printf("kernel: %s\n", cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
    std::vector<float> S(T * NQ), O(D * NP);
    cudaMemcpy(S.data(), dS, T * NQ * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(O.data(), dO, D * NP * 4, cudaMemcpyDeviceToHost);
    double es = 0, eo = 0;
    int bad = 0;
    for (int t = 0; t < T; ++t)
        for (int h = 0; h < NQ; ++h) {
            double ref = 0;
            for (int d = 0; d < D; ++d) ref += (double)Kf[t * D + d] * Qf[h * D + d];
            const double err = fabs(ref - S[t * NQ + h]);
            es = fmax(es, err);
            if (err > 1e-2 && bad++ < 8) printf("S[%d][%d] = %f ref %f\n", t, h, S[t * NQ + h], ref);
        }
    for (int d = 0; d < D; ++d)
        for (int c = 0; c < NP; ++c) {
            double ref = 0;
            for (int t = 0; t < T; ++t) ref += (double)Vf[t * D + d] * Pf[t * NP + c];
            const double err = fabs(ref - O[d * NP + c]);
            eo = fmax(eo, err);
            if (err > 1e-2 && bad++ < 16) printf("O[%d][%d] = %f ref %f\n", d, c, O[d * NP + c], ref);
        }
    printf("max err S %.3g  O %.3g  -> %s\n", es, eo, (es < 1e-3 && eo < 1e-3) ? "PASS" : "FAIL");
    return (es < 1e-3 && eo < 1e-3) ? 0 : 2;
}
