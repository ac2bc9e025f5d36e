/*
 * decode_step.c -- one decode-attention step through the C ABI from plain C99
 * (no C++, no PyTorch): include/pda.h + libpda.so + the CUDA runtime.
 *
 *   make example && ./examples/decode_step
 *
 * Two sequences (context 37 and 256 tokens) over a shuffled 16-token block
 * pool, 4 q heads sharing 2 kv heads (GQA), head_dim 64, fp16 -- BASELINE
 * configs[0]'s shape.  Self-check by a closed form, not by recomputing
 * attention: every V row of kv head k equals the same vector c_k, so each
 * output row must equal c_k whatever the softmax weights are (they sum to 1,
 * P:118); the K values are arbitrary.  Exit code 0 on success.
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime_api.h>

#include "pda.h"

enum { B = 2, HQ = 4, HKV = 2, D = 64, BS = 16, MAXB = 16, NBLK = 32 };

/* float -> IEEE fp16 bits for values exactly representable as normal fp16
   (the example only uses multiples of 1/64 in [-1, 1], and 0) */
static uint16_t f2h(float f) {
    uint32_t x;
    memcpy(&x, &f, 4);
    const uint32_t sign = (x >> 16) & 0x8000u;
    const int exp = (int)((x >> 23) & 0xff) - 127 + 15;
    const uint32_t mant = (x >> 13) & 0x3ffu;
    if ((x & 0x7fffffffu) == 0) return (uint16_t)sign;
    return (uint16_t)(sign | ((uint32_t)exp << 10) | mant);
}

static float h2f(uint16_t h) {
    const uint32_t sign = (uint32_t)(h & 0x8000u) << 16;
    const int exp = (h >> 10) & 0x1f;
    const uint32_t mant = h & 0x3ffu;
    uint32_t x;
    float f;
    if (exp == 0) { /* zero or subnormal */
        f = ldexpf((float)mant, -24);
        return (h & 0x8000u) ? -f : f;
    }
    x = sign | ((uint32_t)(exp - 15 + 127) << 23) | (mant << 13);
    memcpy(&f, &x, 4);
    return f;
}

#define CHECK_CUDA(call)                                                              \
    do {                                                                              \
        cudaError_t e_ = (call);                                                      \
        if (e_ != cudaSuccess) {                                                      \
            fprintf(stderr, "%s failed: %s\n", #call, cudaGetErrorString(e_));        \
            return 2;                                                                 \
        }                                                                             \
    } while (0)

int main(void) {
    const int32_t lens[B] = {37, 256};
    const size_t n_q = (size_t)B * HQ * D, n_kv = (size_t)NBLK * HKV * BS * D;
    uint16_t* q = malloc(n_q * 2);
    uint16_t* k = malloc(n_kv * 2);
    uint16_t* v = malloc(n_kv * 2);
    uint16_t* out = malloc(n_q * 2);
    int32_t bt[B * MAXB];
    uint32_t seed = 12345u;
    size_t i;
    int b, h, d, j, used = 0, bad = 0;
    int perm[NBLK];

    for (i = 0; i < n_q; ++i) {
        seed = seed * 1664525u + 1013904223u;
        q[i] = f2h((float)((int)(seed >> 25) - 64) / 64.0f);
    }
    for (i = 0; i < n_kv; ++i) {
        const int dd = (int)(i % D), kvh = (int)((i / ((size_t)BS * D)) % HKV);
        seed = seed * 1664525u + 1013904223u;
        k[i] = f2h((float)((int)(seed >> 25) - 64) / 64.0f);
        v[i] = f2h((float)((dd * 7 + kvh * 13) % 129 - 64) / 64.0f); /* c_kvh[d] */
    }
    /* shuffled physical placement: a seeded Fisher-Yates permutation of the pool */
    for (j = 0; j < NBLK; ++j) perm[j] = j;
    for (j = NBLK - 1; j > 0; --j) {
        int r, t;
        seed = seed * 1664525u + 1013904223u;
        r = (int)((seed >> 8) % (uint32_t)(j + 1));
        t = perm[j];
        perm[j] = perm[r];
        perm[r] = t;
    }
    for (b = 0; b < B; ++b)
        for (j = 0; j < MAXB; ++j) bt[b * MAXB + j] = j < (lens[b] + BS - 1) / BS ? perm[used++] : perm[NBLK - 1];

    {
        pda_shape shape;
        pda_options opt;
        pda_plan_info plan;
        void *dq, *dk, *dv, *dout, *ws = NULL;
        int32_t *dbt, *dlens;
        size_t wsb;
        pda_status st;

        memset(&shape, 0, sizeof shape);
        shape.num_seqs = B;
        shape.num_q_heads = HQ;
        shape.num_kv_heads = HKV;
        shape.head_dim = D;
        shape.block_size = BS;
        shape.num_blocks = NBLK;
        shape.max_blocks_per_seq = MAXB;
        shape.dtype = PDA_F16;
        shape.out_dtype = PDA_F16;
        shape.kv_dtype = PDA_F16;
        shape.q_len = 1;
        memset(&opt, 0, sizeof opt); /* all defaults: split-K, planner's partitions, prefetch off */

        st = pda_plan(&shape, &opt, &plan);
        if (st != PDA_OK) {
            fprintf(stderr, "pda_plan: %s\n", pda_status_string(st));
            return 1;
        }
        wsb = pda_workspace_bytes(&shape, &opt);
        printf("plan: kernel %d, P = %d tokens, P_max %d, grid (%d, %d, %d), %d threads, %d stages, "
               "workspace %zu B\n", plan.kernel, plan.partition_tokens, plan.p_max, plan.grid_x, plan.grid_y,
               plan.grid_z, plan.threads, plan.smem_stages, wsb);

        CHECK_CUDA(cudaMalloc(&dq, n_q * 2));
        CHECK_CUDA(cudaMalloc(&dk, n_kv * 2));
        CHECK_CUDA(cudaMalloc(&dv, n_kv * 2));
        CHECK_CUDA(cudaMalloc(&dout, n_q * 2));
        CHECK_CUDA(cudaMalloc((void**)&dbt, sizeof bt));
        CHECK_CUDA(cudaMalloc((void**)&dlens, sizeof lens));
        if (wsb) CHECK_CUDA(cudaMalloc(&ws, wsb));
        CHECK_CUDA(cudaMemcpy(dq, q, n_q * 2, cudaMemcpyHostToDevice));
        CHECK_CUDA(cudaMemcpy(dk, k, n_kv * 2, cudaMemcpyHostToDevice));
        CHECK_CUDA(cudaMemcpy(dv, v, n_kv * 2, cudaMemcpyHostToDevice));
        CHECK_CUDA(cudaMemcpy(dbt, bt, sizeof bt, cudaMemcpyHostToDevice));
        CHECK_CUDA(cudaMemcpy(dlens, lens, sizeof lens, cudaMemcpyHostToDevice));

        st = paged_decode_attention(dq, dk, dv, dbt, dlens, 0.125f, dout, &shape, &opt, ws, wsb, NULL);
        if (st != PDA_OK) {
            fprintf(stderr, "paged_decode_attention: %s\n", pda_status_string(st));
            return 1;
        }
        CHECK_CUDA(cudaMemcpy(out, dout, n_q * 2, cudaMemcpyDeviceToHost));
        cudaFree(dq);
        cudaFree(dk);
        cudaFree(dv);
        cudaFree(dout);
        cudaFree(dbt);
        cudaFree(dlens);
        if (ws) cudaFree(ws);
    }

    for (b = 0; b < B; ++b)
        for (h = 0; h < HQ; ++h)
            for (d = 0; d < D; ++d) {
                const int kvh = h / (HQ / HKV);
                const float want = (float)((d * 7 + kvh * 13) % 129 - 64) / 64.0f;
                const float got = h2f(out[((size_t)b * HQ + h) * D + d]);
                if (!(fabsf(got - want) <= 2e-3f)) ++bad;
            }
    printf("out[0,0,0:4] = %.4f %.4f %.4f %.4f; %d of %d outputs off the closed form\n", h2f(out[0]),
           h2f(out[1]), h2f(out[2]), h2f(out[3]), bad, B * HQ * D);
    free(q);
    free(k);
    free(v);
    free(out);
    return bad == 0 ? 0 : 1;
}
