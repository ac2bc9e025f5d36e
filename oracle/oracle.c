/*
 * oracle/oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct fp64 CPU implementation of what the
 * paper's hot path computes: single-query (decode) attention over a paged
 * KV cache, plus the block/prefetch bookkeeping of Algorithm 1.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  The product path
 * (paper_2504_06319_b200/) never includes, links or calls anything here, and
 * this file includes nothing from the product (no shared headers, tables or
 * helpers).  The trace record layout below is restated independently from
 * the documentation in include/pda.h, not included from it.
 *
 * Citations: P:n = /root/reference/PAPER.md line n (read at build time only).
 *
 * Parity pins (tests/test_oracle.py, `-m "not gpu"`):
 *   oracle_paged_attention   pinned: brute force vs numpy/torch fp64 SDPA on
 *                            contiguous gathers, permutation invariance,
 *                            L=1 -> V row, q=0 -> mean(V), const V -> v,
 *                            needle, sum of weights = 1.
 *   oracle_attention_weights pinned: sums to 1, matches numpy softmax.
 *   oracle_fp16/bf16_to_f64  pinned: numpy float16 / torch bfloat16 decode.
 *   oracle_e4m3_to_f64       pinned: torch float8_e4m3fn decode, all 256 codes.
 *   oracle_paged_attention_kv8 pinned: numpy softmax attention on the
 *                            dequantised contiguous gather, closed forms.
 *   oracle_paged_attention_mq pinned: numpy causal attention on contiguous
 *                            gathers (explicit causal mask), q_len = 1 ==
 *                            oracle_paged_attention bitwise.
 *   oracle_plan_splitk       pinned: hand-computed ranges, Alg. 1 guard
 *                            counts, brute-force plan.
 *   oracle_plan_paper        pinned: Alg. 1 guard counts, hand examples.
 *   oracle_eq1/eq2/l2_bound  pinned: 4096 B, 524288 B, 120.
 *   oracle_validate_inputs   pinned: hand-built tables with known counts,
 *                            brute-force recount by perturbation.
 *   oracle_e4m3_encode       pinned: torch float8_e4m3fn cast (in range),
 *                            encode(decode(c)) == c for every finite code,
 *                            exact midpoints (ties to even), saturation.
 *   oracle_kv_append(_e4m3)  pinned: positions by hand (block / slot of the
 *                            last tokens), untouched bytes elsewhere, e4m3
 *                            rows vs the torch cast of x / scale.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_F16 0
#define ORACLE_BF16 1

/* IEEE 754 binary16 -> double, written from the format definition
 * (1 sign bit, 5 exponent bits with bias 15, 10 fraction bits). */
double oracle_fp16_to_f64(uint16_t h) {
    int sign = (h >> 15) & 1;
    int exp = (h >> 10) & 0x1f;
    int frac = h & 0x3ff;
    double v;
    if (exp == 0) {
        v = ldexp((double)frac, -24); /* subnormal: frac * 2^-14 * 2^-10 */
    } else if (exp == 31) {
        v = frac ? NAN : INFINITY;
    } else {
        v = ldexp((double)(frac + 1024), exp - 25); /* (1 + f/1024) * 2^(e-15) */
    }
    return sign ? -v : v;
}

/* bfloat16 -> double: bfloat16 is the upper 16 bits of an IEEE binary32
 * (1 sign bit, 8 exponent bits with bias 127, 7 fraction bits). */
double oracle_bf16_to_f64(uint16_t h) {
    int sign = (h >> 15) & 1;
    int exp = (h >> 7) & 0xff;
    int frac = h & 0x7f;
    double v;
    if (exp == 0) {
        v = ldexp((double)frac, -133); /* frac * 2^-126 * 2^-7 */
    } else if (exp == 255) {
        v = frac ? NAN : INFINITY;
    } else {
        v = ldexp((double)(frac + 128), exp - 134); /* (1 + f/128) * 2^(e-127) */
    }
    return sign ? -v : v;
}

/* OCP FP8 E4M3 (the "e4m3fn" encoding) -> double, from the format definition:
 * 1 sign bit, 4 exponent bits with bias 7, 3 fraction bits; no infinities,
 * S.1111.111 is NaN; max finite 448. */
double oracle_e4m3_to_f64(uint8_t x) {
    int sign = (x >> 7) & 1;
    int exp = (x >> 3) & 0xf;
    int frac = x & 0x7;
    double v;
    if (exp == 15 && frac == 7) {
        v = NAN;
    } else if (exp == 0) {
        v = ldexp((double)frac, -9); /* subnormal: frac/8 * 2^-6 */
    } else {
        v = ldexp((double)(frac + 8), exp - 10); /* (1 + f/8) * 2^(e-7) */
    }
    return sign ? -v : v;
}

static double decode(uint16_t x, int dtype) {
    return dtype == ORACLE_BF16 ? oracle_bf16_to_f64(x) : oracle_fp16_to_f64(x);
}

/* Offset of element d of token slot o of (physical block phys, kv head kvh)
 * in a [num_blocks, Hkv, bs, D] cache.  Layout reading R2 of DESIGN.md: each
 * (block, head) slab is contiguous, "each block exclusively stores KV Cache
 * data for a single attention head" (Section 3.1). */
static size_t kv_offset(int64_t phys, int kvh, int o, int d, int Hkv, int bs, int D) {
    return (((size_t)phys * Hkv + kvh) * bs + o) * D + d;
}

/* Score s_t of token t for row (b, h), as the plain definition
 * s_t = scale * sum_d q[b,h,d] * k_t[d]   (QK^T, Alg. 1 line 9 P:136). */
static double score(const uint16_t* q, const uint16_t* k, int dtype, const int32_t* bt,
                    int b, int h, int kvh, int t, int Hq, int Hkv, int D, int bs,
                    int max_blocks, double scale) {
    int j = t / bs, o = t % bs;
    int64_t phys = bt[(size_t)b * max_blocks + j]; /* bt lookup, Alg. 1 */
    double acc = 0.0;
    for (int d = 0; d < D; ++d) {
        double qd = decode(q[((size_t)b * Hq + h) * D + d], dtype);
        double kd = decode(k[kv_offset(phys, kvh, o, d, Hkv, bs, D)], dtype);
        acc += qd * kd;
    }
    return scale * acc;
}

/* Softmax weights w_t / Z of one row (b, h) over its L = lens[b] tokens.
 * Writes L doubles to w.  Returns L (0 => nothing written). */
int oracle_attention_weights(const uint16_t* q, const uint16_t* k, int dtype,
                             const int32_t* bt, const int32_t* lens, int b, int h,
                             int Hq, int Hkv, int D, int bs, int max_blocks, double scale,
                             double* w) {
    int g = Hq / Hkv;
    int kvh = h / g; /* GQA: q head h reads kv head floor(h / g) */
    int L = lens[b];
    if (L <= 0) return 0;
    double m = -INFINITY;
    for (int t = 0; t < L; ++t) {
        w[t] = score(q, k, dtype, bt, b, h, kvh, t, Hq, Hkv, D, bs, max_blocks, scale);
        if (w[t] > m) m = w[t];
    }
    double Z = 0.0;
    for (int t = 0; t < L; ++t) {
        w[t] = exp(w[t] - m);
        Z += w[t];
    }
    for (int t = 0; t < L; ++t) w[t] /= Z;
    return L;
}

/* One output row: out[b,h,:] = sum_t softmax(s)_t * v_t  ("logits . V").
 * L = 0 gives a zero row (reading R6). */
static void attend_row(const uint16_t* q, const uint16_t* k, const uint16_t* v, int dtype,
                       const int32_t* bt, const int32_t* lens, int b, int h, int Hq, int Hkv,
                       int D, int bs, int max_blocks, double scale, double* w, double* out_row) {
    int g = Hq / Hkv;
    int kvh = h / g;
    for (int d = 0; d < D; ++d) out_row[d] = 0.0;
    int L = oracle_attention_weights(q, k, dtype, bt, lens, b, h, Hq, Hkv, D, bs, max_blocks,
                                     scale, w);
    for (int t = 0; t < L; ++t) {
        int64_t phys = bt[(size_t)b * max_blocks + t / bs];
        int o = t % bs;
        for (int d = 0; d < D; ++d)
            out_row[d] += w[t] * decode(v[kv_offset(phys, kvh, o, d, Hkv, bs, D)], dtype);
    }
}

/* Paged decode attention, fp64.  q: [B, Hq, D]; k, v: [num_blocks, Hkv, bs, D]
 * (raw 16-bit patterns of dtype); bt: [B, max_blocks]; lens: [B]; out: [B, Hq, D].
 * rows: optional list of n_rows row ids r = b * Hq + h to compute (NULL = all);
 * rows not listed are left untouched.  nthreads <= 0: OpenMP default.
 * Returns 0, or -1 on invalid arguments. */
int oracle_paged_attention(const uint16_t* q, const uint16_t* k, const uint16_t* v, int dtype,
                           const int32_t* bt, const int32_t* lens, int B, int Hq, int Hkv,
                           int D, int bs, int max_blocks, double scale, double* out,
                           const int64_t* rows, int64_t n_rows, int nthreads) {
    if (B < 0 || Hq <= 0 || Hkv <= 0 || Hq % Hkv || D <= 0 || bs <= 0 || max_blocks < 0) return -1;
    int64_t total = rows ? n_rows : (int64_t)B * Hq;
    int Lmax = max_blocks * bs;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel
#endif
    {
        double* w = (double*)malloc(sizeof(double) * (Lmax > 0 ? Lmax : 1));
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 1)
#endif
        for (int64_t i = 0; i < total; ++i) {
            int64_t r = rows ? rows[i] : i;
            int b = (int)(r / Hq), h = (int)(r % Hq);
            attend_row(q, k, v, dtype, bt, lens, b, h, Hq, Hkv, D, bs, max_blocks, scale, w,
                       out + (size_t)r * D);
        }
        free(w);
    }
    return 0;
}

/* FP8 KV cache variant: K and V stored as e4m3 codes with
 * per-tensor scales, k_t = k_scale * e4m3(K[...]), v_t = v_scale * e4m3(V[...]);
 * q in fp16/bf16 (q_dtype).  Same plain definition as oracle_paged_attention
 * on the dequantised values:
 *   s_t = scale * sum_d q[b,h,d] * k_t[d];  out = sum_t softmax(s)_t * v_t. */
int oracle_paged_attention_kv8(const uint16_t* q, int q_dtype, const uint8_t* k, const uint8_t* v,
                               double k_scale, double v_scale, const int32_t* bt,
                               const int32_t* lens, int B, int Hq, int Hkv, int D, int bs,
                               int max_blocks, double scale, double* out, const int64_t* rows,
                               int64_t n_rows, int nthreads) {
    if (B < 0 || Hq <= 0 || Hkv <= 0 || Hq % Hkv || D <= 0 || bs <= 0 || max_blocks < 0) return -1;
    int64_t total = rows ? n_rows : (int64_t)B * Hq;
    int Lmax = max_blocks * bs;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel
#endif
    {
        double* w = (double*)malloc(sizeof(double) * (Lmax > 0 ? Lmax : 1));
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 1)
#endif
        for (int64_t i = 0; i < total; ++i) {
            int64_t r = rows ? rows[i] : i;
            int b = (int)(r / Hq), h = (int)(r % Hq);
            int kvh = h / (Hq / Hkv);
            int L = lens[b];
            double* o = out + (size_t)r * D;
            for (int d = 0; d < D; ++d) o[d] = 0.0;
            if (L <= 0) continue;
            double m = -INFINITY;
            for (int t = 0; t < L; ++t) {
                int64_t phys = bt[(size_t)b * max_blocks + t / bs];
                double acc = 0.0;
                for (int d = 0; d < D; ++d)
                    acc += decode(q[((size_t)b * Hq + h) * D + d], q_dtype) *
                           (k_scale * oracle_e4m3_to_f64(k[kv_offset(phys, kvh, t % bs, d, Hkv, bs, D)]));
                w[t] = scale * acc;
                if (w[t] > m) m = w[t];
            }
            double Z = 0.0;
            for (int t = 0; t < L; ++t) {
                w[t] = exp(w[t] - m);
                Z += w[t];
            }
            for (int t = 0; t < L; ++t) {
                int64_t phys = bt[(size_t)b * max_blocks + t / bs];
                for (int d = 0; d < D; ++d)
                    o[d] += (w[t] / Z) *
                            (v_scale * oracle_e4m3_to_f64(v[kv_offset(phys, kvh, t % bs, d, Hkv, bs, D)]));
            }
        }
        free(w);
    }
    return 0;
}

/* Multi-token (speculative) decode: q_len query tokens per
 * sequence, q [B, q_len, Hq, D] -> out [B, q_len, Hq, D].  context_lens[b] = L
 * counts the q_len new tokens, whose K/V are already in the cache; query token
 * i sits at position L - q_len + i and attends causally to tokens
 * [0, L - q_len + i], i.e. it is the single-query definition with context
 * length L_i = L - q_len + i + 1 (L_i <= 0 gives a zero row).  This function
 * evaluates exactly that: for each (b, i) it calls the single-query
 * definition on the sequence truncated to L_i. */
int oracle_paged_attention_mq(const uint16_t* q, const uint16_t* k, const uint16_t* v, int dtype,
                              const int32_t* bt, const int32_t* lens, int B, int q_len, int Hq,
                              int Hkv, int D, int bs, int max_blocks, double scale, double* out,
                              int nthreads) {
    if (q_len <= 0) return -1;
    int32_t* li = (int32_t*)malloc(sizeof(int32_t) * (B > 0 ? B : 1));
    int32_t* bti = (int32_t*)malloc(sizeof(int32_t) * (size_t)(B > 0 ? B : 1) * (max_blocks > 0 ? max_blocks : 1));
    uint16_t* qi = (uint16_t*)malloc(sizeof(uint16_t) * (size_t)(B > 0 ? B : 1) * Hq * D);
    double* oi = (double*)malloc(sizeof(double) * (size_t)(B > 0 ? B : 1) * Hq * D);
    int rc = 0;
    for (int i = 0; i < q_len && rc == 0; ++i) {
        for (int b = 0; b < B; ++b) {
            int L = lens[b] - q_len + i + 1;
            li[b] = L > 0 ? L : 0;
            for (int j = 0; j < max_blocks; ++j) bti[(size_t)b * max_blocks + j] = bt[(size_t)b * max_blocks + j];
            memcpy(qi + (size_t)b * Hq * D, q + (((size_t)b * q_len + i) * Hq) * D, sizeof(uint16_t) * Hq * D);
        }
        rc = oracle_paged_attention(qi, k, v, dtype, bti, li, B, Hq, Hkv, D, bs, max_blocks, scale, oi,
                                    NULL, 0, nthreads);
        for (int b = 0; b < B; ++b)
            memcpy(out + (((size_t)b * q_len + i) * Hq) * D, oi + (size_t)b * Hq * D, sizeof(double) * Hq * D);
    }
    free(li);
    free(bti);
    free(qi);
    free(oi);
    return rc;
}

int oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ---------------------------------------------------------------------------
 * Bookkeeping plans (bit-exact targets for the GPU debug trace).
 *
 * Record layout, restated from the library documentation (include/pda.h):
 *   rec[0] = s, rec[1] = e     (split-K: token range [s, e) of the unit;
 *                               paper kernel: first block index, block end e)
 *   rec[2] = number of visited blocks, rec[3] = number of prefetches,
 *   rec[4 .. 4+R)   visited physical block ids in visit order, rest -1,
 *   rec[4+R .. 4+2R) prefetch target physical ids in issue order, rest -1.
 * ------------------------------------------------------------------------- */

/* Split-K plan.  Units u = ((b * Hkv) + kvh) * P_max + p, partition size
 * P tokens (multiple of bs), R = P / bs.  The unit's blocks are
 * [s/bs, ceil(e/bs)); each is visited in order j = s/bs, s/bs+1, ...; when
 * block j is issued, block j + d is prefetched iff j + d < e_blk
 * (Alg. 1 guard "block_idx + w < e", with the stride w replaced by the
 * distance knob d because one producer issues the blocks in order; reading R8/R9).
 * d <= 0 means prefetch off. */
int oracle_plan_splitk(const int32_t* bt, const int32_t* lens, int B, int Hkv, int bs,
                       int max_blocks, int P, int P_max, int d, int32_t* recs) {
    if (P <= 0 || P % bs) return -1;
    int R = P / bs;
    int rec_len = 4 + 2 * R;
    for (int b = 0; b < B; ++b) {
        int L = lens[b];
        for (int kvh = 0; kvh < Hkv; ++kvh) {
            for (int p = 0; p < P_max; ++p) {
                int32_t* rec = recs + ((size_t)(b * Hkv + kvh) * P_max + p) * rec_len;
                for (int i = 0; i < rec_len; ++i) rec[i] = -1;
                int s = p * P < L ? p * P : L;
                int e = (p + 1) * P < L ? (p + 1) * P : L;
                rec[0] = s;
                rec[1] = e;
                int sb = s / bs, eb = e > s ? (e + bs - 1) / bs : sb; /* empty unit: no blocks */
                int nv = 0, np = 0;
                for (int j = sb; j < eb; ++j) {
                    rec[4 + nv++] = bt[(size_t)b * max_blocks + j];
                    if (d > 0 && j + d < eb) rec[4 + R + np++] = bt[(size_t)b * max_blocks + j + d];
                }
                rec[2] = nv;
                rec[3] = np;
            }
        }
    }
    return 0;
}

/* Paper-kernel plan (Section 3.1, Alg. 1): one CTA per (q head h, seq b)
 * (grid [H, B, 1]), w warps; warp i starts at block_idx = i and strides
 * by w; while on block_idx it prefetches bt[block_idx + d]
 * iff block_idx + d < e (Alg. 1 lines 4-7 with w -> d; d = w is the paper).
 * Records per (b, h, warp) = ((b * Hq) + h) * w + warp, R = ceil(max_blocks / w). */
int oracle_plan_paper(const int32_t* bt, const int32_t* lens, int B, int Hq, int bs,
                      int max_blocks, int w, int d, int32_t* recs) {
    if (w <= 0) return -1;
    int R = (max_blocks + w - 1) / w;
    int rec_len = 4 + 2 * R;
    for (int b = 0; b < B; ++b) {
        int e = (lens[b] + bs - 1) / bs; /* blocks of the sequence */
        for (int h = 0; h < Hq; ++h) {
            for (int wi = 0; wi < w; ++wi) {
                int32_t* rec = recs + ((size_t)(b * Hq + h) * w + wi) * rec_len;
                for (int i = 0; i < rec_len; ++i) rec[i] = -1;
                rec[0] = wi;
                rec[1] = e;
                int nv = 0, np = 0;
                for (int idx = wi; idx < e; idx += w) {
                    rec[4 + nv++] = bt[(size_t)b * max_blocks + idx];
                    if (d > 0 && idx + d < e) rec[4 + R + np++] = bt[(size_t)b * max_blocks + idx + d];
                }
                rec[2] = nv;
                rec[3] = np;
            }
        }
    }
    return 0;
}

/* Stream-kernel plan: all blocks of the step in one ordered item list (rows
 * (b, kvh) in order, each row's blocks j = 0..n_b-1), T items split into
 * NS = min(NS_max, T) contiguous ranges [floor(s*T/NS), floor((s+1)*T/NS)).
 * A segment is the part of a row inside one range; block j of a segment is
 * prefetched-for (target j + d) iff j + d is inside the same segment (the
 * Alg. 1 guard against the unit's end, reading R9).  Records per row
 * r = b * Hkv + kvh, R = max_blocks: visited[j] and target[j] indexed by j.
 * Rows with L = 0 have no blocks and stay all -1. */
int oracle_plan_stream(const int32_t* bt, const int32_t* lens, int B, int Hkv, int bs,
                       int max_blocks, int NS_max, int d, int32_t* recs) {
    int R = max_blocks;
    int rec_len = 4 + 2 * R;
    long long T = 0;
    for (int b = 0; b < B; ++b) {
        int L = lens[b] < max_blocks * bs ? lens[b] : max_blocks * bs;
        if (L > 0) T += (long long)((L + bs - 1) / bs) * Hkv;
    }
    long long NS = T < NS_max ? T : NS_max;
    long long item = 0;
    long long sigma = 0;
    for (int b = 0; b < B; ++b) {
        int L = lens[b] < max_blocks * bs ? lens[b] : max_blocks * bs;
        int n = L > 0 ? (L + bs - 1) / bs : 0;
        for (int kvh = 0; kvh < Hkv; ++kvh) {
            int32_t* rec = recs + ((size_t)b * Hkv + kvh) * rec_len;
            for (int i = 0; i < rec_len; ++i) rec[i] = -1;
            if (n == 0) continue;
            rec[0] = 0;
            rec[1] = L;
            rec[2] = n;
            int np = 0;
            long long row_start = item;
            for (int j = 0; j < n; ++j, ++item) {
                while ((sigma + 1) * T / NS <= item) ++sigma; /* range holding this item */
                long long range_end = (sigma + 1) * T / NS;
                long long seg_end = row_start + n < range_end ? row_start + n : range_end;
                rec[4 + j] = bt[(size_t)b * max_blocks + j];
                if (d > 0 && item + d < seg_end) {
                    rec[4 + R + j] = bt[(size_t)b * max_blocks + j + d];
                    ++np;
                }
            }
            rec[3] = np;
        }
    }
    return 0;
}

/* Eq. 1: M_block = b * d_h * T_block bytes. */
int64_t oracle_eq1_block_bytes(int64_t b, int64_t d_h, int64_t T_block) { return b * d_h * T_block; }

/* Eq. 2: M_total = M_block * (N_thread / 32) * H * B. */
int64_t oracle_eq2_total_bytes(int64_t M_block, int64_t N_thread, int64_t H, int64_t B) {
    return M_block * (N_thread / 32) * H * B;
}

/* L2 residency bound: the largest batch whose per-iteration blocks
 * fit in L2, floor(L2 / M_total(B=1)). */
int64_t oracle_l2_residency_bound(int64_t l2_bytes, int64_t M_total_b1) { return l2_bytes / M_total_b1; }

/* ---------------------------------------------------------------------------
 * Device-data validation (SURVEY 8b convention: "a debug validate kernel flags
 * out-of-range block ids and lengths").  Plain definition: sequence b is
 * valid iff 0 <= L_b <= max_blocks * bs and every block id it references,
 * bt[b][j] for j < ceil(L_b / bs), lies in [0, num_blocks) (the paged
 * lookup of P:105 / Alg. 1 line 3, must land inside the pool).  Ids of
 * a sequence with an invalid length are checked over min(L_b, max) tokens.
 * counts[0] = sequences with an invalid length, counts[1] = referenced block
 * ids out of range, counts[2] = sequences with either problem.
 * ------------------------------------------------------------------------- */
int oracle_validate_inputs(const int32_t* bt, const int32_t* lens, int B, int max_blocks, int bs,
                           int64_t num_blocks, int64_t* counts) {
    counts[0] = counts[1] = counts[2] = 0;
    for (int b = 0; b < B; ++b) {
        int64_t L = lens[b];
        int bad_len = L < 0 || L > (int64_t)max_blocks * bs;
        if (L < 0) L = 0;
        if (L > (int64_t)max_blocks * bs) L = (int64_t)max_blocks * bs;
        int64_t bad_ids = 0;
        for (int64_t j = 0; j < (L + bs - 1) / bs; ++j) {
            int32_t id = bt[(size_t)b * max_blocks + j];
            if (id < 0 || id >= num_blocks) ++bad_ids;
        }
        counts[0] += bad_len;
        counts[1] += bad_ids;
        counts[2] += (bad_len || bad_ids) ? 1 : 0;
    }
    return 0;
}

/* fp32 -> OCP FP8 E4M3 code, round to nearest, ties to the even code, values
 * beyond the largest finite magnitude saturate to +-448, NaN -> 0x7F.  Written
 * as the definition: the nearest of the 127 finite magnitudes (by brute force
 * over the codes, decoded with oracle_e4m3_to_f64), sign copied. */
uint8_t oracle_e4m3_encode(float x) {
    if (isnan(x)) return 0x7F;
    uint8_t sign = signbit(x) ? 0x80 : 0;
    double a = fabs((double)x);
    int best = 0;
    double bd = INFINITY;
    for (int c = 0; c <= 0x7E; ++c) {
        double dist = fabs(oracle_e4m3_to_f64((uint8_t)c) - a);
        if (dist < bd || (dist == bd && (c & 1) == 0)) {
            best = c;
            bd = dist;
        }
    }
    return (uint8_t)(sign | best);
}

/* KV append (the decode step's cache write, "each decoding step" adds one
 * token's K/V; paged layout P:105): new K/V rows k_new, v_new [B, q_len, Hkv, D]
 * of token i of sequence b go to position t = L_b - q_len + i (L_b counts the
 * new tokens, as in oracle_paged_attention_mq), i.e. slot t % bs of physical
 * block bt[b][t / bs], for every kv head; positions t < 0 are skipped.
 * 16-bit caches: the bit patterns are copied.  kv8 != 0: the caches hold
 * e4m3 codes, code = e4m3(fp32(x) / fp32(scale)) with an IEEE fp32 division
 * (the quantisation decision taken in fp32, the precision of the kernel). */
static void append_rows(const uint16_t* k_new, const uint16_t* v_new, int dtype, int kv8, float k_scale,
                        float v_scale, void* k, void* v, const int32_t* bt, const int32_t* lens, int B,
                        int q_len, int Hkv, int D, int bs, int max_blocks) {
    for (int b = 0; b < B; ++b) {
        for (int i = 0; i < q_len; ++i) {
            int t = lens[b] - q_len + i;
            if (t < 0) continue;
            int64_t phys = bt[(size_t)b * max_blocks + t / bs];
            for (int kvh = 0; kvh < Hkv; ++kvh) {
                for (int d = 0; d < D; ++d) {
                    size_t src = (((size_t)b * q_len + i) * Hkv + kvh) * D + d;
                    size_t dst = kv_offset(phys, kvh, t % bs, d, Hkv, bs, D);
                    if (kv8) {
                        float xk = (float)decode(k_new[src], dtype), xv = (float)decode(v_new[src], dtype);
                        ((uint8_t*)k)[dst] = oracle_e4m3_encode(xk / k_scale);
                        ((uint8_t*)v)[dst] = oracle_e4m3_encode(xv / v_scale);
                    } else {
                        ((uint16_t*)k)[dst] = k_new[src];
                        ((uint16_t*)v)[dst] = v_new[src];
                    }
                }
            }
        }
    }
}

int oracle_kv_append(const uint16_t* k_new, const uint16_t* v_new, uint16_t* k, uint16_t* v,
                     const int32_t* bt, const int32_t* lens, int B, int q_len, int Hkv, int D, int bs,
                     int max_blocks) {
    if (B < 0 || q_len <= 0 || Hkv <= 0 || D <= 0 || bs <= 0) return -1;
    append_rows(k_new, v_new, ORACLE_F16, 0, 1.f, 1.f, k, v, bt, lens, B, q_len, Hkv, D, bs, max_blocks);
    return 0;
}

int oracle_kv_append_e4m3(const uint16_t* k_new, const uint16_t* v_new, int dtype, float k_scale,
                          float v_scale, uint8_t* k, uint8_t* v, const int32_t* bt, const int32_t* lens,
                          int B, int q_len, int Hkv, int D, int bs, int max_blocks) {
    if (B < 0 || q_len <= 0 || Hkv <= 0 || D <= 0 || bs <= 0 || !(k_scale > 0.f) || !(v_scale > 0.f)) return -1;
    append_rows(k_new, v_new, dtype, 1, k_scale, v_scale, k, v, bt, lens, B, q_len, Hkv, D, bs, max_blocks);
    return 0;
}
