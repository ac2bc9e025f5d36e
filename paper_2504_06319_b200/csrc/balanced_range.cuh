// balanced_range.cuh -- S0 of the load-balanced persistent kernels (balanced,
// tc): the KV blocks of the whole step form one ordered item list (rows
// (b, kv head) in order, row r holding n_b = ceil(L_b / 16) blocks); with T
// items and G resident CTAs, CTA c owns items [floor(c T / G),
// floor((c + 1) T / G)) -- +-1 block of every other CTA -- cut into
// segments at row boundaries.  Computed on the device by one warp (no host
// sync on the lengths).
#pragma once

#include "kernels.cuh"
#include "ptx.cuh"

namespace pda {
namespace br {

constexpr unsigned kAllLanes = 0xffffffffu;

struct Cursor {
    int b, kvh, j, n, L;  // sequence, kv head, block in row, blocks in row, context length
    long long pre;        // item index of (b, kvh = 0, j = 0)
};

__device__ __forceinline__ int clamp_len(const int32_t* lens, int b, int max_tokens) {
    const int L = __ldg(lens + b);
    return L < max_tokens ? L : max_tokens;
}

__device__ __forceinline__ int blocks_of(int L) { return L > 0 ? (L + kBlockSize - 1) / kBlockSize : 0; }

// Next non-empty row after c's row (kv heads of a sequence, then sequences).
__device__ __forceinline__ void next_row(Cursor& c, const int32_t* lens, int B, int Hkv, int max_tokens) {
    c.j = 0;
    if (++c.kvh < Hkv) return;
    c.kvh = 0;
    c.pre += (long long)c.n * Hkv;
    while (++c.b < B) {
        const int L = clamp_len(lens, c.b, max_tokens);
        if (L > 0) {
            c.L = L;
            c.n = blocks_of(L);
            return;
        }
    }
}

// Move the cursor k items forward; seg counts the row boundaries crossed.
__device__ __forceinline__ void advance(Cursor& c, int k, int& seg, const int32_t* lens, int B, int Hkv,
                                        int max_tokens) {
    c.j += k;
    while (c.j >= c.n) {
        const int over = c.j - c.n;
        next_row(c, lens, B, Hkv, max_tokens);
        c.j = over;
        ++seg;
    }
}

// Lane 0's cursor in every lane, through shuffles (every lane holds the same
// cursor anyway): ptxas can then treat the fields as warp-uniform.
__device__ __forceinline__ void uniform_cursor(Cursor& c) {
    c.b = __shfl_sync(0xffffffffu, c.b, 0);
    c.kvh = __shfl_sync(0xffffffffu, c.kvh, 0);
    c.j = __shfl_sync(0xffffffffu, c.j, 0);
    c.n = __shfl_sync(0xffffffffu, c.n, 0);
    c.L = __shfl_sync(0xffffffffu, c.L, 0);
    c.pre = __shfl_sync(0xffffffffu, c.pre, 0);
}

// CTA owning item k: the largest c with floor(c*T/G) <= k.
__device__ __forceinline__ int cta_of(long long k, long long T, int G) { return (int)(((k + 1) * G - 1) / T); }
__device__ __forceinline__ long long range_start(int c, long long T, int G) { return (long long)c * T / G; }


struct RangePlan {
    long long T, k0, k1;  // items in the step, this CTA's range [k0, k1)
    int Ge;               // CTAs with work (min(T, G))
    int n_segs, end_j;    // segments of the range; block (in its row) of the range's last item
    Cursor start;         // the range's first item
};

// Warp-wide (all 32 lanes, same result in every lane).  seq_prefix (may be
// null): CTA 0 writes the exclusive prefix of blocks per sequence, [B + 1],
// for the combine kernel.
__device__ __forceinline__ RangePlan plan_range(const int32_t* lens, int B, int Hkv, int max_tokens, int c, int G,
                                                long long* seq_prefix, int lane) {
    long long T = 0;
    for (int base = 0; base < B; base += 256) {
        int part = 0;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int b = base + u * 32 + lane;
            if (b < B) part += blocks_of(clamp_len(lens, b, max_tokens));
        }
        T += __reduce_add_sync(kAllLanes, (unsigned)part);
    }
    // the combine kernel needs every sequence's first item: CTA 0 writes the
    // exclusive prefix (in blocks, per kv head) of the step's sequences
    if (c == 0 && seq_prefix != nullptr) {
        long long run = 0;
        for (int base = 0; base <= B; base += 32) {
            const int b = base + lane;
            const long long n = b < B ? blocks_of(clamp_len(lens, b, max_tokens)) : 0;
            long long incl = n;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const long long y = __shfl_up_sync(kAllLanes, incl, o);
                if (lane >= o) incl += y;
            }
            if (b <= B) seq_prefix[b] = run + incl - n;
            run += __shfl_sync(kAllLanes, incl, 31);
        }
    }
    T *= Hkv;
    const int Ge = T < (long long)G ? (int)T : (int)G;
    long long k0 = 0, k1 = 0;
    if (c < Ge) {
        k0 = range_start(c, T, Ge);
        k1 = range_start(c + 1, T, Ge);
    }
    Cursor cur{};
    int n_segs = 0, end_j = 0;
    if (k1 > k0) {
        long long pre = 0;
        for (int base = 0;; base += 32) {
            const int b = base + lane;
            const long long items = b < B ? (long long)blocks_of(clamp_len(lens, b, max_tokens)) * Hkv : 0;
            long long incl = items;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const long long y = __shfl_up_sync(kAllLanes, incl, o);
                if (lane >= o) incl += y;
            }
            const unsigned hit = __ballot_sync(kAllLanes, pre + incl > k0);
            if (hit) {
                const int src = __ffs(hit) - 1;
                const long long before = pre + __shfl_sync(kAllLanes, incl - items, src);
                cur.b = base + src;
                cur.L = clamp_len(lens, cur.b, max_tokens);
                cur.n = blocks_of(cur.L);
                cur.pre = before;
                const long long off = k0 - before;
                cur.kvh = (int)(off / cur.n);
                cur.j = (int)(off % cur.n);
                break;
            }
            pre += __shfl_sync(kAllLanes, incl, 31);
        }
        // walk the range's rows: segments, and where the last one ends
        Cursor e = cur;
        long long rem = k1 - k0;
        n_segs = 1;
        while (rem > e.n - e.j) {
            rem -= e.n - e.j;
            next_row(e, lens, B, Hkv, max_tokens);
            ++n_segs;
        }
        end_j = e.j + (int)rem - 1;
    }
    RangePlan r;
    r.T = T;
    r.k0 = k0;
    r.k1 = k1;
    r.Ge = Ge;
    r.n_segs = n_segs;
    r.end_j = end_j;
    r.start = cur;
    return r;
}

}  // namespace br
}  // namespace pda
