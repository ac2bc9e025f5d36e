// kernels.cuh -- parameter blocks and host launchers shared by pda.cu and
// the kernel translation units (internal; not part of the C ABI).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <atomic>
#include <cstdint>

namespace pda {

// Raise a kernel's dynamic shared-memory limit once per device.  Thread-safe
// (the library promises stateless, thread-safe calls): the per-device "done"
// bits are atomic, and a concurrent duplicate cudaFuncSetAttribute is harmless.
template <typename Kern>
inline cudaError_t ensure_smem_limit(Kern kern, size_t smem, std::atomic<uint64_t>& done) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const uint64_t bit = dev < 64 ? 1ull << dev : 0ull;
    if (bit && (done.load(std::memory_order_acquire) & bit)) return cudaSuccess;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess && bit) done.fetch_or(bit, std::memory_order_release);
    return e;
}

constexpr int kBlockSize = 16;     // tokens per KV block
constexpr int kConsumerWarps = 4;  // split-K kernel consumer warps
#ifndef PDA_TMA3D
#define PDA_TMA3D 1
#endif
// 16-bit D = 128 slabs (two 128-byte column chunks) load as ONE 3-D TMA box
// per slab (K and V: 2 UTMALDG per block instead of 4); 0 = two 2-D boxes
constexpr bool kTma3d = PDA_TMA3D != 0;
#ifndef PDA_SWP
#define PDA_SWP 0
#endif
// split-K self-issue consumers: QK^T of a warp's next block(s) is issued
// before the softmax / PV of the current one (software pipeline across
// blocks); 0 (default) = one block's QK^T -> softmax -> PV chain at a time.
// Measured 2-26 % slower (profiles/r02_ab_swp.log): the next block's stage was
// refilled only one iteration earlier, so waiting for it before the current
// softmax halves the ring's lookahead per warp (even from L2).
constexpr bool kSwp = PDA_SWP != 0;
#ifndef PDA_ELECT_ISSUE
#define PDA_ELECT_ISSUE 1
#endif
// self-issued refills from the converged warp with elect.sync inside each
// statement (no per-load ptxas waterfall loop); 0 = a lane == 0 branch
constexpr bool kElectIssue = PDA_ELECT_ISSUE != 0;
#ifndef PDA_KV_SPLIT
#define PDA_KV_SPLIT 0
#endif
// split K / V ring (self-issue, 4 consumer warps): each stage has a K and a V
// mbarrier; a warp refills the K slabs of its stages as soon as QK^T has read
// them and the V slabs after PV -- K loads go out a softmax + PV earlier.
// Off (default): measured 1 % slower on 16-bit and 4-7 % on e4m3 steps -- the
// second barrier wait, fence and issue per block cost more on the consumer
// chain than the earlier K loads save (profiles/r02_ab_kvsplit.log)
constexpr bool kKvSplit = PDA_KV_SPLIT != 0;
#ifndef PDA_KV8_PAIRS
#define PDA_KV8_PAIRS 1
#endif
// e4m3 rings of 8 / 16 / 24 stages consumed in pairs (one softmax update per
// 32 tokens); 0 = one block at a time (A/B builds)
constexpr bool kKv8Pairs = PDA_KV8_PAIRS != 0;
constexpr int kPaperWarps = 4;     // paper kernel: 128 threads = 4 warps (Table 2)

enum PrefetchMode { kPfOff = 0, kPfBulk = 1, kPfLine = 2 };

constexpr int kMaxPeers = 8;  // fused output all-gather: ranks written by one kernel

// Output destinations of the split-K path: out_peers[0..n_peers) are the [B,
// q_len, Hq_out, D] output buffers of every rank of a tensor-parallel group
// (NVLink peer-mapped, e.g. symmetric memory); this rank's heads land at
// [head_off, head_off + Hq).  Single-GPU: n_peers = 1, Hq_out = Hq, head_off = 0.
struct OutPeers {
    void* ptr[kMaxPeers];
    int n;
    int head_off;
    int Hq_out;
};

// KV append (the decode step's cache write, SURVEY 8f NEXT f3 alternative):
// the new tokens' K/V rows k_new/v_new [B, q_len, Hkv, D] (dtype) go to
// positions L_b - q_len + i of their sequence's paged cache.  k_new == nullptr:
// no append.  An e4m3 cache stores e4m3(x / scale) (fp32 division).
struct AppendParams {
    const uint16_t* k_new;
    const uint16_t* v_new;
    uint8_t* k;  // the caches, as bytes
    uint8_t* v;
    int kv8, bf16;
    float k_scale, v_scale;
};

struct SplitKParams {
    const uint16_t* q;  // [B, Hq, D]
    const uint8_t* k;   // [num_blocks, Hkv, 16, D] (bytes: prefetch addresses)
    const uint8_t* v;
    const int32_t* bt;    // [B, max_blocks]
    const int32_t* lens;  // [B]
    OutPeers outs;        // out [B, q_len, Hq, D] on every destination rank
    float* ws_o;          // [B, Hq, P_max, D]   split-K partial outputs (normalised)
    float* ws_lse;        // [B, Hq, P_max]      log2-sum-exp of each partition
    int32_t* trace;       // debug trace (TRACE instantiation only)
    uint64_t* stamps;     // TRACE only, optional: per unit {start ns, end ns, SM id} (timeline)
    int B, Hq, Hkv, g, max_blocks, part_tokens, p_max;
    int q_len;  // query tokens per sequence (multi-token decode); columns = q_len * g <= 16
    int out_dtype;
    int pf_mode, pf_dist;
    int eviction;  // pda_eviction bits
    int trace_rec_len;
    float scale_log2;  // scale * log2(e) (* k_scale for an e4m3 cache), fp32
    float out_scale;   // v_scale for an e4m3 cache, else 1
    AppendParams app;  // fused KV append (app.k_new == nullptr: none)
    int cluster;       // > 1: launched as clusters of P_max CTAs (one per partition of a
                       // (seq, kv head) row) that merge their partials through DSMEM
    int pdl;           // launched with programmatic stream serialization (PDL)
    int tile_split;    // two head tiles on 8 consumer warps, one tile each (16-bit, self-issue)
    int* query_clusters;  // host-side planner query, not a launch: when set, launch_splitk_m2
                          // stores cudaOccupancyMaxActiveClusters of the kernel it would launch
};

struct PaperParams {
    const uint16_t* q;
    const uint16_t* k;
    const uint16_t* v;
    const int32_t* bt;
    const int32_t* lens;
    void* out;
    int32_t* trace;
    int B, Hq, Hkv, g, max_blocks;
    int out_dtype;
    int pf_mode, pf_dist;
    int eviction;  // pda_eviction bits
    int trace_rec_len;
    float scale_log2;
};

struct StreamParams {
    const uint16_t* q;
    const uint16_t* k;
    const uint16_t* v;
    const int32_t* bt;
    const int32_t* lens;
    void* out;
    float* ws_o;        // [NS][2][NH][D]  partial outputs of a stream's first/last segment
    float* ws_lse;      // [NS][2][NH]
    uint32_t* tickets;  // [B * Hkv] self-resetting arrival counters (zero before first use)
    int32_t* trace;
    int B, Hq, Hkv, g, max_blocks;
    int out_dtype;
    int pf_mode, pf_dist;
    int eviction;  // pda_eviction bits
    int trace_rec_len;
    int NS;  // streams launched (grid * warps per CTA)
    float scale_log2;
};

struct BalancedParams {
    const uint16_t* q;
    const uint16_t* k;
    const uint16_t* v;
    const int32_t* bt;
    const int32_t* lens;
    void* out;
    float* ws_o;             // [G][2][NH][D]  partials of a CTA's first/last segment (normalised)
    float* ws_lse;           // [G][2][NH]     their log2-sum-exp
    long long* seq_prefix;   // [B + 1] blocks of the sequences before b (written by CTA 0)
    int32_t* trace;
    int B, Hq, Hkv, g, max_blocks;
    int out_dtype;
    int pf_mode, pf_dist;
    int eviction;  // pda_eviction bits
    int trace_rec_len;
    float scale_log2;
    int pdl;  // launched with programmatic stream serialization (PDL)
};

struct CombineParams {
    int pdl;  // launched with programmatic stream serialization (PDL)
    const float* ws_o;
    const float* ws_lse;
    const int32_t* lens;
    OutPeers outs;
    int B, Hq, p_max, part_tokens, max_tokens;
    int q_len;
    int out_dtype;
};

// Host launchers (return the launch's cudaError_t).
cudaError_t launch_splitk(const CUtensorMap& tmK, const CUtensorMap& tmV, const SplitKParams& p,
                          bool bf16, int head_dim, int n_tiles, int stages, bool trace,
                          dim3 grid, cudaStream_t stream, bool kv8 = false, bool self_issue = false);
// per-MODE instantiation sets (decode_splitk_m{0,1,2}.cu): plain, debug trace, cluster-launched
#define PDA_SPLITK_MODE_DECL(M)                                                                          \
    cudaError_t launch_splitk_m##M(const CUtensorMap& tmK, const CUtensorMap& tmV, const SplitKParams& p, \
                                   bool bf16, int head_dim, int n_tiles, int stages, dim3 grid,          \
                                   cudaStream_t stream, bool kv8, bool self_issue);
PDA_SPLITK_MODE_DECL(0)
PDA_SPLITK_MODE_DECL(1)
PDA_SPLITK_MODE_DECL(2)
#undef PDA_SPLITK_MODE_DECL
int splitk_threads(bool self_issue = false, bool tile_split = false);

cudaError_t launch_stream(const CUtensorMap& tmK, const CUtensorMap& tmV, const StreamParams& p,
                          bool bf16, int head_dim, int n_tiles, int stages, int warps, bool trace,
                          int grid, cudaStream_t stream);
size_t stream_smem_bytes(int head_dim, int stages, int warps);
bool stream_config_supported(int stages, int warps);

cudaError_t launch_balanced(const CUtensorMap& tmK, const CUtensorMap& tmV, const BalancedParams& p,
                            bool bf16, int head_dim, int n_tiles, int stages, bool trace, int grid,
                            cudaStream_t stream);
size_t balanced_smem_bytes(int head_dim, int n_tiles, int stages);
// balanced_combine_kernel alone (S8 of the persistent kernels' split rows)
cudaError_t launch_balanced_combine(const BalancedParams& p, int grid, int head_dim, cudaStream_t stream);
// the tcgen05 kernel (decode_tc.cu): 16-bit KV, head_dim 128, one query token;
// tmK a 2-D map (64-column boxes), tmV and tmQ 3-D maps (whole 256-B rows)
cudaError_t launch_tc(const CUtensorMap& tmK, const CUtensorMap& tmV, const CUtensorMap& tmQ,
                      const BalancedParams& p, bool bf16, int grid, cudaStream_t stream);
size_t tc_smem_bytes();
int tc_threads();
size_t tc_stamp_bytes(int grid);  // 0 unless built with PDA_TC_STAMPS (measurement builds)

cudaError_t launch_combine(const CombineParams& p, int head_dim, cudaStream_t stream);

cudaError_t launch_paper(const PaperParams& p, bool bf16, int head_dim, bool trace, dim3 grid,
                         cudaStream_t stream);

// Standalone KV append (every kernel other than split-K, and the unfused
// comparison): one launch writing all B * q_len * Hkv new rows.
cudaError_t launch_kv_append(const AppendParams& a, const int32_t* bt, const int32_t* lens, int B,
                             int q_len, int Hkv, int head_dim, int max_blocks, cudaStream_t stream);

// Debug validation of the device-resident block tables / lengths:
// counts[0..3) (int64, device) = invalid lengths, out-of-range referenced
// block ids, invalid sequences.
cudaError_t launch_validate(const int32_t* bt, const int32_t* lens, int B, int max_blocks,
                            int64_t num_blocks, long long* counts, cudaStream_t stream);

cudaError_t launch_read_roofline(const void* buf, size_t bytes, void* sink, int num_sms, int mode,
                                 cudaStream_t stream);

}  // namespace pda
