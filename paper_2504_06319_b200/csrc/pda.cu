// pda.cu -- the C ABI (include/pda.h): argument validation, the split-K
// planner (S0), TMA tensor-map construction and kernel dispatch.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>

#include "../../include/pda.h"
#include "kernels.cuh"

namespace {

constexpr int kDefaultStages = 8;
constexpr int kDefaultStagesKV8 = 16;
constexpr int kDefaultTileSplitStages = 8;  // tile-split kernel ring (12: 180 vs 170 us at B=128 g=16)
constexpr int kDefaultStreamStages = 6;
constexpr int kDefaultStreamWarps = 2;
constexpr int kDefaultBalancedStages = 8;
constexpr size_t kSmemPerSm = 233472;  // 228 KB per SM on B200
constexpr size_t kSmemReservedPerCta = 1024;
constexpr int kDefaultSms = 148;  // B200
constexpr int kMaxCluster = 16;     // non-portable cluster size limit (split-K merge in a cluster)
constexpr int kAutoMaxCluster = 8;  // planner: portable cluster sizes only
constexpr int kSmallGridRows = 8;   // planner: <= 8 (seq, kv head) rows take the small-grid split

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }
int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }
size_t elem_bytes(int dt) { return dt == PDA_F32 ? 4 : 2; }

int q_tokens(const pda_shape* s) { return s->q_len > 1 ? s->q_len : 1; }

pda_status validate(const pda_shape* s, const pda_options* o) {
    if (!s || !o) return PDA_ERR_NULL;
    if (s->num_seqs < 0 || s->num_seqs > 65535 || s->num_q_heads <= 0 || s->num_kv_heads <= 0 ||
        s->num_q_heads % s->num_kv_heads != 0 || s->head_dim <= 0 || s->block_size <= 0 ||
        s->num_blocks <= 0 || s->max_blocks_per_seq <= 0 || s->num_q_heads > 65535)
        return PDA_ERR_SHAPE;
    if ((int64_t)s->num_blocks * s->num_kv_heads * s->block_size >= (int64_t(1) << 31))
        return PDA_ERR_SHAPE;  // TMA row coordinates are int32
    if ((int64_t)s->max_blocks_per_seq * s->block_size >= (int64_t(1) << 30)) return PDA_ERR_SHAPE;
    if (s->dtype != PDA_F16 && s->dtype != PDA_BF16) return PDA_ERR_UNSUPPORTED;
    if (s->out_dtype != s->dtype && s->out_dtype != PDA_F32) return PDA_ERR_UNSUPPORTED;
    if (s->head_dim != 64 && s->head_dim != 128) return PDA_ERR_UNSUPPORTED;
    if (s->kv_dtype != s->dtype && s->kv_dtype != PDA_E4M3) return PDA_ERR_UNSUPPORTED;
    if (s->kv_dtype == PDA_E4M3 &&
        (s->head_dim != 128 || (o && o->kernel != PDA_KERNEL_AUTO && o->kernel != PDA_KERNEL_SPLITK)))
        return PDA_ERR_UNSUPPORTED;
    if (o && (!(o->k_scale >= 0.f) || !(o->v_scale >= 0.f))) return PDA_ERR_SHAPE;
    if (o && (o->issue_mode < 0 || o->issue_mode > 2)) return PDA_ERR_SHAPE;
    if (o && (o->merge < 0 || o->merge > 2)) return PDA_ERR_SHAPE;
    if (o && s->kv_dtype == PDA_E4M3 && o->issue_mode == 1) return PDA_ERR_UNSUPPORTED;
    if (o && o->issue_mode != 1 && (o->kernel == PDA_KERNEL_AUTO || o->kernel == PDA_KERNEL_SPLITK) &&
        o->prefetch != PDA_PF_OFF && o->prefetch_distance > 32)
        return PDA_ERR_UNSUPPORTED;  // self-issue block-id window reaches 32 blocks ahead
    if (s->block_size != pda::kBlockSize) return PDA_ERR_UNSUPPORTED;
    if (s->num_q_heads / s->num_kv_heads > 16) return PDA_ERR_UNSUPPORTED;
    if (s->q_len < 0 || s->q_len > 16) return PDA_ERR_SHAPE;
    if (q_tokens(s) > 1 &&
        (q_tokens(s) * (s->num_q_heads / s->num_kv_heads) > 16 ||
         (o && o->kernel != PDA_KERNEL_AUTO && o->kernel != PDA_KERNEL_SPLITK)))
        return PDA_ERR_UNSUPPORTED;
    if (o->prefetch < PDA_PF_OFF || o->prefetch > PDA_PF_AUTO) return PDA_ERR_SHAPE;
    if (o->prefetch != PDA_PF_OFF && o->prefetch != PDA_PF_AUTO &&
        (o->prefetch_distance < 1 || o->prefetch_distance > (1 << 20)))
        return PDA_ERR_SHAPE;
    if (o->partition_tokens < 0 || o->partition_tokens % s->block_size != 0) return PDA_ERR_SHAPE;
    if (o->kernel < PDA_KERNEL_AUTO || o->kernel > PDA_KERNEL_TC) return PDA_ERR_SHAPE;
    if (o->kernel == PDA_KERNEL_TC &&
        (s->kv_dtype == PDA_E4M3 || s->head_dim != 128 || q_tokens(s) > 1 || o->smem_stages != 0))
        return PDA_ERR_UNSUPPORTED;
    if (o->num_sms < 0 || o->stream_warps < 0 || o->eviction < 0 || o->eviction > PDA_EV_AUTO) return PDA_ERR_SHAPE;
    if (o->kernel == PDA_KERNEL_STREAM) {
        const int st = o->smem_stages ? o->smem_stages : kDefaultStreamStages;
        const int w = o->stream_warps ? o->stream_warps : kDefaultStreamWarps;
        if (!pda::stream_config_supported(st, w)) return PDA_ERR_UNSUPPORTED;
        if (o->prefetch != PDA_PF_OFF && o->prefetch_distance > 32) return PDA_ERR_UNSUPPORTED;
    } else if (o->kernel == PDA_KERNEL_BALANCED) {
        if (o->smem_stages != 0 && o->smem_stages != 4 && o->smem_stages != 8 && o->smem_stages != 12)
            return PDA_ERR_UNSUPPORTED;
        if (o->prefetch != PDA_PF_OFF && o->prefetch_distance > 32) return PDA_ERR_UNSUPPORTED;
    } else if (s->kv_dtype == PDA_E4M3) {
        if (o->smem_stages != 0 && o->smem_stages != 8 && o->smem_stages != 12 && o->smem_stages != 16 &&
            o->smem_stages != 24)
            return PDA_ERR_UNSUPPORTED;
        if (o->prefetch != PDA_PF_OFF && o->prefetch_distance > 32) return PDA_ERR_UNSUPPORTED;
    } else if (o->smem_stages != 0 && o->smem_stages != 4 && o->smem_stages != 8 &&
               o->smem_stages != 12) {
        return PDA_ERR_UNSUPPORTED;
    }
    return PDA_OK;
}

// Split-K ring refill mode: e4m3 always self-issues; 16-bit follows issue_mode,
// auto = self-issue (equal on C2, +1-3 % on GQA / ragged cells).
bool self_issue(const pda_shape* s, const pda_options* o) {
    if (s->kv_dtype == PDA_E4M3) return true;
    return o->issue_mode != 1;
}

// Resident split-K CTAs per SM that the planner assumes when it chooses the
// split: 3 (the default-depth rings), 2 for the two-tile producer-warp kernels.
// The split is chosen BEFORE the ring depth, so the two instantiations built
// for 4 CTAs/SM (16-bit 4-stage, e4m3 12-stage; splitk_min_blocks in
// splitk_impl.cuh) are planned as 3/SM too: a grid of 445-592 units counts as
// multi-wave (combine kernel, not a cluster merge) although it would fit one
// wave at 4/SM.  The split sizes and thresholds below were measured with this
// convention.
// prefetch = AUTO with kernel = AUTO: short-context steps whose q-head rows
// (B * Hq, one CTA each in the paper's grid) fill the chip better than
// split-K's (sequence, kv head) units run the paper-structure kernel with
// Alg. 1's prefetch.  Measured band (105 uniform cells, ctx 128-512, 30
// interleaved rounds each, profiles/r02_short_ctx.jsonl): GQA groups >= 4 with
// 128 <= B * Hq <= 512 (<= 256 at ctx 512) gain 1.12-1.52x over split-K
// (e.g. B=8, 32/8 heads, ctx 256: 12.3 vs 16.4 us); below the band the two
// tie within the 2 us event resolution, above it the paper grid is 0.3-0.9x
// (every CTA walks a whole context); MHA is mixed and stays on split-K.
constexpr int64_t kAutoPaperMaxTokens = 512;
bool auto_paper(const pda_shape* s, const pda_options* o) {
    if (o->kernel != PDA_KERNEL_AUTO || o->prefetch != PDA_PF_AUTO) return false;
    if (s->kv_dtype == PDA_E4M3 || q_tokens(s) > 1) return false;
    const int64_t max_tokens = (int64_t)s->max_blocks_per_seq * s->block_size;
    if (max_tokens > kAutoPaperMaxTokens) return false;
    if (s->num_q_heads / s->num_kv_heads < 4) return false;
    const int64_t rows = (int64_t)s->num_seqs * s->num_q_heads;
    return rows >= 128 && rows <= (max_tokens <= 256 ? 512 : 256);
}

int splitk_ctas_per_sm(const pda_shape* s, const pda_options* o, int n_tiles) {
    return (n_tiles > 1 && s->kv_dtype != PDA_E4M3 && !self_issue(s, o)) ? 2 : 3;
}

// 16-bit steps whose grid of `units` CTAs is one wave at 2 CTAs/SM run the
// split kernel (8 consumer warps, two per block; splitk_impl.cuh TS): with
// two head tiles (g = 16, or q_len * g > 8) one tile each, with one tile one
// half of the output rows d each (D split).  Two tiles: B=128 32/2 ctx 8k 170 vs 174 us,
// B=32 57.3 vs 61.4, B=16 ctx 32k 94.2 vs 98.3, B=64 64/4 170 vs 172; grids of
// more waves keep the 4-warp kernel at 3 CTAs/SM (B=256 ctx 4k 203 vs 195, C5
// with 2 query tokens 2408 vs 2399; profiles/r02_ab_ts.log).  Ring 8 or 12.
// PDA_TILE_SPLIT=0 / 1 forces it off / on (A/B measurements only).
bool tile_split(const pda_shape* s, const pda_options* o, int64_t units, int sms, int stages) {
    if (!self_issue(s, o)) return false;
    if (s->kv_dtype == PDA_E4M3) {
        // e4m3 D split (16 / 24 stages, one head tile): A/B switch only
        static const char* kv8 = std::getenv("PDA_TILE_SPLIT_KV8");
        return kv8 && std::atoi(kv8) != 0 && (stages == 16 || stages == 24) &&
               q_tokens(s) * (s->num_q_heads / s->num_kv_heads) <= 8;
    }
    if (stages != 8 && stages != 12) return false;
    static const char* env = std::getenv("PDA_TILE_SPLIT");
    if (env) return std::atoi(env) != 0;
    return units <= 2 * (int64_t)sms;
}

// Can all n_clusters clusters of `cluster` CTAs of the chosen split-K kernel
// be resident at once?  Asked of the current device
// (cudaOccupancyMaxActiveClusters, cached per configuration): clusters are
// placed per GPC, so a count of CTA slots can say "one wave" when it is not --
// 296 CTAs in clusters of 4 at 2 CTAs/SM on 148 SMs ran as two waves (150 vs
// 104 us with the combine kernel).  Planning for an assumed SM
// count (num_sms given) or without a device: the slot count decides.
bool clusters_fit(const pda_shape* s, const pda_options* o, int n_tiles, int stages, bool ts, int cluster,
                  int64_t n_clusters) {
    if (o->num_sms != 0) return true;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) {
        cudaGetLastError();
        return true;
    }
    const bool kv8 = s->kv_dtype == PDA_E4M3, self = self_issue(s, o);
    const int64_t key = ((((((((int64_t)dev * 2 + (s->dtype == PDA_BF16)) * 256 + s->head_dim) * 4 + n_tiles) * 32 +
                           stages) * 2 + kv8) * 2 + self) * 2 + ts) * 32 + cluster;
    static std::mutex mu;
    static std::map<int64_t, int> cache;
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = cache.find(key);
        if (it != cache.end()) return it->second <= 0 || n_clusters <= it->second;
    }
    pda::SplitKParams p{};
    int n = 0;
    p.cluster = cluster;
    p.tile_split = ts;
    p.query_clusters = &n;
    CUtensorMap none{};
    // the first plan of a configuration may run inside a stream capture: the
    // occupancy query (and the attribute calls before it) are made with this
    // thread's capture mode relaxed, so a global-mode capture stays valid
    cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
    cudaThreadExchangeStreamCaptureMode(&mode);
    if (pda::launch_splitk_m2(none, none, p, s->dtype == PDA_BF16, s->head_dim, n_tiles, stages, dim3(cluster, 1, 1),
                              nullptr, kv8, self) != cudaSuccess) {
        cudaGetLastError();
        n = 0;  // unknown: the slot count decides
    }
    cudaThreadExchangeStreamCaptureMode(&mode);
    std::lock_guard<std::mutex> lk(mu);
    cache[key] = n;
    return n <= 0 || n_clusters <= n;
}

pda_status plan(const pda_shape* s, const pda_options* o, pda_plan_info* pl) {
    pda_status st = validate(s, o);
    if (st != PDA_OK) return st;
    std::memset(pl, 0, sizeof(*pl));
    const int B = s->num_seqs, Hq = s->num_q_heads, Hkv = s->num_kv_heads, D = s->head_dim;
    const int64_t max_tokens = (int64_t)s->max_blocks_per_seq * s->block_size;
    if (o->eviction == PDA_EV_AUTO) {
        // demand evict_first keeps q, tables and split-K partials in L2 on small
        // steps (+5-19 % measured); on multi-GB steps it costs 2-6 %
        const double kv_max = 4.0 * B * (double)max_tokens * Hkv * D;
        pl->eviction = kv_max <= 2147483648.0 ? PDA_EV_DEMAND_FIRST : PDA_EV_NORMAL;
    } else {
        pl->eviction = o->eviction;
    }
    if (o->kernel == PDA_KERNEL_PAPER || auto_paper(s, o)) {
        // grid [H, B, 1], N_thread = 128 (Table 2)
        if (o->kernel != PDA_KERNEL_PAPER && o->eviction == PDA_EV_AUTO)
            pl->eviction = PDA_EV_PREFETCH_LAST;  // prefetch = AUTO's measured variant
        pl->kernel = PDA_KERNEL_PAPER;
        pl->partition_tokens = (int32_t)max_tokens;
        pl->p_max = 1;
        pl->smem_stages = 0;
        pl->grid_x = Hq;
        pl->grid_y = B;
        pl->grid_z = 1;
        pl->threads = pda::kPaperWarps * 32;
        const int R = (int)ceil_div(s->max_blocks_per_seq, pda::kPaperWarps);
        pl->trace_rec_len = 4 + 2 * R;
        pl->trace_records = B * Hq * pda::kPaperWarps;
        pl->workspace_bytes = 0;
        if (o->kernel != PDA_KERNEL_PAPER) {
            // the same call with a fused append / gather runs split-K (run()):
            // report its workspace so one allocation serves both
            pda_options o2 = *o;
            o2.kernel = PDA_KERNEL_SPLITK;
            pda_plan_info p2;
            if (plan(s, &o2, &p2) == PDA_OK) pl->workspace_bytes = p2.workspace_bytes;
        }
        return PDA_OK;
    }
    if (o->kernel == PDA_KERNEL_STREAM) {
        // Persistent grid: as many CTAs as fit on the chip at once; NS streams
        // share all KV blocks of the step equally (S0 happens on the device).
        const int st = o->smem_stages ? o->smem_stages : kDefaultStreamStages;
        const int w = o->stream_warps ? o->stream_warps : kDefaultStreamWarps;
        const int sms = o->num_sms ? o->num_sms : kDefaultSms;
        const size_t smem = pda::stream_smem_bytes(D, st, w);
        int per_sm = (int)(kSmemPerSm / (smem + kSmemReservedPerCta));
        per_sm = per_sm < 2048 / (w * 32) ? per_sm : 2048 / (w * 32);
        per_sm = per_sm < 32 ? per_sm : 32;
        const int nh = (Hq / Hkv) <= 8 ? 8 : 16;
        pl->kernel = PDA_KERNEL_STREAM;
        pl->partition_tokens = (int32_t)max_tokens;
        pl->p_max = 1;
        pl->smem_stages = st;
        pl->grid_x = sms * per_sm;
        pl->grid_y = 1;
        pl->grid_z = 1;
        pl->threads = w * 32;
        pl->trace_rec_len = 4 + 2 * s->max_blocks_per_seq;
        pl->trace_records = B * Hkv;
        const size_t ns = (size_t)pl->grid_x * w;
        pl->workspace_bytes = align256(ns * 2 * nh * D * 4) + align256(ns * 2 * nh * 4) +
                              align256((size_t)B * Hkv * 4);
        return PDA_OK;
    }
    if (o->kernel == PDA_KERNEL_TC) {
        // One persistent CTA per SM (its 3-stage ring of 128-token tiles takes
        // ~219 KB of shared memory); the device splits the step's blocks into
        // G equal ranges (S0), the balanced combine merges split rows.
        const int sms = o->num_sms ? o->num_sms : kDefaultSms;
        const int nh = (Hq / Hkv) <= 8 ? 8 : 16;
        pl->kernel = PDA_KERNEL_TC;
        pl->partition_tokens = (int32_t)max_tokens;
        pl->p_max = 1;
        pl->smem_stages = 3;
        pl->grid_x = sms;
        pl->grid_y = 1;
        pl->grid_z = 1;
        pl->threads = pda::tc_threads();
        pl->trace_rec_len = 0;
        pl->trace_records = 0;
        const size_t gx = (size_t)pl->grid_x;
        pl->workspace_bytes = align256(gx * 2 * nh * D * 4) + align256(gx * 2 * nh * 4) +
                              align256(((size_t)B + 1) * 8) + pda::tc_stamp_bytes(pl->grid_x);
        return PDA_OK;
    }
    if (o->kernel == PDA_KERNEL_BALANCED) {
        // One persistent wave: 2 CTAs per SM (one head tile; 1 for two tiles),
        // fewer if the ring does not fit; the device splits the step's T blocks
        // into G equal ranges (S0) and a combine grid merges the split rows.
        const int n_tiles = (Hq / Hkv) <= 8 ? 1 : 2;
        const int st = o->smem_stages ? o->smem_stages : kDefaultBalancedStages;
        const int sms = o->num_sms ? o->num_sms : kDefaultSms;
        const size_t smem = pda::balanced_smem_bytes(D, n_tiles, st);
        int per_sm = (int)(kSmemPerSm / (smem + kSmemReservedPerCta));
        const int reg_cap = n_tiles == 1 ? 2 : 1;
        per_sm = per_sm < reg_cap ? per_sm : reg_cap;
        per_sm = per_sm > 0 ? per_sm : 1;
        const int nh = 8 * n_tiles;
        pl->kernel = PDA_KERNEL_BALANCED;
        pl->partition_tokens = (int32_t)max_tokens;
        pl->p_max = 1;
        pl->smem_stages = st;
        pl->grid_x = sms * per_sm;
        pl->grid_y = 1;
        pl->grid_z = 1;
        pl->threads = pda::splitk_threads(true);
        pl->trace_rec_len = 4 + 2 * s->max_blocks_per_seq;
        pl->trace_records = B * Hkv;
        const size_t gx = (size_t)pl->grid_x;
        pl->workspace_bytes = align256(gx * 2 * nh * D * 4) + align256(gx * 2 * nh * 4) +
                              align256(((size_t)B + 1) * 8);
        return PDA_OK;
    }
    // S0: split-K plan.  Units (partition, kv head, seq) are independent; pick
    // the partition size so the grid holds >= 4 waves of resident CTAs while a
    // partition keeps >= 512 tokens (32 blocks) to amortise pipeline fill.
    const int n_tiles = q_tokens(s) * (Hq / Hkv) <= 8 ? 1 : 2;
    // e4m3 stages are half the bytes: default to twice the depth (same bytes in flight)
    int stages = o->smem_stages ? o->smem_stages
                                : (s->kv_dtype == PDA_E4M3 ? kDefaultStagesKV8 : kDefaultStages);
    if (o->smem_stages == 0 && s->kv_dtype == PDA_E4M3 && n_tiles == 1 &&
        2.0 * B * (double)max_tokens * Hkv * D <= 1073741824.0) {
        // e4m3 steps up to 1 GiB of KV: 12 stages consumed one block at a time
        // at 4 CTAs/SM beat 16 stages in pairs at 3 (B=64 ctx 4k 81.9 vs 84.0 us,
        // B=64 ctx 512 22.6 vs 28.7, B=4 ctx 4k 20.5 vs 24.6); multi-GB steps keep
        // 16 (C2 321.5 vs 323.7, C5 1268.7 vs 1273.9; profiles/r01_ab_kv8_s12.log)
        stages = 12;
    }
    const int sms = o->num_sms ? o->num_sms : kDefaultSms;
    int64_t P;
    if (o->partition_tokens > 0) {
        P = o->partition_tokens;
    } else {
        const int64_t units0 = (int64_t)B * Hkv;
        const int64_t conc = (int64_t)sms * splitk_ctas_per_sm(s, o, n_tiles);
        int64_t split = 1;
        // partitions of >= 512 tokens; once the grid has >= 256 units, >= 1024
        // (measured: e.g. B=1, ctx 32k: 256 x 1024 tokens 43 us vs 512 x 512 55 us);
        // tiny grids that would stay under one CTA per SM even with 128-token
        // partitions go down to 128 (B=1-4, ctx 512: 12.3-14.3 us vs 16.4 us)
        const int64_t min_part = units0 * ceil_div(max_tokens, 128) <= sms ? 128 : 512;
        // a single, well-filled wave (>= 0.4 of the resident CTA slots) of
        // 512-8192-token partitions beats 1-4 ragged waves: take the smallest
        // split that reaches it (measured: B=4 ctx 32k 88 vs 100 us, B=16 ctx
        // 4k 49 vs 53, C2 at TP 8 94 vs 100; longer partitions prefer many
        // waves: B=16 ctx 32k 280 vs 285)
        // ... and at least one CTA per SM: with two head tiles (2 CTAs/SM) 0.4 of
        // the slots is fewer CTAs than SMs (g = 16, B=64 ctx 8k: 128 CTAs 135 us
        // vs 256 CTAs 100 us; B=16 ctx 32k 141 vs 98)
        int64_t one_wave = 0;
        for (int64_t sp = 1; units0 * sp <= conc && max_tokens / sp >= 512; sp *= 2)
            if (units0 * sp * 5 >= conc * 2 && units0 * sp >= sms && max_tokens / sp <= 8192) {
                one_wave = sp;
                break;
            }
        if (units0 <= kSmallGridRows) {
            // A handful of (sequence, kv head) rows (latency-bound steps): at most
            // 128 CTAs (no cluster -- the combine kernel, see below) of partitions
            // >= min(ctx / 16, 1024) tokens and >= 128.  Measured over 80 small
            // grids x partition counts 1-64 (profiles/r02_small_grid_sweep.jsonl):
            // B=1 8/1 ctx 8k 18.4 vs 27.7 us (64 x 128-token partitions before),
            // ctx 16k 24.5 vs 43.0, ctx 32k (B=1-4) 31-33 vs 33-39; short contexts
            // keep 128-token partitions (B=1-4, ctx 512-2048).  An e4m3 CTA streams
            // half the bytes per block at a similar per-block cost, so e4m3 steps go
            // to 256 CTAs (B=1 32/8 ctx 32k: 32 x 1024 tokens 32.8 vs 16 x 2048 36.9 us).
            const int64_t min_p = std::max<int64_t>(128, std::min<int64_t>(max_tokens / 16, 1024));
            const int64_t max_ctas = s->kv_dtype == PDA_E4M3 ? 256 : 128;
            split = 1;
            while (units0 * split * 2 <= max_ctas && max_tokens / (split * 2) >= min_p) split *= 2;
        } else if (one_wave) {
            split = one_wave;
        } else {
            while (units0 * split < 4 * conc &&
                   max_tokens / (split * 2) >= (units0 * split * 2 > 256 ? 1024 : min_part))
                split *= 2;
        }
        P = ceil_div(ceil_div(max_tokens, split), s->block_size) * s->block_size;
    }
    const int64_t p_max = ceil_div(max_tokens, P);
    if (o->smem_stages == 0 && s->kv_dtype != PDA_E4M3 && n_tiles == 1) {
        // A grid just past one wave at 3 CTAs/SM (8-stage rings) but within two
        // waves at 4 CTAs/SM (4-stage rings, 34 KiB of shared memory; 127
        // registers x 128 threads still fit 4): the shallower ring loses less to
        // wave quantisation than to bytes in flight (measured, L2 flushed: B=64
        // ctx 512 28.7 vs 32.8 us, B=64 ctx 1024 47.1 vs 51.2, B=128 ctx 512
        // 45.1 vs 49.2; past two waves the 8-stage ring wins again: B=256 ctx
        // 1024 133 vs 129, and one-wave grids keep their depth: B=32 ctx 512
        // 22.5 vs 20.5)
        const int64_t units = (int64_t)B * Hkv * p_max;
        if (units > (int64_t)sms * 3 && units <= (int64_t)sms * 4 * 2) stages = 4;
    }
    const bool kv8 = s->kv_dtype == PDA_E4M3;
    const bool ts = tile_split(s, o, (int64_t)B * Hkv * p_max, sms,
                               o->smem_stages || kv8 ? stages : kDefaultTileSplitStages);
    if (ts && o->smem_stages == 0 && !kv8) stages = kDefaultTileSplitStages;
    pl->kernel = PDA_KERNEL_SPLITK;
    pl->partition_tokens = (int32_t)(P < max_tokens ? P : ceil_div(max_tokens, s->block_size) * s->block_size);
    pl->p_max = (int32_t)p_max;
    pl->smem_stages = stages;
    pl->grid_x = (int32_t)p_max;
    pl->grid_y = Hkv;
    pl->grid_z = B;
    pl->threads = pda::splitk_threads(self_issue(s, o), ts);  // 256: the tile-split kernel
    pl->trace_rec_len = 4 + 2 * (pl->partition_tokens / s->block_size);
    pl->trace_records = (int32_t)(B * Hkv * p_max);
    // S8: merge partitions inside a thread-block cluster (DSMEM) when they fit
    // one.  Auto only when the whole grid is one wave of resident CTAs: there
    // the merge saves the combine launch (B=1-4, ctx 4k: 8-10 % faster); with
    // more waves a cluster's CTAs hold their SMs while waiting for the slowest
    // partner (B=16-64, ctx 4k: 14-15 % slower) -- DESIGN.md 7.
    if (p_max > 1 && o->merge != 1) {
        if (o->merge == 2 && p_max > kMaxCluster) return PDA_ERR_UNSUPPORTED;
        const int64_t conc = (int64_t)sms * (ts ? 2 : splitk_ctas_per_sm(s, o, n_tiles));
        const bool one_wave = (int64_t)B * Hkv * p_max <= conc;
        // ... and with at least one CTA per SM: below that the combine kernel
        // (PDL-launched, one memory round trip) is 0-2 us faster than the cluster
        // barriers + DSMEM merge (profiles/r02_small_grid_sweep.jsonl: e.g. B=1,
        // 4 heads, ctx 1k 12.3 vs 14.4 us); from 256 CTAs on the cluster wins
        // or ties (B=8 32/8 ctx 2k 22.5 vs 24.6, B=2 MHA ctx 8k 51.2 vs 53.2)
        const bool fills = (int64_t)B * Hkv * p_max >= sms;
        if (o->merge == 2 ||
            (p_max <= kAutoMaxCluster && one_wave && fills &&
             clusters_fit(s, o, n_tiles, stages, ts, (int)p_max, (int64_t)B * Hkv)))
            pl->cluster = (int32_t)p_max;
    }
    const size_t rows = (size_t)B * q_tokens(s) * Hq;
    pl->workspace_bytes = p_max > 1 && pl->cluster == 0
                              ? align256(rows * p_max * D * 4) + align256(rows * p_max * 4) : 0;
    return PDA_OK;
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

// 2-D view of a [num_blocks, Hkv, 16, D] cache: rows = num_blocks * Hkv * 16,
// cols = D; box = 16 rows x 64 cols (one 128-byte swizzle atom wide).
bool encode_cache_map(CUtensorMap* m, const void* base, const pda_shape* s) {
    auto enc = get_encode();
    if (!enc) return false;
    const bool kv8 = s->kv_dtype == PDA_E4M3;
    if (pda::kTma3d && !kv8 && s->head_dim == 128) {
        // 3-D view (col within a 64-column chunk, row, chunk): one box of
        // 64 x 16 x 2 is a whole slab, written as [chunk][row][128 B]
        const cuuint64_t dims[3] = {64, (cuuint64_t)s->num_blocks * s->num_kv_heads * s->block_size, 2};
        const cuuint64_t strides[2] = {(cuuint64_t)s->head_dim * 2, 128};
        const cuuint32_t box[3] = {64u, (cuuint32_t)s->block_size, 2u};
        const cuuint32_t estr[3] = {1, 1, 1};
        return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    }
    const cuuint64_t dims[2] = {(cuuint64_t)s->head_dim,
                                (cuuint64_t)s->num_blocks * s->num_kv_heads * s->block_size};
    const cuuint64_t strides[1] = {(cuuint64_t)s->head_dim * (kv8 ? 1 : 2)};
    const cuuint32_t box[2] = {kv8 ? 128u : 64u, (cuuint32_t)s->block_size};  // 128-byte rows
    const cuuint32_t estr[2] = {1, 1};
    return enc(m, kv8 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_UINT16, 2,
               const_cast<void*>(base), dims, strides, box,
               estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 16-bit [rows][128] tensor as a 2-D map with 16-row x 64-column boxes (one
// 128-byte swizzle atom wide): the tc kernel's K tile is [chunk][token][128 B].
bool encode_2d_map(CUtensorMap* m, const void* base, uint64_t rows) {
    auto enc = get_encode();
    if (!enc) return false;
    const cuuint64_t dims[2] = {128, rows};
    const cuuint64_t strides[1] = {256};
    const cuuint32_t box[2] = {64u, 16u};
    const cuuint32_t estr[2] = {1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, const_cast<void*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 16-bit [rows][128] tensor as a 4-D map (col in chunk, row in an 8-row half,
// chunk, half) whose 64 x 8 x 2 x 2 box is one 16-row block laid out
// [half][chunk][8 rows][128 B]: the tc kernel's K tile (8-row groups of a
// chunk 2048 B apart, one box per block).
bool encode_k4d_map(CUtensorMap* m, const void* base, uint64_t rows) {
    auto enc = get_encode();
    if (!enc) return false;
    const cuuint64_t dims[4] = {64, 8, 2, rows / 8};
    const cuuint64_t strides[3] = {256, 128, 2048};
    const cuuint32_t box[4] = {64u, 8u, 2u, 2u};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT16, 4, const_cast<void*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 16-bit [rows][128] tensor as a 3-D map (col in chunk, row, chunk) whose
// 64 x 16 x 2 box is 16 whole rows laid out [chunk][row][128 B] (q for the tc kernel).
bool encode_rows_3d_map(CUtensorMap* m, const void* base, uint64_t rows) {
    auto enc = get_encode();
    if (!enc) return false;
    const cuuint64_t dims[3] = {64, rows, 2};
    const cuuint64_t strides[2] = {256, 128};
    const cuuint32_t box[3] = {64u, 16u, 2u};
    const cuuint32_t estr[3] = {1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT16, 3, const_cast<void*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// The caller's tensors may live on any device of the process: run on theirs.
pda_status use_device_of(const void* ptr) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
        cudaGetLastError();
        return PDA_ERR_CUDA;
    }
    if (a.type != cudaMemoryTypeDevice && a.type != cudaMemoryTypeManaged) return PDA_OK;
    int cur = -1;
    cudaGetDevice(&cur);
    if (cur != a.device && cudaSetDevice(a.device) != cudaSuccess) return PDA_ERR_CUDA;
    return PDA_OK;
}

// AppendParams of a call; validates the extra pointers.
pda_status make_append(const void* k_new, const void* v_new, void* k_cache, void* v_cache,
                       const pda_shape* s, const pda_options* o, pda::AppendParams* a) {
    if (!k_new || !v_new || !k_cache || !v_cache) return PDA_ERR_NULL;
    if (!aligned16(k_new) || !aligned16(v_new) || !aligned16(k_cache) || !aligned16(v_cache))
        return PDA_ERR_ALIGN;
    const bool kv8 = s->kv_dtype == PDA_E4M3;
    if (kv8 && !(o->k_scale > 0.f && o->v_scale > 0.f)) return PDA_ERR_SHAPE;  // encoding needs the scales
    a->k_new = static_cast<const uint16_t*>(k_new);
    a->v_new = static_cast<const uint16_t*>(v_new);
    a->k = static_cast<uint8_t*>(k_cache);
    a->v = static_cast<uint8_t*>(v_cache);
    a->kv8 = kv8;
    a->bf16 = s->dtype == PDA_BF16;
    a->k_scale = kv8 ? o->k_scale : 1.f;
    a->v_scale = kv8 ? o->v_scale : 1.f;
    return PDA_OK;
}

// Programmatic dependent launch (default on; PDA_PDL=0 turns it off): a grid
// may be scheduled while the previous grid in the stream drains and waits
// (griddepcontrol.wait) before its first global read -- back-to-back steps
// 0.3-10 % faster (profiles/r01_ab_pdl.log)
bool pdl_enabled() {
    static const char* env = std::getenv("PDA_PDL");
    return !(env && std::atoi(env) == 0);
}

pda_status run(const void* q, const void* k_cache, const void* v_cache, const int32_t* bt,
               const int32_t* lens, float scale, void* out, const pda_shape* s,
               const pda_options* o, void* ws, size_t ws_bytes, int32_t* trace, size_t trace_words,
               cudaStream_t stream, void* const* peers = nullptr, int n_peers = 0, int head_off = 0,
               int hq_out = 0, const pda::AppendParams* app = nullptr, uint64_t* stamps = nullptr,
               size_t stamp_words = 0) {
    pda_options o_splitk;
    if ((app || n_peers > 0) && auto_paper(s, o)) {
        // the paper-structure kernel fuses neither the append nor the gather
        o_splitk = *o;
        o_splitk.kernel = PDA_KERNEL_SPLITK;
        o = &o_splitk;
    }
    pda_plan_info pl;
    pda_status st = plan(s, o, &pl);
    if (st != PDA_OK) return st;
    if (!q || !k_cache || !v_cache || !bt || !lens || !out) return PDA_ERR_NULL;
    if (!aligned16(q) || !aligned16(k_cache) || !aligned16(v_cache) || !aligned16(out) ||
        !aligned16(ws))
        return PDA_ERR_ALIGN;
    if (pl.workspace_bytes > 0 && (!ws || ws_bytes < pl.workspace_bytes)) return PDA_ERR_WORKSPACE;
    if (trace && trace_words < (size_t)pl.trace_records * pl.trace_rec_len) return PDA_ERR_SHAPE;
    if (stamps && (pl.kernel != PDA_KERNEL_SPLITK || !trace)) return PDA_ERR_UNSUPPORTED;
    if (stamps && stamp_words < (size_t)pl.trace_records * 3) return PDA_ERR_SHAPE;
    if (s->num_seqs == 0) return PDA_OK;
    st = use_device_of(out);
    if (st != PDA_OK) return st;

    const float scale_log2 = (float)((double)scale * 1.4426950408889634);
    // prefetch = AUTO: Alg. 1 line prefetch d = 4 on the paper-structure kernel, off elsewhere
    const bool pf_auto = o->prefetch == PDA_PF_AUTO;
    const int prefetch_mode = pf_auto ? (pl.kernel == PDA_KERNEL_PAPER ? PDA_PF_LINE_L2 : PDA_PF_OFF) : o->prefetch;
    const int pf_dist = prefetch_mode == PDA_PF_OFF ? 0 : (pf_auto ? 4 : o->prefetch_distance);
    if (trace && cudaMemsetAsync(trace, 0xff, (size_t)pl.trace_records * pl.trace_rec_len * 4,
                                 stream) != cudaSuccess)
        return PDA_ERR_CUDA;

    cudaError_t err;
    if (app && pl.kernel != PDA_KERNEL_SPLITK) {
        // KV append as its own launch ahead of the kernels that do not fuse it
        err = pda::launch_kv_append(*app, bt, lens, s->num_seqs, q_tokens(s), s->num_kv_heads, s->head_dim,
                                    s->max_blocks_per_seq, stream);
        if (err != cudaSuccess) return PDA_ERR_CUDA;
    }
    if (pl.kernel == PDA_KERNEL_PAPER) {
        pda::PaperParams p{};
        p.q = static_cast<const uint16_t*>(q);
        p.k = static_cast<const uint16_t*>(k_cache);
        p.v = static_cast<const uint16_t*>(v_cache);
        p.bt = bt;
        p.lens = lens;
        p.out = out;
        p.trace = trace;
        p.B = s->num_seqs;
        p.Hq = s->num_q_heads;
        p.Hkv = s->num_kv_heads;
        p.g = s->num_q_heads / s->num_kv_heads;
        p.max_blocks = s->max_blocks_per_seq;
        p.out_dtype = s->out_dtype;
        p.pf_mode = prefetch_mode;
        p.pf_dist = pf_dist;
        p.eviction = pl.eviction;
        p.trace_rec_len = pl.trace_rec_len;
        p.scale_log2 = scale_log2;
        err = pda::launch_paper(p, s->dtype == PDA_BF16, s->head_dim, trace != nullptr,
                                dim3(pl.grid_x, pl.grid_y, pl.grid_z), stream);
        return err == cudaSuccess ? PDA_OK : PDA_ERR_CUDA;
    }

    if (pl.kernel == PDA_KERNEL_TC) {
        if (trace || app || n_peers > 0) return PDA_ERR_UNSUPPORTED;
        CUtensorMap tmK, tmV, tmQ;
        const uint64_t krows = (uint64_t)s->num_blocks * s->num_kv_heads * s->block_size;
        if (!encode_k4d_map(&tmK, k_cache, krows) ||
            !encode_cache_map(&tmV, v_cache, s) ||
            !encode_rows_3d_map(&tmQ, q, (uint64_t)s->num_seqs * s->num_q_heads))
            return PDA_ERR_CUDA;
        const size_t gx = (size_t)pl.grid_x;
        const int nh = (s->num_q_heads / s->num_kv_heads) <= 8 ? 8 : 16;
        pda::BalancedParams bp{};
        bp.q = static_cast<const uint16_t*>(q);
        bp.k = static_cast<const uint16_t*>(k_cache);
        bp.v = static_cast<const uint16_t*>(v_cache);
        bp.bt = bt;
        bp.lens = lens;
        bp.out = out;
        char* wsc = static_cast<char*>(ws);
        bp.ws_o = reinterpret_cast<float*>(wsc);
        bp.ws_lse = reinterpret_cast<float*>(wsc + align256(gx * 2 * nh * 128 * 4));
        bp.seq_prefix = reinterpret_cast<long long*>(wsc + align256(gx * 2 * nh * 128 * 4) + align256(gx * 2 * nh * 4));
        bp.B = s->num_seqs;
        bp.Hq = s->num_q_heads;
        bp.Hkv = s->num_kv_heads;
        bp.g = s->num_q_heads / s->num_kv_heads;
        bp.max_blocks = s->max_blocks_per_seq;
        bp.out_dtype = s->out_dtype;
        bp.eviction = pl.eviction;
        bp.scale_log2 = scale_log2;
        bp.pdl = pdl_enabled();
        err = pda::launch_tc(tmK, tmV, tmQ, bp, s->dtype == PDA_BF16, pl.grid_x, stream);
        return err == cudaSuccess ? PDA_OK : PDA_ERR_CUDA;
    }
    CUtensorMap tmK, tmV;
    if (!encode_cache_map(&tmK, k_cache, s) || !encode_cache_map(&tmV, v_cache, s))
        return PDA_ERR_CUDA;
    if (pl.kernel == PDA_KERNEL_BALANCED) {
        const size_t gx = (size_t)pl.grid_x;
        const int n_tiles = (s->num_q_heads / s->num_kv_heads) <= 8 ? 1 : 2;
        const int nh = 8 * n_tiles;
        pda::BalancedParams bp{};
        bp.q = static_cast<const uint16_t*>(q);
        bp.k = static_cast<const uint16_t*>(k_cache);
        bp.v = static_cast<const uint16_t*>(v_cache);
        bp.bt = bt;
        bp.lens = lens;
        bp.out = out;
        char* wsc = static_cast<char*>(ws);
        bp.ws_o = reinterpret_cast<float*>(wsc);
        bp.ws_lse = reinterpret_cast<float*>(wsc + align256(gx * 2 * nh * s->head_dim * 4));
        bp.seq_prefix = reinterpret_cast<long long*>(wsc + align256(gx * 2 * nh * s->head_dim * 4) +
                                                     align256(gx * 2 * nh * 4));
        bp.trace = trace;
        bp.B = s->num_seqs;
        bp.Hq = s->num_q_heads;
        bp.Hkv = s->num_kv_heads;
        bp.g = s->num_q_heads / s->num_kv_heads;
        bp.max_blocks = s->max_blocks_per_seq;
        bp.out_dtype = s->out_dtype;
        bp.pf_mode = prefetch_mode;
        bp.pf_dist = pf_dist;
        bp.eviction = pl.eviction;
        bp.trace_rec_len = pl.trace_rec_len;
        bp.scale_log2 = scale_log2;
        bp.pdl = pdl_enabled() && trace == nullptr;
        err = pda::launch_balanced(tmK, tmV, bp, s->dtype == PDA_BF16, s->head_dim, n_tiles,
                                   pl.smem_stages, trace != nullptr, pl.grid_x, stream);
        return err == cudaSuccess ? PDA_OK : PDA_ERR_CUDA;
    }
    if (pl.kernel == PDA_KERNEL_STREAM) {
        const int w = pl.threads / 32;
        const size_t ns = (size_t)pl.grid_x * w;
        const int nh = (s->num_q_heads / s->num_kv_heads) <= 8 ? 8 : 16;
        pda::StreamParams sp{};
        sp.q = static_cast<const uint16_t*>(q);
        sp.k = static_cast<const uint16_t*>(k_cache);
        sp.v = static_cast<const uint16_t*>(v_cache);
        sp.bt = bt;
        sp.lens = lens;
        sp.out = out;
        char* wsc = static_cast<char*>(ws);
        sp.ws_o = reinterpret_cast<float*>(wsc);
        sp.ws_lse = reinterpret_cast<float*>(wsc + align256(ns * 2 * nh * s->head_dim * 4));
        sp.tickets = reinterpret_cast<uint32_t*>(wsc + align256(ns * 2 * nh * s->head_dim * 4) +
                                                 align256(ns * 2 * nh * 4));
        sp.trace = trace;
        sp.B = s->num_seqs;
        sp.Hq = s->num_q_heads;
        sp.Hkv = s->num_kv_heads;
        sp.g = s->num_q_heads / s->num_kv_heads;
        sp.max_blocks = s->max_blocks_per_seq;
        sp.out_dtype = s->out_dtype;
        sp.pf_mode = prefetch_mode;
        sp.pf_dist = pf_dist;
        sp.eviction = pl.eviction;
        sp.trace_rec_len = pl.trace_rec_len;
        sp.NS = (int)ns;
        sp.scale_log2 = scale_log2;
        err = pda::launch_stream(tmK, tmV, sp, s->dtype == PDA_BF16, s->head_dim, sp.g <= 8 ? 1 : 2,
                                 pl.smem_stages, w, trace != nullptr, pl.grid_x, stream);
        return err == cudaSuccess ? PDA_OK : PDA_ERR_CUDA;
    }
    pda::SplitKParams p{};
    const bool kv8 = s->kv_dtype == PDA_E4M3;
    const float k_scale = kv8 && o->k_scale > 0.f ? o->k_scale : 1.f;
    p.q = static_cast<const uint16_t*>(q);
    p.k = static_cast<const uint8_t*>(k_cache);
    p.v = static_cast<const uint8_t*>(v_cache);
    p.bt = bt;
    p.lens = lens;
    p.outs.n = n_peers > 0 ? n_peers : 1;
    for (int r = 0; r < p.outs.n; ++r) p.outs.ptr[r] = n_peers > 0 ? peers[r] : out;
    p.outs.head_off = n_peers > 0 ? head_off : 0;
    p.outs.Hq_out = n_peers > 0 ? hq_out : s->num_q_heads;
    const size_t o_bytes =
        align256((size_t)s->num_seqs * q_tokens(s) * s->num_q_heads * pl.p_max * s->head_dim * 4);
    const bool via_ws = pl.p_max > 1 && pl.cluster == 0;
    p.ws_o = via_ws ? static_cast<float*>(ws) : nullptr;
    p.ws_lse = via_ws ? reinterpret_cast<float*>(static_cast<char*>(ws) + o_bytes) : nullptr;
    p.cluster = pl.cluster;
    p.pdl = pdl_enabled() && trace == nullptr;
    p.trace = trace;
    p.stamps = stamps;
    p.B = s->num_seqs;
    p.Hq = s->num_q_heads;
    p.Hkv = s->num_kv_heads;
    p.g = s->num_q_heads / s->num_kv_heads;
    p.max_blocks = s->max_blocks_per_seq;
    p.part_tokens = pl.partition_tokens;
    p.p_max = pl.p_max;
    p.out_dtype = s->out_dtype;
    p.pf_mode = prefetch_mode;
    p.pf_dist = pf_dist;
    p.eviction = pl.eviction;
    p.trace_rec_len = pl.trace_rec_len;
    p.q_len = q_tokens(s);
    p.scale_log2 = (float)((double)scale * k_scale * 1.4426950408889634);
    p.out_scale = kv8 && o->v_scale > 0.f ? o->v_scale : 1.f;
    if (app) p.app = *app;  // fused into the split-K kernel (else p.app.k_new == nullptr)
    // the plan chose the tile-split kernel (its 256-thread block); a fused
    // append keeps the two-tile kernel
    p.tile_split = pl.threads == pda::splitk_threads(true, true) && !app;
    const int n_tiles = p.q_len * p.g <= 8 ? 1 : 2;
    err = pda::launch_splitk(tmK, tmV, p, s->dtype == PDA_BF16, s->head_dim, n_tiles,
                             pl.smem_stages, trace != nullptr,
                             dim3(pl.grid_x, pl.grid_y, pl.grid_z), stream, kv8, self_issue(s, o));
    if (err != cudaSuccess) return PDA_ERR_CUDA;
    if (via_ws) {
        // S8 as its own small kernel: measured faster than merging in the last
        // partition CTA (the fused epilogue's fence + ticket cost every CTA a
        // few microseconds)
        pda::CombineParams c{};
        c.ws_o = p.ws_o;
        c.ws_lse = p.ws_lse;
        c.lens = lens;
        c.outs = p.outs;
        c.B = p.B;
        c.Hq = p.Hq;
        c.p_max = p.p_max;
        c.part_tokens = p.part_tokens;
        c.max_tokens = s->max_blocks_per_seq * s->block_size;
        c.q_len = p.q_len;
        c.out_dtype = s->out_dtype;
        c.pdl = p.pdl;
        err = pda::launch_combine(c, s->head_dim, stream);
        if (err != cudaSuccess) return PDA_ERR_CUDA;
    }
    return PDA_OK;
}

}  // namespace

extern "C" {

pda_status pda_check_args(const pda_shape* shape, const pda_options* opt) {
    return validate(shape, opt);
}

pda_status pda_plan(const pda_shape* shape, const pda_options* opt, pda_plan_info* out) {
    if (!out) return PDA_ERR_NULL;
    return plan(shape, opt, out);
}

size_t pda_workspace_bytes(const pda_shape* shape, const pda_options* opt) {
    pda_plan_info pl;
    return plan(shape, opt, &pl) == PDA_OK ? pl.workspace_bytes : 0;
}

pda_status paged_decode_attention(const void* q, const void* k_cache, const void* v_cache,
                                  const int32_t* block_tables, const int32_t* context_lens,
                                  float scale, void* out, const pda_shape* shape,
                                  const pda_options* opt, void* workspace,
                                  size_t workspace_bytes, void* stream) {
    return run(q, k_cache, v_cache, block_tables, context_lens, scale, out, shape, opt, workspace,
               workspace_bytes, nullptr, 0, static_cast<cudaStream_t>(stream));
}

pda_status paged_decode_attention_trace(const void* q, const void* k_cache, const void* v_cache,
                                        const int32_t* block_tables,
                                        const int32_t* context_lens, float scale, void* out,
                                        const pda_shape* shape, const pda_options* opt,
                                        void* workspace, size_t workspace_bytes, int32_t* trace,
                                        size_t trace_words, void* stream) {
    if (!trace) return PDA_ERR_NULL;
    return run(q, k_cache, v_cache, block_tables, context_lens, scale, out, shape, opt, workspace,
               workspace_bytes, trace, trace_words, static_cast<cudaStream_t>(stream));
}

pda_status paged_decode_attention_timeline(const void* q, const void* k_cache, const void* v_cache,
                                           const int32_t* block_tables, const int32_t* context_lens,
                                           float scale, void* out, const pda_shape* shape,
                                           const pda_options* opt, void* workspace, size_t workspace_bytes,
                                           int32_t* trace, size_t trace_words, uint64_t* stamps,
                                           size_t stamp_words, void* stream) {
    if (!trace || !stamps) return PDA_ERR_NULL;
    return run(q, k_cache, v_cache, block_tables, context_lens, scale, out, shape, opt, workspace,
               workspace_bytes, trace, trace_words, static_cast<cudaStream_t>(stream), nullptr, 0, 0, 0,
               nullptr, stamps, stamp_words);
}

pda_status paged_decode_attention_gather(const void* q, const void* k_cache, const void* v_cache,
                                         const int32_t* block_tables, const int32_t* context_lens,
                                         float scale, void* const* out_peers, int32_t n_peers,
                                         int32_t head_offset, int32_t total_q_heads,
                                         const pda_shape* shape, const pda_options* opt, void* workspace,
                                         size_t workspace_bytes, void* stream) {
    pda_status st = validate(shape, opt);
    if (st != PDA_OK) return st;
    if (!out_peers) return PDA_ERR_NULL;
    if (n_peers < 1 || n_peers > pda::kMaxPeers || head_offset < 0 ||
        head_offset + shape->num_q_heads > total_q_heads)
        return PDA_ERR_SHAPE;
    if (opt->kernel != PDA_KERNEL_AUTO && opt->kernel != PDA_KERNEL_SPLITK) return PDA_ERR_UNSUPPORTED;
    for (int r = 0; r < n_peers; ++r) {
        if (!out_peers[r]) return PDA_ERR_NULL;
        if (!aligned16(out_peers[r])) return PDA_ERR_ALIGN;
    }
    return run(q, k_cache, v_cache, block_tables, context_lens, scale, out_peers[0], shape, opt, workspace,
               workspace_bytes, nullptr, 0, static_cast<cudaStream_t>(stream), out_peers, n_peers, head_offset,
               total_q_heads);
}

pda_status pda_kv_append(const void* k_new, const void* v_new, void* k_cache, void* v_cache,
                         const int32_t* block_tables, const int32_t* context_lens, const pda_shape* shape,
                         const pda_options* opt, void* stream) {
    pda_status st = validate(shape, opt);
    if (st != PDA_OK) return st;
    if (!block_tables || !context_lens) return PDA_ERR_NULL;
    pda::AppendParams a{};
    st = make_append(k_new, v_new, k_cache, v_cache, shape, opt, &a);
    if (st != PDA_OK) return st;
    if (shape->num_seqs == 0) return PDA_OK;
    st = use_device_of(k_cache);
    if (st != PDA_OK) return st;
    return pda::launch_kv_append(a, block_tables, context_lens, shape->num_seqs, q_tokens(shape),
                                 shape->num_kv_heads, shape->head_dim, shape->max_blocks_per_seq,
                                 static_cast<cudaStream_t>(stream)) == cudaSuccess
               ? PDA_OK
               : PDA_ERR_CUDA;
}

pda_status paged_decode_attention_append(const void* q, const void* k_new, const void* v_new, void* k_cache,
                                         void* v_cache, const int32_t* block_tables,
                                         const int32_t* context_lens, float scale, void* out,
                                         const pda_shape* shape, const pda_options* opt, void* workspace,
                                         size_t workspace_bytes, void* stream) {
    pda_status st = validate(shape, opt);
    if (st != PDA_OK) return st;
    pda::AppendParams a{};
    st = make_append(k_new, v_new, k_cache, v_cache, shape, opt, &a);
    if (st != PDA_OK) return st;
    return run(q, k_cache, v_cache, block_tables, context_lens, scale, out, shape, opt, workspace,
               workspace_bytes, nullptr, 0, static_cast<cudaStream_t>(stream), nullptr, 0, 0, 0, &a);
}

pda_status pda_validate_inputs(const int32_t* block_tables, const int32_t* context_lens,
                               const pda_shape* shape, int64_t* counts, void* stream) {
    if (!shape || !block_tables || !context_lens || !counts) return PDA_ERR_NULL;
    if (shape->num_seqs < 0 || shape->max_blocks_per_seq <= 0 || shape->num_blocks <= 0)
        return PDA_ERR_SHAPE;
    if (shape->block_size != pda::kBlockSize) return PDA_ERR_UNSUPPORTED;
    pda_status st = use_device_of(counts);
    if (st != PDA_OK) return st;
    return pda::launch_validate(block_tables, context_lens, shape->num_seqs, shape->max_blocks_per_seq,
                                shape->num_blocks, reinterpret_cast<long long*>(counts),
                                static_cast<cudaStream_t>(stream)) == cudaSuccess
               ? PDA_OK
               : PDA_ERR_CUDA;
}

pda_status pda_decode_step_host(const void* q_host, const int32_t* block_tables_host,
                                const int32_t* context_lens_host, void* out_host, void* q_dev,
                                int32_t* block_tables_dev, int32_t* context_lens_dev,
                                void* out_dev, const void* k_cache, const void* v_cache,
                                float scale, const pda_shape* shape, const pda_options* opt,
                                void* workspace, size_t workspace_bytes, void* stream) {
    pda_status st = validate(shape, opt);
    if (st != PDA_OK) return st;
    if (!q_host || !block_tables_host || !context_lens_host || !out_host || !q_dev ||
        !block_tables_dev || !context_lens_dev || !out_dev)
        return PDA_ERR_NULL;
    st = use_device_of(out_dev);
    if (st != PDA_OK) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const size_t B = shape->num_seqs;
    const size_t q_bytes = B * q_tokens(shape) * shape->num_q_heads * shape->head_dim * 2;
    const size_t bt_bytes = B * shape->max_blocks_per_seq * 4;
    const size_t out_bytes = B * q_tokens(shape) * shape->num_q_heads * shape->head_dim * elem_bytes(shape->out_dtype);
    if (cudaMemcpyAsync(q_dev, q_host, q_bytes, cudaMemcpyHostToDevice, s) != cudaSuccess ||
        cudaMemcpyAsync(block_tables_dev, block_tables_host, bt_bytes, cudaMemcpyHostToDevice, s) !=
            cudaSuccess ||
        cudaMemcpyAsync(context_lens_dev, context_lens_host, B * 4, cudaMemcpyHostToDevice, s) !=
            cudaSuccess)
        return PDA_ERR_CUDA;
    st = run(q_dev, k_cache, v_cache, block_tables_dev, context_lens_dev, scale, out_dev, shape, opt,
             workspace, workspace_bytes, nullptr, 0, s);
    if (st != PDA_OK) return st;
    if (cudaMemcpyAsync(out_host, out_dev, out_bytes, cudaMemcpyDeviceToHost, s) != cudaSuccess)
        return PDA_ERR_CUDA;
    return PDA_OK;
}

pda_status pda_decode_step_host_async(const void* q_host, const int32_t* block_tables_host,
                                      const int32_t* context_lens_host, void* out_host, void* q_dev,
                                      int32_t* block_tables_dev, int32_t* context_lens_dev, void* out_dev,
                                      const void* k_cache, const void* v_cache, float scale,
                                      const pda_shape* shape, const pda_options* opt, void* workspace,
                                      size_t workspace_bytes, void* compute_stream, void* copy_stream,
                                      void* inputs_ready, void* step_done) {
    pda_status st = validate(shape, opt);
    if (st != PDA_OK) return st;
    if (!q_host || !block_tables_host || !context_lens_host || !out_host || !q_dev ||
        !block_tables_dev || !context_lens_dev || !out_dev || !inputs_ready || !step_done)
        return PDA_ERR_NULL;
    st = use_device_of(out_dev);
    if (st != PDA_OK) return st;
    cudaStream_t cs = static_cast<cudaStream_t>(compute_stream);
    cudaStream_t xs = static_cast<cudaStream_t>(copy_stream);
    cudaEvent_t in_ev = static_cast<cudaEvent_t>(inputs_ready);
    cudaEvent_t done_ev = static_cast<cudaEvent_t>(step_done);
    const size_t B = shape->num_seqs;
    const size_t q_bytes = B * q_tokens(shape) * shape->num_q_heads * shape->head_dim * 2;
    const size_t bt_bytes = B * shape->max_blocks_per_seq * 4;
    const size_t out_bytes = B * q_tokens(shape) * shape->num_q_heads * shape->head_dim * elem_bytes(shape->out_dtype);
    // inputs on the copy stream, the kernels on the compute stream once they landed,
    // the output back on the copy stream once the kernels finished
    if (cudaMemcpyAsync(q_dev, q_host, q_bytes, cudaMemcpyHostToDevice, xs) != cudaSuccess ||
        cudaMemcpyAsync(block_tables_dev, block_tables_host, bt_bytes, cudaMemcpyHostToDevice, xs) !=
            cudaSuccess ||
        cudaMemcpyAsync(context_lens_dev, context_lens_host, B * 4, cudaMemcpyHostToDevice, xs) != cudaSuccess ||
        cudaEventRecord(in_ev, xs) != cudaSuccess || cudaStreamWaitEvent(cs, in_ev, 0) != cudaSuccess)
        return PDA_ERR_CUDA;
    st = run(q_dev, k_cache, v_cache, block_tables_dev, context_lens_dev, scale, out_dev, shape, opt, workspace,
             workspace_bytes, nullptr, 0, cs);
    if (st != PDA_OK) return st;
    if (cudaEventRecord(done_ev, cs) != cudaSuccess || cudaStreamWaitEvent(xs, done_ev, 0) != cudaSuccess ||
        cudaMemcpyAsync(out_host, out_dev, out_bytes, cudaMemcpyDeviceToHost, xs) != cudaSuccess)
        return PDA_ERR_CUDA;
    return PDA_OK;
}

pda_status pda_read_roofline_mode(const void* buf, size_t bytes, void* sink, int32_t mode, void* stream) {
    if (!buf || !sink) return PDA_ERR_NULL;
    if (!aligned16(buf) || !aligned16(sink)) return PDA_ERR_ALIGN;
    if (mode < 0 || mode > 2) return PDA_ERR_SHAPE;
    pda_status st = use_device_of(buf);
    if (st != PDA_OK) return st;
    int dev = 0, sms = kDefaultSms;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return pda::launch_read_roofline(buf, bytes, sink, sms, mode, static_cast<cudaStream_t>(stream)) ==
                   cudaSuccess
               ? PDA_OK
               : PDA_ERR_CUDA;
}

pda_status pda_read_roofline(const void* buf, size_t bytes, void* sink, void* stream) {
    return pda_read_roofline_mode(buf, bytes, sink, 0, stream);
}

const char* pda_status_string(pda_status status) {
    switch (status) {
        case PDA_OK: return "PDA_OK";
        case PDA_ERR_NULL: return "PDA_ERR_NULL: a required pointer is NULL";
        case PDA_ERR_SHAPE: return "PDA_ERR_SHAPE: inconsistent or out-of-range sizes/options";
        case PDA_ERR_UNSUPPORTED: return "PDA_ERR_UNSUPPORTED: head_dim/block_size/group/dtype not supported";
        case PDA_ERR_ALIGN: return "PDA_ERR_ALIGN: a base pointer is not 16-byte aligned";
        case PDA_ERR_WORKSPACE: return "PDA_ERR_WORKSPACE: workspace missing or too small";
        case PDA_ERR_CUDA: return "PDA_ERR_CUDA: a CUDA call or kernel launch failed";
    }
    return "PDA_ERR_UNKNOWN";
}

int32_t pda_abi_version(void) { return 14; }

}  // extern "C"
