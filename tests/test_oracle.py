"""Pins of the fp64 oracle against things other than itself (-m "not gpu").

Each test names what fixes the expected value: the paper's printed numbers
(tests/golden/paper_constants.txt), closed forms, invariants, library
routines on contiguous gathers (numpy / torch fp64), or brute force.
"""
import math
import os

import numpy as np
import pytest
import torch

import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "paper_constants.txt")


def golden():
    vals = {}
    for line in open(GOLDEN):
        line = line.split("#", 1)[0].strip()
        if line:
            k, v = line.split("=")
            vals[k.strip()] = int(v)
    return vals


def contiguous_reference(inp, b, h):
    """Gather row (b, h)'s K/V into contiguous fp64 arrays with plain indexing
    and compute softmax attention with numpy (library primitives only)."""
    cfg = inp["cfg"]
    g = cfg.num_q_heads // cfg.num_kv_heads
    kvh = h // g
    L = int(inp["context_lens"][b])
    bs = cfg.block_size
    k = inp["k_cache"].double().numpy()
    v = inp["v_cache"].double().numpy()
    q = inp["q"].double().numpy()[b, h]
    bt = inp["block_tables"].numpy()
    if L == 0:
        return np.zeros(cfg.head_dim)
    K = np.stack([k[bt[b, t // bs], kvh, t % bs] for t in range(L)])
    V = np.stack([v[bt[b, t // bs], kvh, t % bs] for t in range(L)])
    s = inp["scale"] * (K @ q)
    w = np.exp(s - s.max())
    w /= w.sum()
    return w @ V


def run_oracle(oracle_mod, inp, **kw):
    return oracle_mod.paged_attention(inp["q"], inp["k_cache"], inp["v_cache"], inp["block_tables"],
                                      inp["context_lens"], inp["scale"], inp["cfg"].dtype, **kw)


CFGS = [
    synth.C1_TINY,
    synth.Config("mha_d128", 3, 4, 4, 128, (1, 17, 100), "fp16", poison_blocks=2),
    synth.Config("gqa_bf16", 2, 8, 2, 64, (33, 48), "bf16", poison_blocks=1),
    synth.Config("gqa8", 2, 16, 2, 128, (5, 70), "bf16"),
    synth.Config("with_zero", 3, 2, 1, 64, (0, 16, 31), "fp16"),
]


@pytest.mark.parametrize("cfg", CFGS, ids=lambda c: c.name)
def test_oracle_vs_contiguous_numpy(oracle_mod, cfg):
    inp = synth.make_inputs(cfg, seed=3)
    out = run_oracle(oracle_mod, inp)
    assert np.isfinite(out).all(), "NaN poison leaked into the oracle output"
    for b in range(cfg.num_seqs):
        for h in range(cfg.num_q_heads):
            ref = contiguous_reference(inp, b, h)
            np.testing.assert_allclose(out[b, h], ref, rtol=0, atol=1e-12)


def test_oracle_vs_torch_sdpa(oracle_mod):
    """Library routine: torch SDPA in fp64 on the contiguous gather (GQA expanded)."""
    cfg = synth.Config("sdpa", 2, 8, 2, 64, (40, 64), "fp16")
    inp = synth.make_inputs(cfg, seed=5, poison=False)
    out = run_oracle(oracle_mod, inp)
    g = cfg.group
    for b in range(cfg.num_seqs):
        L = int(inp["context_lens"][b])
        ids = inp["block_tables"][b, : math.ceil(L / 16)].long()
        K = inp["k_cache"][ids].double().permute(1, 0, 2, 3).reshape(cfg.num_kv_heads, -1, 64)[:, :L]
        V = inp["v_cache"][ids].double().permute(1, 0, 2, 3).reshape(cfg.num_kv_heads, -1, 64)[:, :L]
        K = K.repeat_interleave(g, 0)
        V = V.repeat_interleave(g, 0)
        q = inp["q"][b].double().unsqueeze(1)  # [Hq, 1, D]
        ref = torch.nn.functional.scaled_dot_product_attention(q, K, V, scale=inp["scale"])
        np.testing.assert_allclose(out[b], ref[:, 0].numpy(), rtol=0, atol=1e-12)


def test_fp16_decode_all_patterns(oracle_mod):
    bits = np.arange(65536, dtype=np.uint16)
    ref = bits.view(np.float16).astype(np.float64)
    got = np.array([oracle_mod.fp16_to_f64(int(x)) for x in bits])
    nan = np.isnan(ref)
    assert (np.isnan(got) == nan).all()
    assert (got[~nan] == ref[~nan]).all()


def test_bf16_decode_all_patterns(oracle_mod):
    bits = np.arange(65536, dtype=np.int32).astype(np.int16)
    ref = torch.from_numpy(bits).view(torch.bfloat16).double().numpy()
    got = np.array([oracle_mod.bf16_to_f64(int(x) & 0xFFFF) for x in bits])
    nan = np.isnan(ref)
    assert (np.isnan(got) == nan).all()
    assert (got[~nan] == ref[~nan]).all()


def test_permutation_invariance_bitwise(oracle_mod):
    inp = synth.make_inputs(synth.C1_TINY, seed=0)
    a = run_oracle(oracle_mod, inp)
    for s in range(3):
        b = run_oracle(oracle_mod, synth.permute_placement(inp, seed=11 + s))
        assert np.array_equal(a, b)


def test_context_len_one_returns_v_row(oracle_mod):
    cfg = synth.Config("l1", 2, 4, 2, 64, (1, 1), "bf16", poison_blocks=3)
    inp = synth.make_inputs(cfg, seed=1)
    out = run_oracle(oracle_mod, inp)
    for b in range(2):
        for h in range(4):
            vrow = inp["v_cache"][int(inp["block_tables"][b, 0]), h // 2, 0].double().numpy()
            assert np.array_equal(out[b, h], vrow)


def test_zero_query_gives_mean_of_v(oracle_mod):
    cfg = synth.Config("q0", 1, 2, 1, 64, (45,), "fp16")
    inp = synth.make_inputs(cfg, seed=2)
    inp["q"].zero_()
    out = run_oracle(oracle_mod, inp)
    ids = inp["block_tables"][0, :3].long()
    V = inp["v_cache"][ids, 0].double().reshape(-1, 64)[:45]
    np.testing.assert_allclose(out[0, 0], V.mean(0).numpy(), rtol=0, atol=1e-14)
    np.testing.assert_allclose(out[0, 1], V.mean(0).numpy(), rtol=0, atol=1e-14)


def test_constant_v_gives_v(oracle_mod):
    cfg = synth.Config("cv", 2, 4, 4, 128, (29, 64), "bf16")
    inp = synth.make_inputs(cfg, seed=4, poison=False)
    inp["v_cache"].fill_(0.375)
    out = run_oracle(oracle_mod, inp)
    np.testing.assert_allclose(out, 0.375, rtol=0, atol=1e-14)


def test_two_token_closed_form(oracle_mod):
    """s0 = 0, s1 = ln 3 => weights (1/4, 3/4); v0 = 1, v1 = -1 => out = -1/2."""
    cfg = synth.Config("two", 1, 1, 1, 64, (2,), "fp16")
    inp = synth.make_inputs(cfg, seed=0, poison=False)
    inp["q"].zero_()
    inp["q"][0, 0, 0] = 1.0
    blk = int(inp["block_tables"][0, 0])
    inp["k_cache"][blk].zero_()
    inp["k_cache"][blk, 0, 1, 0] = 1.0
    inp["v_cache"][blk, 0, 0] = 1.0
    inp["v_cache"][blk, 0, 1] = -1.0
    inp["scale"] = math.log(3.0)
    out = run_oracle(oracle_mod, inp)
    np.testing.assert_allclose(out[0, 0], -0.5, rtol=0, atol=1e-15)
    w = oracle_mod.attention_weights(inp["q"], inp["k_cache"], inp["block_tables"], inp["context_lens"],
                                     0, 0, inp["scale"], "fp16")
    np.testing.assert_allclose(w, [0.25, 0.75], rtol=0, atol=1e-15)


def test_weights_sum_to_one(oracle_mod):
    inp = synth.make_inputs(synth.C1_TINY, seed=7)
    for b in range(2):
        for h in range(4):
            w = oracle_mod.attention_weights(inp["q"], inp["k_cache"], inp["block_tables"],
                                             inp["context_lens"], b, h, inp["scale"], "fp16")
            assert len(w) == int(inp["context_lens"][b])
            assert abs(w.sum() - 1.0) < 1e-12 and (w > 0).all()


@pytest.mark.parametrize("t_star", [0, 5, 15, 16, 31, 36])
def test_needle(oracle_mod, t_star):
    """A key aligned with q at position t* dominates: out ~= v_{t*}."""
    cfg = synth.Config("needle", 1, 1, 1, 64, (37,), "fp16")
    inp = synth.make_inputs(cfg, seed=9)
    inp["q"].zero_()
    inp["q"][0, 0, 0] = 1.0
    bt = inp["block_tables"][0]
    for t in range(37):
        inp["k_cache"][int(bt[t // 16]), 0, t % 16, 0] = 40.0 if t == t_star else 0.0
    inp["scale"] = 1.0
    out = run_oracle(oracle_mod, inp)
    v = inp["v_cache"][int(bt[t_star // 16]), 0, t_star % 16].double().numpy()
    np.testing.assert_allclose(out[0, 0], v, rtol=0, atol=1e-14)


def test_zero_length_row_is_zero(oracle_mod):
    cfg = synth.Config("z", 2, 2, 1, 64, (0, 3), "fp16")
    out = run_oracle(oracle_mod, synth.make_inputs(cfg, seed=0))
    assert (out[0] == 0).all() and np.isfinite(out).all()


def test_gqa_group_sharing(oracle_mod):
    """Identical q across a GQA group => identical outputs; and GQA equals the
    MHA problem with each KV head repeated g times."""
    cfg = synth.Config("gqa", 2, 8, 2, 64, (21, 50), "fp16")
    inp = synth.make_inputs(cfg, seed=6)
    inp["q"][:, 1:4] = inp["q"][:, 0:1]
    out = run_oracle(oracle_mod, inp)
    for h in (1, 2, 3):
        assert np.array_equal(out[:, h], out[:, 0])
    mha = dict(inp)
    mha["k_cache"] = inp["k_cache"].repeat_interleave(4, dim=1)
    mha["v_cache"] = inp["v_cache"].repeat_interleave(4, dim=1)
    mha["cfg"] = cfg.with_heads(8, 8)
    assert np.array_equal(run_oracle(oracle_mod, mha), out)


def test_rows_subset(oracle_mod):
    inp = synth.make_inputs(synth.C1_TINY, seed=1)
    full = run_oracle(oracle_mod, inp)
    part = run_oracle(oracle_mod, inp, rows=[0, 5, 7])
    for r in (0, 5, 7):
        assert np.array_equal(part.reshape(-1, 64)[r], full.reshape(-1, 64)[r])
    assert np.isnan(part.reshape(-1, 64)[1]).all()


def test_sample_rows_compaction(oracle_mod):
    cfg = synth.Config("s", 4, 4, 2, 64, (20, 64, 3, 40), "bf16")
    inp = synth.make_inputs(cfg, seed=8)
    full = run_oracle(oracle_mod, inp)
    sub = synth.sample_rows(inp, [1, 3])
    out = run_oracle(oracle_mod, sub)
    assert np.array_equal(out[0], full[1]) and np.array_equal(out[1], full[3])


# ---- paper constants (tests/golden/paper_constants.txt) ---------------------

def test_eq1_eq2_and_residency_bound(oracle_mod):
    g = golden()
    mb = oracle_mod.eq1_block_bytes(g["table2_b"], g["table2_d_h"], g["table2_T_block"])
    assert mb == g["eq1_block_bytes_llama2_7b"]
    mt = oracle_mod.eq2_total_bytes(mb, g["table2_N_thread"], g["table2_H"], 1)
    assert mt == g["eq2_total_bytes_llama2_7b_b1"]
    assert oracle_mod.l2_residency_bound(60 * 2**20, mt) == g["l2_residency_bound_60MB"]


# ---- bookkeeping plans --------------------------------------------------------

def test_plan_splitk_hand_example(oracle_mod):
    """L = 37 tokens, P = 32: partitions [0,32) -> blocks 0,1 and [32,37) -> block 2;
    distance 1 prefetches block j+1 while issuing block j inside the unit only."""
    bt = np.array([[7, 3, 9, 1]], dtype=np.int32)
    lens = np.array([37], dtype=np.int32)
    recs = oracle_mod.plan_splitk(bt, lens, num_kv_heads=1, block_size=16, partition_tokens=32,
                                  p_max=2, prefetch_distance=1)
    r0, r1 = recs[0, 0, 0], recs[0, 0, 1]
    R = 2
    assert list(r0[:4]) == [0, 32, 2, 1]
    assert list(r0[4:4 + R]) == [7, 3] and list(r0[4 + R:]) == [3, -1]
    assert list(r1[:4]) == [32, 37, 1, 0]
    assert list(r1[4:4 + R]) == [9, -1] and list(r1[4 + R:]) == [-1, -1]


def test_plan_splitk_empty_unit(oracle_mod):
    bt = np.array([[4, 5, 6, 7]], dtype=np.int32)
    lens = np.array([20], dtype=np.int32)
    recs = oracle_mod.plan_splitk(bt, lens, 1, 16, 16, 4, 2)
    assert list(recs[0, 0, 2, :4]) == [20, 20, 0, 0]
    assert list(recs[0, 0, 3, :4]) == [20, 20, 0, 0]
    assert list(recs[0, 0, 1, :4]) == [16, 20, 1, 0]


def test_plan_paper_guard_counts(oracle_mod):
    """one block per warp => zero prefetches; two blocks per warp
    => exactly one prefetch per warp, for its second block (Alg. 1 guard)."""
    w = 4
    bt = np.arange(16, dtype=np.int32)[None, :] + 100
    one = oracle_mod.plan_paper(bt, np.array([16 * w], np.int32), 1, 16, w, w)
    assert (one[0, 0, :, 2] == 1).all() and (one[0, 0, :, 3] == 0).all()
    two = oracle_mod.plan_paper(bt, np.array([2 * 16 * w], np.int32), 1, 16, w, w)
    R = two.shape[-1] // 2 - 2
    for wi in range(w):
        rec = two[0, 0, wi]
        assert rec[2] == 2 and rec[3] == 1
        assert rec[4 + R] == 100 + wi + w  # prefetch target = the warp's second block
        assert list(rec[4:6]) == [100 + wi, 100 + wi + w]
    # total prefetches across warps = max(0, e - w) for d = w
    for e in range(0, 17):
        p = oracle_mod.plan_paper(bt, np.array([16 * e], np.int32), 1, 16, w, w)
        assert p[0, 0, :, 3].sum() == max(0, e - w)
    # a single-block sequence: warp 0 loads it, no prefetch
    p = oracle_mod.plan_paper(bt, np.array([16], np.int32), 1, 16, w, w)
    assert p[0, 0, 0, 2] == 1 and p[0, 0, :, 3].sum() == 0 and (p[0, 0, 1:, 2] == 0).all()


def test_plan_splitk_prefetch_off(oracle_mod):
    bt = np.arange(8, dtype=np.int32)[None, :]
    recs = oracle_mod.plan_splitk(bt, np.array([128], np.int32), 1, 16, 128, 1, 0)
    assert recs[0, 0, 0, 2] == 8 and recs[0, 0, 0, 3] == 0
    assert list(recs[0, 0, 0, 4:12]) == list(range(8))


def test_plan_stream_hand_example(oracle_mod):
    """T = 4 items (row 0: 3 blocks, row 1: 1 block), 2 streams: ranges [0,2), [2,4).
    Row 0 is split after its second block; with d = 1 only block 0 (item 0 -> 1
    inside [0,2)) is prefetched-for."""
    bt = np.array([[10, 11, 12], [20, -1, -1]], dtype=np.int32)
    lens = np.array([40, 16], dtype=np.int32)
    r = oracle_mod.plan_stream(bt, lens, 1, 16, 2, 1)
    R = 3
    row0, row1 = r[0, 0], r[1, 0]
    assert list(row0[:4]) == [0, 40, 3, 1]
    assert list(row0[4:4 + R]) == [10, 11, 12] and list(row0[4 + R:]) == [11, -1, -1]
    assert list(row1[:4]) == [0, 16, 1, 0] and list(row1[4:4 + R]) == [20, -1, -1]
    # more streams than items: every item alone, nothing can be prefetched
    r = oracle_mod.plan_stream(bt, lens, 1, 16, 64, 1)
    assert r[0, 0, 3] == 0 and r[1, 0, 3] == 0
    # one stream: a whole row is one segment -> prefetches = n - d per row
    r = oracle_mod.plan_stream(bt, lens, 1, 16, 1, 1)
    assert r[0, 0, 3] == 2 and list(r[0, 0, 4 + R:]) == [11, 12, -1]


def test_plan_stream_covers_every_block_once(oracle_mod):
    rng = np.random.default_rng(0)
    B, Hkv, mb = 5, 3, 9
    bt = rng.permutation(B * mb).reshape(B, mb).astype(np.int32)
    lens = np.array([0, 1, 144, 17, 70], dtype=np.int32)
    for ns in (1, 2, 7, 40, 1000):
        r = oracle_mod.plan_stream(bt, lens, Hkv, 16, ns, 3)
        for b in range(B):
            n = -(-int(lens[b]) // 16)
            for h in range(Hkv):
                if n == 0:
                    assert (r[b, h] == -1).all()
                    continue
                assert r[b, h, 2] == n and list(r[b, h, 4:4 + n]) == list(bt[b, :n])
                assert (r[b, h, 4 + n:4 + mb] == -1).all()
                # a prefetch target is always the block d ahead in the same row
                pf = r[b, h, 4 + mb:]
                for j in range(mb):
                    if pf[j] != -1:
                        assert j + 3 < n and pf[j] == bt[b, j + 3]
                assert r[b, h, 3] == (pf != -1).sum()


# ---- FP8 (e4m3) KV cache variant -------------------------

def test_e4m3_decode_all_codes(oracle_mod):
    ref = torch.arange(256, dtype=torch.uint8).view(torch.float8_e4m3fn).double().numpy()
    got = np.array([oracle_mod.e4m3_to_f64(c) for c in range(256)])
    nan = np.isnan(ref)
    assert (np.isnan(got) == nan).all() and nan.sum() == 2
    assert (got[~nan] == ref[~nan]).all()
    assert np.nanmax(got) == 448.0


@pytest.mark.parametrize("qdt", ["fp16", "bf16"])
def test_kv8_oracle_vs_dequantised_numpy(oracle_mod, qdt):
    cfg = synth.Config("kv8", 3, 8, 2, 128, (37, 1, 90), qdt, poison_blocks=2)
    inp = synth.quantize_kv_e4m3(synth.make_inputs(cfg, seed=4), k_scale=1 / 200, v_scale=1 / 300)
    out = oracle_mod.paged_attention_kv8(inp["q"], inp["k_cache"], inp["v_cache"], inp["k_scale"],
                                         inp["v_scale"], inp["block_tables"], inp["context_lens"],
                                         inp["scale"], qdt)
    assert np.isfinite(out).all()
    deq = dict(inp)
    deq["k_cache"] = inp["k_cache"].view(torch.float8_e4m3fn).double() * inp["k_scale"]
    deq["v_cache"] = inp["v_cache"].view(torch.float8_e4m3fn).double() * inp["v_scale"]
    for b in range(3):
        for h in range(8):
            np.testing.assert_allclose(out[b, h], contiguous_reference(deq, b, h), rtol=0, atol=1e-12)


def test_kv8_context_one_is_scaled_v_row(oracle_mod):
    cfg = synth.Config("kv8_l1", 1, 2, 1, 64, (1,), "fp16")
    inp = synth.quantize_kv_e4m3(synth.make_inputs(cfg, seed=1), v_scale=0.125)
    out = oracle_mod.paged_attention_kv8(inp["q"], inp["k_cache"], inp["v_cache"], inp["k_scale"],
                                         inp["v_scale"], inp["block_tables"], inp["context_lens"],
                                         inp["scale"], "fp16")
    codes = inp["v_cache"][int(inp["block_tables"][0, 0]), 0, 0]
    vrow = codes.view(torch.float8_e4m3fn).double().numpy() * 0.125
    assert np.array_equal(out[0, 0], vrow) and np.array_equal(out[0, 1], vrow)


# ---- multi-token (speculative) decode --------------------

def causal_reference(inp, b, i, h):
    """numpy: query token i of sequence b at position L - q_len + i attends to
    tokens t <= that position (explicit causal mask over the contiguous gather)."""
    cfg = inp["cfg"]
    q_len = inp["q_len"]
    g = cfg.num_q_heads // cfg.num_kv_heads
    L = int(inp["context_lens"][b])
    bs = cfg.block_size
    k = inp["k_cache"].double().numpy()
    v = inp["v_cache"].double().numpy()
    bt = inp["block_tables"].numpy()
    pos = L - q_len + i
    if pos < 0:
        return np.zeros(cfg.head_dim)
    K = np.stack([k[bt[b, t // bs], h // g, t % bs] for t in range(L)])
    V = np.stack([v[bt[b, t // bs], h // g, t % bs] for t in range(L)])
    s = inp["scale"] * (K @ inp["q"].double().numpy()[b, i, h])
    s[np.arange(L) > pos] = -np.inf
    w = np.exp(s - s.max())
    return (w / w.sum()) @ V


@pytest.mark.parametrize("q_len", [1, 2, 4])
def test_mq_oracle_vs_causal_numpy(oracle_mod, q_len):
    cfg = synth.Config("mq", 3, 8, 2, 64, (37, 2, 70), "fp16", poison_blocks=2)
    inp = synth.with_query_tokens(synth.make_inputs(cfg, seed=5), q_len)
    out = oracle_mod.paged_attention_mq(inp["q"], inp["k_cache"], inp["v_cache"], inp["block_tables"],
                                        inp["context_lens"], inp["scale"], "fp16")
    assert np.isfinite(out).all()
    for b in range(3):
        for i in range(q_len):
            for h in range(8):
                np.testing.assert_allclose(out[b, i, h], causal_reference(inp, b, i, h), rtol=0, atol=1e-12)


def test_mq_len_one_is_single_query_bitwise(oracle_mod):
    inp = synth.make_inputs(synth.C1_TINY, seed=3)
    one = oracle_mod.paged_attention(inp["q"], inp["k_cache"], inp["v_cache"], inp["block_tables"],
                                     inp["context_lens"], inp["scale"], "fp16")
    mq = oracle_mod.paged_attention_mq(inp["q"][:, None], inp["k_cache"], inp["v_cache"], inp["block_tables"],
                                       inp["context_lens"], inp["scale"], "fp16")
    assert np.array_equal(mq[:, 0], one)


def test_mq_last_token_sees_everything_first_token_sees_prefix(oracle_mod):
    """token q_len-1 == single-query over L tokens; token 0 == single-query over L-q_len+1."""
    cfg = synth.Config("mq2", 2, 4, 4, 64, (40, 19), "bf16")
    inp = synth.with_query_tokens(synth.make_inputs(cfg, seed=6), 3)
    mq = oracle_mod.paged_attention_mq(inp["q"], inp["k_cache"], inp["v_cache"], inp["block_tables"],
                                       inp["context_lens"], inp["scale"], "bf16")
    last = oracle_mod.paged_attention(inp["q"][:, 2], inp["k_cache"], inp["v_cache"], inp["block_tables"],
                                      inp["context_lens"], inp["scale"], "bf16")
    first = oracle_mod.paged_attention(inp["q"][:, 0], inp["k_cache"], inp["v_cache"], inp["block_tables"],
                                       inp["context_lens"] - 2, inp["scale"], "bf16")
    assert np.array_equal(mq[:, 2], last) and np.array_equal(mq[:, 0], first)


# ---------------------------------------------------------------------------
# Device-data validation, e4m3 encoding and the KV append
# ---------------------------------------------------------------------------

def test_validate_hand_example(oracle_mod):
    # B=3, max_blocks=3, bs=16, pool of 10 blocks
    bt = np.array([[1, 2, 99],      # L=20 references blocks 0,1 -> ids 1,2 fine (99 unreferenced)
                   [-1, 4, 5],      # L=40 references 3 blocks -> id -1 bad
                   [10, 11, 3]],    # L=60 > 48: bad length; clamped to 48 -> ids 10, 11 bad
                  dtype=np.int32)
    lens = np.array([20, 40, 60], dtype=np.int32)
    assert oracle_mod.validate_inputs(bt, lens, 10) == (1, 3, 2)
    assert oracle_mod.validate_inputs(bt, np.array([0, 0, 0], np.int32), 10) == (0, 0, 0)
    # seq 0: bad length, clamped to 0 tokens; seqs 1, 2 reference ids -1 and 10
    assert oracle_mod.validate_inputs(bt, np.array([-5, 1, 1], np.int32), 10) == (1, 2, 3)


def test_validate_counts_injected_faults(oracle_mod):
    rng = np.random.default_rng(3)
    for trial in range(20):
        B, mb, nb = 6, 8, 50
        bt = rng.integers(0, nb, size=(B, mb), dtype=np.int32)
        lens = rng.integers(0, mb * 16 + 1, size=B).astype(np.int32)
        assert oracle_mod.validate_inputs(bt, lens, nb) == (0, 0, 0)
        # inject faults only at referenced positions, counted independently
        nbad = 0
        bad_seqs = set()
        for b in range(B):
            n = (int(lens[b]) + 15) // 16
            for j in range(n):
                if rng.random() < 0.2:
                    bt[b, j] = rng.choice([-1, nb, nb + 7, -1000])
                    nbad += 1
                    bad_seqs.add(b)
            for j in range(n, mb):  # unreferenced slots may hold anything
                bt[b, j] = -7
        assert oracle_mod.validate_inputs(bt, lens, nb) == (0, nbad, len(bad_seqs))


def test_e4m3_encode_matches_torch_cast(oracle_mod):
    g = torch.Generator().manual_seed(11)
    x = torch.cat([torch.randn(20000, generator=g) * s for s in (1e-3, 0.1, 1.0, 30.0, 150.0)]).clamp(-448, 448)
    ref = x.to(torch.float8_e4m3fn).view(torch.uint8).numpy()
    got = np.array([oracle_mod.e4m3_encode(float(v)) for v in x.numpy()], dtype=np.uint8)
    assert (ref == got).all()


def test_e4m3_encode_roundtrip_and_ties(oracle_mod):
    for c in range(256):
        if c & 0x7F == 0x7F:
            continue  # NaN codes
        v = oracle_mod.e4m3_to_f64(c)
        assert oracle_mod.e4m3_encode(v) == c or (v == 0 and oracle_mod.e4m3_encode(v) in (0, 0x80))
    # exact midpoints between consecutive magnitudes go to the even code (RNE)
    for c in range(0, 0x7E):
        lo, hi = oracle_mod.e4m3_to_f64(c), oracle_mod.e4m3_to_f64(c + 1)
        mid = np.float32((lo + hi) / 2)
        assert float(mid) == (lo + hi) / 2  # representable in fp32
        want = c if c % 2 == 0 else c + 1
        assert oracle_mod.e4m3_encode(float(mid)) == want
        assert oracle_mod.e4m3_encode(-float(mid)) == want | 0x80
        assert torch.tensor([float(mid)]).to(torch.float8_e4m3fn).view(torch.uint8).item() == want


def test_e4m3_encode_saturates_and_nan(oracle_mod):
    for v in (448.0, 449.0, 463.9, 464.0, 500.0, 1e6, float("inf")):
        assert oracle_mod.e4m3_encode(v) == 0x7E
        assert oracle_mod.e4m3_encode(-v) == 0xFE
    assert oracle_mod.e4m3_encode(float("nan")) == 0x7F
    assert oracle_mod.e4m3_encode(1e-9) == 0 and oracle_mod.e4m3_encode(-1e-9) == 0x80


def _append_case(dtype="fp16", lens=(17, 5, 32, 1), q_len=1, seed=4, Hkv=2, D=64):
    rng = np.random.default_rng(seed)
    B, mb, nb = len(lens), 4, 24
    perm = rng.permutation(nb)[: B * mb].reshape(B, mb).astype(np.int32)
    tdt = torch.float16 if dtype == "fp16" else torch.bfloat16
    g = torch.Generator().manual_seed(seed)
    k = (torch.rand(nb, Hkv, 16, D, generator=g) * 2 - 1).to(tdt)
    v = (torch.rand(nb, Hkv, 16, D, generator=g) * 2 - 1).to(tdt)
    kn = (torch.rand(B, q_len, Hkv, D, generator=g) * 2 - 1).to(tdt)
    vn = (torch.rand(B, q_len, Hkv, D, generator=g) * 2 - 1).to(tdt)
    return k, v, kn, vn, perm, np.array(lens, dtype=np.int32)


@pytest.mark.parametrize("q_len,lens", [(1, (17, 5, 32, 1)), (3, (18, 3, 2, 40)), (4, (16, 17, 64, 0))])
def test_kv_append_positions_by_hand(oracle_mod, q_len, lens):
    k, v, kn, vn, bt, L = _append_case(lens=lens, q_len=q_len)
    kc, vc = oracle_mod.kv_append(kn, vn, k, v, bt, L)
    kb, vb = k.view(torch.int16).numpy().view(np.uint16), v.view(torch.int16).numpy().view(np.uint16)
    knb, vnb = kn.view(torch.int16).numpy().view(np.uint16), vn.view(torch.int16).numpy().view(np.uint16)
    ek, ev = kb.copy(), vb.copy()
    for b in range(len(lens)):
        for i in range(q_len):
            t = lens[b] - q_len + i
            if t < 0:
                continue
            ek[bt[b, t // 16], :, t % 16, :] = knb[b, i]
            ev[bt[b, t // 16], :, t % 16, :] = vnb[b, i]
    assert (kc == ek).all() and (vc == ev).all()
    # untouched elsewhere: the number of changed slots is the number of written ones
    n_written = sum(max(0, min(q_len, l)) for l in lens)
    changed = (kc != kb).any(axis=(1, 3)).sum()
    assert changed <= n_written * 1 and n_written >= 1


@pytest.mark.parametrize("dtype", ["fp16", "bf16"])
def test_kv_append_e4m3_matches_torch_cast(oracle_mod, dtype):
    k, v, kn, vn, bt, L = _append_case(dtype=dtype, lens=(19, 33, 2, 64), q_len=2)
    k8 = torch.randint(0, 0x7E, k.shape, dtype=torch.uint8)
    v8 = torch.randint(0, 0x7E, v.shape, dtype=torch.uint8)
    ks, vs = 1 / 224, 0.0123
    kc, vc = oracle_mod.kv_append_e4m3(kn, vn, dtype, ks, vs, k8, v8, bt, L)
    qk = (kn.float() / torch.tensor(ks, dtype=torch.float32)).to(torch.float8_e4m3fn).view(torch.uint8).numpy()
    qv = (vn.float() / torch.tensor(vs, dtype=torch.float32)).to(torch.float8_e4m3fn).view(torch.uint8).numpy()
    ek, ev = k8.numpy().copy(), v8.numpy().copy()
    for b in range(4):
        for i in range(2):
            t = L[b] - 2 + i
            ek[bt[b, t // 16], :, t % 16, :] = qk[b, i]
            ev[bt[b, t // 16], :, t % 16, :] = qv[b, i]
    assert (kc == ek).all() and (vc == ev).all()


def test_attention_after_append_is_attention_over_concatenation(oracle_mod):
    """Decode step semantics: appending token L-1 then attending over L tokens
    equals softmax attention over [old K/V rows ; new row] (numpy)."""
    k, v, kn, vn, bt, L = _append_case(lens=(17, 5, 32, 1), q_len=1, D=64)
    kc, vc = oracle_mod.kv_append(kn, vn, k, v, bt, L)
    g = torch.Generator().manual_seed(9)
    q = (torch.rand(4, 4, 64, generator=g) * 2 - 1).half()
    kct = torch.from_numpy(kc.view(np.int16)).view(torch.float16)
    vct = torch.from_numpy(vc.view(np.int16)).view(torch.float16)
    out = oracle_mod.paged_attention(q, kct, vct, bt, L, 0.125, "fp16")
    for b in range(4):
        for h in range(4):
            kvh = h // 2
            rows = [k[bt[b, t // 16], kvh, t % 16].double().numpy() for t in range(L[b] - 1)]
            vrows = [v[bt[b, t // 16], kvh, t % 16].double().numpy() for t in range(L[b] - 1)]
            K = np.stack(rows + [kn[b, 0, kvh].double().numpy()])
            V = np.stack(vrows + [vn[b, 0, kvh].double().numpy()])
            s = 0.125 * (K @ q[b, h].double().numpy())
            w = np.exp(s - s.max())
            w /= w.sum()
            assert np.abs(out[b, h] - w @ V).max() < 1e-12


# ---------------------------------------------------------------------------
# Property-based pins (hypothesis): random shapes, lengths, placements, scales
# ---------------------------------------------------------------------------
from hypothesis import given, settings, strategies as st  # noqa: E402


@settings(max_examples=30, deadline=None)
@given(B=st.integers(1, 3), Hkv=st.integers(1, 2), g=st.sampled_from([1, 2, 4]), D=st.sampled_from([16, 64]),
       lens=st.lists(st.integers(0, 70), min_size=3, max_size=3), dtype=st.sampled_from(["fp16", "bf16"]),
       seed=st.integers(0, 10_000), scale=st.sampled_from([None, 1.0, 0.3]))
def test_property_oracle_equals_contiguous_softmax(oracle_mod, B, Hkv, g, D, lens, dtype, seed, scale):
    cfg = synth.Config("prop", B, Hkv * g, Hkv, D, tuple(lens[:B]), dtype, poison_blocks=2)
    inp = synth.make_inputs(cfg, seed=seed)
    if scale is not None:
        inp["scale"] = scale
    out = run_oracle(oracle_mod, inp)
    for b in range(B):
        for h in range(Hkv * g):
            np.testing.assert_allclose(out[b, h], contiguous_reference(inp, b, h), rtol=0, atol=1e-12)


@settings(max_examples=20, deadline=None)
@given(lens=st.lists(st.integers(0, 60), min_size=2, max_size=2), q_len=st.integers(1, 4),
       seed=st.integers(0, 10_000))
def test_property_append_then_attend(oracle_mod, lens, q_len, seed):
    """Append q_len rows then multi-token attend == causal attention over the
    old rows with the new rows spliced in at positions L - q_len + i."""
    cfg = synth.Config("prop_app", 2, 4, 2, 16, tuple(max(l, 1) for l in lens), "fp16", poison_blocks=1)
    inp = synth.with_query_tokens(synth.make_inputs(cfg, seed=seed), q_len)
    kn, vn = synth.new_kv_rows(inp, q_len, seed=seed)
    kc, vc = oracle_mod.kv_append(kn, vn, inp["k_cache"], inp["v_cache"], inp["block_tables"], inp["context_lens"])
    kt = torch.from_numpy(kc.view(np.int16)).view(torch.float16)
    vt = torch.from_numpy(vc.view(np.int16)).view(torch.float16)
    out = oracle_mod.paged_attention_mq(inp["q"], kt, vt, inp["block_tables"], inp["context_lens"], inp["scale"],
                                        "fp16")
    bt = inp["block_tables"].numpy()
    for b in range(2):
        L = int(inp["context_lens"][b])
        for i in range(q_len):
            Li = L - q_len + i + 1
            for h in range(4):
                kvh = h // 2
                if Li <= 0:
                    assert (out[b, i, h] == 0).all()
                    continue
                rows_k, rows_v = [], []
                for t in range(Li):
                    j = t - (L - q_len)  # index among the new rows, if this is one
                    if 0 <= j < q_len:
                        rows_k.append(kn[b, j, kvh].double().numpy())
                        rows_v.append(vn[b, j, kvh].double().numpy())
                    else:
                        rows_k.append(inp["k_cache"][bt[b, t // 16], kvh, t % 16].double().numpy())
                        rows_v.append(inp["v_cache"][bt[b, t // 16], kvh, t % 16].double().numpy())
                K, V = np.stack(rows_k), np.stack(rows_v)
                s = inp["scale"] * (K @ inp["q"][b, i, h].double().numpy())
                w = np.exp(s - s.max())
                np.testing.assert_allclose(out[b, i, h], (w / w.sum()) @ V, rtol=0, atol=1e-12)


# ---- SPEC's worked examples (tests/golden/spec_examples.txt), checked through
# the oracle's own computations, not through a re-typed formula ----

def _spec_examples(kind):
    path = os.path.join(os.path.dirname(__file__), "golden", "spec_examples.txt")
    out = []
    for line in open(path):
        line = line.split("#")[0].strip()
        if line.startswith(kind + " "):
            lhs, rhs = line[len(kind):].split("->")
            out.append((tuple(int(x) for x in lhs.split()), int(rhs)))
    assert out, kind
    return out


def test_spec_blocks_per_sequence(oracle_mod):
    """the number of blocks the oracle's plan visits for a
    sequence of L tokens in 16-token blocks (one partition covering it)."""
    for (L, bs), want in _spec_examples("blocks_per_sequence"):
        bt = np.arange(256, dtype=np.int32)[None, :]
        recs = oracle_mod.plan_splitk(bt, np.array([L], dtype=np.int32), num_kv_heads=1, block_size=bs,
                                      partition_tokens=4096, p_max=1, prefetch_distance=0)
        assert recs[0, 0, 0, 2] == want, (L, bs)
        assert list(recs[0, 0, 0, 4:4 + want]) == list(range(want))


def test_spec_kv_head_for_q_head(oracle_mod):
    """q head h reads kv head floor(h / (Hq / Hkv)).  Only kv head k
    carries V = 1 (all others 0), so the oracle's output row of q head h is 1
    (to rounding) iff h reads kv head k, else exactly 0 -- and every kv head serves exactly Hq/Hkv
    q heads (the exhaustive check S:159 asks for)."""
    for (qh, hq, hkv), kvh in _spec_examples("kv_head_for_q_head"):
        cfg = synth.Config("spec_gqa", 1, hq, hkv, 64, (20,), "fp16", poison_blocks=0)
        inp = synth.make_inputs(cfg, seed=3, poison=False)
        readers = {}
        for k in range(hkv):
            v = torch.zeros_like(inp["v_cache"])
            v[:, k] = 1.0
            out = oracle_mod.paged_attention(inp["q"], inp["k_cache"], v, inp["block_tables"],
                                             inp["context_lens"], inp["scale"], "fp16")
            ones = [h for h in range(hq) if np.all(np.abs(out[0, h] - 1.0) <= 1e-12)]  # sum w_t / Z = 1
            zeros = [h for h in range(hq) if np.all(out[0, h] == 0.0)]
            assert sorted(ones + zeros) == list(range(hq))
            readers[k] = ones
        assert qh in readers[kvh]
        assert all(len(r) == hq // hkv for r in readers.values())
