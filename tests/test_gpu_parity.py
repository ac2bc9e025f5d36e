"""GPU parity: the CUDA path through the C ABI vs the fp64 oracle (-m gpu).

Tolerance (BASELINE.json north_star): max abs error <= 2e-3 for fp16/bf16
inputs with fp32 accumulation; bookkeeping (visited blocks, partition
ranges, prefetch targets and counts) bit-exact against oracle plans;
prefetch on/off, placement and run-to-run bitwise invariant.
"""
import math

import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu

TOL = 2e-3


@pytest.fixture(scope="module")
def pda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2504_06319_b200 as m
    m.lib()  # must load; no fallback
    return m


def oracle_out(oracle_mod, inp, rows=None):
    return oracle_mod.paged_attention(inp["q"].cpu(), inp["k_cache"].cpu(), inp["v_cache"].cpu(),
                                      inp["block_tables"].cpu(), inp["context_lens"].cpu(), inp["scale"],
                                      inp["cfg"].dtype, rows=rows)


def to_dev(inp):
    d = dict(inp)
    for k in ("q", "k_cache", "v_cache", "block_tables", "context_lens"):
        d[k] = inp[k].cuda()
    return d


def gpu(pda, inp, **kw):
    # the kernel-level tests pin prefetch (default off); the library default
    # (prefetch AUTO, include/pda.h) has its own test below
    kw.setdefault("prefetch", "off")
    return pda.paged_decode_attention(inp["q"], inp["k_cache"], inp["v_cache"], inp["block_tables"],
                                      inp["context_lens"], inp["scale"], **kw)


def max_err(gpu_out, ref):
    g = gpu_out.double().cpu().numpy()
    assert np.isfinite(g).all(), "non-finite output"
    return float(np.abs(g - ref).max())


SHAPES = [
    synth.C1_TINY,
    synth.Config("mha128_ragged", 4, 4, 4, 128, (1, 15, 17, 300), "fp16", poison_blocks=5),
    synth.Config("gqa4_bf16", 3, 16, 4, 128, (100, 1000, 513), "bf16", poison_blocks=3),
    synth.Config("gqa8_bf16", 2, 16, 2, 128, (777, 64), "bf16", poison_blocks=2),
    synth.Config("gqa16_fp16", 2, 32, 2, 128, (95, 250), "fp16", poison_blocks=2),
    synth.Config("gqa7_d64", 2, 14, 2, 64, (123, 40), "bf16", poison_blocks=2),
    synth.Config("zero_len", 3, 4, 2, 64, (0, 5, 0), "fp16", poison_blocks=1),
]
KERNELS = [dict(kernel="splitk"), dict(kernel="splitk", partition_tokens=16),
           dict(kernel="splitk", partition_tokens=64), dict(kernel="splitk", smem_stages=4),
           dict(kernel="splitk", smem_stages=12, partition_tokens=256), dict(kernel="paper"),
           dict(kernel="splitk", issue_mode="self"), dict(kernel="splitk", issue_mode="self", smem_stages=4,
                                                          partition_tokens=48),
           dict(kernel="stream"), dict(kernel="stream", smem_stages=8, stream_warps=1),
           dict(kernel="stream", smem_stages=4, stream_warps=2),
           dict(kernel="stream", smem_stages=4, stream_warps=4),
           dict(kernel="balanced"), dict(kernel="balanced", smem_stages=4),
           dict(kernel="balanced", smem_stages=12), dict(kernel="balanced", num_sms=3)]


@pytest.mark.parametrize("cfg", SHAPES, ids=lambda c: c.name)
@pytest.mark.parametrize("kw", KERNELS, ids=lambda k: "-".join(f"{a}{b}" for a, b in k.items()))
def test_parity_vs_oracle(pda, oracle_mod, cfg, kw):
    inp = synth.make_inputs(cfg, seed=17)
    ref = oracle_out(oracle_mod, inp)
    dev = to_dev(inp)
    out = gpu(pda, dev, **kw)
    torch.cuda.synchronize()
    assert max_err(out, ref) <= TOL
    out32 = gpu(pda, dev, out_dtype=torch.float32, **kw)
    assert max_err(out32, ref) <= TOL


@pytest.mark.parametrize("cfg", SHAPES[:4], ids=lambda c: c.name)
@pytest.mark.parametrize("kernel", ["splitk", "paper", "stream", "balanced"])
def test_prefetch_is_bitwise_invisible(pda, cfg, kernel):
    """Prefetch changes where data is found, not what is computed."""
    dev = to_dev(synth.make_inputs(cfg, seed=3))
    base = gpu(pda, dev, kernel=kernel, prefetch="off")
    for mode in ("bulk", "line"):
        for d in (1, 2, 4, 7, 64 if kernel == "paper" else 32):
            o = gpu(pda, dev, kernel=kernel, prefetch=mode, prefetch_distance=d)
            assert torch.equal(o, base), (mode, d)


@pytest.mark.parametrize("kernel", ["splitk", "paper", "stream", "balanced"])
def test_eviction_hints_are_bitwise_invisible(pda, kernel):
    """Eviction priority changes cache residency only."""
    dev = to_dev(synth.make_inputs(SHAPES[2], seed=13))
    base = gpu(pda, dev, kernel=kernel, prefetch="off")
    for ev in (1, 2, 3):
        for mode in ("bulk", "line"):
            o = gpu(pda, dev, kernel=kernel, prefetch=mode, prefetch_distance=4, eviction=ev)
            assert torch.equal(o, base), (ev, mode)


@pytest.mark.parametrize("kernel", ["splitk", "paper", "stream", "balanced"])
def test_placement_invariance_bitwise(pda, kernel):
    inp = synth.make_inputs(SHAPES[2], seed=5)
    a = gpu(pda, to_dev(inp), kernel=kernel)
    b = gpu(pda, to_dev(synth.permute_placement(inp, seed=99)), kernel=kernel)
    assert torch.equal(a, b)


@pytest.mark.parametrize("kernel", ["splitk", "paper", "stream", "balanced"])
def test_run_to_run_bitwise(pda, kernel):  # noqa: default options
    dev = to_dev(synth.make_inputs(SHAPES[3], seed=8))
    a = gpu(pda, dev, kernel=kernel, partition_tokens=0 if kernel == "paper" else 128)
    for _ in range(3):
        b = gpu(pda, dev, kernel=kernel, partition_tokens=0 if kernel == "paper" else 128)
        assert torch.equal(a, b)


@pytest.mark.parametrize("dtype", ["fp16", "bf16"])
@pytest.mark.parametrize("kernel", ["splitk", "paper", "stream", "balanced"])
def test_context_len_one_returns_v_row_exactly(pda, dtype, kernel):
    cfg = synth.Config("l1", 3, 8, 2, 128, (1, 1, 1), dtype, poison_blocks=4)
    inp = synth.make_inputs(cfg, seed=2)
    dev = to_dev(inp)
    out = gpu(pda, dev, kernel=kernel)
    for b in range(3):
        blk = int(inp["block_tables"][b, 0])
        for h in range(8):
            assert torch.equal(out[b, h].cpu(), inp["v_cache"][blk, h // 4, 0])


@pytest.mark.parametrize("kernel", ["splitk", "paper", "stream", "balanced"])
def test_needle_every_position(pda, kernel):
    cfg = synth.Config("needle", 1, 2, 1, 64, (37,), "fp16", poison_blocks=2)
    base = synth.make_inputs(cfg, seed=9)
    bt = base["block_tables"][0]
    for t_star in range(37):
        inp = {k: (v.clone() if torch.is_tensor(v) else v) for k, v in base.items()}
        inp["q"].zero_()
        inp["q"][0, :, 0] = 1.0
        for t in range(37):
            inp["k_cache"][int(bt[t // 16]), 0, t % 16, 0] = 40.0 if t == t_star else 0.0
        inp["scale"] = 1.0
        out = gpu(pda, to_dev(inp), kernel=kernel, out_dtype=torch.float32, partition_tokens=0
                  if kernel != "splitk" else 16)
        v = inp["v_cache"][int(bt[t_star // 16]), 0, t_star % 16].float()
        assert torch.allclose(out[0, 0].cpu(), v, atol=1e-5, rtol=0), t_star


def test_gqa_identical_queries_identical_outputs(pda):
    cfg = synth.Config("gqa", 2, 8, 2, 128, (200, 33), "bf16")
    inp = synth.make_inputs(cfg, seed=4)
    inp["q"][:, 1:4] = inp["q"][:, 0:1]
    out = gpu(pda, to_dev(inp))
    for h in (1, 2, 3):
        assert torch.equal(out[:, h], out[:, 0])


def test_split_sizes_agree(pda, oracle_mod):
    cfg = synth.Config("splits", 2, 8, 2, 128, (1000, 517), "fp16", poison_blocks=1)
    inp = synth.make_inputs(cfg, seed=12)
    ref = oracle_out(oracle_mod, inp)
    dev = to_dev(inp)
    outs = [gpu(pda, dev, partition_tokens=p, out_dtype=torch.float32) for p in (16, 64, 256, 1024, 0)]
    for o in outs:
        assert max_err(o, ref) <= 5e-4  # fp32 out: only P / accumulation rounding remains


@pytest.mark.parametrize("issue", ["producer", "self"])
def test_trace_splitk_matches_oracle_plan(pda, oracle_mod, issue):
    cfg = synth.Config("trace", 3, 8, 2, 64, (37, 256, 0), "fp16", poison_blocks=3)
    dev = to_dev(synth.make_inputs(cfg, seed=1))
    for P in (16, 64, 128, 0):
        for mode, d in (("off", 0), ("bulk", 1), ("bulk", 3), ("line", 4), ("bulk", 32 if issue == "self" else 40)):
            _, tr, info = gpu(pda, dev, kernel="splitk", partition_tokens=P, prefetch=mode,
                              prefetch_distance=d or None, trace=True, issue_mode=issue)
            ref = oracle_mod.plan_splitk(dev["block_tables"], dev["context_lens"], cfg.num_kv_heads, 16,
                                         info["partition_tokens"], info["p_max"], d)
            got = tr.cpu().numpy().reshape(ref.shape)
            assert np.array_equal(got, ref), (P, mode, d)


def test_timeline_export_is_consistent(pda, oracle_mod):
    """paged_decode_attention_timeline: same output and trace as the trace
    call, one {start, end, SM} stamp per unit, end >= start, SM ids on chip."""
    cfg = synth.Config("timeline", 3, 8, 2, 64, (37, 256, 0), "fp16", poison_blocks=3)
    dev = to_dev(synth.make_inputs(cfg, seed=1))
    for P in (64, 0):
        out, tr, info = gpu(pda, dev, kernel="splitk", partition_tokens=P, trace=True)
        out2, tr2, info2, st = gpu(pda, dev, kernel="splitk", partition_tokens=P, timeline=True)
        assert torch.equal(out, out2) and torch.equal(tr, tr2)
        st = st.cpu()
        assert st.shape == (info["trace_records"], 3)
        assert (st[:, 0] > 0).all() and (st[:, 1] >= st[:, 0]).all()
        nsm = torch.cuda.get_device_properties(0).multi_processor_count
        assert ((st[:, 2] >= 0) & (st[:, 2] < nsm)).all()
    with pytest.raises(RuntimeError):
        gpu(pda, dev, kernel="paper", timeline=True)


def test_trace_paper_matches_alg1(pda, oracle_mod):
    cfg = synth.Config("trace_p", 3, 4, 2, 128, (16, 128, 300), "fp16", poison_blocks=3)
    dev = to_dev(synth.make_inputs(cfg, seed=2))
    for mode, d in (("off", 0), ("bulk", 4), ("line", 4), ("bulk", 1), ("bulk", 9)):
        _, tr, info = gpu(pda, dev, kernel="paper", prefetch=mode, prefetch_distance=d or None,
                          trace=True)
        ref = oracle_mod.plan_paper(dev["block_tables"], dev["context_lens"], cfg.num_q_heads, 16, 4, d)
        got = tr.cpu().numpy().reshape(ref.shape)
        assert np.array_equal(got, ref), (mode, d)
        if d == 4:  # 1 block/warp -> 0 prefetches; 2 blocks/warp -> 1 per warp
            assert got[0, :, :, 3].sum() == 0
            assert (got[1, :, :, 3] == 1).all()


def test_trace_balanced_matches_oracle_plan(pda, oracle_mod):
    cfg = synth.Config("trace_b", 5, 8, 2, 128, (37, 700, 0, 260, 16), "fp16", poison_blocks=3)
    dev = to_dev(synth.make_inputs(cfg, seed=4))
    for st, sms in ((8, 0), (4, 2), (12, 1), (8, 5)):
        for mode, d in (("off", 0), ("bulk", 1), ("line", 4), ("bulk", 32)):
            _, tr, info = gpu(pda, dev, kernel="balanced", smem_stages=st, num_sms=sms, prefetch=mode,
                              prefetch_distance=d or None, trace=True)
            ref = oracle_mod.plan_stream(dev["block_tables"], dev["context_lens"], cfg.num_kv_heads, 16,
                                         info["grid_x"], d)
            got = tr.cpu().numpy().reshape(ref.shape)
            assert np.array_equal(got, ref), (st, sms, mode, d)


@pytest.mark.parametrize("sms", [1, 2, 5])
def test_balanced_split_rows_tickets_reset(pda, oracle_mod, sms):
    cfg = synth.Config("bsplit", 6, 16, 4, 128, (333, 17, 1, 901, 64, 0), "bf16", poison_blocks=2)
    inp = synth.make_inputs(cfg, seed=8)
    ref = oracle_out(oracle_mod, inp)
    dev = to_dev(inp)
    ws = torch.zeros(64 << 20, dtype=torch.uint8, device="cuda")
    outs = []
    for rep in range(3):
        out = gpu(pda, dev, kernel="balanced", workspace=ws, out_dtype=torch.float32, num_sms=sms)
        assert max_err(out, ref) <= 5e-4
        outs.append(out.clone())
    assert all(torch.equal(o, outs[0]) for o in outs)


def test_trace_stream_matches_oracle_plan(pda, oracle_mod):
    cfg = synth.Config("trace_s", 4, 8, 2, 128, (37, 700, 0, 260), "bf16", poison_blocks=3)
    dev = to_dev(synth.make_inputs(cfg, seed=4))
    for st, w in ((6, 2), (8, 1), (4, 4)):
        for mode, d in (("off", 0), ("bulk", 1), ("line", 4), ("bulk", 32)):
            _, tr, info = gpu(pda, dev, kernel="stream", smem_stages=st, stream_warps=w, prefetch=mode,
                              prefetch_distance=d or None, trace=True)
            ns = info["grid_x"] * info["threads"] // 32
            ref = oracle_mod.plan_stream(dev["block_tables"], dev["context_lens"], cfg.num_kv_heads, 16,
                                         ns, d)
            got = tr.cpu().numpy().reshape(ref.shape)
            assert np.array_equal(got, ref), (st, w, mode, d)


@pytest.mark.parametrize("ns_cap", [1, 3, 17])
def test_stream_few_streams_split_rows(pda, oracle_mod, ns_cap):
    """Force many rows to be split across streams (num_sms small => few streams)
    so the in-kernel ticket/merge path runs for most rows."""
    cfg = synth.Config("split_rows", 5, 16, 4, 128, (333, 17, 1, 901, 64), "bf16", poison_blocks=2)
    inp = synth.make_inputs(cfg, seed=6)
    ref = oracle_out(oracle_mod, inp)
    dev = to_dev(inp)
    ws = torch.zeros(64 << 20, dtype=torch.uint8, device="cuda")
    for rep in range(3):  # tickets must self-reset between calls
        out = pda.paged_decode_attention(dev["q"], dev["k_cache"], dev["v_cache"], dev["block_tables"],
                                         dev["context_lens"], dev["scale"], kernel="stream",
                                         workspace=ws, out_dtype=torch.float32, num_sms=ns_cap)
        assert max_err(out, ref) <= 5e-4


def test_host_e2e_step_matches_device_path(pda):
    cfg = synth.Config("e2e", 4, 8, 2, 128, (300, 64, 1, 999), "bf16")
    inp = synth.make_inputs(cfg, seed=21)
    dev = to_dev(inp)
    ref = gpu(pda, dev)
    step = pda.HostDecodeStep(dev["k_cache"], dev["v_cache"], 4, 8, cfg.max_blocks_per_seq, torch.bfloat16)
    qh = inp["q"].pin_memory()
    bth = inp["block_tables"].pin_memory()
    lh = inp["context_lens"].pin_memory()
    out = step(qh, bth, lh, inp["scale"])
    torch.cuda.synchronize()
    assert torch.equal(out, ref.cpu())


def test_host_e2e_pipelined_slots(pda):
    """Two staging slots on two streams: every step's host output equals the
    device path; steps with different inputs do not mix."""
    cfg = synth.Config("e2e2", 4, 8, 2, 128, (300, 64, 1, 999), "bf16")
    inps = [synth.make_inputs(cfg, seed=s) for s in (31, 32, 33)]
    dev = to_dev(inps[0])
    step = pda.HostDecodeStep(dev["k_cache"], dev["v_cache"], 4, 8, cfg.max_blocks_per_seq, torch.bfloat16,
                              slots=2)
    refs, outs = [], []
    for i, inp in enumerate(inps):
        d = dict(dev, q=inp["q"].cuda())
        refs.append(gpu(pda, d).cpu())
        out = step(inp["q"].pin_memory(), inp["block_tables"].pin_memory() if i == 0 else
                   inps[0]["block_tables"].pin_memory(), inps[0]["context_lens"].pin_memory(), inp["scale"])
        step.join()
        torch.cuda.synchronize()
        outs.append(out.clone())
    for r, o in zip(refs, outs):
        assert torch.equal(o, r)
    assert not torch.equal(outs[0], outs[1])


def test_nan_poison_never_leaks(pda):
    cfg = synth.Config("poison", 4, 8, 8, 128, (17, 31, 33, 1), "fp16", poison_blocks=20)
    dev = to_dev(synth.make_inputs(cfg, seed=3))
    for kw in KERNELS:
        assert torch.isfinite(gpu(pda, dev, **kw)).all()


def test_rejects_cpu_tensors(pda):
    inp = synth.make_inputs(synth.C1_TINY, seed=0)
    with pytest.raises(ValueError):
        gpu(pda, inp)


# ---- FP8 (e4m3) KV cache ---------------------------------

def kv8(inp, ks=1 / 224, vs=1 / 256):
    return synth.quantize_kv_e4m3(inp, k_scale=ks, v_scale=vs)


def oracle_kv8(oracle_mod, inp, rows=None):
    return oracle_mod.paged_attention_kv8(inp["q"].cpu(), inp["k_cache"].cpu(), inp["v_cache"].cpu(),
                                          inp["k_scale"], inp["v_scale"], inp["block_tables"].cpu(),
                                          inp["context_lens"].cpu(), inp["scale"], inp["cfg"].dtype, rows=rows)


def gpu_kv8(pda, inp, **kw):
    return pda.paged_decode_attention(inp["q"], inp["k_cache"], inp["v_cache"], inp["block_tables"],
                                      inp["context_lens"], inp["scale"], k_scale=inp["k_scale"],
                                      v_scale=inp["v_scale"], **kw)


KV8_SHAPES = [
    synth.Config("kv8_mha", 4, 4, 4, 128, (1, 15, 17, 300), "fp16", poison_blocks=5),
    synth.Config("kv8_gqa4_bf16", 3, 16, 4, 128, (100, 1000, 513), "bf16", poison_blocks=3),
    synth.Config("kv8_gqa8", 2, 16, 2, 128, (777, 64), "fp16", poison_blocks=2),
    synth.Config("kv8_gqa16", 2, 32, 2, 128, (95, 250), "bf16", poison_blocks=2),
    synth.Config("kv8_zero", 3, 4, 2, 128, (0, 5, 0), "fp16", poison_blocks=1),
]


@pytest.mark.parametrize("cfg", KV8_SHAPES, ids=lambda c: c.name)
@pytest.mark.parametrize("kw", [dict(), dict(partition_tokens=64), dict(smem_stages=8),
                                dict(smem_stages=16, partition_tokens=256), dict(smem_stages=24),
                                dict(smem_stages=12), dict(smem_stages=12, partition_tokens=48),
                                dict(partition_tokens=16), dict(partition_tokens=48)],
                         ids=lambda k: "-".join(f"{a}{b}" for a, b in k.items()) or "default")
def test_kv8_parity_vs_oracle(pda, oracle_mod, cfg, kw):
    inp = kv8(synth.make_inputs(cfg, seed=17))
    ref = oracle_kv8(oracle_mod, inp)
    dev = to_dev(inp)
    assert max_err(gpu_kv8(pda, dev, **kw), ref) <= TOL
    assert max_err(gpu_kv8(pda, dev, out_dtype=torch.float32, **kw), ref) <= 5e-4


def test_kv8_prefetch_eviction_bitwise_invisible(pda):
    dev = to_dev(kv8(synth.make_inputs(KV8_SHAPES[1], seed=3)))
    base = gpu_kv8(pda, dev, prefetch="off", eviction="normal")
    for mode in ("bulk", "line"):
        for d in (1, 4, 32):
            for ev in ("normal", "both"):
                assert torch.equal(gpu_kv8(pda, dev, prefetch=mode, prefetch_distance=d, eviction=ev), base)


def test_kv8_context_one_is_scaled_v_row(pda):
    cfg = synth.Config("kv8_l1", 2, 8, 2, 128, (1, 1), "fp16", poison_blocks=2)
    inp = kv8(synth.make_inputs(cfg, seed=2), vs=1 / 256)
    out = gpu_kv8(pda, to_dev(inp), out_dtype=torch.float32)
    for b in range(2):
        blk = int(inp["block_tables"][b, 0])
        for h in range(8):
            v = inp["v_cache"][blk, h // 4, 0].view(torch.float8_e4m3fn).float() / 256
            assert torch.equal(out[b, h].cpu(), v)


def test_kv8_trace_matches_oracle_plan(pda, oracle_mod):
    cfg = synth.Config("kv8_trace", 3, 8, 2, 128, (37, 256, 0), "fp16", poison_blocks=3)
    dev = to_dev(kv8(synth.make_inputs(cfg, seed=1)))
    for P, st in ((16, 0), (64, 0), (0, 0), (48, 12), (0, 12)):
        _, tr, info = gpu_kv8(pda, dev, partition_tokens=P, prefetch="line", prefetch_distance=3, trace=True,
                              smem_stages=st)
        ref = oracle_mod.plan_splitk(dev["block_tables"], dev["context_lens"], 2, 16, info["partition_tokens"],
                                     info["p_max"], 3)
        assert np.array_equal(tr.cpu().numpy().reshape(ref.shape), ref)


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("kernel", ["splitk", "balanced"])
def test_tp_shards_match_unsharded(pda, oracle_mod, world, kernel):
    """KV-head tensor parallelism: each rank's shard, computed by the
    CUDA kernel on its own heads and concatenated in rank order, matches the
    unsharded oracle (<= 2e-3); for split-K it also equals the unsharded step
    bit for bit (partition size pinned so the plans match).  The balanced
    kernel cuts its block ranges by the step's total work, which changes with
    the head count, so its shards agree with the unsharded step only to
    rounding -- both are checked against the oracle instead."""
    cfg = synth.Config("tp", 3, 16, 4, 128, (300, 77, 1024), "bf16", poison_blocks=2)
    inp = synth.make_inputs(cfg, seed=31)
    dev = to_dev(inp)
    kw = dict(kernel=kernel, partition_tokens=256) if kernel == "splitk" else dict(kernel=kernel)
    full = gpu(pda, dev, **kw)
    parts = []
    for r in range(world):
        sh = to_dev(synth.shard_kv_heads(inp, r, world))
        parts.append(gpu(pda, sh, **kw))
    got = torch.cat(parts, dim=1)
    ref = oracle_out(oracle_mod, inp)
    assert max_err(got, ref) <= TOL and max_err(full, ref) <= TOL
    if kernel == "splitk":
        assert torch.equal(got, full)


# ---- multi-token (speculative) decode ---------------------

MQ_CASES = [
    (synth.Config("mq_mha", 3, 4, 4, 128, (37, 300, 5), "fp16", poison_blocks=3), 8),
    (synth.Config("mq_gqa4", 2, 16, 4, 128, (700, 33), "bf16", poison_blocks=2), 4),
    (synth.Config("mq_gqa2_d64", 3, 8, 4, 64, (2, 129, 64), "fp16", poison_blocks=2), 4),
    (synth.Config("mq_gqa8", 2, 16, 2, 128, (95, 250), "bf16", poison_blocks=2), 2),
]


@pytest.mark.parametrize("cfg,q_len", MQ_CASES, ids=lambda x: x.name if hasattr(x, "name") else str(x))
@pytest.mark.parametrize("kw", [dict(), dict(partition_tokens=16), dict(partition_tokens=64, smem_stages=4)],
                         ids=lambda k: "-".join(f"{a}{b}" for a, b in k.items()) or "default")
def test_multi_token_parity_vs_oracle(pda, oracle_mod, cfg, q_len, kw):
    inp = synth.with_query_tokens(synth.make_inputs(cfg, seed=21), q_len)
    ref = oracle_mod.paged_attention_mq(inp["q"], inp["k_cache"], inp["v_cache"], inp["block_tables"],
                                        inp["context_lens"], inp["scale"], cfg.dtype)
    dev = to_dev(inp)
    out = gpu(pda, dev, **kw)
    assert out.shape == inp["q"].shape
    assert max_err(out, ref) <= TOL
    assert max_err(gpu(pda, dev, out_dtype=torch.float32, **kw), ref) <= 5e-4


def test_multi_token_q_len_one_matches_single_query_bitwise(pda):
    dev = to_dev(synth.make_inputs(SHAPES[2], seed=4))
    a = gpu(pda, dev, partition_tokens=64)
    q4 = dict(dev, q=dev["q"][:, None].contiguous())
    b = gpu(pda, q4, partition_tokens=64)
    assert torch.equal(a, b[:, 0])


def test_multi_token_e4m3(pda, oracle_mod):
    cfg = synth.Config("mq_kv8", 2, 8, 2, 128, (200, 41), "fp16", poison_blocks=2)
    inp = kv8(synth.with_query_tokens(synth.make_inputs(cfg, seed=5), 3))
    deq = dict(inp)
    deq["k_cache"] = (inp["k_cache"].view(torch.float8_e4m3fn).float() * inp["k_scale"]).double()
    deq["v_cache"] = (inp["v_cache"].view(torch.float8_e4m3fn).float() * inp["v_scale"]).double()
    # reference: the mq oracle on the exactly dequantised cache, via per-token single-query kv8 calls
    ref = np.stack([oracle_mod.paged_attention_kv8(inp["q"][:, i], inp["k_cache"], inp["v_cache"], inp["k_scale"],
                                                   inp["v_scale"], inp["block_tables"],
                                                   inp["context_lens"] - 2 + i, inp["scale"], "fp16")
                    for i in range(3)], axis=1)
    out = gpu_kv8(pda, to_dev(inp), partition_tokens=32)
    assert max_err(out, ref) <= TOL


def test_multi_token_prefetch_bitwise_invisible(pda):
    dev = to_dev(synth.with_query_tokens(synth.make_inputs(MQ_CASES[1][0], seed=6), 4))
    base = gpu(pda, dev, prefetch="off")
    for mode in ("bulk", "line"):
        assert torch.equal(gpu(pda, dev, prefetch=mode, prefetch_distance=3), base)


# ---- fused TP output all-gather ----------------------------

@pytest.mark.parametrize("kw", [dict(), dict(partition_tokens=32), dict(partition_tokens=64, merge="cluster"),
                                dict(q_len=2)],
                         ids=["direct", "combine", "cluster", "multi_token"])
def test_fused_gather_tp_world_vs_oracle(pda, oracle_mod, kw):
    """Fused output all-gather (NEXT f2) for a simulated TP world of 3 ranks on
    one GPU: three local buffers stand in for the ranks' peer-mapped output
    buffers.  Rank r runs its KV-head shard and its kernel stores
    its heads into every buffer at head offset r * Hq/N.  After rank 0 only its
    slice is written (nothing else touched); after all three, every buffer
    holds the whole step and matches the unsharded fp64 oracle on every row
    (<= 2e-3), and each slice equals that rank's plain call bit for bit."""
    kw = dict(kw)
    q_len = kw.pop("q_len", 1)
    world, hq, hkv = 3, 24, 6
    cfg = synth.Config("fg", 3, hq, hkv, 128, (300, 17, 64), "bf16", poison_blocks=2)
    inp = synth.make_inputs(cfg, seed=9)
    if q_len > 1:
        inp = synth.with_query_tokens(inp, q_len)
        q4 = inp["q"]
        ref = oracle_mod.paged_attention_mq(q4, inp["k_cache"], inp["v_cache"], inp["block_tables"],
                                            inp["context_lens"], inp["scale"], cfg.dtype)
    else:
        ref = oracle_out(oracle_mod, inp)
    shape = tuple(inp["q"].shape)
    peers = [torch.full(shape, 7.0, dtype=torch.bfloat16, device="cuda") for _ in range(world)]
    hl = hq // world
    for r in range(world):
        sh = synth.shard_kv_heads(inp, r, world) if q_len == 1 else _shard_mq(inp, r, world)
        dev = to_dev(sh)
        plain = gpu(pda, dev, **kw)
        pda.paged_decode_attention_gather(dev["q"], dev["k_cache"], dev["v_cache"], dev["block_tables"],
                                          dev["context_lens"], dev["scale"], peers, r * hl, hq, **kw)
        torch.cuda.synchronize()
        for pb in peers:
            assert torch.equal(pb[..., r * hl:(r + 1) * hl, :], plain)
            if r == 0:
                assert (pb[..., hl:, :] == 7.0).all()
    for pb in peers:
        assert max_err(pb, ref) <= TOL


def _shard_mq(inp, rank, world):
    """shard_kv_heads for a multi-token q [B, q_len, Hq, D] (heads on dim 2)."""
    flat = dict(inp, q=inp["q"][:, 0])
    sh = synth.shard_kv_heads(flat, rank, world)
    qh = inp["q"].shape[2] // world
    sh["q"] = inp["q"][:, :, rank * qh:(rank + 1) * qh].contiguous()
    return sh


def test_fused_gather_rejects_bad_offsets(pda):
    dev = to_dev(synth.make_inputs(synth.C1_TINY, seed=0))
    buf = torch.zeros((2, 8, 64), dtype=torch.float16, device="cuda")
    with pytest.raises(pda.PdaError):
        pda.paged_decode_attention_gather(dev["q"], dev["k_cache"], dev["v_cache"], dev["block_tables"],
                                          dev["context_lens"], dev["scale"], [buf], 6, 8)
    with pytest.raises(pda.PdaError):
        pda.paged_decode_attention_gather(dev["q"], dev["k_cache"], dev["v_cache"], dev["block_tables"],
                                          dev["context_lens"], dev["scale"], [buf], 0, 8, kernel="paper")


# ---- KV append, fused and standalone (SURVEY 8f NEXT f3 alternative) ------------

APPEND_CFGS = [
    synth.Config("app_mha", 4, 4, 4, 128, (1, 15, 17, 300), "fp16", poison_blocks=3),
    synth.Config("app_gqa4_bf16", 3, 16, 4, 128, (100, 1000, 513), "bf16", poison_blocks=2),
    synth.Config("app_d64", 3, 8, 2, 64, (64, 2, 0), "fp16", poison_blocks=2),
]


def _bytes(t):
    return t.contiguous().view(torch.uint8).cpu().numpy().ravel()


def _oracle_append(oracle_mod, inp, kn, vn):
    if inp.get("kv_dtype") == "e4m3":
        kc, vc = oracle_mod.kv_append_e4m3(kn.cpu(), vn.cpu(), inp["cfg"].dtype, inp["k_scale"], inp["v_scale"],
                                           inp["k_cache"].cpu(), inp["v_cache"].cpu(), inp["block_tables"].cpu(),
                                           inp["context_lens"].cpu())
    else:
        kc, vc = oracle_mod.kv_append(kn.cpu(), vn.cpu(), inp["k_cache"].cpu(), inp["v_cache"].cpu(),
                                      inp["block_tables"].cpu(), inp["context_lens"].cpu())
    return kc.view(np.uint8).ravel(), vc.view(np.uint8).ravel()


def _as_cache(arr_u8, like):
    t = torch.from_numpy(arr_u8.copy())
    return t.view(like.dtype).view(like.shape) if like.dtype != torch.uint8 else t.view(like.shape)


@pytest.mark.parametrize("cfg", APPEND_CFGS, ids=lambda c: c.name)
@pytest.mark.parametrize("q_len", [1, 3])
@pytest.mark.parametrize("e4m3", [False, True])
def test_kv_append_standalone_bitwise_vs_oracle(pda, oracle_mod, cfg, q_len, e4m3):
    if e4m3 and cfg.head_dim != 128:
        pytest.skip("e4m3 caches are head_dim 128 only")
    inp = synth.make_inputs(cfg, seed=12)
    if e4m3:
        inp = kv8(inp)
    kn, vn = synth.new_kv_rows(inp, q_len, seed=3)
    ek, ev = _oracle_append(oracle_mod, inp, kn, vn)
    dev = to_dev(inp)
    kw = dict(k_scale=inp["k_scale"], v_scale=inp["v_scale"]) if e4m3 else {}
    pda.kv_append(kn.cuda(), vn.cuda(), dev["k_cache"], dev["v_cache"], dev["block_tables"], dev["context_lens"],
                  **kw)
    torch.cuda.synchronize()
    assert (_bytes(dev["k_cache"]) == ek).all() and (_bytes(dev["v_cache"]) == ev).all()


FUSED_KW = [dict(), dict(partition_tokens=16), dict(partition_tokens=64, issue_mode="producer"),
            dict(kernel="paper"), dict(kernel="balanced"), dict(kernel="stream")]


@pytest.mark.parametrize("cfg", APPEND_CFGS, ids=lambda c: c.name)
@pytest.mark.parametrize("kw", FUSED_KW, ids=lambda k: "-".join(f"{a}{b}" for a, b in k.items()) or "default")
def test_fused_append_attention_vs_oracle(pda, oracle_mod, cfg, kw):
    """One call = append + attention: the caches afterwards equal the oracle's
    append bitwise, the output matches the oracle attention over the updated
    cache, and equals the two separate calls bitwise."""
    inp = synth.make_inputs(cfg, seed=13)
    kn, vn = synth.new_kv_rows(inp, 1, seed=4)
    ek, ev = _oracle_append(oracle_mod, inp, kn, vn)
    upd = dict(inp, k_cache=_as_cache(ek, inp["k_cache"]), v_cache=_as_cache(ev, inp["v_cache"]))
    ref = oracle_out(oracle_mod, upd)
    dev = to_dev(inp)
    out = gpu(pda, dev, k_new=kn.cuda(), v_new=vn.cuda(), **kw)
    torch.cuda.synchronize()
    assert (_bytes(dev["k_cache"]) == ek).all() and (_bytes(dev["v_cache"]) == ev).all()
    assert max_err(out, ref) <= TOL
    dev2 = to_dev(inp)
    pda.kv_append(kn.cuda(), vn.cuda(), dev2["k_cache"], dev2["v_cache"], dev2["block_tables"],
                  dev2["context_lens"])
    assert torch.equal(gpu(pda, dev2, **kw), out)


@pytest.mark.parametrize("q_len,kw", [(3, dict()), (3, dict(partition_tokens=16)), (4, dict(partition_tokens=32))])
def test_fused_append_multi_token(pda, oracle_mod, q_len, kw):
    """q_len new tokens (they may straddle a block and a partition boundary)."""
    cfg = synth.Config("app_mq", 3, 8, 4, 128, (18, 33, 2), "bf16", poison_blocks=2)
    inp = synth.with_query_tokens(synth.make_inputs(cfg, seed=14), q_len)
    kn, vn = synth.new_kv_rows(inp, q_len, seed=5)
    ek, ev = _oracle_append(oracle_mod, inp, kn, vn)
    upd = dict(inp, k_cache=_as_cache(ek, inp["k_cache"]), v_cache=_as_cache(ev, inp["v_cache"]))
    ref = oracle_mod.paged_attention_mq(upd["q"], upd["k_cache"], upd["v_cache"], upd["block_tables"],
                                        upd["context_lens"], upd["scale"], cfg.dtype)
    dev = to_dev(inp)
    out = gpu(pda, dev, k_new=kn.cuda(), v_new=vn.cuda(), **kw)
    torch.cuda.synchronize()
    assert (_bytes(dev["k_cache"]) == ek).all() and (_bytes(dev["v_cache"]) == ev).all()
    assert max_err(out, ref) <= TOL


@pytest.mark.parametrize("kw", [dict(), dict(partition_tokens=16)], ids=["default", "p16"])
def test_fused_append_e4m3(pda, oracle_mod, kw):
    cfg = synth.Config("app_kv8", 3, 8, 2, 128, (200, 17, 1), "fp16", poison_blocks=2)
    inp = kv8(synth.make_inputs(cfg, seed=15))
    kn, vn = synth.new_kv_rows(inp, 1, seed=6)
    ek, ev = _oracle_append(oracle_mod, inp, kn, vn)
    upd = dict(inp, k_cache=_as_cache(ek, inp["k_cache"]), v_cache=_as_cache(ev, inp["v_cache"]))
    ref = oracle_kv8(oracle_mod, upd)
    dev = to_dev(inp)
    out = gpu_kv8(pda, dev, k_new=kn.cuda(), v_new=vn.cuda(), **kw)
    torch.cuda.synchronize()
    assert (_bytes(dev["k_cache"]) == ek).all() and (_bytes(dev["v_cache"]) == ev).all()
    assert max_err(out, ref) <= TOL


# ---- debug validation of device-resident tables / lengths ------------------------

@pytest.mark.parametrize("seed", [0, 1, 2])
def test_validate_inputs_matches_oracle(pda, oracle_mod, seed):
    rng = np.random.default_rng(seed)
    B, mb, nb = 300, 40, 5000
    bt = rng.integers(0, nb, size=(B, mb), dtype=np.int32)
    lens = rng.integers(0, mb * 16 + 1, size=B).astype(np.int32)
    # faults: ids out of range anywhere (only referenced ones count), bad lengths
    mask = rng.random((B, mb)) < 0.01
    bt[mask] = rng.choice(np.array([-1, nb, 2**31 - 1, -2**31], dtype=np.int64), size=mask.sum()).astype(np.int32)
    bad_len = rng.random(B) < 0.05
    lens[bad_len] = rng.choice(np.array([-1, mb * 16 + 1, 2**31 - 1, -2**31], dtype=np.int64),
                               size=bad_len.sum()).astype(np.int32)
    want = oracle_mod.validate_inputs(bt, lens, nb)
    assert want[1] > 0 and want[0] > 0
    got = pda.validate_inputs(torch.from_numpy(bt).cuda(), torch.from_numpy(lens).cuda(), nb)
    assert got == want
    good = synth.make_inputs(SHAPES[1], seed=1, device="cuda")
    assert pda.validate_inputs(good["block_tables"], good["context_lens"], good["k_cache"].shape[0]) == (0, 0, 0)


# ---- S8 merge inside a thread-block cluster (DSMEM) vs the combine kernel ---------

CLUSTER_CASES = [
    (SHAPES[1], dict(partition_tokens=64)),                      # mha, ragged, P_max 5
    (SHAPES[2], dict(partition_tokens=128)),                     # gqa4 bf16, P_max 8
    (SHAPES[3], dict(partition_tokens=64, merge="cluster")),     # gqa8, P_max 13 (non-portable)
    (SHAPES[4], dict(partition_tokens=32, issue_mode="producer")),  # gqa16 (2 head tiles), producer warp
    (synth.Config("zero_len_long", 3, 4, 2, 64, (0, 100, 0), "fp16", poison_blocks=1),
     dict(partition_tokens=16)),                                 # zero-length rows, P_max 7
]


@pytest.mark.parametrize("cfg,kw", CLUSTER_CASES, ids=lambda x: x.name if hasattr(x, "name") else
                         "-".join(f"{a}{b}" for a, b in x.items()))
def test_cluster_merge_bitwise_equals_combine(pda, oracle_mod, cfg, kw):
    inp = synth.make_inputs(cfg, seed=23)
    dev = to_dev(inp)
    kw = dict(kw)
    # the planner's auto mode merges in clusters only from one CTA per SM on:
    # these small cases force it
    mode = kw.pop("merge", "cluster")
    info = pda.plan(pda.make_shape(dev["q"], dev["k_cache"], dev["block_tables"]),
                    pda.make_options(merge=mode, prefetch="off", **kw))
    assert info["cluster"] == info["p_max"] > 1
    a = gpu(pda, dev, merge=mode, **kw)
    b = gpu(pda, dev, merge="combine", **kw)
    assert torch.equal(a, b)
    assert max_err(a, oracle_out(oracle_mod, inp)) <= TOL


def test_cluster_merge_multi_token_kv8_gather_trace(pda, oracle_mod):
    # multi-token
    dev = to_dev(synth.with_query_tokens(synth.make_inputs(MQ_CASES[1][0], seed=24), 4))
    assert torch.equal(gpu(pda, dev, partition_tokens=64, merge="cluster"),
                       gpu(pda, dev, partition_tokens=64, merge="combine"))
    # e4m3 cache
    d8 = to_dev(kv8(synth.make_inputs(KV8_SHAPES[1], seed=25)))
    assert torch.equal(gpu_kv8(pda, d8, partition_tokens=128, merge="cluster"),
                       gpu_kv8(pda, d8, partition_tokens=128, merge="combine"))
    # fused TP gather destinations
    cfg = synth.Config("cl_fg", 3, 8, 2, 128, (300, 17, 64), "bf16", poison_blocks=2)
    d = to_dev(synth.make_inputs(cfg, seed=26))
    ref = gpu(pda, d, partition_tokens=64, merge="combine")
    peers = [torch.full((3, 16, 128), 7.0, dtype=torch.bfloat16, device="cuda") for _ in range(2)]
    pda.paged_decode_attention_gather(d["q"], d["k_cache"], d["v_cache"], d["block_tables"], d["context_lens"],
                                      d["scale"], peers, 8, 16, partition_tokens=64, merge="cluster")
    torch.cuda.synchronize()
    for pb in peers:
        assert torch.equal(pb[:, 8:], ref) and (pb[:, :8] == 7.0).all()
        assert max_err(pb[:, 8:], oracle_out(oracle_mod, synth.make_inputs(cfg, seed=26))) <= TOL
    # the kernel's own bookkeeping is unchanged by the merge mode
    inp = synth.make_inputs(SHAPES[2], seed=27)
    dv = to_dev(inp)
    _, tr_a, _ = gpu(pda, dv, partition_tokens=128, merge="cluster", trace=True)
    _, tr_b, _ = gpu(pda, dv, partition_tokens=128, merge="combine", trace=True)
    assert torch.equal(tr_a, tr_b)


def test_prepared_decode_matches_wrapper(pda):
    for cfg, kw in ((SHAPES[2], dict(partition_tokens=64)), (SHAPES[0], dict(kernel="paper")),
                    (SHAPES[3], dict(kernel="balanced"))):
        dev = to_dev(synth.make_inputs(cfg, seed=29))
        step = pda.PreparedDecode(dev["q"], dev["k_cache"], dev["block_tables"], prefetch="off", **kw)
        a = step(dev["q"], dev["k_cache"], dev["v_cache"], dev["block_tables"], dev["context_lens"], dev["scale"])
        b = gpu(pda, dev, **kw)
        assert torch.equal(a, b)
        with pytest.raises(ValueError):
            step(dev["q"][:1], dev["k_cache"], dev["v_cache"], dev["block_tables"], dev["context_lens"], dev["scale"])


def test_graphed_decode_replays_with_updated_inputs(pda, oracle_mod):
    cfg = synth.Config("graphed", 3, 8, 2, 128, (300, 17, 64), "bf16", poison_blocks=2)
    a_in, b_in = synth.make_inputs(cfg, seed=30), synth.make_inputs(cfg, seed=31)
    dev = to_dev(a_in)
    prep = pda.PreparedDecode(dev["q"], dev["k_cache"], dev["block_tables"], partition_tokens=64, prefetch="off")
    g = pda.GraphedDecode(prep, dev["q"], dev["k_cache"], dev["v_cache"], dev["block_tables"], dev["context_lens"],
                          dev["scale"])
    out = g.replay().clone()
    assert torch.equal(out, gpu(pda, dev, partition_tokens=64))
    g.q.copy_(b_in["q"].cuda())                      # new queries, same cache
    g.context_lens.copy_(torch.tensor([299, 16, 1], dtype=torch.int32))
    out2 = g.replay().clone()
    ref_in = dict(a_in, q=b_in["q"], context_lens=torch.tensor([299, 16, 1], dtype=torch.int32))
    assert max_err(out2, oracle_out(oracle_mod, ref_in)) <= TOL


def test_c_example_runs(tmp_path):
    """examples/decode_step.c: one decode step from plain C through the C ABI,
    self-checked against the constant-V closed form (exit code 0)."""
    import subprocess
    from test_abi import _build_c_example
    exe = _build_c_example(tmp_path)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 of 512 outputs off the closed form" in r.stdout


@pytest.mark.parametrize("hq,hkv", [(32, 8), (28, 4)])
def test_kernel_gqa_mapping_spec_examples(pda, hq, hkv):
    """SPEC's kv_head_for_q_head examples on the kernel: with V = 1
    only in kv head k, exactly the q heads floor(h / (Hq/Hkv)) == k read 1,
    every other row is exactly 0 -- for each k, default plan and P = 16."""
    cfg = synth.Config("spec_gqa_gpu", 2, hq, hkv, 128, (20, 300), "bf16", poison_blocks=1)
    dev = to_dev(synth.make_inputs(cfg, seed=3))
    g = hq // hkv
    for k in range(hkv):
        v = torch.zeros_like(dev["v_cache"])
        v[:, k] = 1.0
        for kw in (dict(), dict(partition_tokens=16)):
            out = pda.paged_decode_attention(dev["q"], dev["k_cache"], v, dev["block_tables"],
                                             dev["context_lens"], dev["scale"], out_dtype=torch.float32, **kw)
            for h in range(hq):
                row = out[:, h].cpu()
                if h // g == k:
                    assert (row - 1.0).abs().max().item() <= 2e-3, (k, h)
                else:
                    assert torch.count_nonzero(row).item() == 0, (k, h)


def _fuzz_cases(n=96, seed=2025):
    import random
    rng = random.Random(seed)
    cases = []
    for i in range(n):
        kv8_case = i % 4 == 3
        D = 128 if kv8_case else rng.choice([64, 128])
        g = rng.choice([1, 2, 4, 7, 8, 16])
        hkv = rng.choice([1, 2, 4])
        q_len = 1 if kv8_case else rng.choice([1, 1, 2, 3, 4])
        q_len = max(1, min(q_len, 16 // g))
        B = rng.randint(1, 6)
        lens = tuple(rng.choice([0, 1, 15, 16, 17, rng.randint(2, 700)]) for _ in range(B))
        if max(lens) < q_len:
            lens = (q_len,) + lens[1:]
        lens = tuple(max(L, q_len) if L else 0 for L in lens)  # a row with tokens holds its q_len new ones
        stages = rng.choice([0, 8, 12, 16, 24] if kv8_case else [0, 4, 8, 12])
        P = rng.choice([0, 16, 48, 128, 512])
        merge = rng.choice(["auto", "combine", "cluster"])
        dt = rng.choice(["fp16", "bf16"])
        cases.append((i, kv8_case, D, g, hkv, q_len, lens, stages, P, merge, dt))
    return cases


@pytest.mark.parametrize("case", _fuzz_cases(), ids=lambda c: f"fuzz{c[0]}")
def test_fuzz_parity_vs_oracle(pda, oracle_mod, case):
    """Seeded random shapes / lengths / ring depths / partition sizes / merge
    modes (incl. the 4-CTA, two-tile and e4m3 occupancy variants) vs the
    oracle; every planner-valid combination must match within 2e-3."""
    i, kv8_case, D, g, hkv, q_len, lens, stages, P, merge, dt = case
    cfg = synth.Config(f"fuzz{i}", len(lens), g * hkv, hkv, D, lens, dt, poison_blocks=2)
    inp = synth.make_inputs(cfg, seed=100 + i)
    kw = dict(smem_stages=stages, partition_tokens=P)
    if kv8_case:
        inp = kv8(inp)
        ref = oracle_kv8(oracle_mod, inp)
    else:
        inp = synth.with_query_tokens(inp, q_len, seed=i) if q_len > 1 else inp
        q4 = inp["q"] if q_len > 1 else inp["q"][:, None]
        ref = oracle_mod.paged_attention_mq(q4, inp["k_cache"], inp["v_cache"], inp["block_tables"],
                                            inp["context_lens"], inp["scale"], dt)
        if q_len == 1:
            ref = ref[:, 0]
    dev = to_dev(inp)
    if kv8_case:
        dev.update(k_scale=inp["k_scale"], v_scale=inp["v_scale"])
    # the plan this shape gets; cluster merge only where P_max fits a cluster
    s = pda.make_shape(dev["q"], dev["k_cache"], dev["block_tables"])
    info = pda.plan(s, pda.make_options(smem_stages=stages, partition_tokens=P, kernel="splitk",
                                        k_scale=inp.get("k_scale", 0.0), v_scale=inp.get("v_scale", 0.0)))
    if merge == "cluster" and info["p_max"] > 8:
        merge = "auto"
    kw["merge"] = merge
    out = gpu_kv8(pda, dev, **kw) if kv8_case else gpu(pda, dev, **kw)
    assert out.shape == tuple(ref.shape)
    assert max_err(out, ref) <= TOL, kw


def test_prefetch_auto_policy_vs_oracle(pda, oracle_mod):
    """The library default (prefetch AUTO): short-context GQA steps in the
    measured band run the paper-structure kernel with Alg. 1's line prefetch
     and evict_last prefetches; other steps split-K.  Every
    row against the fp64 oracle, and a band step with a fused output gather
    (which keeps split-K) too."""
    for cfg in SHAPES:
        inp = synth.make_inputs(cfg, seed=21)
        dev = to_dev(inp)
        out = pda.paged_decode_attention(dev["q"], dev["k_cache"], dev["v_cache"], dev["block_tables"],
                                         dev["context_lens"], dev["scale"])
        torch.cuda.synchronize()
        assert max_err(out, oracle_out(oracle_mod, inp)) <= TOL, cfg.name
    # a band step (B * Hq = 128, g = 4, ragged <= 256 tokens): the plan is the paper
    # kernel, and it matches the explicit call bit for bit
    band = synth.Config("auto_band", 8, 16, 4, 128, (256, 17, 200, 1, 64, 0, 255, 129), "bf16", poison_blocks=2)
    inp = synth.make_inputs(band, seed=22)
    dev = to_dev(inp)
    a = pda.paged_decode_attention(dev["q"], dev["k_cache"], dev["v_cache"], dev["block_tables"],
                                   dev["context_lens"], dev["scale"])
    b = gpu(pda, dev, kernel="paper", prefetch="line", prefetch_distance=4, eviction="prefetch_last")
    torch.cuda.synchronize()
    assert pda.plan(pda.make_shape(dev["q"], dev["k_cache"], dev["block_tables"]), pda.make_options())["kernel"] == 1
    assert torch.equal(a, b)
    assert max_err(a, oracle_out(oracle_mod, inp)) <= TOL
    # gather with the default options: split-K underneath, every row vs the oracle
    peers = [torch.zeros_like(dev["q"]) for _ in range(2)]
    pda.paged_decode_attention_gather(dev["q"], dev["k_cache"], dev["v_cache"], dev["block_tables"],
                                      dev["context_lens"], dev["scale"], peers, 0, dev["q"].shape[1])
    torch.cuda.synchronize()
    ref = oracle_out(oracle_mod, inp)
    for pb in peers:
        assert max_err(pb, ref) <= TOL


TC_SHAPES = [c for c in SHAPES if c.head_dim == 128] + [
    synth.Config("tc_long_gqa8", 2, 16, 2, 128, (4500, 129), "bf16", poison_blocks=2),
    synth.Config("tc_ragged", 6, 8, 4, 128, (1, 0, 127, 128, 129, 2049), "fp16", poison_blocks=3),
]


@pytest.mark.parametrize("cfg", TC_SHAPES, ids=lambda c: c.name)
@pytest.mark.parametrize("sms", [0, 7, 1])
def test_tc_kernel_vs_oracle(pda, oracle_mod, cfg, sms):
    """The tcgen05 kernel (kernel="tc", decode_tc.cu): every row vs the fp64
    oracle, with the full grid and with 7 / 1 CTAs (ranges that split rows
    many ways, or none), ragged and zero lengths, NaN-poisoned tails."""
    inp = synth.make_inputs(cfg, seed=31)
    dev = to_dev(inp)
    out = gpu(pda, dev, kernel="tc", num_sms=sms)
    torch.cuda.synchronize()
    assert max_err(out, oracle_out(oracle_mod, inp)) <= TOL


def test_tc_kernel_rescale_paths(pda, oracle_mod):
    """Scores that keep growing along the context (a ramp of +0.2 per token in
    the log2 domain) make every tile raise the reference max by far more
    than the 2^8 slack, so O^T and l are rescaled in TMEM on every tile; a
    late needle does it once.  Both vs the fp64 oracle."""
    for kind in ("ramp", "needle"):
        cfg = synth.Config("tc_rescale", 2, 8, 1, 128, (1500, 700), "bf16")
        inp = synth.make_inputs(cfg, seed=5)
        q, k = inp["q"], inp["k_cache"]
        q[:] = 0
        q[..., 0] = 1.0
        bt = inp["block_tables"]
        for b, L in enumerate(cfg.context_lens):
            for tok in range(L):
                blk, row = bt[b, tok // 16], tok % 16
                if kind == "ramp":
                    val = tok * 0.2 / inp["scale"] / 1.4426950408889634
                else:
                    val = (60.0 if tok == L - 3 else 0.0) / inp["scale"] / 1.4426950408889634
                k[blk, :, row, 0] = val
        dev = to_dev(inp)
        out = gpu(pda, dev, kernel="tc")
        torch.cuda.synchronize()
        assert max_err(out, oracle_out(oracle_mod, inp)) <= TOL, kind


def _score_pattern(inp, kind):
    """Set k[..., 0] (with q = e_0) so that the log2-domain score of token t
    follows `kind`: ramp (+0.2 per token: the running max rises on every
    block, by 3.2 per block), steep (+1 per token: by 16 per block), descend
    (the first block holds the max), step (a plateau 12 units higher from the
    middle on: one late jump), needle (one token 60 above the rest)."""
    q, k = inp["q"], inp["k_cache"]
    q[:] = 0
    q[..., 0] = 1.0
    unit = 1.0 / inp["scale"] / 1.4426950408889634
    bt = inp["block_tables"]
    for b, L in enumerate(inp["cfg"].context_lens):
        for tok in range(L):
            v = {"ramp": 0.2 * tok, "steep": 1.0 * tok, "descend": -0.1 * tok,
                 "step": 12.0 if tok >= L // 2 else 0.0, "needle": 60.0 if tok == L - 3 else 0.0}[kind]
            k[bt[b, tok // 16], :, tok % 16, 0] = v * unit


RESCALE_CFGS = [synth.Config("rs_g8", 2, 8, 1, 128, (1500, 700), "bf16"),
             synth.Config("rs_mha", 2, 4, 4, 128, (900, 333), "fp16")]


@pytest.mark.parametrize("cfg", RESCALE_CFGS, ids=lambda c: c.name)
@pytest.mark.parametrize("kind", ["ramp", "steep", "descend", "step", "needle"])
@pytest.mark.parametrize("kw", [dict(), dict(num_sms=1), dict(partition_tokens=256), dict(kernel="balanced"),
                                dict(kernel="stream")],
                         ids=lambda k: "-".join(f"{a}{b}" for a, b in k.items()) or "default")
def test_softmax_rescale_patterns_vs_oracle(pda, oracle_mod, cfg, kind, kw):
    """Online-softmax rescale paths (S5): score patterns whose running max
    rises on every block, once late, or never after the first block, through
    the split kernel (default plan, one wave), the 4-warp kernel (num_sms=1:
    a multi-wave plan), a fixed partition, the balanced and the stream
    kernels, all vs the fp64 oracle."""
    inp = synth.make_inputs(cfg, seed=11)
    _score_pattern(inp, kind)
    out = gpu(pda, to_dev(inp), **kw)
    assert max_err(out, oracle_out(oracle_mod, inp)) <= TOL


@pytest.mark.parametrize("kind", ["ramp", "steep", "descend", "step", "needle"])
@pytest.mark.parametrize("kw", [dict(), dict(smem_stages=16, partition_tokens=256), dict(smem_stages=12)],
                         ids=lambda k: "-".join(f"{a}{b}" for a, b in k.items()) or "default")
def test_softmax_rescale_patterns_kv8_vs_oracle(pda, oracle_mod, kind, kw):
    """Same patterns through the e4m3 path (one-block and paired-block
    softmax), K scale chosen so the pattern fits e4m3's range."""
    cfg = synth.Config("rs_kv8", 2, 8, 2, 128, (1500, 700), "fp16")
    inp = synth.make_inputs(cfg, seed=12)
    _score_pattern(inp, kind)
    kf = inp["k_cache"].float()
    kmax = float(kf[kf.isfinite()].abs().max())  # poison blocks hold NaN
    inp = kv8(inp, ks=kmax / 400.0)  # code = k / ks <= 400 < 448
    out = gpu_kv8(pda, to_dev(inp), **kw)
    assert max_err(out, oracle_kv8(oracle_mod, inp)) <= TOL


@pytest.mark.parametrize("B,ctx,p_max,cluster", [
    (74, 16384, 4, 0),   # 296 CTAs (2/SM, tile split) in clusters of 4: not all resident -> combine
    (128, 8192, 2, 2),   # 256 CTAs in clusters of 2: resident -> cluster merge
    (32, 32768, 8, 8),   # 256 CTAs in clusters of 8
])
def test_planner_clusters_only_when_resident(pda, B, ctx, p_max, cluster):
    """The auto cluster merge (S8 over DSMEM) asks the device whether every
    (seq, kv head) cluster fits at once (cudaOccupancyMaxActiveClusters): a
    CTA-slot count said one wave for 296 CTAs in clusters of 4 on 148 SMs,
    which ran as two waves (150 vs 104 us with the combine kernel)."""
    from paper_2504_06319_b200 import _lib
    s = _lib.Shape(num_seqs=B, num_q_heads=8, num_kv_heads=1, head_dim=128, block_size=16, num_blocks=100000,
                   max_blocks_per_seq=ctx // 16, dtype=1, out_dtype=1, kv_dtype=1, q_len=1)
    o = _lib.Options(prefetch=0, prefetch_distance=0, partition_tokens=0, smem_stages=0, kernel=2, num_sms=0,
                     stream_warps=0, eviction=0, issue_mode=0, k_scale=0.0, v_scale=0.0, merge=0)
    p = pda.plan(s, o)
    assert (p["p_max"], p["cluster"]) == (p_max, cluster)
    assert (p["workspace_bytes"] > 0) == (cluster == 0)


def test_first_plan_inside_graph_capture(tmp_path):
    """The planner's first cluster-residency query for a configuration may run
    inside a (global-mode) CUDA graph capture: it relaxes the thread's capture
    mode, so the capture stays valid and the replay matches an eager call.
    A fresh process, so the query cache is empty."""
    import subprocess
    import sys
    code = r'''
import sys, torch
sys.path.insert(0, %r)
import paper_2504_06319_b200 as pda, synth
cfg = synth.uniform("cap", 128, 8, 1, 128, 8192, "bf16")
d = synth.make_inputs(cfg, seed=5, device="cuda")
args = (d["q"], d["k_cache"], d["v_cache"], d["block_tables"], d["context_lens"], d["scale"])
out = torch.empty_like(d["q"])
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):  # the first plan of this configuration happens here
    pda.paged_decode_attention(*args, out=out, prefetch="off")
g.replay()
ref = pda.paged_decode_attention(*args, prefetch="off")
torch.cuda.synchronize()
info = pda.plan(pda.make_shape(d["q"], d["k_cache"], d["block_tables"]), pda.make_options(prefetch="off"))
assert info["cluster"] == 2, info
assert torch.equal(out, ref)
print("ok")
''' % (str(__import__("pathlib").Path(__file__).resolve().parents[1]),)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr
