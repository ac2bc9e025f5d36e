"""Tensor-parallel host logic on CPU (gloo, world size 2): KV-head sharding,
the output all-gather and the head order of the gathered view.

Each rank's local attention is computed here by the oracle (test-only; the
product's per-rank compute is the CUDA kernel), so the check isolates the
sharding + gather logic of paper_2504_06319_b200.tp: the gathered output
must equal the unsharded oracle output bit for bit (rows are independent).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def worker(rank, world, port, cfg_name, result_q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import synth
        from paper_2504_06319_b200.tp import gather_heads, shard_range
        cfg = {"gqa": synth.Config("tp_gqa", 3, 8, 4, 64, (37, 5, 100), "fp16", poison_blocks=2),
               "mha": synth.Config("tp_mha", 2, 4, 4, 128, (16, 33), "bf16")}[cfg_name]
        full = synth.make_inputs(cfg, seed=7)
        shard = synth.shard_kv_heads(full, rank, world)
        lo, hi = shard_range(cfg.num_q_heads, rank, world)
        assert torch.equal(shard["q"], full["q"][:, lo:hi])
        local = oracle.paged_attention(shard["q"], shard["k_cache"], shard["v_cache"],
                                       shard["block_tables"], shard["context_lens"], shard["scale"],
                                       cfg.dtype)
        gathered = gather_heads(torch.from_numpy(local))
        got = gathered.reshape(cfg.num_seqs, cfg.num_q_heads, cfg.head_dim).numpy()
        ref = oracle.paged_attention(full["q"], full["k_cache"], full["v_cache"], full["block_tables"],
                                     full["context_lens"], full["scale"], cfg.dtype)
        result_q.put((rank, bool(np.array_equal(got, ref))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg_name", ["gqa", "mha"])
def test_tp_shard_gather_equals_unsharded(cfg_name):
    import oracle
    oracle.build()
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, cfg_name, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    assert all(p.exitcode == 0 for p in procs)
    res = dict(q.get(timeout=10) for _ in range(world))
    assert res == {0: True, 1: True}


def test_shard_range_validation():
    from paper_2504_06319_b200.tp import shard_range
    assert shard_range(32, 3, 8) == (12, 16)
    with pytest.raises(ValueError):
        shard_range(6, 0, 4)
