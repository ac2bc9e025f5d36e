"""Tensor parallelism on real GPUs (-m gpu): one process per GPU, NCCL.

The paper runs vLLM tensor parallelism, "each GPU processes 1/N of the
heads": rank r holds KV heads [r*Hkv/N, (r+1)*Hkv/N)
of the Llama-3-70B step (BASELINE configs[4], C5: B=256, 64/8 heads, ctx
16384, bf16), computes them with the CUDA kernel and the step ends with the
output all-gather -- NCCL all_gather_into_tensor (S9) or the fused gather
(NEXT f2: the kernel's stores go straight into every rank's symmetric-memory
buffer).  Every rank's gathered [B, Hq, D] output is checked against the fp64
oracle of the unsharded step on every row (<= 2e-3), the fused and NCCL
gathers must agree bit for bit, and three consecutive fused steps (which
alternate the two symmetric buffers) must all stay correct.

N = 1 runs the same code path (a world-1 NCCL group, symmetric memory over one
device) on a single-GPU box; N = 2, 4, 8 run when that many GPUs are visible
and are skipped otherwise.
"""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOL = 2e-3
SEED = 1234


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, ref_path, result_q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import torch.distributed as dist
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    res = {"rank": rank}
    try:
        import synth
        from paper_2504_06319_b200.tp import TPDecodeAttention
        cfg = synth.C5_LLAMA3_70B
        full = synth.make_inputs(cfg, seed=SEED, device="cuda")  # same seeded draw on every rank
        shard = synth.shard_kv_heads(full, rank, world)
        del full
        torch.cuda.empty_cache()
        lc = shard["cfg"]
        ref = np.load(ref_path)

        def err(out):
            g = out.reshape(cfg.num_seqs, cfg.num_q_heads, cfg.head_dim).double().cpu().numpy()
            return float(np.abs(g - ref).max()) if np.isfinite(g).all() else float("inf")

        args = (shard["q"], shard["block_tables"], shard["context_lens"], shard["scale"])
        nccl = TPDecodeAttention(shard["k_cache"], shard["v_cache"], lc.num_seqs, lc.num_q_heads,
                                 lc.max_blocks_per_seq, torch.bfloat16)
        a = nccl(*args).clone()
        torch.cuda.synchronize()
        res["nccl_err"] = err(a)
        fused = TPDecodeAttention(shard["k_cache"], shard["v_cache"], lc.num_seqs, lc.num_q_heads,
                                  lc.max_blocks_per_seq, torch.bfloat16, fused_gather=True)
        outs = [fused(*args).clone() for _ in range(3)]  # buffers 0, 1, 0
        torch.cuda.synchronize()
        res["fused_err"] = max(err(o) for o in outs)
        res["fused_eq_nccl"] = all(torch.equal(o.view(torch.int16), a.view(torch.int16)) for o in outs)
    except Exception as e:  # noqa: BLE001 -- reported to the parent
        res["error"] = repr(e)
    finally:
        result_q.put(res)
        dist.destroy_process_group()


_REF = {}


def _reference_path(oracle_mod):
    """Oracle of the unsharded C5 step, every row, computed once per session."""
    if "path" not in _REF:
        import synth
        from test_gpu_full_size import oracle_every_row
        inp = synth.make_inputs(synth.C5_LLAMA3_70B, seed=SEED, device="cuda:0")
        ref = oracle_every_row(oracle_mod, inp)
        del inp
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        fd, path = tempfile.mkstemp(suffix=".npy")
        os.close(fd)
        np.save(path, ref)
        _REF["path"] = path
    return _REF["path"]


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_tp_nccl_and_fused_gather_vs_oracle(oracle_mod, world):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs, {torch.cuda.device_count()} visible")
    import torch.multiprocessing as mp
    ref_path = _reference_path(oracle_mod)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, ref_path, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=900) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
    for r in sorted(results, key=lambda x: x["rank"]):
        assert "error" not in r, r
        assert r["nccl_err"] <= TOL, r
        assert r["fused_err"] <= TOL, r
        assert r["fused_eq_nccl"], r
    assert all(p.exitcode == 0 for p in procs)
