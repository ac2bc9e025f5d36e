"""Tensor-parallel decode attention: KV heads sharded across ranks (one
process per GPU), NCCL all-gather of the per-rank output heads.

The paper runs vLLM tensor parallelism, where "each GPU processes 1/N of the
heads".  A GQA group is never split: rank r owns KV heads
[r*Hkv/N, (r+1)*Hkv/N) and the q heads that read them,
[r*Hq/N, (r+1)*Hq/N); block tables and context lengths are replicated.  The
only exchange is the output all-gather: each rank's
[B, Hq/N, D] slice goes out with one all_gather_into_tensor on the compute
stream; the gathered [N, B, Hq/N, D] buffer is returned as a [B, N, Hq/N, D]
view whose flattening is [B, Hq, D] -- no extra copy on the step.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import _lib


def shard_range(num_heads: int, rank: int, world: int):
    if num_heads % world:
        raise ValueError(f"{num_heads} heads do not divide over {world} ranks")
    n = num_heads // world
    return rank * n, (rank + 1) * n


def gather_heads(out_local: torch.Tensor, group=None, gathered: torch.Tensor | None = None):
    """All-gather [B, Hq/N, D] slices -> [B, N, Hq/N, D] view (head order = rank order)."""
    world = dist.get_world_size(group)
    B, hl, D = out_local.shape
    if gathered is None:
        gathered = torch.empty((world * B, hl, D), dtype=out_local.dtype, device=out_local.device)
    if out_local.is_cuda and dist.get_backend(group) == "gloo":
        # testing path (several ranks sharing one GPU): gloo gathers host tensors
        host = torch.empty(gathered.shape, dtype=gathered.dtype)
        dist.all_gather_into_tensor(host, out_local.cpu(), group=group)
        gathered.copy_(host)
    else:
        dist.all_gather_into_tensor(gathered, out_local.contiguous(), group=group)
    return gathered.view(world, B, hl, D).permute(1, 0, 2, 3)


class TPDecodeAttention:
    """One rank's share of a tensor-parallel decode attention step.

    k_cache / v_cache hold only this rank's KV heads ([num_blocks, Hkv/N, 16, D]);
    q_local holds this rank's q heads.  __call__ runs the CUDA decode kernels
    on the local shard and all-gathers the heads -- with NCCL
    (all_gather_into_tensor, default), or, with fused_gather=True, inside the
    kernel's own stores into every rank's symmetric-memory output buffer
    followed by one symmetric-memory barrier.

    The returned [B, N, Hq/N, D] view aliases an internal buffer: with the NCCL
    gather it is valid until the next call, with the fused gather (two
    alternating buffers) until the call after next; reads must be enqueued on
    the calling stream (or finished) before then.
    """

    def __init__(self, k_cache, v_cache, num_seqs, num_q_heads_local, max_blocks, dtype, group=None,
                 fused_gather=False, **opts):
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.fused = fused_gather
        D = k_cache.shape[-1]
        dev = k_cache.device
        self.k, self.v = k_cache, v_cache
        self.opts = opts
        self.out_local = torch.empty((num_seqs, num_q_heads_local, D), dtype=dtype, device=dev)
        self.gathered = torch.empty((self.world * num_seqs, num_q_heads_local, D), dtype=dtype,
                                    device=dev)
        shape = _lib.make_shape(self.out_local, k_cache,
                                torch.empty((num_seqs, max_blocks), dtype=torch.int32, device="meta"))
        opt = _lib.make_options(**{k: v for k, v in opts.items() if k in _lib.OPTION_KEYS})
        self.plan = _lib.plan(shape, opt)
        wsb = self.plan["workspace_bytes"]
        self.ws = torch.zeros(max(1, wsb), dtype=torch.uint8, device=dev)  # stream tickets start at 0
        # the per-step call with shape / options / plan prepared once (host cost ~5 us, not ~18)
        self.prepared = _lib.PreparedDecode(self.out_local, k_cache,
                                            torch.empty((num_seqs, max_blocks), dtype=torch.int32, device="meta"),
                                            **{k: v for k, v in opts.items() if k in _lib.OPTION_KEYS})
        self.hq_local = num_q_heads_local
        if self.fused:
            # Two symmetric output buffers, alternated step by step: this rank's
            # kernel stores into its PEERS' buffers, so reusing one buffer would
            # let a fast rank's step k+1 overwrite step k's output while a slower
            # peer still reads it (write-after-read).  With step k in set k % 2,
            # the barrier that ends step k+1 orders every rank's stream-ordered
            # reads of step k before any rank's step k+2 stores (include/pda.h).
            import torch.distributed._symmetric_memory as symm_mem
            hq = num_q_heads_local * self.world
            grp = group if group is not None else dist.group.WORLD
            self.out_full = [symm_mem.empty((num_seqs, hq, D), dtype=dtype, device=dev) for _ in range(2)]
            self.symm = [symm_mem.rendezvous(buf, grp) for buf in self.out_full]
            self.peer_ptrs = [list(h.buffer_ptrs) for h in self.symm]
            self.step_index = 0

    def launches_per_step(self) -> int:
        # split-K launches its combine kernel when sequences are split and the
        # partitions do not merge inside a cluster; the balanced kernel always
        # launches its combine grid
        pl = self.plan
        if pl["kernel"] == 4:
            return 2
        return 1 + (1 if pl["kernel"] == 2 and pl["p_max"] > 1 and not pl["cluster"] else 0)

    def __call__(self, q_local, block_tables, context_lens, scale):
        if self.fused:
            k = self.step_index & 1
            self.step_index += 1
            _lib.paged_decode_attention_gather(q_local, self.k, self.v, block_tables, context_lens, scale,
                                               self.peer_ptrs[k], self.rank * self.hq_local,
                                               self.hq_local * self.world, workspace=self.ws, **self.opts)
            self.symm[k].barrier(channel=0)  # every rank's stores have landed everywhere
            out = self.out_full[k]
            return out.view(out.shape[0], 1, *out.shape[1:])
        self.prepared(q_local, self.k, self.v, block_tables, context_lens, scale, out=self.out_local)
        if self.world == 1:
            return self.out_local.unsqueeze(1)
        return gather_heads(self.out_local, self.group, self.gathered)
