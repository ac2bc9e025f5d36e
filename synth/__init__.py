"""Seeded synthetic decode-attention workloads (shared by tests, bench, smoke).

This module holds NO arithmetic of the method: it only draws inputs
(q, paged K/V caches, block tables, context lengths) with the shapes and
structure of the paper's Llama-class workloads (Llama2-7B
32:32 MHA, Llama3-8B 32:8 GQA, head_dim 128, 16-token blocks P:105) and of
BASELINE.json's configs.  Both the oracle side and the CUDA side consume
what it returns; neither side's code lives here.

Input recipe:
  * q, k, v ~ U(-1, 1), rounded to the dtype (fp16 / bf16).
  * Physical block placement: a seeded random permutation of the block pool
    (vLLM-style fragmentation), one table per sequence shared by all heads.
  * Poison: unreferenced pool blocks, block-table padding entries and the
    token slots >= L inside each sequence's last block are NaN, so any read
    outside the context shows up as a NaN in the result.
  * Ragged lengths (sweep cells): L_b ~ U[ceil(ctx/2), ctx] with L_0 = ctx.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional, Sequence

import torch

BLOCK_SIZE = 16  # tokens per KV block (Table 2)


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    num_seqs: int
    num_q_heads: int
    num_kv_heads: int
    head_dim: int
    context_lens: tuple  # one length per sequence
    dtype: str = "fp16"  # "fp16" | "bf16"
    block_size: int = BLOCK_SIZE
    poison_blocks: int = 0  # extra unreferenced NaN blocks in the pool
    note: str = ""

    @property
    def group(self) -> int:
        return self.num_q_heads // self.num_kv_heads

    @property
    def max_blocks_per_seq(self) -> int:
        return max(1, max(math.ceil(L / self.block_size) for L in self.context_lens))

    @property
    def used_blocks(self) -> int:
        return sum(math.ceil(L / self.block_size) for L in self.context_lens)

    @property
    def num_blocks(self) -> int:
        # +1: a dedicated NaN block that block-table padding points at
        return self.used_blocks + self.poison_blocks + 1

    def kv_bytes(self) -> int:
        """Algorithmic K+V bytes of one step: sum_b 2 * Hkv * L_b * D * 2 B."""
        return sum(2 * self.num_kv_heads * L * self.head_dim * 2 for L in self.context_lens)

    def other_bytes(self, out_elem_bytes: int = 2) -> int:
        """q + out + block-table entries actually used + lens."""
        B, Hq, D = self.num_seqs, self.num_q_heads, self.head_dim
        bt = sum(math.ceil(L / self.block_size) for L in self.context_lens) * 4
        return B * Hq * D * 2 + B * Hq * D * out_elem_bytes + bt + 4 * B

    def with_heads(self, num_q_heads: int, num_kv_heads: int, name: Optional[str] = None) -> "Config":
        return dataclasses.replace(self, num_q_heads=num_q_heads, num_kv_heads=num_kv_heads,
                                   name=name or self.name)


def uniform(name, B, Hq, Hkv, D, ctx, dtype, **kw) -> Config:
    return Config(name, B, Hq, Hkv, D, tuple([ctx] * B), dtype, **kw)


def ragged(name, B, Hq, Hkv, D, ctx, dtype, seed=0, **kw) -> Config:
    """L_b ~ U[ceil(ctx/2), ctx], L_0 = ctx (DESIGN.md input recipe, sweep cells)."""
    g = torch.Generator().manual_seed(1000 + seed)
    lo = math.ceil(ctx / 2)
    lens = torch.randint(lo, ctx + 1, (B,), generator=g).tolist()
    lens[0] = ctx
    return Config(name, B, Hq, Hkv, D, tuple(lens), dtype, **kw)


# BASELINE.json configs ------------------------------------------------------
C1_TINY = Config("c1_tiny", 2, 4, 2, 64, (37, 256), "fp16", poison_blocks=13,
                 note="BASELINE configs[0]: tiny paged decode, shuffled block table")
C2_LLAMA2_7B = uniform("c2_llama2_7b", 64, 32, 32, 128, 4096, "fp16",
                       note="BASELINE configs[1]: Llama-2-7B shape, B=64, ctx=4096, fp16")
C3_LLAMA3_8B = uniform("c3_llama3_8b", 128, 32, 8, 128, 8192, "bf16",
                       note="BASELINE configs[2]: Llama-3-8B GQA shape, B=128, ctx=8192, bf16")
C5_LLAMA3_70B = uniform("c5_llama3_70b", 256, 64, 8, 128, 16384, "bf16",
                        note="BASELINE configs[4]: Llama-3-70B shape, B=256, ctx=16384 (TP shards KV heads)")

PRESETS = {c.name: c for c in (C1_TINY, C2_LLAMA2_7B, C3_LLAMA3_8B, C5_LLAMA3_70B)}
PRESETS.update({"c1": C1_TINY, "c2": C2_LLAMA2_7B, "c3": C3_LLAMA3_8B, "c5": C5_LLAMA3_70B})


def sweep_cell(batch: int, ctx: int, seed: int = 0, dtype: str = "bf16") -> Config:
    """BASELINE configs[3]: batch x context sweep cell, Llama-3-8B shape, ragged lens."""
    return ragged(f"c4_b{batch}_ctx{ctx}", batch, 32, 8, 128, ctx, dtype, seed=seed)


def torch_dtype(dtype: str):
    return {"fp16": torch.float16, "bf16": torch.bfloat16, "fp32": torch.float32}[dtype]


def make_inputs(cfg: Config, seed: int = 0, device="cpu", poison: bool = True,
                shuffle: bool = True, values: str = "uniform") -> dict:
    """Draw one decode step's inputs for `cfg`.

    Returns dict with q [B,Hq,D], k_cache/v_cache [num_blocks,Hkv,bs,D] (dtype),
    block_tables [B, max_blocks] int32, context_lens [B] int32, scale (1/sqrt(D)),
    all on `device`.  Large caches are drawn directly on the device with a
    seeded device generator.  values: "uniform" U(-1,1) | "normal" N(0,1).
    """
    device = torch.device(device)
    dt = torch_dtype(cfg.dtype)
    B, Hq, Hkv, D, bs = cfg.num_seqs, cfg.num_q_heads, cfg.num_kv_heads, cfg.head_dim, cfg.block_size
    nb, mb = cfg.num_blocks, cfg.max_blocks_per_seq
    gcpu = torch.Generator().manual_seed(seed)
    gdev = torch.Generator(device=device).manual_seed(seed + 1) if device.type == "cuda" else gcpu

    def draw(shape):
        # drawn in fp32 chunks (bounded temporaries for multi-GB caches), rounded to dtype
        out = torch.empty(shape, dtype=dt, device=device)
        flat = out.view(-1)
        chunk = 1 << 28
        for s in range(0, flat.numel(), chunk):
            n = min(chunk, flat.numel() - s)
            if values == "normal":
                x = torch.randn(n, generator=gdev, device=device, dtype=torch.float32)
            else:
                x = torch.rand(n, generator=gdev, device=device, dtype=torch.float32).mul_(2).sub_(1)
            flat[s:s + n] = x
        return out

    q = draw((B, Hq, D))
    k = draw((nb, Hkv, bs, D))
    v = draw((nb, Hkv, bs, D))

    # physical placement: shuffled pool; the last pool block is the padding block
    pool = torch.randperm(nb - 1, generator=gcpu) if shuffle else torch.arange(nb - 1)
    pad_block = nb - 1
    bt = torch.full((B, mb), pad_block, dtype=torch.int32)
    pos = 0
    used = []
    for b, L in enumerate(cfg.context_lens):
        n = math.ceil(L / bs)
        bt[b, :n] = pool[pos:pos + n].to(torch.int32)
        used.append(pool[pos:pos + n])
        pos += n
    lens = torch.tensor(cfg.context_lens, dtype=torch.int32)

    if poison:
        nan = float("nan")
        unused = pool[pos:].tolist() + [pad_block]
        if unused:
            idx = torch.tensor(unused, dtype=torch.long, device=device)
            k.index_fill_(0, idx, nan)
            v.index_fill_(0, idx, nan)
        for b, L in enumerate(cfg.context_lens):
            tail = L % bs
            if tail:
                last = int(bt[b, L // bs])
                k[last, :, tail:, :] = nan
                v[last, :, tail:, :] = nan

    return dict(q=q, k_cache=k, v_cache=v, block_tables=bt.to(device), context_lens=lens.to(device),
                scale=1.0 / math.sqrt(D), cfg=cfg)


def with_query_tokens(inputs: dict, q_len: int, seed: int = 0) -> dict:
    """Multi-token (speculative) decode variant: q becomes [B, q_len, Hq, D]
    (fresh U(-1, 1) draws, same dtype/device); context_lens keep counting the
    new tokens, whose K/V are already in the cache."""
    q = inputs["q"]
    g = torch.Generator(device=q.device).manual_seed(seed + 77) if q.is_cuda else torch.Generator().manual_seed(seed + 77)
    B, Hq, D = q.shape
    x = torch.rand((B, q_len, Hq, D), generator=g, device=q.device, dtype=torch.float32).mul_(2).sub_(1)
    out = dict(inputs)
    out["q"] = x.to(q.dtype)
    out["q_len"] = q_len
    return out


def new_kv_rows(inputs: dict, q_len: int = 1, seed: int = 0):
    """The decode step's new K/V rows to append, k_new/v_new [B, q_len, Hkv, D]
    (U(-1, 1) in the cache dtype, or q's dtype for an e4m3 cache; same device)."""
    cfg, q = inputs["cfg"], inputs["q"]
    dt = q.dtype
    g = torch.Generator(device=q.device).manual_seed(seed + 131) if q.is_cuda else torch.Generator().manual_seed(seed + 131)
    shape = (cfg.num_seqs, q_len, cfg.num_kv_heads, cfg.head_dim)
    k = torch.rand(shape, generator=g, device=q.device, dtype=torch.float32).mul_(2).sub_(1).to(dt)
    v = torch.rand(shape, generator=g, device=q.device, dtype=torch.float32).mul_(2).sub_(1).to(dt)
    return k, v


def quantize_kv_e4m3(inputs: dict, k_scale: float = 1.0 / 224, v_scale: float = 1.0 / 224) -> dict:
    """FP8 KV-cache variant of `inputs`: K and V stored as
    OCP e4m3 codes (uint8) of x / scale with per-tensor scales, NaN poison kept
    as the e4m3 NaN code 0x7F.  The dequantised cache is scale * e4m3(code)."""
    out = dict(inputs)
    for name, sc in (("k_cache", k_scale), ("v_cache", v_scale)):
        x = inputs[name].float()
        nan = torch.isnan(x)
        codes = (x / sc).nan_to_num(0.0).to(torch.float8_e4m3fn).view(torch.uint8)
        codes[nan] = 0x7F
        out[name] = codes
    out.update(k_scale=k_scale, v_scale=v_scale, kv_dtype="e4m3")
    return out


def permute_placement(inputs: dict, seed: int) -> dict:
    """Re-place every physical block at a new random position and rewrite the
    block tables consistently (same logical cache, different placement)."""
    k, v, bt = inputs["k_cache"], inputs["v_cache"], inputs["block_tables"]
    nb = k.shape[0]
    g = torch.Generator().manual_seed(seed)
    perm = torch.randperm(nb, generator=g)  # new position of old block i is perm[i]
    inv = torch.empty_like(perm)
    inv[perm] = torch.arange(nb)
    k2 = k[inv.to(k.device)]
    v2 = v[inv.to(v.device)]
    bt2 = perm.to(torch.int32).to(bt.device)[bt.long()]
    out = dict(inputs)
    out.update(k_cache=k2, v_cache=v2, block_tables=bt2)
    return out


def shard_kv_heads(inputs: dict, rank: int, world: int) -> dict:
    """Tensor-parallel shard: rank r keeps KV heads [r*Hkv/N, (r+1)*Hkv/N) and
    their GQA q heads (heads split per GPU).  Tables/lens replicated."""
    cfg: Config = inputs["cfg"]
    Hq, Hkv = cfg.num_q_heads, cfg.num_kv_heads
    assert Hkv % world == 0, "KV heads must divide the TP degree"
    kh, qh = Hkv // world, Hq // world
    out = dict(inputs)
    out.update(q=inputs["q"][:, rank * qh:(rank + 1) * qh].contiguous(),
               k_cache=inputs["k_cache"][:, rank * kh:(rank + 1) * kh].contiguous(),
               v_cache=inputs["v_cache"][:, rank * kh:(rank + 1) * kh].contiguous(),
               cfg=cfg.with_heads(qh, kh, name=f"{cfg.name}_tp{world}"))
    return out


def sample_rows(inputs: dict, seqs: Sequence[int]) -> dict:
    """Compact sub-problem holding only sequences `seqs` (all heads): their
    blocks are gathered into a fresh pool and the tables renumbered.  Used to
    check full-size runs row by row on the host."""
    cfg: Config = inputs["cfg"]
    bt = inputs["block_tables"].cpu()
    lens = inputs["context_lens"].cpu()
    bs = cfg.block_size
    rows_bt, blocks = [], []
    off = 0
    for b in seqs:
        n = math.ceil(int(lens[b]) / bs)
        blocks.append(bt[b, :n].long())
        rows_bt.append(torch.arange(off, off + n))
        off += n
    ids_all = torch.cat(blocks) if blocks else torch.zeros(0, dtype=torch.long)
    mb = max(1, max((len(x) for x in blocks), default=1))
    new_bt = torch.zeros((len(seqs), mb), dtype=torch.int32)
    for i, r in enumerate(rows_bt):
        new_bt[i, :len(r)] = r.to(torch.int32)
    dev = inputs["k_cache"].device
    k = inputs["k_cache"][ids_all.to(dev)].cpu()
    v = inputs["v_cache"][ids_all.to(dev)].cpu()
    if k.shape[0] == 0:
        k = inputs["k_cache"][:1].cpu()
        v = inputs["v_cache"][:1].cpu()
    return dict(q=inputs["q"][list(seqs)].cpu(), k_cache=k, v_cache=v, block_tables=new_bt,
                context_lens=lens[list(seqs)].clone(), scale=inputs["scale"], cfg=cfg)

