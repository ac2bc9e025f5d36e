"""Host-only checks of the C ABI (-m "not gpu"): the library loads, exports
every symbol include/pda.h declares, validates arguments synchronously
without a CUDA context, and plans launches deterministically."""
import ctypes
import os
import subprocess

import pytest

import paper_2504_06319_b200 as pda
from paper_2504_06319_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def built():
    from paper_2504_06319_b200 import build
    build.build()


def test_exports_every_header_symbol():
    syms = pda.header_symbols()
    assert {"paged_decode_attention", "paged_decode_attention_trace", "paged_decode_attention_gather",
            "pda_check_args", "pda_plan",
            "pda_workspace_bytes", "pda_decode_step_host", "pda_read_roofline", "pda_status_string",
            "pda_abi_version"} <= set(syms)
    L = pda.lib()
    for s in syms:
        assert hasattr(L, s), f"libpda.so does not export {s}"
    nm = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    for s in syms:
        assert f" T {s}" in nm


def test_sass_targets_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True, text=True).stdout
    for mnemonic in ("UTMALDG", "UBLKPF", "HMMA.16816.F32", "LDSM", "MOVM", "SYNCS",
                     "FENCE.VIEW.ASYNC.G", "F2FP.SATFINITE.E4M3"):
        assert mnemonic in sass, f"{mnemonic} missing from SASS"


def shape(**kw):
    d = dict(num_seqs=2, num_q_heads=4, num_kv_heads=2, head_dim=64, block_size=16, num_blocks=32,
             max_blocks_per_seq=16, dtype=0, out_dtype=0)
    d.update(kw)
    d.setdefault("kv_dtype", d["dtype"])
    d.setdefault("q_len", 1)
    return _lib.Shape(**d)


def opts(**kw):
    d = dict(prefetch=1, prefetch_distance=4, partition_tokens=0, smem_stages=0, kernel=0, num_sms=0,
             stream_warps=0, eviction=0, issue_mode=0, k_scale=0.0, v_scale=0.0, merge=0)
    d.update(kw)
    return _lib.Options(**d)


@pytest.mark.parametrize("kw,status", [
    ({}, 0),
    (dict(head_dim=96), 3),
    (dict(block_size=32), 3),
    (dict(num_q_heads=6, num_kv_heads=4), 2),
    (dict(num_q_heads=34, num_kv_heads=2), 3),
    (dict(dtype=2), 3),
    (dict(out_dtype=1), 3),
    (dict(out_dtype=2), 0),
    (dict(num_seqs=-1), 2),
    (dict(num_blocks=0), 2),
    (dict(kv_dtype=3), 3),                 # e4m3 needs head_dim 128
    (dict(kv_dtype=3, head_dim=128), 0),
    (dict(kv_dtype=1), 3),                 # bf16 cache with an fp16 q
    (dict(q_len=4), 0),                    # 4 tokens x g=2 = 8 columns
    (dict(q_len=9), 3),                    # 18 columns > 16
    (dict(q_len=17), 2),
])
def test_check_args_shape(kw, status):
    assert pda.check_args(shape(**kw), opts()) == status


@pytest.mark.parametrize("kw,status", [
    (dict(prefetch=1, prefetch_distance=0), 2),
    (dict(prefetch=0, prefetch_distance=0), 0),
    (dict(prefetch=3), 0),                               # PDA_PF_AUTO
    (dict(prefetch=4), 2),
    (dict(partition_tokens=24), 2),
    (dict(partition_tokens=32), 0),
    (dict(kernel=2, smem_stages=6), 3),
    (dict(smem_stages=6), 3),
    (dict(smem_stages=12), 0),
    (dict(kernel=4, smem_stages=6), 3),
    (dict(kernel=4, smem_stages=12), 0),
    (dict(kernel=4, prefetch_distance=33), 3),
    (dict(kernel=5), 3),                                 # tc: head_dim 128 only
    (dict(kernel=6), 2),
    (dict(kernel=7), 2),
    (dict(kernel=2, prefetch_distance=400), 3),          # self-issue window: d <= 32
    (dict(kernel=2, prefetch_distance=400, issue_mode=1), 0),
    (dict(kernel=3), 0),
    (dict(kernel=3, smem_stages=6, stream_warps=2), 0),
    (dict(kernel=3, smem_stages=12), 3),
    (dict(kernel=3, prefetch_distance=33), 3),
    (dict(kernel=3, prefetch_distance=32), 0),
    (dict(eviction=5), 2),
    (dict(k_scale=-1.0), 2),
    (dict(issue_mode=3), 2),
    (dict(issue_mode=2), 0),
    (dict(eviction=4), 0),
    (dict(eviction=3), 0),
])
def test_check_args_options(kw, status):
    assert pda.check_args(shape(), opts(**kw)) == status


def test_null_args():
    L = pda.lib()
    assert L.pda_check_args(None, ctypes.byref(opts())) == 1
    assert L.pda_workspace_bytes(None, None) == 0
    rc = L.paged_decode_attention(None, None, None, None, None, 1.0, None, ctypes.byref(shape()),
                                  ctypes.byref(opts()), None, 0, None)
    assert rc == 1


def test_misaligned_pointer_rejected_before_launch():
    L = pda.lib()
    base = 0x10000000
    rc = L.paged_decode_attention(base + 2, base, base, base, base, 1.0, base, ctypes.byref(shape()),
                                  ctypes.byref(opts()), None, 0, None)
    assert rc == 4


def test_workspace_required():
    L = pda.lib()
    s, o = shape(max_blocks_per_seq=64), opts(partition_tokens=256, merge=1)  # combine kernel
    need = pda.workspace_bytes(s, o)
    assert need > 0
    # auto: merge in a cluster of 4 once the grid has a CTA per SM (num_sms=16 here: 16 units)
    assert pda.workspace_bytes(s, opts(partition_tokens=256, num_sms=16)) == 0
    assert pda.workspace_bytes(s, opts(partition_tokens=256)) == need  # 16 CTAs < 148 SMs: combine kernel
    base = 0x10000000
    rc = L.paged_decode_attention(base, base, base, base, base, 1.0, base, ctypes.byref(s),
                                  ctypes.byref(o), None, 0, None)
    assert rc == 5


def test_plan_no_split_llama2():
    # C2: B=64, 32 kv heads, ctx 4096: 2048 units already fill >= 4 waves -> one partition
    s = shape(num_seqs=64, num_q_heads=32, num_kv_heads=32, head_dim=128, num_blocks=16385,
              max_blocks_per_seq=256)
    p = pda.plan(s, opts(kernel=2))
    assert p["p_max"] == 1 and p["partition_tokens"] == 4096 and p["workspace_bytes"] == 0
    assert (p["grid_x"], p["grid_y"], p["grid_z"]) == (1, 32, 64) and p["threads"] == 128  # self-issue
    assert pda.plan(s, opts(kernel=2, issue_mode=1))["threads"] == 160  # + producer warp
    assert p["trace_rec_len"] == 4 + 2 * 256 and p["trace_records"] == 64 * 32


def test_plan_split_llama3_8b():
    # C3: 1024 units < 4 waves of 444 -> split 2 -> P = 4096
    s = shape(num_seqs=128, num_q_heads=32, num_kv_heads=8, head_dim=128, num_blocks=65537,
              max_blocks_per_seq=512, dtype=1, out_dtype=1)
    p = pda.plan(s, opts(kernel=2))
    assert p["p_max"] == 2 and p["partition_tokens"] == 4096
    assert p["cluster"] == 0  # 2048 CTAs > one wave: combine kernel (auto)
    assert pda.plan(s, opts(kernel=2, merge=2))["cluster"] == 2
    pc = pda.plan(s, opts(kernel=2, merge=1))
    B, Hq, P, D = 128, 32, 2, 128
    assert pc["cluster"] == 0 and pc["workspace_bytes"] == B * Hq * P * D * 4 + B * Hq * P * 4


def test_plan_explicit_partition_and_paper():
    s = shape()
    p = pda.plan(s, opts(kernel=2, partition_tokens=48))
    assert p["partition_tokens"] == 48 and p["p_max"] == 6 and p["trace_rec_len"] == 4 + 2 * 3
    pp = pda.plan(s, opts(kernel=1))
    assert pp["kernel"] == 1 and (pp["grid_x"], pp["grid_y"]) == (4, 2) and pp["threads"] == 128
    assert pp["trace_rec_len"] == 4 + 2 * 4 and pp["trace_records"] == 2 * 4 * 4


def test_plan_stream_persistent_grid():
    # D=128, 6 stages x 2 warps x 8 KiB = 96 KiB (+1 KiB align) -> 2 CTAs per SM on 148 SMs
    s = shape(num_seqs=64, num_q_heads=32, num_kv_heads=32, head_dim=128, num_blocks=16385,
              max_blocks_per_seq=256)
    p = pda.plan(s, opts(kernel=3))
    assert p["kernel"] == 3 and p["grid_x"] == 296 and p["threads"] == 64 and p["smem_stages"] == 6
    ns, nh, D = 296 * 2, 8, 128
    assert p["workspace_bytes"] == ns * 2 * nh * D * 4 + ns * 2 * nh * 4 + 64 * 32 * 4
    assert p["trace_rec_len"] == 4 + 2 * 256 and p["trace_records"] == 64 * 32
    p1 = pda.plan(s, opts(kernel=3, smem_stages=8, stream_warps=1))
    assert p1["grid_x"] == 148 * 3 and p1["threads"] == 32


def test_plan_balanced_persistent_wave():
    # D=128, g<=8: ring 8 x 8 KiB + two parked segment slots (2 x 16.75 KiB) ~ 99 KiB -> 2 CTAs/SM
    s = shape(num_seqs=64, num_q_heads=32, num_kv_heads=32, head_dim=128, num_blocks=16385,
              max_blocks_per_seq=256)
    assert pda.plan(s, opts())["kernel"] == 2  # AUTO = split-K
    p = pda.plan(s, opts(kernel=4))
    assert p["kernel"] == 4 and p["grid_x"] == 296 and p["threads"] == 128 and p["smem_stages"] == 8
    G, nh, D = 296, 8, 128

    def a256(x):
        return (x + 255) // 256 * 256
    assert p["workspace_bytes"] == a256(G * 2 * nh * D * 4) + a256(G * 2 * nh * 4) + a256((64 + 1) * 8)
    # g = 16 needs two head tiles: one parked slot of 2 x 8 columns, 1 CTA/SM
    s16 = shape(num_seqs=8, num_q_heads=32, num_kv_heads=2, head_dim=128, num_blocks=600,
                max_blocks_per_seq=64)
    assert pda.plan(s16, opts(kernel=4))["grid_x"] == 148
    assert pda.plan(s, opts(kernel=4, num_sms=5))["grid_x"] == 10


def test_eviction_auto_resolution():
    small = shape(num_seqs=16, num_q_heads=32, num_kv_heads=8, head_dim=128, num_blocks=5000,
                  max_blocks_per_seq=256)   # 16 x 4096 tokens x 8 heads x 512 B = 0.27 GB
    big = shape(num_seqs=64, num_q_heads=32, num_kv_heads=32, head_dim=128, num_blocks=16385,
                max_blocks_per_seq=256)     # 4.3 GB
    assert pda.plan(small, opts(eviction=4))["eviction"] == 1
    assert pda.plan(big, opts(eviction=4))["eviction"] == 0
    assert pda.plan(big, opts(eviction=2))["eviction"] == 2


def test_multi_token_needs_splitk_and_sizes_workspace():
    s = shape(q_len=4, max_blocks_per_seq=64)
    assert pda.check_args(s, opts(kernel=1)) == 3 and pda.check_args(s, opts(kernel=4)) == 3
    p = pda.plan(s, opts(kernel=2, partition_tokens=256, merge=1))
    rows = 2 * 4 * 4  # B * q_len * Hq
    assert p["p_max"] == 4 and p["workspace_bytes"] == rows * 4 * 64 * 4 + ((rows * 4 * 4 + 255) // 256) * 256


def test_e4m3_cache_needs_splitk():
    s = shape(head_dim=128, kv_dtype=3)
    assert pda.check_args(s, opts(kernel=2)) == 0
    for k in (1, 3, 4):
        assert pda.check_args(s, opts(kernel=k)) == 3


def test_status_strings():
    for code in range(7):
        assert pda.status_string(code).startswith("PDA_")
    assert pda.lib().pda_abi_version() == 14


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2504_06319_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "from oracle" not in text, f
                assert "oracle.c" not in text and "liboracle" not in text, f


def test_append_entries_reject_before_launch():
    """pda_kv_append / paged_decode_attention_append / pda_validate_inputs:
    argument errors come back synchronously, before any CUDA call."""
    L = pda.lib()
    base = 0x10000000
    s, o = shape(), opts()
    # NULL new rows / caches
    assert L.pda_kv_append(None, base, base, base, base, base, ctypes.byref(s), ctypes.byref(o), None) == 1
    assert L.pda_kv_append(base, base, base, base, None, base, ctypes.byref(s), ctypes.byref(o), None) == 1
    # misaligned new rows
    assert L.pda_kv_append(base + 4, base, base, base, base, base, ctypes.byref(s), ctypes.byref(o), None) == 4
    # e4m3 cache without scales: the encoding is undefined
    s8 = shape(head_dim=128, kv_dtype=3)
    assert L.pda_kv_append(base, base, base, base, base, base, ctypes.byref(s8), ctypes.byref(o), None) == 2
    # fused entry: same checks, then the attention's own
    rc = L.paged_decode_attention_append(base, None, base, base, base, base, base, 1.0, base, ctypes.byref(s),
                                         ctypes.byref(o), None, 0, None)
    assert rc == 1
    rc = L.paged_decode_attention_append(base, base, base + 8, base, base, base, base, 1.0, base, ctypes.byref(s),
                                         ctypes.byref(o), None, 0, None)
    assert rc == 4
    # validation entry
    assert L.pda_validate_inputs(None, base, ctypes.byref(s), base, None) == 1
    assert L.pda_validate_inputs(base, base, ctypes.byref(shape(block_size=32)), base, None) == 3
    assert L.pda_validate_inputs(base, base, ctypes.byref(shape(num_blocks=0)), base, None) == 2


def test_host_async_entry_rejects_before_launch():
    L = pda.lib()
    base = 0x10000000
    s, o = shape(), opts()
    args = [base] * 10
    rc = L.pda_decode_step_host_async(*args[:8], base, base, 1.0, ctypes.byref(s), ctypes.byref(o), None, 0,
                                      None, None, None, base)
    assert rc == 1  # NULL inputs_ready event


def test_cluster_merge_planning():
    """Auto: clusters for 2 <= P_max <= 8 on one-wave grids with a CTA per SM;
    explicit cluster up to 16; beyond: unsupported."""
    s = shape(max_blocks_per_seq=64)  # 1024 tokens
    assert pda.plan(s, opts(partition_tokens=128, num_sms=32))["cluster"] == 8  # 32 CTAs on 32 SMs
    assert pda.plan(s, opts(partition_tokens=128))["cluster"] == 0  # 32 CTAs < 148 SMs: combine
    p16 = pda.plan(s, opts(partition_tokens=64))
    assert p16["cluster"] == 0 and p16["workspace_bytes"] > 0  # auto: 16 > 8 -> combine kernel
    assert pda.plan(s, opts(partition_tokens=64, merge=2))["cluster"] == 16
    assert pda.check_args(s, opts(merge=3)) == 2
    info = _lib.PlanInfo()
    assert pda.lib().pda_plan(ctypes.byref(s), ctypes.byref(opts(partition_tokens=32, merge=2)),
                              ctypes.byref(info)) == 3  # 32 partitions do not fit a cluster
    assert pda.plan(s, opts(partition_tokens=1024))["cluster"] == 0  # single partition


@pytest.mark.parametrize("B,ctx,P,p_max,cluster", [
    (1, 512, 128, 4, 0),      # tiny grid: down to 128-token partitions, combine kernel (< 1 CTA per SM)
    (4, 512, 128, 4, 0),
    (16, 512, 512, 1, 0),     # 128 units at 512: no split
    (1, 4096, 256, 16, 0),    # 8 rows (small grid): 16 x 256-token partitions, combine kernel
    (16, 4096, 2048, 2, 2),   # 256 units: one well-filled wave of 2048-token partitions
    (64, 4096, 1024, 4, 0),   # 512 rows: four waves of 1024-token partitions, combine kernel
    (16, 32768, 2048, 16, 0),  # long partitions prefer many waves
    (1, 32768, 2048, 16, 0),  # small grid: partitions >= 1024 tokens, <= 128 CTAs, combine kernel
])
def test_planner_partitions_and_merge(B, ctx, P, p_max, cluster):
    _check_planner(B, ctx, P, p_max, cluster, 8)


@pytest.mark.parametrize("B,ctx,P,p_max,cluster", [
    (64, 8192, 4096, 2, 2),    # g = 16 (2 CTAs/SM): one wave of >= one CTA per SM, not 128 CTAs
    (16, 32768, 4096, 8, 8),
])
def test_planner_one_wave_fills_every_sm(B, ctx, P, p_max, cluster):
    _check_planner(B, ctx, P, p_max, cluster, 2)


@pytest.mark.parametrize("B,hkv,ctx,kv8,P,p_max", [
    (1, 1, 8192, False, 512, 16),    # small grid: <= 128 CTAs of >= min(ctx/16, 1024)-token partitions
    (1, 1, 4096, False, 256, 16),
    (2, 1, 32768, False, 1024, 32),
    (4, 8, 2048, False, 512, 4),     # 32 rows > 8: the general rules (>= 512-token partitions)
    (1, 8, 32768, False, 2048, 16),  # 8 rows x 16 = 128 CTAs
    (1, 8, 32768, True, 1024, 32),   # e4m3: up to 256 CTAs
])
def test_planner_small_grids(B, hkv, ctx, kv8, P, p_max):
    """<= 8 (seq, kv head) rows: the measured small-grid split (DESIGN.md 6,
    profiles/r02_small_grid_sweep.jsonl); such grids merge with the combine kernel."""
    s = shape(num_seqs=B, num_q_heads=8 * hkv, num_kv_heads=hkv, head_dim=128, num_blocks=100000,
              max_blocks_per_seq=ctx // 16, dtype=1, out_dtype=1, kv_dtype=3 if kv8 else 1)
    p = pda.plan(s, opts(kernel=2))
    assert (p["partition_tokens"], p["p_max"]) == (P, p_max)
    assert p["cluster"] == 0  # fewer CTAs than SMs: combine kernel


def _check_planner(B, ctx, P, p_max, cluster, hkv):
    s = shape(num_seqs=B, num_q_heads=32, num_kv_heads=hkv, head_dim=128, num_blocks=100000,
              max_blocks_per_seq=ctx // 16, dtype=1, out_dtype=1)
    p = pda.plan(s, opts(kernel=2))
    assert (p["partition_tokens"], p["p_max"], p["cluster"]) == (P, p_max, cluster)


@pytest.mark.parametrize("B, ctx, stages", [
    (64, 512, 4),     # 512 units: past one wave at 3 CTAs/SM (444), one wave at 4 (592)
    (128, 512, 4),    # 1024 units: within two waves at 4 CTAs/SM
    (64, 1024, 4),
    (32, 512, 8),     # 256 units: one wave either way, keep the deeper ring
    (256, 512, 8),    # 2048 units: many waves, deeper ring wins
    (256, 1024, 8),
    (64, 4096, 8),    # split to 2048 units of 1024 tokens
])
def test_planner_ring_depth(B, ctx, stages):
    s = shape(num_seqs=B, num_q_heads=32, num_kv_heads=8, head_dim=128, num_blocks=100000,
              max_blocks_per_seq=ctx // 16, dtype=1, out_dtype=1)
    assert pda.plan(s, opts(kernel=2))["smem_stages"] == stages
    assert pda.plan(s, opts(kernel=2, smem_stages=12))["smem_stages"] == 12  # explicit depth wins
    kv8 = shape(num_seqs=B, num_q_heads=32, num_kv_heads=8, head_dim=128, num_blocks=100000,
                max_blocks_per_seq=ctx // 16, dtype=1, out_dtype=1, kv_dtype=3)
    # e4m3: 12 single-block stages at 4 CTAs/SM up to 1 GiB of e4m3 KV, else 16 in pairs
    assert pda.plan(kv8, opts(kernel=2))["smem_stages"] == (12 if 2 * B * ctx * 8 * 128 <= 1 << 30 else 16)
    big8 = shape(num_seqs=64, num_q_heads=32, num_kv_heads=32, head_dim=128, num_blocks=16385,
                 max_blocks_per_seq=256, kv_dtype=3)  # C2 in e4m3: 2.1 GB
    assert pda.plan(big8, opts(kernel=2))["smem_stages"] == 16


def _build_c_example(tmp_path):
    """examples/decode_step.c compiled and linked as plain C11 against the
    header and libpda.so (the boundary needs no C++ and no PyTorch)."""
    exe = tmp_path / "decode_step"
    cmd = ["gcc", "-std=c11", "-pedantic", "-Wall", "-Wextra", "-Werror", f"-I{ROOT}/include",
           "-I/usr/local/cuda/include", f"{ROOT}/examples/decode_step.c", f"-L{os.path.dirname(_lib.LIB_PATH)}",
           "-lpda", "-L/usr/local/cuda/lib64", "-lcudart", "-lm",
           f"-Wl,-rpath,{os.path.dirname(_lib.LIB_PATH)}", "-o", str(exe)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_header_is_c99_and_c_example_links(tmp_path):
    src = tmp_path / "h.c"
    src.write_text('#include "pda.h"\nint main(void) { return pda_abi_version() > 0 ? 0 : 1; }\n')
    r = subprocess.run(["gcc", "-std=c99", "-pedantic", "-Wall", "-Wextra", "-Werror", f"-I{ROOT}/include",
                        "-fsyntax-only", str(src)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert _build_c_example(tmp_path).exists()


def test_default_split_k_kernels_do_not_spill():
    """The occupancy each split-K instantiation is built for (its
    __launch_bounds__ minimum CTAs/SM, which the planner assumes) must not
    cost spills in the self-issue kernels the library runs by default
    (ptxas -v report of the plain-MODE translation unit)."""
    import re
    rep = os.path.join(os.path.dirname(_lib.LIB_PATH), "_build", "decode_splitk_m0.o.ptxas.txt")
    text = open(rep).read()
    blocks = re.findall(r"Function properties for (\S+)\n\s+(\d+) bytes stack frame, (\d+) bytes spill stores", text)
    # template tail ...E<KV8>E<SELF>E<TS>: SELF = 1, tile split TS = 0 or 1
    tail = re.compile(r"ELb1ELb[01]EEEv14CUtensorMap_stS2_NS_12SplitKParamsE$")
    self_issue = [(n, int(sp)) for n, _, sp in blocks if "splitk_kernel" in n and tail.search(n)]
    assert len(self_issue) >= 20, "expected every self-issue instantiation in the ptxas report"
    # accepted: the two-tile e4m3 kernel at 3 CTAs/SM spills a few words (measured
    # 11-12 % faster than its spill-free 2-CTA/SM build, splitk_impl.cuh)
    kv8_two_tile = re.compile(r"ELi128ELi2ELi\d+ELi0ELb1ELb1E")
    spilled = [n for n, sp in self_issue if sp and not (kv8_two_tile.search(n) and sp <= 64)]
    assert not spilled, spilled


from hypothesis import given, settings, strategies as st  # noqa: E402


@settings(max_examples=300, deadline=None)
@given(B=st.integers(1, 1024), g=st.sampled_from([1, 2, 4, 5, 7, 8, 16]), hkv=st.sampled_from([1, 2, 4, 8, 32]),
       D=st.sampled_from([64, 128]), max_blocks=st.integers(1, 4096), q_len=st.integers(1, 4),
       kv8=st.booleans(), dt=st.sampled_from([0, 1]))
def test_planner_invariants(B, g, hkv, D, max_blocks, q_len, kv8, dt):
    """Any valid shape: the split-K plan covers every token exactly once with
    whole blocks, its grid matches (P_max, Hkv, B), the ring depth is one the
    kernels instantiate, clusters only merge what fits, the workspace is the
    documented partial size, and the planner is deterministic."""
    if kv8 and D != 128:
        return
    if q_len * g > 16:
        q_len = max(1, 16 // g)
    s = shape(num_seqs=B, num_q_heads=g * hkv, num_kv_heads=hkv, head_dim=D, num_blocks=max_blocks + 1,
              max_blocks_per_seq=max_blocks, dtype=dt, out_dtype=dt, kv_dtype=3 if kv8 else dt, q_len=q_len)
    p = pda.plan(s, opts(kernel=2, prefetch=0))
    assert p == pda.plan(s, opts(kernel=2, prefetch=0))
    max_tokens = max_blocks * 16
    P, pm = p["partition_tokens"], p["p_max"]
    assert P % 16 == 0 and P > 0
    assert pm == -(-max_tokens // P) and (pm - 1) * P < max_tokens <= pm * P
    assert (p["grid_x"], p["grid_y"], p["grid_z"]) == (pm, hkv, B)
    assert p["smem_stages"] in ((8, 12, 16, 24) if kv8 else (4, 8, 12))
    if p["cluster"]:
        assert p["cluster"] == pm and 1 < pm <= 8 and p["workspace_bytes"] == 0
    if pm > 1 and not p["cluster"]:
        rows = B * q_len * g * hkv
        al = lambda x: (x + 255) // 256 * 256
        assert p["workspace_bytes"] == al(rows * pm * D * 4) + al(rows * pm * 4)
    if pm == 1:
        assert p["workspace_bytes"] == 0
    assert p["trace_records"] == B * hkv * pm and p["trace_rec_len"] == 4 + 2 * (P // 16)


def test_prefetch_auto_policy():
    """PDA_PF_AUTO (include/pda.h): with kernel AUTO a short-context step
    (16-bit, one query token, <= 512 tokens) with GQA groups >= 4 and
    128 <= B * Hq <= 512 (<= 256 above 256 tokens) plans the paper-structure
    kernel (its prefetch evict_last under eviction AUTO) and reports split-K's
    workspace, which the same call needs with a fused append / gather; every
    other step plans split-K exactly as with prefetch off."""
    def sh(B, hq, hkv, ctx, **kw):
        return shape(num_seqs=B, num_q_heads=hq, num_kv_heads=hkv, head_dim=128, max_blocks_per_seq=ctx // 16,
                     num_blocks=B * ctx // 16, **kw)
    band = sh(8, 32, 8, 256)  # B * Hq = 256, g = 4, ctx 256
    p = pda.plan(band, opts(prefetch=3, eviction=4))
    ref = pda.plan(band, opts(prefetch=0, eviction=4, kernel=2))
    assert p["kernel"] == 1 and p["eviction"] == 2
    assert p["workspace_bytes"] == ref["workspace_bytes"]
    # explicit prefetch or an explicit kernel: no policy
    assert pda.plan(band, opts(prefetch=2, eviction=4))["kernel"] == 2
    assert pda.plan(band, opts(prefetch=3, kernel=2))["kernel"] == 2
    # the band's edges
    assert pda.plan(sh(4, 32, 8, 256), opts(prefetch=3))["kernel"] == 1      # 128 rows
    assert pda.plan(sh(16, 32, 8, 256), opts(prefetch=3))["kernel"] == 1     # 512 rows
    assert pda.plan(sh(8, 32, 8, 512), opts(prefetch=3))["kernel"] == 1      # 256 rows at ctx 512
    for off in (sh(2, 32, 8, 256), sh(32, 32, 8, 256), sh(16, 32, 8, 512), sh(8, 32, 8, 528),
                sh(8, 32, 32, 256), sh(8, 32, 16, 256), sh(8, 32, 8, 256, q_len=2),
                sh(8, 32, 8, 256, kv_dtype=3)):
        assert pda.plan(off, opts(prefetch=3)) == pda.plan(off, opts(prefetch=0))


def test_tc_and_tile_split_plans():
    """kernel=tc: one persistent CTA per SM (grid = num_sms), 320 threads, the
    balanced-style workspace; unsupported shapes are refused before launch.
    Tile split: two-tile 16-bit steps whose grid is one wave at 2 CTAs/SM run
    256-thread CTAs with an 8-stage ring; multi-wave, e4m3 or 4-stage grids
    keep the 4-warp two-tile kernel."""
    s = shape(num_q_heads=16, num_kv_heads=2, head_dim=128)
    p = pda.plan(s, opts(kernel=5, prefetch=0))
    assert (p["kernel"], p["grid_x"], p["grid_y"], p["grid_z"], p["threads"]) == (5, 148, 1, 1, 320)
    assert pda.plan(s, opts(kernel=5, prefetch=0, num_sms=7))["grid_x"] == 7
    assert p["workspace_bytes"] >= 148 * 2 * 8 * 128 * 4
    for bad in (dict(head_dim=64), dict(q_len=2, head_dim=128), dict(kv_dtype=3, head_dim=128)):
        assert pda.check_args(shape(**bad), opts(kernel=5, prefetch=0)) == 3
    assert pda.check_args(shape(head_dim=128), opts(kernel=5, prefetch=0, smem_stages=8)) == 3
    # g = 16: B=2 x 2 kv heads -> a one-wave grid at 2 CTAs/SM -> tile split
    g16 = shape(num_q_heads=32, num_kv_heads=2, head_dim=128)
    p = pda.plan(g16, opts(prefetch=0))
    assert p["threads"] == 256 and p["smem_stages"] == 8
    assert pda.plan(g16, opts(prefetch=0, smem_stages=4))["threads"] == 128
    assert pda.plan(g16, opts(prefetch=0, issue_mode=1))["threads"] == 160   # producer-warp form
    # many rows: more than one wave -> the two-tile kernel
    big = shape(num_seqs=512, num_q_heads=32, num_kv_heads=2, head_dim=128, num_blocks=8192)
    assert pda.plan(big, opts(prefetch=0))["threads"] == 128
