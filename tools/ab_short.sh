# short-context multi-wave grids: unit size vs ring depth
python tools/psweep.py u_128_32_8_128_1024_bf16 '[dict(), dict(partition_tokens=512), dict(partition_tokens=512, smem_stages=8), dict(partition_tokens=256), dict(smem_stages=8)]'
python tools/psweep.py u_128_28_4_128_1024_bf16 '[dict(), dict(partition_tokens=512), dict(partition_tokens=512, smem_stages=8), dict(partition_tokens=256), dict(smem_stages=8)]'
python tools/psweep.py u_32_16_16_128_1024_bf16 '[dict(), dict(partition_tokens=512), dict(partition_tokens=512, smem_stages=8), dict(partition_tokens=256), dict(smem_stages=8)]'
python tools/psweep.py u_512_32_2_128_1024_bf16 '[dict(), dict(partition_tokens=512), dict(partition_tokens=256)]'
python tools/timeline.py u_128_32_8_128_1024_bf16
