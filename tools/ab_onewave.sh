# one-wave grids: power-of-two split (default) vs the largest split that still fits one wave
python tools/psweep.py u_1_32_32_128_32768_bf16 '[dict(), dict(partition_tokens=2528), dict(partition_tokens=2736), dict(partition_tokens=2048)]'
python tools/psweep.py u_32_28_4_128_8192_bf16 '[dict(), dict(partition_tokens=2736), dict(partition_tokens=2048)]'
python tools/psweep.py u_8_16_16_128_8192_bf16 '[dict(), dict(partition_tokens=2736), dict(partition_tokens=2048)]'
python tools/psweep.py c4_b16_ctx4096 '[dict(), dict(partition_tokens=1376), dict(partition_tokens=1024)]'
python tools/psweep.py c4_b4_ctx32768 '[dict(), dict(partition_tokens=2528), dict(partition_tokens=2048)]'
python tools/psweep.py u_8_32_32_128_8192_bf16 '[dict(), dict(partition_tokens=4096)]'
