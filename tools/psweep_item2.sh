# split-K configurations on the batch >= 64, ctx >= 4k cells below 6.4 TB/s, plus the tc kernel
python tools/psweep.py u_128_8_1_128_8192_bf16 '[dict(), dict(partition_tokens=2736), dict(partition_tokens=2048), dict(partition_tokens=2048, smem_stages=8), dict(partition_tokens=1024), dict(partition_tokens=4096, smem_stages=12), dict(partition_tokens=4096, merge="combine"), dict(partition_tokens=1536), dict(partition_tokens=1360), dict(kernel="tc"), dict(kernel="balanced")]'
python tools/psweep.py c4_b64_ctx4096 '[dict(), dict(partition_tokens=512), dict(partition_tokens=768), dict(partition_tokens=1360), dict(partition_tokens=2048), dict(smem_stages=4), dict(smem_stages=12), dict(kernel="tc")]'
python tools/psweep.py u_128_32_2_128_8192_bf16 '[dict(), dict(partition_tokens=4096), dict(partition_tokens=2736), dict(partition_tokens=2048), dict(partition_tokens=4096, smem_stages=12), dict(kernel="tc")]'
python tools/psweep.py u_64_32_8_128_4096_bf16 '[dict(), dict(partition_tokens=2048), dict(partition_tokens=1024), dict(kernel="tc")]'
python tools/psweep.py u_256_32_8_128_4096_bf16 '[dict(), dict(partition_tokens=2048), dict(kernel="tc")]'
