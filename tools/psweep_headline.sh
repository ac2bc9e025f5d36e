# the headline configs: planner choice vs finer partitions (smaller drain) and ring variants
timeout 300 python tools/psweep.py c2 '[dict(), dict(partition_tokens=2048), dict(partition_tokens=1024), dict(smem_stages=12), dict(partition_tokens=2048, smem_stages=4)]'
timeout 300 python tools/psweep.py c3 '[dict(), dict(partition_tokens=2048), dict(partition_tokens=8192), dict(smem_stages=12)]'
timeout 300 python tools/psweep.py c5 '[dict(), dict(partition_tokens=8192), dict(partition_tokens=4096)]'
