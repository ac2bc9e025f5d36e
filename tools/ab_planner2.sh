# planner candidates: cap partitions at 8192/4096 tokens on long multi-wave steps; 4-stage rings (4 CTAs/SM) for short multi-wave units
python tools/psweep.py c5 '[dict(), dict(partition_tokens=8192), dict(partition_tokens=4096)]'
python tools/psweep.py u_256_64_8_128_32768_bf16 '[dict(), dict(partition_tokens=8192), dict(partition_tokens=4096)]'
python tools/psweep.py c4_b128_ctx32768 '[dict(), dict(partition_tokens=8192), dict(partition_tokens=4096)]'
python tools/psweep.py c4_b256_ctx16384 '[dict(), dict(partition_tokens=8192), dict(partition_tokens=4096)]'
python tools/psweep.py c2 '[dict(), dict(partition_tokens=2048)]'
python tools/psweep.py u_256_32_32_128_8192_fp16 '[dict(), dict(partition_tokens=4096)]'
for c in c4_b256_ctx512 c4_b64_ctx512 c4_b128_ctx512 c4_b256_ctx1024 c4_b64_ctx1024 u_256_32_8_128_512_bf16 u_64_32_32_128_512_fp16 u_128_32_32_128_1024_fp16 c4_b32_ctx512 c4_b256_ctx2048; do
python tools/psweep.py $c '[dict(), dict(smem_stages=4)]'
done
