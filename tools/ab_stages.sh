# drain vs partition size (multi-wave ragged) and ring depth on one-wave grids
python tools/psweep.py c4_b256_ctx4096 '[dict(), dict(partition_tokens=2048), dict(partition_tokens=1024)]'
python tools/psweep.py c4_b256_ctx32768 '[dict(), dict(partition_tokens=8192), dict(partition_tokens=4096)]'
python tools/psweep.py c3 '[dict(), dict(partition_tokens=2048), dict(partition_tokens=1024)]'
for c in c4_b16_ctx4096 c4_b4_ctx32768 c4_b16_ctx512 c4_b4_ctx4096 c4_b1_ctx32768 c4_b1_ctx4096 c4_b64_ctx512; do
python tools/psweep.py $c '[dict(), dict(smem_stages=4), dict(smem_stages=12)]'
done
