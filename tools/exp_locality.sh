# DRAM locality: shuffled (default) vs contiguous block placement on the one-wave cells and C2/C3
for c in u_128_8_1_128_8192_bf16 u_148_8_1_128_8192_bf16 u_128_32_2_128_8192_bf16 c4_b64_ctx4096 c2 c3; do
  timeout 200 python tools/psweep.py $c '[dict()]' | sed 's/^/{"place": "shuffled"} /'
  PSWEEP_CONTIGUOUS=1 timeout 200 python tools/psweep.py $c '[dict()]' | sed 's/^/{"place": "contiguous"} /'
done
timeout 200 python tools/psweep.py u_74_8_1_128_16384_bf16 '[dict(), dict(merge="combine"), dict(merge="cluster")]'
timeout 200 python tools/psweep.py u_32_8_1_128_32768_bf16 '[dict(), dict(merge="combine"), dict(merge="cluster")]'
